# TMA-fed biharmonic pair kernel: L2 promotion of the tensor map (0 none ..
# 3 256 B) vs the cp.async-fed pair kernel (SHEN_PAIR_TMA=0); bench + DRAM bytes
mkdir -p gpurun_out/tma
for v in "1 0" "1 1" "1 2" "0 0"; do
  set -- $v
  export SHEN_PAIR_TMA=$1 SHEN_TMA_PROMO=$2
  tag=tma$1_p$2
  timeout 300 python bench.py --no-e2e --no-cpu --steps 5 > gpurun_out/tma/$tag.json 2> gpurun_out/tma/$tag.err
  python -c "
import json; d=json.load(open('gpurun_out/tma/$tag.json')); p=d['per_operator']
print('$tag', 'B', round(p['biharmonic']['ms'],3), round(p['biharmonic']['ms_median'],3), 'clk', d['clocks']['sm_mhz'])"
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:'bih_pair' -s 1 -c 1 --csv python bench.py --no-e2e --no-cpu --steps 1 --warmup 1 \
    > gpurun_out/tma/$tag.ncu.csv 2>&1
  grep -E "dram__bytes|gpu__time" gpurun_out/tma/$tag.ncu.csv | awk -F'","' '{print "   ", $(NF-2), $NF}'
done
