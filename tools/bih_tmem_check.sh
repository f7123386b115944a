# biharmonic pair kernel with TMEM-parked y checkpoints: parity + bench + DRAM bytes
mkdir -p gpurun_out/bt
timeout 900 python -m pytest tests/test_solvers_gpu.py -q -x -k "biharmonic" 2>&1 | tail -2
timeout 300 python bench.py --no-e2e --no-cpu --steps 5 > gpurun_out/bt/bench.json 2> gpurun_out/bt/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bt/bench.json')); p=d['per_operator']
print('value', d['value'], 'H', p['helmholtz']['ms'], 'B', p['biharmonic']['ms'], p['biharmonic']['ms_median'], 'clk', d['clocks'])"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  --clock-control none -k regex:bih_pair -s 1 -c 1 --csv python bench.py --no-e2e --no-cpu --steps 1 --warmup 1 \
  > gpurun_out/bt/ncu.csv 2>&1
grep -E "dram__bytes|lts__t_sector_hit|gpu__time" gpurun_out/bt/ncu.csv | awk -F'","' '{print "   ", $(NF-2), $NF}'
