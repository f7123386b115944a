# full GPU test suite, one default bench line, and the DRAM bytes of both
# streaming kernels on a config-4 launch (ncu, one launch each)
mkdir -p gpurun_out/qc
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python bench.py --no-e2e --no-cpu --steps 5 > gpurun_out/qc/bench.json 2> gpurun_out/qc/bench.err
python -c "
import json; d=json.load(open('gpurun_out/qc/bench.json')); p=d['per_operator']
print('value', d['value'], 'H', p['helmholtz']['ms'], p['helmholtz']['ms_median'], 'B', p['biharmonic']['ms'], p['biharmonic']['ms_median'], 'clk', d['clocks'])"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  --clock-control none -k regex:'helm_stream|bih_pair' -s 2 -c 2 --csv python bench.py --no-e2e --no-cpu --steps 1 --warmup 1 \
  > gpurun_out/qc/ncu.csv 2>&1
grep -E "dram__bytes|lts__t_sector_hit|gpu__time" gpurun_out/qc/ncu.csv | awk -F'","' '{print "   ", substr($5,1,30), $(NF-2), $NF}'
