# pair kernel: evict-first policy on the streamed RHS rows on/off, time + DRAM bytes
mkdir -p gpurun_out
for v in 1 0 1 0; do
  touch paper_1701_03787_b200/csrc/shen_solve_stream.cu
  make -s -C paper_1701_03787_b200/csrc EXTRA="-DSHEN_PAIR_EF=$v" > /dev/null 2>&1
  echo "EF=$v $(python bench.py --no-e2e --no-cpu --steps 5 | python -c 'import json,sys; d=json.load(sys.stdin); print({k:(round(v["ms"],2),round(v["ms_best"],2)) for k,v in d["per_operator"].items()}, d["clocks"]["sm_mhz"])')"
done
for v in 1 0; do
  touch paper_1701_03787_b200/csrc/shen_solve_stream.cu
  make -s -C paper_1701_03787_b200/csrc EXTRA="-DSHEN_PAIR_EF=$v" > /dev/null 2>&1
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      -k regex:bih_pair -c 1 --log-file gpurun_out/pair_ef_$v.csv python bench.py --no-e2e --no-cpu --steps 1 --warmup 1 > /dev/null 2>&1
  echo "EF=$v $(grep -E 'dram__bytes|gpu__time' gpurun_out/pair_ef_$v.csv | awk -F'","' '{print $(NF-2), $NF}' | tr '\n' ' ')"
done
touch paper_1701_03787_b200/csrc/shen_solve_stream.cu
make -s -C paper_1701_03787_b200/csrc > /dev/null 2>&1
