# biharmonic ring depth 2 vs 3 (rebuilds shen_solve_stream.o in place)
for v in 3 2 3 2; do
  touch paper_1701_03787_b200/csrc/shen_solve_stream.cu
  make -s -C paper_1701_03787_b200/csrc EXTRA="-DSHEN_BIH_RING=$v" > /dev/null 2>&1
  echo "RING=$v $(python bench.py --no-e2e --no-cpu --steps 5 | python -c 'import json,sys; d=json.load(sys.stdin); print({k:(round(v["ms"],2),round(v["ms_best"],2)) for k,v in d["per_operator"].items()}, d["clocks"]["sm_mhz"])')"
done
touch paper_1701_03787_b200/csrc/shen_solve_stream.cu
make -s -C paper_1701_03787_b200/csrc > /dev/null 2>&1
