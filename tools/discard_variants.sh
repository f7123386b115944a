# y-checkpoint L2 discard on/off (rebuilds shen_solve_stream.o in place)
python -m pytest tests/test_solvers_gpu.py -q -x -k "stream" 2>&1 | tail -1
for v in 1 0 1 0; do
  touch paper_1701_03787_b200/csrc/shen_solve_stream.cu
  make -s -C paper_1701_03787_b200/csrc EXTRA="-DSHEN_YCKPT_DISCARD=$v" > /dev/null 2>&1
  echo "DISCARD=$v $(python bench.py --no-e2e --no-cpu --steps 5 | python -c 'import json,sys; d=json.load(sys.stdin); print({k:round(v["ms"],2) for k,v in d["per_operator"].items()}, d["clocks"]["sm_mhz"], d["clocks"]["reasons"])')"
done
touch paper_1701_03787_b200/csrc/shen_solve_stream.cu
make -s -C paper_1701_03787_b200/csrc > /dev/null 2>&1
