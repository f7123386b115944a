# CTA-size sweep of the streaming solves (bench lines into gpurun_out/):
# warps_per_sm 8 / 12 / default per operator
mkdir -p gpurun_out
python -m pytest tests/test_solvers_gpu.py -q -x 2>&1 | tail -1
for w in 8 12 0; do
  SHEN_STREAM_WARPS=$w python bench.py --no-e2e --no-cpu --steps 3 > gpurun_out/sw_$w.json 2>&1
done
