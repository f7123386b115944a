# sweep CTA size / ring depth of the streaming solves (bench lines into gpurun_out/)
mkdir -p gpurun_out
python -m pytest tests/test_solvers_gpu.py -q -x 2>&1 | tail -1
SHEN_STREAM_WARPS=8 python bench.py --no-e2e --no-cpu --steps 3 > gpurun_out/sw_8r3.json 2>&1
SHEN_BIH_RING2=1 SHEN_STREAM_WARPS=8 python bench.py --no-e2e --no-cpu --steps 3 > gpurun_out/sw_8r2.json 2>&1
SHEN_STREAM_WARPS=12 python bench.py --no-e2e --no-cpu --steps 3 > gpurun_out/sw_12.json 2>&1
