# e2e (numpy API, page-locked buffers) vs number of pipeline slabs
mkdir -p gpurun_out
for k in 8 16 32; do
SHEN_PIPE_SLABS=$k python bench.py --no-cpu --steps 1 --warmup 3 --kx-rows 64 > gpurun_out/e2e_$k.json 2>&1
done
