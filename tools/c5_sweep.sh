# BASELINE config 5: wall-normal size sweep at 512 x 257 wavenumbers (bench lines)
mkdir -p gpurun_out
for N in 129 257 513 1025 2049; do
  python bench.py --config c5:$N --no-e2e --no-cpu --steps 10 > gpurun_out/c5_$N.json 2> gpurun_out/c5_$N.err
done
