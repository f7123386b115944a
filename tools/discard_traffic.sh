# DRAM bytes of the streaming kernels with the y-checkpoint discard on/off
mkdir -p gpurun_out
for v in 1 0; do
  touch paper_1701_03787_b200/csrc/shen_solve_stream.cu
  make -s -C paper_1701_03787_b200/csrc EXTRA="-DSHEN_YCKPT_DISCARD=$v" > /dev/null 2>&1
  python bench.py --no-e2e --no-cpu --steps 1 --warmup 1 > /dev/null 2>&1 || exit 1
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      -k regex:stream_kernel -c 6 --log-file gpurun_out/discard_$v.csv \
      python bench.py --no-e2e --no-cpu --steps 1 --warmup 1 > /dev/null 2>&1
done
touch paper_1701_03787_b200/csrc/shen_solve_stream.cu
make -s -C paper_1701_03787_b200/csrc > /dev/null 2>&1
