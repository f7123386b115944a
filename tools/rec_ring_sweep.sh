# recover_ring_kernel ring depth sweep (rebuilds shen_recover.o in place)
for d in 4 8 10 12; do
  touch paper_1701_03787_b200/csrc/shen_recover.cu
  make -s -C paper_1701_03787_b200/csrc EXTRA="-DSHEN_REC_RING=$d" > /dev/null 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:recover --log-file gpurun_out/rec_$d.csv \
      python bench.py --config step --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
  echo "RING=$d $(grep gpu__time gpurun_out/rec_$d.csv | tail -1 | awk -F'","' '{print $NF}')"
done
touch paper_1701_03787_b200/csrc/shen_recover.cu
make -s -C paper_1701_03787_b200/csrc > /dev/null 2>&1
