# C3 transform evidence (run under gpurun, one GPU):
#   1. the c3 bench line (no profiler)
#   2. the ncu launch list of the same command (every transform-stage launch)
#   3. one ncu --set full capture of the four wall-normal launches of a step
#      (raw metrics + source page exported, the .ncu-rep itself not kept)
set -e
mkdir -p gpurun_out
python bench.py --config c3 > gpurun_out/c3_bench.json 2> gpurun_out/c3_bench.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/c3_launches.csv python bench.py --config c3 --steps 1 --warmup 3 > gpurun_out/c3_under_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/c3_launches.csv --json gpurun_out/c3_launches_summary.json > gpurun_out/c3_launches_summary.txt
ncu --set full --import-source on --clock-control none -k regex:'wall_' -s 12 -c 4 -o /tmp/c3_wall_full -f \
    python bench.py --config c3 --steps 1 --warmup 3 > gpurun_out/c3_ncu_full.log 2>&1
ncu -i /tmp/c3_wall_full.ncu-rep --page raw --csv > gpurun_out/c3_wall_full_raw.csv
ncu -i /tmp/c3_wall_full.ncu-rep --page details --csv > gpurun_out/c3_wall_full_details.csv
# 4. one ncu --set full capture of each plane FFT kernel at the c3 size (257 planes)
for k in rfft2 irfft2; do
  ncu --set full --import-source on --clock-control none --kernel-name-base function -k regex:"^${k}_256_kernel" \
      -s 3 -c 1 -o /tmp/c3_plane_$k -f python tools/plane_fft_check.py > gpurun_out/c3_plane_$k.log 2>&1
  ncu -i /tmp/c3_plane_$k.ncu-rep --page details --csv > gpurun_out/c3_plane_${k}_details.csv
  ncu -i /tmp/c3_plane_$k.ncu-rep --page raw --csv > gpurun_out/c3_plane_${k}_raw.csv
done
