# Round profiling recipe (run under gpurun, one GPU); ROUND=r02 by default.
#   1. the default bench line (no profiler)
#   2. the ncu launch list of the same command (duration + DRAM bytes per launch)
#   3. one ncu --set full capture of each streaming kernel on the full config-4
#      launch (the first H and B launches of a warm-up step); the .ncu-rep
#      stays on the box, its raw page and summaries come back
set -e
R=${ROUND:-r02}
mkdir -p gpurun_out
python bench.py > gpurun_out/${R}_bench_default.json 2> gpurun_out/${R}_bench_default.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/${R}_launches_default.csv python bench.py > gpurun_out/${R}_bench_under_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/${R}_launches_default.csv --json gpurun_out/${R}_launches_default_summary.json \
    > gpurun_out/${R}_launches_default_summary.txt
ncu --set full --import-source on --clock-control none -k regex:'stream_kernel|pair_kernel' -c 2 -o /tmp/stream_full -f \
    python bench.py --no-e2e --no-cpu --steps 1 --warmup 1 > gpurun_out/${R}_ncu_full.log 2>&1
ncu -i /tmp/stream_full.ncu-rep --page raw --csv > /tmp/stream_full_raw.csv
python tools/full_capture_summary.py /tmp/stream_full_raw.csv gpurun_out/${R}_ncu_full_stream_c4.csv gpurun_out/traffic_c4.json
