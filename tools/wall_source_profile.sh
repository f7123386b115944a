# Source-level stall profile of the wall-normal kernels (one launch each, C3 sizes)
set -e
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:'wall_forward' -s 6 -c 1 -o /tmp/wf -f \
    python bench.py --config c3 --steps 1 --warmup 3 > gpurun_out/wf_ncu.log 2>&1
ncu -i /tmp/wf.ncu-rep --page source --csv --print-source sass > gpurun_out/wf_source_sass.csv 2>&1 || true
ncu --set full --import-source on --clock-control none -k regex:'wall_inverse' -s 6 -c 1 -o /tmp/wi -f \
    python bench.py --config c3 --steps 1 --warmup 3 > gpurun_out/wi_ncu.log 2>&1
ncu -i /tmp/wi.ncu-rep --page source --csv --print-source sass > gpurun_out/wi_source_sass.csv 2>&1 || true
ls -la gpurun_out/*source*
