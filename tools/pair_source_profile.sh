# Source-level stall profile of the biharmonic pair kernel (one launch, config 4, the 512 folded kx rows of a 4-way split)
set -e
mkdir -p gpurun_out
python bench.py --no-e2e --no-cpu --steps 1 --warmup 1 --kx-fold 4 > gpurun_out/pair_plain.json 2> gpurun_out/pair_plain.err
ncu --set full --import-source on --clock-control none -k regex:'pair_kernel' -c 1 -o /tmp/pk -f \
    python bench.py --no-e2e --no-cpu --steps 1 --warmup 1 --kx-fold 4 > gpurun_out/pk_ncu.log 2>&1
ncu -i /tmp/pk.ncu-rep --page source --csv --print-source sass > gpurun_out/pk_source_sass.csv 2>&1 || true
ncu -i /tmp/pk.ncu-rep --page details --csv > gpurun_out/pk_details.csv 2>&1 || true
ls -la gpurun_out/pk_*
