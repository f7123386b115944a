# Helmholtz mirror-pair kernel: parity (bitwise vs one-system kernel), then
# CTA size x ring depth x L2 policy at BASELINE config 4 (bench lines + one
# ncu DRAM-bytes capture per variant into gpurun_out/hp/).
mkdir -p gpurun_out/hp
timeout 900 python -m pytest tests/test_solvers_gpu.py -q -x -k "mirror_pairs" 2>&1 | tail -2
for v in ${VARIANTS:-"8 3 0" "8 3 2" "6 3 0" "6 3 2" "4 4 0" "4 4 1" "4 4 2" "4 3 2"}; do
  set -- $v
  tag=w$1_r$2_h$3
  export SHEN_HELM_PAIRS=1 SHEN_HELM_PAIR_WARPS=$1 SHEN_HELM_PAIR_RING=$2 SHEN_HELM_HINT=$3
  timeout 300 python bench.py --no-e2e --no-cpu --steps 3 > gpurun_out/hp/$tag.json 2> gpurun_out/hp/$tag.err
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:helm_pair -s 1 -c 1 --csv python bench.py --no-e2e --no-cpu --steps 1 --warmup 1 \
    > gpurun_out/hp/$tag.ncu.csv 2>&1
  python - "$tag" <<'PY'
import json, sys
t = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/hp/{t}.json"))
    h = d["per_operator"]["helmholtz"]
    print(t, "H ms", round(h["ms"], 3), "med", round(h["ms_median"], 3), "frac", round(h["frac"], 3), "clk", d["clocks"]["sm_mhz"])
except Exception as e:
    print(t, "bench failed", e)
PY
  grep -E "dram__bytes|lts__t_sector_hit|gpu__time" gpurun_out/hp/$tag.ncu.csv | awk -F'","' '{print "   ", $(NF-2), $NF}'
done
