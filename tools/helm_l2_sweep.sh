# Helmholtz stream solve: CTA size x ring depth x L2 policy of the two RHS
# reads (SHEN_HELM_HINT: 0 none, 1 fwd evict_last + bwd evict_first,
# 2 bwd evict_first, 3 fwd evict_last).  Bench lines + one ncu DRAM-bytes
# capture per variant into gpurun_out/hl2/.
mkdir -p gpurun_out/hl2
for v in ${VARIANTS:-"12 3 0" "12 3 1" "12 3 2" "8 4 0" "8 4 1" "6 4 0" "6 4 1" "6 6 1" "4 6 0" "4 6 1" "4 6 2"}; do
  set -- $v
  tag=w$1_r$2_h$3
  SHEN_STREAM_WARPS=$1 SHEN_HELM_RING=$2 SHEN_HELM_HINT=$3 timeout 300 python bench.py --no-e2e --no-cpu --steps 3 \
    > gpurun_out/hl2/$tag.json 2> gpurun_out/hl2/$tag.err
  SHEN_STREAM_WARPS=$1 SHEN_HELM_RING=$2 SHEN_HELM_HINT=$3 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:helm_stream -s 1 -c 1 --csv python bench.py --no-e2e --no-cpu --steps 1 --warmup 1 \
    > gpurun_out/hl2/$tag.ncu.csv 2>&1
  python - "$tag" <<'PY'
import json, sys
t = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/hl2/{t}.json"))
    h = d["per_operator"]["helmholtz"]
    print(t, "H ms", round(h["ms"], 3), "med", round(h["ms_median"], 3), "frac", round(h["frac"], 3), "clk", d["clocks"]["sm_mhz"])
except Exception as e:
    print(t, "bench failed", e)
PY
  grep -E "dram__bytes|lts__t_sector_hit|gpu__time" gpurun_out/hl2/$tag.ncu.csv | awk -F'","' '{print "   ", $(NF-2), $NF}'
done
