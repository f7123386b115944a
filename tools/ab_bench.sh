# Alternate the product library and variants (SHEN_LIB_VARIANT) in one GPU
# session, so power-state drift hits every arm alike; prints per-run H and B ms.
#   bash tools/ab_bench.sh "tagA tagB" [rounds]
variants="base $1"; rounds=${2:-3}
mkdir -p gpurun_out/ab
for r in $(seq $rounds); do
  for v in $variants; do
    if [ "$v" = base ]; then unset SHEN_LIB_VARIANT; else export SHEN_LIB_VARIANT=$v; fi
    timeout 300 python bench.py --no-e2e --no-cpu --steps 5 > gpurun_out/ab/$v.$r.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab/$v.$r.json')); p=d['per_operator']
print('$v', $r, 'H', round(p['helmholtz']['ms_median'],3), 'B', round(p['biharmonic']['ms_median'],3), 'clk', d['clocks']['sm_mhz'])"
  done
done
