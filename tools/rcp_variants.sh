# fast reciprocal (cubic vs two Newton steps) x biharmonic quotient refinement:
# residual statistics + timing per variant (rebuilds the whole library: build
# and solve must share the arithmetic)
set -e
python -m pytest tests/test_solvers_gpu.py tests/test_reference_cases_gpu.py -q -x 2>&1 | tail -1
for v in "1 1" "0 0" "1 0" "1 1" "0 0"; do
  set -- $v
  make -s -C paper_1701_03787_b200/csrc clean > /dev/null 2>&1 || true
  make -s -j16 -C paper_1701_03787_b200/csrc EXTRA="-DSHEN_RCP_CUBIC=$1 -DSHEN_BIH_QDIV=$2" > /dev/null 2>&1
  echo "CUBIC=$1 QDIV=$2 $(python bench.py --no-e2e --no-cpu --steps 5 | python -c 'import json,sys; d=json.load(sys.stdin); print({k:round(v["ms"],2) for k,v in d["per_operator"].items()}, d["clocks"]["sm_mhz"], d["clocks"]["reasons"])')"
  python tools/residual_stats.py 32 2>&1 | tail -2
done
make -s -C paper_1701_03787_b200/csrc clean > /dev/null 2>&1 || true
make -s -j16 -C paper_1701_03787_b200/csrc > /dev/null 2>&1
