# rhs_u: register-window kernel (variant 2) vs cp.async-ring kernel (variant 3, ring depth D)
python -m pytest tests/test_rhs_gpu.py -q -x 2>&1 | tail -1
echo "V2 $(SHEN_RHS_VARIANT=2 python tools/bench_rhs.py 256 | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["rhs_u"]["ms"],2), round(d["rhs_u"]["GBps_alg"]))')"
for D in 2 4 6; do
  touch paper_1701_03787_b200/csrc/shen_rhs.cu
  make -s -C paper_1701_03787_b200/csrc EXTRA="-DSHEN_RHS_RING=$D" > /dev/null 2>&1
  echo "V3 D=$D $(SHEN_RHS_VARIANT=3 python tools/bench_rhs.py 256 | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["rhs_u"]["ms"],2), round(d["rhs_u"]["GBps_alg"]))')"
done
SHEN_RHS_VARIANT=3 python -m pytest tests/test_rhs_gpu.py tests/test_stepper_gpu.py -q -x 2>&1 | tail -1
