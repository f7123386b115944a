# rhs kernels: unroll / register-budget variants (rebuilds shen_rhs.o in place)
python -m pytest tests/test_rhs_gpu.py -q -x 2>&1 | tail -1
for v in "1 3" "2 3" "2 2" "4 2"; do
  set -- $v
  touch paper_1701_03787_b200/csrc/shen_rhs.cu
  make -s -C paper_1701_03787_b200/csrc EXTRA="-DSHEN_RHS_UNROLL=$1 -DSHEN_RHS_U_MINB=$2" > /dev/null 2>&1
  echo "UNROLL=$1 MINB=$2 $(python tools/bench_rhs.py 256 | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["rhs_u"]["ms"],2), round(d["rhs_u"]["GBps_alg"]), round(d["rhs_g"]["ms"],2), round(d["rhs_g"]["GBps_alg"]))')"
done
