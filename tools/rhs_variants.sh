# rhs_u per-parity kernel: prefetch distance / register budget variants (rebuilds shen_rhs.o in place)
for v in "0 3" "1 3" "2 2" "3 2"; do
  set -- $v
  touch paper_1701_03787_b200/csrc/shen_rhs.cu
  make -s -C paper_1701_03787_b200/csrc EXTRA="-DSHEN_RHS_UPAR_PF=$1 -DSHEN_RHS_UPAR_MINB=$2" > /dev/null 2>&1
  echo "PF=$1 MINB=$2 $(python tools/bench_rhs.py 256 | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["rhs_u"]["ms"],2), round(d["rhs_u"]["GBps_alg"]))')"
done
