timeout 300 python -m pytest tests/test_gpu_factor.py tests/test_gpu_laplace.py -q -x 2>&1 | tail -2
for hv in "64 40" "256 40" "1024 24" "0 1000"; do set -- $hv
  echo "== heavy_rows=$1 heavy_deps=$2"; VL_HEAVY_LEVEL_ROWS=$1 VL_HEAVY_DEPS=$2 timeout 200 python tools/kbench.py --n 1000000 --ts 1 --orders 1 --reps 10 2>&1 | grep '"t"'
done
for tr in 0 1; do KP_TR=$tr KP_TS=1 timeout 300 python tools/trsv_diag.py 2>&1 | grep -E "total|hop|L0"; done
