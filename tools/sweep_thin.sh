timeout 300 python -m pytest tests/test_gpu_factor.py tests/test_gpu_laplace.py -q -x 2>&1 | tail -2
for tp in 0 1 2 4 8; do
  echo "== thin_passes=$tp"; VL_THIN_PASSES=$tp timeout 200 python tools/kbench.py --n 1000000 --ts 1,50 --orders 1 --reps 5 2>&1 | grep '"t"'
done
VL_THIN_PASSES=2 KP_TS=1 timeout 300 python tools/trsv_diag.py 2>&1 | grep -E "total|hop|L0"
