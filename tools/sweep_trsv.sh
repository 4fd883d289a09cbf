for bps in 1 2 4; do for sm in 0 32 128; do
  echo "=== bps=$bps spin=$sm"; VL_TRSV_BPS=$bps VL_SPIN_MAX_NS=$sm timeout 200 python tools/kbench.py --n 1000000 --ts 1,50 --orders 1 --reps 5 2>&1 | grep '"t"'
done; done
