for bps in 1 2 4 8; do for sm in 0 200; do
  echo "== bps=$bps smax=$sm"; VL_TRSV_BPS=$bps VL_SPIN_MAX_NS=$sm timeout 200 python tools/kbench.py --n 1000000 --ts 1,50 --orders 1 --reps 5 2>&1 | grep '"t"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['t'], 'Binv', d['Binv']['ms'], 'Btinv', d['Btinv']['ms'])"
done; done
