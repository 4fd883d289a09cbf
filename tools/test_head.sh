timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
echo "== with small head (VL_HEAD_MAX=150) for the parity suite"
VL_HEAD_MAX=150 timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for h in 0 1; do echo "== use_head=$h"; VL_USE_HEAD=$h timeout 200 python tools/kbench.py --n 1000000 --ts 1,50 --orders 1 --reps 5 2>&1 | grep '"t"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['t'], 'Binv', d['Binv']['ms'], 'Btinv', d['Btinv']['ms'])"; done
for hm in 512 1024 2048 4096; do echo "== head_max=$hm"; VL_HEAD_MAX=$hm timeout 200 python tools/kbench.py --n 1000000 --ts 1,50 --orders 1 --reps 5 2>&1 | grep -E '"t"|factor' | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['t'], 'Binv', d['Binv']['ms'], 'Btinv', d['Btinv']['ms'])
    else: print(l.strip())"; done
