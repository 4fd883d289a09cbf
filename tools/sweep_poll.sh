# poll-one vs poll-all and spin cap sweep for the single-column solves
for lib in libvlgpx.so libvlgpx_p0.so; do for sm in 0 32 64 128 256; do
  echo "== lib=$lib smax=$sm"; VLGPX_LIB=paper_2310_12000_b200/$lib VL_SPIN_MAX_NS=$sm timeout 200 python tools/kbench.py --n 1000000 --ts 1 --orders 1 --reps 10 2>&1 | grep '"t"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['t'], 'Binv', d['Binv']['ms'], 'Btinv', d['Btinv']['ms'])"
done; done
