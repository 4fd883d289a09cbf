#!/bin/bash
# runtime knobs re-swept after the solve-order change (pcgbench, n = 1e6)
out=gpurun_out/r2k_knobs.jsonl
: > $out
run() { label=$1; shift; env "$@" python tools/pcgbench.py --ts 1,50 --iters 120,20 --label $label >> $out 2>>gpurun_out/r2k_knobs.err; }
run base X=1
for v in 0 16 32 128 256; do run spin$v VL_SPIN_MAX_NS=$v; done
for v in 2048 4096 6144; do run head$v VL_HEAD_MAX=$v; done
for v in 2 3; do run bps$v VL_TRSV_BPS=$v; done
cat $out
