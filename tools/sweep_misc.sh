#!/bin/bash
# one-off A/B runs of the solve-order options (pcgbench, n = 1e6)
out=gpurun_out/r2k_misc.jsonl
: > $out
run() { label=$1; shift; env "$@" python tools/pcgbench.py --ts ${TS:-1,50} --iters 120,20 --label $label >> $out 2>>gpurun_out/r2k_misc.err; }
run default X=1
run tail0 VL_TILE_TAIL=0
run gather_ca VLGPX_LIB=$PWD/paper_2310_12000_b200/libvlgpx_vCA.so
run slab_sort VL_SLAB_SORT=1
cat $out
