#!/bin/bash
# t = 50 PCG iteration: gather batch size / CTAs per SM variants x tile settings
out=gpurun_out/r2k_tiles2.jsonl
: > $out
for v in ${VARIANTS:-default vA vB vC}; do
  lib=""; [ $v != default ] && lib=$PWD/paper_2310_12000_b200/libvlgpx_$v.so
  for ks in ${SWEEP:-0_0 32_4 32_8 32_16}; do
    K=${ks%_*}; S=${ks#*_}
    if [ $K = 0 ]; then tiles=0; else tiles=1; fi
    VLGPX_LIB=$lib VL_USE_TILES=$tiles VL_TILE_K=$K VL_TILE_S=$S python tools/pcgbench.py --ts 50 --iters 20 --label "${v}_K${K}_S${S}" >> $out 2>>gpurun_out/r2k_tiles2.err
  done
done
cat $out
