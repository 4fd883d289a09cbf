#!/bin/bash
# t = 50 VADU PCG iteration time under the tile-blocked solve order (pattern.cpp):
# level order (VL_USE_TILES=0) against tile_K x tile_S settings.
out=gpurun_out/r2k_tiles.jsonl
: > $out
VL_USE_TILES=0 python tools/pcgbench.py --ts 50 --iters 20 --label level >> $out 2>gpurun_out/r2k_tiles.err
for ks in ${SWEEP:-32_8 16_8 64_8 32_4 32_16 32_32 100_8}; do
  set -- ${ks%_*} ${ks#*_}
  VL_TILE_K=$1 VL_TILE_S=$2 python tools/pcgbench.py --ts 50 --iters 20 --label "K$1_S$2" >> $out 2>>gpurun_out/r2k_tiles.err
done
cat $out
