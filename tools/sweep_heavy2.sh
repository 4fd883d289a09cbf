#!/bin/bash
# single-RHS solves: levels up to VL_HEAVY_LEVEL_ROWS rows / rows with more than VL_HEAVY_DEPS dependencies as warp-per-row items
out=gpurun_out/r2k_heavy.jsonl
: > $out
for hv in ${SWEEP:-64_64 128_64 256_64 512_64 1024_64 64_32 64_128 256_32}; do
  VL_HEAVY_LEVEL_ROWS=${hv%_*} VL_HEAVY_DEPS=${hv#*_} python tools/pcgbench.py --ts 1 --iters 120 --label "heavy$hv" >> $out 2>>gpurun_out/r2k_heavy.err
done
cat $out
