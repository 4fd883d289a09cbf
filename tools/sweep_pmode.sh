#!/bin/bash
# t = 1 PCG product modes (pcg.cu): 3 = separate B^T product pass (default), 1 = product fused into the backward solve
out=gpurun_out/r2k_pmode.jsonl
: > $out
for pm in ${SWEEP:-3 1}; do
  VL_PMODE1=$pm python tools/pcgbench.py --ts 1 --iters 120 --label "pmode$pm" >> $out 2>>gpurun_out/r2k_pmode.err
done
cat $out
