#!/bin/bash
# backward solve with late children listed last (pattern.cpp, VL_CHILD_LATE)
out=gpurun_out/r2k_child.jsonl
: > $out
for d in ${SWEEP:-0 1 3 8 1000}; do
  VL_CHILD_LATE=$d python tools/pcgbench.py --ts 1,50 --iters 120,20 --label "late$d" >> $out 2>>gpurun_out/r2k_child.err
done
cat $out
