#!/bin/bash
# A/B of library variants (paper_2310_12000_b200/libvlgpx_<v>.so) on the t = 1 PCG iteration
out=gpurun_out/r2k_variants.jsonl
: > $out
for v in ${VARIANTS:-default}; do
  lib=""; [ $v != default ] && lib=$PWD/paper_2310_12000_b200/libvlgpx_$v.so
  VLGPX_LIB=$lib python tools/pcgbench.py --ts ${TS:-1} --iters ${ITERS:-120} --label $v >> $out 2>>gpurun_out/r2k_variants.err
done
cat $out
