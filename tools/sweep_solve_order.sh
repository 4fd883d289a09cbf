#!/bin/bash
# A/B sweeps behind DESIGN 7.6 (tools/pcgbench.py at n = 1e6; one JSON line per run into gpurun_out/).
#   tiles    VL_TILE_K x VL_TILE_S against the level order        SWEEP="32_4 64_6 ..."
#   late     VL_CHILD_LATE window                                 SWEEP="0 3 16 1000"
#   heavy    VL_HEAVY_LEVEL_ROWS x VL_HEAVY_DEPS (t = 1)          SWEEP="512_64 ..."
#   knobs    VL_SPIN_MAX_NS / VL_SPIN_MAX_NS1 / VL_HEAD_MAX / VL_TRSV_BPS
#   pmode    t = 1 PCG product mode 3 (separate product) against 1 (fused into the backward solve)
#   variants library variants paper_2310_12000_b200/libvlgpx_<v>.so   VARIANTS="default vA ..."
what=${1:-tiles}
out=gpurun_out/sweep_$what.jsonl
: > $out
run() { label=$1; ts=$2; it=$3; shift 3; env "$@" python tools/pcgbench.py --ts $ts --iters $it --label $label >> $out 2>>gpurun_out/sweep_$what.err; }
case $what in
  tiles)
    run level 50 20 VL_USE_TILES=0
    for ks in ${SWEEP:-32_4 32_8 32_16 64_6 64_8}; do run K${ks%_*}_S${ks#*_} 50 20 VL_TILE_K=${ks%_*} VL_TILE_S=${ks#*_}; done ;;
  late)
    for d in ${SWEEP:-0 1 3 8 16 1000}; do run late$d 1,50 120,20 VL_CHILD_LATE=$d; done ;;
  heavy)
    for hv in ${SWEEP:-64_64 256_64 512_64 1024_64 512_48 512_96}; do run heavy$hv 1 120 VL_HEAVY_LEVEL_ROWS=${hv%_*} VL_HEAVY_DEPS=${hv#*_}; done ;;
  knobs)
    run base 1,50 120,20 X=1
    for v in 16 32 64 128 256; do run spin1_$v 1 120 VL_SPIN_MAX_NS1=$v; done
    for v in 0 32 128; do run spinT_$v 50 20 VL_SPIN_MAX_NS=$v; done
    for v in 2048 4096 6144; do run head$v 1,50 120,20 VL_HEAD_MAX=$v; done
    for v in 2 3; do run bps$v 50 20 VL_TRSV_BPS=$v; done ;;
  pmode)
    for pm in 3 1; do run pmode$pm 1 120 VL_PMODE1=$pm; done ;;
  variants)
    for v in ${VARIANTS:-default}; do
      lib=""; [ $v != default ] && lib=$PWD/paper_2310_12000_b200/libvlgpx_$v.so
      run $v ${TS:-1,50} ${ITERS:-120,20} VLGPX_LIB=$lib
    done ;;
esac
cat $out
