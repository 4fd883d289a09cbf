# tile-order ncu: DRAM traffic / L2 hit of the t = 50 solves, level order vs tile order (pcgbench, 3 iterations)
cd $GRAFT_REPO_ROOT
: > gpurun_out/r2k_ncu_tiles_summary.txt
for cfg in "0 32 4" "1 32 4" "1 32 8"; do
  set -- $cfg
  echo "## VL_USE_TILES=$1 VL_TILE_K=$2 VL_TILE_S=$3" >> gpurun_out/r2k_ncu_tiles_summary.txt
  VL_USE_TILES=$1 VL_TILE_K=$2 VL_TILE_S=$3 ncu --set full --clock-control none --kernel-name-base demangled \
    -k regex:"trsv_kernel<\\(int\\)32" -s 4 -c 2 -f -o /tmp/pk python tools/pcgbench.py --ts 50 --iters 4 > gpurun_out/r2k_ncu.log 2>&1; echo rc=$?
  python tools/ncu_summary.py /tmp/pk.ncu-rep >> gpurun_out/r2k_ncu_tiles_summary.txt 2>&1
  ncu -i /tmp/pk.ncu-rep --page raw --csv | gzip > gpurun_out/r2k_ncu_tiles_$1_$2_$3_raw.csv.gz
done
cat gpurun_out/r2k_ncu_tiles_summary.txt | cut -c1-250
