cd $GRAFT_REPO_ROOT
timeout 300 python tools/dbg_lz.py 30000 > gpurun_out/r2d_dbg_lz.log 2>&1; echo dbg rc=$?; tail -25 gpurun_out/r2d_dbg_lz.log
for L in libvlgpx.so libvlgpx_v2.so libvlgpx_v3.so; do
  VLGPX_LIB=$PWD/paper_2310_12000_b200/$L timeout 400 python tools/pcgbench.py --ts 1 --iters 120 --label $L >> gpurun_out/r2d_pcgbench.jsonl 2>> gpurun_out/r2d_pcgbench.err; echo pcg $L rc=$?
done
cat gpurun_out/r2d_pcgbench.jsonl
timeout 600 python bench.py --steps 5 --warmup 3 --no-c4 --no-cpu-baseline > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err; echo bench rc=$?; head -c 600 gpurun_out/r2d_bench.json
