cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_predict.py -x -q > gpurun_out/r2e_pytest_predict.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/r2e_pytest_predict.log
for L in ts ts4; do
  VLGPX_LIB=$PWD/paper_2310_12000_b200/libvlgpx_$L.so timeout 600 python tools/trsv_diag2.py > gpurun_out/r2e_trsv_diag2_$L.log 2>&1; echo diag $L rc=$?
done
for L in libvlgpx.so libvlgpx_v4.so libvlgpx_v5.so libvlgpx_v6.so libvlgpx.so; do
  VLGPX_LIB=$PWD/paper_2310_12000_b200/$L timeout 400 python tools/pcgbench.py --ts 1 --iters 120 --label $L >> gpurun_out/r2e_pcgbench.jsonl 2>> gpurun_out/r2e_pcgbench.err; echo pcg $L rc=$?
done
cat gpurun_out/r2e_pcgbench.jsonl
