# Lanczos tests, per-row solve timeline (TS build), PCG A/B of library variants
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_predict.py -x -q > gpurun_out/r2c_pytest_predict.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/r2c_pytest_predict.log
VLGPX_LIB=$PWD/paper_2310_12000_b200/libvlgpx_ts.so timeout 600 python tools/trsv_diag2.py > gpurun_out/r2c_trsv_diag2.log 2>&1; echo diag rc=$?
for L in libvlgpx.so libvlgpx_v1.so libvlgpx.so libvlgpx_v1.so; do
  VLGPX_LIB=$PWD/paper_2310_12000_b200/$L timeout 400 python tools/pcgbench.py --label $L >> gpurun_out/r2c_pcgbench.jsonl 2>> gpurun_out/r2c_pcgbench.err; echo pcg $L rc=$?
done
