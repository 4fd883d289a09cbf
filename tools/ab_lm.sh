# A/B of lane-parallel metadata in the multi-column solves (VL_LANEMETA build define)
cd $GRAFT_REPO_ROOT
for L in libvlgpx.so libvlgpx_nolm.so; do
  VLGPX_LIB=$PWD/paper_2310_12000_b200/$L timeout 300 python tools/c5_sweep.py --ns 1000000 --ms 20 --ts 16,64 --kinds knn,random --reps 10 --check 1 > gpurun_out/lm_c5_$L.log 2>&1; echo c5 $L rc=$?
  VLGPX_LIB=$PWD/paper_2310_12000_b200/$L timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench_lm_$L.json 2> gpurun_out/bench_lm_$L.err; echo bench $L rc=$?
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_lm.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_lm.log
