# A/B of the in-tree library against a saved previous build (libvlgpx_prev.so)
cd $GRAFT_REPO_ROOT
for L in libvlgpx.so libvlgpx_prev.so; do
  VLGPX_LIB=$PWD/paper_2310_12000_b200/$L timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench_ab_$L.json 2> gpurun_out/bench_ab_$L.err; echo bench $L rc=$?
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_ab.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_ab.log
