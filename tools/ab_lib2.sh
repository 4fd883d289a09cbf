# A/B of the in-tree library against libvlgpx_prev.so + launch list of the new one (head kernels)
cd $GRAFT_REPO_ROOT
for L in libvlgpx.so libvlgpx_prev.so; do
  VLGPX_LIB=$PWD/paper_2310_12000_b200/$L timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench_ab_$L.json 2> gpurun_out/bench_ab_$L.err; echo bench $L rc=$?
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_ab.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_ab.log
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:head_ -c 200 --csv --log-file gpurun_out/head_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/head_launches.csv > gpurun_out/head_launches_summary.txt
