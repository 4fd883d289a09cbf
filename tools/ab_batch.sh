# per-direction batch width check (CSR: 8-entry batches at 3 CTAs/SM)
cd $GRAFT_REPO_ROOT
timeout 300 python tools/c5_sweep.py --ns 1000000 --ms 20 --ts 16,64 --kinds knn,random --reps 10 --check 1 > gpurun_out/bt2_c5.log 2>&1; echo c5 rc=$?
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench_bt2.json 2> gpurun_out/bench_bt2.err; echo bench rc=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_bt2.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_bt2.log
