# config-5 kernel sweep + kNN factor, scipy-checked (tools/c5_sweep.py)
cd $GRAFT_REPO_ROOT
timeout 900 python tools/c5_sweep.py --out gpurun_out/c5_sweep_b.jsonl > gpurun_out/c5_sweep_b.log 2>&1; echo c5 rc=$?
timeout 300 python tools/c5_sweep.py --ns 1000000 --ms 20 --kinds knn --out gpurun_out/c5_knn_b.jsonl > gpurun_out/c5_knn_b.log 2>&1; echo knn rc=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_b.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_b.log
timeout 400 python bench.py > gpurun_out/bench_c5run.json 2> gpurun_out/bench_c5run.err; echo bench rc=$?
