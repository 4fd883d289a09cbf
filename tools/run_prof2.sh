cd $GRAFT_REPO_ROOT
SKIP_P1=1 bash tools/prof_r1s3.sh
timeout 600 python -m pytest tests/test_gpu_factor.py -m gpu -x -q -k random_parents > gpurun_out/pytest_rp.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_rp.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
