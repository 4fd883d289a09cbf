cd $GRAFT_REPO_ROOT
python tools/dense_bench.py
python -m pytest tests/test_gpu_dense.py tests/test_gpu_probes.py tests/test_gpu_laplace.py tests/test_gpu_scale.py tests/test_gpu_multirank.py tests/test_gpu_predict.py -q -rs -x 2>&1 | grep -v Warning | tail -30
python tools/c2_lrac_tol.py 4e-5
timeout 600 python tools/bench_c2.py --precs lrac,vadu --steps 2 --newton-grad-tol 4e-5 --prof > gpurun_out/r2k_c2.json 2>/dev/null; echo c2 rc=$?
