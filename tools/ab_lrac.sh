# LRAC path at config 2: hand-written dense kernels vs the previous cuBLAS build (_ab_prev/)
cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_dense.py -q > gpurun_out/r2h_pytest_dense.log 2>&1; echo dense rc=$?
python tools/c2_lrac_tol.py 1e-5,2e-5,4e-5
C2_ROOT=$PWD/_ab_prev python tools/c2_lrac_tol.py 1e-5,2e-5,4e-5
timeout 600 python tools/bench_c2.py --precs lrac --steps 2 --newton-grad-tol 4e-5 --prof > gpurun_out/r2h_c2_new.json 2>/dev/null; echo c2new rc=$?
cd _ab_prev && timeout 600 python tools/bench_c2.py --precs lrac --steps 2 --newton-grad-tol 4e-5 --prof > ../gpurun_out/r2h_c2_prev.json 2>/dev/null; echo c2prev rc=$?
