cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2g_pytest.log 2>&1; echo rc=$?; tail -4 gpurun_out/r2g_pytest.log | cut -c1-300
