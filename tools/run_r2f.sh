cd $GRAFT_REPO_ROOT
VL_DEBUG_SYNC=1 timeout 300 python -m pytest tests/test_gpu_predict.py -x -q -k "mode_and_blocks" > gpurun_out/r2f_dbg.log 2>&1; echo rc=$?; grep -m3 "kernel failed\|Error" gpurun_out/r2f_dbg.log | cut -c1-900
