cd $GRAFT_REPO_ROOT
VL_DEBUG_NEWTON=1 timeout 300 python tools/c2_lrac_tol.py 1e-5 2>&1 | head -60
cd _ab_prev && VL_DEBUG_NEWTON=1 C2_ROOT=$PWD timeout 300 python ../tools/c2_lrac_tol.py 1e-5 2>&1 | head -45
