# single-RHS PCG per-iteration time vs the lagged item start (VL_TRSV_LAG) and its backoff cap
cd $GRAFT_REPO_ROOT
for cfg in "0 256" "2 256" "3 256" "4 256" "6 256" "3 128" "3 1024" "8 256"; do
  set -- $cfg
  VL_TRSV_LAG=$1 VL_LAG_NS=$2 timeout 300 python tools/pcgbench.py --ts 1 --iters 120 --label "lag$1_ns$2" 2>&1 | tail -1
done
