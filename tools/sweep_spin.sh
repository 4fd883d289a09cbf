# bench at several nanosleep caps of the dependency polls (Ctx::spin_max_ns)
cd $GRAFT_REPO_ROOT
for S in 32 64 128 256; do VL_SPIN_MAX_NS=$S timeout 400 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/bench_spin$S.json 2>/dev/null; echo spin $S rc=$?; done
