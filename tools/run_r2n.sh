cd $GRAFT_REPO_ROOT
python bench.py --steps 5 --warmup 3 > gpurun_out/r2n_bench.json 2> gpurun_out/r2n_bench.err; echo bench rc=$?
python tools/dense_bench.py 2>&1 | head -1
timeout 600 python tools/bench_c2.py --precs lrac --steps 2 --newton-grad-tol 4e-5 --prof > gpurun_out/r2n_c2.json 2>/dev/null; echo c2 rc=$?
timeout 2400 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2n_ref.json 2> gpurun_out/r2n_ref.err; echo ref rc=$?
