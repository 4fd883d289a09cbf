# round-2 measurement pass: config-4 check, launch list of one bench step, dense kernels,
# config-5 sweep, config-2 VADU vs LRAC, complete CPU evaluations (reference arm)
cd $GRAFT_REPO_ROOT
python -c "import bench, json; print(json.dumps(bench.config4_prediction()))" > gpurun_out/r2b_c4.json 2> gpurun_out/r2b_c4.err; echo c4 rc=$?
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-c4 --e2e-steps 1"
$CMD > gpurun_out/r2b_plain.json 2> gpurun_out/r2b_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 11000 -c 12000 --csv --log-file gpurun_out/r2b_launches.csv $CMD > gpurun_out/r2b_ncu_launches.log 2>&1
echo "launches rc=$?"
gzip -f gpurun_out/r2b_launches.csv
python tools/dense_bench.py > gpurun_out/r2b_dense.log 2>&1; echo dense rc=$?
timeout 900 python tools/c5_sweep.py --ns 1000000,10000000 --ms 20 --out gpurun_out/r2b_c5.jsonl > gpurun_out/r2b_c5.log 2>&1; echo c5 rc=$?
timeout 300 python tools/c5_sweep.py --ns 1000000 --ms 20 --kinds knn --out gpurun_out/r2b_c5_knn.jsonl > gpurun_out/r2b_c5_knn.log 2>&1; echo knn rc=$?
timeout 600 python tools/bench_c2.py --precs vadu,lrac --steps 2 --newton-grad-tol 4e-5 --prof > gpurun_out/r2b_c2.json 2>gpurun_out/r2b_c2.err; echo c2 rc=$?
timeout 3000 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2b_ref.json 2> gpurun_out/r2b_ref.err; echo ref rc=$?
