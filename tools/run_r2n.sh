# round-2 pass after the solve-order change: GPU tests, bench line, launch list, ncu --set full of the top kernels
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2n_pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/r2n_pytest_gpu.log | cut -c1-200
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r2n.json 2> gpurun_out/bench_r2n.err; echo bench rc=$?; head -c 300 gpurun_out/bench_r2n.json; echo
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-c4 --e2e-steps 1"
ncu --metrics gpu__time_duration.sum --clock-control none -s 22000 -c 12000 --csv --log-file gpurun_out/r2n_launches.csv $CMD > gpurun_out/r2n_ncu_launches.log 2>&1; echo launches rc=$?
gzip -f gpurun_out/r2n_launches.csv
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"trsv1_kernel|K2Body" -s 300 -c 3 -o /tmp/p1 $CMD > gpurun_out/r2n_ncu_p1.log 2>&1; echo p1 rc=$?
python tools/ncu_summary.py /tmp/p1.ncu-rep > gpurun_out/r2n_ncu_full_summary.txt 2>&1
ncu -i /tmp/p1.ncu-rep --page raw --csv | gzip > gpurun_out/r2n_ncu_p1_raw.csv.gz
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"trsv_kernel<\\(int\\)32" -s 8 -c 2 -o /tmp/p2 $CMD > gpurun_out/r2n_ncu_p2.log 2>&1; echo p2 rc=$?
python tools/ncu_summary.py /tmp/p2.ncu-rep >> gpurun_out/r2n_ncu_full_summary.txt 2>&1
ncu -i /tmp/p2.ncu-rep --page raw --csv | gzip > gpurun_out/r2n_ncu_p2_raw.csv.gz
cat gpurun_out/r2n_ncu_full_summary.txt | cut -c1-250
timeout 900 python tools/c5_sweep.py --out gpurun_out/c5_sweep_r2n.jsonl > gpurun_out/c5_sweep_r2n.log 2>&1; echo c5 rc=$?
timeout 300 python tools/c5_sweep.py --ns 1000000 --ms 20 --kinds knn --out gpurun_out/c5_knn_r2n.jsonl > gpurun_out/c5_knn_r2n.log 2>&1; echo knn rc=$?
timeout 600 python tools/bench_c2.py > gpurun_out/c2_r2n.jsonl 2> gpurun_out/c2_r2n.err; echo c2 rc=$?; tail -3 gpurun_out/c2_r2n.jsonl | cut -c1-300
