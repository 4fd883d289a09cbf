# round-end style check: GPU tests, smoke, default bench, launch list of one bench step
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/final_smoke.log
timeout 600 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo bench rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv --log-file gpurun_out/final_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/final_ncu.log 2>&1; echo ncu rc=$?
python tools/launch_summary.py gpurun_out/final_launches.csv > gpurun_out/final_launches_summary.txt; gzip -f gpurun_out/final_launches.csv
