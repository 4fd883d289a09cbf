# launch list + full capture of the dominant kernel for the bench command
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_r1.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
$CMD > gpurun_out/prof_plain2.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"trsv1_kernel|trsv_kernel|rows_kernel" -s 2000 -c 6 -o gpurun_out/prof_r1_full $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
tail -3 gpurun_out/ncu_full.log
