# ncu --set full captures of the current bench step's top kernels (single-RHS solves,
# single-RHS B^T product, t = 50 solves); raw CSV exported on the box
cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err || exit 1
if [ -z "$SKIP_P1" ]; then
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"trsv1_kernel|K2Body" -s 300 -c 3 -o /tmp/p1 $CMD > gpurun_out/ncu_p1.log 2>&1; echo p1 rc=$?
ncu -i /tmp/p1.ncu-rep --page raw --csv > gpurun_out/ncu_p1_raw.csv
fi
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"trsv_kernel<\\(int\\)32" -s 8 -c 2 -o /tmp/p2 $CMD > gpurun_out/ncu_p2.log 2>&1; echo p2 rc=$?
ncu -i /tmp/p2.ncu-rep --page raw --csv > gpurun_out/ncu_p2_raw.csv
ncu -i /tmp/p2.ncu-rep --page details --csv > gpurun_out/ncu_p2_details.csv
ls -la gpurun_out/*.csv
