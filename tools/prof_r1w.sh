# ncu --set full of the t=1 kernels changed after the session-3 captures
# (streamed B^T product K2Body, head GEMV, backward head rhs), one bench step
cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/prof_w_plain.json 2> gpurun_out/prof_w_plain.err || exit 1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"K2Body|head_gemv_kernel|head_rhs_kernel" -s 300 -c 4 -o /tmp/pw $CMD > gpurun_out/ncu_w.log 2>&1; echo ncu rc=$?
python tools/ncu_summary.py /tmp/pw.ncu-rep > gpurun_out/r1w_ncu_full_summary.txt 2>&1
ncu -i /tmp/pw.ncu-rep --page raw --csv | gzip > gpurun_out/r1w_ncu_raw.csv.gz
