cd $GRAFT_REPO_ROOT
run() { VLGPX_LIB=$PWD/paper_2310_12000_b200/$1 timeout 400 python tools/pcgbench.py --ts 1 --iters 120 --label "$2" >> gpurun_out/r2h_pcgbench.jsonl 2>> gpurun_out/r2h_pcgbench.err; echo pcg $2 rc=$?; }
run libvlgpx.so base
run libvlgpx_v7.so gather_ca
VL_SLAB_SORT=1 run libvlgpx.so slab_sort
VL_SLAB_SORT=1 run libvlgpx_v7.so gather_ca+slab_sort
run libvlgpx_v2.so stream_pf8
run libvlgpx_v3.so stream_pf20
run libvlgpx.so base
cat gpurun_out/r2h_pcgbench.jsonl
VLGPX_LIB=$PWD/paper_2310_12000_b200/libvlgpx_v7.so timeout 600 python -m pytest tests/test_gpu_factor.py tests/test_gpu_laplace.py tests/test_gpu_scale.py -x -q 2>&1 | tail -3
