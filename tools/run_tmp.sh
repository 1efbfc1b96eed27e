cd $GRAFT_REPO_ROOT
B="timeout 300 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu-baseline --no-amortization --no-e2e"
$B > gpurun_out/e_base.json 2> gpurun_out/e_base.err
SC_OVERLAP=2 $B > gpurun_out/e_ov2.json 2> gpurun_out/e_ov2.err
SC_OVERLAP=4 $B > gpurun_out/e_ov4.json 2> gpurun_out/e_ov4.err
SC_OVERLAP=8 $B > gpurun_out/e_ov8.json 2> gpurun_out/e_ov8.err
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "warp or cfg2" > gpurun_out/t_warp.log 2>&1
