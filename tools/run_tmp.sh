cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CFGS=cfg2 KERNELS="trsm_warp_kernel syrk_warp16_kernel factor_kernel implicit_fwd_kernel" TAG=r02 BENCH_CFGS="cfg2" bash tools/gpu_prof.sh > gpurun_out/prof.log 2>&1
bash tools/ablation.sh > gpurun_out/abl.log 2>&1
python tools/ablation_md.py gpurun_out/ablation.jsonl r02 > gpurun_out/ablation_r02.md 2>&1
