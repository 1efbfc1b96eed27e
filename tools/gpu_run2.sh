cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in cfg2 cfg3; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --cpu-budget 2 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:trsm_smem -s 1 -c 1 -o gpurun_out/prof_cfg2_trsm -f python bench.py --config cfg2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_trsm.log 2>&1
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:prep_small -s 1 -c 1 -o gpurun_out/prof_cfg2_prepsmall -f python bench.py --config cfg2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_ps.log 2>&1
