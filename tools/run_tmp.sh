cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out /tmp/prof
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/variants.txt
STEPS=10 VARIANTS="" bash tools/variants.sh
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:syrk_warp16 -s 0 -c 1 -o gpurun_out/s16b -f python bench.py --config cfg2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-amortization --no-factor --per-config "" > gpurun_out/ncu_s16.log 2>&1
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:trsm_warp -s 0 -c 1 -o gpurun_out/w3 -f python bench.py --config cfg2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-amortization --no-factor --per-config "" > gpurun_out/ncu_w3.log 2>&1
