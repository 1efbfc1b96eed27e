#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x -k "global or cfg5 or full_size or classes or perturbed or warp" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/variants.txt
VARIANTS="zall:" CFGS="cfg2 cfg3 cfg4" STEPS=5 bash tools/variants.sh
