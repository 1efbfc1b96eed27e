#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_factor.py tests/test_gpu_parity.py -q -x -k "factor or implicit or perturbed" > gpurun_out/t_factor.log 2>&1; echo "rc=$?" >> gpurun_out/t_factor.log
timeout 900 python bench.py --cpu-budget 2 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
