#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "perturbed" > gpurun_out/t_pert.log 2>&1; echo "rc=$?" >> gpurun_out/t_pert.log
timeout 1500 python bench.py --config cfg3 --perturbed --steps 5 --no-cpu-baseline --no-e2e --per-config "" --no-amortization > gpurun_out/bench_cfg3_perturbed.json 2> gpurun_out/bench_cfg3_perturbed.err
timeout 1500 python bench.py --config cfg2 --perturbed --steps 5 --no-cpu-baseline --no-e2e --per-config "" --no-amortization > gpurun_out/bench_cfg2_perturbed.json 2> gpurun_out/bench_cfg2_perturbed.err
