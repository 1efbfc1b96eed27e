#!/bin/bash
# ncu evidence: launch list of a short bench and one --set full capture of each assembly kernel
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFG=${CFG:-cfg2}
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv \
  python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_$CFG.log 2>&1
for K in ${KERNELS:-prep_panel_kernel trsm_smem_kernel syrk_pair_kernel}; do
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o gpurun_out/prof_${CFG}_$K -f \
    python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_${CFG}_$K.log 2>&1
done
