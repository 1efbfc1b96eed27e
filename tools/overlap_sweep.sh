#!/bin/bash
# phase overlap (SC_OVERLAP=K chunks: TRSM of chunk k+1 beside the SYRK of chunk k) x warp-TRSM CTAs/SM
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f gpurun_out/variants.txt
for K in 0 2 4 8; do
  ENVS="SC_OVERLAP=$K" VARIANTS="minb2:" CFGS="cfg2" STEPS=10 bash tools/variants.sh
  sed -i "s/^\(base\|minb2\) cfg2/\1 ov$K cfg2/" gpurun_out/variants.txt
done
