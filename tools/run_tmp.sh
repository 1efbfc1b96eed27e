#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f gpurun_out/variants.txt
VARIANTS="b8: b2:" CFGS="cfg2" STEPS=10 bash tools/variants.sh
VARIANTS="" CFGS="cfg2" STEPS=10 bash tools/variants.sh
