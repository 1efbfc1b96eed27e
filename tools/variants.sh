#!/bin/bash
# A/B of compile-time variants: VARIANTS="name:DEF1=v,DEF2=v ..." CFGS="cfg2 ..." -> gpurun_out/variants.txt
# (each variant built here as paper_2509_21037_b200/libsc_b200_<name>.so and selected with SC_B200_LIB)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for spec in base: $VARIANTS; do
  IFS=: read name defs <<< "$spec"
  lib=paper_2509_21037_b200/libsc_b200.so
  [ "$name" != "base" ] && lib=paper_2509_21037_b200/libsc_b200_$name.so
  for cfg in ${CFGS:-cfg2}; do
    timeout 600 env SC_B200_LIB=$PWD/$lib ${ENVS} python bench.py --config $cfg --steps ${STEPS:-5} --warmup 3 --no-e2e --no-cpu-baseline --no-amortization --no-factor --per-config "" > gpurun_out/v.json 2> gpurun_out/v.err
    python -c "
import json
try:
    d=json.loads(open('gpurun_out/v.json').read().strip().splitlines()[-1])
    print('$name $cfg', round(d['value']), {k: round(v,3) for k,v in d['phase_ms'].items()}, round(d['roofline']['frac'],3))
except Exception as e:
    print('$name $cfg FAILED', open('gpurun_out/v.err').read()[-600:])
" >> gpurun_out/variants.txt
  done
done
