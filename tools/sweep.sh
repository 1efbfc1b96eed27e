#!/bin/bash
# short bench sweep: SWEEP="cfg:tile:panel[:extra] ..." -> gpurun_out/sweep.txt
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for spec in $SWEEP; do
  IFS=: read cfg tile panel strip extra <<< "$spec"
  timeout 600 env ${extra//,/ } python bench.py --config $cfg --tile $tile --panel $panel --strip ${strip:-auto} --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-amortization > gpurun_out/sw.json 2> gpurun_out/sw.err
  python -c "
import json,sys
try:
    d=json.load(open('gpurun_out/sw.json'))
    print('$spec', round(d['value']), {k: round(v,3) for k,v in d['phase_ms'].items()}, d['config'].get('tile_cols'), d['config'].get('x_strip'), d['config'].get('trsm_tasks_2cta'), round(d['roofline']['frac'],3))
except Exception as e:
    print('$spec FAILED', open('gpurun_out/sw.err').read()[-600:])
" >> gpurun_out/sweep.txt
done
