#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_factor.py tests/test_gpu_parity.py -q -x -k "factor or implicit or perturbed or cfg2_class or warp" > gpurun_out/t_factor.log 2>&1; echo "rc=$?" >> gpurun_out/t_factor.log
rm -f gpurun_out/factor_sweep.txt
for c in cfg2 cfg3; do
  timeout 900 python bench.py --config $c --steps 5 --no-cpu-baseline --no-e2e --per-config "" > gpurun_out/b.json 2> gpurun_out/b.err
  python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1])
f=d['factor']; a=d['amortization']
print('$c', round(d['value']), d['phase_ms'], 'factor ms %.3f'%f['ms'], 'impl ms %.3f stage %.3f'%(a['t_apply_implicit_gpu_ms'], a['t_factor_staging_gpu_ms']))
" >> gpurun_out/factor_sweep.txt 2>&1 || tail -3 gpurun_out/b.err >> gpurun_out/factor_sweep.txt
done
