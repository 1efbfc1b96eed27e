#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f gpurun_out/factor_sweep.txt
for zw in d:d 0.2:8 0.1:4 0.05:2 0.1:8; do
  IFS=: read z w <<< "$zw"
  E=""; [ $z != d ] && E="SC_FACTOR_ZMAX=$z SC_FACTOR_WSMALL=$w"
  for c in cfg2 cfg3; do
    env $E timeout 900 python bench.py --config $c --steps 5 --no-cpu-baseline --no-e2e --per-config "" > gpurun_out/b.json 2> gpurun_out/b.err
    python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1])
f=d['factor']; a=d['amortization']
print('$zw', '$c', 'factor ms %.3f'%f['ms'], 'GF/s %.0f'%f['gflops_useful'], 'tasks', f['tasks'], 'lev', f['max_level'], 'impl ms %.3f stage ms %.3f'%(a['t_apply_implicit_gpu_ms'], a['t_factor_staging_gpu_ms']))
" >> gpurun_out/factor_sweep.txt 2>&1 || tail -3 gpurun_out/b.err >> gpurun_out/factor_sweep.txt
  done
done
