#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_factor.py -q -x > gpurun_out/t_factor.log 2>&1; echo "rc=$?" >> gpurun_out/t_factor.log
rm -f gpurun_out/factor_sweep.txt
for v in base old; do
  lib=$PWD/paper_2509_21037_b200/libsc_b200_$v.so; [ $v = base ] && lib=$PWD/paper_2509_21037_b200/libsc_b200.so
  for c in cfg2 cfg3 cfg4; do
    SC_B200_LIB=$lib timeout 900 python bench.py --config $c --steps 5 --no-cpu-baseline --no-e2e --per-config "" --no-amortization > gpurun_out/b.json 2> gpurun_out/b.err
    python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1])
f=d['factor']
print('$v', '$c', 'factor ms %.3f'%f['ms'], 'GF/s %.0f'%f['gflops_useful'], 'tasks', f['tasks'])
" >> gpurun_out/factor_sweep.txt 2>&1 || tail -3 gpurun_out/b.err >> gpurun_out/factor_sweep.txt
  done
done
