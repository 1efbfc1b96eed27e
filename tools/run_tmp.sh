#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out /tmp/prof
L=paper_2509_21037_b200
for v in base pf pf3 minb3 minb5 minb6; do
  lib=$PWD/$L/libsc_b200_$v.so; [ $v = base ] && lib=$PWD/$L/libsc_b200.so
  for c in cfg2 cfg3; do
    [ $c = cfg3 ] && [[ $v == minb* ]] && continue
    SC_B200_LIB=$lib timeout 900 python bench.py --config $c --steps 5 --no-cpu-baseline --no-e2e --per-config "" > gpurun_out/b.json 2> gpurun_out/b.err
    python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1])
f=d['factor']; a=d['amortization']
print('$v', '$c', 'factor ms %.3f'%f['ms'], 'tasks', f['tasks'], 'impl ms %.3f stage ms %.3f'%(a['t_apply_implicit_gpu_ms'], a['t_factor_staging_gpu_ms']), 'asm %.3f'%d['ms_per_step'], {k: round(x,3) for k,x in d['phase_ms'].items()})
" >> gpurun_out/variant_sweep.txt 2>&1 || tail -3 gpurun_out/b.err >> gpurun_out/variant_sweep.txt
  done
done
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:implicit_ -s 2 -c 2 -o /tmp/prof/prof_cfg2_implicit -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --per-config "" --no-factor > /tmp/prof/ncu_i.log 2>&1
python tools/ncu_summary.py /tmp/prof/prof_cfg2_implicit.ncu-rep > gpurun_out/ncu_implicit_cfg2.txt 2>&1
python tools/ncu_hot.py /tmp/prof/prof_cfg2_implicit.ncu-rep 25 >> gpurun_out/ncu_implicit_cfg2.txt 2>&1
tail -3 /tmp/prof/ncu_i.log >> gpurun_out/ncu_implicit_cfg2.txt
