cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -q -m gpu -x --durations=8 > gpurun_out/t_all.log 2>&1
B="timeout 300 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu-baseline --no-amortization --no-e2e --per-config none"
$B > gpurun_out/f_base.json 2> gpurun_out/f_base.err
timeout 300 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu-baseline --no-amortization --no-e2e --per-config none > gpurun_out/f_base2.json 2>&1
