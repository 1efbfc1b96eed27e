#!/bin/bash
# ncu evidence for CFGS: launch list of a short bench (serialised, cold-cache per launch) and one
# `--set full` capture of each phase's first kernel; then the round's bench lines.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out /tmp/prof
NCU=/usr/local/cuda/bin/ncu
# reports stay on the box (/tmp/prof, too large to bring back); summaries go to gpurun_out/profiles
for CFG in ${CFGS:-cfg2 cfg3 cfg4}; do
  timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/prof/launches_$CFG.csv \
    python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-amortization --no-factor --per-config "" > /tmp/prof/ncu_launch_$CFG.log 2>&1
  for K in ${KERNELS:-prep_small_kernel prep_panel_kernel trsm_smem_kernel syrk_pair_kernel}; do
    case $K in  # the factorization / implicit kernels run in bench's factor / amortization legs
      factor_kernel) X="--no-amortization" ;;
      implicit_*) X="--no-factor" ;;
      *) X="--no-amortization --no-factor" ;;
    esac
    timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$K -s 0 -c 1 -o /tmp/prof/prof_${CFG}_$K -f \
      python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --per-config "" $X > /tmp/prof/ncu_full_${CFG}_$K.log 2>&1
  done
done
mkdir -p gpurun_out/profiles
python tools/make_profiles.py ${TAG:-r01} /tmp/prof gpurun_out/profiles > gpurun_out/make_profiles.log 2>&1
for CFG in ${CFGS:-cfg2 cfg3 cfg4}; do  # per-line stall tables of the TRSM / SYRK captures
  for K in trsm_smem_kernel trsm_warp_kernel syrk_pair_kernel syrk_warp16_kernel factor_kernel implicit_fwd_kernel; do
    [ -f /tmp/prof/prof_${CFG}_$K.ncu-rep ] && python tools/ncu_lines.py /tmp/prof/prof_${CFG}_$K.ncu-rep 25 > gpurun_out/profiles/lines_${CFG}_${K}_${TAG:-r01}.txt 2>&1
  done
done
ls -la /tmp/prof > gpurun_out/prof_ls.txt
for c in ${BENCH_CFGS:-cfg2 cfg3 cfg4}; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --cpu-budget 10 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
