cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sanitizer
for CFG in cfg1 t3e; do for TOOL in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $TOOL --print-limit 20 python tools/sanitize_run.py $CFG > gpurun_out/sanitizer/${TOOL}_${CFG}.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitizer/${TOOL}_${CFG}.txt
done; done
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
