#!/bin/bash
# paper-variant ablation on B200 -- skip mode (none = original algorithm without the
# stepped/sparse-RHS skipping, envelope = the paper's stepped envelope, exact = etree reach) x tile
# width, same kernels; one short bench per variant -> gpurun_out/ablation.jsonl
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for spec in ${ABL:-cfg2:none:0 cfg2:envelope:0 cfg2:exact:0 cfg3:none:0 cfg3:envelope:0 cfg3:exact:0 cfg3:exact:32}; do
  IFS=: read cfg skip tile <<< "$spec"
  timeout 900 python bench.py --config $cfg --skip $skip --tile $tile --steps 3 --warmup 3 --no-e2e --no-cpu-baseline \
    --no-amortization > gpurun_out/abl.json 2> gpurun_out/abl.err && cat gpurun_out/abl.json >> gpurun_out/ablation.jsonl \
    || echo "{\"spec\": \"$spec\", \"failed\": true}" >> gpurun_out/ablation.jsonl
done
