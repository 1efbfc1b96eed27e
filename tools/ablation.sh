#!/bin/bash
# paper-variant ablation on B200, one short bench per variant -> gpurun_out/ablation.jsonl
#   cfg:skip:tile:strip:trsm:panel[:syrk]   (0 / auto = the plan's default; syrk = output (default) | input)
# Groups (same kernels, one knob at a time):
#   skip  -- none (original algorithm) / envelope (paper's stepped shape) /
#            exact (etree reach), at the SAME tile width, strip placement and TRSM kernel;
#   tile  -- RHS splitting granularity T;
#   panel -- factor splitting block width (the paper's uniform block-size sweep, Fig. 5 / Table 1);
#   syrk  -- SYRK input splitting (block rows summed into F') vs output splitting
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f gpurun_out/ablation.jsonl
DEF="cfg2:none:16:global:warp:0 cfg2:envelope:16:global:warp:0 cfg2:exact:16:global:warp:0
cfg2:exact:8:global:warp:0 cfg2:exact:16:auto:cta:0 cfg2:exact:32:auto:cta:0 cfg2:exact:64:auto:cta:0
cfg2:exact:16:global:warp:8 cfg2:exact:16:global:warp:16
cfg3:none:16:global:cta:0 cfg3:envelope:16:global:cta:0 cfg3:exact:16:global:cta:0
cfg3:exact:32:global:cta:0 cfg3:exact:64:global:cta:0 cfg3:exact:16:shared:cta:0
cfg3:exact:16:global:cta:16 cfg3:exact:16:global:cta:32
cfg4:envelope:16:global:cta:0 cfg4:exact:16:global:cta:0
cfg2:envelope:16:global:warp:0:input cfg2:exact:16:global:warp:0:input
cfg3:envelope:16:global:cta:0:input cfg3:exact:16:global:cta:0:input cfg4:exact:16:global:cta:0:input"
for spec in ${ABL:-$DEF}; do
  IFS=: read cfg skip tile strip trsm panel syrk <<< "$spec"
  timeout 900 python bench.py --config $cfg --skip $skip --tile $tile --strip $strip --trsm $trsm --panel $panel --syrk ${syrk:-output} \
    --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-amortization --no-factor --per-config "" \
    > gpurun_out/abl.json 2> gpurun_out/abl.err
  python - "$spec" <<'PY' >> gpurun_out/ablation.jsonl
import json, sys
spec = sys.argv[1]
try:
    d = json.loads(open("gpurun_out/abl.json").read().strip().splitlines()[-1])
    d["spec"] = spec
    print(json.dumps(d))
except Exception:
    print(json.dumps({"spec": spec, "failed": True, "err": open("gpurun_out/abl.err").read()[-400:]}))
PY
done
