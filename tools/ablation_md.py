"""gpurun_out/ablation.jsonl -> markdown tables (profiles/ablation_<tag>.md).

    python tools/ablation_md.py gpurun_out/ablation.jsonl r02 > profiles/ablation_r02.md
"""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip()]
tag = sys.argv[2] if len(sys.argv) > 2 else "r02"
print(f"# Paper-variant ablation on 1 B200 (SURVEY §8.5 f3), {tag}\n")
print("`tools/ablation.sh`: one `bench.py` line per variant (3 timed steps after 3 warm-up, L device-resident,")
print("inputs larger than L2).  Spec = cfg:skip:T:strip:trsm:panel[:syrk] (0 = plan default; syrk input = input-split SYRK).  `useful GF/s` divides the")
print("same etree-exact flop count by each variant's step time, so it compares variants directly; `executed GF/s`")
print("is what the kernels computed.\n")
hdr = "| spec | subdomains/s | TRSM ms | SYRK ms | prep ms | executed GF/s | useful GF/s | T | panel | strip | trsm | syrk | vs skip none |"
print(hdr)
print("|" + "---|" * (hdr.count("|") - 1))
base = {}
for d in rows:
    if d.get("failed"):
        continue
    cfg, skip = d["spec"].split(":")[:2]
    if skip == "none":
        base[cfg] = d["value"]
for d in rows:
    if d.get("failed"):
        print(f"| {d['spec']} | failed | | | | | | | | | | | |")
        continue
    cfg = d["spec"].split(":")[0]
    c = d["config"]
    ph = d["phase_ms"]
    rel = f"{d['value'] / base[cfg]:.1f}x" if cfg in base else ""
    print(f"| {d['spec']} | {d['value']:.0f} | {ph['trsm']:.2f} | {ph['syrk']:.2f} | {ph['prep']:.2f} | "
          f"{d['gflops_executed']:.0f} | {d['gflops_useful']:.0f} | {c['tile_cols']} | {c['panel_cols']} | "
          f"{c['x_strip']} | {c['trsm_kernel']} | {c.get('syrk_split', 'output')} | {rel} |")
