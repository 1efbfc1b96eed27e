"""Top SASS instructions by warp-stall samples from an ncu report (source page)."""
import csv
import io
import subprocess
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
ia, isrc, isamp = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[isamp]) for r in data if r[isamp].isdigit())
order = sorted(range(len(data)), key=lambda k: -int(data[k][isamp]) if data[k][isamp].isdigit() else 0)
print(f"total samples {tot}")
for k in order[:top]:
    r = data[k]
    print(f"{int(r[isamp]) / tot * 100:5.1f}%  #{k:5d}  {r[isrc].strip()}")

# aggregate by opcode
agg = {}
for r in data:
    if not r[isamp].isdigit():
        continue
    src = r[isrc].strip()
    toks = src.split()
    op = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "?")
    op = op.split(".")[0]
    agg[op] = agg.get(op, 0) + int(r[isamp])
print("by opcode:", ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:14]))
