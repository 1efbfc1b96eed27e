"""Warp-stall samples per CUDA source line from an ncu report (needs -lineinfo + --import-source)."""
import csv
import io
import subprocess
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
isamp = hdr.index("Warp Stall Sampling (All Samples)")
iinst = hdr.index("Instructions Executed")
lines = []
for r in rows:
    if len(r) > isamp and r[0].isdigit() and r[2] == "-" and r[isamp].isdigit():
        ni = int(r[iinst]) if r[iinst].isdigit() else 0
        lines.append((int(r[isamp]), int(r[0]), r[1].strip(), ni))
tot = sum(x[0] for x in lines) or 1
toti = sum(x[3] for x in lines) or 1
print(f"total samples {tot}, warp instructions {toti}")
for s, ln, src, ni in sorted(lines, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}% smp {100 * ni / toti:5.1f}% inst  L{ln:5d}  {src[:100]}")
if "--inst" in sys.argv:
    print("-- by instructions")
    for s, ln, src, ni in sorted(lines, key=lambda x: -x[3])[:top]:
        print(f"{100 * s / tot:5.1f}% smp {100 * ni / toti:5.1f}% inst  L{ln:5d}  {src[:100]}")

# per-line stall-reason breakdown for the top lines (columns named like "Warp Stall Sampling (...)")
reason_cols = [k for k, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
if len(sys.argv) > 3 and reason_cols and sys.argv[3] != "--inst":
    want = set(int(x) for x in sys.argv[3].split(","))
    for r in rows:
        if len(r) > isamp and r[0].isdigit() and r[2] == "-" and int(r[0]) in want:
            br = sorted(((float(r[k]) if r[k].replace(".", "").isdigit() else 0.0, hdr[k]) for k in reason_cols), reverse=True)
            print(f"L{r[0]}: " + ", ".join(f"{h}={v:.0f}" for v, h in br[:6] if v > 0))
