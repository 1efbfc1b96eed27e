"""Copy the ncu evidence of a gpurun into profiles/ (tracked): per-kernel summaries of the
`--set full` captures, the launch lists, and profiles/traffic_<cfg>.json (DRAM bytes per launch of
each phase's kernel, read by bench.py for roofline.traffic).

    python tools/make_profiles.py r01 gpurun_out [dst_dir]
"""
import csv
import glob
import io
import json
import os
import shutil
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import stalls, summary  # noqa: E402

tag = sys.argv[1]
src = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
dst = sys.argv[3] if len(sys.argv) > 3 else os.path.join(root, "profiles")
os.makedirs(dst, exist_ok=True)

PHASE = {"prep_panel_kernel": "prep", "prep_small_kernel": "prep", "trsm_smem_kernel": "trsm", "trsm_warp_kernel": "trsm",
         "factor_kernel": "factor", "implicit_fwd_kernel": "implicit_fwd", "implicit_bwd_kernel": "implicit_bwd",
         "syrk_pair_kernel": "syrk", "syrk_warp16_kernel": "syrk"}


def to_bytes(s):
    v, unit = s.split()[0], s.split()[1] if len(s.split()) > 1 else "byte"
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


traffic = {}
for rep in sorted(glob.glob(os.path.join(src, "prof_*.ncu-rep"))):
    base = os.path.basename(rep)[len("prof_"):-len(".ncu-rep")]
    cfg, kernel = base.split("_", 1)
    lines = []
    for d in summary(rep):
        for k, v in d.items():
            lines.append(f"{k}: {v}")
        t = to_bytes(d.get("dram__bytes_read.sum", "0 byte")) + to_bytes(d.get("dram__bytes_write.sum", "0 byte"))
        ph = PHASE.get(kernel)
        if ph:
            traffic.setdefault(cfg, {})
            traffic[cfg][ph] = traffic[cfg].get(ph, 0.0) + t
    lines.append(f"stalls: {stalls(rep)}")
    hot = subprocess.run([sys.executable, os.path.join(root, "tools", "ncu_hot.py"), rep, "12"], capture_output=True,
                         text=True).stdout
    lines.append(hot)
    with open(os.path.join(dst, f"ncu_{cfg}_{kernel}_{tag}.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
for cfg, t in traffic.items():
    with open(os.path.join(dst, f"traffic_{cfg}.json"), "w") as f:
        json.dump({"bytes_per_launch": t, "source": f"ncu --set full ({tag}), dram__bytes_read.sum + dram__bytes_write.sum",
                   **t}, f, indent=1)
for lc in glob.glob(os.path.join(src, "launches_*.csv")):
    shutil.copy(lc, os.path.join(dst, os.path.basename(lc).replace(".csv", f"_{tag}.csv")))
for bj in glob.glob(os.path.join(src, "bench_*.json")):
    shutil.copy(bj, os.path.join(dst, os.path.basename(bj).replace(".json", f"_{tag}.json")))
print("profiles written to", dst)
