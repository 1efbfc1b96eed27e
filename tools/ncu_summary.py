"""Summarise an ncu report (raw page) into the metrics we track."""
import csv
import io
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
        "launch__grid_size", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__average_warp_latency_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_barrier"]


def summary(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {}
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                d[w] = f"{vals[i]} {units[i]}".strip()
        d["kernel"] = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        res.append(d)
    return res


def stalls(path, top=8):
    """Top warp-stall reasons (pct of samples) from the details page."""
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    vals = rows[2]
    items = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
            try:
                items.append((float(vals[i].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    items.sort(reverse=True)
    tot = sum(v for v, _ in items) or 1
    return [(n, round(100 * v / tot, 1)) for v, n in items[:top]]


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("==", p)
        for d in summary(p):
            for k, v in d.items():
                print(f"  {k}: {v}")
        print("  stalls:", stalls(p))
