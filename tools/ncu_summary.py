"""Summarise ncu output for profiles/: the launch list (per-kernel device time and share
of the step, from `ncu --metrics gpu__time_duration.sum --csv`) and one `--set full`
capture (DRAM bytes, throughput, occupancy, pipe utilisation per captured launch).

    python tools/ncu_summary.py <launches.csv> <prof.ncu-rep> <out.json>
"""
import csv, io, json, subprocess, sys
from collections import OrderedDict


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    out = []
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        us = {"ns": v / 1e3, "nsecond": v / 1e3, "us": v, "usecond": v, "ms": v * 1e3, "msecond": v * 1e3}[unit]
        out.append((r[ki], us))
    agg = OrderedDict()
    for k, us in out:
        short = k.split("(")[0].replace("void ", "").split("::")[-1]
        a = agg.setdefault(short, [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(a[1] for a in agg.values())
    return {"launches": len(out), "total_us": tot,
            "kernels": {k: {"n": a[0], "total_us": a[1], "avg_us": a[1] / a[0], "share": a[1] / tot} for k, a in agg.items()}}


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.sum", "lts__t_bytes.sum", "launch__occupancy_limit_registers",
        "sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def full(path):
    p = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(p.stdout)))
    if not rows:
        return []
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")][:80]}
        for w in WANT:
            if w in h:
                i = h.index(w)
                d[w] = f"{r[i]} {units[i]}".strip()
        res.append(d)
    return res


if __name__ == "__main__":
    out = {"launch_list": launches(sys.argv[1]) if sys.argv[1] != "-" else None,
           "full_capture": full(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else None}
    json.dump(out, open(sys.argv[3], "w"), indent=1)
    print(json.dumps(out, indent=1)[:3000])
