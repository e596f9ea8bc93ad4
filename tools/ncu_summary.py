"""Summarise an ncu report (--set full) into a small JSON for profiles/.

usage: python tools/ncu_summary.py <report.ncu-rep> [--out profiles/x.json]
Per profiled launch: kernel, duration, DRAM bytes read/write, DMMA pipe
activity, achieved occupancy, registers, top stall reasons.
"""

import argparse
import csv
import io
import json
import subprocess

KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active": "dmma_pipe_active_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_active_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__inst_executed.sum": "inst_executed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
}
STALLS = [
    "barrier", "long_scoreboard", "short_scoreboard", "wait", "math_pipe_throttle", "mio_throttle",
    "lg_throttle", "not_selected", "selected", "branch_resolving", "no_instruction", "dispatch_stall",
]


def summarise(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    units = dict(zip(hdr, rows[1]))
    scale = {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        rec = {"kernel": d.get("Kernel Name", "")[:120]}
        for k, name in KEYS.items():
            v = d.get(k)
            if v not in (None, ""):
                try:
                    rec[name] = float(v.replace(",", "")) * scale.get(units.get(k, ""), 1.0)
                except ValueError:
                    rec[name] = v
        stalls = {}
        for s in STALLS:
            v = d.get(f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio")
            if v not in (None, ""):
                stalls[s] = float(v)
        rec["stall_cycles_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
        if "dram_read_bytes" in rec and "dram_write_bytes" in rec:
            rec["dram_bytes"] = rec["dram_read_bytes"] + rec["dram_write_bytes"]
        out.append(rec)
    return out


def families(launches):
    """Per kernel family: launches, total / average duration, DRAM bytes,
    duration-weighted DMMA pipe activity, and the K2 bytes of the capture
    (every gj_* / band_* / pattern / plan launch: one call when the capture is one call)."""
    fam = {}
    for r in launches:
        k = r["kernel"].split("(")[0].replace("void ", "").split("<")[0].replace("rdb::", "")
        f = fam.setdefault(k, {"launches": 0, "total_ns": 0.0, "dram_bytes": 0.0, "_dmma": 0.0})
        f["launches"] += 1
        f["total_ns"] += r.get("duration_ns", 0.0)
        f["dram_bytes"] += r.get("dram_bytes", 0.0)
        f["_dmma"] += r.get("dmma_pipe_active_pct", 0.0) * r.get("duration_ns", 0.0)
    tot = sum(f["total_ns"] for f in fam.values()) or 1.0
    for f in fam.values():
        f["avg_ns"] = f["total_ns"] / f["launches"]
        f["share"] = f["total_ns"] / tot
        f["dmma_pipe_active_pct"] = f.pop("_dmma") / max(f["total_ns"], 1.0)
    k2 = sum(f["dram_bytes"] for k, f in fam.items()
             if k.startswith(("gj_", "band_")) or "pattern" in k)
    return fam, k2


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--out")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    res = {"report": a.report, "note": a.note, "launches": summarise(a.report)}
    res["families"], res["k2_dram_bytes_per_call"] = families(res["launches"])
    txt = json.dumps(res, indent=1)
    if a.out:
        open(a.out, "w").write(txt + "\n")
    print(txt)
