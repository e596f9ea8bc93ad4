"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel launch counts, total device time and share of the step.

usage: python tools/launch_shares.py gpurun_out/launches.csv [--out profiles/x.json]
"""

import argparse
import collections
import csv
import json


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--out")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    lines = [ln for ln in open(a.csv) if not ln.startswith("==")]
    rows = list(csv.reader(lines))
    h = rows[0]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    other = collections.defaultdict(list)
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("void ", "").split("<")[0]
        if r[mi] == "gpu__time_duration.sum":
            scale = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(r[ui], 1.0)
            tot[name] += float(r[vi].replace(",", "")) * scale
            cnt[name] += 1
        else:
            try:
                other[(name, r[mi])].append(float(r[vi].replace(",", "")))
            except ValueError:
                pass
    total = sum(tot.values())
    res = {"note": a.note, "total_ns": total, "kernels": {}}
    for k in sorted(tot, key=lambda k: -tot[k]):
        res["kernels"][k] = {"launches": cnt[k], "total_ns": tot[k], "avg_ns": tot[k] / cnt[k],
                             "share": tot[k] / total}
    for (k, m), vals in other.items():
        res["kernels"].setdefault(k, {})[m + ".avg"] = sum(vals) / len(vals)
    txt = json.dumps(res, indent=1)
    if a.out:
        open(a.out, "w").write(txt + "\n")
    print(txt)


if __name__ == "__main__":
    main()
