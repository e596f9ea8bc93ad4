"""Top stall-sampled source lines (CUDA source and SASS) of one kernel in an
ncu report: python tools/ncu_source_top.py rep.ncu-rep [N] > out.txt"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for view in ("cuda", "sass"):
    out = subprocess.run(["/usr/local/cuda/bin/ncu", "-i", rep, "--page", "source", "--csv", "--print-source", view],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if not rows:
        continue
    hdr_i = next((i for i, r in enumerate(rows) if any("Warp Stall Sampling (All" in c for c in r)), None)
    if hdr_i is None:
        print(f"== {view}: no stall columns ({out[:200]!r})")
        continue
    hdr = rows[hdr_i]
    col = next(i for i, c in enumerate(hdr) if "Warp Stall Sampling (All" in c)
    body = [r for r in rows[hdr_i + 1:] if len(r) > col]
    def val(r):
        try:
            return float(r[col].replace(",", ""))
        except ValueError:
            return 0.0
    tot = sum(val(r) for r in body) or 1.0
    print(f"== {view}: {len(body)} lines, total samples {tot:.0f}; columns: {hdr[:4]} ...")
    for r in sorted(body, key=val, reverse=True)[:top]:
        print(f"{100 * val(r) / tot:6.2f}%  " + " | ".join(c.strip()[:110] for c in r[:3]))
