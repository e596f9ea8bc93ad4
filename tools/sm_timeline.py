"""Per-SM busy timeline of one config-2 K2 call (where SMs sit idle between
the launches of the concurrent sub-batch / look-ahead streams).

Needs the diagnostic build (every warp of the K2 kernels logs globaltimer at
entry and exit, its SM id and a kernel kind into a per-SM segment of a buffer;
common.cuh RDB_TRACE_SCOPE):
    make BUILD=build_trace LIB=tools/_var/lib_trace.so EXTRA=-DRDB_TRACE
usage: python tools/sm_timeline.py [tools/_var/lib_trace.so] [--out f.json]
Prints SM utilisation over the call (union of warp intervals per SM / (SMs x
wall)), SM-time per kernel kind, and a coarse busy-SM count per time bin.
"""

import argparse
import ctypes
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2308_07403_b200 import _lib as L  # noqa: E402
from paper_2308_07403_b200 import batch as B  # noqa: E402
from paper_2308_07403_b200 import workloads as wl  # noqa: E402

KINDS = {0: "P1 plan", 1: "P1 nested (DW band)", 5: "P1 band path", 2: "rowpanel NB128", 3: "update NB128",
         4: "DW row panel", 10: "DW update (all)", 11: "DW update (next band 2x2)", 12: "DW update (rest)",
         8: "wide row", 9: "wide update", 20: "local gemm", 30: "plan walk", 33: "DW sparse step-0 gather", 31: "plan scan", 32: "dw classify",
         14: "W2 outer row panel", 15: "W2 outer update", 50: "K3 log_ceil", 51: "K1 build_m_bits", 6: "DW sparse step-0 row panel", 7: "DW sparse step-0 update", 40: "band factor", 41: "band chain", 42: "band detect"}
REC = np.dtype([("t0", "<u8"), ("t1", "<u8"), ("sm", "<i4"), ("kind", "<i4")])


def union_len(iv):
    """Total length of the union of [t0, t1) intervals (sorted by t0)."""
    tot, cur0, cur1 = 0, None, None
    for a, b in iv:
        if cur1 is None or a > cur1:
            if cur1 is not None:
                tot += cur1 - cur0
            cur0, cur1 = a, b
        else:
            cur1 = max(cur1, b)
    if cur1 is not None:
        tot += cur1 - cur0
    return tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("lib", nargs="?", default="tools/_var/lib_trace.so")
    ap.add_argument("--out", default=None)
    ap.add_argument("--bin-us", type=float, default=25.0)
    ap.add_argument("--full", action="store_true", help="trace the whole K1 -> K2 -> K3 call")
    ap.add_argument("--reps", type=int, default=1, help="traced calls (summary of each; the last is kept)")
    a = ap.parse_args()
    lib = L.load_library(a.lib)
    L._lib = lib
    lib.rdb_trace_attach.argtypes = [ctypes.c_void_p, ctypes.c_uint]
    lib.rdb_trace_counts.argtypes = [ctypes.POINTER(ctypes.c_uint)]
    dev = torch.device("cuda", 0)
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    bits, gammas, _ = wl.cfg2_batch(256)
    buf = B.BatchBuffers.allocate(1024, 256, dev)
    buf.bits.copy_(torch.from_numpy(bits.view(np.int32)))
    buf.gammas.copy_(torch.from_numpy(gammas))
    sh = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        B.run_chunk(buf, 256, sh)
    torch.cuda.synchronize()
    cap = 1 << 24
    tbuf = torch.zeros(cap * REC.itemsize, dtype=torch.uint8, device=dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for rep in range(a.reps):
        buf.stage_build(256, sh)
        torch.cuda.synchronize()
        L.check(lib.rdb_trace_attach(tbuf.data_ptr(), cap), "trace_attach")
        ev[0].record()
        if a.full:
            B.run_chunk(buf, 256, sh)
        else:
            buf.stage_invert(256, sh)
        ev[1].record()
        torch.cuda.synchronize()
        call_ms = ev[0].elapsed_time(ev[1])
        cnt = (ctypes.c_uint * 2)()
        lib.rdb_trace_counts(cnt)
        raw = tbuf.cpu().numpy().view(REC)
        recs = raw[raw["t1"] != 0]  # per-SM segments, unused slots zero
        tbuf.zero_()
        L.check(lib.rdb_trace_attach(None, 0), "trace_detach")
        t_lo, t_hi = int(recs["t0"].min()), int(recs["t1"].max())
        per_sm_n = np.bincount(recs["sm"], minlength=nsm)
        print(json.dumps({"segment_capacity": cap // 4 // 192, "records_per_sm_max": int(per_sm_n.max()),
                          "records_per_sm_min": int(per_sm_n.min()), "trace_counts": [int(cnt[0]), int(cnt[1])]}),
              flush=True)
        wall = t_hi - t_lo
        busy = 0
        per_sm = {}
        for sm in np.unique(recs["sm"]):
            r = recs[recs["sm"] == sm]
            o = np.argsort(r["t0"])
            iv = list(zip(r["t0"][o].tolist(), r["t1"][o].tolist()))
            per_sm[int(sm)] = union_len(iv)
            busy += per_sm[int(sm)]
        kinds = {}
        for k in np.unique(recs["kind"]):
            rk = recs[recs["kind"] == k]
            tot = 0
            for sm in np.unique(rk["sm"]):
                r = rk[rk["sm"] == sm]
                o = np.argsort(r["t0"])
                tot += union_len(list(zip(r["t0"][o].tolist(), r["t1"][o].tolist())))
            kinds[KINDS.get(int(k), str(int(k)))] = {"sm_ms": tot / 1e6, "share_of_sm_time": tot / (nsm * wall),
                                                     "warp_records": int(rk.size)}
        # busy SMs per bin (an SM counts for the part of the bin it is busy)
        nb = int(np.ceil(wall / (a.bin_us * 1e3)))
        occ = np.zeros(nb)
        edges = t_lo + np.arange(nb + 1) * a.bin_us * 1e3
        for sm in np.unique(recs["sm"]):
            r = recs[recs["sm"] == sm]
            o = np.argsort(r["t0"])
            cur0 = cur1 = None
            merged = []
            for x, y in zip(r["t0"][o].tolist(), r["t1"][o].tolist()):
                if cur1 is None or x > cur1:
                    if cur1 is not None:
                        merged.append((cur0, cur1))
                    cur0, cur1 = x, y
                else:
                    cur1 = max(cur1, y)
            merged.append((cur0, cur1))
            for x, y in merged:
                i0 = int((x - t_lo) // (a.bin_us * 1e3))
                i1 = min(int((y - t_lo) // (a.bin_us * 1e3)), nb - 1)
                for i in range(i0, i1 + 1):
                    ov = min(y, edges[i + 1]) - max(x, edges[i])
                    if ov > 0:
                        occ[i] += ov / (a.bin_us * 1e3)
        out = {
            "call_ms_events": call_ms,
            "traced_wall_ms": wall / 1e6,
            "sms": nsm,
            "sm_utilisation": busy / (nsm * wall),
            "idle_sm_ms": (nsm * wall - busy) / 1e6,
            "records": int(recs.size),
            "kinds": dict(sorted(kinds.items(), key=lambda kv: -kv[1]["sm_ms"])),
            "bin_us": a.bin_us,
            "busy_sms_per_bin": [round(float(x), 1) for x in occ],
        }
        print(json.dumps({k: out[k] for k in ("call_ms_events", "traced_wall_ms", "sm_utilisation", "idle_sm_ms")}),
              flush=True)
    print(json.dumps({k: v for k, v in out.items() if k != "busy_sms_per_bin"}, indent=1))
    lo = [(i, round(float(x), 1)) for i, x in enumerate(occ) if x < 0.85 * nsm]
    print("bins below 85% busy (index, busy SMs):", lo[:200])
    # what runs in those bins: SMs per kernel kind active in the bin
    low = {}
    for i, _ in lo:
        b0, b1 = edges[i], edges[i + 1]
        act = recs[(recs["t0"] < b1) & (recs["t1"] > b0)]
        low[i] = {KINDS.get(int(k), str(int(k))): int(np.unique(act["sm"][act["kind"] == k]).size)
                  for k in np.unique(act["kind"])}
        print(f"  bin {i} ({(b0 - t_lo) / 1e3:.0f} us): {low[i]}")
    out["low_bins"] = low
    # every bin: SMs per kind (kinds with at least 8 SMs)
    allb = []
    for i in range(nb):
        b0, b1 = edges[i], edges[i + 1]
        act = recs[(recs["t0"] < b1) & (recs["t1"] > b0)]
        d = {KINDS.get(int(k), str(int(k))): int(np.unique(act["sm"][act["kind"] == k]).size)
             for k in np.unique(act["kind"])}
        allb.append({k: v for k, v in d.items() if v >= 8})
    out["bins_kinds"] = allb
    if a.out:
        Path(a.out).write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
