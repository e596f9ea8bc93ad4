"""A/B timing of the batched K2 (config-2 batch of 256) under scheduling knobs
read per call from the environment (csrc/gj_invert.cu): the co-scheduling grid
cap, dynamic tile tickets, the sub-batch split. D must stay bitwise identical.

usage: python tools/k2_modes.py [--out gpurun_out/k2_modes.json]
"""

import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2308_07403_b200 import _lib as L  # noqa: E402
from paper_2308_07403_b200 import batch as B  # noqa: E402
from paper_2308_07403_b200 import workloads as wl  # noqa: E402

MODES = {
    "default": {},
    "static_capped": {"RDB_GJ_DYNAMIC": "0"},
    "static_uncapped": {"RDB_GJ_DYNAMIC": "0", "RDB_GJ_COSCHED": "0"},
    "no_dense_wide": {"RDB_GJ_DW": "0"},
    "dw_no_lookahead": {"RDB_GJ_DW_LA": "0"},
    "dw_la_reserve8": {"RDB_GJ_DW_LA_RESERVE": "8"},
    "dw_la_reserve24": {"RDB_GJ_DW_LA_RESERVE": "24"},
    "dw_la_reserve48": {"RDB_GJ_DW_LA_RESERVE": "48"},
    "dw_la_reserve64": {"RDB_GJ_DW_LA_RESERVE": "64"},
    "dw_la_reserve80": {"RDB_GJ_DW_LA_RESERVE": "80"},
    "dw_la_reserve100": {"RDB_GJ_DW_LA_RESERVE": "100"},
    "dw_no_helper": {"RDB_GJ_DW_HELPER": "0"},
    "dw_no_s0": {"RDB_GJ_DW_S0": "0"},
    "no_synth": {"RDB_GJ_DW_SYNTH": "0"},
    "no_dw2": {"RDB_GJ_DW2": "0"},
    "dw_helper_reserve32": {"RDB_GJ_DW_LA_RESERVE": "32"},
    "dw_helper_reserve80": {"RDB_GJ_DW_LA_RESERVE": "80"},
    "dw_helper_reserve100": {"RDB_GJ_DW_LA_RESERVE": "100"},
    "dw_helper_reserve90": {"RDB_GJ_DW_LA_RESERVE": "90"},
    "dw_helper_reserve106": {"RDB_GJ_DW_LA_RESERVE": "106"},
    "dw_helper_reserve120": {"RDB_GJ_DW_LA_RESERVE": "120"},
    "no_split": {"RDB_GJ_SPLIT_MIN": "0"},
    "no_split_no_dw": {"RDB_GJ_SPLIT_MIN": "0", "RDB_GJ_DW": "0"},
    "split3_capped": {"RDB_GJ_SPLIT_PARTS": "3"},
    "split4": {"RDB_GJ_SPLIT_PARTS": "4"},
    "reserve40": {"RDB_GJ_DW_LA_RESERVE": "40"},
    "reserve56": {"RDB_GJ_DW_LA_RESERVE": "56"},
    "reserve72": {"RDB_GJ_DW_LA_RESERVE": "72"},
    "split3_reserve48": {"RDB_GJ_SPLIT_PARTS": "3", "RDB_GJ_DW_LA_RESERVE": "48"},
}
KNOBS = ("RDB_GJ_LA_SIDE", "RDB_GJ_WIDE_MIN", "RDB_GJ_COSCHED", "RDB_GJ_DYNAMIC", "RDB_GJ_SPLIT_MIN", "RDB_GJ_SPLIT_PARTS", "RDB_GJ_DW", "RDB_GJ_DW_LA", "RDB_GJ_DW_LA_RESERVE", "RDB_GJ_DW_HELPER", "RDB_GJ_DW_S0", "RDB_GJ_DW_SYNTH", "RDB_GJ_DW2")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--reps", type=int, default=9)
    ap.add_argument("--modes", default=",".join(MODES))
    ap.add_argument("--single", default="2048,4096")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    L.load_library()
    bits, gammas, _ = wl.cfg2_batch(256)
    buf = B.BatchBuffers.allocate(1024, 256, dev)
    buf.bits.copy_(torch.from_numpy(bits.view(np.int32)))
    buf.gammas.copy_(torch.from_numpy(gammas))
    sh = torch.cuda.current_stream().cuda_stream
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ref_d = None
    out = []
    for name in args.modes.split(","):
        for k in KNOBS:
            os.environ.pop(k, None)
        os.environ.update(MODES[name])
        for _ in range(2):
            B.run_chunk(buf, 256, sh)
        torch.cuda.synchronize()
        if ref_d is None:
            ref_d = buf.d.clone()
        same = bool(torch.equal(ref_d, buf.d))
        ts, tstep = [], []
        for _ in range(args.reps):
            buf.stage_build(256, sh)
            ev[0].record()
            buf.stage_invert(256, sh)
            ev[1].record()
            torch.cuda.synchronize()
            ts.append(ev[0].elapsed_time(ev[1]))
            ev[2].record()
            B.run_chunk(buf, 256, sh)
            ev[3].record()
            torch.cuda.synchronize()
            tstep.append(ev[2].elapsed_time(ev[3]))
        rec = {"mode": name, "env": MODES[name], "k2_ms_median": float(np.median(ts)), "k2_ms_min": float(np.min(ts)),
               "step_ms_median": float(np.median(tstep)), "d_identical_to_default": same}
        print(json.dumps(rec), flush=True)
        out.append(rec)
    # single-matrix look-ahead path (configs 1 and 4): ticketed vs static update tiles
    for n in (int(x) for x in args.single.split(",") if x):
        gen = torch.Generator(device=dev).manual_seed(7)
        m0 = (torch.rand((n, n), generator=gen, device=dev) < 0.1).to(torch.float64).mul_(-1e-3)
        m0.diagonal().fill_(1.0)
        m1 = m0.clone()
        work = torch.empty(L.lib().rdb_invert_workspace_bytes(n, 1), dtype=torch.uint8, device=dev)
        info = L.pivot_info_tensor(1, dev)
        ref = None
        for name, env in (("default", {}), ("diag_lookahead", {"RDB_GJ_LA_SIDE": "0"}),
                          ("row_lookahead_8", {"RDB_GJ_LA_SIDE": "8"}), ("row_lookahead_24", {"RDB_GJ_LA_SIDE": "24"}),
                          ("row_lookahead_32", {"RDB_GJ_LA_SIDE": "32"}), ("static", {"RDB_GJ_DYNAMIC": "0"})):
            for k in KNOBS:
                os.environ.pop(k, None)
            os.environ.update(env)
            work = torch.empty(L.lib().rdb_invert_workspace_bytes(n, 1), dtype=torch.uint8, device=dev)
            ts = []
            for _ in range(args.reps):
                m1.copy_(m0)
                ev[0].record()
                L.check(L.lib().rdb_invert(m1.data_ptr(), n, n, work.data_ptr(), info.data_ptr(), sh), "invert")
                ev[1].record()
                torch.cuda.synchronize()
                ts.append(ev[0].elapsed_time(ev[1]))
            if ref is None:
                ref = m1.clone()
            rec = {"single_n": n, "mode": name, "ms_median": float(np.median(ts)),
                   "tflops": 2.0 * n**3 / (float(np.median(ts)) * 1e-3) / 1e12,
                   "y_identical": bool(torch.equal(ref, m1))}
            print(json.dumps(rec), flush=True)
            out.append(rec)
    if args.out:
        Path(args.out).write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
