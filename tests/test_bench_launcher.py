"""bench.py's multi-GPU launcher on CPU: `--gpus 2` outside torch.distributed
re-launches itself under torch.distributed.run with two ranks (gloo here, the
launch probe hook); each rank sees WORLD_SIZE == --gpus and the max-over-ranks
reduction the bench uses for its timings."""

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_bench_self_launches_n_ranks():
    env = dict(os.environ, RDB_BENCH_LAUNCH_PROBE="1")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2"], env=env, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    # the two ranks print concurrently (lines may interleave): decode every object in the stream
    dec, lines, pos, text = json.JSONDecoder(), [], 0, out.stdout
    while (pos := text.find("{", pos)) >= 0:
        obj, end = dec.raw_decode(text, pos)
        lines.append(obj)
        pos = end
    assert sorted(x["rank"] for x in lines) == [0, 1]
    assert all(x["world"] == 2 and x["max_rank"] == 1.0 and x["local_world"] == 2 for x in lines)


def test_bench_rejects_world_mismatch():
    env = dict(os.environ, RDB_BENCH_LAUNCH_PROBE="1", WORLD_SIZE="1", RANK="0", LOCAL_RANK="0",
               MASTER_ADDR="127.0.0.1", MASTER_PORT="29555")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2"], env=env, capture_output=True,
                         text=True, timeout=120)
    assert out.returncode != 0 and "WORLD_SIZE=1" in out.stderr
