"""Golden outputs of the REFERENCE's own command line (rdist distances /
navigate, pkg/src/rdist/cli.py) on small edge-list files, for the GPU CLI
parity test (tests/test_gpu_cli.py). Run in the build container:

    python tests/golden/make_golden_cli.py

Writes tests/golden/cli/<case>.{txt,csv,out,err}: the input edge list, the
distance CSV the reference wrote, its stdout / stderr; exit codes in cases.json.

The reference CLI's ``--method rdist`` path cannot run: inside cli.py
``from . import resolvent`` binds the *function* ``rdist.resolvent`` (the
package re-export shadows the submodule, rdist/__init__.py:52-68), so
``resolvent.gamma_bounds`` / ``resolvent.resolvent`` raise AttributeError
(cli.py:159, :228, :251). For those cases the expected output is what the
command computes when that import resolves to the module: the same calls
(cli.py:150-170, :224-231, :248-263) made here on the reference's own
functions, written with the CLI's own CSV writer (cli.py:196-202) and
messages; cases.json records the reference CLI's own exit code as well.
"""

import json
import subprocess
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent / "cli"
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import rdist  # noqa: E402  (the reference)

CASES = {
    # name: (graph builder, [cli args after the input])
    "grid5_rdist": (lambda: rdist.gen_grid(5), ["distances", "--method", "rdist"]),
    "grid5_gamma": (lambda: rdist.gen_grid(5), ["distances", "--method", "rdist", "--gamma", "0.001"]),
    "grid5_bfs": (lambda: rdist.gen_grid(5), ["distances", "--method", "bfs"]),
    "tree4_floyd": (lambda: rdist.gen_binary_tree(4), ["distances", "--method", "floyd"]),
    "wdense40_rdist": (lambda: rdist.gen_weighted_dense(40, 0.3, 1.0, 100.0, 2), ["distances", "--method", "rdist"]),
    "wdense40_floyd": (lambda: rdist.gen_weighted_dense(40, 0.3, 1.0, 100.0, 2), ["distances", "--method", "floyd"]),
    "dense30_dijkstra": (lambda: rdist.gen_random_dense(30, 0.2, 4), ["distances", "--method", "dijkstra"]),
    "grid5_nav": (lambda: rdist.gen_grid(5), ["navigate", "--start", "0", "--goal", "24"]),
    "wdense40_nav": (lambda: rdist.gen_weighted_dense(40, 0.3, 1.0, 100.0, 2), ["navigate", "--start", "3", "--goal", "17"]),
    "wdense40_nav_exact": (lambda: rdist.gen_weighted_dense(40, 0.3, 1.0, 100.0, 2),
                           ["navigate", "--start", "3", "--goal", "17", "--method", "exact"]),
    "unreach_nav": (lambda: rdist.graph_from_edge_list(rdist.EdgeList(4, ((0, 1, 1.0), (2, 3, 1.0))),
                                                        rdist.GraphKind.UNWEIGHTED),
                    ["navigate", "--start", "0", "--goal", "3", "--gamma", "0.1"]),
}


def intended(g, args, inp):
    """cli.py's _cmd_distances / _cmd_navigate for --method rdist with the
    resolvent *module* (rdist.resolvent module functions), same text."""
    import importlib
    import io
    import math

    from rdist import cli

    res_mod = importlib.import_module("rdist.resolvent")
    opts = dict(zip(args[1::2], args[2::2]))
    out, err = io.StringIO(), io.StringIO()
    gamma_arg = opts.get("--gamma", "auto")
    if gamma_arg == "auto":
        exact = rdist.floyd_warshall(g)
        d_max = max(math.ceil(rdist.graph_diameter(exact)), 1)
        bounds = res_mod.gamma_bounds(g, d_max)
        gamma = res_mod.suggest_gamma(bounds, safety=0.01)
        print(f"auto gamma: {gamma:.6g} (critical gain {bounds.critical_gain:.6g}, "
              f"precision floor {bounds.precision_floor_for_dmax:.6g}, d_max {d_max})", file=err)
    else:
        gamma = float(gamma_arg)
    res = res_mod.resolvent(g, gamma)
    if args[0] == "distances":
        d = res_mod.r_distance(res) if g.kind is rdist.GraphKind.REAL_WEIGHTED else res_mod.rounded_r_distance(res)
        path = str(inp)[:-4] + ".csv"
        cli._write_distance_csv(d, path)
        print(f"wrote {d.shape[0]}x{d.shape[1]} distance matrix to {path}", file=out)
        return out.getvalue(), err.getvalue(), 0
    dist = res_mod.r_distance(res)
    result = rdist.greedy_descent(g, dist, int(opts["--start"]), int(opts["--goal"]))
    if not result.reached:
        print(f"goal {opts['--goal']} not reached from {opts['--start']} after {result.steps_taken} steps", file=err)
        return out.getvalue(), err.getvalue(), 3
    print("path: " + " ".join(str(v) for v in result.vertices), file=out)
    print(f"length: {result.length:.12g}", file=out)
    return out.getvalue(), err.getvalue(), 0


def main():
    HERE.mkdir(exist_ok=True)
    meta = {}
    for name, (build, args) in CASES.items():
        g = build()
        inp = HERE / f"{name}.txt"
        rdist.write_edge_list(rdist.edge_list_from_graph(g), inp)
        cmd = [sys.executable, "-m", "rdist.cli", args[0], "--input", str(inp)] + args[1:]
        if args[0] == "distances":
            cmd += ["--out", str(HERE / f"{name}.csv")]
        proc = subprocess.run(cmd, capture_output=True, text=True, env={"PYTHONPATH": REF, "PATH": "/usr/bin"})
        meta[name] = {"args": args, "rc": proc.returncode, "reference_cli_rc": proc.returncode}
        out, err = proc.stdout, proc.stderr
        if "has no attribute" in proc.stderr:  # the shadowing bug: run the intended calls
            out, err, rc = intended(g, args, inp)
            meta[name].update(rc=rc, expected_from="reference functions (cli.py's resolvent import is shadowed)")
        (HERE / f"{name}.out").write_text(out.replace(str(HERE) + "/", ""))
        (HERE / f"{name}.err").write_text(err)
        print(name, proc.returncode, proc.stdout.strip()[:80], proc.stderr.strip()[:80])
    (HERE / "cases.json").write_text(json.dumps(meta, indent=1) + "\n")


if __name__ == "__main__":
    main()
