"""Command line for the hot path: ``distances`` and ``navigate``.

Mirrors the reference's ``rdist distances`` / ``rdist navigate``
(pkg/src/rdist/cli.py:88-104 parser, :133-160 graph loading and the 'auto'
gain, :196-265 the two commands): same flags, output text, CSV format
(cli.py:196-202) and exit codes (0 ok, 1 runtime failure, 2 usage, 3
unreachable goal). Every method runs on the GPU: ``rdist`` is the resolvent
pipeline (K1 -> K2 -> K3), ``bfs`` the all-source BFS (K8), ``floyd`` and
``dijkstra`` the exact weighted distances of the Floyd–Warshall kernel (K10;
on positive weights both name the same shortest-path lengths — exact on
integer weights, the reference's floyd_warshall bit for bit on real weights).
The 'auto' gain takes d_max from the exact GPU distances, as the reference
takes it from floyd_warshall. The reference's other subcommands (generate,
sweep, correlate, bench) and the analog navigation method are outside the
accelerated path.

    python -m paper_2308_07403_b200 distances --input g.txt --out d.csv
    python -m paper_2308_07403_b200 navigate --input g.txt --start 0 --goal 5
"""

from __future__ import annotations

import argparse
import math
import sys

EXIT_OK = 0
EXIT_FAILURE = 1
EXIT_USAGE = 2
EXIT_UNREACHABLE = 3


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="rdist", description="Shortest-path distances from a single matrix inversion.")
    sub = parser.add_subparsers(dest="command", required=True)

    dist = sub.add_parser("distances", help="write a distance matrix as CSV")
    dist.add_argument("--input", "--in", dest="input", required=True)
    dist.add_argument("--method", choices=["rdist", "floyd", "dijkstra", "bfs"], default="rdist")
    dist.add_argument("--gamma", default="auto", help="'auto' or a float in (0,1)")
    dist.add_argument("--safety", type=float, default=0.01)
    dist.add_argument("--kind", choices=["auto", "unweighted", "integer", "real"], default="auto")
    dist.add_argument("--out", required=True)

    nav = sub.add_parser("navigate", help="greedy path from start to goal")
    nav.add_argument("--input", "--in", dest="input", required=True)
    nav.add_argument("--start", type=int, required=True)
    nav.add_argument("--goal", type=int, required=True)
    nav.add_argument("--method", choices=["rdist", "exact", "analog"], default="rdist")
    nav.add_argument("--gamma", default="auto")
    nav.add_argument("--safety", type=float, default=0.01)
    nav.add_argument("--kind", choices=["auto", "unweighted", "integer", "real"], default="auto")
    return parser


def _load_graph(path: str, kind_name: str):
    from . import graphs

    edges = graphs.read_edge_list(path)
    if kind_name == "auto":
        kind = graphs.infer_kind(edges)
    else:
        kind = {"unweighted": graphs.GraphKind.UNWEIGHTED, "integer": graphs.GraphKind.INTEGER_WEIGHTED,
                "real": graphs.GraphKind.REAL_WEIGHTED}[kind_name]
    return graphs.graph_from_edge_list(edges, kind)


def _exact(g):
    """Exact distances on the device: BFS for unweighted graphs, else Floyd–Warshall."""
    from . import oracles
    from .graphs import kind_value

    return oracles.bfs_apsp(g) if kind_value(g) == "unweighted" else oracles.floyd_warshall(g)


def _resolve_gamma(g, gamma_arg: str, safety: float) -> float:
    """A literal gain, or 'auto': d_max from the exact distances, then
    gamma_bounds / suggest_gamma (cli.py:133-160); exits 1 when infeasible."""
    # (the resolvent *module*: the package re-export `resolvent` is the function,
    # which is why the reference's own `from . import resolvent` fails here)
    from . import oracles
    from .resolvent import gamma_bounds, suggest_gamma

    if gamma_arg != "auto":
        return float(gamma_arg)
    d_max = max(math.ceil(oracles.graph_diameter(_exact(g))), 1)
    bounds = gamma_bounds(g, d_max)
    if not bounds.feasible:
        raise SystemExit(
            f"error: no valid gamma exists: the precision floor "
            f"{bounds.precision_floor_for_dmax:.6g} for diameter {d_max} meets or "
            f"exceeds the critical gain {bounds.critical_gain:.6g}; the longest "
            f"distance must stay below {bounds.max_feasible_distance:.1f}"
        )
    gamma = suggest_gamma(bounds, safety=safety)
    print(f"auto gamma: {gamma:.6g} (critical gain {bounds.critical_gain:.6g}, "
          f"precision floor {bounds.precision_floor_for_dmax:.6g}, d_max {d_max})", file=sys.stderr)
    return gamma


def _cmd_distances(args) -> int:
    from . import graphs, oracles
    from .resolvent import r_distance, resolvent, rounded_r_distance

    g = _load_graph(args.input, args.kind)
    if args.method == "bfs":
        d = oracles.bfs_apsp(g)
    elif args.method in ("floyd", "dijkstra"):
        d = oracles.floyd_warshall(g)
    else:
        gamma = _resolve_gamma(g, args.gamma, args.safety)
        res = resolvent(g, gamma)
        d = r_distance(res) if g.kind is graphs.GraphKind.REAL_WEIGHTED else rounded_r_distance(res)
    graphs.write_distance_csv(d, args.out)
    print(f"wrote {d.shape[0]}x{d.shape[1]} distance matrix to {args.out}")
    return EXIT_OK


def _cmd_navigate(args) -> int:
    from . import navigation
    from .resolvent import r_distance, resolvent

    g = _load_graph(args.input, args.kind)
    if args.method == "analog":
        print("error: the analog network method is not part of the accelerated path", file=sys.stderr)
        return EXIT_USAGE
    if args.method == "rdist":
        gamma = _resolve_gamma(g, args.gamma, args.safety)
        dist = r_distance(resolvent(g, gamma))
    else:
        dist = _exact(g)
    result = navigation.greedy_descent(g, dist, args.start, args.goal)
    if not result.reached:
        print(f"goal {args.goal} not reached from {args.start} after {result.steps_taken} steps", file=sys.stderr)
        return EXIT_UNREACHABLE
    print("path: " + " ".join(str(v) for v in result.vertices))
    print(f"length: {result.length:.12g}")
    return EXIT_OK


def main(argv: list[str] | None = None) -> int:
    parser = build_parser()
    args = parser.parse_args(argv)
    handlers = {"distances": _cmd_distances, "navigate": _cmd_navigate}
    try:
        return handlers[args.command](args)
    except SystemExit as exc:
        if isinstance(exc.code, str):
            print(exc.code, file=sys.stderr)
            return EXIT_FAILURE
        raise
    except (OSError, ValueError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_FAILURE


if __name__ == "__main__":
    sys.exit(main())
