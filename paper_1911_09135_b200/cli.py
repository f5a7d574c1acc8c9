"""Command line over the B200 engine: one run, a scheduler comparison with a
label-equality check, and a huge-vertex threshold sweep.

Mirrors the reference CLI's three commands (`cli.py:173-290`: `run`,
`compare`, `sweep-threshold`), their options and report files, so scripts
written against ``simtgraph`` keep working:

    python -m paper_1911_09135_b200.cli compare --format rmat --scale 20 --app bfs \\
        --schedulers twc,alb,lb --out-dir reports
    python -m paper_1911_09135_b200.cli sweep-threshold --format rmat --scale 20 \\
        --app sssp --thresholds 256,4096,auto,inf

Every run goes through ``engine.run_app`` (the whole BSP loop on the device).
Exit codes as the reference: 0 success, 1 label mismatch or backend failure,
2 usage / configuration error.  Labels are compared exactly, pr within the
reference's cross-scheduler tolerance (`cli.py:25`); on this device pr sums
are bit-exact, so pr labels agree exactly too except under the blocked LB
distribution.
"""

from __future__ import annotations

import argparse
import csv
import sys
from pathlib import Path

import numpy as np

from . import engine
from .errors import ConfigError, ParseError, RangeError, SimtGraphError
from .graph import RMAT_SKEWED, attach_random_weights, generate_rmat, load_graph
from .schedulers import Scheduler
from .simt import KernelConfig

PR_LABEL_ATOL = 1e-7
INT64_MAX = np.iinfo(np.int64).max


def _threshold(text):
    """'auto' -> None (the launched thread count), 'inf' -> no huge bin, else an int."""
    if text is None or text == "auto":
        return None
    if text in ("inf", "+inf"):
        return INT64_MAX
    try:
        return int(text)
    except ValueError:
        raise ConfigError(f"threshold must be an integer, 'auto', or 'inf', got {text!r}")


def scheduler_of(token: str, distribution=None, threshold=None) -> Scheduler:
    """``alb``, ``alb-blocked``, ``lb-cyclic``, ``twc`` ... (kind[-distribution])."""
    kind, _, dist = token.partition("-")
    if dist and dist not in ("cyclic", "blocked"):
        raise ConfigError(f"bad scheduler token {token!r}")
    return Scheduler(kind=kind, distribution=dist or distribution or None,
                     threshold=_threshold(threshold))


def build_graph(a):
    if a.input == "rmat" or a.format == "rmat":
        probs = tuple(float(x) for x in a.rmat_probs.split(","))
        g = generate_rmat(a.scale, a.edge_factor, a.seed, probs)
        if a.app == "sssp" and a.weights:
            g = attach_random_weights(g, a.seed + 1, 1, a.weights)
    elif a.input:
        g = load_graph(a.input, a.format or None)
    else:
        raise ConfigError("no input: pass --input PATH or --format rmat")
    if a.symmetrize:
        g = g.symmetrized()
    return g


def run_one(a, graph, sched: Scheduler):
    config = KernelConfig(a.cta, a.tpb, a.warp)
    res = engine.run_app(graph, a.app, sched, config, devices=a.devices,
                         max_rounds=a.max_rounds or None, source=a.source, k=a.k,
                         damping=a.damping, tol=a.tol)
    res.spec = {k: v for k, v in vars(a).items() if k != "func"}
    return res


def labels_equal(app, x, y) -> bool:
    if app == "pr":
        return bool(np.allclose(x, y, rtol=0.0, atol=PR_LABEL_ATOL))
    return bool(np.array_equal(x, y))


def _write_csv(path: Path, rows):
    path.parent.mkdir(parents=True, exist_ok=True)
    with open(path, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=list(rows[0]))
        w.writeheader()
        w.writerows(rows)


def cmd_run(a):
    graph = build_graph(a)
    sched = scheduler_of(a.scheduler, a.distribution, a.threshold)
    res = run_one(a, graph, sched)
    name = f"{a.app}_{sched.describe()}"
    paths = engine.write_reports(res, a.out_dir, name)
    s = engine.report(res)
    print(f"{a.app} {sched.describe()} rounds={s['rounds']} "
          f"edges={s['totals']['edges_processed']} "
          f"lb_launches={s['totals']['kernel_launches'].get('lb', 0)} "
          f"device_ms={res.device_ms:.3f} -> {paths['summary']}")
    return 0


def cmd_compare(a):
    tokens = [t.strip() for t in a.schedulers.split(",") if t.strip()]
    if not tokens:
        raise ConfigError("empty scheduler list")
    graph = build_graph(a)
    rows, results = [], []
    for tok in tokens:
        sched = scheduler_of(tok, a.distribution, a.threshold)
        res = run_one(a, graph, sched)
        s = engine.report(res)
        results.append((tok, res))
        rows.append({"scheduler": sched.describe(), "rounds": s["rounds"],
                     "edges": s["totals"]["edges_processed"],
                     "lb_launches": s["totals"]["kernel_launches"].get("lb", 0),
                     "device_ms": round(res.device_ms, 4),
                     "gteps": round(s["totals"]["edges_processed"] / max(res.device_ms, 1e-9) / 1e6, 3)})
        engine.write_reports(res, a.out_dir, f"{a.app}_{sched.describe()}")
    table = Path(a.out_dir) / f"{a.app}_compare.csv"
    _write_csv(table, rows)
    print(f"{'scheduler':<18}{'rounds':>7}{'edges':>13}{'lb':>5}{'ms':>10}{'GTEPS':>9}")
    for r in rows:
        print(f"{r['scheduler']:<18}{r['rounds']:>7}{r['edges']:>13}{r['lb_launches']:>5}"
              f"{r['device_ms']:>10.3f}{r['gteps']:>9.2f}")
    base_tok, base = results[0]
    for tok, other in results[1:]:
        if not labels_equal(a.app, base.labels, other.labels):
            diff = np.flatnonzero(base.labels != other.labels)[:10]
            print(f"label mismatch: {base_tok} vs {tok} at vertices {diff.tolist()}",
                  file=sys.stderr)
            return 1
    print(f"labels identical across {len(results)} schedulers -> {table}")
    return 0


def cmd_sweep(a):
    values = [t.strip() for t in a.thresholds.split(",") if t.strip()]
    if not values:
        raise ConfigError("empty threshold list")
    graph = build_graph(a)
    rows, first = [], None
    for text in values:
        sched = scheduler_of("alb", a.distribution, text)
        res = run_one(a, graph, sched)
        s = engine.report(res)
        if first is None:
            first = res
        elif not labels_equal(a.app, first.labels, res.labels):
            print(f"label mismatch at threshold {text}", file=sys.stderr)
            return 1
        rows.append({"threshold": text, "rounds": s["rounds"],
                     "lb_launches": s["totals"]["kernel_launches"].get("lb", 0),
                     "device_ms": round(res.device_ms, 4),
                     "gteps": round(s["totals"]["edges_processed"] / max(res.device_ms, 1e-9) / 1e6, 3)})
    path = Path(a.out_dir) / f"{a.app}_threshold_sweep.csv"
    _write_csv(path, rows)
    print(f"{'threshold':>10}{'rounds':>7}{'lb':>5}{'ms':>10}{'GTEPS':>9}")
    for r in rows:
        print(f"{r['threshold']:>10}{r['rounds']:>7}{r['lb_launches']:>5}{r['device_ms']:>10.3f}"
              f"{r['gteps']:>9.2f}")
    print(f"-> {path}")
    return 0


def parser() -> argparse.ArgumentParser:
    common = argparse.ArgumentParser(add_help=False)
    common.add_argument("--input", default="", help="graph path, or 'rmat'")
    common.add_argument("--format", default="", choices=["", "el", "wel", "bin", "rmat"])
    common.add_argument("--scale", type=int, default=14)
    common.add_argument("--edge-factor", type=int, default=16)
    common.add_argument("--rmat-probs", default=",".join(str(p) for p in RMAT_SKEWED))
    common.add_argument("--symmetrize", action="store_true")
    common.add_argument("--app", default="bfs", choices=["bfs", "sssp", "cc", "pr", "kcore"])
    common.add_argument("--source", type=int, default=0)
    common.add_argument("--k", type=int, default=2)
    common.add_argument("--damping", type=float, default=0.85)
    common.add_argument("--tol", type=float, default=1e-6)
    common.add_argument("--distribution", default="", choices=["", "cyclic", "blocked"])
    common.add_argument("--threshold", default="auto")
    common.add_argument("--cta", type=int, default=KernelConfig().num_ctas)
    common.add_argument("--tpb", type=int, default=KernelConfig().threads_per_cta)
    common.add_argument("--warp", type=int, default=KernelConfig().warp_size)
    common.add_argument("--devices", type=int, default=1)
    common.add_argument("--seed", type=int, default=1)
    common.add_argument("--weights", type=int, default=0,
                        help="rmat sssp: attach integer weights in [1, W] (seed + 1); "
                             "0 = unweighted, as the reference CLI")
    common.add_argument("--max-rounds", type=int, default=0)
    common.add_argument("--out-dir", default="reports")
    p = argparse.ArgumentParser(prog="simtgraph-b200", description=__doc__.splitlines()[0])
    sub = p.add_subparsers(dest="command", required=True)
    r = sub.add_parser("run", parents=[common], help="one run, reports written")
    r.add_argument("--scheduler", default="alb")
    r.set_defaults(func=cmd_run)
    c = sub.add_parser("compare", parents=[common], help="several schedulers, labels must agree")
    c.add_argument("--schedulers", default="twc,alb")
    c.set_defaults(func=cmd_compare)
    s = sub.add_parser("sweep-threshold", parents=[common], help="alb across thresholds")
    s.add_argument("--thresholds", default="256,512,1024,2048,4096")
    s.set_defaults(func=cmd_sweep)
    return p


def main(argv=None) -> int:
    try:
        a = parser().parse_args(argv)
    except SystemExit as e:  # argparse usage errors
        return 2 if e.code else 0
    a.distribution = a.distribution or None
    try:
        return a.func(a)
    except (ConfigError, ParseError, RangeError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    except SimtGraphError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
