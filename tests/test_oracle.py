"""CPU: pin the oracle (numpy + C restatements) to the reference's golden
vectors before trusting it as the GPU checker.  No GPU needed."""

from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle_c as C
from oracle import oracle_np as O

GOLDEN = Path(__file__).parent / "golden"
SMALL = ("rmat10", "uniform10", "rmat12", "rmat14")


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _graph(name):
    kind, scale = name[:-2], int(name[-2:])
    return O.rmat_csr(scale, 16, 1, O.SKEWED if kind == "rmat" else (0.25,) * 4)


def _golden():
    return json.loads((GOLDEN / "golden.json").read_text())


def _cases(names):
    g = _golden()
    out = []
    for name in names:
        for key in g["runs"][name]:
            if key != "graph":
                out.append((name, key))
    return out


@pytest.mark.parametrize("name", ["rmat10", "uniform10", "rmat12", "rmat14", "rmat16", "uniform16"])
def test_generator_and_views(name, golden):
    ref = golden["runs"][name]["graph"]
    off, tgt = _graph(name)
    assert _sha(off) == ref["offsets_sha256"] and _sha(tgt) == ref["targets_sha256"]
    assert _sha(O.transpose(off, tgt)[1]) == ref["csc_targets_sha256"]
    soff, stgt, _ = O.symmetrize(off, tgt)
    assert _sha(soff) == ref["sym_offsets_sha256"] and _sha(stgt) == ref["sym_targets_sha256"]
    assert _sha(O.random_weights(len(tgt), 2)) == ref["weights_sha256"]


@pytest.mark.parametrize("name,key", _cases(SMALL))
def test_numpy_oracle_run_level(name, key, golden):
    info = golden["runs"][name][key]
    app, sched, d = key.split("/")
    kind = sched.split("-")[0]
    thr = int(sched.split("-t")[1]) if "-t" in sched else None
    off, tgt = _graph(name)
    w = O.random_weights(len(tgt), 2) if app == "sssp" else None
    lab, log = O.run_graph(off, tgt, w, app, kind=kind, threshold=thr, blocked=(kind == "lb"),
                           devices=int(d[1:]))
    assert O.labels_sha256(lab) == info["labels_sha256"]
    assert [r.as_list() for r in log] == info["per_round"]


@pytest.mark.parametrize("name", ["rmat10", "uniform10", "rmat12", "rmat14", "rmat16", "uniform16"])
@pytest.mark.parametrize("app", ["bfs", "sssp", "cc", "pr", "kcore"])
@pytest.mark.parametrize("threads", [1, 4])
def test_c_oracle_bit_exact(name, app, threads, golden):
    """Including pr: per-row sequential sums reproduce np.add.at bit for bit."""
    info = golden["runs"][name][f"{app}/alb/d1"]
    off, tgt = _graph(name)
    w = O.random_weights(len(tgt), 2) if app == "sssp" else None
    lab, log, st = C.run(app, *C.prepare(off, tgt, w, app), threads=threads)
    assert st == 0
    assert O.labels_sha256(lab) == info["labels_sha256"]
    assert log.tolist() == [r[:2] for r in info["per_round"]]


def test_c_generator_matches_numpy():
    for scale, probs in ((9, O.SKEWED), (11, (0.25,) * 4), (12, (0.45, 0.15, 0.15, 0.25))):
        s, d = C.rmat_pairs(scale, 16, 1, probs, threads=3)
        s2, d2, _ = O.rmat_pairs(scale, 16, 1, probs)
        assert np.array_equal(s, s2) and np.array_equal(d, d2)
        off, tgt, _ = C.csr_from_pairs(s, d, 1 << scale)
        off2, tgt2, _ = O.csr_from_pairs(s2, d2, None, 1 << scale)
        assert np.array_equal(off, off2) and np.array_equal(tgt, tgt2)


def _kernel_fixtures():
    z = np.load(GOLDEN / "kernels_small.npz")
    return z, int(z["count"])


@pytest.fixture(scope="module")
def views():
    off, tgt = O.rmat_csr(10)
    w = O.random_weights(len(tgt), 2).astype(np.float64)
    soff, stgt, _ = O.symmetrize(off, tgt)
    return {"bfs": (off, tgt, np.empty(0)), "sssp": (off, tgt, w),
            "cc": (soff, stgt, np.empty(0)), "pr": (*O.transpose(off, tgt)[:2], np.empty(0)),
            "kcore": (*O.transpose(soff, stgt)[:2], np.empty(0))}


@pytest.mark.parametrize("i", range(_kernel_fixtures()[1]))
def test_numpy_oracle_kernel_level(i, views):
    """Oracle kernels == the reference's lb/twc/vertex/edge kernel outputs."""
    z, _ = _kernel_fixtures()
    p = f"k{i}_"
    kind, app = str(z[p + "kind"]), str(z[p + "app"])
    ctas, tpb, ws = (int(x) for x in z["config"])
    off, tgt, w = views[app]
    values, aux, op = z[p + "values"], z[p + "aux"], int(z[p + "opcode"])
    out = values.copy() if op != 3 else np.zeros_like(values)
    pce = np.zeros(ctas, np.int64)
    if kind == "lb":
        pwp = np.zeros(ctas * tpb // ws, np.int64)
        acc = O.lb_kernel(off, tgt, w, z[p + "huge"], z[p + "cumulative"], values, out, aux, op,
                          int(z[p + "blocked"]), ctas, tpb, ws, pce, pwp)
        assert acc == int(z[p + "accesses"])
        assert np.array_equal(pwp, z[p + "per_warp_paths"])
    elif kind == "twc":
        O.twc_kernel(off, tgt, w, z[p + "small"], z[p + "medium"], z[p + "large"], values, out,
                     aux, op, ctas, tpb, ws, pce)
    else:
        fn = O.vertex_kernel if kind == "vertex" else O.edge_kernel
        fn(off, tgt, w, z[p + "frontier"], values, out, aux, op, ctas, tpb, pce)
    assert np.array_equal(pce, z[p + "per_cta_edges"])
    assert np.array_equal(out, z[p + "out"])


def test_labels_small_fixture(golden):
    z = np.load(GOLDEN / "labels_small.npz")
    for name in ("rmat10", "uniform10"):
        off, tgt = _graph(name)
        for app in ("bfs", "sssp", "cc", "pr", "kcore"):
            w = O.random_weights(len(tgt), 2) if app == "sssp" else None
            lab, _ = O.run_graph(off, tgt, w, app)
            assert np.array_equal(lab, z[f"{name}_{app}"])


def test_spec_examples():
    """SPEC.md examples restated by the oracle (SURVEY App. B small fixtures)."""
    spec = _golden()["spec"]
    off, tgt, _ = O.csr_from_pairs([0, 1], [1, 2], None, 3)
    assert O.run(off, tgt, None, "bfs")[0].tolist() == spec["path_bfs"]
    off, tgt, w = O.csr_from_pairs([0, 0, 2], [1, 2, 1], [5, 1, 2], 3)
    assert O.run(off, tgt, w, "sssp")[0].tolist() == spec["triangle_sssp"]
    off, tgt, _ = O.csr_from_pairs([0, 2], [1, 3], None, 4)
    assert O.run_graph(off, tgt, None, "cc")[0].tolist() == spec["two_comp_cc"]
    off, tgt, _ = O.csr_from_pairs([0, 1], [1, 0], None, 2)
    assert O.run(off, tgt, None, "pr")[0].tolist() == spec["two_cycle_pr"]
