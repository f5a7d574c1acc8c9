"""Kernel-level plugin parity: cuda_backend.{lb,twc,vertex,edge}_kernel against
the reference's own kernel outputs captured in tests/golden/kernels_small.npz
(out arrays, per_cta_edges, per_warp_paths, search accesses — all exact,
including float64 pull sums, which the plugin accumulates in the reference's
array order)."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _fixtures():
    from pathlib import Path
    z = np.load(Path(__file__).parent / "golden" / "kernels_small.npz")
    return z, int(z["count"])


@pytest.fixture(scope="module")
def views():
    from oracle import oracle_np as O
    off, tgt = O.rmat_csr(10)
    w = O.random_weights(len(tgt), 2).astype(np.float64)
    soff, stgt, _ = O.symmetrize(off, tgt)
    coff, ctgt, _ = O.transpose(off, tgt)
    scoff, sctgt, _ = O.transpose(soff, stgt)
    return {"bfs": (off, tgt, np.empty(0)), "sssp": (off, tgt, w), "cc": (soff, stgt, np.empty(0)),
            "pr": (coff, ctgt, np.empty(0)), "kcore": (scoff, sctgt, np.empty(0))}


@pytest.mark.parametrize("i", range(_fixtures()[1]))
def test_kernel_fixture(i, views):
    from paper_1911_09135_b200 import cuda_backend as K
    z, _ = _fixtures()
    p = f"k{i}_"
    kind, app = str(z[p + "kind"]), str(z[p + "app"])
    ctas, tpb, ws = (int(x) for x in z["config"])
    off, tgt, w = views[app]
    values, aux, op = z[p + "values"], z[p + "aux"], int(z[p + "opcode"])
    out = values.copy() if op != 3 else np.zeros_like(values)
    pce = np.zeros(ctas, np.int64)
    if kind == "lb":
        pwp = np.zeros(ctas * tpb // ws, np.int64)
        acc = K.lb_kernel(off, tgt, w, z[p + "huge"], z[p + "cumulative"], values, out, aux, op,
                          int(z[p + "blocked"]), ctas, tpb, ws, pce, pwp)
        assert acc == int(z[p + "accesses"])
        assert np.array_equal(pwp, z[p + "per_warp_paths"])
    elif kind == "twc":
        K.twc_kernel(off, tgt, w, z[p + "small"], z[p + "medium"], z[p + "large"], values, out,
                     aux, op, ctas, tpb, ws, pce)
    else:
        fn = K.vertex_kernel if kind == "vertex" else K.edge_kernel
        fn(off, tgt, w, z[p + "frontier"], values, out, aux, op, ctas, tpb, pce)
    assert np.array_equal(pce, z[p + "per_cta_edges"]), kind
    assert np.array_equal(out, z[p + "out"]), (kind, app)


@pytest.mark.parametrize("app", ["bfs", "sssp", "cc", "pr", "kcore"])
@pytest.mark.parametrize("kind", ["alb", "twc", "lb", "vertex", "edge"])
def test_reference_loop_over_cuda_plugin_matches_golden(golden, app, kind):
    """The reference's host loop (restated in oracle_np.run, engine.py:205-235)
    driving the CUDA kernel plugin reproduces the reference's full report:
    labels, search accesses, launches and the modeled per-CTA load."""
    from oracle import oracle_np as O
    from paper_1911_09135_b200 import cuda_backend
    info = golden["runs"]["rmat10"].get(f"{app}/{kind}/d1")
    if info is None:
        pytest.skip("no golden for this scheduler")
    off, tgt = O.rmat_csr(10)
    w = O.random_weights(len(tgt), 2) if app == "sssp" else None
    lab, log = O.run_graph(off, tgt, w, app, kind=kind,
                           blocked=(kind in ("lb", "edge")), K=cuda_backend)
    launches = {}
    for r in log:
        for k, n in r.launches.items():
            launches[k] = launches.get(k, 0) + n
    assert O.labels_sha256(lab) == info["labels_sha256"]
    assert sum(r.accesses for r in log) == info["search_memory_accesses"]
    assert dict(sorted(launches.items())) == info["kernel_launches"]
    assert max(r.cta_cv() for r in log) == pytest.approx(info["worst_cta_cv"], abs=0)
