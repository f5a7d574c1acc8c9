"""CPU: host-side logic of the drop-in package (no kernel calls) and the C ABI
surface (library loads, exports every symbol include/*.h declares)."""

from __future__ import annotations

import io
import re
import warnings
from pathlib import Path

import numpy as np
import pytest

import paper_1911_09135_b200 as sg
from paper_1911_09135_b200 import native
from paper_1911_09135_b200.errors import (ConfigError, ConvergenceError, ParseError, RangeError,
                                          SimtGraphError)
from paper_1911_09135_b200.schedulers import (Scheduler, assign_blocked, assign_cyclic,
                                              split_frontier)
from paper_1911_09135_b200.simt import KernelConfig, RoundMetrics, ThreadCoord
from paper_1911_09135_b200.worklist import (PrefixWork, Worklist, find_owner, remap_threshold)

ROOT = Path(__file__).resolve().parents[1]


# ------------------------------------------------------------------ C ABI
def _header_functions():
    text = "".join(p.read_text() for p in (ROOT / "include").glob("*.h"))
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = native.load()
    declared = _header_functions()
    assert len(declared) >= 15
    missing = [n for n in declared if not hasattr(lib, n)]
    assert not missing, missing
    assert set(native.EXPORTS) <= set(declared)


def test_library_is_sm100a_only():
    import subprocess
    so = native.LIB_PATH
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(so)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_round_struct_layout():
    import ctypes
    assert native.ROUND_DTYPE.itemsize == 11 * 8
    assert ctypes.sizeof(native.Params) == 4 * 4 + 8 * 2 + 8 * 2 + 8 * 2 + 4 * 2


def test_no_cpu_fallback_without_gpu_or_library(monkeypatch, tmp_path):
    monkeypatch.setattr(native, "_lib", None)
    with pytest.raises(SimtGraphError):
        native.load(tmp_path / "missing.so")


# ------------------------------------------------------- schedulers / simt
def test_kernel_config_and_threads():
    c = KernelConfig()
    assert (c.num_ctas, c.threads_per_cta, c.warp_size, c.total_threads) == (84, 256, 32, 21504)
    assert c.num_warps == 672
    with pytest.raises(ConfigError):
        KernelConfig(2, 48, 32)
    with pytest.raises(ConfigError):
        KernelConfig(0, 64, 32)
    t = ThreadCoord.from_global(100, KernelConfig(2, 64, 32))
    assert (t.cta_id, t.warp_id, t.lane_id) == (1, 3, 4)


def test_scheduler_resolution():
    assert Scheduler("alb").resolved_distribution() == "cyclic"
    assert Scheduler("lb").resolved_distribution() == "blocked"
    assert Scheduler("alb").resolved_threshold(KernelConfig()) == 21504
    assert Scheduler("alb", threshold=1024).describe() == "alb-cyclic-t1024"
    assert Scheduler("lb").describe() == "lb-blocked"
    with pytest.raises(ConfigError):
        Scheduler("magic")
    with pytest.raises(ConfigError):
        Scheduler("alb", distribution="zigzag")
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        assert Scheduler("alb", threshold=0).resolved_threshold(KernelConfig()) == 1
        assert w


def test_assignments_spec_examples():
    cfg = KernelConfig(1, 20, 4)
    assert list(assign_cyclic(100, cfg, 4)) == [4, 24, 44, 64, 84]
    assert list(assign_cyclic(5, cfg, 7)) == []
    assert list(assign_blocked(100, cfg, 4)) == [20, 21, 22, 23, 24]
    # SPEC.md:285 claims empty; the reference code returns [76]
    assert list(assign_blocked(77, cfg, 19)) == [76]
    seen = sorted(x for t in range(20) for x in assign_cyclic(77, cfg, t))
    assert seen == list(range(77))
    seen = sorted(x for t in range(20) for x in assign_blocked(77, cfg, t))
    assert seen == list(range(77))


def test_split_frontier_bins():
    cfg = KernelConfig(2, 64, 32)
    fr = np.arange(6, dtype=np.int64)
    deg = np.array([0, 31, 32, 63, 64, 500])
    huge, bins = split_frontier(fr, deg, 500, cfg)
    assert huge.tolist() == [5]
    assert bins.small.tolist() == [0, 1] and bins.medium.tolist() == [2, 3]
    assert bins.large.tolist() == [4]
    huge, bins = split_frontier(fr, deg, None, cfg)
    assert len(huge) == 0 and bins.large.tolist() == [4, 5]


def test_find_owner_spec_and_linear_scan():
    p = PrefixWork(np.array([10, 11, 12]), np.array([40, 64, 77]))
    assert find_owner(p, 4)[:2] == (10, 4)
    assert find_owner(p, 40)[:2] == (11, 0)
    assert find_owner(p, 76)[:2] == (12, 12)
    with pytest.raises(RangeError):
        find_owner(p, 77)
    rng = np.random.default_rng(3)
    for n in range(1, 40):
        cum = np.cumsum(rng.integers(1, 9, n))
        p = PrefixWork(np.arange(n), cum)
        for g in range(int(cum[-1])):
            o, off, probes = find_owner(p, g)
            lin = int(np.flatnonzero(cum > g)[0])
            assert o == lin and off == g - (cum[lin - 1] if lin else 0)
            assert len(probes) <= int(np.ceil(np.log2(n))) + 1


def test_worklist():
    wl = Worklist(5)
    wl.push(3)
    wl.push(1)
    wl.push(3)
    assert wl.ids().tolist() == [3, 1] and len(wl) == 2 and 3 in wl
    assert wl.to_dense().ids().tolist() == [1, 3]
    with pytest.raises(RangeError):
        wl.push(5)
    with pytest.raises(RangeError):
        Worklist.from_ids(3, [0, 7])
    assert Worklist.from_ids(6, [4, 2, 4, 0]).ids().tolist() == [4, 2, 0]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        assert remap_threshold(-3) == 1


def test_round_metrics_charge_search():
    m = RoundMetrics(KernelConfig(1, 64, 32))
    m.begin_pass()
    for _ in range(32):
        m.charge_search(0, (3, 1, 2))
    assert m.search_memory_accesses == 3 and m.per_warp_search_paths[0] == 1
    m.charge_search(0, (3, 4))
    assert m.search_memory_accesses == 5 and m.per_warp_search_paths[0] == 2


# ----------------------------------------------------------------- graph
def test_graph_validation_and_from_edges():
    g = sg.Graph.from_edges([0, 0, 1], [1, 2, 2], None, 3)
    assert g.out_offsets.tolist() == [0, 2, 3, 3] and g.num_edges == 3
    assert g.out_degrees().tolist() == [2, 1, 0]
    with pytest.raises(ConfigError):
        sg.Graph(np.array([1, 2]), np.array([0], np.int32))
    with pytest.raises(RangeError):
        sg.Graph(np.array([0, 1]), np.array([5], np.int32))
    with pytest.raises(ConfigError):
        sg.Graph(np.array([0, 1]), np.array([0], np.int32), np.array([1, 2]))


def test_edge_list_loader():
    g = sg.graph.load_edge_list("0 1\n0 2\n1 2")
    assert g.num_vertices == 3 and g.out_offsets.tolist() == [0, 2, 3, 3]
    e = sg.graph.load_edge_list("")
    assert e.num_vertices == 0 and e.num_edges == 0
    w = sg.graph.load_edge_list("0 1 5\n1 0 7", weighted=True)
    assert w.edge_weights.tolist() == [5, 7]
    h = sg.graph.load_edge_list("# vertices 10\n0 1\n")
    assert h.num_vertices == 10
    with pytest.raises(ParseError) as ei:
        sg.graph.load_edge_list("0 1\n0\n")
    assert ei.value.line == 2
    with pytest.raises(ParseError):
        sg.graph.load_edge_list("0 x\n")
    with pytest.raises(RangeError):
        sg.graph.load_edge_list(f"0 {2**31}\n")
    with pytest.raises(ConfigError):
        sg.graph.load_edge_list("0 1 -3\n", weighted=True)
    with pytest.raises(RangeError):
        sg.graph.load_edge_list("# vertices 2\n0 5\n")


def test_binary_round_trip(tmp_path):
    g = sg.Graph.from_edges([0, 0, 3, 2], [1, 3, 0, 2], [4, 5, 6, 7], 4)
    buf = io.BytesIO()
    g.save_binary(buf)
    raw = buf.getvalue()
    assert raw[:4] == b"SGB1" and len(raw) == 4 + 8 + 16 + 8 * 5 + 4 * 4 + 8 * 4
    h = sg.Graph.load_binary(io.BytesIO(raw))
    assert np.array_equal(h.out_offsets, g.out_offsets)
    assert np.array_equal(h.out_targets, g.out_targets)
    assert np.array_equal(h.edge_weights, g.edge_weights)
    p = tmp_path / "g.bin"
    g.save_binary(str(p))
    with open(p, "rb") as f:  # a stream parses on the host (a path streams into HBM: GPU tests)
        assert sg.Graph.load_binary(f).num_edges == 4
    with pytest.raises(ParseError):
        sg.Graph.load_binary(io.BytesIO(b"NOPE" + raw[4:]))
    with pytest.raises(ConfigError):
        sg.graph.load_graph(tmp_path / "g.xyz")


def test_generate_rmat_validation_is_host_side():
    with pytest.raises(ConfigError):
        sg.generate_rmat(0, 16, 1)
    with pytest.raises(ConfigError):
        sg.generate_rmat(4, 16, 1, (0.5, 0.5, 0.5, 0.5))


# ------------------------------------------------------------------ apps
def test_app_parameters():
    from paper_1911_09135_b200.apps import make_app
    assert make_app("pagerank").name == "pr"
    with pytest.raises(ConfigError):
        make_app("pr", damping=1.0)
    with pytest.raises(ConfigError):
        make_app("pr", tol=0.0)
    with pytest.raises(ConfigError):
        make_app("kcore", k=0)
    with pytest.raises(ConfigError):
        make_app("triangles")


# ------------------------------------------------------- partition / sync
def test_partition_and_sync_match_oracle():
    from oracle import oracle_np as O
    from paper_1911_09135_b200.engine import make_partition, sync_labels
    from paper_1911_09135_b200.schedulers import TraversalView
    off, tgt = O.rmat_csr(10)
    view = TraversalView(off, tgt, None, "push")
    for d in (1, 2, 3, 8):
        part = make_partition(view, d)
        blocks, owner, mc = O.edge_cut(off, tgt, d)
        assert part.ranges == blocks
        assert np.array_equal(part.owner, owner) and np.array_equal(part.mirror_count, mc)
    part = make_partition(view, 2)
    a = np.array([5.0, 1.0, np.inf] + [0.0] * (len(off) - 4))
    b = np.array([3.0, 2.0, 7.0] + [0.0] * (len(off) - 4))
    merged, sent = sync_labels(part, [a, b], "min", baseline=np.full(len(a), np.inf))
    assert merged[:3].tolist() == [3.0, 1.0, 7.0]
    with pytest.raises(ConfigError):
        sync_labels(part, [a], "max")


def test_convergence_error_carries_log():
    e = ConvergenceError("x", metrics_log=[1, 2])
    assert e.metrics_log == [1, 2] and isinstance(e, SimtGraphError)
