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
from paper_1911_09135_b200.schedulers import Scheduler, remap_threshold
from paper_1911_09135_b200.simt import KernelConfig, RoundMetrics

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
    c = KernelConfig(2, 64, 32)
    assert (c.cta_of_thread(100), c.warp_of_thread(100)) == (1, 3)


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


def test_remap_threshold_and_round_metrics():
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        assert remap_threshold(-3) == 1 and w
    assert remap_threshold(7) == 7
    m = RoundMetrics.from_device(KernelConfig(), 123, 4, {"inspect": 1, "twc": 1})
    assert m.total_edges() == 123 and m.inspect_degree_reads == 4
    assert m.as_dict()["kernel_launches"] == {"inspect": 1, "twc": 1}


def test_report_schema_from_device_log():
    """engine.report / write_reports over a synthetic device round log keep
    the reference's schema (engine.py:269-350)."""
    log = np.zeros(3, dtype=native.ROUND_DTYPE)
    log["frontier_size"] = [1, 5, 2]
    log["active_edges"] = [4, 9, 0]
    log["launches_twc"] = 1
    log["launches_lb"] = [0, 1, 0]
    sch = Scheduler("alb")
    recs = sg.engine.records_from_log(log, sch, KernelConfig())
    res = sg.engine.RunResult(np.zeros(3), recs, "bfs", sch, KernelConfig(), 1, 3, 4)
    rep = sg.report(res)
    assert rep["rounds"] == 3 and rep["totals"]["edges_processed"] == 13
    assert rep["totals"]["kernel_launches"] == {"inspect": 3, "lb": 1, "twc": 3}
    assert rep["scheduler"] == "alb-cyclic" and rep["schema_version"] == 1
    assert set(rep) >= {"app", "devices", "backend", "config", "graph", "load", "coo_bytes",
                        "labels_sha256", "spec"}


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


# ------------------------------------------------------------ partition
def test_edge_cut_bounds_match_oracle():
    from oracle import oracle_np as O
    off, tgt = O.rmat_csr(10)
    for d in (1, 2, 3, 8):
        blocks, _, _ = O.edge_cut(off, tgt, d)
        assert sg.engine.edge_cut_bounds(off, d) == blocks


def test_convergence_error_carries_log():
    e = ConvergenceError("x", metrics_log=[1, 2])
    assert e.metrics_log == [1, 2] and isinstance(e, SimtGraphError)


def test_cli_parsing_and_scheduler_tokens():
    """CLI (reference cli.py:173-290 commands): scheduler tokens, thresholds,
    usage errors -> exit code 2 without touching the device."""
    from paper_1911_09135_b200 import cli
    from paper_1911_09135_b200.errors import ConfigError
    s = cli.scheduler_of("alb-blocked", None, "4096")
    assert (s.kind, s.distribution, s.threshold) == ("alb", "blocked", 4096)
    assert cli.scheduler_of("alb", None, "inf").threshold == cli.INT64_MAX
    assert cli.scheduler_of("lb", "cyclic", "auto").describe() == "lb-cyclic"
    with pytest.raises(ConfigError):
        cli.scheduler_of("alb-diagonal")
    with pytest.raises(ConfigError):
        cli._threshold("many")
    assert cli.main(["compare", "--app", "nope"]) == 2
    assert cli.main(["sweep-threshold", "--thresholds", ""]) == 2  # empty list: ConfigError
    a = cli.parser().parse_args(["compare", "--format", "rmat", "--scale", "10",
                                 "--schedulers", "twc,alb,lb"])
    assert a.func is cli.cmd_compare and a.schedulers == "twc,alb,lb"
