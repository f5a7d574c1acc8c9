"""SGB1 files straight into HBM (sg_graph_load_sgb1) against the reference's
load_binary semantics (graph.py:136-177): the same arrays, and for malformed
files the same exception class and message as the host parse of the same
bytes (which builds the Graph exactly as the reference does, so its
validation, graph.py:44-57, reports short or bad sections)."""

from __future__ import annotations

import hashlib
import io
import struct

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sg():
    import paper_1911_09135_b200 as sg
    from paper_1911_09135_b200 import native
    if native.device_count() < 1:
        pytest.fail("no CUDA device visible")
    return sg


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("scale,weighted", [(10, False), (14, True), (18, True)])
def test_round_trip_device(sg, tmp_path, scale, weighted):
    g = sg.generate_rmat(scale, 16, 1)
    if weighted:
        g = sg.attach_random_weights(g, 2)
    p = tmp_path / "g.bin"  # load_graph picks the format by extension
    g.save_binary(str(p))
    h = sg.Graph.load_binary(str(p))
    assert h.num_vertices == g.num_vertices and h.num_edges == g.num_edges
    assert h.is_weighted == weighted
    assert _sha(h.out_offsets) == _sha(g.out_offsets)
    assert _sha(h.out_targets) == _sha(g.out_targets)
    if weighted:
        assert _sha(h.edge_weights) == _sha(g.edge_weights)
    app = "sssp" if weighted else "bfs"
    a, b = sg.run_app(g, app), sg.run_app(h, app)
    assert np.array_equal(a.labels, b.labels)
    assert sg.graph.load_graph(p).num_edges == g.num_edges  # load_graph dispatches here too


def _raw(g):
    buf = io.BytesIO()
    g.save_binary(buf)
    return buf.getvalue()


def _both(sg, tmp_path, raw):
    """(exception type, message) of the host parse and of the device loader."""
    out = []
    for kind in ("host", "device"):
        try:
            if kind == "host":
                sg.Graph.load_binary(io.BytesIO(raw))
            else:
                p = tmp_path / "x.sgb"
                p.write_bytes(raw)
                sg.Graph.load_binary(str(p))
            out.append(None)
        except Exception as e:  # noqa: BLE001
            out.append((type(e), str(e)))
    return out


def test_malformed_files_match_reference_errors(sg, tmp_path):
    from paper_1911_09135_b200.errors import ConfigError, ParseError, RangeError
    g = sg.Graph.from_edges([0, 0, 3, 2, 1], [1, 3, 0, 2, 2], [4, 5, 6, 7, 8], 4)
    raw = _raw(g)
    hdr, nv, ne = 28, 4, 5
    cases = {
        "magic": (b"NOPE" + raw[4:], ParseError),
        "version": (raw[:4] + struct.pack("<I", 2) + raw[8:], ParseError),
        "short offsets": (raw[:hdr + 8 * 3], ConfigError),
        "short targets": (raw[:hdr + 8 * (nv + 1) + 4 * 3], ConfigError),
        "short weights": (raw[:hdr + 8 * (nv + 1) + 4 * ne + 8 * 2], ConfigError),
    }
    bad = bytearray(raw)  # a target == V
    struct.pack_into("<i", bad, hdr + 8 * (nv + 1) + 4 * 2, nv)
    cases["target range"] = (bytes(bad), RangeError)
    bad = bytearray(raw)  # a negative target
    struct.pack_into("<i", bad, hdr + 8 * (nv + 1), -1)
    cases["negative target"] = (bytes(bad), RangeError)
    bad = bytearray(raw)  # offsets decrease (3 -> 1)
    struct.pack_into("<q", bad, hdr + 8 * 2, 4)
    struct.pack_into("<q", bad, hdr + 8 * 3, 1)
    cases["decreasing offsets"] = (bytes(bad), ConfigError)
    bad = bytearray(raw)  # offsets[0] != 0
    struct.pack_into("<q", bad, hdr, 1)
    cases["offset start"] = (bytes(bad), ConfigError)
    for name, (data, exc) in cases.items():
        host, dev = _both(sg, tmp_path, data)
        assert host is not None and host[0] is exc, (name, host)
        assert dev == host, (name, dev, host)
    with pytest.raises(FileNotFoundError):
        sg.Graph.load_binary(str(tmp_path / "missing.sgb"))


def test_empty_and_edgeless(sg, tmp_path):
    for g in (sg.Graph(np.zeros(1, np.int64), np.zeros(0, np.int32)),
              sg.Graph(np.zeros(6, np.int64), np.zeros(0, np.int32))):
        p = tmp_path / "e.sgb"
        g.save_binary(str(p))
        h = sg.Graph.load_binary(str(p))
        assert h.num_vertices == g.num_vertices and h.num_edges == 0
        assert np.array_equal(h.out_offsets, g.out_offsets)
