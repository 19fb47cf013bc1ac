"""Graph ingestion (SPEC.md:121-129 load_graph, :160 formats) and the partition cache (CPU)."""

import numpy as np
import pytest

import paper_1810_08403_b200 as sg
from oracle import graph as og
from oracle import rng


def _w(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return p


def test_load_graph_kats(tmp_path):
    # 2-line edge file "0 1 / 1 0", 2 feature rows -> V=2, E=2
    e = _w(tmp_path, "e.txt", "0 1\n1 0\n")
    f = _w(tmp_path, "f.csv", "1.5,2\n3,4.25\n")
    g = sg.load_graph(e, f)
    assert (g.V, g.E) == (2, 2)
    assert g.src.tolist() == [0, 1] and g.dst.tolist() == [1, 0]
    assert g.features.tolist() == [[1.5, 2.0], [3.0, 4.25]]
    # :127 empty edge file accepted
    g0 = sg.load_graph(_w(tmp_path, "empty.txt", ""), f)
    assert (g0.V, g0.E) == (2, 0)
    # :128 edge "5 0" with V=2 -> error naming the offending line
    bad = _w(tmp_path, "bad.txt", "0 1\n# comment\n5 0\n")
    with pytest.raises(sg.GraphFormatError, match="line 3.*out of range"):
        sg.load_graph(bad, f)


def test_load_graph_errors_name_lines(tmp_path):
    with pytest.raises(sg.GraphFormatError, match="line 2"):
        sg.load_graph(_w(tmp_path, "a.txt", "0 1\n0 x\n"))
    with pytest.raises(sg.GraphFormatError, match="line 3"):
        sg.load_graph(_w(tmp_path, "b.txt", "0 1 0.5\n1 0 2\n1 1\n"))
    with pytest.raises(sg.GraphFormatError, match="line 2"):
        sg.read_features(_w(tmp_path, "f.csv", "1,2\n3\n"), "csv")
    with pytest.raises(sg.GraphFormatError, match="rows"):
        sg.load_graph(_w(tmp_path, "c.txt", "0 1\n"), _w(tmp_path, "g.csv", "1\n2\n3\n"), num_vertices=2)
    with pytest.raises(sg.GraphFormatError, match="line 2"):
        sg.read_labels(_w(tmp_path, "l.txt", "1\n-2\n"))
    with pytest.raises(sg.GraphFormatError):
        sg.load_graph(tmp_path / "missing.txt")


def test_edge_values_labels_comments_and_whitespace(tmp_path):
    e = _w(tmp_path, "e.txt", "% header\n\n 0\t2  0.25\r\n2 1 -1e-3\n1 1 7\n")
    lab = _w(tmp_path, "y.txt", "0\n2\n1\n")
    g = sg.load_graph(e, label_file=lab)
    assert (g.V, g.E) == (3, 3)
    assert g.edge_values.tolist() == [0.25, -1e-3, 7.0]
    assert g.labels.tolist() == [0, 2, 1]
    assert g.src.tolist() == [0, 2, 1] and g.dst.tolist() == [2, 1, 1]  # self-loop kept


def test_large_edge_file_parallel_parse_roundtrip(tmp_path):
    s, d = rng.rmat_edges(5000, 300000, seed=4)
    p = tmp_path / "big.txt"
    with open(p, "w") as fh:
        fh.write("\n".join(f"{a} {b}" for a, b in zip(s.tolist(), d.tolist())))  # no final newline
    g = sg.load_graph(p, num_vertices=5000)
    assert np.array_equal(g.src, s) and np.array_equal(g.dst, d)


def test_features_binary_and_csv_roundtrip(tmp_path):
    X = rng.features(50, 7, seed=1, dtype=np.float64)
    sg.write_features_bin(tmp_path / "x.bin", X)
    assert np.array_equal(sg.read_features(tmp_path / "x.bin"), X)  # auto-detected binary
    raw = (tmp_path / "x.bin").read_bytes()
    assert np.frombuffer(raw[:16], "<u8").tolist() == [50, 7]
    np.savetxt(tmp_path / "x.csv", X, delimiter=",", fmt="%.17g")
    assert np.array_equal(sg.read_features(tmp_path / "x.csv"), X)
    (tmp_path / "trunc.bin").write_bytes(raw[:-8])
    with pytest.raises(sg.GraphFormatError, match="bytes"):
        sg.read_features(tmp_path / "trunc.bin", "bin")


def test_partition_cache_roundtrip(tmp_path):
    s, d = rng.rmat_edges(700, 9000, seed=2)
    g = sg.Graph(700, s, d)
    p1 = sg.partition_2d(g, 200, cache_dir=tmp_path)
    p2 = sg.partition_2d(g, 200, cache_dir=tmp_path)
    assert not p1.cache_hit and p2.cache_hit
    ref = og.partition_2d(s, d, 700, 200)
    for i in range(ref.P):
        for j in range(ref.P):
            a, b = p2.chunk(i, j), ref.chunk(i, j)
            for k in ("csc_ptr", "csc_idx", "csc_eid", "csr_ptr", "csr_idx", "csr_eid"):
                assert np.array_equal(np.asarray(a[k]), b[k]), (i, j, k)
    # a different edge list or interval size is a different cache entry
    g2 = sg.Graph(700, d, s)
    assert not sg.partition_2d(g2, 200, cache_dir=tmp_path).cache_hit
    assert not sg.partition_2d(g, 300, cache_dir=tmp_path).cache_hit
