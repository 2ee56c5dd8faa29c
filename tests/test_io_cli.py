"""File I/O and CLI.

CPU: parsing, error paths and round trips.  GPU: the device edge-list
builder (lcc_build_graph) against golden outputs of the reference's own
``build_graph_arrays`` (tests/golden/build.npz, made by
tests/golden/make_golden.py), the SPEC I/O examples, and the ``cluster`` /
``eval`` / ``rmat`` commands end to end.
"""
import json
import os

import numpy as np
import pytest

from paper_2108_01731_b200 import io as lio
from paper_2108_01731_b200.eval import EvalReport
from paper_2108_01731_b200.graph import GraphError


@pytest.mark.gpu
def test_build_matches_reference_golden(golden):
    """The device build (lcc_build_graph) against the reference's own
    build_graph_arrays output: CSR, weights and total_weight bit for bit."""
    from paper_2108_01731_b200.graph import build_graph_arrays
    z = golden("build.npz")
    for t in z["cases"]:
        p = f"b{t}_"
        g = build_graph_arrays(z[p + "u"], z[p + "v"], z[p + "w"], n=int(z[p + "n"][0]))
        ip, ind, w = g.to_host()
        assert g.m == int(z[p + "m"][0])
        assert np.array_equal(ip, z[p + "indptr"])
        assert np.array_equal(ind, z[p + "indices"])
        w = np.ones(ind.size) if w is None else w
        assert np.array_equal(w, z[p + "weights"])  # bit-identical sums and averages
        assert g.total_weight == float(z[p + "total"][0])


def test_parse_edge_list(tmp_path):
    f = tmp_path / "e.txt"
    f.write_text("# c\na b\nb c 2.5\n")
    u, v, w, idmap = lio.parse_edge_list(str(f), weighted=True)
    assert idmap == ["a", "b", "c"] and u.tolist() == [0, 1] and v.tolist() == [1, 2] and w.tolist() == [1.0, 2.5]
    f.write_text("3 1\n")
    u, v, w, idmap = lio.parse_edge_list(str(f))
    assert idmap is None and w is None and u.tolist() == [3]


@pytest.mark.gpu
def test_read_edge_list_spec_examples(tmp_path):
    f = tmp_path / "path.txt"
    f.write_text("0 1\n1 2\n")
    g, idmap = lio.read_edge_list(str(f))
    assert (g.n, g.m, idmap) == (3, 2, None) and g.weights is None
    f.write_text("# comment\n0 1 2.5\n")
    g, _ = lio.read_edge_list(str(f), weighted=True)
    assert g.m == 1 and np.array_equal(g.weights.cpu().numpy(), [2.5, 2.5])
    f.write_text("a b\nb c\n")
    g, idmap = lio.read_edge_list(str(f))
    assert idmap == ["a", "b", "c"] and g.n == 3 and g.m == 2
    f.write_text("0 1\n0 1\n1 0\n2 2\n")  # same-orientation sum, orientation average, loop dropped
    g, _ = lio.read_edge_list(str(f))
    assert g.m == 1 and np.array_equal(g.weights.cpu().numpy(), [1.5, 1.5]) and g.n == 3


def test_read_errors(tmp_path):
    f = tmp_path / "bad.txt"
    f.write_text("0 1\n0\n")
    with pytest.raises(GraphError, match=":2:"):
        lio.read_edge_list(str(f))
    f.write_text("0 1 x\n")
    with pytest.raises(GraphError, match="bad weight"):
        lio.read_edge_list(str(f), weighted=True)
    with pytest.raises(FileNotFoundError):
        lio.read_edge_list(str(tmp_path / "missing.txt"))
    gt = tmp_path / "gt.txt"
    gt.write_text("1 2 3\n\n4 5\n")
    assert lio.read_ground_truth(str(gt), n=6).communities() == [[1, 2, 3], [4, 5]]
    gt.write_text("1 9\n")
    with pytest.raises(GraphError, match="unknown vertex"):
        lio.read_ground_truth(str(gt), n=6)


def test_clustering_and_metrics_round_trip(tmp_path):
    f = tmp_path / "c.txt"
    lio.write_clustering(str(f), np.array([0, 0], np.int32))
    assert f.read_text() == "0 0\n1 0\n"
    lab = np.array([0, 0, 2, 2, 0, 5], np.int32)
    lio.write_clustering(str(f), lab)
    assert np.array_equal(lio.read_clustering(str(f)), lab)
    idmap = ["x", "y", "z", "w", "u", "v"]
    lio.write_clustering(str(f), lab, idmap)
    assert f.read_text().splitlines()[2] == "z z"
    assert np.array_equal(lio.read_clustering(str(f), idmap), lab)
    m = tmp_path / "m.json"
    rep = EvalReport(objective=1.5, num_clusters=3, ari=None, runtime_ms=2.0, seed=7)
    lio.write_metrics(str(m), rep)
    d = json.loads(m.read_text())
    assert list(d)[:8] == ["objective", "num_clusters", "avg_precision", "avg_recall", "ari", "nmi",
                           "runtime_ms", "seed"]
    assert d["ari"] is None and lio.read_metrics(str(m)).objective == 1.5


@pytest.mark.gpu
def test_cli_cluster_eval_rmat(tmp_path):
    from paper_2108_01731_b200 import cli
    from paper_2108_01731_b200.gen import sbm
    g, truth = sbm(n=1000, communities=10, p_in=0.5, p_out=0.01, seed=3)
    src = np.repeat(np.arange(g.n), np.diff(g.indptr))
    keep = src < g.indices
    ef = tmp_path / "g.txt"
    np.savetxt(ef, np.stack([src[keep], g.indices[keep]], 1), fmt="%d")
    gt = tmp_path / "gt.txt"
    gt.write_text("\n".join(" ".join(map(str, np.flatnonzero(truth == t))) for t in range(10)) + "\n")
    lab = tmp_path / "labels.txt"
    lio.write_clustering(str(lab), truth.astype(np.int32))
    out, met = tmp_path / "out.txt", tmp_path / "met.json"
    rc = cli.main(["cluster", "--input", str(ef), "--resolution", "0.05", "--schedule", "sync",
                   "--ground-truth", str(gt), "--labels", str(lab), "--out", str(out), "--metrics", str(met)])
    assert rc == 0
    d = json.loads(met.read_text())
    assert d["avg_precision"] >= 0.95 and d["avg_recall"] >= 0.95 and d["ari"] > 0.9 and d["nmi"] > 0.9
    assert d["objective"] > 0 and d["num_clusters"] >= 10 and d["runtime_ms"] > 0
    # eval of the written clustering reproduces the metrics
    met2 = tmp_path / "met2.json"
    assert cli.main(["eval", "--input", str(ef), "--resolution", "0.05", "--clustering", str(out),
                     "--ground-truth", str(gt), "--labels", str(lab), "--metrics", str(met2)]) == 0
    d2 = json.loads(met2.read_text())
    for k in ("objective", "num_clusters", "avg_precision", "avg_recall", "ari", "nmi"):
        assert d2[k] == pytest.approx(d[k], rel=1e-12)
    # errors: lambda out of range, unknown engine, missing file -> exit 1
    assert cli.main(["cluster", "--input", str(ef), "--resolution", "1.5"]) == 1
    assert cli.main(["cluster", "--input", str(ef), "--engine", "seq"]) == 1
    assert cli.main(["cluster", "--input", str(tmp_path / "nope.txt")]) == 1
    # rmat: deterministic given the seed
    r1, r2 = tmp_path / "r1.txt", tmp_path / "r2.txt"
    assert cli.main(["rmat", "--scale", "10", "--edge-factor", "5", "--seed", "4", "--out", str(r1)]) == 0
    assert cli.main(["rmat", "--scale", "10", "--edge-factor", "5", "--seed", "4", "--out", str(r2)]) == 0
    assert r1.read_text() == r2.read_text() and os.path.getsize(r1) > 1000
    assert cli.main(["rmat", "--scale", "4", "--edges", "0", "--out", str(r1)]) == 0
    assert cli.main(["rmat", "--scale", "4", "--edges", "5", "--a", "0.9", "--out", str(r1)]) == 1
