"""File ingestion and output (the reference's ``io-gen-cli`` module,
``SPEC.md:390-450``).

* ``read_edge_list(path, weighted)`` -- "u v" / "u v w" lines, '#' comments;
  non-integer ids are remapped densely (first appearance order) and the
  mapping is returned; the CSR is built on the device by
  ``graph.build_graph_arrays`` (``lcc_build_graph``: the reference's
  ``build_graph_arrays`` contract, graph.py:98-164, bit for bit).  Unit
  weights are stored implicitly (``weights is None``) so the device path
  reads no weight array.
* ``read_ground_truth(path, id_map)`` -- one community per line.
* ``read_clustering`` / ``write_clustering`` -- "vertex_id cluster_id" lines
  in original ids; ``write_metrics`` -- one JSON object with the EvalReport
  keys (``SPEC.md:419``).

This is host-side plumbing around the device path (file parsing); the CSR
build, the clustering and every metric run in the sm_100a library.
"""
from __future__ import annotations

import json
import os
import numpy as np

from .eval import EvalReport, GroundTruth
from .graph import GraphError, build_graph_arrays


def _parse_id(tok: str):
    try:
        return int(tok)
    except ValueError:
        return tok


def read_edge_list(path: str, weighted: bool = False):
    """SPEC.md:398-406.  Returns ``(graph, id_map)``: ``graph`` is the device
    CSR (``DeviceGraph``) and ``id_map[i]`` the original id of vertex i, or
    None when the file's ids are non-negative integers (kept as they are)."""
    u, v, w, id_map = parse_edge_list(path, weighted)
    return build_graph_arrays(u, v, w, n=None if u.size else 0), id_map


def parse_edge_list(path: str, weighted: bool = False):
    """The file-parsing half of ``read_edge_list``: ``(u, v, w, id_map)``
    host arrays (int64 ids, float64 weights or None when unweighted)."""
    if not os.path.exists(path):
        raise FileNotFoundError(path)
    us, vs, ws = [], [], []
    with open(path) as f:
        for ln, line in enumerate(f, 1):
            s = line.strip()
            if not s or s.startswith("#"):
                continue
            tok = s.split()
            if len(tok) < 2 or len(tok) > 3 or (len(tok) == 3 and not weighted):
                raise GraphError(f"{path}:{ln}: malformed line {s!r}")
            us.append(_parse_id(tok[0]))
            vs.append(_parse_id(tok[1]))
            if weighted:
                if len(tok) == 3:
                    try:
                        ws.append(float(tok[2]))
                    except ValueError:
                        raise GraphError(f"{path}:{ln}: bad weight {tok[2]!r}") from None
                else:
                    ws.append(1.0)
    ids = us + vs
    id_map = None
    if all(isinstance(x, int) and x >= 0 for x in ids):
        u = np.asarray(us, np.int64)
        v = np.asarray(vs, np.int64)
    else:
        pos: dict = {}
        order = []
        for a, b in zip(us, vs):
            for x in (a, b):
                if x not in pos:
                    pos[x] = len(order)
                    order.append(x)
        u = np.asarray([pos[x] for x in us], np.int64)
        v = np.asarray([pos[x] for x in vs], np.int64)
        id_map = order
    w = np.asarray(ws, np.float64) if weighted else None
    return u, v, w, id_map


def _index(id_map):
    return None if id_map is None else {x: i for i, x in enumerate(id_map)}


def read_ground_truth(path: str, id_map=None, n: int | None = None) -> GroundTruth:
    """one community per line, member ids whitespace separated."""
    idx = _index(id_map)
    comms = []
    with open(path) as f:
        for ln, line in enumerate(f, 1):
            tok = line.split()
            if not tok or tok[0].startswith("#"):
                continue
            mem = []
            for t in tok:
                x = _parse_id(t)
                if idx is not None:
                    if x not in idx:
                        raise GraphError(f"{path}:{ln}: unknown vertex id {t!r}")
                    x = idx[x]
                elif not isinstance(x, int) or x < 0 or (n is not None and x >= n):
                    raise GraphError(f"{path}:{ln}: unknown vertex id {t!r}")
                mem.append(x)
            comms.append(mem)
    return GroundTruth.from_sets(comms)


def _orig(i: int, id_map):
    return i if id_map is None else id_map[i]


def write_clustering(path: str, c, id_map=None) -> None:
    """lines "vertex_id cluster_id" in original ids; the
    cluster id is the original id of the cluster's smallest member."""
    lab = c.labels() if hasattr(c, "labels") else np.asarray(c)
    with open(path, "w") as f:
        if id_map is None:
            np.savetxt(f, np.stack([np.arange(lab.size), lab], 1), fmt="%d")
        else:
            for i, x in enumerate(lab.tolist()):
                f.write(f"{_orig(i, id_map)} {_orig(int(x), id_map)}\n")


def read_clustering(path: str, id_map=None, n: int | None = None) -> np.ndarray:
    """Inverse of ``write_clustering``: labels[n] (internal ids; any int values)."""
    idx = _index(id_map)
    pairs = []
    with open(path) as f:
        for ln, line in enumerate(f, 1):
            tok = line.split()
            if not tok or tok[0].startswith("#"):
                continue
            if len(tok) != 2:
                raise GraphError(f"{path}:{ln}: malformed line {line.strip()!r}")
            a, b = _parse_id(tok[0]), _parse_id(tok[1])
            if idx is not None:
                if a not in idx or b not in idx:
                    raise GraphError(f"{path}:{ln}: unknown vertex id")
                a, b = idx[a], idx[b]
            pairs.append((a, b))
    if not pairs:
        return np.zeros(0 if n is None else n, np.int32)
    arr = np.asarray(pairs, np.int64)
    size = int(arr[:, 0].max()) + 1 if n is None else n
    if arr[:, 0].min() < 0 or arr[:, 0].max() >= size:
        raise GraphError(f"{path}: vertex id out of range")
    lab = np.full(size, -1, np.int64)
    lab[arr[:, 0]] = arr[:, 1]
    if (lab < 0).any():
        raise GraphError(f"{path}: some vertices have no cluster")
    return lab.astype(np.int32)


def write_metrics(path: str, report: EvalReport) -> None:
    """one JSON object with the EvalReport keys (missing -> null)."""
    with open(path, "w") as f:
        f.write(report.to_json() + "\n")


def read_metrics(path: str) -> EvalReport:
    d = json.load(open(path))
    known = {k: d.pop(k) for k in list(d) if k in EvalReport.__dataclass_fields__ and k != "extra"}
    return EvalReport(**known, extra=d)
