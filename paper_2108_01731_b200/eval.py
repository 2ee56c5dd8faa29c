"""Quality evaluation (the reference's ``eval`` module, ``SPEC.md:329-388``;
SURVEY.md §8f row 2).

Same operation names, argument meanings and errors as the SPEC:
``avg_precision_recall(c, gt)``, ``ari(c, labels)``, ``nmi(c, labels)``,
``cluster_stats(c)`` plus the ``GroundTruth`` / ``EvalReport`` types.  Every
metric is computed on the device by the sm_100a library (contingency tables
by radix sort + run-length encoding, ``csrc/eval.cu``); this module only
moves arrays and maps status codes.
"""
from __future__ import annotations

import ctypes
import json
from dataclasses import asdict, dataclass, field

import numpy as np
import torch

from . import _lib
from .graph import GraphError, _device, _to_dev, stream_ptr
from .objective import Clustering


@dataclass
class GroundTruth:
    """Overlapping ground-truth communities: each a
    non-empty set of vertex ids < n.  Stored as CSR (``offsets``, ``members``)."""
    offsets: np.ndarray   # int64 [k+1]
    members: np.ndarray   # int32 [offsets[-1]]

    @classmethod
    def from_sets(cls, communities) -> "GroundTruth":
        offs = [0]
        mem: list[np.ndarray] = []
        for t in communities:
            a = np.unique(np.asarray(list(t), dtype=np.int64))
            if a.size == 0:
                raise GraphError("ground-truth communities must be non-empty")
            mem.append(a)
            offs.append(offs[-1] + a.size)
        members = np.concatenate(mem).astype(np.int32) if mem else np.zeros(0, np.int32)
        return cls(np.asarray(offs, dtype=np.int64), members)

    @property
    def num_communities(self) -> int:
        return int(self.offsets.size - 1)

    def communities(self) -> list[list[int]]:
        return [self.members[self.offsets[i]:self.offsets[i + 1]].tolist() for i in range(self.num_communities)]


@dataclass
class EvalReport:
    """SPEC.md:338-341; key names are the stable JSON names of ``write_metrics``."""
    objective: float | None = None
    num_clusters: int | None = None
    avg_precision: float | None = None
    avg_recall: float | None = None
    ari: float | None = None
    nmi: float | None = None
    runtime_ms: float | None = None
    seed: int | None = None
    extra: dict = field(default_factory=dict)

    def to_json(self) -> str:
        d = asdict(self)
        extra = d.pop("extra")
        d.update({k: v for k, v in extra.items() if k not in d})
        return json.dumps(d, sort_keys=False)


def _labels(c, dev) -> torch.Tensor:
    lab = c.assignment if isinstance(c, Clustering) else _to_dev(c, torch.int32, dev)
    return lab.contiguous()


def _pair(c, labels):
    dev = _device()
    a = _labels(c, dev)
    b = _labels(labels, dev)
    if a.numel() != b.numel():
        raise GraphError("labels length must equal n")
    ari_v, nmi_v = ctypes.c_double(), ctypes.c_double()
    _lib.check(_lib.load().lcc_partition_scores(a.numel(), a.data_ptr(), b.data_ptr(), ctypes.byref(ari_v),
                                                ctypes.byref(nmi_v), stream_ptr()))
    return ari_v.value, nmi_v.value


def ari(c, labels) -> float:
    """Adjusted Rand index via the pair-counting contingency table."""
    return _pair(c, labels)[0]


def nmi(c, labels) -> float:
    """Normalised mutual information, arithmetic-mean normalisation."""
    return _pair(c, labels)[1]


def ari_nmi(c, labels) -> tuple[float, float]:
    """Both pair metrics from one contingency table."""
    return _pair(c, labels)


def avg_precision_recall(c, gt: GroundTruth) -> tuple[float, float]:
    """best-matching cluster per community (largest overlap,
    ties to the lowest cluster id); unweighted means of precision and recall."""
    if gt.num_communities == 0:
        raise GraphError("empty ground truth")
    dev = _device()
    C = _labels(c, dev)
    off = torch.as_tensor(np.ascontiguousarray(gt.offsets, dtype=np.int64)).to(dev)
    mem = torch.as_tensor(np.ascontiguousarray(gt.members, dtype=np.int32)).to(dev)
    p, r = ctypes.c_double(), ctypes.c_double()
    _lib.check(_lib.load().lcc_avg_precision_recall(C.numel(), C.data_ptr(), gt.num_communities, off.data_ptr(),
                                                    mem.data_ptr(), ctypes.byref(p), ctypes.byref(r), stream_ptr()))
    return p.value, r.value


def cluster_stats(c) -> tuple[int, int, int, float]:
    """(num_clusters, min size, max size, mean size)."""
    dev = _device()
    C = _labels(c, dev)
    num, mn, mx, mean = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_double()
    _lib.check(_lib.load().lcc_cluster_stats(C.numel(), C.data_ptr() if C.numel() else None, ctypes.byref(num),
                                             ctypes.byref(mn), ctypes.byref(mx), ctypes.byref(mean), stream_ptr()))
    return num.value, mn.value, mx.value, mean.value
