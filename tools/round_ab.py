"""A/B of one async round-1 call through CudaBackend.round at config 4:
explicit frontier vs none (all vertices), with and without the fused
neighbour marks.  Run on a GPU box: python tools/round_ab.py
(AB_SYNC=1: the synchronous round instead)"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2108_01731_b200 import _lib  # noqa: E402
from paper_2108_01731_b200.dist import CudaBackend, make_part  # noqa: E402
from paper_2108_01731_b200.graph import stream_ptr  # noqa: E402

dg = bench.build_graph_device(24, 16, 24)
n = dg.n
part = make_part(dg.indptr, dg.indices, None, float(dg.nnz // 2), 0, n, torch.device("cuda", 0))
be = CudaBackend()
lib = be.lib
iota = torch.arange(n, dtype=torch.int32, device="cuda")
mark = torch.empty(n, dtype=torch.uint8, device="cuda")
moved = torch.empty(n, dtype=torch.uint8, device="cuda")


D = torch.empty(n, dtype=torch.int32, device="cuda")
SCHED = _lib.SYNC if os.environ.get("AB_SYNC") else _lib.ASYNC


def raw(frontier, use_mark):
    C = iota.clone()
    K2 = torch.zeros(2 * n, dtype=torch.float64, device="cuda")
    K2[:n] = 1.0
    g, p = be._g(part), be._p(None, 0.85)
    cnt = ctypes.c_int64()
    _lib.check(lib.lcc_best_moves_round(ctypes.byref(g), ctypes.byref(p), C.data_ptr(), K2.data_ptr(),
                                        None if frontier is None else frontier.data_ptr(), n, SCHED,
                                        1000, 0, D.data_ptr() if SCHED == _lib.SYNC else None, moved.data_ptr(), mark.data_ptr() if use_mark else None,
                                        ctypes.byref(cnt), None, stream_ptr()))


for name, fr, mk in [("frontier=iota mark=0", iota, False), ("frontier=None mark=0", None, False),
                     ("frontier=iota mark=1", iota, True), ("frontier=None mark=1", None, True)]:
    for _ in range(3):
        raw(fr, mk)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        raw(fr, mk)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / 10:.3f} ms per round", flush=True)
