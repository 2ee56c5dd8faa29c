"""Repeat parallel_cc on a bench graph and print, per call, the wall time,
levels/rounds and the per-level trace lines (LCC_TRACE), to study the async
run-to-run variance.  Usage: python tools/e2e_trace.py N [cfg4|cfg5] [host]
(host: the CSR starts in pinned host memory, as in the bench e2e)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("LCC_TRACE", "1")
import paper_2108_01731_b200 as L  # noqa: E402
from paper_2108_01731_b200.gen import powerlaw_communities_device, rmat_device  # noqa: E402


def main(n, cfg="cfg4", host=False):
    dg = rmat_device(24, 16, seed=24) if cfg == "cfg4" else powerlaw_communities_device()
    if host:
        class H:
            pass
        h = H()
        h.n, h.m, h.weights, h.total_weight = dg.n, dg.m, None, dg.total_weight
        h.indptr, h.indices = dg.indptr.cpu().pin_memory(), dg.indices.cpu().pin_memory()
        dg = h
        torch.cuda.empty_cache()
    p = L.ClusteringParams(0.85)
    for i in range(n):
        torch.cuda.synchronize()
        print(f"=== call {i}", file=sys.stderr, flush=True)
        t0 = time.perf_counter()
        cl = L.parallel_cc(dg, p, L.ParOptions())
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        st = cl.meta["stats"]
        print(f"=== call {i} wall {1e3 * dt:.1f} ms levels {st.levels} rounds {st.rounds} "
              f"device {st.ms_total:.1f} ms best-move {st.ms_best_moves:.1f} ms", file=sys.stderr, flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 6, sys.argv[2] if len(sys.argv) > 2 else "cfg4",
         len(sys.argv) > 3 and sys.argv[3] == "host")
