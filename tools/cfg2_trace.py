"""LCC_TRACE of one config-2 clustering (LFR-style 1.2M, modularity, async)."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("LCC_TRACE", "1")
import paper_2108_01731_b200 as L
from paper_2108_01731_b200.gen import lfr_like
hg, _ = lfr_like(n=1_200_000, seed=2)
dg = L.DeviceGraph.from_graph(hg)
p = L.modularity_params(dg, 1.0)
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    cl = L.parallel_cc(dg, p, L.ParOptions())
    torch.cuda.synchronize()
    st = cl.meta["stats"]
    print(f"=== rep {rep} {1e3*(time.perf_counter()-t0):.1f} ms rounds {st.rounds} levels {st.levels} device {st.ms_total:.1f} bm {st.ms_best_moves:.1f} kernels {st.ms_kernels:.1f} launches {st.kernel_launches}", file=sys.stderr, flush=True)
