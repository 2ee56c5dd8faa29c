"""Repeat parallel_cc on the config-5 graph (device resident) with LCC_TRACE:
per-call wall time, levels and rounds.  Usage: python tools/cfg5_trace.py [reps]"""
import os, sys, time, torch
sys.path.insert(0, '.')
import paper_2108_01731_b200 as L
from paper_2108_01731_b200.gen import powerlaw_communities_device
dg = powerlaw_communities_device()
torch.cuda.empty_cache()
p = L.ClusteringParams(0.85)
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    cl = L.parallel_cc(dg, p, L.ParOptions())
    torch.cuda.synchronize(); t = time.perf_counter() - t0
    st = cl.meta["stats"]
    print(f"=== rep {rep} {t:.2f} s levels {st.levels} rounds {st.rounds}", file=sys.stderr, flush=True)
    del cl
