"""Config-4 async clustering objective, optionally after a sync round on the
same graph (regression probe).  Usage: python tools/q_async.py [sync-first]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_01731_b200 as L  # noqa: E402
from paper_2108_01731_b200.gen import rmat_device  # noqa: E402

dg = rmat_device(24, 16, seed=24)
p = L.ClusteringParams(0.85)
if len(sys.argv) > 1:
    L.best_moves_round(dg, p, L.singletons(dg.n, p), frontier=None, schedule=L.Schedule.Synchronous)
for _ in range(2):
    cl = L.parallel_cc(dg, p, L.ParOptions())
    st = cl.meta["stats"]
    print(os.environ.get("LCC_LIB_PATH", "default"), sys.argv[1:], "objective", L.cc_objective(dg, p, cl),
          "rounds", st.rounds, "levels", st.levels, flush=True)
