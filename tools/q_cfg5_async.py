"""Config-5 async clustering objective and time under schedule settings
(quality probe against the CPU parallel-async oracle's 7,446,638.65,
profiles/r02_parity_cfg5.jsonl).  Usage: python tools/q_cfg5_async.py CHUNKS..."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_01731_b200 as L  # noqa: E402
from paper_2108_01731_b200.gen import powerlaw_communities_device, rmat_device  # noqa: E402

cfg = os.environ.get("Q_CFG", "cfg5")
dg = powerlaw_communities_device() if cfg == "cfg5" else rmat_device(24, 16, seed=24)
p = L.ClusteringParams(0.85)
L.parallel_cc(dg, p, L.ParOptions())  # warm-up (pool growth, kernel loading)
for ch in [int(x) for x in sys.argv[1:]] or [0]:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cl = L.parallel_cc(dg, p, L.ParOptions(async_chunks=ch))
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    st = cl.meta["stats"]
    print(f"{cfg} chunks {ch} wave {os.environ.get('LCC_WAVE', '')} subconc {os.environ.get('LCC_SUBCONC', '')} objective "
          f"{L.cc_objective(dg, p, cl):.2f} time {t:.2f} s rounds {st.rounds} levels {st.levels} "
          f"clusters {cl.num_clusters}", flush=True)
    del cl
