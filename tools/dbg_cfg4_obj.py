"""Regression probe: config-4 async objective after other clusterings in the
same process.  Usage: python tools/dbg_cfg4_obj.py [cfg2|cfg3|none] [cold]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_01731_b200 as L  # noqa: E402
from paper_2108_01731_b200 import gen  # noqa: E402

pre = sys.argv[1] if len(sys.argv) > 1 else "none"
if pre == "cfg2":
    hg, _ = gen.lfr_like(n=1_200_000, seed=2)
    p2 = L.modularity_params(hg, 1.0)
    cl = L.parallel_cc(hg, p2, L.ParOptions())
    print("cfg2 modularity", L.modularity_value(hg, 1.0, cl), flush=True)
if pre == "cfg2test":  # the parity test's cfg2 step, oracle runs included
    from tests.test_parity_full import test_cfg2_lfr_modularity_async_full
    test_cfg2_lfr_modularity_async_full()
    print("cfg2 test done", flush=True)
if "cfg4test" in sys.argv:  # then the parity test's cfg4 step itself
    from tests.test_parity_full import test_cfg4_rmat_full
    try:
        test_cfg4_rmat_full()
        print("cfg4 test passed", flush=True)
    except AssertionError as e:
        print("cfg4 test failed", e, flush=True)
    sys.exit(0)
if "round1" in sys.argv:  # a sync round + its oracle check before the clusterings
    from tests.test_parity_full import _round1_exact
    _round1_exact(gen.rmat_device(24, 16, seed=24), 0.85)
    print("round1 done", flush=True)
if pre == "oracle":  # only an OpenMP oracle clustering before
    from oracle import oracle as O
    from paper_2108_01731_b200.gen import rmat_pairs_host, csr_from_pairs
    u, v = rmat_pairs_host(16, 16 << 16, 0.57, 0.19, 0.19, 1)
    go = O.as_graph(csr_from_pairs(1 << 16, u, v))
    O.parallel_cc(go, None, 0.85, O.Opts(schedule=O.ASYNC, async_parallel=True, threads=os.cpu_count()))
    print("oracle done", flush=True)
if pre == "cfg3":
    hg, _ = gen.knn_mixture(seed=3)
    cl = L.parallel_cc(hg, L.ClusteringParams(0.1), L.ParOptions(schedule="sync"))
    print("cfg3 objective", L.cc_objective(hg, L.ClusteringParams(0.1), cl), flush=True)
dg = gen.rmat_device(24, 16, seed=24)
p = L.ClusteringParams(0.85)
cold = "cold" in sys.argv
for _ in range(4 if cold else 2):
    if cold:  # the library's scratch handed back: the next call grows the pool afresh
        L.release_memory()
    cl = L.parallel_cc(dg, p, L.ParOptions())
    print(os.environ.get("LCC_LIB_PATH", "default"), pre, "cfg4 objective", L.cc_objective(dg, p, cl), flush=True)
