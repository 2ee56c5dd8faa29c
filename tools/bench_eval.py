"""Measure the eval row at config-4 size: ARI + NMI of
two 16.8M-vertex labelings, average precision/recall over 5000 overlapping
communities (the paper's "top 5000 ground-truth communities")
and cluster statistics -- device time through the public API against
sklearn / the numpy oracle on the host cores.  One JSON line on stdout.
Usage: python tools/bench_eval.py [n]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_01731_b200.eval as E  # noqa: E402


def timed(f, reps=5):
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        r = f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return r, 1e3 * float(np.median(ts))


def main(n):
    rng = np.random.default_rng(24)
    a = rng.integers(0, n // 8, n).astype(np.int32)   # ~2M clusters
    b = np.where(rng.random(n) < 0.8, a, rng.integers(0, n // 8, n)).astype(np.int32)
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    comms = [rng.choice(n, size=int(rng.integers(2, 2000)), replace=False) for _ in range(5000)]
    gt = E.GroundTruth.from_sets(comms)
    (ari, nmi), t_pair = timed(lambda: E.ari_nmi(da, db))
    (p, r), t_pr = timed(lambda: E.avg_precision_recall(da, gt))
    st, t_st = timed(lambda: E.cluster_stats(da))
    out = dict(metric="eval (SURVEY §8f row 2)", n=n, clusters=int(st[0]), communities=gt.num_communities,
               community_members=int(gt.offsets[-1]), ari=ari, nmi=nmi, precision=p, recall=r,
               device_ms=dict(ari_nmi=t_pair, precision_recall=t_pr, cluster_stats=t_st),
               gelem_per_s_ari_nmi=n / t_pair / 1e6)
    # CPU reference: sklearn (the SPEC's standard formulas) on a bounded sample
    from sklearn.metrics import adjusted_rand_score, normalized_mutual_info_score
    m = min(n, 4_000_000)
    t0 = time.perf_counter()
    adjusted_rand_score(a[:m], b[:m])
    normalized_mutual_info_score(a[:m], b[:m], average_method="arithmetic")
    t_cpu = time.perf_counter() - t0
    out["cpu_baseline"] = dict(kind="sklearn", sample=f"first {m} labels", seconds=t_cpu,
                               gelem_per_s=m / t_cpu / 1e9, cores=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24)
