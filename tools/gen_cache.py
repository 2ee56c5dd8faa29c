"""Write a bench workload's CPU sample to disk, in a process of its own.

``bench.py --impl reference`` times the CPU oracle port on a vertex sample of
the same graph; the graph itself is generated on the device (configs 4-5:
billions of entries).  This script runs that generator in a separate
process and writes the sampled rows as .npy files, so the reference arm's
own process never loads this repository's CUDA library (it maps only
oracle/_build).

    python tools/gen_cache.py --config cfg5 --stride 8 --out DIR

DIR/indptr.npy   int64 [n+1]: rows of sampled vertices (v % stride == 0)
                 hold their full neighbour lists, every other row is empty
DIR/indices.npy  int32: the sampled rows' neighbours
DIR/meta.json    n, m, lambda, schedule, sample vertices / entries, workload
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", required=True)
    ap.add_argument("--stride", type=int, default=8)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    import numpy as np
    import torch
    import bench
    args = bench.parse([f"--config={a.config}"])
    wl = bench.Workload(args, a.config)
    ip, ix, F, edges = bench.sample_rows(wl.dg, a.stride)
    os.makedirs(a.out, exist_ok=True)
    np.save(os.path.join(a.out, "indptr.npy"), ip)
    np.save(os.path.join(a.out, "indices.npy"), ix)
    k = None if wl.k is None else wl.k.cpu().numpy()
    if k is not None:
        np.save(os.path.join(a.out, "k.npy"), k)
    meta = {"n": wl.dg.n, "m": wl.dg.m, "lambda": wl.lam, "schedule": wl.schedule, "stride": a.stride,
            "sample_vertices": int(F), "sample_entries": int(edges), "workload": wl.desc,
            "total_weight": wl.dg.total_weight}
    with open(os.path.join(a.out, "meta.json"), "w") as f:
        json.dump(meta, f)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
