"""CPU backend for the sharded driver (paper_2108_01731_b200/dist.py): the
per-rank compute is the oracle, so the exchange logic can be tested with
gloo on a GPU-less machine.  Test infrastructure only."""
import os

import numpy as np
import torch

from oracle import oracle as O


def _np(t):
    return None if t is None else t.detach().cpu().numpy()


class OracleBackend:
    device = torch.device("cpu")

    def _g(self, part):
        w = _np(part.weights)
        return O.Graph(part.n, np.ascontiguousarray(_np(part.indptr)), np.ascontiguousarray(_np(part.indices)),
                       None if w is None else np.ascontiguousarray(w, dtype=np.float64), part.total_weight)

    def round(self, part, k, lam, C, K, frontier, schedule, thr, chunks):
        g = self._g(part)
        kk = _np(k)
        Cn, Kn = _np(C).copy(), _np(K).copy()
        F = _np(frontier).astype(np.int32)
        if schedule == O.SYNC:
            D, moved, cnt = O.sync_round(g, kk, lam, Cn, Kn, F)
            return torch.from_numpy(D), torch.from_numpy(moved), cnt
        K2 = np.zeros(2 * part.n); K2[:part.n] = Kn
        moved, cnt = O.async_round(g, kk, lam, Cn, K2, F)
        return torch.from_numpy(Cn), torch.from_numpy(moved), cnt

    def apply(self, labels, label_range, k):
        C, K = O.canonicalize(labels.numel(), _np(labels).astype(np.int32), label_range, _np(k))
        return torch.from_numpy(C), torch.from_numpy(K)

    def frontier_mask(self, part, policy, moved, Cold, Cnew):
        ids = O.frontier(self._g(part), policy, _np(moved).astype(np.uint8), _np(Cold).astype(np.int32),
                         _np(Cnew).astype(np.int32))
        m = torch.zeros(part.n, dtype=torch.uint8)
        m[torch.from_numpy(ids.astype(np.int64))] = 1
        return m

    def compress(self, part, k, lam, C, K):
        lvl = O.compress(self._g(part), _np(k), lam, _np(C).astype(np.int32), _np(K))
        cg = lvl.graph
        w = cg.weights if cg.weights is not None else np.ones(cg.indices.size)
        return (cg.n, torch.from_numpy(cg.indptr), torch.from_numpy(cg.indices), torch.from_numpy(w),
                torch.from_numpy(lvl.k), torch.from_numpy(lvl.mapping))

    def parallel_cc(self, indptr, indices, weights, total_weight, k, lam, opts):
        w = None if weights is None else np.ascontiguousarray(_np(weights), dtype=np.float64)
        g = O.Graph(indptr.numel() - 1, _np(indptr), _np(indices).astype(np.int32), w, total_weight)
        o = O.Opts(schedule=int(opts.schedule), frontier=int(opts.frontier_policy), refine=bool(opts.refine),
                   num_iter=int(opts.num_iter))
        return torch.from_numpy(O.parallel_cc(g, _np(k), lam, o))

    def merge(self, n, rows, cols, w, integral):
        r, c, ww = _np(rows).astype(np.int64), _np(cols).astype(np.int64), _np(w).astype(np.float64)
        key = r * (1 << 32) + c
        uk, inv = np.unique(key, return_inverse=True)
        sums = np.bincount(inv, weights=ww, minlength=uk.size) if uk.size else np.zeros(0)
        ip = np.zeros(n + 1, np.int64)
        np.cumsum(np.bincount(uk >> 32, minlength=n), out=ip[1:])
        wt = torch.from_numpy(sums.astype(np.int32)) if integral else torch.from_numpy(sums)
        return torch.from_numpy(ip), torch.from_numpy((uk & 0xffffffff).astype(np.int32)), wt

    def flatten(self, mapping, Cc, k):
        C, K = O.flatten(mapping.numel(), _np(mapping).astype(np.int32), _np(Cc).astype(np.int32), _np(k))
        return torch.from_numpy(C), torch.from_numpy(K)


def run_rank(rank, world, port, fn, args, out_path):
    """torch.multiprocessing entry: init gloo on 127.0.0.1, run fn, save result."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = fn(rank, world, *args)
        if rank == 0:
            torch.save(res, out_path)
    finally:
        dist.destroy_process_group()
