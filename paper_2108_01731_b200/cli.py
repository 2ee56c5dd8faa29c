"""Command-line interface (the reference's ``io-gen-cli`` module,
``SPEC.md:390-450``).

    python -m paper_2108_01731_b200.cli cluster --input G.txt [--weighted]
        [--objective cc|modularity] [--resolution L | --gamma G] [--engine par]
        [--schedule sync|async] [--frontier all|cluster-nbrs|vertex-nbrs]
        [--refine | --no-refine] [--num-iter N] [--seed S] [--threads T]
        [--ground-truth PATH] [--labels PATH] [--out PATH] [--metrics PATH]
    python -m paper_2108_01731_b200.cli rmat --scale S (--edges M | --edge-factor F)
        [--a A --b B --c C --d D] [--seed S] --out PATH
    python -m paper_2108_01731_b200.cli eval --input G.txt --clustering PATH [...]

``run(config)`` is the library form.  Runtime is wall clock of the
clustering alone (no file I/O), as the paper reports it.
Only the parallel engine exists in this build: the sequential engines are
SURVEY.md §8f row 4 and raise a clear error.  Exit code 0 on success,
1 with a one-line diagnostic otherwise.
"""
from __future__ import annotations

import argparse
import sys
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import io as lio
from .eval import EvalReport, GroundTruth, ari_nmi, avg_precision_recall
from .graph import DeviceGraph, GraphError
from .louvain_par import ParOptions, parallel_cc
from .objective import ClusteringParams, cc_objective, clustering_from_labels, modularity_params


@dataclass
class RunConfig:
    """SPEC.md:395-397."""
    input: str
    weighted: bool = False
    objective: str = "cc"             # cc | modularity
    resolution: float = 0.85          # lambda (cc)
    gamma: float = 1.0                # modularity resolution
    engine: str = "par"
    options: ParOptions = field(default_factory=ParOptions)
    ground_truth: str | None = None
    labels: str | None = None
    out: str | None = None
    metrics: str | None = None


def _params(g: DeviceGraph, cfg: RunConfig) -> ClusteringParams:
    if cfg.objective == "cc":
        if not (0.0 < cfg.resolution < 1.0):
            raise GraphError("resolution (lambda) must lie in (0, 1)")
        return ClusteringParams(cfg.resolution)
    if cfg.objective == "modularity":
        return modularity_params(g, cfg.gamma)
    raise GraphError(f"unknown objective {cfg.objective!r}")


def _evaluate(g, p, c, cfg: RunConfig, id_map, rep: EvalReport) -> EvalReport:
    rep.objective = cc_objective(g, p, c)
    from .eval import cluster_stats
    num, mn, mx, mean = cluster_stats(c)
    rep.num_clusters = num
    rep.extra.update(min_cluster_size=mn, max_cluster_size=mx, mean_cluster_size=mean)
    if cfg.ground_truth:
        gt = lio.read_ground_truth(cfg.ground_truth, id_map, n=g.n)
        rep.avg_precision, rep.avg_recall = avg_precision_recall(c, gt)
    if cfg.labels:
        lab = lio.read_clustering(cfg.labels, id_map, n=g.n)
        rep.ari, rep.nmi = ari_nmi(c, lab)
    return rep


def run(cfg: RunConfig) -> EvalReport:
    """load, build params, cluster, evaluate, write outputs."""
    if cfg.engine not in ("par", "parallel"):
        raise GraphError(f"engine {cfg.engine!r} is not part of this build (only the parallel engine; "
                         "the sequential comparator is SURVEY.md §8f row 4)")
    host, id_map = lio.read_edge_list(cfg.input, cfg.weighted)
    g = DeviceGraph.from_graph(host)
    p = _params(g, cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    c = parallel_cc(g, p, cfg.options)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    rep = _evaluate(g, p, c, cfg, id_map, EvalReport(runtime_ms=ms, seed=int(cfg.options.seed)))
    if cfg.out:
        lio.write_clustering(cfg.out, c, id_map)
    if cfg.metrics:
        lio.write_metrics(cfg.metrics, rep)
    return rep


def _common(ap):
    ap.add_argument("--input", required=True)
    ap.add_argument("--weighted", action="store_true")
    ap.add_argument("--objective", choices=["cc", "modularity"], default="cc")
    ap.add_argument("--resolution", type=float, default=0.85)
    ap.add_argument("--gamma", type=float, default=1.0)
    ap.add_argument("--ground-truth")
    ap.add_argument("--labels")
    ap.add_argument("--metrics")


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="lambdacc-b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    c = sub.add_parser("cluster")
    _common(c)
    c.add_argument("--engine", default="par")
    c.add_argument("--schedule", choices=["sync", "async"], default="async")
    c.add_argument("--frontier", choices=["all", "cluster-nbrs", "vertex-nbrs"], default="vertex-nbrs")
    c.add_argument("--refine", dest="refine", action="store_true", default=True)
    c.add_argument("--no-refine", dest="refine", action="store_false")
    c.add_argument("--num-iter", type=int, default=10)
    c.add_argument("--seed", type=int, default=0)
    c.add_argument("--threads", type=int, default=0)
    c.add_argument("--out")
    r = sub.add_parser("rmat")
    r.add_argument("--scale", type=int, required=True)
    grp = r.add_mutually_exclusive_group(required=True)
    grp.add_argument("--edges", type=int)
    grp.add_argument("--edge-factor", type=int)
    r.add_argument("--a", type=float, default=0.5)
    r.add_argument("--b", type=float, default=0.1)
    r.add_argument("--c", type=float, default=0.1)
    r.add_argument("--d", type=float, default=0.3)
    r.add_argument("--seed", type=int, default=0)
    r.add_argument("--out", required=True)
    e = sub.add_parser("eval")
    _common(e)
    e.add_argument("--clustering", required=True)
    args = ap.parse_args(argv)
    try:
        if args.cmd == "cluster":
            frontier = {"all": "all", "cluster-nbrs": "cluster_neighbors", "vertex-nbrs": "vertex_neighbors"}
            opts = ParOptions(schedule=args.schedule, frontier_policy=frontier[args.frontier], refine=args.refine,
                              num_iter=args.num_iter, seed=args.seed, threads=args.threads)
            cfg = RunConfig(args.input, args.weighted, args.objective, args.resolution, args.gamma, args.engine,
                            opts, args.ground_truth, args.labels, args.out, args.metrics)
            rep = run(cfg)
            print(rep.to_json())
        elif args.cmd == "rmat":
            gen_rmat_file(args.scale, args.edges, args.edge_factor, args.a, args.b, args.c, args.d, args.seed,
                          args.out)
        else:
            cfg = RunConfig(args.input, args.weighted, args.objective, args.resolution, args.gamma,
                            ground_truth=args.ground_truth, labels=args.labels, metrics=args.metrics)
            host, id_map = lio.read_edge_list(cfg.input, cfg.weighted)
            g = DeviceGraph.from_graph(host)
            p = _params(g, cfg)
            lab = lio.read_clustering(args.clustering, id_map, n=g.n)
            if lab.size and (lab.min() < 0 or lab.max() >= g.n):
                raise GraphError("cluster ids must be vertex ids of the graph")
            cl = clustering_from_labels(lab, p)
            rep = _evaluate(g, p, cl, cfg, id_map, EvalReport())
            if cfg.metrics:
                lio.write_metrics(cfg.metrics, rep)
            print(rep.to_json())
    except (GraphError, FileNotFoundError, ValueError) as ex:
        print(f"error: {ex}", file=sys.stderr)
        return 1
    return 0


def gen_rmat_file(scale: int, edges: int | None, edge_factor: int | None, a: float, b: float, c: float,
                  d: float, seed: int, out: str) -> int:
    """SPEC.md:421-429 through the device generator; writes "u v" lines."""
    if scale > 30 or scale < 0:
        raise GraphError("scale must lie in [0, 30]")
    if abs(a + b + c + d - 1.0) > 1e-9 or min(a, b, c, d) < 0:
        raise GraphError("a + b + c + d must equal 1 (all >= 0)")
    samples = edges if edges is not None else edge_factor << scale
    from .gen import rmat_device
    g = rmat_device(scale, 0, a, b, c, seed=seed, samples=samples)
    indptr = g.indptr.cpu().numpy()
    indices = g.indices.cpu().numpy()
    src = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(indptr))
    keep = src < indices
    with open(out, "w") as f:
        f.write(f"# rmat scale={scale} samples={samples} a={a} b={b} c={c} d={d} seed={seed} m={int(keep.sum())}\n")
        np.savetxt(f, np.stack([src[keep], indices[keep]], 1), fmt="%d")
    return int(keep.sum())


if __name__ == "__main__":
    sys.exit(main())
