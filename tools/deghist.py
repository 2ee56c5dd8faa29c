import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2108_01731_b200.gen import rmat_device
g = rmat_device(24, 16, seed=24)
deg = (g.indptr[1:] - g.indptr[:-1]).cpu().numpy()
edges = [-1, 0, 1, 2, 4, 8, 16, 32, 128, 512, 1023, 2048, 10240, 100000, 10**9]
tot = deg.sum()
for a, b in zip(edges[:-1], edges[1:]):
    m = (deg > a) & (deg <= b)
    print(f"({a},{b}]: verts {m.sum():>10} edges {deg[m].sum():>12} ({100*deg[m].sum()/tot:.1f}%)")
print("max", deg.max(), "n", deg.size, "2m", tot)
