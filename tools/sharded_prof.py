"""Where the sharded driver's round-1 step spends its time at world size 1
(torch.profiler CUDA + CPU totals).  Run on a GPU box:
  torchrun --nproc-per-node 1 --master-addr 127.0.0.1 tools/sharded_prof.py"""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2108_01731_b200 as L  # noqa: E402
from paper_2108_01731_b200.dist import CudaBackend, ShardStats, make_part, sharded_best_moves  # noqa: E402

torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
dg = bench.build_graph_device(24, 16, 24)
n = dg.n
part = make_part(dg.indptr, dg.indices, None, float(dg.nnz // 2), 0, n, torch.device("cuda", 0))
be = CudaBackend()
opts = L.ParOptions(schedule="async", num_iter=1)
iota = torch.arange(n, dtype=torch.int32, device="cuda")


def step():
    C = iota.clone()
    K = torch.ones(n, dtype=torch.float64, device="cuda")
    sharded_best_moves(part, None, 0.85, C, K, opts, be, None, ShardStats())


for _ in range(3):
    step()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        step()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=60))
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=15, max_name_column_width=60))
dist.destroy_process_group()
