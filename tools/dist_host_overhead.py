"""Host (CPU) time to enqueue one sharded training step (dist engine, NCCL, world 1):
if it approached the per-rank GPU time at N = 8 the GPUs would starve."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1810_08403_b200 as sg  # noqa: E402
from paper_1810_08403_b200 import dist as D  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29555")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
V, E, F, H, C = 232965, 114615892, 602, 128, 41
g = sg.rmat_graph(V, E, seed=0)
for model in ("gcn", "ggcn"):
    shard = D.ShardIndex(g, 1, 0, device="cuda:0", gcn_weights=model == "gcn")
    m = D.DistSAGA(shard, [F, H, C] if model == "gcn" else [128, 128, C], D.CudaCompute("cuda:0"), model=model)
    m.load_features(torch.from_numpy(sg.synthetic_features(V, m.dims[0], seed=1)))
    m.load_labels(np.random.default_rng(3).integers(0, C, V))
    for _ in range(2):
        m.train_step(0.01)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m.train_step(0.01)
    host = time.perf_counter() - t0
    torch.cuda.synchronize()
    gpu = time.perf_counter() - t0
    print(model, f"host enqueue {host * 1e3:.2f} ms, step wall {gpu * 1e3:.2f} ms", flush=True)
dist.destroy_process_group()
