"""Training steps of a bench.py workload after warm-up (for ncu captures).

    python tools/profile_step.py [config] [steps]      (default: reddit 2)

    ncu --set full --clock-control none -k regex:'prop_kernel|gemm_tma' --launch-skip 8 \
        --launch-count 8 -o gpurun_out/step python tools/profile_step.py reddit
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1810_08403_b200 as sg  # noqa: E402
from bench import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "reddit"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = dict(CONFIGS[name])
if len(sys.argv) > 3:  # override edge count (smaller power-law captures)
    cfg["E"] = int(float(sys.argv[3]))
V, E, F, H, C = cfg["V"], cfg["E"], cfg["F"], cfg["H"], cfg["C"]
g = (sg.rmat_graph if cfg["graph"] == "rmat" else sg.uniform_graph)(V, E, seed=0)
grid = sg.ChunkGrid(g, V, gcn_weights=cfg["model"] == "gcn")
m = (sg.gcn_model if cfg["model"] == "gcn" else sg.ggcn_model)(grid, [F, H, C])
m.load_features(torch.from_numpy(sg.synthetic_features(V, F, seed=1)))
m.load_labels(np.random.default_rng(3).integers(0, C, V))
for _ in range(steps):
    m.train_step(0.01)
torch.cuda.synchronize()
print("loss", m.loss.item())
