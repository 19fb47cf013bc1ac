import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1810_08403_b200 as sg
V, E = 232965, 114615892 // 4
g = sg.rmat_graph(V, E, seed=0)
grid = sg.ChunkGrid(g, V, gcn_weights=False)
m = sg.mpgcn_model(grid, [128, 64, 41])
m.load_features(torch.from_numpy(sg.synthetic_features(V, 128, seed=1)))
m.load_labels(np.random.default_rng(3).integers(0, 41, V))
for _ in range(2):
    m.train_step(0.01)
torch.cuda.synchronize()
st = {}
for _ in range(3):
    m.prof = []
    m.train_step(0.01)
    torch.cuda.synchronize()
    for k, v in m.stage_times().items():
        st[k] = st.get(k, 0) + v / 3
print(json.dumps({"lib": os.environ.get("SG_LIB_PATH", "default")[-20:], **{k: round(v, 2) for k, v in st.items() if "prop" in k}}))
