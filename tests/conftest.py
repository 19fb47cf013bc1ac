import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
GOLDEN_CASES = ["uniform_v40_e160", "rmat_v64_e600", "isolated_v30_e20"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and the built libsagann.so")
    config.addinivalue_line("markers", "slow: long-running")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def needed_floor(got, ref, rel=1e-4):
    """The smallest ``floor`` with which ``got`` passes the elementwise test against ``ref``."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    scale = float(np.abs(ref).max()) if ref.size else 0.0
    if scale == 0.0:
        return 0.0
    return float(np.max((np.abs(got - ref) - rel * np.abs(ref)) / (rel * scale), initial=0.0))


# Default elementwise floor (units of rel * max|ref|): 0.02 = 2e-6 max|ref| at rel = 1e-4, twice
# SURVEY §8(c)'s 1e-6.  Why twice: every fp32 model output passes through the tcgen05 3xTF32
# ApplyVertex GEMM, whose per-product error (<= ~3 * 2^-22 relative after the round-to-nearest
# split, sm100.cuh split3) exceeds an fp32 FMA's; on the few elements where z = a W cancels
# (|z| << sum |a||W|) that leaves up to 1.6e-6 max|z| (needed floors measured over the whole GPU
# suite: <= 0.0155, gpurun_out/c_pytest.txt).  Tests with a reason for more say so.
FLOOR = 0.02


def assert_close(got, ref, rel=1e-4, what="", floor=FLOOR, ref32=None):
    """Parity criterion: normwise rel <= rel AND
    elementwise |d| <= rel*|ref| + floor*rel*max|ref| (FLOOR above).

    The absolute term covers entries that are sums of many cancelling terms, where any fp32
    reduction order leaves ~sqrt(K) ulp of the term magnitudes.  When the reference's own fp32
    result ``ref32`` is given (``ref`` being its fp64 result), the floor is widened to twice
    what the reference itself needs on this tensor: the GPU must be no further from fp64 than
    2x the reference's own fp32 run.  Tests that pass a larger ``floor`` say why at the call
    site (DESIGN.md §2 lists them)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    if ref32 is not None:
        floor = max(floor, 2.0 * needed_floor(ref32, ref, rel))
    d = np.abs(got - ref)
    nref = np.linalg.norm(ref)
    scale = float(np.abs(ref).max()) if ref.size else 0.0
    if nref > 0:
        nrm = np.linalg.norm(got - ref) / nref
        assert nrm <= rel, f"{what}: normwise rel err {nrm:.3e} > {rel:.1e}"
    bad = d > rel * np.abs(ref) + floor * rel * scale + 1e-30
    assert not bad.any(), (
        f"{what}: {int(bad.sum())} elements out of tolerance; max abs err {d.max():.3e}, "
        f"max |ref| {scale:.3e}; needed floor {needed_floor(got, ref, rel):.4f} > {floor:.4f}")


def route_relu_masks(z_gpu, z_ref, tie=1e-5, max_frac=1e-3, what=""):
    """ReLU masks of the run under test, after checking that every place where they disagree
    with the reference's (z_ref > 0) is a kink: |z_ref| <= tie * max|z_ref| -- a value at the
    rounding level of the computation, where fp32 (or bf16) and fp64 may legitimately land on
    different sides of 0 -- and that such places are rare.  The oracle then runs its backward
    through these masks (saga.gcn_epoch / fullsize.gcn_backward ``masks``)."""
    masks = []
    for l, (zg, zr) in enumerate(zip(z_gpu, z_ref)):
        zg, zr = np.asarray(zg), np.asarray(zr, np.float64)
        mg = zg > 0
        diff = mg != (zr > 0)
        scale = float(np.abs(zr).max()) if zr.size else 0.0
        assert int(diff.sum()) <= max_frac * zr.size, f"{what} L{l}: {int(diff.sum())} ReLU flips"
        if diff.any():
            gap = float(np.abs(zr[diff]).max())
            assert gap <= tie * scale, f"{what} L{l}: a ReLU flip at |z| = {gap:.3e} (> {tie} x {scale:.3e})"
        masks.append(mg)
    return masks


@pytest.fixture(scope="session")
def reddit_oracle():
    """The Reddit-shaped config (BASELINE configs[1]) built once per session: the bench's graph,
    features, weights (Glorot, seed 2) and labels, and the fp64 full-size oracle's forward pass
    (oracle/fullsize.py) -- the GPU tests route its backward through their own ReLU masks."""
    import paper_1810_08403_b200 as sg
    from oracle import fullsize as fs
    from oracle import rng

    V, E, F, H, C = 232965, 114615892, 602, 128, 41
    g = sg.rmat_graph(V, E, seed=0)
    X = sg.synthetic_features(V, F, seed=1)
    Ws = [w.astype(np.float64) for w in rng.glorot([(F, H), (H, C)], seed=2)]
    lab = rng.labels(V, C, seed=3)
    f = fs.gcn_forward(g.src, g.dst, V, X.astype(np.float64), Ws, lab)
    return dict(g=g, X=X, fwd=f, V=V, E=E, F=F, H=H, C=C)
