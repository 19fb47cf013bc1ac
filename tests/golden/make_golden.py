"""Generate golden fixtures by running the REAL reference (run here, not on the GPU box).

    PYTHONPATH=/root/repo python tests/golden/make_golden.py

Imports the unmodified reference ``sagastream.tensor`` from
/root/reference/pkg/src (read-only), composes the SAGA-NN GCN and G-GCN layers
from its primitives with its own ``Tape``/``backward`` (PAPER.md:552-564,
:172-173), and writes inputs + layer outputs + loss + parameter gradients to
``tests/golden/*.npz``.  Inputs come from the oracle's seeded generators so the
fixtures are reproducible.  The reference's scalar-seed defect
(tensor.py:33 vs :166) is worked around with a 0-d duck-typed
seed, as SURVEY.md Appendix B.7 pins.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, "/root/reference/pkg/src")

from sagastream import tensor as T  # noqa: E402  (the reference itself)

from oracle import graph as og  # noqa: E402
from oracle import rng  # noqa: E402


class Seed:
    """0-d seed shim: tensor.py:99-104 compares seed.shape to the recorded ()."""

    def __init__(self, dtype):
        self.shape = ()
        self.dtype = np.dtype(dtype)
        self.data = np.array(1.0, dtype=dtype)


def tens(x, dtype):
    return T.Tensor(np.asarray(x, dtype=dtype), dtype=dtype)


def run_gcn(X, Ws, labels, src, dst, w, V, dtype):
    tape = T.Tape()
    Wt = [tens(W, dtype) for W in Ws]
    for W in Wt:
        tape.watch(W)
    h = tens(X, dtype)
    wcol = tens(w.reshape(-1, 1), dtype)
    acts = []
    for W in Wt:
        es = T.take_rows(h, src, tape)                   # Scatter
        acc = T.mul(es, wcol, tape)                       # ApplyEdge: src x edge.data
        accum = T.segment_sum(acc, dst, V, tape)          # Gather(sum)
        z = T.matmul(accum, W, tape)                      # ApplyVertex
        h = T.relu(z, tape)
        acts.append((accum.to_numpy(), z.to_numpy(), h.to_numpy()))
    loss = T.softmax_cross_entropy(h, labels, tape)
    grads = T.backward(tape, Seed(dtype))
    return acts, loss.to_numpy(), [grads[W.tid] for W in Wt]


def run_ggcn(X, layers, labels, src, dst, V, dtype, hoisted=True):
    tape = T.Tape()
    lt = [tuple(tens(m, dtype) for m in L) for L in layers]
    for L in lt:
        for m in L:
            tape.watch(m)
    h = tens(X, dtype)
    acts = []
    counter = T.MatmulCounter()
    T.instrument_matmuls(counter)
    try:
        for (WH, WC, W) in lt:
            counter.stage = "apply_edge"
            if hoisted:
                P_ = T.matmul(h, WH, tape)
                Q_ = T.matmul(h, WC, tape)
                pre = T.add(T.take_rows(P_, src, tape), T.take_rows(Q_, dst, tape), tape)
            else:
                hs_ = T.take_rows(h, src, tape)
                hd_ = T.take_rows(h, dst, tape)
                pre = T.add(T.matmul(hs_, WH, tape), T.matmul(hd_, WC, tape), tape)
            eta = T.sigmoid(pre, tape)
            acc = T.mul(eta, T.take_rows(h, src, tape), tape)
            accum = T.segment_sum(acc, dst, V, tape)
            counter.stage = "apply_vertex"
            z = T.matmul(accum, W, tape)
            h = T.relu(z, tape)
            acts.append((accum.to_numpy(), z.to_numpy(), h.to_numpy()))
    finally:
        T.instrument_matmuls(None)
    loss = T.softmax_cross_entropy(h, labels, tape)
    grads = T.backward(tape, Seed(dtype))
    return acts, loss.to_numpy(), [tuple(grads[m.tid] for m in L) for L in lt], counter.counts


def run_mpgcn(X, layers, labels, src, dst, V, dtype, hoisted=True):
    """MP-GCN: acc = sigmoid(W_pool src + b), Gather(max), ReLU(W accum)."""
    tape = T.Tape()
    lt = [tuple(tens(m, dtype) for m in L) for L in layers]
    for L in lt:
        for m in L:
            tape.watch(m)
    h = tens(X, dtype)
    acts = []
    for (Wp, b, W) in lt:
        if hoisted:
            Y = T.sigmoid(T.add(T.matmul(h, Wp, tape), b, tape), tape)
            ys = T.take_rows(Y, src, tape)
        else:
            hs_ = T.take_rows(h, src, tape)
            ys = T.sigmoid(T.add(T.matmul(hs_, Wp, tape), b, tape), tape)
        accum = T.segment_max(ys, dst, V, tape=tape)
        z = T.matmul(accum, W, tape)
        h = T.relu(z, tape)
        acts.append((accum.to_numpy(), z.to_numpy(), h.to_numpy()))
    loss = T.softmax_cross_entropy(h, labels, tape)
    grads = T.backward(tape, Seed(dtype))
    return acts, loss.to_numpy(), [tuple(grads[m.tid] for m in L) for L in lt]


def run_commnet(X, layers, labels, src, dst, V, dtype):
    """CommNet: acc = edge.src, Gather(sum), ReLU(W_H vertex + W_C accum)."""
    tape = T.Tape()
    lt = [tuple(tens(m, dtype) for m in L) for L in layers]
    for L in lt:
        for m in L:
            tape.watch(m)
    h = tens(X, dtype)
    acts = []
    for (WH, WC) in lt:
        es = T.take_rows(h, src, tape)                    # Scatter; ApplyEdge = passthrough
        accum = T.segment_sum(es, dst, V, tape)           # Gather(sum)
        z = T.add(T.matmul(h, WH, tape), T.matmul(accum, WC, tape), tape)
        h = T.relu(z, tape)
        acts.append((accum.to_numpy(), z.to_numpy(), h.to_numpy()))
    loss = T.softmax_cross_entropy(h, labels, tape)
    grads = T.backward(tape, Seed(dtype))
    return acts, loss.to_numpy(), [tuple(grads[m.tid] for m in L) for L in lt]


def run_ggnn(X, layers, Wo, types, n_types, labels, src, dst, V, dtype):
    """GG-NN: acc = A(edge.data) (x) edge.src with the
    per-type matmul hoisted to the vertices (Y_t = h A_t, then a per-type
    Scatter routed by select_rows_by_label, tensor.py:358-386), Gather(sum), ApplyVertex =
    GRU(vertex, accum) in the Li et al. form without biases:
        z = s(a Wz + h Uz), r = s(a Wr + h Ur), c = tanh(a Wh + (r*h) Uh),
        h' = (1 - z)*h + z*c
    then a linear readout logits = h_L Wo and softmax-CE (no ReLU)."""
    tape = T.Tape()
    lt = []
    for (As, Wz, Uz, Wr, Ur, Wh, Uh) in layers:
        lt.append(([tens(m, dtype) for m in As],) + tuple(tens(m, dtype) for m in (Wz, Uz, Wr, Ur, Wh, Uh)))
    Wot = tens(Wo, dtype)
    for L in lt:
        for m in L[0]:
            tape.watch(m)
        for m in L[1:]:
            tape.watch(m)
    tape.watch(Wot)
    h = tens(X, dtype)
    ones = tens(np.ones(X.shape), dtype)
    acts = []
    for (As, Wz, Uz, Wr, Ur, Wh, Uh) in lt:
        Ys = [T.matmul(h, A, tape) for A in As]
        acc = T.select_rows_by_label(types, [T.take_rows(Y, src, tape) for Y in Ys], tape)
        a = T.segment_sum(acc, dst, V, tape)
        z = T.sigmoid(T.add(T.matmul(a, Wz, tape), T.matmul(h, Uz, tape), tape), tape)
        r = T.sigmoid(T.add(T.matmul(a, Wr, tape), T.matmul(h, Ur, tape), tape), tape)
        c = T.tanh(T.add(T.matmul(a, Wh, tape), T.matmul(T.mul(r, h, tape), Uh, tape), tape), tape)
        h = T.add(T.mul(T.sub(ones, z, tape), h, tape), T.mul(z, c, tape), tape)
        acts.append((a.to_numpy(), h.to_numpy()))
    logits = T.matmul(h, Wot, tape)
    loss = T.softmax_cross_entropy(logits, labels, tape)
    grads = T.backward(tape, Seed(dtype))
    gl = [([grads[m.tid] for m in L[0]],) + tuple(grads[m.tid] for m in L[1:]) for L in lt]
    return acts, logits.to_numpy(), loss.to_numpy(), gl, grads[Wot.tid]


CASES = [
    # name, V, E, F, H, C, generator, seed
    ("uniform_v40_e160", 40, 160, 12, 8, 3, "uniform", 11),
    ("rmat_v64_e600", 64, 600, 10, 6, 4, "rmat", 12),
    ("isolated_v30_e20", 30, 20, 7, 5, 3, "uniform", 13),  # many zero in-degree vertices
]


def make_case(name, V, E, F, H, C, gen, seed):
    if gen == "uniform":
        src, dst = rng.uniform_edges(V, E, seed=seed)
    else:
        src, dst = rng.rmat_edges(V, E, seed=seed)
    part = og.partition_2d(src, dst, V, V)
    order = part.csc_eid  # the dest-sorted (CSC) edge list the hot path runs on
    s, d = src[order].astype(np.int64), dst[order].astype(np.int64)
    out = dict(V=V, E=E, F=F, H=H, C=C, src_in=src, dst_in=dst, src=s, dst=d)
    lab = rng.labels(V, C, seed=3)
    out["labels"] = lab
    for dt, tag in ((np.float64, "f64"), (np.float32, "f32")):
        X = rng.features(V, F, seed=1, dtype=dt)
        w = og.gcn_edge_weights(s, d, V, dtype=dt)
        Ws = rng.glorot([(F, H), (H, C)], seed=2, dtype=dt)
        acts, loss, gW = run_gcn(X, Ws, lab, s, d, w, V, dt)
        out[f"gcn_{tag}_X"] = X
        out[f"gcn_{tag}_w"] = w
        for l, W in enumerate(Ws):
            out[f"gcn_{tag}_W{l}"] = W
            out[f"gcn_{tag}_a{l}"], out[f"gcn_{tag}_z{l}"], out[f"gcn_{tag}_h{l}"] = acts[l]
            out[f"gcn_{tag}_dW{l}"] = gW[l]
        out[f"gcn_{tag}_loss"] = loss
        # G-GCN: F -> F (gates) -> H ; H -> H -> C
        Ls = rng.glorot([(F, F), (F, F), (F, H), (H, H), (H, H), (H, C)], seed=2, dtype=dt)
        layers = [tuple(Ls[0:3]), tuple(Ls[3:6])]
        for hoisted in (True, False):
            acts, loss, gL, counts = run_ggcn(X, layers, lab, s, d, V, dt, hoisted)
            hp = "h" if hoisted else "u"
            for l, L in enumerate(layers):
                for k, m in enumerate(L):
                    out[f"ggcn_{tag}_L{l}_{k}"] = m
                    out[f"ggcn{hp}_{tag}_dL{l}_{k}"] = gL[l][k]
                out[f"ggcn{hp}_{tag}_a{l}"], out[f"ggcn{hp}_{tag}_z{l}"], out[f"ggcn{hp}_{tag}_h{l}"] = acts[l]
            out[f"ggcn{hp}_{tag}_loss"] = loss
            out[f"ggcn{hp}_{tag}_mm_edge"] = counts.get("apply_edge", 0)
        # MP-GCN: F -> pool 9 -> H ; H -> pool 7 -> C  (W_pool, b, W per layer)
        r = np.random.default_rng(2)
        Lm = []
        for fi, fp, fo in ((F, 9, H), (H, 7, C)):
            Lm.append((r.uniform(-0.5, 0.5, (fi, fp)).astype(dt), r.uniform(-0.2, 0.2, (fp,)).astype(dt),
                       r.uniform(-0.5, 0.5, (fp, fo)).astype(dt)))
        for hoisted in (True, False):
            acts, loss, gL = run_mpgcn(X, Lm, lab, s, d, V, dt, hoisted)
            hp = "h" if hoisted else "u"
            for l, L in enumerate(Lm):
                for k, m in enumerate(L):
                    out[f"mpgcn_{tag}_L{l}_{k}"] = m
                    out[f"mpgcn{hp}_{tag}_dL{l}_{k}"] = gL[l][k]
                out[f"mpgcn{hp}_{tag}_a{l}"], out[f"mpgcn{hp}_{tag}_z{l}"], _ = acts[l]
            out[f"mpgcn{hp}_{tag}_loss"] = loss
        # CommNet: F -> H -> C, params [W_H, W_C] per layer
        Lc = rng.glorot([(F, H), (F, H), (H, C), (H, C)], seed=2, dtype=dt)
        layers = [tuple(Lc[0:2]), tuple(Lc[2:4])]
        acts, loss, gL = run_commnet(X, layers, lab, s, d, V, dt)
        for l, L in enumerate(layers):
            for k, m in enumerate(L):
                out[f"commnet_{tag}_L{l}_{k}"] = m
                out[f"commnet_{tag}_dL{l}_{k}"] = gL[l][k]
            out[f"commnet_{tag}_a{l}"], out[f"commnet_{tag}_z{l}"], _ = acts[l]
        out[f"commnet_{tag}_loss"] = loss
        # GG-NN: 2 propagation steps at state width F, 3 edge types, readout F -> C
        nt = 3
        types_in = rng.labels(E, nt, seed=5)
        types = types_in[order]
        out["ggnn_types"] = types
        r = np.random.default_rng(7)
        Lg = []
        for _ in range(2):
            As = [r.uniform(-0.4, 0.4, (F, F)).astype(dt) for _ in range(nt)]
            Lg.append((As,) + tuple(r.uniform(-0.4, 0.4, (F, F)).astype(dt) for _ in range(6)))
        Wo = r.uniform(-0.5, 0.5, (F, C)).astype(dt)
        acts, logits, loss, gl, gWo = run_ggnn(X, Lg, Wo, types, nt, lab, s, d, V, dt)
        for l, L in enumerate(Lg):
            for t, A in enumerate(L[0]):
                out[f"ggnn_{tag}_L{l}_A{t}"] = A
                out[f"ggnn_{tag}_dL{l}_A{t}"] = gl[l][0][t]
            for k in range(6):
                out[f"ggnn_{tag}_L{l}_{k}"] = L[1 + k]
                out[f"ggnn_{tag}_dL{l}_{k}"] = gl[l][1 + k]
            out[f"ggnn_{tag}_a{l}"], out[f"ggnn_{tag}_h{l}"] = acts[l]
        out[f"ggnn_{tag}_Wo"] = Wo
        out[f"ggnn_{tag}_dWo"] = gWo
        out[f"ggnn_{tag}_logits"] = logits
        out[f"ggnn_{tag}_loss"] = loss
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print("wrote", name)


if __name__ == "__main__":
    for case in CASES:
        make_case(*case)
