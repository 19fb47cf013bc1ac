"""GG-NN executor on the chunk grid.

The layer program is ``build_ggnn(F, n_types)``: ApplyEdge = A(edge.data) (x) edge.src,
Gather(sum), ApplyVertex = GRU(vertex, accum).  ``optimize`` hoists the typed matmul to
the vertices: Y = h [A_0 | A_1 | ...] is ONE GEMM per layer, and the SAG
phase becomes a fused PASS gather over Y viewed as [V * n_types, bs] with a per-graph
typed index (row src * n_types + type) -- no per-edge matmul, no edge tensor in HBM.
Its dual is a PASS gather over a per-type CSR (rows src * n_types + type, each row's
edges in CSR order), i.e. take_rows' backward per type (tensor.py:431-434).

ApplyVertex runs the GRU as stacked GEMMs on the tcgen05 GEMM (a [Wz|Wr|Wh], h [Uz|Ur],
(r*h) Uh) with the element-wise stages fused in four kernels (csrc/gru.cu).  A linear
readout logits = h_L Wo feeds softmax-CE (no ReLU).  Parity: tests/test_gpu_kernels.py
(typed gather bitwise vs the oracle; model vs the real reference's golden outputs).
"""

import numpy as np
import torch

from . import _lib
from . import graph as G
from . import kernels as K
from . import program as prog
from .errors import ConfigError, NumericError, ProgramError, ShapeError


def _ld(n, align=4):
    return (n + align - 1) // align * align


def _buf(r, c, device):
    return torch.zeros((r, c), dtype=torch.float32, device=device)


class GGNNModel:
    """``layers`` GG-NN propagation steps at state width F over ``n_types`` edge types,
    then a readout to ``C`` classes.  ``edge_types``: the type of every INPUT edge
    (the Graph's edge order).  Parameters per layer (the reference's order):
    ([A_0 .. A_{T-1}], W_z, U_z, W_r, U_r, W_h, U_h), then W_o."""

    def __init__(self, grid, F, n_types, C, edge_types, layers=2, weights=None, seed=2,
                 device="cuda", strict=True, gemm_prec=_lib.GEMM_TF32X3):
        if not torch.cuda.is_available():
            raise RuntimeError("GGNNModel needs a CUDA device (no CPU fallback)")
        q, reports = prog.optimize(prog.build_ggnn(F, n_types))
        if q.fused is None or q.fused.kind != "typed" or prog.vertex_form(q)[0] != "gru":
            raise ProgramError("GG-NN program did not lower to a typed gather + GRU")
        self.reports = reports
        types = np.asarray(edge_types, np.int64).reshape(-1)
        if types.shape[0] != grid.E:
            raise ShapeError(f"need one edge type per edge ({grid.E}), got {types.shape[0]}")
        if types.size and (types.min() < 0 or types.max() >= n_types):
            raise ShapeError("edge label out of range for the parameter family")
        if grid.V * n_types >= 2 ** 31:
            raise ConfigError("V * edge types must fit the int32 typed index")
        self.grid, self.F, self.T, self.C, self.L = grid, int(F), int(n_types), int(C), int(layers)
        self.device, self.strict, self.prec = torch.device(device), strict, gemm_prec
        self.bs = _ld(self.F)
        self.ws = K.Workspace(self.device)
        self._index(types)
        self._alloc()
        self.set_weights(*(weights if weights is not None else self.init_weights(seed)))

    # ------------------------------------------------------------------ typed indices
    def _index(self, types):
        g, T = self.grid, self.T
        part, split = g.part, g.split_edges
        self.tcsc, self.tcsr = {}, {}
        for (i, j) in g.csc:
            ch = part.chunk(i, j)
            n_i, n_j = int(part.sizes[i]), int(part.sizes[j])
            idx = (ch["csc_idx"].astype(np.int64) * T + types[ch["csc_eid"]]).astype(np.int32)
            self.tcsc[(i, j)] = G.PassIndex(ch["csc_ptr"], idx, None, n_j, split, self.device)
            src_local = np.repeat(np.arange(n_i, dtype=np.int64), np.diff(ch["csr_ptr"]))
            key = src_local * T + types[ch["csr_eid"]]
            order = np.argsort(key, kind="stable")
            ptr = np.zeros(n_i * T + 1, np.int64)
            np.cumsum(np.bincount(key, minlength=n_i * T), out=ptr[1:])
            self.tcsr[(i, j)] = G.PassIndex(ptr, ch["csr_idx"][order].astype(np.int32), None,
                                            n_i * T, split, self.device)

    # ------------------------------------------------------------------ buffers
    def _alloc(self):
        V, F, T, bs, dev = self.grid.V, self.F, self.T, self.bs, self.device
        Cp = _ld(self.C)
        self.h = [_buf(V, bs, dev)[:, :F] for _ in range(self.L + 1)]
        self.X = self.h[0]
        self.Y = [_buf(V, T * bs, dev) for _ in range(self.L)]
        self.a = [_buf(V, bs, dev)[:, :F] for _ in range(self.L)]
        self.G1 = [_buf(V, 3 * bs, dev) for _ in range(self.L)]
        self.G2 = [_buf(V, 2 * bs, dev) for _ in range(self.L)]
        self.G3 = [_buf(V, bs, dev) for _ in range(self.L)]
        self.z, self.r, self.rh, self.c = ([_buf(V, bs, dev)[:, :F] for _ in range(self.L)] for _ in range(4))
        self.logits = _buf(V, Cp, dev)[:, : self.C]
        self.dlogits = _buf(V, Cp, dev)[:, : self.C]
        self.g = [_buf(V, bs, dev)[:, :F] for _ in range(self.L + 1)]  # g[l] = dLoss/dh[l]
        self.D3 = _buf(V, 3 * bs, dev)          # [gzp | grp | gcp], padding columns stay 0
        self.grh = _buf(V, bs, dev)[:, :F]
        self.ga = _buf(V, bs, dev)[:, :F]
        self.dY = _buf(V, T * bs, dev)
        self.tmp = _buf(V, bs, dev)[:, :F]
        # parameters: padded stacks (column blocks at stride bs), grads alike
        self.P = []
        for _ in range(self.L):
            self.P.append({"A": _buf(F, T * bs, dev), "W3": _buf(F, 3 * bs, dev),
                           "U2": _buf(F, 2 * bs, dev), "Uh": _buf(F, bs, dev)})
        self.dP = [{k: torch.zeros_like(v) for k, v in p.items()} for p in self.P]
        self.Wo = _buf(F, Cp, dev)
        self.dWo = torch.zeros_like(self.Wo)
        self.labels = torch.zeros(V, dtype=torch.int64, device=dev)
        self.loss = torch.zeros(1, dtype=torch.float32, device=dev)
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)
        self.nonfinite = torch.zeros(1, dtype=torch.int32, device=dev)

    # ------------------------------------------------------------------ parameters
    def init_weights(self, seed=2):
        """Glorot-uniform (F, F) matrices from default_rng(seed) in parameter order."""
        rng = np.random.default_rng(seed)
        F = self.F

        def glorot(r, c):
            lim = np.sqrt(6.0 / (r + c))
            return rng.uniform(-lim, lim, (r, c)).astype(np.float32)

        layers = []
        for _ in range(self.L):
            As = [glorot(F, F) for _ in range(self.T)]
            layers.append((As,) + tuple(glorot(F, F) for _ in range(6)))
        return layers, glorot(F, self.C)

    def _blocks(self, l):
        """Views of layer l's parameters (and gradients) as the reference's matrices."""
        F, bs = self.F, self.bs
        out = []
        for P in (self.P[l], self.dP[l]):
            As = [P["A"][:, t * bs: t * bs + F] for t in range(self.T)]
            W3, U2, Uh = P["W3"], P["U2"], P["Uh"]
            out.append((As, W3[:, :F], U2[:, :F], W3[:, bs:bs + F], U2[:, bs:bs + F],
                        W3[:, 2 * bs:2 * bs + F], Uh[:, :F]))
        return out

    def set_weights(self, layers, Wo):
        if len(layers) != self.L:
            raise ShapeError(f"need {self.L} layers of parameters")
        for l, L in enumerate(layers):
            As, *rest = L
            if len(As) != self.T:
                raise ShapeError(f"need {self.T} edge-type matrices")
            dst = self._blocks(l)[0]
            for t, A in enumerate(As):
                dst[0][t].copy_(torch.as_tensor(np.asarray(A, np.float32)))
            for d, w in zip(dst[1:], rest):
                d.copy_(torch.as_tensor(np.asarray(w, np.float32)))
        self.Wo[:, : self.C].copy_(torch.as_tensor(np.asarray(Wo, np.float32)))

    def _host(self, which):
        layers = []
        for l in range(self.L):
            As, *rest = self._blocks(l)[which]
            layers.append(([a.cpu().numpy().copy() for a in As],) + tuple(x.cpu().numpy().copy() for x in rest))
        Wo = (self.Wo if which == 0 else self.dWo)[:, : self.C].cpu().numpy().copy()
        return layers, Wo

    def weights(self):
        return self._host(0)

    def grads(self):
        return self._host(1)

    def load_features(self, X):
        X = torch.as_tensor(X)
        if X.shape[0] != self.grid.V or X.shape[1] < self.F:
            raise ShapeError(f"features must be [V={self.grid.V}, {self.F}]")
        self.X.copy_(X[:, : self.F], non_blocking=True)

    def load_labels(self, y):
        self.labels.copy_(torch.as_tensor(np.asarray(y, np.int64)), non_blocking=True)

    # ------------------------------------------------------------------ helpers
    def _rows(self, t, k):
        b = self.grid.begin(k)
        return t[b: b + self.grid.size(k)]

    def _typed_rows(self, Ybuf, k):
        """Interval k's rows of a [V, T*bs] per-type table viewed [n_k * T, bs][:, :F]."""
        n = self.grid.size(k)
        return self._rows(Ybuf, k).reshape(n * self.T, self.bs)[:, : self.F]

    def _gemm(self, A, B, C, **kw):
        K.gemm(A, B, C, prec=self.prec, ws=self.ws, **kw)

    def _check(self, rc):
        _lib.check(rc)

    # ------------------------------------------------------------------ step
    def forward(self):
        g, P = self.grid, self.grid.P
        F, bs, V = self.F, self.bs, self.grid.V
        lib, st = _lib.lib, _lib.stream_handle()
        for l in range(self.L):
            h, Pm = self.h[l], self.P[l]
            self._gemm(h, Pm["A"], self.Y[l])                        # Y = h [A_0 | A_1 | ...]
            for j in range(P):                                        # typed Gather(sum)
                chain = [i for i in range(P) if (i, j) in self.tcsc]
                if not chain:
                    self._rows(self.a[l], j).zero_()
                for k, i in enumerate(chain):
                    K.propagate(self.tcsc[(i, j)], _lib.PROP_PASS, self._typed_rows(self.Y[l], i),
                                self._rows(self.a[l], j), F, accumulate=k > 0, ws=self.ws)
            self._gemm(self.a[l], Pm["W3"], self.G1[l])              # a [Wz | Wr | Wh]
            self._gemm(h, Pm["U2"], self.G2[l])                      # h [Uz | Ur]
            self._check(lib.sg_gru_gates(V, F, self.G1[l].data_ptr(), 3 * bs, self.G2[l].data_ptr(),
                                         2 * bs, bs, h.data_ptr(), bs, self.z[l].data_ptr(),
                                         self.r[l].data_ptr(), self.rh[l].data_ptr(), bs, st))
            self._gemm(self.rh[l], Pm["Uh"], self.G3[l])             # (r*h) Uh
            self._check(lib.sg_gru_out(V, F, self.G1[l].data_ptr(), 3 * bs, bs, self.G3[l].data_ptr(),
                                       bs, self.z[l].data_ptr(), h.data_ptr(), bs, self.c[l].data_ptr(),
                                       self.h[l + 1].data_ptr(), bs, bs, st))
        self._gemm(self.h[self.L], self.Wo, self.logits_full())      # readout
        return self.logits

    def logits_full(self):
        return self.logits._base if self.logits._base is not None else self.logits

    def backward(self):
        g, P = self.grid, self.grid.P
        F, bs, V = self.F, self.bs, self.grid.V
        lib, st = _lib.lib, _lib.stream_handle()
        K.softmax_xent(self.logits, self.labels, self.loss, self.dlogits, self.err, relu_input=False,
                       ws=self.ws)
        hL = self.h[self.L]
        self._gemm(self.dlogits, self.Wo[:, : self.C], self.g[self.L], trans_b=True)
        self._gemm(hL, self.dlogits, self.dWo[:, : self.C], trans_a=True)
        for l in range(self.L - 1, -1, -1):
            h, Pm, dPm = self.h[l], self.P[l], self.dP[l]
            gh = self.g[l]
            self._check(lib.sg_gru_bwd1(V, F, self.g[l + 1].data_ptr(), bs, self.z[l].data_ptr(),
                                        self.c[l].data_ptr(), bs, h.data_ptr(), bs, self.D3.data_ptr(),
                                        3 * bs, bs, gh.data_ptr(), bs, st))
            gcp = self.D3[:, 2 * bs: 2 * bs + F]
            self._gemm(gcp, Pm["Uh"][:, :F], self.grh, trans_b=True)     # grh = gcp Uh^T
            self._gemm(self.rh[l], gcp, dPm["Uh"][:, :F], trans_a=True)   # dUh = (r*h)^T gcp
            self._check(lib.sg_gru_bwd2(V, F, self.grh.data_ptr(), bs, self.r[l].data_ptr(), bs,
                                        h.data_ptr(), bs, gh.data_ptr(), bs, self.D3.data_ptr(), 3 * bs,
                                        bs, st))
            self._gemm(self.D3, Pm["W3"], self.ga, trans_b=True)          # ga = D3 [Wz|Wr|Wh]^T
            self._gemm(self.a[l], self.D3, dPm["W3"], trans_a=True)       # [dWz|dWr|dWh] = a^T D3
            D2 = self.D3[:, : 2 * bs]
            self._gemm(D2, Pm["U2"], self.tmp, trans_b=True)              # [gzp|grp] [Uz|Ur]^T
            self._gemm(h, D2, dPm["U2"], trans_a=True)                    # [dUz|dUr] = h^T [gzp|grp]
            K.ewise(0, gh, self.tmp, gh)
            for i in range(P):                                            # typed dual (CSR)
                chain = [j for j in range(P) if (i, j) in self.tcsr]
                if not chain:
                    self._rows(self.dY, i).zero_()
                for k, j in enumerate(chain):
                    K.propagate(self.tcsr[(i, j)], _lib.PROP_PASS, self._rows(self.ga, j),
                                self._typed_rows(self.dY, i), F, accumulate=k > 0, ws=self.ws)
            self._gemm(h, self.dY, dPm["A"], trans_a=True)                # [dA_t] = h^T dY
            self._gemm(self.dY, Pm["A"], self.tmp, trans_b=True)          # sum_t dY_t A_t^T
            K.ewise(0, gh, self.tmp, gh)
        if self.strict:
            self.nonfinite.zero_()
            K.check_finite(self.loss, self.nonfinite)
            for dPm in self.dP:
                for t in dPm.values():
                    K.check_finite(t, self.nonfinite)
            K.check_finite(self.dWo, self.nonfinite)
        return self.loss

    def sgd(self, lr):
        for Pm, dPm in zip(self.P, self.dP):
            for k in Pm:
                K.sgd(Pm[k], dPm[k], lr)
        K.sgd(self.Wo, self.dWo, lr)

    def train_step(self, lr=0.01):
        self.forward()
        self.backward()
        self.sgd(lr)
        return self.loss

    def check_status(self):
        if int(self.err.item()):
            raise ShapeError("label out of range [0, classes)")
        if self.strict and int(self.nonfinite.item()):
            raise NumericError("non-finite value produced in the training step")


def ggnn_model(grid, F, n_types, C, edge_types, **kw):
    return GGNNModel(grid, F, n_types, C, edge_types, **kw)
