"""Chunk-dataflow executor for SAGA-NN models (forward, backward, SGD) on one GPU.

Lowers each optimized LayerProgram (program.optimize) onto the fused sm_100a
kernels, following the reference's dataflow-builder / scheduler contracts:

* forward, Locality order: for every destination interval
  j, all source intervals i in ascending order run ``fused_gather_chunk`` into
  the resident accumulator A_j, then ApplyVertex;
* backward, stages in reverse: backward
  ApplyVertex (GEMMs) -> backward Gather/ApplyEdge/Scatter fused into one pass
  over the transposed (CSR) index, with the ReLU mask of the layer below fused
  into its epilogue;
* loss: softmax cross-entropy on ReLU(z_L) (tensor.py:487-506),
  update W <- W - lr dW.

All device buffers are allocated once; ``capture()`` records a whole training
step into a CUDA graph, so an epoch is one graph launch.
"""

import os

import numpy as np
import torch

from . import _lib
from . import kernels as K
from . import program as prog
from .errors import ConfigError, NumericError, ProgramError, ShapeError


def _ld(n, align=4):
    return (n + align - 1) // align * align


def _mat(V, n, device, align=4, dtype=torch.float32):
    """[V, n] view of a zero-padded [V, ld] buffer (16-byte aligned rows: ld a multiple of 4
    fp32 / 8 bf16 elements)."""
    if dtype == torch.bfloat16:
        align = max(align, 8)
    return torch.zeros((V, _ld(n, align)), dtype=dtype, device=device)[:, :n]


def _param(L, r, c, device):
    """A parameter and its gradient as [r, c] views of zero-padded [r, ld] buffers (16-B
    rows, so the tensor-core GEMM takes the TMA path); SGD runs over the whole buffers
    (the padding columns of W and dW stay zero)."""
    wb = torch.zeros((r, _ld(c)), dtype=torch.float32, device=device)
    gb = torch.zeros_like(wb)
    L.sgd_pairs.append((wb, gb))
    return wb[:, :c], gb[:, :c]


class _Layer:
    pass


def lower_programs(programs, reorder=False):
    """hoist + fuse + validate each LayerProgram and pick its kernel lowering (host only,
    no device work): fused gather kind (gcn / pass / ggcn / max / max_pool) and
    ApplyVertex form.  Raises ProgramError for programs the executor cannot run
    exactly as written (instead of running a different model)."""
    layers = []
    for p in programs:
        q, reports = prog.optimize(p, reorder=reorder)
        diags = prog.validate_program(q)
        if diags:
            raise ProgramError("; ".join(diags))
        if q.fused is None or q.fused.kind not in ("gcn", "pass", "ggcn", "max", "max_pool"):
            raise ProgramError(f"layer ApplyEdge {p.apply_edge!r} has no fused kernel "
                               f"({reports[-1].blocker or (q.fused and q.fused.kind)})")
        form = prog.vertex_form(q)
        if form is None or form[0] not in ("w", "hc"):
            raise ProgramError("ApplyVertex must be ReLU(W accum) or ReLU(W_H vertex + "
                               "W_C accum) for the fused executor"
                               + (" (GRU ApplyVertex: use ggnn.GGNNModel)"
                                  if form is not None else ""))
        if form[0] == "hc" and q.fused.kind not in ("gcn", "pass"):
            raise ProgramError("ReLU(W_H vertex + W_C accum) is lowered for sum gathers only")
        L = _Layer()
        L.prog, L.kind, L.F, L.O = q, q.fused.kind, q.f_in, q.f_out
        L.vform, L.wname = form[0], form[1:]
        L.gate = q.fused.params
        # reorder_linear_gather: Y = h W per vertex, then propagate Y (width O)
        L.reorder = bool(getattr(q, "reorder", False))
        # accumulator width: the pooled width for MP-GCN, else the input width
        L.Aw = q.params[L.gate[0]][1] if L.kind == "max_pool" else q.f_in
        layers.append(L)
    return layers


class SAGAModel:
    """An L-layer SAGA-NN model bound to a ChunkGrid and executed by libsagann kernels.

    ``programs`` are LayerPrograms (e.g. ``build_gcn``/``build_ggcn``); each is run
    through ``hoist_vertex_computation`` + ``fuse_sag`` and must lower to a fused
    gather (gcn / pass / ggcn) followed by ApplyVertex = ReLU(W accum)."""

    def __init__(self, programs, grid, weights=None, *, seed=2, gemm_prec=_lib.GEMM_TF32X3,
                 device="cuda", strict=True, schedule="locality", reorder=False, dtype="f32"):
        if not torch.cuda.is_available():
            raise RuntimeError("SAGAModel needs a CUDA device (no CPU fallback)")
        if schedule not in ("locality", "dest_order"):
            raise ConfigError(f"unknown schedule '{schedule}'; valid: locality, dest_order")
        self.schedule = schedule
        self.grid, self.device, self.strict = grid, torch.device(device), strict
        self.V = grid.V
        self.gemm_prec = gemm_prec
        self.ws = K.Workspace(self.device)
        self.reorder = bool(reorder)
        self.layers = lower_programs(programs, self.reorder)
        if dtype not in ("f32", "bf16"):
            raise ConfigError(f"unknown dtype '{dtype}'; valid: f32, bf16")
        # bf16 storage mode: the GATHERED rows are bf16 -- the input features, every hidden
        # activation h (the next layer's gathered rows) and the backward's dA -- so the
        # propagation passes read half the bytes; every gather accumulates and writes fp32 (a,
        # dz), the ApplyVertex GEMMs run 3xTF32 on fp32 operands and round only their h / dA
        # outputs to bf16.  (bf16 aggregates / gradients as GEMM operands cost 5-7% of dW0.)
        self.bf16 = dtype == "bf16"
        if self.bf16:
            if any(L.kind not in ("gcn", "pass") or L.vform != "w" or L.reorder for L in self.layers):
                raise ConfigError("bf16 storage is implemented for sum-gather layers with "
                                  "ApplyVertex = ReLU(W accum) (GCN), without reorder")
        dims = [(L.F, L.O) for L in self.layers]
        for a, b in zip(dims, dims[1:]):
            if a[1] != b[0]:
                raise ShapeError(f"layer widths do not chain: {a} -> {b}")
        self._alloc()
        self.set_weights(weights if weights is not None else self.init_weights(seed))
        self.graph = None
        self.prof = None

    # ------------------------------------------------------------------ parameters
    def param_shapes(self):
        out = []
        for L in self.layers:
            if L.kind == "ggcn":
                out += [(L.F, L.F), (L.F, L.F), (L.F, L.O)]
            elif L.kind == "max_pool":
                out += [(L.F, L.Aw), (L.Aw,), (L.Aw, L.O)]
            elif L.vform == "hc":
                out += [(L.F, L.O), (L.F, L.O)]
            else:
                out += [(L.F, L.O)]
        return out

    def init_weights(self, seed=2):
        """Glorot-uniform matrices (zero biases) from default_rng(seed) in parameter order
        (SURVEY.md §8(d))."""
        rng = np.random.default_rng(seed)
        out = []
        for shape in self.param_shapes():
            if len(shape) == 1:
                out.append(np.zeros(shape, np.float32))
                continue
            fin, fout = shape
            lim = np.sqrt(6.0 / (fin + fout))
            out.append(rng.uniform(-lim, lim, (fin, fout)).astype(np.float32))
        return out

    def set_weights(self, weights):
        flat = list(weights)
        if len(flat) != len(self.param_shapes()):
            raise ShapeError("wrong number of weight matrices")
        k = 0
        for L in self.layers:
            for t in L.params:
                w = torch.as_tensor(np.asarray(flat[k], np.float32))
                if w.dim() == 1 and t.dim() == 2 and t.shape[0] == 1:
                    w = w.reshape(1, -1)  # bias vector
                if tuple(w.shape) != tuple(t.shape):
                    raise ShapeError(f"weight {k} has shape {tuple(w.shape)}, want {tuple(t.shape)}")
                t.copy_(w)
                k += 1

    @staticmethod
    def _host(t, L):
        x = t.detach().cpu().numpy().copy()
        return x.reshape(-1) if t is getattr(L, "bias", None) or t is getattr(L, "dbias", None) else x

    def weights(self):
        return [self._host(t, L) for L in self.layers for t in L.params]

    def grads(self):
        return [self._host(t, L) for L in self.layers for t in L.dparams]

    # ------------------------------------------------------------------ buffers
    def _alloc(self):
        V, dev = self.V, self.device
        for n, L in enumerate(self.layers):
            F, O = L.F, L.O
            L.sgd_pairs = []
            if L.vform != "hc":
                L.W, L.dW = _param(L, L.Aw, O, dev)
            if L.vform == "hc":
                # CommNet: z = [h | accum] @ [W_H; W_C] as ONE GEMM over a per-vertex [h | a]
                # buffer (16-B padded halves, zero pad rows in the stacked weights); its
                # backward dz @ [W_H; W_C]^T writes [dh_direct | da] in one pass too.
                ldF = _ld(F)
                L.HA = torch.zeros((V, 2 * ldF), dtype=torch.float32, device=dev)
                L.hin, L.a = L.HA[:, :F], L.HA[:, ldF:ldF + F]
                L.W, L.dW = _param(L, 2 * ldF, O, dev)
                L.WH, L.WC = L.W[:F], L.W[ldF:ldF + F]
                L.dWH, L.dWC = L.dW[:F], L.dW[ldF:ldF + F]
                L.dHA = torch.zeros((V, 2 * ldF), dtype=torch.float32, device=dev)
                L.da = L.dHA[:, ldF:ldF + F]
                L.gin = L.HA
                L.params, L.dparams = [L.WH, L.WC], [L.dWH, L.dWC]
                L.z = _mat(V, O, dev)
                L.dz = _mat(V, O, dev)
                continue
            if L.kind in ("max", "max_pool"):
                A = L.Aw
                L.hin = None
                L.arg = torch.zeros((V, _ld(A)), dtype=torch.int32, device=dev)[:, :A]
                L.da = _mat(V, A, dev)
                L.dY = _mat(V, A, dev)
                L.params, L.dparams = [L.W], [L.dW]
                if L.kind == "max_pool":
                    L.Y = _mat(V, A, dev)
                    L.Wp, L.dWp = _param(L, F, A, dev)
                    L.bias, L.dbias = _param(L, 1, A, dev)
                    L.params, L.dparams = [L.Wp, L.bias, L.W], [L.dWp, L.dbias, L.dW]
                    self._ones = torch.ones((V, 1), dtype=torch.float32, device=dev)
                L.a = _mat(V, A, dev)
                L.z = _mat(V, O, dev)
                L.dz = _mat(V, O, dev)
                continue
            if L.kind == "ggcn":
                L.goff = _ld(F)
                L.HP = torch.zeros((V, 2 * L.goff), dtype=torch.float32, device=dev)
                L.GQ = torch.zeros((V, 2 * L.goff), dtype=torch.float32, device=dev)
                L.hin = L.HP[:, :F]
                L.Pv = L.HP[:, L.goff:L.goff + F]
                L.Qv = L.GQ[:, L.goff:L.goff + F]
                L.dAv = L.GQ[:, :F]
                L.WH, L.dWH = _param(L, F, F, dev)
                L.WC, L.dWC = _param(L, F, F, dev)
                L.dQ, L.dP, L.dHt = _mat(V, F, dev), _mat(V, F, dev), _mat(V, F, dev)
                L.S = _mat(V, F, dev)  # sum_e (h eta)(1 - eta) per destination (GGCN_FWD_S)
                L.params = [L.WH, L.WC, L.W]
                L.dparams = [L.dWH, L.dWC, L.dW]
            else:
                L.hin = None  # set below (previous layer's ReLU output or X)
                L.da = _mat(V, F, dev) if not L.reorder else None
                L.params = [L.W]
                L.dparams = [L.dW]
                if L.reorder:
                    L.Y, L.dY = _mat(V, O, dev), _mat(V, O, dev)
            L.a = _mat(V, F, dev) if not getattr(L, "reorder", False) else None
            L.z = _mat(V, O, dev)
            L.dz = _mat(V, O, dev)
        for n, L in enumerate(self.layers):
            if getattr(L, "gin", None) is None:
                L.gin = L.a  # the ApplyVertex GEMM operand
            if L.vform == "hc" and n > 0:
                # the layer below's dz IS the direct half of this layer's [dh | da] buffer:
                # the CSR pass then accumulates the gathered half onto it in place
                self.layers[n - 1].dz = L.dHA[:, : L.F]
        for n, L in enumerate(self.layers):
            if L.hin is None:
                L.hin = _mat(V, L.F, dev) if n == 0 else None
        for n, L in enumerate(self.layers[:-1]):
            nxt = self.layers[n + 1]
            if nxt.hin is None:
                nxt.hin = _mat(V, nxt.F, dev)
            L.hout = nxt.hin
        self.layers[-1].hout = None
        if self.bf16:
            self._alloc_bf16()
        self.X = self.layers[0].hin
        self.labels = torch.zeros(V, dtype=torch.int64, device=dev)
        self.loss = torch.zeros(1, dtype=torch.float32, device=dev)
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)
        self.nonfinite = torch.zeros(1, dtype=torch.int32, device=dev)
        self.tmp1 = _mat(V, max(L.F for L in self.layers), dev)
        self.tmp2 = _mat(V, max(L.F for L in self.layers), dev)

    def _alloc_bf16(self):
        """bf16 buffers of the bf16 storage mode: the layer-1 features, the hidden activations
        h_out = relu(z) (GEMM epilogue output, the next layer's gathered rows) and the gathered
        gradients dA (GEMM output); a, z, dz stay fp32.  The backward ReLU mask is h_out > 0
        (<=> z > 0), so the hidden z is not stored."""
        V, dev, bf = self.V, self.device, torch.bfloat16
        last = self.layers[-1]
        for n, L in enumerate(self.layers):
            if n == 0:
                L.hin = _mat(V, L.F, dev, dtype=bf)
            L.da = _mat(V, L.F, dev, dtype=bf) if n > 0 else None
            if L is not last:
                L.hout = _mat(V, L.O, dev, dtype=bf)
                L.z = None
                self.layers[n + 1].hin = L.hout

    def load_features(self, X):
        X = torch.as_tensor(X)
        if tuple(X.shape[:1]) != (self.V,) or X.shape[1] < self.layers[0].F:
            raise ShapeError(f"features must be [V={self.V}, {self.layers[0].F}]")
        dst = self._xbufs[self._cur] if getattr(self, "_graphs", None) else self.X
        dst.copy_(X[:, : self.layers[0].F], non_blocking=True)

    def load_labels(self, labels):
        self.labels.copy_(torch.as_tensor(np.asarray(labels, np.int64)), non_blocking=True)

    def prefetch_inputs(self, X_host, labels_host):
        """Stage the NEXT step's features and labels (pinned host tensors) on a copy stream.

        The H2D copy overlaps the current step's kernels.  With two captured graphs
        (``capture(double_buffer=True)``) the features land directly in the feature buffer
        the next graph reads (the one the running step does not), so nothing is moved on
        the device; otherwise the next step makes the compute stream wait for the copy and
        moves the staged inputs into place (a D2D copy).  A host tensor laid out like the
        device buffer (``[V, ld]``, 16-B padded rows) is copied as one contiguous block."""
        F = self.layers[0].F
        if getattr(self, "_copy_stream", None) is None:
            self._copy_stream = torch.cuda.Stream(device=self.device)
            self._stage_y = torch.empty_like(self.labels)
            self._stage_X = None if getattr(self, "_graphs", None) else torch.empty_like(self.X._base)[:, :F]
            self._staged = None
            self._consumed = None
        cs = self._copy_stream
        graphs = getattr(self, "_graphs", None)
        if graphs is not None:
            tgt = 1 - self._cur
            dst = self._xbufs[tgt]
            if self._done[tgt] is not None:
                cs.wait_event(self._done[tgt])  # the last step that read this buffer is done
        else:
            tgt, dst = None, self._stage_X
        if self._consumed is not None:
            # the previous staged labels (single _stage_y buffer, both modes) and features
            # (single-graph mode) have been moved into place
            cs.wait_event(self._consumed)
        with torch.cuda.stream(cs):
            if X_host.is_contiguous() and tuple(X_host.shape) == tuple(dst._base.shape):
                dst._base.copy_(X_host, non_blocking=True)
            else:
                dst.copy_(X_host[:, :F], non_blocking=True)
            self._stage_y.copy_(labels_host, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
        self._staged = ev
        self._staged_tgt = tgt

    def _take_staged(self):
        if getattr(self, "_staged", None) is None:
            return
        cur = torch.cuda.current_stream(self.device)
        cur.wait_event(self._staged)
        if self._staged_tgt is not None:
            self._cur = self._staged_tgt          # the next graph reads the buffer just filled
        else:
            self.X.copy_(self._stage_X)
        self.labels.copy_(self._stage_y)
        ev = torch.cuda.Event()
        ev.record(cur)
        self._consumed = ev
        self._staged = None

    # ------------------------------------------------------------------ passes
    def _rows(self, t, k):
        b = self.grid.begin(k)
        return t[b: b + self.grid.size(k)]

    def _fwd_propagate(self, L, stream=None, src=None, out=None, F=None):
        """Forward gather over the CSC chunks: src (default L.hin) -> out (default L.a)."""
        g, P = self.grid, self.grid.P
        src = L.hin if src is None else src
        out = L.a if out is None else out
        F = L.F if F is None else F
        for j in range(P):
            if not any((i, j) in g.csc for i in range(P)):
                self._rows(out, j).zero_()
                if L.kind == "ggcn":
                    self._rows(L.S, j).zero_()
        for (i, j), first, _ in self._chunk_order(list(g.csc), 1):
            pi = g.csc[(i, j)]
            if L.kind == "ggcn":
                # the forward also sums S = (h eta)(1 - eta) per destination, so the backward's
                # dQ = dA (.) S needs no second pass over the CSC (GGCN_FWD_S)
                K.propagate(pi, _lib.PROP_GGCN_FWD_S, self._rows(L.HP, i), self._rows(L.a, j), L.F,
                            g_off=L.goff, R=self._rows(L.Qv, j), out1=self._rows(L.S, j),
                            accumulate=not first, ws=self.ws, stream=stream)
            else:
                mode = _lib.PROP_GCN if L.kind == "gcn" else _lib.PROP_PASS
                K.propagate(pi, mode, self._rows(src, i), self._rows(out, j), F,
                            accumulate=not first, ws=self.ws, stream=stream)

    def _chunk_order(self, keys, out_axis):
        """Chunk visit order of the scheduler for a pass whose output
        interval is key[out_axis].  'locality': output-interval outer, so the accumulator
        A_j stays hot across its chunks; 'dest_order': input-interval outer.  Both visit the
        chunks of one output interval in ascending input interval, so results are bitwise
        identical.  Yields (key, first_for_output, last_for_output)."""
        P = self.grid.P
        inner = 1 - out_axis
        per_out = {o: sorted(k for k in keys if k[out_axis] == o) for o in range(P)}
        if self.schedule == "locality":
            order = [k for o in range(P) for k in per_out[o]]
        else:
            order = sorted(keys, key=lambda k: (k[inner], k[out_axis]))
        for k in order:
            chain = per_out[k[out_axis]]
            yield k, k == chain[0], k == chain[-1]

    def _bwd_propagate_gcn(self, L, out, mask, stream=None, onto=False, src=None, F=None):
        """dH[v] = sum_{out(v)} w_e dA[u] over CSR chunks, j ascending; ReLU mask on the last.
        ``onto``: continue from the value already in ``out`` (CommNet's direct W_H term).
        ``src`` (default L.da) / ``F`` (default L.F): the gathered gradient and its width."""
        g, P = self.grid, self.grid.P
        src = L.da if src is None else src
        F = L.F if F is None else F
        mode = _lib.PROP_GCN if L.kind == "gcn" else _lib.PROP_PASS
        for i in range(P):
            if not any((i, j) in g.csr for j in range(P)):
                if onto:
                    o = self._rows(out, i)
                    K.ewise(8, o, self._rows(mask, i), o, stream)
                else:
                    self._rows(out, i).zero_()
        for (i, j), first, last in self._chunk_order(list(g.csr), 0):
            K.propagate(g.csr[(i, j)], mode, self._rows(src, j), self._rows(out, i), F,
                        mask=self._rows(mask, i) if (last and mask is not None) else None,
                        accumulate=onto or not first, ws=self.ws, stream=stream)

    def _bwd_propagate_ggcn(self, L, stream=None):
        g, P = self.grid, self.grid.P
        # dQ[u] = sum_in(u) ((dA[u] h[v]) eta)(1 - eta) = dA[u] (.) S[u] with S from the forward
        K.ewise(2, L.dAv, L.S, L.dQ, stream)
        for i in range(P):  # pass B over CSR: dP[v], dH_take[v]
            chain = [j for j in range(P) if (i, j) in g.csr]
            if not chain:
                self._rows(L.dP, i).zero_()
                self._rows(L.dHt, i).zero_()
            for k, j in enumerate(chain):
                K.propagate(g.csr[(i, j)], _lib.PROP_GGCN_BWD_SRC, self._rows(L.GQ, j),
                            self._rows(L.dP, i), L.F, g_off=L.goff, R=self._rows(L.HP, i),
                            r_off=L.goff, out1=self._rows(L.dHt, i), accumulate=k > 0, ws=self.ws,
                            stream=stream)

    def _fwd_max(self, L, Y, stream=None):
        """Gather(max) over the CSC chunks of each destination interval, source intervals
        ascending, carrying the running max/argmax (global positions = chunk base + CSC
        position, so the result is segment_max over the flattened edge list)."""
        g, P = self.grid, self.grid.P
        for j in range(P):
            if not any((i, j) in g.csc for i in range(P)):
                self._rows(L.a, j).zero_()
                self._rows(L.arg, j).fill_(-1)
        for (i, j), first, last in self._chunk_order(list(g.csc), 1):
            K.max_gather(g.csc[(i, j)], self._rows(Y, i), self._rows(L.a, j), self._rows(L.arg, j),
                         L.Aw, pos_base=g.edge_base[(i, j)], accumulate=not first, finalize=last,
                         stream=stream, ws=self.ws)

    def _bwd_max(self, L, out, mask, stream=None):
        """dY[v] = sum over out-edges (destination intervals ascending, CSR order) of dA[dst]
        routed to the argmax edge; ReLU mask of the layer below fused on the last chunk."""
        g, P = self.grid, self.grid.P
        for i in range(P):
            if not any((i, j) in g.csr for j in range(P)):
                self._rows(out, i).zero_()
        for (i, j), first, last in self._chunk_order(list(g.csr), 0):
            K.max_gather_bwd(g.csr[(i, j)], g.csr_positions(i, j), self._rows(L.da, j),
                             self._rows(L.arg, j), self._rows(out, i), L.Aw,
                             mask=self._rows(mask, i) if (last and mask is not None) else None,
                             pos_base=g.edge_base[(i, j)], accumulate=not first, stream=stream,
                             ws=self.ws)

    def _gemm(self, A, B, C, **kw):
        # strict mode (tensor.py:161-163) fused into every GEMM epilogue: z, the hoisted P / Q,
        # dA and dW of every layer raise the device flag if non-finite (a non-finite aggregate
        # or gathered gradient row reaches a GEMM output, so the gathers are covered too)
        K.gemm(A, B, C, prec=self.gemm_prec, ws=self.ws,
               nonfinite=self.nonfinite if self.strict else None, **kw)

    def _ewise(self, op, a, b, out, stream=None):
        _lib.check(_lib.lib.sg_ewise(op, a.shape[0], a.shape[1], a.data_ptr(), a.stride(0),
                                     b.data_ptr(), b.shape[0], b.shape[1], b.stride(0),
                                     out.data_ptr(), out.stride(0), _lib.stream_handle(stream)))

    # ------------------------------------------------------------------ step
    _NVTX = os.environ.get("SG_NVTX", "0") == "1"

    def _mark(self, name):
        """Stage boundary event (enabled by setting ``self.prof = []``); with SG_NVTX=1 also
        an NVTX marker per SAGA stage for timeline tools (SURVEY.md §5 tracing)."""
        if self._NVTX:
            torch.cuda.nvtx.mark(f"sg:{name}")
        if self.prof is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self.prof.append((name, e))

    def forward(self, stream=None):
        """All layers forward; returns z_L (pre-ReLU logits)."""
        self._mark("start")
        if self.strict:
            self.nonfinite.zero_()
        if self.bf16:
            return self._forward_bf16(stream)
        for n, L in enumerate(self.layers):
            if L.kind == "ggcn":
                self._gemm(L.hin, L.WH, L.Pv)   # hoisted P = h W_H
                self._gemm(L.hin, L.WC, L.Qv)   # hoisted Q = h W_C
                self._mark(f"L{n}.fwd.hoist_gemm")
            if L.reorder:  # Y = h W, then z = A Y (reorder_linear_gather)
                self._gemm(L.hin, L.W, L.Y)
                self._mark(f"L{n}.fwd.apply_vertex")
                self._fwd_propagate(L, stream, src=L.Y, out=L.z, F=L.O)
                if L.hout is not None:
                    K.ewise(7, L.z, None, L.hout, stream)   # h' = relu(z)
                self._mark(f"L{n}.fwd.propagate")
                continue
            if L.kind in ("max", "max_pool"):
                Y = L.hin
                if L.kind == "max_pool":       # hoisted edge network Y = sigmoid(h W_pool + b)
                    self._gemm(L.hin, L.Wp, L.Y)
                    K.ewise(0, L.Y, L.bias, L.Y, stream)
                    K.ewise(5, L.Y, None, L.Y, stream)
                    Y = L.Y
                    self._mark(f"L{n}.fwd.hoist_gemm")
                self._fwd_max(L, Y, stream)
            else:
                self._fwd_propagate(L, stream)
            self._mark(f"L{n}.fwd.propagate")
            self._gemm(L.gin, L.W, L.z, relu_out=L.hout)  # ApplyVertex: z = a W, h' = relu(z)
            self._mark(f"L{n}.fwd.apply_vertex")
        return self.layers[-1].z

    def _forward_bf16(self, stream=None):
        last = self.layers[-1]
        for n, L in enumerate(self.layers):
            self._fwd_propagate(L, stream)              # bf16 rows in, fp32 sums and a out
            self._mark(f"L{n}.fwd.propagate")
            # z = a W (3xTF32); hidden layers keep only h' = relu(z) in bf16, the top layer z fp32
            self._gemm(L.a, L.W, L.z, relu_out=None if L is last else L.hout)
            self._mark(f"L{n}.fwd.apply_vertex")
        return last.z

    def _backward_bf16(self, stream=None):
        for n in range(len(self.layers) - 1, -1, -1):
            L = self.layers[n]
            self._gemm(L.a, L.dz, L.dW, trans_a=True)        # dW = a^T dz (fp32)
            if n > 0:
                below = self.layers[n - 1]
                self._gemm(L.dz, L.W, L.da, trans_b=True)    # dA = dz W^T, stored bf16
                self._mark(f"L{n}.bwd.apply_vertex")
                # CSR dual: bf16 dA rows in, fp32 dz out, ReLU mask h_out (bf16) of the layer below
                self._bwd_propagate_gcn(L, below.dz, below.hout, stream)
                self._mark(f"L{n}.bwd.propagate")
            else:
                self._mark(f"L{n}.bwd.apply_vertex")

    def backward(self, stream=None):
        """Loss + all parameter gradients (reverse stage order)."""
        last = self.layers[-1]
        K.softmax_xent(last.z, self.labels, self.loss, last.dz, self.err, relu_input=True,
                       ws=self.ws, stream=stream)
        self._mark("loss")
        if self.bf16:
            self._backward_bf16(stream)
            if self.strict:
                K.check_finite(self.loss, self.nonfinite, stream)
            return self.loss
        for n in range(len(self.layers) - 1, -1, -1):
            L = self.layers[n]
            below = self.layers[n - 1] if n > 0 else None
            if L.reorder:
                # dY = A^T dz (CSR pass), dW = h^T dY, dh = dY W^T (+ ReLU mask of the layer below)
                self._bwd_propagate_gcn(L, L.dY, None, stream, src=L.dz, F=L.O)
                self._mark(f"L{n}.bwd.propagate")
                self._gemm(L.hin, L.dY, L.dW, trans_a=True)
                if below is not None:
                    self._gemm(L.dY, L.W, below.dz, trans_b=True)
                    K.ewise(8, below.dz, below.z, below.dz, stream)
                self._mark(f"L{n}.bwd.apply_vertex")
                continue
            self._gemm(L.gin, L.dz, L.dW, trans_a=True)         # dW = a^T dz
            if L.kind in ("max", "max_pool"):
                self._gemm(L.dz, L.W, L.da, trans_b=True)       # dA = dz W^T
                self._mark(f"L{n}.bwd.apply_vertex")
                if L.kind == "max":
                    if below is not None:  # max routing + ReLU mask of the layer below, one pass
                        self._bwd_max(L, below.dz, below.z, stream)
                    self._mark(f"L{n}.bwd.propagate")
                    continue
                self._bwd_max(L, L.dY, None, stream)
                self._mark(f"L{n}.bwd.propagate")
                K.ewise(9, L.dY, L.Y, L.dY, stream)                  # sigmoid bwd (tensor.py:232)
                self._gemm(self._ones, L.dY, L.dbias, trans_a=True)  # db = column sums
                self._gemm(L.hin, L.dY, L.dWp, trans_a=True)         # dW_pool = h^T dpre
                if below is not None:
                    t1 = self.tmp1[:, : L.F]
                    self._gemm(L.dY, L.Wp, t1, trans_b=True)
                    K.ewise(8, t1, below.z, below.dz, stream)
                self._mark(f"L{n}.bwd.hoist_gemm")
                continue
            if L.kind == "ggcn":
                self._gemm(L.dz, L.W, L.dAv, trans_b=True)      # dA = dz W^T
                self._mark(f"L{n}.bwd.apply_vertex")
                self._bwd_propagate_ggcn(L, stream)
                self._mark(f"L{n}.bwd.propagate")
                self._gemm(L.hin, L.dQ, L.dWC, trans_a=True)    # dW_C = h^T dQ
                self._gemm(L.hin, L.dP, L.dWH, trans_a=True)    # dW_H = h^T dP
                if below is not None:
                    t1, t2 = self.tmp1[:, : L.F], self.tmp2[:, : L.F]
                    self._gemm(L.dQ, L.WC, t1, trans_b=True)
                    self._ewise(0, L.dHt, t1, t1, stream)       # take_rows part + Q part
                    self._gemm(L.dP, L.WH, t2, trans_b=True)
                    self._ewise(0, t1, t2, t1, stream)          # + P part (tape order)
                    self._ewise(8, t1, below.z, below.dz, stream)  # relu bwd of the layer below
                self._mark(f"L{n}.bwd.hoist_gemm")
            elif L.vform == "hc":
                if below is not None:  # [dh_direct | da] = dz [W_H; W_C]^T, then += gathered da
                    self._gemm(L.dz, L.W, L.dHA, trans_b=True)
                    self._mark(f"L{n}.bwd.apply_vertex")
                    self._bwd_propagate_gcn(L, below.dz, below.z, stream, onto=True)
                    self._mark(f"L{n}.bwd.propagate")
                else:
                    self._mark(f"L{n}.bwd.apply_vertex")
            else:
                if below is not None:
                    self._gemm(L.dz, L.W, L.da, trans_b=True)   # dA = dz W^T
                    self._mark(f"L{n}.bwd.apply_vertex")
                    self._bwd_propagate_gcn(L, below.dz, below.z, stream)
                    self._mark(f"L{n}.bwd.propagate")
                else:
                    self._mark(f"L{n}.bwd.apply_vertex")
        if self.strict:
            # every GEMM output (z, P, Q, dA, dW) was checked in its epilogue; the loss here
            K.check_finite(self.loss, self.nonfinite, stream)
        return self.loss

    def sgd(self, lr, stream=None):
        for L in self.layers:
            for W, dW in L.sgd_pairs:  # whole padded buffers (padding stays zero)
                K.sgd(W, dW, lr, stream)
        self._mark("sgd")

    def stage_times(self):
        """{stage: ms} from the recorded marks (call after synchronize)."""
        out = {}
        for (_, a), (name, b) in zip(self.prof, self.prof[1:]):
            if name != "start":
                out[name] = out.get(name, 0.0) + a.elapsed_time(b)
        return out

    def train_step(self, lr=0.01):
        if self._NVTX:
            torch.cuda.nvtx.range_push("sg:train_step")
        self._take_staged()
        self.forward()
        self.backward()
        self.sgd(lr)
        if self._NVTX:
            torch.cuda.nvtx.range_pop()
        return self.loss

    # ------------------------------------------------------------------ checkpoint
    def save_checkpoint(self, path, epoch=0):
        """Parameters + epoch (+ the graph's content key, so a resume on another graph is
        refused) as one .npz (SURVEY.md §5 checkpoint/resume)."""
        from . import graph as G

        g = self.grid.graph
        arrs = {f"p{k}": w for k, w in enumerate(self.weights())}
        np.savez(path, epoch=np.int64(epoch), graph_key=np.array(G.graph_key(g, self.grid.part.interval_size)),
                 n_params=np.int64(len(arrs)), **arrs)

    def load_checkpoint(self, path):
        """Restore parameters saved by save_checkpoint; returns the saved epoch."""
        from . import graph as G

        with np.load(path) as z:
            key = str(z["graph_key"])
            if key != G.graph_key(self.grid.graph, self.grid.part.interval_size):
                raise ConfigError(f"checkpoint {path} was written for another graph ({key})")
            n = int(z["n_params"])
            self.set_weights([z[f"p{k}"] for k in range(n)])
            return int(z["epoch"])

    # ------------------------------------------------------------------ CUDA graph
    def capture(self, lr=0.01, warmup=1, double_buffer=True):
        """Record one full training step (forward, backward, SGD) as a CUDA graph.

        ``double_buffer``: also record a second graph whose layer-1 input is a second
        feature buffer, so ``prefetch_inputs`` can copy the next step's features straight
        into the buffer the running step does not read (no device-side move); replays
        alternate between the two (GCN / passthrough first layers)."""
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            snapshot = [t.clone() for L in self.layers for t in L.params]
            for _ in range(warmup):  # sizes the workspace before capture
                self.train_step(lr)
            k = 0
            for L in self.layers:
                for t in L.params:
                    t.copy_(snapshot[k])
                    k += 1
        torch.cuda.current_stream().wait_stream(s)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.train_step(lr)
        self._graphs = None
        L0 = self.layers[0]
        if double_buffer and L0.kind in ("gcn", "pass") and L0.hin is self.X:
            X2 = torch.zeros_like(self.X._base)[:, : L0.F]
            X2.copy_(self.X)
            L0.hin = X2
            try:
                g2 = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g2):
                    self.train_step(lr)
            finally:
                L0.hin = self.X
            self._graphs = [self.graph, g2]
            self._xbufs = [self.X, X2]
            self._done = [None, None]
            self._cur = 0
            self._copy_stream = None  # re-created for the double-buffered layout
        return self.graph

    def replay(self):
        self._take_staged()
        if getattr(self, "_graphs", None) is None:
            self.graph.replay()
            return self.loss
        self._graphs[self._cur].replay()
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))
        self._done[self._cur] = ev
        return self.loss

    def check_status(self):
        """Read the device flags (syncs): raise like the reference's strict mode."""
        if int(self.err.item()):
            raise ShapeError("label out of range [0, classes)")
        if self.strict and int(self.nonfinite.item()):
            raise NumericError("non-finite value produced in the training step")


def gcn_model(grid, dims, **kw):
    """2-layer (or L-layer) GCN: dims = [F, H, ..., C]."""
    return SAGAModel([prog.build_gcn(a, b) for a, b in zip(dims, dims[1:])], grid, **kw)


def ggcn_model(grid, dims, **kw):
    return SAGAModel([prog.build_ggcn(a, b) for a, b in zip(dims, dims[1:])], grid, **kw)


def commnet_model(grid, dims, **kw):
    """CommNet: params per layer [W_H, W_C]."""
    return SAGAModel([prog.build_commnet(a, b) for a, b in zip(dims, dims[1:])], grid, **kw)


def mpgcn_model(grid, dims, pool=None, **kw):
    """MP-GCN: per layer W_pool [F, pool], b [pool], W [pool, O].
    ``pool`` defaults to each layer's input width."""
    pool = list(pool) if pool is not None else list(dims[:-1])
    if len(pool) != len(dims) - 1:
        raise ShapeError("need one pool width per layer")
    return SAGAModel([prog.build_mpgcn(a, p, b) for a, p, b in zip(dims, pool, dims[1:])], grid, **kw)


def run_train(config):
    """SPEC.md:595-603 run_train on a synthetic graph; returns a metrics dict.

    config keys (SPEC.md:622 subset + synthetic graph): model ('gcn'|'ggcn'|'mpgcn'|'commnet'|'ggnn'),
    graph ('rmat'|'uniform'), V, E, features F, hidden, classes, layers, epochs,
    lr, seed, interval_size."""
    from . import graph as G

    known = {"model", "graph", "V", "E", "features", "hidden", "classes", "layers", "epochs", "lr",
             "seed", "interval_size", "split_edges", "edge_types", "checkpoint"}
    bad = set(config) - known
    if bad:
        raise ConfigError(f"unknown config keys {sorted(bad)}")
    model = config.get("model", "gcn")
    builders = {"gcn": gcn_model, "ggcn": ggcn_model, "mpgcn": mpgcn_model,
                "commnet": commnet_model, "ggnn": None}
    if model not in builders:
        raise ConfigError(f"unknown model '{model}'; valid: {', '.join(builders)}")
    V, E = int(config["V"]), int(config["E"])
    gen = G.rmat_graph if config.get("graph", "uniform") == "rmat" else G.uniform_graph
    g = gen(V, E, seed=int(config.get("seed", 0)))
    F, H, C = int(config["features"]), int(config.get("hidden", 16)), int(config["classes"])
    nl = int(config.get("layers", 2))
    dims = [F] + [H] * (nl - 1) + [C]
    interval = config.get("interval_size")
    if not interval:
        # the chunk scheduler's choice for a resident model on this device (schedule.py)
        from . import schedule as S

        free = torch.cuda.mem_get_info()[0] if torch.cuda.is_available() else None
        interval = S.build_schedule(g, dims, budget=free,
                                    model="ggcn" if model == "ggcn" else "gcn").interval_size
    grid = G.ChunkGrid(g, interval, split_edges=int(config.get("split_edges", G.DEFAULT_SPLIT_EDGES)))
    if model == "ggnn":  # GG-NN: state width F, synthetic edge labels, readout to C classes
        from .ggnn import ggnn_model

        nt = int(config.get("edge_types", 3))
        types = np.random.default_rng(5).integers(0, nt, E)
        grid = G.ChunkGrid(g, interval, gcn_weights=False,
                           split_edges=int(config.get("split_edges", G.DEFAULT_SPLIT_EDGES)))
        m = ggnn_model(grid, F, nt, C, types, layers=nl)
    else:
        m = builders[model](grid, dims)
    m.load_features(torch.from_numpy(G.synthetic_features(V, F, seed=1)))
    m.load_labels(np.random.default_rng(3).integers(0, C, V))
    ckpt = config.get("checkpoint")
    start = 0
    if ckpt and os.path.exists(ckpt) and hasattr(m, "load_checkpoint"):
        start = m.load_checkpoint(ckpt)   # resume: parameters and epoch counter
    losses = []
    for _ in range(start, int(config.get("epochs", 10))):
        m.train_step(float(config.get("lr", 0.01)))
        m.check_status()
        losses.append(float(m.loss.item()))
    if ckpt and hasattr(m, "save_checkpoint"):
        m.save_checkpoint(ckpt, start + len(losses))
    return {"model": model, "V": V, "E": E, "epochs": len(losses), "start_epoch": start,
            "loss": losses}


def run_bench(config):
    """SPEC.md:604-612 run_bench: every scheduling strategy on the same partitioned graph.

    One row per strategy of schedule.STRATEGIES ('locality', 'dest_order', 'stage_based'):
    the scheduler's swap bytes and modelled makespan (schedule.build_schedule under the
    config's ``budget_bytes``), and -- for the strategies the device executor runs (the resident
    chunk orders 'locality' / 'dest_order'; 'stage_based', which materialises every stage's
    edge tensors, is modelled only) -- the measured epoch time and the loss after ``epochs``
    training epochs from the same seed (scheduling never changes values: SPEC.md:371).  The
    ring / non-ring multi-device simulations of the reference's report are out of scope
    (DESIGN.md §7).  Config keys: those of run_train plus ``budget_bytes``."""
    import time

    from . import graph as G
    from . import schedule as S

    cfg = dict(config)
    budget = cfg.pop("budget_bytes", None)
    known = {"model", "graph", "V", "E", "features", "hidden", "classes", "layers", "epochs", "lr",
             "seed", "interval_size", "split_edges"}
    bad = set(cfg) - known
    if bad:
        raise ConfigError(f"unknown config keys {sorted(bad)}")
    model = cfg.get("model", "gcn")
    if model not in ("gcn", "ggcn"):
        raise ConfigError(f"run_bench model must be gcn or ggcn (got '{model}')")
    V, E = int(cfg["V"]), int(cfg["E"])
    gen = G.rmat_graph if cfg.get("graph", "uniform") == "rmat" else G.uniform_graph
    g = gen(V, E, seed=int(cfg.get("seed", 0)))
    F, H, C = int(cfg["features"]), int(cfg.get("hidden", 16)), int(cfg["classes"])
    nl = int(cfg.get("layers", 2))
    dims = [F] + [H] * (nl - 1) + [C]
    epochs, lr = int(cfg.get("epochs", 1)), float(cfg.get("lr", 0.01))
    X = torch.from_numpy(G.synthetic_features(V, F, seed=1))
    labels = np.random.default_rng(3).integers(0, C, V)
    rows = []
    for strategy in S.STRATEGIES:
        sch = S.build_schedule(g, dims, budget=budget, model=model, strategy=strategy)
        row = {"strategy": strategy, "mode": sch.mode, "P": sch.P,
               "swap_h2d_bytes": int(sch.swap_h2d_bytes), "swap_d2h_bytes": int(sch.swap_d2h_bytes),
               "makespan_ms_model": round(sch.makespan_ms, 4), "measured_ms": None, "loss": None}
        if sch.mode == "resident" and strategy in ("locality", "dest_order"):
            interval = cfg.get("interval_size") or sch.interval_size
            grid = G.ChunkGrid(g, interval, gcn_weights=model == "gcn",
                               split_edges=cfg.get("split_edges", G.DEFAULT_SPLIT_EDGES))
            build = gcn_model if model == "gcn" else ggcn_model
            m = build(grid, dims, schedule=strategy)
            m.load_features(X)
            m.load_labels(labels)
            losses = []
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(epochs):
                m.train_step(lr)
                losses.append(float(m.loss.item()))
            torch.cuda.synchronize()
            m.check_status()
            row["P"] = grid.P
            row["measured_ms"] = round((time.perf_counter() - t0) * 1e3 / max(epochs, 1), 4)
            row["loss"] = losses
        rows.append(row)
    return {"model": model, "V": V, "E": E, "dims": dims, "budget_bytes": budget, "rows": rows}
