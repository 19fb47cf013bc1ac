"""Chunk-level stage ops and the unfused SAGA-NN executor.

The fused executor (``engine.SAGAModel``) lowers the programs ``fuse_sag`` recognises onto one
sm_100a propagation kernel per chunk.  Everything else -- an ApplyEdge that is not one of the
fused shapes, or a program run without the hoist -- runs here, stage by stage, exactly as the
SPEC's propagation-kernels module describes:

=========================  =====================================================  ================================
SPEC op                    here                                                   kernels
=========================  =====================================================  ================================
scatter_chunk   :392-399   ``scatter_chunk``: edge.src / edge.dest rows in CSC     sg_take_rows
                           edge order (+ hoisted per-vertex tables, edge.data)
apply_edge_chunk :400-406  ``apply_edge_chunk``: the traced ApplyEdge graph        sg_ewise, sg_gemm (tcgen05)
                           evaluated on the chunk's edge tensors
gather_chunk    :407-416   ``gather_chunk``: A_j <- A_j (+)= rows in CSC order     sg_propagate(PASS, accumulate) /
                           (sum), running max + argmax (max)                      sg_max_gather (chained)
fused_gather_chunk :417-423 ``engine.SAGAModel`` (fused executor)                  sg_propagate modes
backward_gather :427-436   ``backward_gather``: sum -> dA[dest(e)], max -> routed  sg_take_rows / sg_max_gather_bwd
                           to the argmax edge
backward_apply_edge        torch autograd through ``ops`` (tensor.py closures)     sg_ewise_bwd, sg_reduce_sum, sg_gemm
backward_scatter           ``ops.take_rows`` backward: np.add.at in edge order     sg_segment_sort + sg_propagate(PASS)
=========================  =====================================================  ================================

torch autograd stands in for the reference's Tape (tensor.py:69-130); every forward and
backward computation is one of this repo's kernels.  Like the reference Tape, the edge
tensors of every chunk are kept for the backward (O(E x width) device memory per layer), so
this executor is the general path, not the fast one: ``fuse_sag``-able programs belong on the
fused executor ("fused == unfused bitwise for GCN" is what the tests check).
"""

import numpy as np
import torch

from . import _lib
from . import kernels as K
from . import ops
from . import program as prog
from .errors import ConfigError, NumericError, ProgramError, ShapeError
from .graph import PassIndex


class EdgeChunkDev:
    """Device view of one EdgeChunk C_ij for the unfused stage ops: per CSC edge its local
    source row and local destination row (int64, take_rows indices), its edge data, and the
    identity pass indexes the gathers run on (edge e of the chunk is row e of the edge tensor)."""

    def __init__(self, grid, i, j, edge_data=None):
        ch = grid.part.chunk(i, j)
        dev = grid.device
        self.i, self.j, self.nnz = i, j, int(ch["nnz"])
        self.n_src, self.n_dst = grid.size(i), grid.size(j)
        ptr = np.ascontiguousarray(ch["csc_ptr"], np.int64)
        dst = np.repeat(np.arange(self.n_dst, dtype=np.int64), np.diff(ptr))
        self.src = torch.from_numpy(ch["csc_idx"].astype(np.int64)).to(dev)
        self.dst = torch.from_numpy(dst).to(dev)
        self.eid = ch["csc_eid"]
        if edge_data is not None:
            self.data = edge_data[torch.from_numpy(self.eid).to(edge_data.device)].contiguous()
        elif (i, j) in grid.csc and grid.csc[(i, j)].w is not None:
            self.data = grid.csc[(i, j)].w.reshape(-1, 1)     # GCN weight, CSC order
        else:
            self.data = None
        T = grid.split_edges
        # Gather: rows of the [nnz, F] edge tensor in CSC order, grouped by local destination
        self.gather_pi = PassIndex(ptr, np.arange(self.nnz, dtype=np.int32), None, self.n_dst, T, dev)
        # backward of the max gather: edge-row e has one "out-edge", to dest(e), at position e
        self._bwd_pi = None
        self._T = T

    def max_bwd_index(self):
        if self._bwd_pi is None:
            dev = self.src.device
            self._bwd_pi = PassIndex(np.arange(self.nnz + 1, dtype=np.int64), self.dst.cpu().numpy().astype(np.int32),
                                     None, self.nnz, self._T, dev)
            self._pos = torch.arange(self.nnz, dtype=torch.int32, device=dev)
        return self._bwd_pi, self._pos


# ------------------------------------------------------------------ forward stage ops
def scatter_chunk(vc_src, vc_dest, ec, need=("src", "dest"), tables=None):
    """per-edge rows in CSC edge order.  ``vc_src`` / ``vc_dest`` are the
    source / destination VertexChunks (row slices of the vertex features); ``tables`` maps
    hoisted per-vertex table names to (side, (src-interval slice, dest-interval slice)).
    Returns the ApplyEdge bindings {'edge.src', 'edge.dest', 'edge.data', 'pre_*'}."""
    out = {}
    if "src" in need:
        out["edge.src"] = ops.take_rows(vc_src, ec.src)
    if "dest" in need:
        out["edge.dest"] = ops.take_rows(vc_dest, ec.dst)
    if ec.data is not None:
        out["edge.data"] = ec.data
    for name, (side, (t_src, t_dst)) in (tables or {}).items():
        out[name] = ops.take_rows(t_src, ec.src) if side == "src" else ops.take_rows(t_dst, ec.dst)
    return out


def apply_edge_chunk(expr, edge_tensors, params):
    """row e = expr evaluated on edge e (the traced ApplyEdge graph on the
    chunk's edge tensors; matmul rows run on the tcgen05 GEMM)."""
    b = dict(params)
    b.update(edge_tensors)
    return evaluate(expr, b)


def gather_chunk(acc, ec, accumulator, A_j, *, first, last=True, argmax=None, pos_base=0,
                 empty_fill=0.0):
    """SPEC.md:407-416 (in place on A_j): sum -> A_j[u] (+)= acc rows of u's in-edges in CSC
    order (``first`` starts from the identity; rows with more than T edges combine their
    subgroups in order); max -> running max with the lowest position winning
    ties, ``argmax`` = pos_base + edge row (int32), rows still empty at ``last`` filled with
    ``empty_fill``."""
    acc = acc.contiguous()
    F = acc.shape[1]
    if accumulator == "sum":
        K.propagate(ec.gather_pi, _lib.PROP_PASS, acc, A_j, F, accumulate=not first)
    elif accumulator == "max":
        K.max_gather(ec.gather_pi, acc, A_j, argmax, F, empty_fill, pos_base=pos_base,
                     accumulate=not first, finalize=last)
    else:
        raise ProgramError(f"accumulator '{accumulator}' has no gather (concat is out of scope)")
    return A_j


# ------------------------------------------------------------------ backward stage ops
def backward_gather(dA_j, ec, accumulator, argmax=None, pos_base=0):
    """sum -> d acc_e = dA_j[dest(e)]; max -> dA_j routed to the edge that won
    each column (argmax), zero elsewhere."""
    if accumulator == "sum":
        return _take(dA_j, ec.dst)
    pi, pos = ec.max_bwd_index()
    F = dA_j.shape[1]
    out = torch.empty((ec.nnz, F), dtype=dA_j.dtype, device=dA_j.device)
    K.max_gather_bwd(pi, pos, dA_j.contiguous(), argmax, out, F, pos_base=pos_base)
    return out


def _take(a, idx):
    a = a.contiguous()
    out = torch.empty((idx.numel(), a.shape[1]), dtype=a.dtype, device=a.device)
    err = torch.zeros(1, dtype=torch.int32, device=a.device)
    _lib.check(_lib.lib.sg_take_rows(K.dtype_code(a), a.data_ptr(), a.stride(0), a.shape[0],
                                     idx.data_ptr(), idx.numel(), out.data_ptr(), out.stride(0),
                                     a.shape[1], err.data_ptr(), _lib.stream_handle()))
    return out


class _GatherColumn(torch.autograd.Function):
    """gather_chunk over every chunk C_ij of destination column j in source-interval order
    (Locality) into a fresh A_j; backward = backward_gather per chunk."""

    @staticmethod
    def forward(ctx, accumulator, chunks, n_rows, F, empty_fill, *accs):
        dev = accs[0].device if accs else torch.device("cuda")
        A = torch.empty((n_rows, F), dtype=torch.float32, device=dev)
        arg = None
        if not chunks:
            A.fill_(0.0 if accumulator == "sum" else empty_fill)
        elif accumulator == "sum":
            for k, (ec, acc) in enumerate(zip(chunks, accs)):
                gather_chunk(acc, ec, "sum", A, first=k == 0)
        else:
            arg = torch.empty((n_rows, F), dtype=torch.int32, device=dev)
            base = 0
            for k, (ec, acc) in enumerate(zip(chunks, accs)):
                gather_chunk(acc, ec, "max", A, first=k == 0, last=k == len(chunks) - 1,
                             argmax=arg, pos_base=base, empty_fill=empty_fill)
                base += ec.nnz
        ctx.accumulator, ctx.chunks, ctx.arg = accumulator, chunks, arg
        if arg is not None:
            ctx.mark_non_differentiable(arg)
        return A

    @staticmethod
    def backward(ctx, g):
        g = g.contiguous()
        outs, base = [], 0
        for ec in ctx.chunks:
            outs.append(backward_gather(g, ec, ctx.accumulator, ctx.arg, base))
            base += ec.nnz
        return (None, None, None, None, None) + tuple(outs)


# ------------------------------------------------------------------ expression evaluation
def evaluate(e, bindings):
    """program.evaluate_expr plus the GRU ApplyVertex spelled out in
    primitive ops.  Typed GG-NN edges have their own executor (ggnn.GGNNModel)."""
    memo = {}

    def ev(x):
        if id(x) in memo:
            return memo[id(x)]
        if x.op in ("input", "param", "pre"):
            if x.name not in bindings:
                raise ProgramError(f"missing binding for '{x.name}'")
            v = bindings[x.name]
        elif x.op == "matmul":
            v = ops.matmul(ev(x.args[0]), ev(x.args[1]))
        elif x.op in ("sigmoid", "tanh", "relu"):
            v = getattr(ops, x.op)(ev(x.args[0]))
        elif x.op in prog.ELEMENTWISE:
            v = ops.elementwise(x.op, ev(x.args[0]), ev(x.args[1]))
        elif x.op == "gru":
            h, a = ev(x.args[0]), ev(x.args[1])
            Wz, Uz, Wr, Ur, Wh, Uh = (ev(w) for w in x.args[2:])
            z = ops.sigmoid(ops.add(ops.matmul(a, Wz), ops.matmul(h, Uz)))
            r = ops.sigmoid(ops.add(ops.matmul(a, Wr), ops.matmul(h, Ur)))
            c = ops.tanh(ops.add(ops.matmul(a, Wh), ops.matmul(ops.mul(r, h), Uh)))
            one = torch.ones((z.shape[1],), dtype=z.dtype, device=z.device)   # a_lead broadcast
            v = ops.add(ops.mul(ops.sub(one, z), h), ops.mul(z, c))
        else:
            raise ProgramError(f"op '{x.op}' has no unfused lowering (typed edges: ggnn.GGNNModel)")
        memo[id(x)] = v
        return v

    return ev(e)


# ------------------------------------------------------------------ the unfused executor
class UnfusedSAGAModel:
    """Multi-layer SAGA-NN model run stage by stage on a ChunkGrid (SPEC.md:297-305,
    392-436): per layer the hoisted per-vertex tables (``hoist=True``), then
    for each destination interval j and each source interval i in ascending order
    scatter_chunk -> apply_edge_chunk -> gather_chunk into A_j, then ApplyVertex over all
    vertices; softmax cross-entropy on the last layer's output (tensor.py:487-506); the
    backward is the reverse sweep (torch autograd over the libsagann ops).

    Runs any program ``validate_program`` accepts whose ops have a lowering (element-wise,
    matmul, GRU; sum or max accumulator).  Parameters are initialised exactly like
    ``engine.SAGAModel`` (Glorot-uniform from default_rng(seed), zero biases, program order), so
    the two executors can be compared on the same weights."""

    def __init__(self, programs, grid, weights=None, *, seed=2, hoist=True, edge_data=None,
                 empty_fill=0.0):
        if not torch.cuda.is_available():
            raise RuntimeError("UnfusedSAGAModel needs a CUDA device (no CPU fallback)")
        self.grid, self.V = grid, grid.V
        self.device = torch.device(grid.device)
        self.empty_fill = float(empty_fill)
        self.layers = []
        for p in programs:
            q = prog.hoist_vertex_computation(p)[0] if hoist else p
            diags = prog.validate_program(q)
            if diags:
                raise ProgramError("; ".join(diags))
            if q.accumulator not in ("sum", "max"):
                raise ProgramError(f"accumulator '{q.accumulator}' is not executable")
            for x in prog.nodes(q.apply_edge) + prog.nodes(q.apply_vertex):
                if x.op in ("typed_matmul", "select_type"):
                    raise ProgramError("typed ApplyEdge: use ggnn.GGNNModel")
            self.layers.append(q)
        for a, b in zip(self.layers, self.layers[1:]):
            if a.f_out != b.f_in:
                raise ShapeError(f"layer widths do not chain: {a.f_out} -> {b.f_in}")
        if edge_data is not None:
            edge_data = torch.as_tensor(edge_data, dtype=torch.float32, device=self.device)
            if edge_data.dim() == 1:
                edge_data = edge_data.reshape(-1, 1)
            if edge_data.shape[0] != grid.E:
                raise ShapeError(f"edge_data has {edge_data.shape[0]} rows, the graph {grid.E} edges")
        self.chunks = {j: [EdgeChunkDev(grid, i, j, edge_data) for i in range(grid.P)
                           if grid.part.chunk(i, j)["nnz"] > 0] for j in range(grid.P)}
        self.params = [{n: torch.zeros(tuple(s) if len(s) >= 2 else (s[0],), dtype=torch.float32,
                                       device=self.device, requires_grad=True)
                        for n, s in q.params.items()} for q in self.layers]
        self.set_weights(weights if weights is not None else self.init_weights(seed))
        self.X = self.labels = self.loss = None
        self.A, self.H = [], []

    # ------------------------------------------------------------------ parameters
    def param_shapes(self):
        return [tuple(s) for q in self.layers for s in q.params.values()]

    def init_weights(self, seed=2):
        rng = np.random.default_rng(seed)
        out = []
        for shape in self.param_shapes():
            if len(shape) == 1:
                out.append(np.zeros(shape, np.float32))
                continue
            if len(shape) != 2:
                raise ProgramError("typed parameter families are not executable here")
            lim = np.sqrt(6.0 / (shape[0] + shape[1]))
            out.append(rng.uniform(-lim, lim, shape).astype(np.float32))
        return out

    def set_weights(self, weights):
        flat = [np.asarray(w, np.float32) for w in weights]
        ts = [t for P in self.params for t in P.values()]
        if len(flat) != len(ts):
            raise ShapeError("wrong number of weight matrices")
        with torch.no_grad():
            for t, w in zip(ts, flat):
                if w.size != t.numel():
                    raise ShapeError(f"weight of shape {w.shape}, want {tuple(t.shape)}")
                t.copy_(torch.from_numpy(w.reshape(t.shape)))

    def weights(self):
        return [t.detach().cpu().numpy().copy() for P in self.params for t in P.values()]

    def grads(self):
        return [(t.grad if t.grad is not None else torch.zeros_like(t)).cpu().numpy().copy()
                for P in self.params for t in P.values()]

    # ------------------------------------------------------------------ data
    def load_features(self, X):
        X = torch.as_tensor(X, dtype=torch.float32)
        if X.shape != (self.V, self.layers[0].f_in):
            raise ShapeError(f"features {tuple(X.shape)}, want ({self.V}, {self.layers[0].f_in})")
        self.X = X.to(self.device).contiguous()

    def load_labels(self, labels):
        self.labels = torch.as_tensor(np.asarray(labels), dtype=torch.int64).to(self.device)

    # ------------------------------------------------------------------ one layer
    def _layer(self, q, P, h):
        g = self.grid
        # hoisted per-vertex tables (P = h W_H, ...), computed once per layer on |V| rows
        tables = {}
        for name, (side, vx) in q.precompute.items():
            b = dict(P)
            b["vertex"] = h
            tables[name] = (side, evaluate(vx, b))
        names = prog.inputs_of(q.apply_edge)
        need = tuple(s for s, n in (("src", "edge.src"), ("dest", "edge.dest")) if n in names)
        if "edge.data" in names and any(ec.data is None for c in self.chunks.values() for ec in c):
            raise ConfigError("program reads edge.data: build the grid with GCN weights or pass edge_data")
        A_parts = []
        for j in range(g.P):
            j0, nj = g.begin(j), g.size(j)
            accs, chs = [], self.chunks[j]
            for ec in chs:                                    # source intervals ascending
                i0, ni = g.begin(ec.i), g.size(ec.i)
                tb = {n: (s, (t[i0:i0 + ni], t[j0:j0 + nj])) for n, (s, t) in tables.items()}
                et = scatter_chunk(h[i0:i0 + ni], h[j0:j0 + nj], ec, need, tb)
                acc = apply_edge_chunk(q.apply_edge, et, P)
                if acc.dim() == 1:
                    acc = acc.reshape(-1, 1)
                accs.append(acc)
            width = accs[0].shape[1] if accs else (q.apply_edge.width or q.f_in)
            A_parts.append(_GatherColumn.apply(q.accumulator, chs, nj, width, self.empty_fill, *accs))
        A = torch.cat(A_parts, 0) if len(A_parts) > 1 else A_parts[0]
        b = dict(P)
        b.update({"vertex": h, "accum": A})
        return A, evaluate(q.apply_vertex, b)

    def forward(self):
        if self.X is None:
            raise ConfigError("load_features first")
        for P in self.params:
            for t in P.values():
                t.grad = None
        h = self.X
        self.A, self.H = [], []
        for q, P in zip(self.layers, self.params):
            A, h = self._layer(q, P, h)
            self.A.append(A)
            self.H.append(h)
        if self.labels is not None:
            self.loss = ops.softmax_cross_entropy(h, self.labels)
        return h

    def backward(self):
        if self.loss is None:
            raise ConfigError("forward with labels first")
        self.loss.backward()

    def sgd(self, lr):
        """W <- W - lr * dW with the libsagann sgd kernel."""
        for P in self.params:
            for t in P.values():
                if t.grad is not None:
                    K.sgd(t.data, t.grad, lr)

    def train_step(self, lr=0.01):
        self.forward()
        self.backward()
        self.sgd(lr)
        return self.loss

    def check_status(self):
        if self.loss is not None and not bool(torch.isfinite(self.loss.detach()).all()):
            raise NumericError("non-finite loss")


def unfused_model(programs, grid, **kw):
    return UnfusedSAGAModel(programs, grid, **kw)
