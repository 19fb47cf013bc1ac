"""The reference's primitive API (tensor.py) on CUDA tensors, backed by libsagann kernels.

Same names, argument meaning and error behaviour as
``/root/reference/pkg/src/sagastream/tensor.py``; torch autograd replaces the
``Tape`` (tensor.py:69-121) and every forward/backward launches one of this
repo's sm_100a kernels:

=====================  ==============================  ================================
reference              here                            kernel
=====================  ==============================  ================================
take_rows  :424-436    take_rows                       sg_take_rows / sort + PASS gather
segment_sum :439-450   segment_sum                     sg_segment_sort + sg_propagate(PASS)
segment_max :453-484   segment_max                     sg_segment_max (/ _plan) / _bwd
mul/add/... :204-303   mul, add, sub, div, maximum...  sg_ewise
matmul     :306-319    matmul                          sg_gemm
softmax_cross_entropy  softmax_cross_entropy           sg_softmax_xent
=====================  ==============================  ================================

Strict mode (tensor.py:18-19, :161-163) checks every op output for NaN/Inf
on the device and raises NumericError; it synchronises, like the reference's
eager check.  Set ``ops.strict = False`` to skip it.
"""

import torch

from . import _lib
from . import kernels as K
from .errors import NumericError, ShapeError
from .graph import PassIndex

strict = True

_OPS = {"add": 0, "sub": 1, "mul": 2, "div": 3, "max": 4, "sigmoid": 5, "tanh": 6, "relu": 7}


def _check_device(*ts):
    for t in ts:
        if not t.is_cuda:
            raise RuntimeError("libsagann ops need CUDA tensors (no CPU fallback)")


def _finalize(t, op):
    if strict:
        flag = torch.zeros(1, dtype=torch.int32, device=t.device)
        if t.numel():
            K.check_finite(t.reshape(-1, t.shape[-1]) if t.dim() > 1 else t.reshape(1, -1), flag)
        if int(flag.item()):
            raise NumericError(f"non-finite value produced by '{op}'")
    return t


def _as2d(t):
    return t if t.dim() == 2 else t.reshape(-1, 1) if t.dim() == 1 else t.reshape(t.shape[0], -1)


# ------------------------------------------------------------------ segment index
def _segment_index(seg, num_segments):
    seg = torch.as_tensor(seg, device="cuda").to(torch.int64).contiguous()
    n = seg.numel()
    ptr = torch.empty(num_segments + 1, dtype=torch.int64, device=seg.device)
    perm = torch.empty(max(n, 1), dtype=torch.int32, device=seg.device)
    err = torch.zeros(1, dtype=torch.int32, device=seg.device)
    wsb = int(_lib.lib.sg_sort_workspace_bytes(n, num_segments))
    ws = torch.empty(wsb, dtype=torch.uint8, device=seg.device)
    _lib.check(_lib.lib.sg_segment_sort(seg.data_ptr(), n, num_segments, ptr.data_ptr(),
                                        perm.data_ptr(), err.data_ptr(), ws.data_ptr(), wsb,
                                        _lib.stream_handle()))
    if int(err.item()):
        raise ShapeError("segment id out of range")
    return PassIndex.from_device(ptr, perm[:n] if n else perm[:0])


def _gather_sum(a, pi, num_segments):
    a2 = _as2d(a).contiguous()
    F = a2.shape[1]
    out = torch.empty((num_segments, F), dtype=a.dtype, device=a.device)
    if pi.nnz == 0 or F == 0:
        out.zero_()
    else:
        K.propagate(pi, _lib.PROP_PASS, a2, out, F)
    return out.reshape((num_segments,) + tuple(a.shape[1:]))


class _SegmentSum(torch.autograd.Function):
    @staticmethod
    def forward(ctx, a, seg, num_segments):
        pi = _segment_index(seg, num_segments)
        ctx.seg = seg
        return _gather_sum(a, pi, num_segments)

    @staticmethod
    def backward(ctx, g):
        return take_rows(g, ctx.seg), None, None  # tensor.py:447-448 g[seg]


class _TakeRows(torch.autograd.Function):
    @staticmethod
    def forward(ctx, a, idx):
        a2 = _as2d(a).contiguous()
        n = idx.numel()
        out = torch.empty((n, a2.shape[1]), dtype=a.dtype, device=a.device)
        err = torch.zeros(1, dtype=torch.int32, device=a.device)
        _lib.check(_lib.lib.sg_take_rows(K.dtype_code(a2), a2.data_ptr(), a2.stride(0), a2.shape[0],
                                         idx.data_ptr(), n, out.data_ptr(), out.stride(0),
                                         a2.shape[1], err.data_ptr(), _lib.stream_handle()))
        if int(err.item()):
            raise ShapeError("row index out of range")
        ctx.idx, ctx.n = idx, a.shape[0]
        return out.reshape((n,) + tuple(a.shape[1:]))

    @staticmethod
    def backward(ctx, g):
        # tensor.py:431-434: sequential np.add.at into the source rows
        return _gather_sum(g, _segment_index(ctx.idx, ctx.n), ctx.n), None


def take_rows(a, idx, tape=None):
    """Scatter: y[k] = a[idx[k]] (tensor.py:424-436)."""
    _check_device(a)
    idx = torch.as_tensor(idx, device=a.device).to(torch.int64).contiguous()
    return _finalize(_TakeRows.apply(a, idx), "take_rows")


def segment_sum(a, segment_ids, num_segments, tape=None):
    """Gather(sum): rows added in row order (tensor.py:439-450)."""
    _check_device(a)
    seg = torch.as_tensor(segment_ids, device=a.device).to(torch.int64).contiguous()
    if seg.numel() != a.shape[0]:
        raise ShapeError("segment id count does not match row count")
    return _finalize(_SegmentSum.apply(a, seg, int(num_segments)), "segment_sum")


class _SegmentMax(torch.autograd.Function):
    @staticmethod
    def forward(ctx, a, seg, num_segments, empty_fill):
        pi = _segment_index(seg, num_segments)
        a2 = _as2d(a).contiguous()
        F = a2.shape[1]
        out = torch.empty((num_segments, F), dtype=a.dtype, device=a.device)
        arg = torch.empty((num_segments, F), dtype=torch.int64, device=a.device)
        if pi.n_splits > 0 and a2.dtype == torch.float32:
            # segments with more than T rows (hubs): plan-driven, bit-identical result
            nb = int(_lib.lib.sg_max_plan_workspace_bytes(pi.n_splits, pi.n_slots, F))
            ws = torch.empty(max(nb, 256), dtype=torch.uint8, device=a.device)
            _lib.check(_lib.lib.sg_segment_max_plan(
                pi.ptr.data_ptr(), pi.idx.data_ptr(), pi.items.data_ptr(), pi.n_items,
                pi.splits.data_ptr(), pi.n_splits, pi.n_slots, a2.data_ptr(), a2.stride(0),
                out.data_ptr(), F, arg.data_ptr(), F, F, float(empty_fill), ws.data_ptr(), ws.numel(),
                _lib.stream_handle()))
        else:
            _lib.check(_lib.lib.sg_segment_max(K.dtype_code(a2), pi.ptr.data_ptr(), pi.idx.data_ptr(),
                                               num_segments, a2.data_ptr(), a2.stride(0), out.data_ptr(),
                                               F, arg.data_ptr(), F, F, float(empty_fill),
                                               _lib.stream_handle()))
        ctx.save_for_backward(arg)
        ctx.shape, ctx.n = a.shape, a.shape[0]
        ctx.mark_non_differentiable(arg)
        return out.reshape((num_segments,) + tuple(a.shape[1:])), arg

    @staticmethod
    def backward(ctx, g, _garg):
        (arg,) = ctx.saved_tensors
        g2 = _as2d(g).contiguous()
        gx = torch.zeros((ctx.n, g2.shape[1]), dtype=g.dtype, device=g.device)
        _lib.check(_lib.lib.sg_segment_max_bwd(K.dtype_code(g2), g2.data_ptr(), g2.stride(0),
                                               arg.data_ptr(), arg.stride(0), arg.shape[0],
                                               gx.data_ptr(), gx.stride(0), g2.shape[1],
                                               _lib.stream_handle()))
        return gx.reshape(ctx.shape), None, None, None


def segment_max(a, segment_ids, num_segments, empty_fill=0.0, tape=None):
    """Gather(max); gradient to the lowest row attaining the max (tensor.py:453-484)."""
    _check_device(a)
    seg = torch.as_tensor(segment_ids, device=a.device).to(torch.int64).contiguous()
    if seg.numel() != a.shape[0]:
        raise ShapeError("segment id count does not match row count")
    out, _ = _SegmentMax.apply(a, seg, int(num_segments), float(empty_fill))
    return _finalize(out, "segment_max")


# ------------------------------------------------------------------ elementwise
def _broadcast_kind(sa, sb):
    """tensor.py:171-188."""
    sa, sb = tuple(sa), tuple(sb)
    if sa == sb:
        return "equal"
    if len(sb) < len(sa) and sb == sa[len(sa) - len(sb):]:
        return "b_lead"
    if len(sa) < len(sb) and sa == sb[len(sb) - len(sa):]:
        return "a_lead"
    if len(sa) == 2 and len(sb) == 2 and sb == (sa[0], 1):
        return "b_row"
    if len(sa) == 2 and len(sb) == 2 and sa == (sb[0], 1):
        return "a_row"
    raise ShapeError(f"shapes {sa} and {sb} are not broadcast-compatible")


def _ewise_raw(op, a, b=None):
    a2 = _as2d(a).contiguous()
    out = torch.empty_like(a2)
    if b is None:
        bp, br, bc, ldb = None, 0, 0, 0
    else:
        b2 = b.contiguous()
        if b2.shape == a.shape:
            b2 = _as2d(b2)
            br, bc = b2.shape
        elif b2.dim() == 2 and b2.shape[1] == 1:      # b_row
            br, bc = b2.shape[0], 1
        else:                                          # b_lead: broadcast along leading axis
            b2 = b2.reshape(1, -1)
            br, bc = 1, b2.shape[1]
        bp, ldb = b2.data_ptr(), b2.stride(0) if b2.dim() == 2 else bc
    _lib.check(_lib.lib.sg_ewise(_OPS[op], a2.shape[0], a2.shape[1], a2.data_ptr(), a2.stride(0),
                                 bp, br, bc, ldb, out.data_ptr(), out.stride(0),
                                 _lib.stream_handle()))
    return out.reshape(a.shape)


def _reduce_to(g, shape, kind, side):
    """tensor.py:191-201, on the device (sg_reduce_sum: fixed-order sums, no torch reduction)."""
    if kind == "equal" or (kind == "b_lead" and side == "a") or (kind == "a_lead" and side == "b") \
            or (kind == "b_row" and side == "a") or (kind == "a_row" and side == "b"):
        return g
    g2 = _as2d(g).contiguous()
    if kind in ("a_lead", "b_lead"):
        n = 1
        for d in shape:
            n *= d
        g2 = g2.reshape(-1, n)
        out = torch.empty(n, dtype=g.dtype, device=g.device)
        ws = torch.empty(int(_lib.lib.sg_reduce_workspace_bytes(n)), dtype=torch.uint8, device=g.device)
        _lib.check(_lib.lib.sg_reduce_sum(0, g2.data_ptr(), g2.stride(0), g2.shape[0], n, out.data_ptr(),
                                          ws.data_ptr(), ws.numel(), _lib.stream_handle()))
        return out.reshape(shape)
    out = torch.empty((g2.shape[0], 1), dtype=g.dtype, device=g.device)
    _lib.check(_lib.lib.sg_reduce_sum(1, g2.data_ptr(), g2.stride(0), g2.shape[0], g2.shape[1],
                                      out.data_ptr(), None, 0, _lib.stream_handle()))
    return out


def _b_view(b, a_shape):
    """(tensor, b_rows, b_cols, ldb) of operand b broadcast against a [rows, cols] view of a."""
    b2 = b.contiguous()
    if tuple(b2.shape) == tuple(a_shape):
        b2 = _as2d(b2)
        return b2, b2.shape[0], b2.shape[1], b2.stride(0)
    if b2.dim() == 2 and b2.shape[1] == 1:             # b_row
        return b2, b2.shape[0], 1, b2.stride(0)
    b2 = b2.reshape(1, -1)                             # b_lead
    return b2, 1, b2.shape[1], b2.shape[1]


class _Binary(torch.autograd.Function):
    @staticmethod
    def forward(ctx, op, a, b):
        kind = _broadcast_kind(a.shape, b.shape)
        if op == "div" and strict and bool((b == 0).any()):
            raise NumericError("division by zero")
        if kind in ("a_lead", "a_row"):
            y = _ewise_raw(op, a.expand(b.shape).contiguous(), b)
        else:
            y = _ewise_raw(op, a, b)
        ctx.op, ctx.kind = op, kind
        ctx.a_shape, ctx.b_shape = tuple(a.shape), tuple(b.shape)
        ctx.save_for_backward(a, b)
        return y

    @staticmethod
    def backward(ctx, g):
        # both partials in one sg_ewise_bwd pass (tensor.py:255-265), then _reduce_to
        a, b = ctx.saved_tensors
        op, kind = ctx.op, ctx.kind
        if kind in ("a_lead", "a_row"):
            a = a.expand(b.shape)
            ae, be = a.contiguous(), b
        else:
            ae, be = a, b
        a2 = _as2d(ae).contiguous()
        g2 = _as2d(g).contiguous()
        b2, br, bc, ldb = _b_view(be, ae.shape)
        ga = torch.empty_like(a2)
        gb = torch.empty_like(a2)
        _lib.check(_lib.lib.sg_ewise_bwd(_OPS[op], a2.shape[0], a2.shape[1], g2.data_ptr(), g2.stride(0),
                                         a2.data_ptr(), a2.stride(0), b2.data_ptr(), br, bc, ldb,
                                         ga.data_ptr(), ga.stride(0), gb.data_ptr(), gb.stride(0),
                                         _lib.stream_handle()))
        ga, gb = ga.reshape(ae.shape), gb.reshape(ae.shape)
        return None, _reduce_to(ga, ctx.a_shape, kind, "a"), _reduce_to(gb, ctx.b_shape, kind, "b")


class _Unary(torch.autograd.Function):
    @staticmethod
    def forward(ctx, op, a):
        y = _ewise_raw(op, a)
        ctx.op = op
        ctx.save_for_backward(a, y)
        return y

    @staticmethod
    def backward(ctx, g):
        # tensor.py:231-236 on the device: sigmoid g*y*(1-y) (op 9), tanh g*(1-y*y) (op 10),
        # relu g*(x>0) (op 8, gradient 0 at 0)
        a, y = ctx.saved_tensors
        code, other = {"sigmoid": (9, y), "tanh": (10, y), "relu": (8, a)}[ctx.op]
        g2 = _as2d(g).contiguous()
        o2 = _as2d(other).contiguous()
        out = torch.empty_like(g2)
        _lib.check(_lib.lib.sg_ewise(code, g2.shape[0], g2.shape[1], g2.data_ptr(), g2.stride(0),
                                     o2.data_ptr(), o2.shape[0], o2.shape[1], o2.stride(0),
                                     out.data_ptr(), out.stride(0), _lib.stream_handle()))
        return None, out.reshape(g.shape)


def _binary(op, a, b):
    _check_device(a, b)
    return _finalize(_Binary.apply(op, a, b), op)


def add(a, b, tape=None):
    return _binary("add", a, b)


def sub(a, b, tape=None):
    return _binary("sub", a, b)


def mul(a, b, tape=None):
    return _binary("mul", a, b)


def div(a, b, tape=None):
    return _binary("div", a, b)


def maximum(a, b, tape=None):
    return _binary("max", a, b)


def sigmoid(a, tape=None):
    _check_device(a)
    return _finalize(_Unary.apply("sigmoid", a), "sigmoid")


def tanh(a, tape=None):
    _check_device(a)
    return _finalize(_Unary.apply("tanh", a), "tanh")


def relu(a, tape=None):
    _check_device(a)
    return _finalize(_Unary.apply("relu", a), "relu")


def elementwise(op, a, b=None, tape=None):
    """tensor.py:211-223 dispatcher."""
    if op in ("sigmoid", "tanh", "relu"):
        if b is not None:
            raise ShapeError(f"'{op}' is unary")
        return {"sigmoid": sigmoid, "tanh": tanh, "relu": relu}[op](a)
    if op in ("add", "sub", "mul", "div", "max"):
        if b is None:
            raise ShapeError(f"'{op}' needs two operands")
        return _binary(op, a, b)
    raise ShapeError(f"unknown elementwise op '{op}'")


# ------------------------------------------------------------------ matmul / loss
class _Matmul(torch.autograd.Function):
    @staticmethod
    def forward(ctx, a, b):
        out = torch.empty((a.shape[0], b.shape[1]), dtype=torch.float32, device=a.device)
        K.gemm(a.contiguous(), b.contiguous(), out, prec=_lib.GEMM_TF32X3)
        ctx.save_for_backward(a, b)
        return out

    @staticmethod
    def backward(ctx, g):
        a, b = ctx.saved_tensors
        g = g.contiguous()
        ga = torch.empty_like(a)
        gb = torch.empty_like(b)
        # tcgen05 3xTF32 (fp32-parity error bound), like the forward
        K.gemm(g, b.contiguous(), ga, trans_b=True, prec=_lib.GEMM_TF32X3)   # g @ w.T  (tensor.py:317)
        K.gemm(a.contiguous(), g, gb, trans_a=True, prec=_lib.GEMM_TF32X3)   # x.T @ g
        return ga, gb


def matmul(a, b, tape=None):
    """ApplyVertex matmul (tensor.py:306-319)."""
    _check_device(a, b)
    if a.dim() != 2 or b.dim() != 2:
        raise ShapeError(f"matmul needs 2-D operands, got {tuple(a.shape)} x {tuple(b.shape)}")
    if a.shape[1] != b.shape[0]:
        raise ShapeError(f"matmul inner extents differ: {tuple(a.shape)} x {tuple(b.shape)}")
    return _finalize(_Matmul.apply(a.float(), b.float()), "matmul")


class _Xent(torch.autograd.Function):
    @staticmethod
    def forward(ctx, z, labels):
        z = z.contiguous()
        loss = torch.empty(1, dtype=torch.float32, device=z.device)
        dz = torch.empty_like(z)
        err = torch.zeros(1, dtype=torch.int32, device=z.device)
        K.softmax_xent(z, labels, loss, dz, err, relu_input=False)
        if int(err.item()):
            raise ShapeError("label out of range")
        ctx.save_for_backward(dz)
        return loss.reshape(())

    @staticmethod
    def backward(ctx, g):
        (dz,) = ctx.saved_tensors
        return dz * g, None


def softmax_cross_entropy(logits, labels, tape=None):
    """Mean softmax cross-entropy (tensor.py:487-506)."""
    _check_device(logits)
    lab = torch.as_tensor(labels, device=logits.device).to(torch.int64).contiguous()
    if logits.dim() != 2 or lab.shape[0] != logits.shape[0]:
        raise ShapeError("logits must be [n, classes] with one label per row")
    return _finalize(_Xent.apply(logits.float(), lab), "softmax_xent")
