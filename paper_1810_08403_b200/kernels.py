"""Typed torch-tensor wrappers over the libsagann device entry points.

Every function here launches one of the repo's own sm_100a kernels on the
current torch stream (or the given one) and raises the mirrored reference
exception on a bad status.  torch is used only for device memory and streams.
"""

import ctypes
import os

import torch

from . import _lib
from . import graph
from ._lib import check, lib, stream_handle, tptr
from .errors import ShapeError

_DT = {torch.float32: _lib.SG_F32, torch.bfloat16: _lib.SG_BF16}


def dtype_code(t):
    try:
        return _DT[t.dtype]
    except KeyError:
        raise TypeError(f"unsupported dtype {t.dtype}; expected float32 or bfloat16") from None


def ld(t):
    """Leading dimension (row stride, elements) of a row-major 2-D view."""
    if t.dim() != 2:
        raise ValueError("expected a 2-D tensor")
    if t.numel() == 0:
        return max(t.shape[1], 1)
    if t.stride(1) != 1 and t.shape[1] > 1:
        raise ValueError("expected a 2-D tensor with unit column stride")
    return max(t.stride(0), t.shape[1]) if t.shape[0] == 1 else t.stride(0)


class Workspace:
    """Grow-only device scratch buffer (caller-owned workspace of the C-ABI)."""

    def __init__(self, device):
        self.device = device
        self.buf = torch.empty(0, dtype=torch.uint8, device=device)

    def get(self, nbytes):
        nbytes = max(int(nbytes), 256)
        if self.buf.numel() < nbytes:
            self.buf = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        return self.buf


# hub-row cache: opt-in (SG_HUB=1).  With the canonical (source-sorted) CSC the L1 serves the
# hot rows and the 64-KB shared-memory carve-out cost more than it saved (Reddit L0 15.5 vs
# 14.2 ms, profiles/r01_hub_cluster_ab.txt)
HUB_CACHE = os.environ.get("SG_HUB", "0") == "1"


def _vec_ok(t, vw):
    return t is None or (ld(t) % vw == 0 and t.data_ptr() % 16 == 0)


def _hub_for(pi, mode, dt, G, out0, mask, F, g_off):
    """The pass's hub-row cache if this call can use it (GCN / PASS, 16-B rows, > 16 vectors)."""
    if not HUB_CACHE or mode not in (_lib.PROP_PASS, _lib.PROP_GCN) or not hasattr(pi, "hub"):
        return None
    vw = 4 if dt == _lib.SG_F32 else 8
    if g_off % vw or not (_vec_ok(G, vw) and _vec_ok(out0, vw) and _vec_ok(mask, vw)):
        return None
    cap = int(lib.sg_propagate_hub_capacity(F, dt))
    return pi.hub(cap) if cap > 0 else None


def propagate(pi, mode, G, out0, F, *, g_off=0, R=None, r_off=0, out1=None, mask=None,
              accumulate=False, ws=None, stream=None, hub=True):
    """One fused Scatter-ApplyEdge-Gather pass over PassIndex ``pi`` (sg_propagate; with the
    hub-row cache, sg_propagate_hub, when the pass has hubs -- bitwise identical)."""
    dt = dtype_code(G)
    if dt == _lib.SG_BF16 and out0.dtype == torch.float32:
        dt = _lib.SG_BF16_F32OUT       # bf16 rows in, fp32 aggregate out
    elif out0.dtype != G.dtype:
        raise TypeError(f"propagate: {G.dtype} rows into a {out0.dtype} output is not supported")
    h = _hub_for(pi, mode, dt, G, out0, mask, F, g_off) if hub and R is None and out1 is None else None
    if (h is None and graph.STAGED and mode in (_lib.PROP_PASS, _lib.PROP_GCN) and dt == _lib.SG_F32
            and R is None and out1 is None and g_off == 0 and hasattr(pi, "stage_plan")
            and _vec_ok(G, 4) and _vec_ok(out0, 4) and _vec_ok(mask, 4)):
        sp = pi.stage_plan(F)
        if sp is not None:
            wsb = int(lib.sg_propagate_workspace_bytes(0, sp.n_splits, sp.n_slots, F, mode))
            buf = ws.get(wsb) if ws is not None else torch.empty(wsb, dtype=torch.uint8, device=G.device)
            check(lib.sg_propagate_staged(
                mode, tptr(sp.pieces), tptr(sp.group_batch), sp.n_groups, tptr(sp.batch_src_off),
                tptr(sp.batch_src), tptr(sp.batch_ent_off), tptr(sp.entries), tptr(sp.batch_pofs), sp.G,
                sp.S, sp.EMAX, sp.stages, sp.n_splits, sp.n_slots, tptr(G), ld(G), tptr(out0), ld(out0), tptr(mask),
                ld(mask) if mask is not None else 0, F, int(bool(accumulate)), tptr(buf), buf.numel(),
                stream_handle(stream)))
            return
    wsb = pi.workspace_bytes(F, mode)
    buf = ws.get(wsb) if ws is not None else torch.empty(wsb, dtype=torch.uint8, device=G.device)
    idx, rows, n_hub = (h[0], h[1], h[2]) if h is not None else (pi.idx, None, 0)
    check(lib.sg_propagate_hub(
        mode, dt, tptr(pi.ptr), tptr(idx), tptr(pi.w), pi.n_rows, tptr(pi.items), pi.n_items,
        tptr(pi.splits), pi.n_splits, pi.n_slots, tptr(G), ld(G), g_off,
        tptr(R), ld(R) if R is not None else 0, r_off, tptr(out0), ld(out0),
        tptr(out1), ld(out1) if out1 is not None else 0, tptr(mask),
        ld(mask) if mask is not None else 0, F, int(bool(accumulate)), tptr(rows), n_hub,
        tptr(buf), buf.numel(), stream_handle(stream)))


def gemm(A, B, C, *, trans_a=False, trans_b=False, relu_out=None, prec=_lib.GEMM_F32, ws=None,
         stream=None, nonfinite=None):
    """C = op(A) @ op(B) (+ relu_out = relu(C)) through sg_gemm_ex.

    fp32 A/B for GEMM_F32 / GEMM_TF32X3, bf16 A/B for GEMM_BF16; C and relu_out fp32 or bf16
    (bf16 outputs with GEMM_BF16 or GEMM_TF32X3); C may be None when relu_out is given.
    ``nonfinite`` (int32 device flag) is OR-ed with 1 if C has a non-finite element."""
    M = A.shape[1] if trans_a else A.shape[0]
    K = A.shape[0] if trans_a else A.shape[1]
    N = B.shape[0] if trans_b else B.shape[1]
    Kb = B.shape[1] if trans_b else B.shape[0]
    if K != Kb:
        raise ShapeError(f"matmul inner extents differ: {K} vs {Kb}")
    want = _lib.SG_BF16 if prec == _lib.GEMM_BF16 else _lib.SG_F32
    if dtype_code(A) != want or dtype_code(B) != want:
        raise TypeError(f"gemm precision {prec} takes {'bf16' if want else 'fp32'} operands")
    wsb = int(lib.sg_gemm_workspace_bytes(M, N, K, prec))
    buf = (ws.get(wsb) if ws is not None else torch.empty(max(wsb, 256), dtype=torch.uint8,
                                                            device=A.device))
    d = _lib.GemmDesc()
    d.prec, d.trans_a, d.trans_b = prec, int(trans_a), int(trans_b)
    d.epilogue = _lib.EPI_RELU_DUAL if relu_out is not None else _lib.EPI_NONE
    d.M, d.N, d.K = M, N, K
    d.A, d.lda, d.B, d.ldb = tptr(A), ld(A), tptr(B), ld(B)
    d.C, d.ldc = tptr(C), (ld(C) if C is not None else 0)
    d.c_dtype = dtype_code(C) if C is not None else _lib.SG_F32
    d.D, d.ldd = tptr(relu_out), (ld(relu_out) if relu_out is not None else 0)
    d.d_dtype = dtype_code(relu_out) if relu_out is not None else _lib.SG_F32
    d.nonfinite = tptr(nonfinite)
    d.workspace, d.workspace_bytes = tptr(buf), buf.numel()
    check(lib.sg_gemm_ex(ctypes.byref(d), stream_handle(stream)))


def softmax_xent(Z, labels, loss, dZ, err, *, relu_input=True, n_total=0, ws=None, stream=None):
    n, C = Z.shape
    wsb = int(lib.sg_xent_workspace_bytes(n))
    buf = ws.get(wsb) if ws is not None else torch.empty(wsb, dtype=torch.uint8, device=Z.device)
    check(lib.sg_softmax_xent(tptr(Z), ld(Z), int(relu_input), tptr(labels), n, C, int(n_total), tptr(loss),
                              tptr(dZ), ld(dZ), tptr(err), tptr(buf), buf.numel(),
                              stream_handle(stream)))


def _max_ws(pi, F, ws, device):
    nb = int(lib.sg_max_plan_workspace_bytes(pi.n_splits, pi.n_slots, F))
    return ws.get(nb) if ws is not None else torch.empty(max(nb, 256), dtype=torch.uint8, device=device)


def _check_pos_range(pi, pos_base):
    """Max-gather positions are int32 with -1 = empty (segment.cu): refuse a pass whose
    global positions pos_base .. pos_base + nnz would wrap (graphs with >= 2^31 edges)."""
    if int(pos_base) < 0 or int(pos_base) + int(getattr(pi, "nnz", 0)) > 2**31 - 1:
        raise ShapeError(f"max gather positions {pos_base} + {getattr(pi, 'nnz', 0)} exceed int32")


def max_gather(pi, Y, out, arg, F, empty_fill=0.0, *, pos_base=0, accumulate=False, finalize=True,
               stream=None, ws=None):
    """Fused Gather(max) over CSC pass index ``pi`` (argmax = pos_base + CSC position, int32).
    Passes with split rows (hubs) run the plan-driven kernel (bit-identical result)."""
    _check_pos_range(pi, pos_base)
    if getattr(pi, "n_splits", 0) > 0:
        buf = _max_ws(pi, F, ws, Y.device)
        check(lib.sg_max_gather_plan(tptr(pi.ptr), tptr(pi.idx), tptr(pi.items), pi.n_items,
                                     tptr(pi.splits), pi.n_splits, pi.n_slots, tptr(Y), ld(Y), tptr(out),
                                     ld(out), tptr(arg), ld(arg), F, float(empty_fill), int(pos_base),
                                     int(bool(accumulate)), int(bool(finalize)), tptr(buf), buf.numel(),
                                     stream_handle(stream)))
        return
    check(lib.sg_max_gather(tptr(pi.ptr), tptr(pi.idx), pi.n_rows, tptr(Y), ld(Y), tptr(out), ld(out),
                            tptr(arg), ld(arg), F, float(empty_fill), int(pos_base),
                            int(bool(accumulate)), int(bool(finalize)), stream_handle(stream)))


def max_gather_bwd(pi, pos, G, arg, out, F, mask=None, *, pos_base=0, accumulate=False, stream=None,
                   ws=None):
    """Backward of max_gather over CSR pass index ``pi`` (pos = CSC position per CSR edge).
    Passes with split rows sum a heavy row's subgroups in subgroup order."""
    _check_pos_range(pi, pos_base)
    if getattr(pi, "n_splits", 0) > 0:
        buf = _max_ws(pi, F, ws, G.device)
        check(lib.sg_max_gather_bwd_plan(tptr(pi.ptr), tptr(pi.idx), tptr(pos), tptr(pi.items), pi.n_items,
                                         tptr(pi.splits), pi.n_splits, pi.n_slots, tptr(G), ld(G), tptr(arg),
                                         ld(arg), tptr(out), ld(out), F, tptr(mask),
                                         ld(mask) if mask is not None else 0, int(pos_base),
                                         int(bool(accumulate)), tptr(buf), buf.numel(), stream_handle(stream)))
        return
    check(lib.sg_max_gather_bwd(tptr(pi.ptr), tptr(pi.idx), tptr(pos), pi.n_rows, tptr(G), ld(G),
                                tptr(arg), ld(arg), tptr(out), ld(out), F, tptr(mask),
                                ld(mask) if mask is not None else 0, int(pos_base),
                                int(bool(accumulate)), stream_handle(stream)))


def ewise(op, a, b, out, stream=None):
    """sg_ewise on 2-D views; b is [rows, cols], [rows, 1] (b_row) or [1, cols] (b_lead)."""
    check(lib.sg_ewise(op, a.shape[0], a.shape[1], tptr(a), ld(a), tptr(b),
                       b.shape[0] if b is not None else 0, b.shape[1] if b is not None else 0,
                       ld(b) if b is not None else 0, tptr(out), ld(out), stream_handle(stream)))


def sgd(W, dW, lr, stream=None):
    check(lib.sg_sgd(tptr(W), tptr(dW), W.numel(), float(lr), stream_handle(stream)))


def check_finite(X, flag, stream=None):
    X2 = X if X.dim() == 2 else X.reshape(1, -1)
    check(lib.sg_check_finite(dtype_code(X2), tptr(X2), X2.shape[0], X2.shape[1], ld(X2),
                              tptr(flag), stream_handle(stream)))


def convert(X, Y, stream=None):
    check(lib.sg_convert(dtype_code(X), dtype_code(Y), tptr(X), ld(X), tptr(Y), ld(Y), X.shape[0],
                         X.shape[1], stream_handle(stream)))
