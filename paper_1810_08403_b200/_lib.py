"""ctypes binding of libsagann.so (the C-ABI declared in include/sagann.h).

This is the reference-side binding a Python caller needs: plain pointers and
sizes cross the boundary, status codes come back and are mapped to the
reference's exception classes (errors.py).  There is no fallback: if the
shared library is missing the import fails loudly (build it with
``python -c "import __graft_entry__ as g; g.build()"`` or ``make -C
paper_1810_08403_b200/csrc``).
"""

import ctypes
import os
import re

import numpy as np

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
# SG_LIB_PATH: an alternate in-tree build for A/B timing (e.g. libsagann_ab.so)
LIB_PATH = os.environ.get("SG_LIB_PATH") or os.path.join(_HERE, "libsagann.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "sagann.h")

SG_OK, SG_ESHAPE, SG_ENUMERIC, SG_EBUDGET, SG_ECUDA, SG_ENCCL, SG_EINVAL, SG_EFORMAT = range(8)
SG_F32, SG_BF16, SG_BF16_F32OUT = 0, 1, 2
PROP_PASS, PROP_GCN, PROP_GGCN_FWD, PROP_GGCN_BWD_DST, PROP_GGCN_BWD_SRC, PROP_GGCN_FWD_S = range(6)
EPI_NONE, EPI_RELU_DUAL = 0, 1
GEMM_F32, GEMM_TF32X3, GEMM_BF16 = 0, 1, 2

ITEM_DTYPE = np.dtype([("row_begin", "<i4"), ("row_end", "<i4"), ("e_begin", "<i8"),
                       ("e_end", "<i8"), ("split", "<i4"), ("sub", "<i4")])
SPLIT_DTYPE = np.dtype([("row", "<i4"), ("n_sub", "<i4"), ("slot0", "<i8")])
assert ITEM_DTYPE.itemsize == 32 and SPLIT_DTYPE.itemsize == 16

_i64, _i32, _f64, _f32 = ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_float
_u64, _p = ctypes.c_uint64, ctypes.c_void_p
_s = ctypes.c_char_p

class GemmDesc(ctypes.Structure):
    """sg_gemm_desc (include/sagann.h)."""
    _fields_ = [("prec", ctypes.c_int), ("trans_a", ctypes.c_int), ("trans_b", ctypes.c_int),
                ("epilogue", ctypes.c_int), ("M", ctypes.c_int64), ("N", ctypes.c_int64),
                ("K", ctypes.c_int64), ("A", ctypes.c_void_p), ("lda", ctypes.c_int64),
                ("B", ctypes.c_void_p), ("ldb", ctypes.c_int64), ("C", ctypes.c_void_p),
                ("ldc", ctypes.c_int64), ("c_dtype", ctypes.c_int), ("D", ctypes.c_void_p),
                ("ldd", ctypes.c_int64), ("d_dtype", ctypes.c_int), ("nonfinite", ctypes.c_void_p),
                ("workspace", ctypes.c_void_p), ("workspace_bytes", ctypes.c_int64)]


_SIGS = {
    "sg_gemm_ex": (ctypes.c_int, [ctypes.POINTER(GemmDesc), ctypes.c_void_p]),
    "sg_last_error": (ctypes.c_char_p, []),
    "sg_version": (_i32, []),
    "sg_device_sm_count": (_i32, [_i32, _p]),
    "sg_launch_count": (_i64, []),
    "sg_host_gen_rmat": (_i32, [_i64, _i64, _u64, _f64, _f64, _f64, _i64, _p, _p]),
    "sg_host_gen_uniform": (_i32, [_i64, _i64, _u64, _i64, _p, _p]),
    "sg_host_gen_features": (_i32, [_i64, _i64, _u64, _i64, _p, _i64]),
    "sg_host_degrees": (_i32, [_p, _p, _i64, _i64, _p, _p]),
    "sg_host_reencode_balance": (_i32, [_p, _p, _i64, _i64, _i64, _p]),
    "sg_host_partition_layout": (_i32, [_i64, _i64, _p, _p]),
    "sg_host_partition_2d": (_i32, [_p, _p, _i64, _i64, _i64] + [_p] * 9),
    "sg_host_gcn_weights": (_i32, [_p, _p, _p, _p, _p, _i64, _p]),
    "sg_host_plan": (_i32, [_p, _i64, _i64, _i64, _i64, _p, _p, _p, _p, _p]),
    "sg_host_plan_order": (_i32, [_p, _i64, _p]),
    "sg_host_stage_plan": (_i32, [_p, _p, _p, _i64, _i64, _i32, _i32, _i32] + [_p] * 8),
    "sg_stage_group_pieces": (_i32, [_i64]),
    "sg_stage_smem_bytes": (_i64, [_i32, _i32, _i32, _i64, _i32]),
    "sg_propagate_staged": (_i32, [_i32, _p, _p, _i64, _p, _p, _p, _p, _p, _i32, _i32, _i32, _i32, _i64, _i64,
                                   _p, _i64, _p, _i64, _p, _i64, _i64, _i32, _p, _i64, _p]),
    "sg_host_scan_edges": (_i32, [_s, _i64, _p, _p, _p]),
    "sg_host_read_edges": (_i32, [_s, _i64, _p, _p, _p]),
    "sg_host_scan_matrix_text": (_i32, [_s, _p, _p]),
    "sg_host_read_matrix_text": (_i32, [_s, _i64, _i64, _p]),
    "sg_host_read_matrix_bin_header": (_i32, [_s, _p, _p]),
    "sg_host_read_matrix_bin": (_i32, [_s, _i64, _i64, _p]),
    "sg_host_write_matrix_bin": (_i32, [_s, _i64, _i64, _p]),
    "sg_host_scan_labels": (_i32, [_s, _p]),
    "sg_host_read_labels": (_i32, [_s, _i64, _p]),
    "sg_host_hash64": (_u64, [_p, _i64, _u64]),
    "sg_propagate_workspace_bytes": (_i64, [_i64, _i64, _i64, _i64, _i32]),
    "sg_propagate": (_i32, [_i32, _i32, _p, _p, _p, _i64, _p, _i64, _p, _i64, _i64,
                            _p, _i64, _i64, _p, _i64, _i64, _p, _i64, _p, _i64, _p, _i64,
                            _i64, _i32, _p, _i64, _p]),
    "sg_propagate_hub_capacity": (_i64, [_i64, _i32]),
    "sg_propagate_hub": (_i32, [_i32, _i32, _p, _p, _p, _i64, _p, _i64, _p, _i64, _i64,
                                _p, _i64, _i64, _p, _i64, _i64, _p, _i64, _p, _i64, _p, _i64,
                                _i64, _i32, _p, _i64, _p, _i64, _p]),
    "sg_segment_max": (_i32, [_i32, _p, _p, _i64, _p, _i64, _p, _i64, _p, _i64, _i64, _f32, _p]),
    "sg_segment_max_bwd": (_i32, [_i32, _p, _i64, _p, _i64, _i64, _p, _i64, _i64, _p]),
    "sg_max_gather": (_i32, [_p, _p, _i64, _p, _i64, _p, _i64, _p, _i64, _i64, _f32, _i64, _i32,
                             _i32, _p]),
    "sg_max_gather_bwd": (_i32, [_p, _p, _p, _i64, _p, _i64, _p, _i64, _p, _i64, _i64, _p, _i64,
                                 _i64, _i32, _p]),
    "sg_take_rows":(_i32, [_i32, _p, _i64, _i64, _p, _i64, _p, _i64, _i64, _p, _p]),
    "sg_sort_workspace_bytes": (_i64, [_i64, _i64]),
    "sg_segment_sort": (_i32, [_p, _i64, _i64, _p, _p, _p, _p, _i64, _p]),
    "sg_gemm_workspace_bytes": (_i64, [_i64, _i64, _i64, _i32]),
    "sg_gemm": (_i32, [_i32, _i32, _i32, _i64, _i64, _i64, _p, _i64, _p, _i64, _p, _i64, _i32,
                       _p, _i64, _p, _i64, _p]),
    "sg_xent_workspace_bytes": (_i64, [_i64]),
    "sg_softmax_xent": (_i32, [_p, _i64, _i32, _p, _i64, _i64, _i64, _p, _p, _i64, _p, _p, _i64, _p]),
    "sg_sgd": (_i32, [_p, _p, _i64, _f32, _p]),
    "sg_check_finite": (_i32, [_i32, _p, _i64, _i64, _i64, _p, _p]),
    "sg_ewise": (_i32, [_i32, _i64, _i64, _p, _i64, _p, _i64, _i64, _i64, _p, _i64, _p]),
    "sg_ewise_bwd": (_i32, [_i32, _i64, _i64, _p, _i64, _p, _i64, _p, _i64, _i64, _i64, _p, _i64, _p,
                            _i64, _p]),
    "sg_reduce_workspace_bytes": (_i64, [_i64]),
    "sg_reduce_sum": (_i32, [_i32, _p, _i64, _i64, _i64, _p, _p, _i64, _p]),
    "sg_max_plan_workspace_bytes": (_i64, [_i64, _i64, _i64]),
    "sg_max_gather_plan": (_i32, [_p, _p, _p, _i64, _p, _i64, _i64, _p, _i64, _p, _i64, _p, _i64, _i64,
                                  _f32, _i64, _i32, _i32, _p, _i64, _p]),
    "sg_segment_max_plan": (_i32, [_p, _p, _p, _i64, _p, _i64, _i64, _p, _i64, _p, _i64, _p, _i64, _i64,
                                   _f32, _p, _i64, _p]),
    "sg_max_gather_bwd_plan": (_i32, [_p, _p, _p, _p, _i64, _p, _i64, _i64, _p, _i64, _p, _i64, _p, _i64,
                                      _i64, _p, _i64, _i64, _i32, _p, _i64, _p]),
    "sg_gru_gates": (_i32, [_i64, _i64, _p, _i64, _p, _i64, _i64, _p, _i64, _p, _p, _p, _i64, _p]),
    "sg_gru_out": (_i32, [_i64, _i64, _p, _i64, _i64, _p, _i64, _p, _p, _i64, _p, _p, _i64, _i64, _p]),
    "sg_gru_bwd1": (_i32, [_i64, _i64, _p, _i64, _p, _p, _i64, _p, _i64, _p, _i64, _i64, _p, _i64, _p]),
    "sg_gru_bwd2": (_i32, [_i64, _i64, _p, _i64, _p, _i64, _p, _i64, _p, _i64, _p, _i64, _i64, _p]),
    "sg_convert": (_i32, [_i32, _i32, _p, _i64, _p, _i64, _i64, _i64, _p]),
}


def header_symbols(path=HEADER_PATH):
    """Every function the C-ABI header declares (used by the export test)."""
    txt = open(path).read()
    return sorted(set(re.findall(r"\b(sg_[a-z0-9_]+)\s*\(", txt)))


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libsagann.so not found at {LIB_PATH}: build it with `make -C "
            f"{os.path.join(_HERE, 'csrc')}` (no CPU fallback exists)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()

_EXC = {
    SG_EFORMAT: errors.GraphFormatError,
    SG_ESHAPE: errors.ShapeError,
    SG_ENUMERIC: errors.NumericError,
    SG_EBUDGET: errors.BudgetError,
}


def check(rc):
    """Map a C-ABI status to the mirrored reference exception."""
    if rc != SG_OK:
        msg = lib.sg_last_error().decode(errors="replace")
        raise _EXC.get(rc, errors.NativeError)(msg)
    return rc


def nptr(a):
    """Host pointer of a C-contiguous numpy array (or None)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "numpy buffer must be C-contiguous"
    return a.ctypes.data


def tptr(t):
    """Device pointer of a torch tensor (or None)."""
    return None if t is None else t.data_ptr()


def stream_handle(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
