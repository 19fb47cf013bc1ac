"""Pure-numpy restatement of the reference primitives (test infrastructure only).

Each function follows ``/root/reference/pkg/src/sagastream/tensor.py`` line for
line in arithmetic and order (so fp32/fp64 results are bit-identical to the
reference's), minus the ``Tensor``/``Tape`` object plumbing: forward and backward
are separate functions and the caller composes them in tape order.
"""

import numpy as np

STRICT = True  # tensor.py:18-19


class EngineError(Exception):
    """errors.py:4"""


class ShapeError(EngineError):
    """errors.py:8"""


class NumericError(EngineError):
    """errors.py:12"""


def finalize(arr, op):
    """tensor.py:161-163 -- strict-mode non-finite check on every op output."""
    if STRICT and not np.all(np.isfinite(arr)):
        raise NumericError(f"non-finite value produced by '{op}'")
    return arr


# ----------------------------------------------------------------- elementwise
def sigmoid(x):
    """tensor.py:205 ``1.0 / (1.0 + np.exp(-x))``."""
    return finalize(1.0 / (1.0 + np.exp(-x)), "sigmoid")


def sigmoid_bwd(g, y):
    """tensor.py:231-232 ``g * y * (1.0 - y)``."""
    return g * y * (1.0 - y)


def tanh(x):
    return finalize(np.tanh(x), "tanh")


def relu(x):
    """tensor.py:207 ``np.maximum(x, 0.0)``."""
    return finalize(np.maximum(x, 0.0), "relu")


def relu_bwd(g, x):
    """tensor.py:235-236 ``g * (x > 0.0)`` -- gradient at 0 is 0."""
    return g * (x > 0.0)


def broadcast_kind(sa, sb):
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


def add(x, w):
    """tensor.py:246-247."""
    broadcast_kind(x.shape, w.shape)
    return finalize(x + w, "add")


def mul(x, w):
    """tensor.py:248-249."""
    broadcast_kind(x.shape, w.shape)
    return finalize(x * w, "mul")


def mul_bwd(g, x, w):
    """tensor.py:262-263 ``ga, gb = g * w, g * x`` (before _reduce_to)."""
    return g * w, g * x


# ----------------------------------------------------------------- matmul
def matmul(x, w):
    """tensor.py:306-312."""
    if x.ndim != 2 or w.ndim != 2:
        raise ShapeError(f"matmul needs 2-D operands, got {x.shape} x {w.shape}")
    if x.shape[1] != w.shape[0]:
        raise ShapeError(f"matmul inner extents differ: {x.shape} x {w.shape}")
    return finalize(x @ w, "matmul")


def matmul_bwd(g, x, w):
    """tensor.py:316-317 ``(g @ w.T, x.T @ g)``."""
    return g @ w.T, x.T @ g


# ----------------------------------------------------------------- structural
def take_rows(a, idx):
    """tensor.py:424-436 -- Scatter: ``y[k] = a[idx[k]]``."""
    indices = np.asarray(idx, dtype=np.int64)
    if indices.size and (indices.min() < 0 or indices.max() >= a.shape[0]):
        raise ShapeError("row index out of range")
    return finalize(a[indices], "take_rows")


def take_rows_bwd(g, idx, n_rows):
    """tensor.py:431-434 -- backward-Scatter: sequential ``np.add.at``."""
    out = np.zeros((n_rows,) + g.shape[1:], dtype=g.dtype)
    np.add.at(out, np.asarray(idx, dtype=np.int64), g)
    return out


def segment_sum(a, segment_ids, num_segments):
    """tensor.py:439-450 -- Gather(sum): rows added in row order."""
    seg = np.asarray(segment_ids, dtype=np.int64)
    if seg.shape[0] != a.shape[0]:
        raise ShapeError("segment id count does not match row count")
    out = np.zeros((num_segments,) + a.shape[1:], dtype=a.dtype)
    np.add.at(out, seg, a)
    return finalize(out, "segment_sum")


def segment_sum_bwd(g, segment_ids):
    """tensor.py:447-448 ``g[seg]``."""
    return g[np.asarray(segment_ids, dtype=np.int64)]


def segment_max(a, segment_ids, num_segments, empty_fill=0.0):
    """tensor.py:453-484 -- Gather(max) with argmax.

    Vectorised but equivalent to the reference loop (``tensor.py:465-469``):
    strict ``>`` from a -inf init means the LOWEST row index attaining the max
    wins; empty segments (argmax -1) are filled with ``empty_fill``.
    Returns ``(out, argmax)``; argmax is int64 [num_segments, F], -1 if empty.
    """
    seg = np.asarray(segment_ids, dtype=np.int64)
    if seg.shape[0] != a.shape[0]:
        raise ShapeError("segment id count does not match row count")
    out = np.full((num_segments,) + a.shape[1:], -np.inf, dtype=a.dtype)
    np.maximum.at(out, seg, a)
    rows = np.arange(a.shape[0], dtype=np.int64)
    cand = np.where(a == out[seg] if a.ndim == 1 else a == out[seg],
                    rows.reshape((-1,) + (1,) * (a.ndim - 1)),
                    np.iinfo(np.int64).max)
    arg = np.full((num_segments,) + a.shape[1:], np.iinfo(np.int64).max, dtype=np.int64)
    np.minimum.at(arg, seg, cand)
    # a row equal to -inf never wins against the -inf init (strict '>')
    arg[np.isneginf(out)] = -1
    arg[arg == np.iinfo(np.int64).max] = -1
    empty = arg[..., 0] < 0 if arg.ndim > 1 else arg < 0
    out[empty] = empty_fill
    return finalize(out, "segment_max"), arg


def segment_max_bwd(g, arg, n_rows):
    """tensor.py:473-482 -- route each output element to its argmax row."""
    gx = np.zeros((n_rows,) + g.shape[1:], dtype=g.dtype)
    valid = arg >= 0
    rows = arg[valid]
    if arg.ndim == 2:
        cols = np.nonzero(valid)[1]
        np.add.at(gx, (rows, cols), g[valid])
    else:
        np.add.at(gx, rows, g[valid])
    return gx


# ----------------------------------------------------------------- loss
def softmax_cross_entropy(z, labels):
    """tensor.py:487-506. Returns ``(loss_0d, p)``; loss keeps z's dtype."""
    lab = np.asarray(labels, dtype=np.int64)
    if z.ndim != 2 or lab.shape[0] != z.shape[0]:
        raise ShapeError("logits must be [n, classes] with one label per row")
    zmax = z.max(axis=1, keepdims=True)
    ez = np.exp(z - zmax)
    denom = ez.sum(axis=1, keepdims=True)
    p = ez / denom
    n = z.shape[0]
    logp = (z - zmax) - np.log(denom)
    loss = -logp[np.arange(n), lab].mean()
    return finalize(np.asarray(loss), "softmax_xent"), p


def softmax_cross_entropy_bwd(g, p, labels):
    """tensor.py:501-504 ``g * (p - onehot) / n``."""
    lab = np.asarray(labels, dtype=np.int64)
    n = p.shape[0]
    gz = p.copy()
    gz[np.arange(n), lab] -= 1.0
    return g * gz / n
