"""SAGA-NN layer oracle: GCN and G-GCN forward/backward (test infrastructure only).

Two restatements of the same math:

* ``ref_*`` -- the literal reference composition: the SAGA-NN stages written
  with the ``tensor.py`` primitives over the whole CSC-ordered edge list, in
  tape order (Scatter = take_rows tensor.py:424, ApplyEdge = mul/add/sigmoid
  tensor.py:204-303, Gather = segment_sum tensor.py:439, ApplyVertex =
  matmul + relu tensor.py:306/207, loss tensor.py:487, backward = the reverse
  sweep of tensor.py:91-121).  Checked bit-for-bit against golden fixtures
  produced by the real reference (tests/golden/make_golden.py).
* chunked -- the SPEC's engine semantics: Locality order over the 2D grid
  (for each destination interval j, all source intervals i in
  ascending order accumulate into A_j), per-destination accumulation in CSC
  order and large groups split into consecutive subgroups of
  ``T`` edges combined in fixed order.  With
  P = 1 and no split this is the reference composition exactly.
"""

import numpy as np

from . import primitives as prim


# ------------------------------------------------------------------ gather core
def seq_sum_rows(ptr, t, A=None, T=None, F=None, dtype=None):
    """Sum per-edge terms ``t`` (CSC/CSR order) into rows, deterministic order.

    Row u with ``n_u <= T`` edges continues the chain ``acc = A[u]; acc += t_e``
    in edge order; a row with ``n_u > T`` edges is split into consecutive
    subgroups of ``T`` edges, each summed from 0, and the partials are added
    onto ``A[u]`` in subgroup order.  ``T=None`` never splits.
    """
    ptr = np.asarray(ptr, np.int64)
    n = len(ptr) - 1
    if A is None:
        A = np.zeros((n, t.shape[1] if F is None else F), dtype=t.dtype if dtype is None else dtype)
    out = A.copy()
    nnz = int(ptr[-1])
    if nnz == 0:
        return out
    deg = np.diff(ptr)
    rows = np.repeat(np.arange(n, dtype=np.int64), deg)
    if T is None:
        np.add.at(out, rows, t)
        return out
    esplit = (deg > T)[rows]
    keep = ~esplit
    np.add.at(out, rows[keep], t[keep])
    if esplit.any():
        pos = np.arange(nnz, dtype=np.int64) - ptr[rows]
        r_s, sub = rows[esplit], pos[esplit] // T
        change = np.ones(r_s.shape[0], dtype=bool)
        change[1:] = (r_s[1:] != r_s[:-1]) | (sub[1:] != sub[:-1])
        gid = np.cumsum(change) - 1
        partial = np.zeros((int(gid[-1]) + 1, t.shape[1]), dtype=t.dtype)
        np.add.at(partial, gid, t[esplit])
        np.add.at(out, r_s[change], partial)
    return out


def local_rows(ptr):
    ptr = np.asarray(ptr, np.int64)
    return np.repeat(np.arange(len(ptr) - 1, dtype=np.int64), np.diff(ptr))


def _rows(part, X, k):
    b = part.begin(k)
    return X[b: b + int(part.sizes[k])]


# ------------------------------------------------------------------ GCN propagation
def gcn_propagate_fwd(part, H, w_edge, T=None):
    """fused_gather_chunk for GCN over all columns, Locality order.

    ``A[u] = sum_{e in in(u)} w_e * H[src_e]`` with ``t_e = H[src] * w_e``
    exactly as ``mul(take_rows(H, src), w)`` (tensor.py:249)."""
    A = np.zeros((part.V, H.shape[1]), dtype=H.dtype)
    for j in range(part.P):
        Aj = np.zeros((int(part.sizes[j]), H.shape[1]), dtype=H.dtype)
        for i in range(part.P):
            ch = part.chunk(i, j)
            if ch["nnz"] == 0:
                continue  # SPEC.md:427 empty chunk -> A_j unchanged
            t = _rows(part, H, i)[ch["csc_idx"]]
            if w_edge is not None:
                t = t * w_edge[ch["csc_eid"]][:, None]
            Aj = seq_sum_rows(ch["csc_ptr"], t, Aj, T)
        A[part.begin(j): part.begin(j) + int(part.sizes[j])] = Aj
    return A


def gcn_propagate_bwd(part, G, w_edge, T=None):
    """backward Gather+ApplyEdge+Scatter for GCN over the transposed (CSR) index.

    ``dH[v] = sum_{e in out(v)} G[dst_e] * w_e`` (tensor.py:447-448, :263, :431-434);
    per source interval i, destination intervals j ascending."""
    out = np.zeros((part.V, G.shape[1]), dtype=G.dtype)
    for i in range(part.P):
        Oi = np.zeros((int(part.sizes[i]), G.shape[1]), dtype=G.dtype)
        for j in range(part.P):
            ch = part.chunk(i, j)
            if ch["nnz"] == 0:
                continue
            t = _rows(part, G, j)[ch["csr_idx"]]
            if w_edge is not None:
                t = t * w_edge[ch["csr_eid"]][:, None]
            Oi = seq_sum_rows(ch["csr_ptr"], t, Oi, T)
        out[part.begin(i): part.begin(i) + int(part.sizes[i])] = Oi
    return out


# ------------------------------------------------------------------ G-GCN propagation
def ggcn_propagate_fwd(part, h, P_, Q_, T=None):
    """Fused gated gather (post-hoist G-GCN):
    ``A[u] = sum sigmoid(P[v] + Q[u]) * h[v]`` -- add(Ps, Qd) -> sigmoid -> mul(eta, hs)."""
    A = np.zeros((part.V, h.shape[1]), dtype=h.dtype)
    for j in range(part.P):
        Aj = np.zeros((int(part.sizes[j]), h.shape[1]), dtype=h.dtype)
        Qj = _rows(part, Q_, j)
        for i in range(part.P):
            ch = part.chunk(i, j)
            if ch["nnz"] == 0:
                continue
            src = ch["csc_idx"]
            u = local_rows(ch["csc_ptr"])
            eta = prim.sigmoid(_rows(part, P_, i)[src] + Qj[u])
            t = eta * _rows(part, h, i)[src]
            Aj = seq_sum_rows(ch["csc_ptr"], t, Aj, T)
        A[part.begin(j): part.begin(j) + int(part.sizes[j])] = Aj
    return A


def ggcn_propagate_bwd(part, h, P_, Q_, Ga, T=None):
    """G-GCN backward duals with eta recomputed.

    Pass A (CSC): dQ[u] = sum_in(u) t_e.  Pass B (CSR): dP[v] = sum_out(v) t_e and
    dh_take[v] = sum_out(v) Ga[u] * eta_e, where g_eta = Ga[u] * h[v] (mul bwd,
    tensor.py:263) and t_e = g_eta * eta * (1 - eta) (sigmoid bwd, tensor.py:232)."""
    F = h.shape[1]
    dQ = np.zeros((part.V, F), dtype=h.dtype)
    dP = np.zeros((part.V, F), dtype=h.dtype)
    dH = np.zeros((part.V, F), dtype=h.dtype)
    for j in range(part.P):  # pass A
        Gj, Qj = _rows(part, Ga, j), _rows(part, Q_, j)
        acc = np.zeros((int(part.sizes[j]), F), dtype=h.dtype)
        for i in range(part.P):
            ch = part.chunk(i, j)
            if ch["nnz"] == 0:
                continue
            v = ch["csc_idx"]
            u = local_rows(ch["csc_ptr"])
            eta = prim.sigmoid(_rows(part, P_, i)[v] + Qj[u])
            t = prim.sigmoid_bwd(Gj[u] * _rows(part, h, i)[v], eta)
            acc = seq_sum_rows(ch["csc_ptr"], t, acc, T)
        dQ[part.begin(j): part.begin(j) + int(part.sizes[j])] = acc
    for i in range(part.P):  # pass B
        Pi, hi = _rows(part, P_, i), _rows(part, h, i)
        accP = np.zeros((int(part.sizes[i]), F), dtype=h.dtype)
        accH = np.zeros((int(part.sizes[i]), F), dtype=h.dtype)
        for j in range(part.P):
            ch = part.chunk(i, j)
            if ch["nnz"] == 0:
                continue
            u = ch["csr_idx"]
            v = local_rows(ch["csr_ptr"])
            Gu = _rows(part, Ga, j)[u]
            eta = prim.sigmoid(Pi[v] + _rows(part, Q_, j)[u])
            t = prim.sigmoid_bwd(Gu * hi[v], eta)
            accP = seq_sum_rows(ch["csr_ptr"], t, accP, T)
            accH = seq_sum_rows(ch["csr_ptr"], Gu * eta, accH, T)
        dP[part.begin(i): part.begin(i) + int(part.sizes[i])] = accP
        dH[part.begin(i): part.begin(i) + int(part.sizes[i])] = accH
    return dQ, dP, dH


# ------------------------------------------------------------------ models (chunked)
def gcn_epoch(part, X, Ws, labels, w_edge, T=None, masks=None):
    """2-layer (or L-layer) GCN forward + backward.

    ``masks`` (optional, one bool array per layer): the ReLU-backward masks to use instead of
    z_l > 0 -- a run under test may resolve a ReLU kink (|z| at rounding level) the other way,
    and routing the oracle through the same masks compares everything else exactly (the way
    mpgcn_epoch(args=...) routes near-tie argmaxes).
    Returns dict(loss, a=[...], z=[...], out=[...], grads=[dW...])."""
    hs, As, Zs = [X], [], []
    for W in Ws:
        a = gcn_propagate_fwd(part, hs[-1], w_edge, T)
        z = prim.matmul(a, W)
        As.append(a)
        Zs.append(z)
        hs.append(prim.relu(z))
    loss, p = prim.softmax_cross_entropy(hs[-1], labels)
    g = prim.softmax_cross_entropy_bwd(np.asarray(1.0, dtype=X.dtype), p, labels)
    grads = [None] * len(Ws)
    for l in range(len(Ws) - 1, -1, -1):
        gz = prim.relu_bwd(g, Zs[l]) if masks is None else g * masks[l]
        ga, grads[l] = prim.matmul_bwd(gz, As[l], Ws[l])
        if l > 0:
            g = gcn_propagate_bwd(part, ga, w_edge, T)
    return dict(loss=loss, p=p, a=As, z=Zs, out=hs[1:], grads=grads)


def ggcn_epoch(part, X, layers, labels, T=None):
    """2-layer G-GCN, hoisted (P = h W_H, Q = h W_C), forward + backward.

    ``layers`` = [(W_H, W_C, W), ...]; grads returned in the same structure."""
    hs, cache = [X], []
    for (WH, WC, W) in layers:
        h = hs[-1]
        P_ = prim.matmul(h, WH)
        Q_ = prim.matmul(h, WC)
        a = ggcn_propagate_fwd(part, h, P_, Q_, T)
        z = prim.matmul(a, W)
        cache.append((h, P_, Q_, a, z))
        hs.append(prim.relu(z))
    loss, p = prim.softmax_cross_entropy(hs[-1], labels)
    g = prim.softmax_cross_entropy_bwd(np.asarray(1.0, dtype=X.dtype), p, labels)
    grads = [None] * len(layers)
    for l in range(len(layers) - 1, -1, -1):
        WH, WC, W = layers[l]
        h, P_, Q_, a, z = cache[l]
        gz = prim.relu_bwd(g, z)
        ga, gW = prim.matmul_bwd(gz, a, W)
        dQ, dP, dH = ggcn_propagate_bwd(part, h, P_, Q_, ga, T)
        gh_q, gWC = prim.matmul_bwd(dQ, h, WC)
        gh_p, gWH = prim.matmul_bwd(dP, h, WH)
        grads[l] = (gWH, gWC, gW)
        g = (dH + gh_q) + gh_p  # tape order: take_rows(h) part, then Q-, then P-matmul
    return dict(loss=loss, p=p, out=hs[1:], cache=cache, grads=grads)


def commnet_epoch(part, X, layers, labels, T=None):
    """2-layer CommNet: ApplyEdge = edge.src (passthrough), Gather(sum),
    ApplyVertex = ReLU(h W_H + accum W_C) (tensor.py:274 add of the two matmuls).
    ``layers`` = [(W_H, W_C), ...].  The gradient of h sums the direct (W_H) partial and
    the take_rows partial in the tape's reverse order (tensor.py:109-116)."""
    hs, cache = [X], []
    for (WH, WC) in layers:
        h = hs[-1]
        a = gcn_propagate_fwd(part, h, None, T)
        z = prim.add(prim.matmul(h, WH), prim.matmul(a, WC))
        cache.append((h, a, z))
        hs.append(prim.relu(z))
    loss, p = prim.softmax_cross_entropy(hs[-1], labels)
    g = prim.softmax_cross_entropy_bwd(np.asarray(1.0, dtype=X.dtype), p, labels)
    grads = [None] * len(layers)
    for l in range(len(layers) - 1, -1, -1):
        WH, WC = layers[l]
        h, a, z = cache[l]
        gz = prim.relu_bwd(g, z)
        ga, gWC = prim.matmul_bwd(gz, a, WC)
        gh, gWH = prim.matmul_bwd(gz, h, WH)
        grads[l] = (gWH, gWC)
        if l > 0:
            g = gh + gcn_propagate_bwd(part, ga, None, T)
    return dict(loss=loss, a=[c[1] for c in cache], z=[c[2] for c in cache], out=hs[1:],
                grads=grads)


def mpgcn_epoch(part, X, layers, labels, args=None):
    """2-layer MP-GCN, hoisted: Y = sigmoid(h W_pool + b) per vertex,
    Gather(max) over in-edges (segment_max, tensor.py:453-484, argmax = first CSC
    position), ApplyVertex ReLU(accum W).  ``layers`` = [(W_pool, b, W), ...].

    The edge list is the 2D grid flattened source-interval-major (chunk C_ij for i, then
    j, each in CSC order): per destination that is source interval ascending then
    in-chunk CSC order, per source destination interval ascending
    then CSR order -- the engine's chunk order in both directions.  Positions (argmax)
    index this list; with P = 1 it is the plain CSC edge list.

    ``args`` (optional, one [V, pool] CSC-position array per layer) pins the max
    selection: max is discontinuous at ties, so a checker comparing an fp32 run with
    this fp64 oracle routes both through the SAME argmax (after verifying separately
    that every disagreement is a near-tie)."""
    from .graph import flatten_edges

    src, dst = flatten_edges(part)
    V = part.V
    hs, cache = [X], []
    for (Wp, b, W) in layers:
        h = hs[-1]
        Y = prim.sigmoid(prim.add(prim.matmul(h, Wp), b))
        ys = prim.take_rows(Y, src)
        a, arg = prim.segment_max(ys, dst, V)
        if args is not None:
            arg = np.asarray(args[len(cache)], dtype=np.int64)
            cols = np.broadcast_to(np.arange(arg.shape[1]), arg.shape)
            a = np.where(arg >= 0, ys[np.maximum(arg, 0), cols] if len(src) else 0, 0).astype(Y.dtype)
        z = prim.matmul(a, W)
        cache.append((h, Y, a, arg, z))
        hs.append(prim.relu(z))
    loss, p = prim.softmax_cross_entropy(hs[-1], labels)
    g = prim.softmax_cross_entropy_bwd(np.asarray(1.0, dtype=X.dtype), p, labels)
    grads = [None] * len(layers)
    for l in range(len(layers) - 1, -1, -1):
        Wp, b, W = layers[l]
        h, Y, a, arg, z = cache[l]
        gz = prim.relu_bwd(g, z)
        ga, gW = prim.matmul_bwd(gz, a, W)
        gys = prim.segment_max_bwd(ga, arg, len(src))          # tensor.py:473-482
        gY = prim.take_rows_bwd(gys, src, V)                    # tensor.py:431-434
        gpre = prim.sigmoid_bwd(gY, Y)
        gb = gpre.sum(axis=0)                                   # _reduce_to b_lead (tensor.py:199)
        gh, gWp = prim.matmul_bwd(gpre, h, Wp)
        grads[l] = (gWp, gb, gW)
        g = gh
    return dict(loss=loss, out=hs[1:], cache=cache, grads=grads)


# ------------------------------------------------------------------ GG-NN
def typed_csc_rows(part, i, j, types_in, n_types):
    """Rows of the per-type table Y (viewed [V * n_types, F], row v * n_types + t) that the
    CSC edges of chunk C_ij gather: (begin_i + local src) * n_types + type."""
    ch = part.chunk(i, j)
    return (part.begin(i) + ch["csc_idx"].astype(np.int64)) * n_types + \
        np.asarray(types_in, np.int64)[ch["csc_eid"]]


def typed_csr(part, i, j, types_in, n_types):
    """Per-type CSR of chunk C_ij: rows keyed (local src) * n_types + type, each row's edges
    in CSR order (stable), i.e. the order take_rows' backward adds them (tensor.py:431-434).
    Returns (ptr [n_i * n_types + 1], local destination per edge)."""
    ch = part.chunk(i, j)
    n_i = int(part.sizes[i])
    src_local = local_rows(ch["csr_ptr"])
    key = src_local * n_types + np.asarray(types_in, np.int64)[ch["csr_eid"]]
    order = np.argsort(key, kind="stable")
    ptr = np.zeros(n_i * n_types + 1, np.int64)
    np.add.at(ptr, key + 1, 1)
    return np.cumsum(ptr), ch["csr_idx"].astype(np.int64)[order]


def ggnn_propagate_fwd(part, Yflat, types_in, n_types, T=None):
    """GG-NN Scatter + ApplyEdge + Gather after the per-type hoist:
    a[u] = sum_{e in in(u)} Y_{type_e}[src_e] with Y stacked per vertex ([V, n_types*F],
    row v holds Y_0[v] | Y_1[v] | ...), Locality order over the grid."""
    V, F = part.V, Yflat.shape[1] // n_types
    Yrows = Yflat.reshape(V * n_types, F)
    A = np.zeros((V, F), dtype=Yflat.dtype)
    for j in range(part.P):
        Aj = np.zeros((int(part.sizes[j]), F), dtype=Yflat.dtype)
        for i in range(part.P):
            ch = part.chunk(i, j)
            if ch["nnz"] == 0:
                continue
            Aj = seq_sum_rows(ch["csc_ptr"], Yrows[typed_csc_rows(part, i, j, types_in, n_types)], Aj, T)
        A[part.begin(j): part.begin(j) + int(part.sizes[j])] = Aj
    return A


def ggnn_propagate_bwd(part, Ga, types_in, n_types, T=None):
    """Backward of the typed gather: dY_t[v] = sum_{e in out(v), type_e = t} Ga[dst_e]
    (segment_sum bwd tensor.py:447-448, select_rows bwd :380-386, take_rows bwd :431-434),
    over the per-type CSR, destination intervals ascending.  Returns [V, n_types*F]."""
    V, F = part.V, Ga.shape[1]
    out = np.zeros((V * n_types, F), dtype=Ga.dtype)
    for i in range(part.P):
        n_i = int(part.sizes[i])
        acc = np.zeros((n_i * n_types, F), dtype=Ga.dtype)
        for j in range(part.P):
            if part.chunk(i, j)["nnz"] == 0:
                continue
            ptr, dst_local = typed_csr(part, i, j, types_in, n_types)
            Gj = Ga[part.begin(j): part.begin(j) + int(part.sizes[j])]
            acc = seq_sum_rows(ptr, Gj[dst_local], acc, T)
        b = part.begin(i) * n_types
        out[b: b + n_i * n_types] = acc
    return out.reshape(V, n_types * F)


def gru_fwd(a, h, Wz, Uz, Wr, Ur, Wh, Uh):
    """GRU(vertex, accum) in the Li et al. (GG-NN) form, no biases, with the
    reference's op order (tensor.py add / sigmoid / tanh / mul / sub):
    z = s(aWz + hUz); r = s(aWr + hUr); c = tanh(aWh + (r*h)Uh); h' = (1 - z)*h + z*c."""
    z = prim.sigmoid(prim.add(prim.matmul(a, Wz), prim.matmul(h, Uz)))
    r = prim.sigmoid(prim.add(prim.matmul(a, Wr), prim.matmul(h, Ur)))
    rh = prim.mul(r, h)
    c = prim.tanh(prim.add(prim.matmul(a, Wh), prim.matmul(rh, Uh)))
    omz = prim.finalize(np.ones_like(z) - z, "sub")
    hn = prim.add(prim.mul(omz, h), prim.mul(z, c))
    return hn, (z, r, rh, c, omz)


def gru_bwd(g, a, h, params, cache):
    """Reverse sweep of gru_fwd in tape order (tensor.py:106-117): returns (g_a, g_h,
    [gWz, gUz, gWr, gUr, gWh, gUh]); partials of h and a are summed in the order the tape
    visits their consumers."""
    Wz, Uz, Wr, Ur, Wh, Uh = params
    z, r, rh, c, omz = cache
    g_z = g * c                                   # mul(z, c)
    g_c = g * z
    g_omz = g * h                                 # mul(omz, h)
    g_h = g * omz
    g_z = g_z + (-g_omz)                          # sub(ones, z)
    g_cp = g_c * (1.0 - c * c)                    # tanh bwd (tensor.py:234)
    g_rh, gUh = prim.matmul_bwd(g_cp, rh, Uh)     # matmul(rh, Uh)
    g_r = g_rh * h                                # mul(r, h)
    g_h = g_h + g_rh * r
    g_a, gWh = prim.matmul_bwd(g_cp, a, Wh)       # matmul(a, Wh)
    g_rp = prim.sigmoid_bwd(g_r, r)
    gh_r, gUr = prim.matmul_bwd(g_rp, h, Ur)      # matmul(h, Ur)
    g_h = g_h + gh_r
    ga_r, gWr = prim.matmul_bwd(g_rp, a, Wr)      # matmul(a, Wr)
    g_a = g_a + ga_r
    g_zp = prim.sigmoid_bwd(g_z, z)
    gh_z, gUz = prim.matmul_bwd(g_zp, h, Uz)      # matmul(h, Uz)
    g_h = g_h + gh_z
    ga_z, gWz = prim.matmul_bwd(g_zp, a, Wz)      # matmul(a, Wz)
    g_a = g_a + ga_z
    return g_a, g_h, [gWz, gUz, gWr, gUr, gWh, gUh]


def ggnn_epoch(part, X, layers, Wo, types_in, labels, T=None):
    """GG-NN: per layer (As, Wz, Uz, Wr, Ur, Wh, Uh) with
    As the n_types edge-type matrices; Y_t = h A_t hoisted per vertex, typed Gather(sum),
    GRU ApplyVertex; readout logits = h_L Wo (no ReLU), softmax-CE.  ``types_in``: edge
    type per INPUT edge id.  Returns dict(loss, logits, a, out, grads) with grads per layer
    ([dA_t...], dWz, dUz, dWr, dUr, dWh, dUh) and grads_Wo."""
    nt = len(layers[0][0])
    hs, cache = [X], []
    for (As, *gp) in layers:
        h = hs[-1]
        Yflat = np.concatenate([prim.matmul(h, A) for A in As], axis=1)
        a = ggnn_propagate_fwd(part, Yflat, types_in, nt, T)
        hn, gc = gru_fwd(a, h, *gp)
        cache.append((h, a, gc))
        hs.append(hn)
    logits = prim.matmul(hs[-1], Wo)
    loss, p = prim.softmax_cross_entropy(logits, labels)
    g_logits = prim.softmax_cross_entropy_bwd(np.asarray(1.0, dtype=X.dtype), p, labels)
    g, gWo = prim.matmul_bwd(g_logits, hs[-1], Wo)
    grads = [None] * len(layers)
    for l in range(len(layers) - 1, -1, -1):
        As, *gp = layers[l]
        h, a, gc = cache[l]
        g_a, g_h, gps = gru_bwd(g, a, h, gp, gc)
        F = h.shape[1]
        dY = ggnn_propagate_bwd(part, g_a, types_in, nt, T)
        gAs = [None] * nt
        for t in range(nt - 1, -1, -1):            # matmul(h, A_t) visited last-first
            gh_t, gAs[t] = prim.matmul_bwd(dY[:, t * F:(t + 1) * F], h, As[t])
            g_h = g_h + gh_t
        grads[l] = (gAs, *gps)
        g = g_h
    return dict(loss=loss, logits=logits, a=[c[1] for c in cache], out=hs[1:], grads=grads,
                grads_Wo=gWo)


def sgd(params, grads, lr):
    """W <- W - lr * dW."""
    return [W - lr * g for W, g in zip(params, grads)]


# ------------------------------------------------------------------ literal reference composition
def ref_gcn_layer(h, W, src, dst, w_col, V):
    """GCN layer as PAPER.md:552-564 on the primitives; edges in CSC order."""
    es = prim.take_rows(h, src)              # Scatter
    acc = prim.mul(es, w_col)                # ApplyEdge: edge.src x edge.data
    accum = prim.segment_sum(acc, dst, V)    # Gather(sum)
    z = prim.matmul(accum, W)                # ApplyVertex
    return es, accum, z, prim.relu(z)


def ref_gcn_epoch(X, Ws, labels, src, dst, w, V):
    w_col = w.reshape(-1, 1)
    hs, cache = [X], []
    for W in Ws:
        es, a, z, out = ref_gcn_layer(hs[-1], W, src, dst, w_col, V)
        cache.append((a, z))
        hs.append(out)
    loss, p = prim.softmax_cross_entropy(hs[-1], labels)
    g = prim.softmax_cross_entropy_bwd(np.asarray(1.0, dtype=X.dtype), p, labels)
    grads = [None] * len(Ws)
    for l in range(len(Ws) - 1, -1, -1):
        a, z = cache[l]
        gz = prim.relu_bwd(g, z)
        ga, grads[l] = prim.matmul_bwd(gz, a, Ws[l])
        gacc = prim.segment_sum_bwd(ga, dst)
        ges = gacc * w_col                      # mul bwd, ga = g * w (tensor.py:263)
        g = prim.take_rows_bwd(ges, src, V)     # backward-Scatter (tensor.py:431-434)
    return dict(loss=loss, a=[c[0] for c in cache], z=[c[1] for c in cache],
                out=hs[1:], grads=grads)


def ref_ggcn_layer(h, WH, WC, W, src, dst, V, hoisted=True):
    """G-GCN layer per the listing PAPER.md:172-173 / SPEC.md:193 (W_H on src)."""
    if hoisted:
        P_ = prim.matmul(h, WH)
        Q_ = prim.matmul(h, WC)
        pre = prim.add(prim.take_rows(P_, src), prim.take_rows(Q_, dst))
    else:
        hs_ = prim.take_rows(h, src)
        hd_ = prim.take_rows(h, dst)
        pre = prim.add(prim.matmul(hs_, WH), prim.matmul(hd_, WC))
    eta = prim.sigmoid(pre)
    acc = prim.mul(eta, prim.take_rows(h, src))
    accum = prim.segment_sum(acc, dst, V)
    z = prim.matmul(accum, W)
    return accum, z, prim.relu(z)
