"""Graph-store restatement (test infrastructure only).

Follows the graph-store module of ``/root/reference/SPEC.md``:
``reencode_balance`` (heuristic :154) and ``partition_2d``
(invariants :150-152, layout :113-118), with the ambiguities
pinned as in SURVEY.md Appendix B.4-B.5.  The product's C++ partitioner
(``csrc/host_graph.cpp``) must reproduce these arrays byte for byte.
"""

import numpy as np


def degrees(src, dst, V):
    """(deg_out, deg_in) as int64 [V]."""
    dout = np.bincount(np.asarray(src, np.int64), minlength=V).astype(np.int64)
    din = np.bincount(np.asarray(dst, np.int64), minlength=V).astype(np.int64)
    return dout, din


def gcn_edge_weights(src, dst, V, dtype=np.float32):
    """w_e = 1/sqrt(deg_out(src) * deg_in(dst)), computed in fp64."""
    dout, din = degrees(src, dst, V)
    w = 1.0 / np.sqrt(dout[src].astype(np.float64) * din[dst].astype(np.float64))
    return w.astype(dtype)


def interval_layout(V, interval_size):
    """P = ceil(V / interval_size); all intervals equal except possibly the last."""
    if interval_size < 1:
        raise ValueError("interval_size must be >= 1")
    P = max(1, -(-V // interval_size))
    sizes = np.full(P, interval_size, dtype=np.int64)
    sizes[-1] = V - (P - 1) * interval_size
    return P, sizes


def max_chunk_edges(src, dst, V, interval_size):
    P, _ = interval_layout(V, interval_size)
    if len(src) == 0:
        return 0
    key = (np.asarray(src, np.int64) // interval_size) * P + np.asarray(dst, np.int64) // interval_size
    return int(np.bincount(key, minlength=P * P).max())


def reencode_balance(src, dst, V, num_intervals):
    """SPEC.md:130-138 with the SURVEY Appendix B.5 pins.

    degree = in + out; order = degree descending, ties by ascending id;
    round-robin over intervals skipping full ones (capacity interval_size, the
    last interval short); new ids in arrival order inside an interval; fall
    back to identity if the re-encoded max chunk edge count is worse.
    Returns ``perm`` with ``perm[old] = new`` (int64 [V]).
    """
    if num_intervals < 1:
        raise ValueError("num_intervals must be >= 1")
    size = max(1, -(-V // num_intervals))
    P, caps = interval_layout(V, size)
    dout, din = degrees(src, dst, V)
    deg = dout + din
    order = np.lexsort((np.arange(V), -deg))
    fill = np.zeros(P, dtype=np.int64)
    perm = np.empty(V, dtype=np.int64)
    cur = 0
    for v in order:
        while fill[cur] >= caps[cur]:
            cur = (cur + 1) % P
        perm[v] = cur * size + fill[cur]
        fill[cur] += 1
        cur = (cur + 1) % P
    src = np.asarray(src, np.int64)
    dst = np.asarray(dst, np.int64)
    if max_chunk_edges(perm[src], perm[dst], V, size) > max_chunk_edges(src, dst, V, size):
        return np.arange(V, dtype=np.int64)
    return perm


class Partition:
    """P x P grid of edge chunks C_ij (i = source interval, j = destination interval).

    Flattened, chunk id ``c = i * P + j``:

    * ``edge_off[c]:edge_off[c+1]`` -- the chunk's edges in ``csc_*`` / ``csr_*``;
    * ``csc_ptr[cptr_off[c] : cptr_off[c] + n_j + 1]`` -- chunk-local column
      pointers by local destination; ``csc_idx`` = local source id,
      ``csc_eid`` = input edge id.  Canonical: sorted by local source within a
      destination, multi-edges (same source) in input order.
    * ``csr_ptr[rptr_off[c] : rptr_off[c] + n_i + 1]`` -- chunk-local row
      pointers by local source; ``csr_idx`` = local destination id,
      ``csr_eid`` = input edge id.  Stable by CSC position within a source
      (so backward-Scatter visits edges in the forward edge-list order,
      tensor.py:431-434).
    """

    def __init__(self, V, interval_size, P, sizes, edge_off, cptr_off, rptr_off,
                 csc_ptr, csc_idx, csc_eid, csr_ptr, csr_idx, csr_eid):
        self.V, self.interval_size, self.P, self.sizes = V, interval_size, P, sizes
        self.edge_off, self.cptr_off, self.rptr_off = edge_off, cptr_off, rptr_off
        self.csc_ptr, self.csc_idx, self.csc_eid = csc_ptr, csc_idx, csc_eid
        self.csr_ptr, self.csr_idx, self.csr_eid = csr_ptr, csr_idx, csr_eid

    def begin(self, i):
        return i * self.interval_size

    def chunk(self, i, j):
        c = i * self.P + j
        e0, e1 = int(self.edge_off[c]), int(self.edge_off[c + 1])
        nj, ni = int(self.sizes[j]), int(self.sizes[i])
        cp = self.csc_ptr[self.cptr_off[c]: self.cptr_off[c] + nj + 1]
        rp = self.csr_ptr[self.rptr_off[c]: self.rptr_off[c] + ni + 1]
        return dict(i=i, j=j, nnz=e1 - e0,
                    csc_ptr=cp, csc_idx=self.csc_idx[e0:e1], csc_eid=self.csc_eid[e0:e1],
                    csr_ptr=rp, csr_idx=self.csr_idx[e0:e1], csr_eid=self.csr_eid[e0:e1])


def partition_2d(src, dst, V, interval_size):
    """P = ceil(V/interval_size), explicit empty chunks, CSC + CSR per chunk."""
    P, sizes = interval_layout(V, interval_size)
    src = np.asarray(src, np.int64)
    dst = np.asarray(dst, np.int64)
    E = src.shape[0]
    si, sj = src // interval_size, dst // interval_size
    ls, ld = src - si * interval_size, dst - sj * interval_size
    cid = si * P + sj
    # canonical CSC: by (chunk, local dst), then local src ("CSC sorted by local
    # dest id" with row indices sorted inside a column); multi-edges keep input order
    by_src = np.argsort(ls, kind="stable")
    csc_eid = by_src[np.argsort((cid * interval_size + ld)[by_src], kind="stable")].astype(np.int64)
    # CSR: stable by (chunk, local src) over the CSC order
    csr_perm = np.argsort((cid * interval_size + ls)[csc_eid], kind="stable")
    csr_eid = csc_eid[csr_perm]
    counts = np.bincount(cid, minlength=P * P) if E else np.zeros(P * P, np.int64)
    edge_off = np.zeros(P * P + 1, np.int64)
    edge_off[1:] = np.cumsum(counts)
    ccnt = np.bincount(cid * interval_size + ld, minlength=P * P * interval_size) if E \
        else np.zeros(P * P * interval_size, np.int64)
    rcnt = np.bincount(cid * interval_size + ls, minlength=P * P * interval_size) if E \
        else np.zeros(P * P * interval_size, np.int64)
    cptr, rptr = [], []
    cptr_off = np.zeros(P * P + 1, np.int64)
    rptr_off = np.zeros(P * P + 1, np.int64)
    for i in range(P):
        for j in range(P):
            c = i * P + j
            nj, ni = int(sizes[j]), int(sizes[i])
            cp = np.zeros(nj + 1, np.int64)
            cp[1:] = np.cumsum(ccnt[c * interval_size: c * interval_size + nj])
            rp = np.zeros(ni + 1, np.int64)
            rp[1:] = np.cumsum(rcnt[c * interval_size: c * interval_size + ni])
            cptr.append(cp)
            rptr.append(rp)
            cptr_off[c + 1] = cptr_off[c] + nj + 1
            rptr_off[c + 1] = rptr_off[c] + ni + 1
    return Partition(V, interval_size, P, sizes, edge_off, cptr_off, rptr_off,
                     np.concatenate(cptr), ls[csc_eid].astype(np.int32), csc_eid,
                     np.concatenate(rptr), ld[csr_eid].astype(np.int32), csr_eid)


def flatten_edges(part, src_global=True):
    """Reassemble all chunks into (src, dst) lists (SPEC.md:147,150 property)."""
    out_s, out_d = [], []
    for i in range(part.P):
        for j in range(part.P):
            ch = part.chunk(i, j)
            cp = ch["csc_ptr"]
            ld = np.repeat(np.arange(len(cp) - 1), np.diff(cp))
            out_s.append(ch["csc_idx"].astype(np.int64) + part.begin(i))
            out_d.append(ld + part.begin(j))
    return np.concatenate(out_s), np.concatenate(out_d)
