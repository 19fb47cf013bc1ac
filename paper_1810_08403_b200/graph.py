"""Graph store: synthetic graphs, reencode_balance, partition_2d and the device ChunkGrid.

Mirrors the graph-store module of the reference SPEC (``SPEC.md:96-165``):
``Graph`` (:101-106), ``VertexChunk``/``EdgeChunk`` (:107-118),
``reencode_balance`` (:130-138) and ``partition_2d`` (:139-147).  All index
construction runs in native C++ (libsagann ``sg_host_*``); the resulting CSC
(destination-sorted, forward) and CSR (source-sorted, the "transposed chunk
index" used by backward) layouts are uploaded once per graph into a
``ChunkGrid`` together with the per-pass work plans the propagation kernels
consume.
"""

import os

import numpy as np

from . import _lib
from ._lib import check, lib, nptr
from .errors import GraphFormatError, ShapeError

RMAT_ABC = (0.57, 0.19, 0.19)
DEFAULT_SPLIT_EDGES = 4096     # subgroup size T for heavy rows


def auto_split_edges(nnz, warps=148 * 24, items_per_warp=4):
    """Subgroup size T for a pass of ``nnz`` edges: the largest power of two in [256, 4096] that
    still gives every resident warp ~items_per_warp work items.  A split subgroup is one warp's
    sequential sum, so T edges are the pass's critical path: 4096 for a whole-graph pass (Reddit:
    114.6M edges), smaller for the small chunks of a sharded grid (8 GPUs: ~1.8M edges per chunk,
    where T = 4096 made each chunk pass wait ~1.5 ms on its last subgroup, tools/dist_proxy.py).
    T is part of the sum order: the oracle takes the same T."""
    t = 4096
    while t > 256 and nnz < t * warps * items_per_warp:
        t //= 2
    return t


def resolve_split_edges(split_edges, nnz):
    return auto_split_edges(nnz) if split_edges in (None, "auto") else int(split_edges)
HUB_MIN_COVER = 0.03           # use the hub-row cache when its rows cover >= 3% of a pass's edges


class Graph:
    """Edge list over vertices [0, V); self-loops and multi-edges kept (:124)."""

    def __init__(self, V, src, dst):
        src = np.ascontiguousarray(src, dtype=np.int32)
        dst = np.ascontiguousarray(dst, dtype=np.int32)
        if src.shape != dst.shape or src.ndim != 1:
            raise GraphFormatError("src and dst must be 1-D arrays of equal length")
        if V < 0 or V > np.iinfo(np.int32).max:
            raise GraphFormatError(f"vertex count {V} out of range")
        if src.size and (min(src.min(), dst.min()) < 0 or max(src.max(), dst.max()) >= V):
            raise GraphFormatError(f"edge endpoint out of range [0, {V})")
        self.V, self.src, self.dst = int(V), src, dst

    @property
    def E(self):
        return int(self.src.shape[0])

    def degrees(self):
        dout = np.empty(self.V, np.int64)
        din = np.empty(self.V, np.int64)
        check(lib.sg_host_degrees(nptr(self.src), nptr(self.dst), self.E, self.V, nptr(dout), nptr(din)))
        return dout, din

    def gcn_weights(self, eid=None, degrees=None):
        """w_e = 1/sqrt(deg_out(src) deg_in(dst)) in fp32, for edges ``eid``."""
        dout, din = degrees if degrees is not None else self.degrees()
        n = self.E if eid is None else eid.shape[0]
        w = np.empty(n, np.float32)
        check(lib.sg_host_gcn_weights(nptr(self.src), nptr(self.dst), nptr(dout), nptr(din),
                                      nptr(eid) if eid is not None else None, n, nptr(w)))
        return w

    def permute(self, perm):
        perm = np.asarray(perm, np.int64)
        return Graph(self.V, perm[self.src], perm[self.dst])


def rmat_graph(V, E, seed=0, abc=RMAT_ABC):
    """R-MAT(a, b, c, 1-a-b-c) graph, ids folded into [0, V)."""
    a, b, c = abc
    t1, t2 = a, a + b
    t3 = t2 + c
    src = np.empty(E, np.int32)
    dst = np.empty(E, np.int32)
    check(lib.sg_host_gen_rmat(V, E, seed, t1, t2, t3, 0, nptr(src), nptr(dst)))
    return Graph(V, src, dst)


def uniform_graph(V, E, seed=0):
    src = np.empty(E, np.int32)
    dst = np.empty(E, np.int32)
    check(lib.sg_host_gen_uniform(V, E, seed, 0, nptr(src), nptr(dst)))
    return Graph(V, src, dst)


def synthetic_features(V, F, seed=1, ld=None):
    """U[-1, 1) features, fp32 [V, ld] with zeroed padding columns."""
    ld = F if ld is None else ld
    x = np.zeros((V, ld), np.float32)
    check(lib.sg_host_gen_features(V, F, seed, 0, nptr(x), ld))
    return x


def reencode_balance(g, num_intervals):
    """SPEC.md:130-138.  Returns (re-encoded Graph, perm) with perm[old] = new."""
    perm = np.empty(g.V, np.int64)
    check(lib.sg_host_reencode_balance(nptr(g.src), nptr(g.dst), g.E, g.V, num_intervals, nptr(perm)))
    return g.permute(perm), perm


class Partition:
    """P x P grid of EdgeChunks; chunk id c = i * P + j.

    Same flattened layout as the oracle's ``Partition``: chunk-local CSC
    pointers by local destination (canonical: by local source, multi-edges in input
    order) and chunk-local CSR
    pointers by local source (stable by CSC position)."""

    def __init__(self, g, interval_size):
        if interval_size < 1:
            raise ShapeError("interval_size must be >= 1")
        P = np.zeros(1, np.int64)
        plen = np.zeros(1, np.int64)
        check(lib.sg_host_partition_layout(g.V, interval_size, nptr(P), nptr(plen)))
        P, plen = int(P[0]), int(plen[0])
        E = g.E
        self.V, self.E, self.P, self.interval_size = g.V, E, P, int(interval_size)
        self.sizes = np.full(P, interval_size, np.int64)
        self.sizes[-1] = g.V - (P - 1) * interval_size
        self.edge_off = np.zeros(P * P + 1, np.int64)
        self.cptr_off = np.zeros(P * P + 1, np.int64)
        self.rptr_off = np.zeros(P * P + 1, np.int64)
        self.csc_ptr = np.zeros(plen, np.int64)
        self.csr_ptr = np.zeros(plen, np.int64)
        self.csc_idx = np.empty(E, np.int32)
        self.csr_idx = np.empty(E, np.int32)
        self.csc_eid = np.empty(E, np.int64)
        self.csr_eid = np.empty(E, np.int64)
        check(lib.sg_host_partition_2d(
            nptr(g.src), nptr(g.dst), E, g.V, interval_size, nptr(self.edge_off),
            nptr(self.cptr_off), nptr(self.rptr_off), nptr(self.csc_ptr), nptr(self.csc_idx),
            nptr(self.csc_eid), nptr(self.csr_ptr), nptr(self.csr_idx), nptr(self.csr_eid)))

    def begin(self, i):
        return i * self.interval_size

    def chunk(self, i, j):
        c = i * self.P + j
        e0, e1 = int(self.edge_off[c]), int(self.edge_off[c + 1])
        nj, ni = int(self.sizes[j]), int(self.sizes[i])
        return dict(i=i, j=j, nnz=e1 - e0, e0=e0,
                    csc_ptr=self.csc_ptr[self.cptr_off[c]: self.cptr_off[c] + nj + 1],
                    csc_idx=self.csc_idx[e0:e1], csc_eid=self.csc_eid[e0:e1],
                    csr_ptr=self.csr_ptr[self.rptr_off[c]: self.rptr_off[c] + ni + 1],
                    csr_idx=self.csr_idx[e0:e1], csr_eid=self.csr_eid[e0:e1])


    # ---------------------------------------------------------------- on-disk cache
    _ARRAYS = ("sizes", "edge_off", "cptr_off", "rptr_off", "csc_ptr", "csr_ptr", "csc_idx", "csr_idx",
               "csc_eid", "csr_eid")

    def save(self, path):
        """Write the partition as a directory of .npy arrays (memory-mappable on load)."""
        import os

        os.makedirs(path, exist_ok=True)
        for k in self._ARRAYS:
            np.save(os.path.join(path, k + ".npy"), getattr(self, k))
        np.save(os.path.join(path, "meta.npy"),
                np.array([self.V, self.E, self.P, self.interval_size], np.int64))

    @classmethod
    def load(cls, path, mmap=True):
        import os

        self = cls.__new__(cls)
        V, E, P, isz = (int(x) for x in np.load(os.path.join(path, "meta.npy")))
        self.V, self.E, self.P, self.interval_size = V, E, P, isz
        for k in self._ARRAYS:
            setattr(self, k, np.load(os.path.join(path, k + ".npy"), mmap_mode="r" if mmap else None))
        return self


def graph_key(g, interval_size):
    """Content key of (graph, interval_size) for the partition cache (native 64-bit hash)."""
    h = lib.sg_host_hash64(nptr(g.src), g.src.nbytes, np.uint64(g.V).item())
    h = lib.sg_host_hash64(nptr(g.dst), g.dst.nbytes, h)
    return f"v{g.V}_e{g.E}_i{int(interval_size)}_{h:016x}"


def partition_2d(g, interval_size, cache_dir=None):
    """P = ceil(V / interval_size), explicit empty chunks.

    ``cache_dir``: reuse a partition saved there for the same edge list and interval
    size (content hash of src/dst), else build and save it ("partition
    cache")."""
    if cache_dir is None:
        return Partition(g, interval_size)
    import os

    path = os.path.join(cache_dir, "partition_" + graph_key(g, interval_size))
    if os.path.exists(os.path.join(path, "meta.npy")):
        part = Partition.load(path)
        part.cache_hit = True
        return part
    part = Partition(g, interval_size)
    tmp = path + f".tmp{os.getpid()}"
    part.save(tmp)
    if not os.path.exists(path):
        os.replace(tmp, path)  # atomic publish; a concurrent writer's copy is equivalent
    part.cache_hit = False
    return part


# ------------------------------------------------------------------ ingestion
def _path(p):
    return str(p).encode()


def read_features(path, fmt="auto"):
    """Feature file: text CSV (row v = features of vertex v) or raw binary
    (u64 rows, u64 cols, row-major f64).  ``fmt`` = 'csv' | 'bin' | 'auto' (by content)."""
    if fmt == "auto":
        fmt = "csv"
        try:
            r = np.zeros(1, np.int64)
            c = np.zeros(1, np.int64)
            if lib.sg_host_read_matrix_bin_header(_path(path), nptr(r), nptr(c)) == _lib.SG_OK:
                fmt = "bin"
        except Exception:  # noqa: BLE001
            fmt = "csv"
    r = np.zeros(1, np.int64)
    c = np.zeros(1, np.int64)
    if fmt == "bin":
        check(lib.sg_host_read_matrix_bin_header(_path(path), nptr(r), nptr(c)))
        out = np.empty((int(r[0]), int(c[0])), np.float64)
        check(lib.sg_host_read_matrix_bin(_path(path), int(r[0]), int(c[0]), nptr(out)))
        return out
    if fmt != "csv":
        raise GraphFormatError(f"unknown feature format '{fmt}' (csv | bin | auto)")
    check(lib.sg_host_scan_matrix_text(_path(path), nptr(r), nptr(c)))
    out = np.empty((int(r[0]), int(c[0])), np.float64)
    check(lib.sg_host_read_matrix_text(_path(path), int(r[0]), int(c[0]), nptr(out)))
    return out


def write_features_bin(path, X):
    X = np.ascontiguousarray(X, np.float64)
    if X.ndim != 2:
        raise ShapeError("features must be a 2-D matrix")
    check(lib.sg_host_write_matrix_bin(_path(path), X.shape[0], X.shape[1], nptr(X)))


def read_labels(path):
    n = np.zeros(1, np.int64)
    check(lib.sg_host_scan_labels(_path(path), nptr(n)))
    out = np.empty(int(n[0]), np.int64)
    check(lib.sg_host_read_labels(_path(path), int(n[0]), nptr(out)))
    return out


def load_graph(edge_file, feature_file=None, label_file=None, *, num_vertices=None,
               feature_format="auto"):
    """load_graph: edge list + optional features / labels.

    V = ``num_vertices`` if given, else the feature row count, else max id + 1.  Ids are
    bounds-checked against V with the offending line named; self-loops and multi-edges
    are kept as given.  Returns a Graph with ``features`` (f64 [V, F] or None),
    ``labels`` (int64 [V] or None) and ``edge_values`` (f64 [E] or None) attached."""
    X = read_features(feature_file, feature_format) if feature_file is not None else None
    if num_vertices is not None:
        V = int(num_vertices)
        if X is not None and X.shape[0] != V:
            raise GraphFormatError(f"feature file has {X.shape[0]} rows, expected {V} vertices")
    elif X is not None:
        V = X.shape[0]
    else:
        V = -1
    E = np.zeros(1, np.int64)
    mx = np.zeros(1, np.int64)
    hv = np.zeros(1, np.int32)
    check(lib.sg_host_scan_edges(_path(edge_file), V, nptr(E), nptr(mx), nptr(hv)))
    E = int(E[0])
    if V < 0:
        V = int(mx[0]) + 1
    src = np.empty(E, np.int32)
    dst = np.empty(E, np.int32)
    val = np.empty(E, np.float64) if hv[0] else None
    check(lib.sg_host_read_edges(_path(edge_file), E, nptr(src), nptr(dst), nptr(val)))
    g = Graph(V, src, dst)
    g.features, g.edge_values = X, val
    g.labels = None
    if label_file is not None:
        y = read_labels(label_file)
        if y.shape[0] != V:
            raise GraphFormatError(f"label file has {y.shape[0]} rows, expected {V} vertices")
        g.labels = y
    return g


# split subgroups ordered by their first source (sg_host_plan_order): SG_PLAN_ORDER=row keeps
# the (row, subgroup) order for A/B runs
PLAN_ORDER = os.environ.get("SG_PLAN_ORDER", "src")


def plan(ptr, split_edges=DEFAULT_SPLIT_EDGES, pack_edges=None, max_rows=256, idx=None):
    """Work plan of one propagation pass over a CSC/CSR pointer array (native); with the pass's
    index ``idx``, split subgroups are queued by first source (sg_host_plan_order)."""
    ptr = np.ascontiguousarray(ptr, np.int64)
    n_rows = ptr.shape[0] - 1
    nnz = int(ptr[-1]) if n_rows >= 0 else 0
    if pack_edges is None:
        pack_edges = int(min(max(32, nnz // (148 * 64)), split_edges))
    cnt = np.zeros(3, np.int64)
    check(lib.sg_host_plan(nptr(ptr), n_rows, pack_edges, max_rows, split_edges, None, None,
                           nptr(cnt[0:1]), nptr(cnt[1:2]), nptr(cnt[2:3])))
    items = np.zeros(int(cnt[0]), _lib.ITEM_DTYPE)
    splits = np.zeros(max(int(cnt[1]), 1), _lib.SPLIT_DTYPE)
    check(lib.sg_host_plan(nptr(ptr), n_rows, pack_edges, max_rows, split_edges, nptr(items),
                           nptr(splits), nptr(cnt[0:1]), nptr(cnt[1:2]), nptr(cnt[2:3])))
    if idx is not None and PLAN_ORDER == "src" and len(items):
        check(lib.sg_host_plan_order(nptr(items), len(items), nptr(np.ascontiguousarray(idx, np.int32))))
    return items, splits[: int(cnt[1])], int(cnt[2])


# source-staged sum passes (sg_propagate_staged, bitwise identical to sg_propagate) for fp32 rows
# of 64..640 columns: opt-in (SG_STAGED=1).  It halves the L2 -> SM row traffic of the Reddit
# layer-1 pass (103 vs 190 GB) but measured 3-4x slower than the row-per-warp kernel in every
# variant tried (profiles/r02_staged_ab.txt), so the row kernel stays the default.
STAGED = os.environ.get("SG_STAGED", "0") == "1"
STAGE_MIN_F, STAGE_MAX_F = 64, 640
STAGES = int(os.environ.get("SG_STAGES", "3"))
_STAGE_SMEM = 227 * 1024


class StagePlan:
    """sg_host_stage_plan of one pass for rows of F columns: pieces (rows / T-edge subgroups)
    grouped by first source, each group's merged source list cut into shared-memory batches,
    every piece's edges as run entries (slot in batch, run length, weight)."""

    def __init__(self, ptr, idx, w, split_edges, F, device):
        import torch

        G = int(lib.sg_stage_group_pieces(F))
        if G <= 0:
            raise ShapeError(f"no staged gather for F = {F}")
        emax = 1024
        row_bytes = (F + 3) // 4 * 16
        pofs = (G + 1 + 7) // 8 * 8 * 2
        nst = STAGES
        stage = (_STAGE_SMEM - 256) // nst // 128 * 128
        S = int(min(256, (stage - emax * 8 - pofs) // row_bytes))   # <= 4 producer warps x 64 rows
        ptr = np.ascontiguousarray(ptr, np.int64)
        idx = np.ascontiguousarray(idx, np.int32)
        w = None if w is None else np.ascontiguousarray(w, np.float32)
        n_rows = ptr.shape[0] - 1
        sz = np.zeros(6, np.int64)
        args = (nptr(ptr), nptr(idx), nptr(w), n_rows, int(split_edges), G, S, emax)
        check(lib.sg_host_stage_plan(*args, None, None, None, None, None, None, None, nptr(sz)))
        ng, nb, ns, ne = (int(x) for x in sz[:4])
        pieces = np.zeros((max(ng, 1) * G, 4), np.int32)
        gb = np.zeros(ng + 1, np.int32)
        bso = np.zeros(nb + 1, np.int64)
        bs = np.zeros(max(ns, 1), np.int32)
        beo = np.zeros(nb + 1, np.int64)
        ent = np.zeros(max(ne, 2), np.uint64)
        pst = (G + 1 + 7) // 8 * 8
        pofs_a = np.zeros(max(nb, 1) * pst, np.uint16)
        check(lib.sg_host_stage_plan(*args, nptr(pieces), nptr(gb), nptr(bso), nptr(bs), nptr(beo),
                                     nptr(ent), nptr(pofs_a), nptr(sz)))
        self.G, self.S, self.EMAX, self.F, self.stages = G, S, emax, F, nst
        self.n_groups, self.n_batches, self.n_src, self.n_ent = ng, nb, ns, ne
        self.n_splits, self.n_slots = int(sz[4]), int(sz[5])
        t = lambda a: torch.from_numpy(a).to(device)  # noqa: E731
        self.pieces, self.group_batch, self.batch_src_off = t(pieces), t(gb), t(bso)
        self.batch_src, self.batch_ent_off = t(bs), t(beo)
        self.entries = t(ent.view(np.int64))
        self.batch_pofs = t(pofs_a.view(np.int16))


class PassIndex:
    """Device-resident index of one propagation pass over one chunk (CSC or CSR)."""

    def __init__(self, ptr, idx, w, n_rows, split_edges, device):
        import torch

        split_edges = resolve_split_edges(split_edges, int(ptr[-1]))
        self.split_edges = split_edges
        items, splits, n_slots = plan(ptr, split_edges, idx=idx)
        self.n_rows = int(n_rows)
        self.nnz = int(ptr[-1])
        self.n_items, self.n_splits, self.n_slots = len(items), len(splits), n_slots
        self.ptr = torch.from_numpy(np.ascontiguousarray(ptr, np.int64)).to(device)
        self.idx = torch.from_numpy(np.ascontiguousarray(idx, np.int32)).to(device)
        self.w = None if w is None else torch.from_numpy(np.ascontiguousarray(w, np.float32)).to(device)
        self.items = torch.from_numpy(items.view(np.uint8)).to(device)
        self.splits = torch.from_numpy(splits.view(np.uint8)).to(device) if len(splits) else None
        self.max_degree = int(np.diff(ptr).max()) if n_rows > 0 else 0
        # host arrays kept (views of the partition) for the staged-gather plans, built lazily
        self._host = (ptr, idx, w)
        self._stage = {}

    @classmethod
    def from_device(cls, ptr, idx, split_edges=DEFAULT_SPLIT_EDGES):
        """Index over device (ptr int64, idx int32) tensors; only the plan is built on the host."""
        import torch

        self = cls.__new__(cls)
        ptr_h = ptr.cpu().numpy()
        items, splits, n_slots = plan(ptr_h, split_edges)
        self.n_rows = ptr_h.shape[0] - 1
        self.nnz = int(ptr_h[-1])
        self.n_items, self.n_splits, self.n_slots = len(items), len(splits), n_slots
        self.ptr, self.idx, self.w = ptr, idx, None
        self.items = torch.from_numpy(items.view(np.uint8)).to(ptr.device)
        self.splits = torch.from_numpy(splits.view(np.uint8)).to(ptr.device) if len(splits) else None
        self.max_degree = int(np.diff(ptr_h).max()) if self.n_rows > 0 else 0
        return self

    def workspace_bytes(self, F, mode):
        return int(lib.sg_propagate_workspace_bytes(self.n_items, self.n_splits, self.n_slots, F, mode))

    def stage_plan(self, F):
        """The staged-gather plan of this pass for rows of F columns (None if not applicable)."""
        host = getattr(self, "_host", None)
        if host is None or self.nnz == 0 or not (STAGE_MIN_F <= F <= STAGE_MAX_F):
            return None
        G = int(lib.sg_stage_group_pieces(F))
        key = (G, (F + 3) // 4)
        if key not in self._stage:
            try:
                self._stage[key] = StagePlan(host[0], host[1], host[2], self.split_edges, F,
                                             self.ptr.device)
            except Exception:   # e.g. a row not sorted by source: the row-per-warp kernel runs
                self._stage[key] = None
        return self._stage[key]

    def hub(self, n_cap, min_cover=HUB_MIN_COVER):
        """Hub-row cache of this pass for at most ``n_cap`` rows (sg_propagate_hub).

        The most referenced gathered rows (count >= 2; descending count, ties by row id)
        get slots 0..n-1; returns (encoded idx, hub rows, n, edge coverage) with each edge
        to slot k carrying k | 0x80000000, or None when the hubs would cover fewer than
        ``min_cover`` of the edges (e.g. uniform graphs).  Built on the device, cached."""
        import torch

        if not hasattr(self, "_hubs"):
            self._hubs = {}
        if n_cap in self._hubs:
            return self._hubs[n_cap]
        res = None
        if self.nnz > 0 and n_cap > 0:
            idx = self.idx.long()
            counts = torch.bincount(idx)
            vals, order = torch.sort(counts, descending=True, stable=True)
            n = min(int(n_cap), int((vals >= 2).sum().item()))
            cover = float(vals[:n].sum().item()) / self.nnz if n else 0.0
            if n > 0 and cover >= min_cover:
                rows = order[:n]
                slot = torch.full((counts.numel(),), -1, dtype=torch.int64, device=idx.device)
                slot[rows] = torch.arange(n, device=idx.device)
                s = slot[idx]
                enc = torch.where(s >= 0, s - (1 << 31), idx).to(torch.int32)
                res = (enc, rows.to(torch.int32).contiguous(), n, cover)
                del s, slot
            del idx, counts
        self._hubs[n_cap] = res
        return res


class ChunkGrid:
    """Device chunk grid: per non-empty chunk C_ij a CSC pass index (forward,
    SPEC.md:142 "CSC sorted by local dest id") and a CSR pass index (backward),
    each with its static GCN edge weights in that edge order."""

    def __init__(self, g, interval_size=None, device="cuda", split_edges=DEFAULT_SPLIT_EDGES,
                 gcn_weights=True, partition=None):
        self.graph = g
        self.part = partition if partition is not None else partition_2d(g, interval_size or max(g.V, 1))
        self.V, self.E, self.P = g.V, g.E, self.part.P
        self.split_edges = split_edges
        self.device = device
        degs = g.degrees() if gcn_weights else None
        self.csc, self.csr = {}, {}
        # offset of each chunk's edges in the source-interval-major flattening (global
        # edge positions, e.g. the max-gather argmax)
        self.edge_base = {}
        total = 0
        for i in range(self.P):
            for j in range(self.P):
                ch = self.part.chunk(i, j)
                self.edge_base[(i, j)] = total
                total += int(ch["nnz"])
                if ch["nnz"] == 0:
                    continue
                wc = g.gcn_weights(ch["csc_eid"], degs) if gcn_weights else None
                wr = g.gcn_weights(ch["csr_eid"], degs) if gcn_weights else None
                self.csc[(i, j)] = PassIndex(ch["csc_ptr"], ch["csc_idx"], wc, self.part.sizes[j],
                                             split_edges, device)
                self.csr[(i, j)] = PassIndex(ch["csr_ptr"], ch["csr_idx"], wr, self.part.sizes[i],
                                             split_edges, device)

    def begin(self, k):
        return self.part.begin(k)

    def size(self, k):
        return int(self.part.sizes[k])

    def csr_positions(self, i, j):
        """CSC position of every CSR edge of chunk C_ij (int32, device), for routing max
        gradients to the argmax edge.  The CSR order is a stable sort of the CSC order by
        local source, so this is argsort(csc_idx, stable)."""
        if not hasattr(self, "_csr_pos"):
            self._csr_pos = {}
        if (i, j) not in self._csr_pos:
            import torch

            ch = self.part.chunk(i, j)
            pos = np.argsort(ch["csc_idx"], kind="stable").astype(np.int32)
            self._csr_pos[(i, j)] = torch.from_numpy(pos).to(self.device)
        return self._csr_pos[(i, j)]

    def workspace_bytes(self, F, mode):
        m = 0
        for d in (self.csc, self.csr):
            for pi in d.values():
                m = max(m, pi.workspace_bytes(F, mode))
        return max(m, 256)
