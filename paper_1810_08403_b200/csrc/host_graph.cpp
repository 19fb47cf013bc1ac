// Host-side graph store: synthetic generators, degrees, reencode_balance,
// partition_2d and propagation work plans.  Native C++ (OpenMP), no GPU needed.
//
// Semantics follow /root/reference/SPEC.md graph-store (:96-165) with the pins
// of SURVEY.md Appendix B.5 and a canonical CSC (ties within a destination by local source,
// multi-edges in input order); the generator is the counter-based splitmix64
// scheme restated in oracle/rng.py.  tests/test_host_graph.py checks every
// output array byte for byte against the oracle.
#include <omp.h>

#include <algorithm>
#include <cstring>
#include <cmath>
#include <numeric>
#include <vector>

#include "common.h"

namespace {

inline uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
inline uint64_t stream_key(uint64_t seed, uint64_t stream) { return splitmix64(seed * 256ull + stream); }
inline double u53(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }

constexpr uint64_t kStreamUniform = 1, kStreamFeature = 2, kStreamRmat = 3;

int rmat_scale(int64_t V) {
  int s = 0;
  while ((int64_t(1) << s) < V) ++s;
  return s < 1 ? 1 : s;
}

int max_threads() { return std::max(1, omp_get_max_threads()); }

// Stable counting sort of positions [0, n) (in the order given by `in`, or
// identity when null) by key(pos) in [0, n_keys): writes out[] and ptr[n_keys+1].
template <class KeyFn>
void stable_counting_sort(const int64_t* in, int64_t n, int64_t n_keys, KeyFn key, int64_t* out,
                          int64_t* ptr) {
  int T = max_threads();
  // bound the per-thread histogram footprint
  while (T > 1 && (int64_t)T * (n_keys + 1) > (int64_t(1) << 26)) --T;
  if (n < (int64_t(1) << 16)) T = 1;
  std::vector<int64_t> hist((size_t)T * (size_t)(n_keys + 1), 0);
#pragma omp parallel num_threads(T)
  {
    int t = omp_get_thread_num();
    int64_t b = n * t / T, e = n * (t + 1) / T;
    int64_t* h = hist.data() + (size_t)t * (n_keys + 1);
    for (int64_t p = b; p < e; ++p) h[key(in ? in[p] : p)]++;
  }
  // ptr[k] = sum over all threads of counts of keys < k; per-thread offsets
  int64_t run = 0;
  for (int64_t k = 0; k < n_keys; ++k) {
    ptr[k] = run;
    for (int t = 0; t < T; ++t) {
      int64_t c = hist[(size_t)t * (n_keys + 1) + k];
      hist[(size_t)t * (n_keys + 1) + k] = run;
      run += c;
    }
  }
  ptr[n_keys] = run;
#pragma omp parallel num_threads(T)
  {
    int t = omp_get_thread_num();
    int64_t b = n * t / T, e = n * (t + 1) / T;
    int64_t* h = hist.data() + (size_t)t * (n_keys + 1);
    for (int64_t p = b; p < e; ++p) {
      int64_t v = in ? in[p] : p;
      out[h[key(v)]++] = v;
    }
  }
}

int64_t max_chunk_edges(const int32_t* src, const int32_t* dst, const int64_t* perm, int64_t E,
                        int64_t V, int64_t size) {
  int64_t P = std::max<int64_t>(1, (V + size - 1) / size);
  std::vector<int64_t> cnt((size_t)(P * P), 0);
  for (int64_t e = 0; e < E; ++e) {
    int64_t s = perm ? perm[src[e]] : src[e];
    int64_t d = perm ? perm[dst[e]] : dst[e];
    cnt[(size_t)((s / size) * P + d / size)]++;
  }
  return E ? *std::max_element(cnt.begin(), cnt.end()) : 0;
}

}  // namespace

extern "C" {

int sg_host_gen_rmat(int64_t V, int64_t E, uint64_t seed, double t1, double t2, double t3,
                     int64_t edge_begin, int32_t* src, int32_t* dst) {
  SG_REQUIRE(V >= 1 && V <= INT32_MAX && E >= 0, SG_EINVAL, "gen_rmat: bad V=%lld E=%lld",
             (long long)V, (long long)E);
  const int s = rmat_scale(V);
  const uint64_t key = stream_key(seed, kStreamRmat);
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < E; ++k) {
    uint64_t sv = 0, dv = 0;
    const uint64_t base = key + (uint64_t)(edge_begin + k) * (uint64_t)s;
    for (int l = 0; l < s; ++l) {
      double u = u53(splitmix64(base + (uint64_t)l));
      uint64_t sb = u >= t2;
      uint64_t db = (u >= t1 && u < t2) || u >= t3;
      sv = (sv << 1) | sb;
      dv = (dv << 1) | db;
    }
    src[k] = (int32_t)(sv % (uint64_t)V);
    dst[k] = (int32_t)(dv % (uint64_t)V);
  }
  return SG_OK;
}

int sg_host_gen_uniform(int64_t V, int64_t E, uint64_t seed, int64_t edge_begin, int32_t* src,
                        int32_t* dst) {
  SG_REQUIRE(V >= 1 && V <= INT32_MAX && E >= 0, SG_EINVAL, "gen_uniform: bad V/E");
  const uint64_t key = stream_key(seed, kStreamUniform);
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < E; ++k) {
    uint64_t i = (uint64_t)(edge_begin + k) * 2ull;
    src[k] = (int32_t)(splitmix64(key + i) % (uint64_t)V);
    dst[k] = (int32_t)(splitmix64(key + i + 1ull) % (uint64_t)V);
  }
  return SG_OK;
}

int sg_host_gen_features(int64_t V, int64_t F, uint64_t seed, int64_t row_begin, float* x,
                         int64_t ldx) {
  SG_REQUIRE(V >= 0 && F >= 0 && ldx >= F, SG_EINVAL, "gen_features: bad shape");
  const uint64_t key = stream_key(seed, kStreamFeature);
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < V; ++v) {
    for (int64_t f = 0; f < F; ++f) {
      uint64_t h = splitmix64(key + (uint64_t)(row_begin + v) * (uint64_t)F + (uint64_t)f);
      float k = (float)(h >> 40);
      volatile float p = k * (float)(1.0 / 8388608.0);  // exact; no contraction
      x[v * ldx + f] = p - 1.0f;
    }
  }
  return SG_OK;
}

int sg_host_degrees(const int32_t* src, const int32_t* dst, int64_t E, int64_t V, int64_t* dout,
                    int64_t* din) {
  std::fill(dout, dout + V, 0);
  std::fill(din, din + V, 0);
  for (int64_t e = 0; e < E; ++e) {
    SG_REQUIRE(src[e] >= 0 && src[e] < V && dst[e] >= 0 && dst[e] < V, SG_ESHAPE,
               "edge %lld endpoint out of range [0,%lld)", (long long)e, (long long)V);
  }
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < E; ++e) {
    __atomic_fetch_add(&dout[src[e]], 1, __ATOMIC_RELAXED);
    __atomic_fetch_add(&din[dst[e]], 1, __ATOMIC_RELAXED);
  }
  return SG_OK;
}

int sg_host_reencode_balance(const int32_t* src, const int32_t* dst, int64_t E, int64_t V,
                             int64_t num_intervals, int64_t* perm) {
  SG_REQUIRE(num_intervals >= 1, SG_EINVAL, "num_intervals must be >= 1");
  const int64_t size = std::max<int64_t>(1, (V + num_intervals - 1) / num_intervals);
  const int64_t P = std::max<int64_t>(1, (V + size - 1) / size);
  std::vector<int64_t> dout(V), din(V);
  int rc = sg_host_degrees(src, dst, E, V, dout.data(), din.data());
  if (rc) return rc;
  std::vector<int64_t> order(V);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    return dout[a] + din[a] > dout[b] + din[b];  // degree desc; ties keep ascending id
  });
  std::vector<int64_t> fill(P, 0), cap(P, size);
  cap[P - 1] = V - (P - 1) * size;
  int64_t cur = 0;
  for (int64_t v : order) {
    while (fill[cur] >= cap[cur]) cur = (cur + 1) % P;
    perm[v] = cur * size + fill[cur];
    fill[cur]++;
    cur = (cur + 1) % P;
  }
  if (max_chunk_edges(src, dst, perm, E, V, size) > max_chunk_edges(src, dst, nullptr, E, V, size))
    std::iota(perm, perm + V, 0);
  return SG_OK;
}

int sg_host_partition_layout(int64_t V, int64_t interval_size, int64_t* P, int64_t* ptr_len) {
  SG_REQUIRE(interval_size >= 1 && V >= 0, SG_EINVAL, "interval_size must be >= 1");
  int64_t p = std::max<int64_t>(1, (V + interval_size - 1) / interval_size);
  *P = p;
  *ptr_len = p * (V + p);
  return SG_OK;
}

int sg_host_partition_2d(const int32_t* src, const int32_t* dst, int64_t E, int64_t V,
                         int64_t size, int64_t* edge_off, int64_t* cptr_off, int64_t* rptr_off,
                         int64_t* csc_ptr, int32_t* csc_idx, int64_t* csc_eid, int64_t* csr_ptr,
                         int32_t* csr_idx, int64_t* csr_eid) {
  int64_t P, plen;
  int rc = sg_host_partition_layout(V, size, &P, &plen);
  if (rc) return rc;
  for (int64_t e = 0; e < E; ++e)
    SG_REQUIRE(src[e] >= 0 && src[e] < V && dst[e] >= 0 && dst[e] < V, SG_ESHAPE,
               "edge %lld endpoint out of range [0,%lld)", (long long)e, (long long)V);
  auto nsz = [&](int64_t k) { return k == P - 1 ? V - (P - 1) * size : size; };
  // 1) stable bucket by chunk id (input order inside a chunk)
  std::vector<int64_t> by_chunk((size_t)E);
  auto cid = [&](int64_t e) { return (int64_t)(src[e] / size) * P + dst[e] / size; };
  stable_counting_sort(nullptr, E, P * P, cid, by_chunk.data(), edge_off);
  // pointer-array offsets (chunk c = i*P + j has n_j + 1 CSC and n_i + 1 CSR entries)
  cptr_off[0] = rptr_off[0] = 0;
  for (int64_t c = 0; c < P * P; ++c) {
    cptr_off[c + 1] = cptr_off[c] + nsz(c % P) + 1;
    rptr_off[c + 1] = rptr_off[c] + nsz(c / P) + 1;
  }
  // 2) per chunk: canonical CSC -- by local dst, then local src ("CSC sorted by
  //    local dest id"; row indices sorted within a column as in a canonical sparse matrix,
  //    multi-edges in input order) as two stable counting sorts (src, then dst); then CSR by
  //    local src over the CSC order (so by dst within a source row)
  for (int64_t c = 0; c < P * P; ++c) {
    const int64_t i = c / P, j = c % P, e0 = edge_off[c], e1 = edge_off[c + 1], n = e1 - e0;
    const int64_t bi = i * size, bj = j * size;
    int64_t* cp = csc_ptr + cptr_off[c];
    int64_t* rp = csr_ptr + rptr_off[c];
    // src-sorted order staged in csr_eid (overwritten by the CSR sort below); its pointer
    // array goes to rp, rewritten below as well
    stable_counting_sort(by_chunk.data() + e0, n, nsz(i), [&](int64_t e) { return src[e] - bi; },
                         csr_eid + e0, rp);
    stable_counting_sort(csr_eid + e0, n, nsz(j), [&](int64_t e) { return dst[e] - bj; },
                         csc_eid + e0, cp);
    stable_counting_sort(csc_eid + e0, n, nsz(i), [&](int64_t e) { return src[e] - bi; },
                         csr_eid + e0, rp);
#pragma omp parallel for schedule(static)
    for (int64_t k = e0; k < e1; ++k) {
      csc_idx[k] = (int32_t)(src[csc_eid[k]] - bi);
      csr_idx[k] = (int32_t)(dst[csr_eid[k]] - bj);
    }
  }
  return SG_OK;
}

int sg_host_gcn_weights(const int32_t* src, const int32_t* dst, const int64_t* dout,
                        const int64_t* din, const int64_t* eid, int64_t n, float* w) {
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < n; ++k) {
    int64_t e = eid ? eid[k] : k;
    double p = (double)dout[src[e]] * (double)din[dst[e]];
    w[k] = (float)(1.0 / std::sqrt(p));
  }
  return SG_OK;
}

int sg_host_plan(const int64_t* ptr, int64_t n_rows, int64_t pack_edges, int64_t max_rows,
                 int64_t split_edges, sg_item* items, sg_split* splits, int64_t* n_items,
                 int64_t* n_splits, int64_t* n_slots) {
  SG_REQUIRE(pack_edges >= 1 && max_rows >= 1 && split_edges >= 1, SG_EINVAL,
             "plan: pack_edges, max_rows and split_edges must be >= 1");
  SG_REQUIRE(n_rows <= INT32_MAX, SG_EINVAL, "plan: too many rows");
  // pass 1: count split rows / slots
  int64_t ns = 0, nslot = 0, nsplit_items = 0;
  for (int64_t r = 0; r < n_rows; ++r) {
    int64_t d = ptr[r + 1] - ptr[r];
    if (d > split_edges) {
      int64_t k = (d + split_edges - 1) / split_edges;
      ns++;
      nslot += k;
      nsplit_items += k;
    }
  }
  // split items first (largest work), then packed rows in row order
  int64_t it = 0, si = 0, slot = 0, pk = nsplit_items;
  int64_t r = 0;
  while (r < n_rows) {
    int64_t d = ptr[r + 1] - ptr[r];
    if (d > split_edges) {
      int64_t k = (d + split_edges - 1) / split_edges;
      if (items) {
        splits[si] = sg_split{(int32_t)r, (int32_t)k, slot};
        for (int64_t s = 0; s < k; ++s) {
          int64_t e0 = ptr[r] + s * split_edges;
          items[it + s] = sg_item{(int32_t)r, (int32_t)(r + 1), e0,
                                  std::min(e0 + split_edges, ptr[r + 1]), (int32_t)si, (int32_t)s};
        }
      }
      it += k;
      si++;
      slot += k;
      r++;
      continue;
    }
    int64_t start = r, edges = 0;
    while (r < n_rows && r - start < max_rows) {
      int64_t dr = ptr[r + 1] - ptr[r];
      if (dr > split_edges) break;
      if (r > start && edges + dr > pack_edges) break;
      edges += dr;
      r++;
    }
    if (items) items[pk] = sg_item{(int32_t)start, (int32_t)r, ptr[start], ptr[r], -1, 0};
    pk++;
  }
  *n_items = pk;
  *n_splits = ns;
  *n_slots = nslot;
  return SG_OK;
}

int sg_host_stage_plan(const int64_t* ptr, const int32_t* idx, const float* w, int64_t n_rows,
                       int64_t split_edges, int32_t group_pieces, int32_t batch_rows,
                       int32_t batch_entries, sg_stage_piece* pieces, int32_t* group_batch,
                       int64_t* batch_src_off, int32_t* batch_src, int64_t* batch_ent_off,
                       uint64_t* entries, uint16_t* batch_pofs, int64_t* sizes) {
  SG_REQUIRE(ptr && idx && sizes && n_rows >= 0 && n_rows <= INT32_MAX, SG_EINVAL, "stage_plan: bad args");
  SG_REQUIRE(split_edges >= 1 && group_pieces >= 1 && group_pieces <= 1024 && batch_rows >= 1 &&
                 batch_rows <= 65535 && batch_entries >= 1 && batch_entries <= 65535,
             SG_EINVAL, "stage_plan: bad limits");
  const int G = group_pieces;
  const int pstride = (G + 1 + 7) / 8 * 8;
  // pieces: whole rows, and split rows' T-edge subgroups numbered as sg_host_plan does
  struct P { int64_t e0, e1; sg_stage_piece p; int32_t first; };
  std::vector<P> ps;
  ps.reserve(n_rows);
  int64_t si = 0, slot = 0;
  for (int64_t r = 0; r < n_rows; ++r) {
    const int64_t d = ptr[r + 1] - ptr[r];
    for (int64_t e = ptr[r] + 1; e < ptr[r + 1]; ++e)
      SG_REQUIRE(idx[e] >= idx[e - 1], SG_EINVAL, "stage_plan: row %lld is not sorted by source", (long long)r);
    if (d > split_edges) {
      const int64_t k = (d + split_edges - 1) / split_edges;
      SG_REQUIRE(k < 65536, SG_EINVAL, "stage_plan: too many subgroups in row %lld", (long long)r);
      for (int64_t s = 0; s < k; ++s) {
        const int64_t e0 = ptr[r] + s * split_edges, e1 = std::min(e0 + split_edges, ptr[r + 1]);
        ps.push_back(P{e0, e1, sg_stage_piece{(int32_t)r, (int32_t)si, (int32_t)slot, (int32_t)((s << 16) | k)},
                       idx[e0]});
      }
      si++;
      slot += k;
    } else {
      ps.push_back(P{ptr[r], ptr[r + 1], sg_stage_piece{(int32_t)r, -1, 0, 0},
                     d > 0 ? idx[ptr[r]] : INT32_MAX});
    }
  }
  SG_REQUIRE(slot <= INT32_MAX, SG_EINVAL, "stage_plan: too many split slots");
  // pieces that start at the same source share the most sources: adjacent, then grouped
  std::stable_sort(ps.begin(), ps.end(), [](const P& a, const P& b) { return a.first < b.first; });
  const int64_t n_groups = ((int64_t)ps.size() + G - 1) / G;

  // per group: runs of equal (source, weight) per piece, merged source list, batches
  struct Grp {
    std::vector<int32_t> src;                 // staged sources, batch by batch
    std::vector<int64_t> src_off, ent_off;    // per batch (relative)
    std::vector<uint64_t> ent;
    std::vector<uint16_t> pofs;
    int64_t n_ent = 0;
    int bad = 0;
  };
  std::vector<Grp> gs(n_groups);
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t g = 0; g < n_groups; ++g) {
    Grp& gr = gs[g];
    const int64_t q0 = g * G, q1 = std::min<int64_t>(q0 + G, (int64_t)ps.size());
    // runs: (source, weight bits, count) per piece
    struct Run { int32_t src; uint32_t wb; uint32_t cnt; };
    std::vector<std::vector<Run>> runs(q1 - q0);
    std::vector<int32_t> all;
    for (int64_t q = q0; q < q1; ++q) {
      auto& rv = runs[q - q0];
      for (int64_t e = ps[q].e0; e < ps[q].e1; ++e) {
        uint32_t wb = 0;
        if (w) std::memcpy(&wb, w + e, 4);
        if (!rv.empty() && rv.back().src == idx[e] && rv.back().wb == wb && rv.back().cnt < 65535)
          rv.back().cnt++;
        else
          rv.push_back(Run{idx[e], wb, 1});
        all.push_back(idx[e]);
      }
    }
    std::sort(all.begin(), all.end());
    all.erase(std::unique(all.begin(), all.end()), all.end());
    // entries per source (across pieces), to close batches
    std::vector<int32_t> cu(all.size(), 0);
    for (auto& rv : runs)
      for (const Run& x : rv) cu[std::lower_bound(all.begin(), all.end(), x.src) - all.begin()]++;
    std::vector<size_t> cur(runs.size(), 0);
    size_t u = 0;
    gr.src_off.push_back(0);
    gr.ent_off.push_back(0);
    while (u < all.size()) {
      // close the batch at batch_rows sources or batch_entries entries
      size_t u1 = u;
      int64_t ne = 0;
      while (u1 < all.size() && (int64_t)(u1 - u) < batch_rows && ne + cu[u1] <= batch_entries) ne += cu[u1++];
      if (u1 == u) { gr.bad = 1; break; }
      const int32_t lo = all[u], hi = all[u1 - 1];
      for (size_t k = u; k < u1; ++k) gr.src.push_back(all[k]);
      // entries, piece-major (positions beyond the group's pieces stay empty)
      const size_t eb = gr.ent.size();
      for (int q = 0; q < G; ++q) {
        gr.pofs.push_back((uint16_t)(gr.ent.size() - eb));
        if (q >= (int)runs.size()) continue;
        auto& rv = runs[q];
        size_t& c = cur[q];
        while (c < rv.size() && rv[c].src <= hi) {
          const uint64_t sl = (uint64_t)(std::lower_bound(all.begin() + u, all.begin() + u1, rv[c].src) -
                                         (all.begin() + u));
          (void)lo;
          gr.ent.push_back(sl | ((uint64_t)rv[c].cnt << 16) | ((uint64_t)rv[c].wb << 32));
          c++;
        }
      }
      const size_t n_b = gr.ent.size() - eb;
      for (int q = G; q < pstride; ++q) gr.pofs.push_back((uint16_t)n_b);
      if (n_b & 1) gr.ent.push_back(0);   // 16-byte aligned batches for the bulk copies
      gr.src_off.push_back((int64_t)gr.src.size());
      gr.ent_off.push_back((int64_t)gr.ent.size());
      gr.n_ent += (int64_t)n_b;
      u = u1;
    }
    if (gr.src_off.size() == 1 && !gr.bad) {
      // a group of edgeless rows: one empty batch, so the kernel still writes its outputs
      for (int q = 0; q < pstride; ++q) gr.pofs.push_back(0);
      gr.src_off.push_back(0);
      gr.ent_off.push_back(0);
    }
  }
  for (auto& gr : gs) SG_REQUIRE(!gr.bad, SG_EINVAL, "stage_plan: a source has more than %d entries", batch_entries);
  // groups by descending entry count (longest first on the persistent CTAs)
  std::vector<int64_t> order(n_groups);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return gs[a].n_ent > gs[b].n_ent; });
  int64_t nb = 0, nsrc = 0, nent = 0;
  for (auto& gr : gs) {
    nb += (int64_t)gr.src_off.size() - 1;
    nsrc += (int64_t)gr.src.size();
    nent += (int64_t)gr.ent.size();
  }
  sizes[0] = n_groups; sizes[1] = nb; sizes[2] = nsrc; sizes[3] = nent; sizes[4] = si; sizes[5] = slot;
  if (!pieces) return SG_OK;
  SG_REQUIRE(group_batch && batch_src_off && batch_src && batch_ent_off && entries && batch_pofs, SG_EINVAL,
             "stage_plan: null output");
  SG_REQUIRE(nb <= INT32_MAX, SG_EINVAL, "stage_plan: too many batches");
  // output offsets in execution order
  std::vector<int64_t> gb(n_groups + 1, 0), gsrc(n_groups + 1, 0), gent(n_groups + 1, 0);
  for (int64_t k = 0; k < n_groups; ++k) {
    const Grp& gr = gs[order[k]];
    gb[k + 1] = gb[k] + (int64_t)gr.src_off.size() - 1;
    gsrc[k + 1] = gsrc[k] + (int64_t)gr.src.size();
    gent[k + 1] = gent[k] + (int64_t)gr.ent.size();
  }
  batch_src_off[nb] = nsrc;
  batch_ent_off[nb] = nent;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t k = 0; k < n_groups; ++k) {
    const int64_t g = order[k];
    const Grp& gr = gs[g];
    group_batch[k] = (int32_t)gb[k];
    for (int q = 0; q < G; ++q) {
      const int64_t pq = g * G + q;
      pieces[k * G + q] = pq < (int64_t)ps.size() ? ps[pq].p : sg_stage_piece{-1, -1, 0, 0};
    }
    const int64_t nbg = (int64_t)gr.src_off.size() - 1;
    for (int64_t b = 0; b < nbg; ++b) {
      batch_src_off[gb[k] + b] = gsrc[k] + gr.src_off[b];
      batch_ent_off[gb[k] + b] = gent[k] + gr.ent_off[b];
    }
    std::memcpy(batch_src + gsrc[k], gr.src.data(), gr.src.size() * 4);
    std::memcpy(entries + gent[k], gr.ent.data(), gr.ent.size() * 8);
    std::memcpy(batch_pofs + gb[k] * pstride, gr.pofs.data(), gr.pofs.size() * 2);
  }
  group_batch[n_groups] = (int32_t)nb;
  return SG_OK;
}

int sg_host_plan_order(sg_item* items, int64_t n_items, const int32_t* idx) {
  SG_REQUIRE(n_items >= 0 && (n_items == 0 || (items && idx)), SG_EINVAL, "plan_order: null pointer");
  int64_t ns = 0;
  while (ns < n_items && items[ns].split >= 0) ns++;  // split items lead the plan
  // subgroups that start at the same source traverse the same source rows at about the same
  // rate: adjacent in the queue, the warps of one CTA (which take consecutive items) share
  // them through L1.  Stable on (first source, row, subgroup); the per-row combination order
  // is by subgroup index, so results do not depend on this order.
  std::stable_sort(items, items + ns, [idx](const sg_item& a, const sg_item& b) {
    const int32_t sa = idx[a.e_begin], sb = idx[b.e_begin];
    if (sa != sb) return sa < sb;
    if (a.row_begin != b.row_begin) return a.row_begin < b.row_begin;
    return a.sub < b.sub;
  });
  return SG_OK;
}

}  // extern "C"
