/*
 * sagann.h -- C-ABI of the B200-native SAGA-NN layer hot path (libsagann.so).
 *
 * The reference (/root/reference/pkg/src/sagastream) is pure Python/numpy and
 * has no FFI; each entry point below replaces the reference interface named in
 * its comment (file:line).  Conventions:
 *   - plain pointers and sizes only; every buffer is caller-owned (device memory
 *     for sg_* kernels, host memory for sg_host_*); no hidden allocations;
 *   - row-major matrices with an explicit leading dimension (elements);
 *   - kernels are asynchronous on the given stream (a cudaStream_t, passed as
 *     void*; NULL = legacy default stream) and deterministic run to run (no
 *     float atomics);
 *   - every call returns a status code (SG_OK = 0) and never throws; the message
 *     of the last failure on the calling thread is sg_last_error().  Status codes
 *     mirror the reference's exceptions (errors.py:4-29): SG_ESHAPE -> ShapeError,
 *     SG_ENUMERIC -> NumericError, SG_EBUDGET -> BudgetError.
 */
#ifndef SAGANN_H
#define SAGANN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum sg_status {
  SG_OK = 0,
  SG_ESHAPE = 1,   /* ShapeError   (errors.py:8)  */
  SG_ENUMERIC = 2, /* NumericError (errors.py:12) */
  SG_EBUDGET = 3,  /* BudgetError  (errors.py:24) */
  SG_ECUDA = 4,
  SG_ENCCL = 5,
  SG_EINVAL = 6,
  SG_EFORMAT = 7   /* GraphFormatError (errors.py): malformed input file, line named */
};

enum sg_dtype {
  SG_F32 = 0,
  SG_BF16 = 1,
  /* sg_propagate only: bf16 gathered / row-side operands and mask (G, R, mask), fp32
   * outputs (out0, out1) -- bf16 storage of the gathered rows, fp32 aggregates */
  SG_BF16_F32OUT = 2
};

/* Propagation modes of sg_propagate (one fused Scatter-ApplyEdge-Gather pass). */
enum sg_prop_mode {
  SG_PROP_PASS = 0,         /* t_e = G[idx_e]                 (passthrough / segment_sum)   */
  SG_PROP_GCN = 1,          /* t_e = G[idx_e] * w_e           (GCN fwd on CSC, bwd on CSR)  */
  SG_PROP_GGCN_FWD = 2,     /* G=[h|P], R=Q:  t = sig(P[v]+Q[u]) * h[v]                     */
  SG_PROP_GGCN_BWD_DST = 3, /* CSC. G=[h|P], R=[dA|Q]: dQ[u] = sum ((dA[u]*h[v])*eta)*(1-eta) */
  SG_PROP_GGCN_BWD_SRC = 4, /* CSR. G=[dA|Q], R=[h|P]: dP[v] = sum t_e, dH[v] = sum dA[u]*eta */
  SG_PROP_GGCN_FWD_S = 5    /* GGCN_FWD + out1: S[u] = sum (h[v]*eta)*(1-eta), so the backward
                               dQ[u] = dA[u] * S[u] (dA[u] is constant over u's in-edges) */
};

enum sg_epilogue { SG_EPI_NONE = 0, SG_EPI_RELU_DUAL = 1 };
enum sg_gemm_prec { SG_GEMM_F32 = 0, SG_GEMM_TF32X3 = 1, SG_GEMM_BF16 = 2 };

/* Work item of a propagation pass (32 bytes).  A non-split item covers the whole
 * rows [row_begin, row_end); a split item covers edges [e_begin, e_end) of one
 * row (row_end = row_begin + 1), subgroup `sub` of split record `split`. */
typedef struct sg_item {
  int32_t row_begin, row_end;
  int64_t e_begin, e_end;
  int32_t split, sub;
} sg_item;

/* A row whose edge count exceeds the split threshold T. */
typedef struct sg_split {
  int32_t row, n_sub;
  int64_t slot0; /* partial rows slot0 .. slot0 + n_sub - 1 in the workspace */
} sg_split;

const char* sg_last_error(void);
int sg_version(void);
int sg_device_sm_count(int device, int* sm_count);
/* Number of device kernels this library has launched in this process (bench evidence). */
int64_t sg_launch_count(void);

/* ---------------------------------------------------------------- host: graph store
 * Synthetic generators (counter-based, identical to oracle/rng.py). */
int sg_host_gen_rmat(int64_t V, int64_t E, uint64_t seed, double t1, double t2, double t3,
                     int64_t edge_begin, int32_t* src, int32_t* dst);
int sg_host_gen_uniform(int64_t V, int64_t E, uint64_t seed, int64_t edge_begin,
                        int32_t* src, int32_t* dst);
int sg_host_gen_features(int64_t V, int64_t F, uint64_t seed, int64_t row_begin,
                         float* x, int64_t ldx);
/* degrees: deg_out / deg_in (int64 [V]). */
int sg_host_degrees(const int32_t* src, const int32_t* dst, int64_t E, int64_t V,
                    int64_t* dout, int64_t* din);
/* reencode_balance: perm[old] = new. */
int sg_host_reencode_balance(const int32_t* src, const int32_t* dst, int64_t E, int64_t V,
                             int64_t num_intervals, int64_t* perm);
/* partition_2d.  sg_host_partition_layout gives P and the length
 * of each pointer array (= P * (V + P)); sg_host_partition_2d fills the layout of
 * oracle/graph.py:Partition (chunk id c = i * P + j).  Canonical CSC: a destination's edges
 * by local source, multi-edges in input order ("CSC sorted by local dest id");
 * CSR stable over the CSC order. */
int sg_host_partition_layout(int64_t V, int64_t interval_size, int64_t* P, int64_t* ptr_len);
int sg_host_partition_2d(const int32_t* src, const int32_t* dst, int64_t E, int64_t V,
                         int64_t interval_size, int64_t* edge_off, int64_t* cptr_off,
                         int64_t* rptr_off, int64_t* csc_ptr, int32_t* csc_idx, int64_t* csc_eid,
                         int64_t* csr_ptr, int32_t* csr_idx, int64_t* csr_eid);
/* GCN static edge weight w = 1/sqrt(deg_out(src) * deg_in(dst)),
 * evaluated in fp64 and rounded to fp32, for edges eid[0..n). */
int sg_host_gcn_weights(const int32_t* src, const int32_t* dst, const int64_t* dout,
                        const int64_t* din, const int64_t* eid, int64_t n, float* w);
/* Work plan of a CSC/CSR pass: rows with > split_edges edges become split rows
 * (subgroups of split_edges edges); other rows are packed in order
 * into items of <= pack_edges edges and <= max_rows rows.  Call with items ==
 * NULL to count. */
int sg_host_plan(const int64_t* ptr, int64_t n_rows, int64_t pack_edges, int64_t max_rows,
                 int64_t split_edges, sg_item* items, sg_split* splits, int64_t* n_items,
                 int64_t* n_splits, int64_t* n_slots);
/* Reorder a plan's split items (in place) by the source of their first edge (idx[e_begin]),
 * then row and subgroup, so that subgroups covering the same sources are adjacent in the work
 * queue (results are independent of the item order). */
int sg_host_plan_order(sg_item* items, int64_t n_items, const int32_t* idx);

/* One destination row of a staged gather (or one T-edge subgroup of a row with more than T
 * edges, SPEC.md:443 -- the same subgroups, split ids and partial slots as sg_host_plan).
 * row < 0: an unused position of the group. */
typedef struct sg_stage_piece {
  int32_t row, split, slot0, sub_nsub; /* sub_nsub = sub << 16 | n_sub (split pieces) */
} sg_stage_piece;

/* Work plan of the source-staged gather (sg_propagate_staged).  Pieces (whole rows and split
 * subgroups) are ordered by their first source and cut into groups of group_pieces; a group's
 * pieces gather from the merged, ascending list of the sources they reference, which the
 * kernel stages into shared memory batch_rows rows at a time, so a source row shared by
 * several pieces of a group crosses L2 -> SM once.  Per batch: the staged source rows
 * (batch_src), and the entries of every piece that reference them, piece-major, each a run of
 * equal consecutive (source, weight) edges: bits 0-15 the row's slot in the batch, 16-31 the
 * run length, 32-63 the weight (0 without w); batch_pofs[b * pofs_stride + q] is the first entry
 * of piece q (q = 0 .. group_pieces, pofs_stride = group_pieces + 1 rounded up to 8).  Each
 * piece's edges are visited in index order, so every row sums its terms in the same order as
 * sg_propagate (bitwise identical).  Groups are listed by descending entry count.
 * Requires idx non-decreasing within every row (the canonical CSC / CSR of ChunkGrid);
 * returns SG_EINVAL otherwise or when one source's entries exceed batch_entries.
 * Call with pieces == NULL to size: sizes = {n_groups, n_batches, n_src, n_ent, n_splits,
 * n_slots}. */
int sg_host_stage_plan(const int64_t* ptr, const int32_t* idx, const float* w, int64_t n_rows,
                       int64_t split_edges, int32_t group_pieces, int32_t batch_rows,
                       int32_t batch_entries, sg_stage_piece* pieces, int32_t* group_batch,
                       int64_t* batch_src_off, int32_t* batch_src, int64_t* batch_ent_off,
                       uint64_t* entries, uint16_t* batch_pofs, int64_t* sizes);

/* ---------------------------------------------------------------- host: ingestion
 * load_graph's file formats.  Edge file: one "src dest
 * [edge_value]" per line, whitespace separated (blank, '#' and '%' lines skipped).
 * Feature file: text CSV or binary (u64 rows, u64 cols, row-major f64, little endian).
 * Label file: one integer per line.  Scan first (sizes; vertex_limit >= 0 bounds-checks
 * ids), then read into caller buffers.  Errors (SG_EFORMAT) name the 1-based line. */
int sg_host_scan_edges(const char* path, int64_t vertex_limit, int64_t* n_edges, int64_t* max_id,
                       int* has_value);
int sg_host_read_edges(const char* path, int64_t n_edges, int32_t* src, int32_t* dst, double* value);
int sg_host_scan_matrix_text(const char* path, int64_t* rows, int64_t* cols);
int sg_host_read_matrix_text(const char* path, int64_t rows, int64_t cols, double* out);
int sg_host_read_matrix_bin_header(const char* path, int64_t* rows, int64_t* cols);
int sg_host_read_matrix_bin(const char* path, int64_t rows, int64_t cols, double* out);
int sg_host_write_matrix_bin(const char* path, int64_t rows, int64_t cols, const double* data);
int sg_host_scan_labels(const char* path, int64_t* n);
int sg_host_read_labels(const char* path, int64_t n, int64_t* out);
/* Order-sensitive 64-bit content hash (keys the on-disk partition cache). */
uint64_t sg_host_hash64(const void* data, int64_t nbytes, uint64_t seed);

/* ---------------------------------------------------------------- device: propagation
 * One fused Scatter-ApplyEdge-Gather pass over a CSC (forward) or CSR (backward)
 * index: for each row r, out[r] (+)= sum over e in [ptr[r], ptr[r+1]) of t_e in
 * edge order (split rows: subgroup partials combined in fixed order by a second launch on
 * the same stream).
 * Replaces take_rows -> mul/add/sigmoid -> segment_sum (tensor.py:424-450,
 * :204-303) and SPEC stage ops fused_gather_chunk / backward_* (SPEC.md:419-436).
 *   G, ldg, g_off : gathered rows (second operand segment at column g_off)
 *   R, ldr, r_off : row-side rows (may be NULL for PASS / GCN)
 *   out0/out1     : outputs (out1 for GGCN_BWD_SRC: dH_take; for GGCN_FWD_S: S)
 *   mask, ldm     : optional ReLU-backward mask: out0 = acc * (mask > 0) (tensor.py:236)
 *   workspace     : >= sg_propagate_workspace_bytes(...) bytes of device memory
 */
int64_t sg_propagate_workspace_bytes(int64_t n_items, int64_t n_splits, int64_t n_slots,
                                     int64_t F, int mode);
int sg_propagate(int mode, int dtype, const int64_t* ptr, const int32_t* idx, const float* w,
                 int64_t n_rows, const sg_item* items, int64_t n_items, const sg_split* splits,
                 int64_t n_splits, int64_t n_slots, const void* G, int64_t ldg, int64_t g_off,
                 const void* R, int64_t ldr, int64_t r_off, void* out0, int64_t ld0, void* out1,
                 int64_t ld1, const void* mask, int64_t ldm, int64_t F, int accumulate,
                 void* workspace, int64_t workspace_bytes, void* stream);

/* Source-staged sum pass (GCN / PASS modes, fp32, F <= 640, 16-byte aligned rows): the same
 * function as sg_propagate -- bitwise identical outputs, same split slots / workspace
 * (sg_propagate_workspace_bytes with the plan's n_splits, n_slots) -- driven by a
 * sg_host_stage_plan.  Each persistent CTA takes groups of pieces from a queue and stages the
 * group's source rows into shared memory with TMA bulk copies (cp.async.bulk, mbarrier
 * complete_tx), batch_rows rows per batch, 2-3 stages deep; every source row a group shares
 * is read from L2 once per group instead of once per edge.  group_pieces must be
 * sg_stage_group_pieces(F); the dynamic shared memory is sg_stage_smem_bytes(...) (<= 227 KB).
 * mask (optional): ReLU-backward epilogue as in sg_propagate. */
int32_t sg_stage_group_pieces(int64_t F);
int64_t sg_stage_smem_bytes(int32_t group_pieces, int32_t batch_rows, int32_t batch_entries, int64_t F,
                            int32_t stages);
int sg_propagate_staged(int mode, const sg_stage_piece* pieces, const int32_t* group_batch, int64_t n_groups,
                        const int64_t* batch_src_off, const int32_t* batch_src, const int64_t* batch_ent_off,
                        const uint64_t* entries, const uint16_t* batch_pofs, int32_t group_pieces,
                        int32_t batch_rows, int32_t batch_entries, int32_t stages, int64_t n_splits,
                        int64_t n_slots, const float* G, int64_t ldg, float* out, int64_t ldo, const float* mask,
                        int64_t ldm, int64_t F, int accumulate, void* workspace, int64_t workspace_bytes,
                        void* stream);

/* sg_propagate with a hub-row cache (GCN / PASS modes, rows wider than 16 vectors).
 * The n_hub most referenced gathered rows (hub_rows[0..n_hub), int32 row ids of G) are
 * copied into each block's shared memory once; idx must be the hub-encoded index in
 * which an edge to hub slot k carries (int32)(k | 0x80000000) instead of its row id.
 * Results are bitwise identical to sg_propagate over the plain index.
 * n_hub <= sg_propagate_hub_capacity(F, dtype); n_hub = 0 is plain sg_propagate. */
int64_t sg_propagate_hub_capacity(int64_t F, int dtype);
int sg_propagate_hub(int mode, int dtype, const int64_t* ptr, const int32_t* idx, const float* w,
                     int64_t n_rows, const sg_item* items, int64_t n_items, const sg_split* splits,
                     int64_t n_splits, int64_t n_slots, const void* G, int64_t ldg, int64_t g_off,
                     const void* R, int64_t ldr, int64_t r_off, void* out0, int64_t ld0, void* out1,
                     int64_t ld1, const void* mask, int64_t ldm, int64_t F, int accumulate,
                     const int32_t* hub_rows, int64_t n_hub, void* workspace, int64_t workspace_bytes,
                     void* stream);

/* Gather(max) with argmax (segment_max, tensor.py:453-484):
 * out[r] = max over rows X[idx_e] (strict >, lowest edge position wins), -inf
 * init, empty rows get empty_fill and argmax -1; argmax holds idx_e (int64). */
int sg_segment_max(int dtype, const int64_t* ptr, const int32_t* idx, int64_t n_rows,
                   const void* X, int64_t ldx, void* out, int64_t ldo, int64_t* argmax,
                   int64_t lda, int64_t F, float empty_fill, void* stream);
/* backward of segment_max: gx[argmax[r,f], f] = g[r, f] (gx pre-zeroed by caller). */
int sg_segment_max_bwd(int dtype, const void* g, int64_t ldg, const int64_t* argmax, int64_t lda,
                       int64_t n_rows, void* gx, int64_t ldx, int64_t F, void* stream);
/* Fused Gather(max) over a CSC index (MP-GCN ApplyEdge hoisted to Y, PAPER.md:574-586;
 * segment_max, tensor.py:453-484): out[u] = max over in-edges of Y[idx_e]; argpos[u,f]
 * = global position (pos_base + CSC position) of the first maximum (int32), -1 for
 * empty rows.  2D grid: pos_base = the chunk's offset in the source-interval-major
 * flattening; the chunks of one destination interval run in source order with
 * accumulate = 1 after the first (running max/argmax read back from out/argpos), and
 * finalize = 1 on the last writes empty_fill into rows that saw no edge.
 * fp32; Y rows with ld % 4 == 0 are read as 16-B vectors. */
int sg_max_gather(const int64_t* ptr, const int32_t* idx, int64_t n_rows, const float* Y, int64_t ldy,
                  float* out, int64_t ldo, int32_t* argpos, int64_t lda, int64_t F, float empty_fill,
                  int64_t pos_base, int accumulate, int finalize, void* stream);
/* Its backward over the transposed (CSR) index: out[v] (+)= sum over out-edges k (CSR
 * order) of G[idx_k] where argpos[idx_k] == pos_base + pos_k (the edge's global
 * position), else +0.0; accumulate continues the previous chunk of the source interval;
 * optional ReLU mask (pass it on the last chunk).  Bitwise equal to segment_max's
 * backward followed by take_rows' backward (tensor.py:473-482, :431-434). */
int sg_max_gather_bwd(const int64_t* ptr, const int32_t* idx, const int32_t* pos, int64_t n_rows,
                      const float* G, int64_t ldg, const int32_t* argpos, int64_t lda, float* out,
                      int64_t ldo, int64_t F, const float* mask, int64_t ldm, int64_t pos_base,
                      int accumulate, void* stream);
/* Plan-driven variants of sg_max_gather / sg_max_gather_bwd for passes with split rows
 * (R-MAT hubs): the pass's work plan (sg_host_plan) is pulled from an atomic queue and a
 * heavy row's subgroups run in parallel.  The forward result is bit-identical to the
 * sequential one (max / argmax are exact; partials are combined lowest position first); the
 * backward sums a split row's subgroups in subgroup order (as sg_propagate).
 * workspace >= sg_max_plan_workspace_bytes(n_splits, n_slots, F). */
int64_t sg_max_plan_workspace_bytes(int64_t n_splits, int64_t n_slots, int64_t F);
int sg_max_gather_plan(const int64_t* ptr, const int32_t* idx, const sg_item* items, int64_t n_items,
                       const sg_split* splits, int64_t n_splits, int64_t n_slots, const float* Y, int64_t ldy,
                       float* out, int64_t ldo, int32_t* argpos, int64_t lda, int64_t F, float empty_fill,
                       int64_t pos_base, int accumulate, int finalize, void* workspace,
                       int64_t workspace_bytes, void* stream);
/* segment_max (tensor.py:453-484) over a segment index with split segments, fp32: as
 * sg_segment_max (argmax = the gathered row idx[e], int64) but plan-driven like
 * sg_max_gather_plan (bit-identical to the sequential result). */
int sg_segment_max_plan(const int64_t* ptr, const int32_t* idx, const sg_item* items, int64_t n_items,
                        const sg_split* splits, int64_t n_splits, int64_t n_slots, const float* X, int64_t ldx,
                        float* out, int64_t ldo, int64_t* argmax, int64_t lda, int64_t F, float empty_fill,
                        void* workspace, int64_t workspace_bytes, void* stream);
int sg_max_gather_bwd_plan(const int64_t* ptr, const int32_t* idx, const int32_t* pos, const sg_item* items,
                           int64_t n_items, const sg_split* splits, int64_t n_splits, int64_t n_slots,
                           const float* G, int64_t ldg, const int32_t* argpos, int64_t lda, float* out,
                           int64_t ldo, int64_t F, const float* mask, int64_t ldm, int64_t pos_base,
                           int accumulate, void* workspace, int64_t workspace_bytes, void* stream);
/* Scatter (take_rows, tensor.py:424-436): out[k] = X[idx[k]] (int64 idx, bounds
 * checked on device: *err_flag set to 1 if any index is out of [0, n_src)). */
int sg_take_rows(int dtype, const void* X, int64_t ldx, int64_t n_src, const int64_t* idx,
                 int64_t n, void* out, int64_t ldo, int64_t F, int32_t* err_flag, void* stream);
/* Stable counting sort of segment ids (int64 [n], values in [0, n_seg)) into a
 * CSC-like (ptr [n_seg+1], perm int32 [n]); perm is stable (row order within a
 * segment), so sg_propagate(PASS) over it equals np.add.at (tensor.py:445).
 * Sets *err_flag if an id is out of range.  workspace >= sg_sort_workspace_bytes. */
int64_t sg_sort_workspace_bytes(int64_t n, int64_t n_seg);
int sg_segment_sort(const int64_t* seg, int64_t n, int64_t n_seg, int64_t* ptr, int32_t* perm,
                    int32_t* err_flag, void* workspace, int64_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------- device: dense
 * ApplyVertex GEMM (matmul, tensor.py:306-319): C[M,N] = op(A)[M,K] . op(B)[K,N],
 * row-major; trans_a: A is stored [K,M]; trans_b: B is stored [N,K].  Epilogue
 * RELU_DUAL also writes D = relu(C) (tensor.py:207).  Split-K reductions are
 * deterministic (fixed order).  prec: SG_GEMM_F32 (SIMT fp32), SG_GEMM_TF32X3
 * (tcgen05 kind::tf32, 3xTF32 split, TMEM accumulators), SG_GEMM_BF16 (tcgen05
 * kind::f16 on bf16 operands, fp32 TMEM accumulation; through sg_gemm the A/B pointers
 * are bf16 and C/D fp32 -- use sg_gemm_ex for bf16 outputs). */
int64_t sg_gemm_workspace_bytes(int64_t M, int64_t N, int64_t K, int prec);
int sg_gemm(int prec, int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, const float* A,
            int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc, int epilogue,
            float* D, int64_t ldd, void* workspace, int64_t workspace_bytes, void* stream);

/* The general form of sg_gemm (same operation and precisions):
 *   A, B      : fp32 for F32 / TF32X3, bf16 (SG_BF16) for SG_GEMM_BF16 (bf16 rows need
 *               ld % 8 == 0 and 16-B aligned bases: the TMA tensor-map constraints);
 *   C, c_dtype: output (fp32 or bf16; bf16 with TF32X3 needs the TMA-eligible 16-B aligned
 *               operands); may be NULL when epilogue == RELU_DUAL (only D), not with F32;
 *   D, d_dtype: D = relu(C) (np.maximum semantics: NaN propagates), fp32 or bf16;
 *   nonfinite : optional device flag, |= 1 if any element of C is non-finite (the
 *               strict-mode check of tensor.py:161-163 fused into the epilogue).
 * bf16 outputs are rounded once from the fp32 accumulator (round to nearest even).
 * Split-K (long K) needs fp32 outputs. */
typedef struct sg_gemm_desc {
  int prec, trans_a, trans_b, epilogue;
  int64_t M, N, K;
  const void* A;
  int64_t lda;
  const void* B;
  int64_t ldb;
  void* C;
  int64_t ldc;
  int c_dtype;
  void* D;
  int64_t ldd;
  int d_dtype;
  int32_t* nonfinite;
  void* workspace;
  int64_t workspace_bytes;
} sg_gemm_desc;
int sg_gemm_ex(const sg_gemm_desc* desc, void* stream);

/* Softmax cross-entropy head (tensor.py:487-506) on logits = relu(Z) when
 * relu_input (the last layer's ReLU) else Z, over n local rows:
 * writes -sum(log p[label]) / n_total to *loss (device fp32 scalar) and
 * dZ = (p - onehot) / n_total, times the ReLU mask when relu_input.  n_total is the
 * global row count when rows are sharded across ranks (<= 0 means n).  labels int64
 * [n]; *err_flag <- 1 on a bad label. */
int64_t sg_xent_workspace_bytes(int64_t n);
int sg_softmax_xent(const float* Z, int64_t ldz, int relu_input, const int64_t* labels, int64_t n,
                    int64_t C, int64_t n_total, float* loss, float* dZ, int64_t lddz,
                    int32_t* err_flag, void* workspace, int64_t workspace_bytes, void* stream);

/* Plain gradient descent W <- W - lr * dW. */
int sg_sgd(float* W, const float* dW, int64_t n, float lr, void* stream);
/* Strict mode (tensor.py:18-19, :161-163): *flag |= 1 if any non-finite element. */
int sg_check_finite(int dtype, const void* X, int64_t rows, int64_t cols, int64_t ld,
                    int32_t* flag, void* stream);
/* Elementwise ops used by unfused ApplyEdge programs (tensor.py:204-303):
 * op 0 add, 1 sub, 2 mul, 3 div, 4 max, 5 sigmoid, 6 tanh, 7 relu,
 * 8 relu-backward (a * (b > 0), tensor.py:236),
 * 9 sigmoid-backward (a * b * (1 - b) with b = y, tensor.py:232),
 * 10 tanh-backward (a * (1 - b * b) with b = y, tensor.py:234); b is broadcast
 * per row when b_cols == 1 (the "b_row" kind, tensor.py:184-185), along the
 * leading axis when b_rows == 1 ("b_lead"). */
int sg_ewise(int op, int64_t rows, int64_t cols, const float* a, int64_t lda, const float* b,
             int64_t b_rows, int64_t b_cols, int64_t ldb, float* out, int64_t ldo, void* stream);
/* Backward of binary op 0-4 (the bwd closure of _binary, tensor.py:255-265): given the
 * upstream gradient g and the forward operands a (full [rows, cols]) and b (broadcast as in
 * sg_ewise), writes both full-shape partials ga, gb (add: g, g; sub: g, -g; mul: g*b, g*a;
 * div: g/b, -g*a/(b*b); max: g*(a>=b), g*!(a>=b) -- ties route to a).  The caller reduces
 * a broadcast side back to its shape with sg_reduce_sum (_reduce_to, tensor.py:191-201). */
int sg_ewise_bwd(int op, int64_t rows, int64_t cols, const float* g, int64_t ldg, const float* a,
                 int64_t lda, const float* b, int64_t b_rows, int64_t b_cols, int64_t ldb, float* ga,
                 int64_t ldga, float* gb, int64_t ldgb, void* stream);
/* _reduce_to's sums (tensor.py:197-201): axis 1 -> out[rows] = row sums (row-scalar side),
 * axis 0 -> out[cols] = column sums over the broadcast leading axis (fixed-order partials in
 * the caller-owned workspace of sg_reduce_workspace_bytes(cols) bytes).  Deterministic. */
int64_t sg_reduce_workspace_bytes(int64_t cols);
int sg_reduce_sum(int axis, const float* X, int64_t ld, int64_t rows, int64_t cols, float* out,
                  void* workspace, int64_t workspace_bytes, void* stream);
/* GG-NN ApplyVertex = GRU(vertex, accum) (Li et al. form,
 * no biases), the element-wise stages around the ApplyVertex GEMMs.  G1 = a [Wz|Wr|Wh],
 * G2 = h [Uz|Ur], G3 = (r*h) Uh, gate blocks at column stride bs (>= F); z/r/rh/c share ldo.
 *   gates: z = s(G1z + G2z), r = s(G1r + G2r), rh = r*h       (s = 1/(1+exp(-x)), tensor.py:205)
 *   out:   c = tanh(G1h + G3), hn = (1-z)*h + z*c
 *   bwd1:  D3[:,0] = gzp, D3[:,2bs] = gcp, gh = g*(1-z)       (tape reverse order, tensor.py:231-263)
 *   bwd2:  gh += grh*r, D3[:,bs] = grp                        (grh = gcp Uh^T) */
int sg_gru_gates(int64_t V, int64_t F, const float* G1, int64_t ld1, const float* G2, int64_t ld2,
                 int64_t bs, const float* h, int64_t ldh, float* z, float* r, float* rh, int64_t ldo,
                 void* stream);
int sg_gru_out(int64_t V, int64_t F, const float* G1, int64_t ld1, int64_t bs, const float* G3,
               int64_t ld3, const float* z, const float* h, int64_t ldh, float* c, float* hn,
               int64_t ldo, int64_t ldn, void* stream);
int sg_gru_bwd1(int64_t V, int64_t F, const float* g, int64_t ldg, const float* z, const float* c,
                int64_t ldo, const float* h, int64_t ldh, float* D3, int64_t ld3, int64_t bs, float* gh,
                int64_t ldgh, void* stream);
int sg_gru_bwd2(int64_t V, int64_t F, const float* grh, int64_t ldr, const float* r, int64_t ldo,
                const float* h, int64_t ldh, float* gh, int64_t ldgh, float* D3, int64_t ld3, int64_t bs,
                void* stream);
/* fp32 <-> bf16 row copy with padding (feature staging). */
int sg_convert(int src_dtype, int dst_dtype, const void* X, int64_t ldx, void* Y, int64_t ldy,
               int64_t rows, int64_t cols, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SAGANN_H */
