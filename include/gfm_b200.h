/*
 * gfm_b200 -- C ABI of the B200-native (sm_100a) gfmkit training hot path.
 *
 * The reference (gfmkit, /root/reference/pkg/src/gfmkit) is pure Python +
 * numpy and has no FFI; each entry point below replaces the numpy operation
 * cited beside it (file:line relative to that package).  INTEGRATION.md shows
 * the ctypes binding a gfmkit maintainer would add.
 *
 * Conventions
 *  - Every function is stream-ordered on `stream` (a cudaStream_t passed as
 *    void*), works on caller-owned DEVICE buffers, allocates nothing, and
 *    returns 0 or a nonzero status (cudaError_t value, or GFM_EINVAL);
 *    gfm_last_error() then holds a message (thread-local).
 *  - Indices are int32.  Floating buffers are float32 (GFM_F32) or float64
 *    (GFM_F64) per the `dtype` argument; positions are always float64.
 *  - Node features are row-major [n_nodes][H].  A batch is a dst-sorted CSR
 *    (rowptr[N+1], col_src[E], edge_dst[E], edge_w[E], edge_dx[E][3]) plus the
 *    src-sorted CSC view (csc_ptr[N+1], csc_eid[E] = CSR position,
 *    csc_dst[E]); CSR order equals the reference's stable dst sort
 *    (model.py:260) so argmax indices and segment orders agree.
 *  - Functions that size grids from an upper bound `e_cap` read the actual
 *    edge count from rowptr[n_nodes] on the device (CUDA-graph friendly).
 *  - Results are deterministic: no floating-point atomics; every reduction
 *    has a fixed order chosen from shapes only.
 */
#ifndef GFM_B200_H
#define GFM_B200_H

#include <stddef.h>

#if defined(__GNUC__)
#define GFM_API __attribute__((visibility("default")))
#else
#define GFM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define GFM_ABI_VERSION 3

enum { GFM_F32 = 0, GFM_F64 = 1 };
enum { GFM_EINVAL = -1 };
/* aggregation parts (bit order = column-block order of the output) */
enum { GFM_PART_SUM = 1, GFM_PART_MEAN = 2, GFM_PART_MAX = 4, GFM_PART_STD = 8 };
enum { GFM_FLAG_SCALAR = 1 }; /* force the scalar (numpy-order) kernels */
/* aggregation: argmax is a uint8 [N][H] buffer holding the LOW BYTE of the CSR
 * position (unique within a row; valid when every CSR row has <= 256 edges,
 * e.g. a neighbour cap <= 256) -- 4x fewer bytes gathered by the backward */
enum { GFM_FLAG_ARGMAX_U8 = 2 };
/* gfm_agg_bwd: G | coef already in `workspace` and `dagg` is the max part's
 * gradient [N][H] (as written by gfm_layer_bwd_data_agg) -- no prep pass */
enum { GFM_FLAG_AGG_PREPPED = 4 };
/* gfm_agg_bwd: edge_w is in CSC order (w[q] for CSC slot q, e.g. from
 * gfm_permute) -- a coalesced load instead of a dependent gather w[eid] */
enum { GFM_FLAG_W_CSC = 8 };
/* gfm_agg_bwd: the gathered rows are local (batches of small graphs: a
 * node's neighbours sit in the same few hundred rows, mostly L2 hits) --
 * shallower gather batches; without it the backward keeps more rows in
 * flight for scattered (HBM-latency-bound) sources */
enum { GFM_FLAG_GATHER_LOCAL = 16 };
/* float32 GEMM engine: tcgen05 3xTF32 (default, fp32-level accuracy),
 * tcgen05 1xTF32 (faster, ~1e-3 relative), the SIMT fp32 engine, or MIXED:
 * 3xTF32 everywhere except the weight-gradient GEMMs (gfm_linear_bwd_weight*,
 * gfm_embedding_grad), which run 1xTF32 */
enum { GFM_GEMM_SIMT = 0, GFM_GEMM_TC3 = 1, GFM_GEMM_TC1 = 2, GFM_GEMM_MIXED = 3 };

/* ---- housekeeping ---------------------------------------------------- */
GFM_API int gfm_abi_version(void);
GFM_API const char* gfm_last_error(void);
GFM_API int gfm_device_sm_count(void);
GFM_API int gfm_stream_sync(void* stream);
GFM_API int gfm_set_gemm_mode(int mode);
GFM_API int gfm_get_gemm_mode(void);
/* tcgen05 3xTF32 GEMMs on CTA pairs (cta_group::2, M = 256 MMAs, each CTA
 * staging half of the B tile): 1 on, 0 off; returns the previous setting */
GFM_API int gfm_set_tc_pairs(int on);
/* CTA-pair GEMM launches since the library was loaded (diagnostics) */
GFM_API long long gfm_tc_pair_launches(void);

/* ---- K1/K2: batch geometry (preprocess.py:90-104, model.py:234-285) --- */
/* gnode[i] = graph of node i (model.py:243) */
GFM_API int gfm_graph_of_node(const int* node_offsets, int n_graphs, int* gnode, void* stream);
/* Device sample store gather, replacing DDStore.fetch_batch + decode_record
 * + make_batch's host concatenation (ddstore.py:316-490, records.py:154-183,
 * model.py:237-250): output structure b = resident structure idx[b], its
 * atoms written at dst_off[b] (caller-computed, e.g. a fixed runner layout).
 * z int32, pos float64 in and out; energy/forces float64 in, `dtype` out. */
GFM_API int gfm_gather_structures(const int* idx, int n_out, const int* src_off,
                                  const int* dst_off, const int* z_in, const double* pos_in,
                                  const double* energy_in, const double* forces_in, int* z_out,
                                  double* pos_out, void* energy_out, void* forces_out, int dtype,
                                  void* stream);
/* out[0..n] = exclusive prefix sum of in[0..n) (np.cumsum, model.py:238) */
/* Device batch assembly from a store group's per-structure CSR blocks
 * (replaces make_batch's host concatenation + CSR/CSC build for records
 * that keep their own edges, model.py:234-285).  The group (n_s structures)
 * was packed once by gfm_csr_build in float64: s_off [n_s+1], s_z, s_pos,
 * s_e, s_f, s_rowptr / s_col / s_w / s_dx / s_cscptr / s_cscid / s_cscdst.
 * Output graph b = structure idx[b]; meta (device) = [B_true, N_true |
 * node offsets (n_cap_graphs+1) | n_per (n_cap_graphs) | edge offsets
 * (n_cap_graphs+1)].  Writes the batch's inputs and its CSR / CSC in the
 * compute dtype; nodes past N_true up to n_nodes are edge-free with gnode -1.
 * Capture-safe: every size is read from `meta`. */
GFM_API int gfm_gather_batch(const int* idx, const int* meta, int n_cap_graphs, int n_nodes,
                             const int* s_off, const int* s_z, const double* s_pos,
                             const double* s_e, const double* s_f, const int* s_rowptr,
                             const int* s_col, const double* s_w, const double* s_dx,
                             const int* s_cscptr, const int* s_cscid, const int* s_cscdst, int* z,
                             double* pos, void* e, void* f, int* gnode, int* rowptr, int* col_src,
                             int* edge_dst, void* w, void* dx, int* csc_ptr, int* csc_eid,
                             int* csc_dst, int dtype, void* stream);
/* Variable-length row-block gather (sharded store pack / unpack, the
 * NVLink shard exchange replacing DDStore's remote fetch, ddstore.py:441-464):
 * output block b = input block idx[b] (idx NULL: identity), rows
 * [src_off[s], src_off[s+1]) copied to rows from dst_off[b], `width` 32-bit
 * words per row; add[b] (optional) is added to every word (node-id shift). */
GFM_API int gfm_gather_blocks(const int* idx, int n_out, const long long* src_off,
                              const long long* dst_off, int width, const void* in, void* out,
                              const int* add, void* stream);
/* out[q] = in[idx[q]] for q < min(n, *n_dev) (n_dev may be NULL): e.g. the
 * edge weights in CSC order, w_csc = edge_w[csc_eid] (GFM_FLAG_W_CSC) */
GFM_API int gfm_permute(const int* idx, int n, const int* n_dev, const void* in, void* out,
                        int dtype, void* stream);
GFM_API size_t gfm_scan_workspace_bytes(int n);
GFM_API int gfm_exclusive_scan(const int* in, int n, int* out, void* workspace, void* stream);
/* Radius graph replacing build_cutoff_edges (preprocess.py:90-104), emitted
 * directly as the dst-sorted CSR make_batch builds (model.py:256-267).  The
 * float64 predicate sqrt((dx^2+dy^2)+dz^2) <= rc is bit-exact against numpy.
 * cells: NULL or per-graph orthorhombic box [n_graphs][3] (minimum image,
 * needs rc < L/2); max_nbr > 0 keeps the max_nbr nearest sources per
 * destination by (distance, source index).  Two passes: count -> scan ->
 * fill. */
GFM_API int gfm_radius_count(const double* pos, const int* node_offsets, const int* gnode, int n_nodes,
                     const double* cells, double rc, int max_nbr, int* deg, void* stream);
GFM_API int gfm_radius_fill(const double* pos, const int* node_offsets, const int* gnode, int n_nodes,
                    const double* cells, double rc, int max_nbr, const int* rowptr, int* col_src,
                    int* edge_dst, void* edge_w, void* edge_dx, int dtype, void* stream);
/* make_batch for arbitrary record edge lists (model.py:245-267): stable dst
 * sort -> CSR (order[p] = original edge index, model.py:260), w/dx from
 * float64 positions (+ optional per-edge periodic shift), and the stable src
 * sort -> CSC.  src/dst are global node ids in original order; edge_offsets
 * [n_graphs+1] delimit each graph's edges. */
GFM_API size_t gfm_csr_workspace_bytes(int n_nodes, int n_edges, int n_graphs);
GFM_API int gfm_csr_build(const int* src, const int* dst, const int* edge_offsets, int n_graphs,
                  const double* pos, const double* shift, int n_nodes, int n_edges, int* rowptr,
                  int* col_src, int* edge_dst, void* edge_w, void* edge_dx, int* order,
                  int* csc_ptr, int* csc_eid, int* csc_dst, int dtype, void* workspace,
                  void* stream);
/* CSC view of a CSR produced by gfm_radius_fill (workspace sized by
 * gfm_csr_workspace_bytes(n_nodes, e_cap, n_graphs)). */
GFM_API int gfm_csc_from_csr(const int* rowptr, const int* col_src, const int* edge_dst,
                     const int* node_offsets, int n_graphs, int n_nodes, int e_cap, int* csc_ptr,
                     int* csc_eid, int* csc_dst, void* workspace, void* stream);

/* Fused batch assembly (replaces graph_of_node + radius_count + scan +
 * radius_fill + csc_from_csr): one CTA per graph (graphs of up to 256 atoms;
 * GFM_EINVAL otherwise -- use the separate calls), same predicate, cap, order
 * and outputs.  `workspace`: gfm_radius_batch_workspace_bytes (scratch).
 * Capacity semantics (ragged batches in a fixed-shape captured step): n_nodes
 * may exceed node_offsets[n_graphs]; the tail nodes get rowptr = csc_ptr = E
 * (no edges) and gnode = -1.  The edge buffers hold e_cap edges: a batch with
 * more is emitted edge-free and raises the int overflow flag at index
 * gfm_radius_batch_overflow_index(n_graphs) of the workspace (no
 * out-of-bounds writes). */
GFM_API size_t gfm_radius_batch_workspace_bytes(int n_graphs);
GFM_API int gfm_radius_batch_overflow_index(int n_graphs);
GFM_API int gfm_radius_batch(const double* pos, const int* node_offsets, int n_graphs, int n_nodes,
                             int max_atoms, const double* cells, double rc, int max_nbr,
                             int* gnode, int* rowptr, int* col_src, int* edge_dst, void* edge_w,
                             void* edge_dx, int* csc_ptr, int* csc_eid, int* csc_dst, int e_cap,
                             void* workspace, int dtype, void* stream);

/* ---- K3/K4/K11: embedding and aggregation (model.py:293-341, 351-356) - */
/* h = emb[z - 1] (model.py:351) */
GFM_API int gfm_embed(const int* z, int n, const void* emb, int H, void* h, int dtype, void* stream);
/* number of column blocks for a parts mask */
GFM_API int gfm_agg_parts_count(int parts);
/* agg[N][K*H] = per-dst reduction of msg = h[src] * w over the CSR rows
 * (_aggregate, model.py:293-322; std/pna are extensions).  argmax [N][H]
 * (max part) holds the first CSR position attaining the max; stat_mean
 * [N][H] (std part) keeps the mean for the backward. */
GFM_API int gfm_agg_fwd(const void* h, int n_nodes, int H, const int* rowptr, const int* col_src,
                const void* edge_w, int parts, void* agg, int* argmax, void* stat_mean, int dtype,
                int flags, void* stream);
/* Backward as a CSC gather, no atomics (_aggregate_backward model.py:325-341
 * + np.add.at(dh_in, src, dmsg * w) model.py:561): dh holds dz W on entry;
 * out = (dh + gather) [* (1 - gate^2) when gate != NULL, model.py:553]. */
GFM_API size_t gfm_agg_bwd_workspace_bytes(int n_nodes, int H, int parts, int dtype);
GFM_API int gfm_agg_bwd(const void* dagg, const void* agg, const void* stat_mean, const int* argmax,
                const void* h_in, const int* rowptr, const int* csc_ptr, const int* csc_eid,
                const int* csc_dst, const void* edge_w, int n_nodes, int H, int parts, void* dh,
                const void* gate, void* out, void* workspace, int dtype, int flags, void* stream);

/* ---- K5/K9: dense layers (model.py:357-358, 365-372, 520-533, 549-558) */
/* Y = act([X1 | X2] [W1 | W2]^T + bias), act 0 = identity, 1 = tanh */
GFM_API int gfm_linear_fwd(const void* X1, int ld1, int K1, const void* X2, int ld2, int K2,
                   const void* W1, int ldw1, const void* W2, int ldw2, const void* bias, int M,
                   const int* M_dev, int N, int act, void* Y, int ldy, int dtype, void* stream);
/* [out1 | out2] = dY [W1 | W2]; with gate: out1 *= (1 - gate^2) */
GFM_API int gfm_linear_bwd_data(const void* dY, int ldd, int M, const int* M_dev, int N, const void* W1,
                        int ldw1, int K1, const void* W2, int ldw2, int K2, void* out1, int ldo1,
                        void* out2, int ldo2, const void* gate, int ldg, int dtype, void* stream);
/* Layer backward-data fused with the PNA (parts = 15) aggregation-backward
 * prep, float32 tensor-core engine only: dh_in = dz W; with dagg = dz U
 * (never stored) G = dsum + dmean/deg - coef*mean, coef = dstd/(deg*std),
 * dmax = the max part -- then gfm_agg_bwd(..., dagg = dmax, workspace =
 * [G | coef], GFM_FLAG_AGG_PREPPED).  G and coef are [N][H] at the head of
 * the gfm_agg_bwd workspace; `workspace` here holds U permuted channel-major
 * (gfm_layer_bwd_data_agg_workspace_bytes). */
GFM_API size_t gfm_layer_bwd_data_agg_workspace_bytes(int H);
GFM_API int gfm_layer_bwd_data_agg(const void* dz, int M, int H, const void* W, const void* U,
                                   const void* agg, const void* stat_mean, const int* rowptr,
                                   void* dh_in, void* G, void* coef, void* dmax, void* workspace,
                                   void* stream);
/* g1 = dY^T X1, g2 = dY^T X2, gb = colsum(dY): deterministic split-K.
 * with_bias: 0 = no gb; 1 = gb (the float32 tensor-core path writes a [M][4]
 * ones operand into the workspace); 2 = as 1 when this workspace already
 * holds that ones operand from an earlier call with the same M (skips it). */
GFM_API size_t gfm_linear_bwd_weight_workspace_bytes(int M, int N, int K1, int K2, int with_bias,
                                             int dtype);
GFM_API int gfm_linear_bwd_weight(const void* dY, int ldd, int M, const int* M_dev, int N,
                          const void* X1, int ld1, int K1, const void* X2, int ld2, int K2,
                          int with_bias, void* g1, void* g2, void* gb, void* workspace, int dtype,
                          void* stream);

/* ---- K7/K10: force head (model.py:377-389, 535-547) ------------------- */
/* Node-factored: the pair pre-activation (h[dst] + h[src]) V^T + c equals
 * P[dst] + P[src] + c with P = h V^T (written to caller-owned P [N][H] and
 * reused by the backward); then t = tanh(.), m = t.u and f[dst] += m dx over
 * the dst-CSR in one gather pass. */
GFM_API int gfm_force_fwd(const void* h, int H, int n_nodes, const int* rowptr,
                          const int* col_src, const void* edge_dx, const void* V, const void* c,
                          const void* u, void* P, void* f_pred, int dtype, int flags,
                          void* stream);
/* grads of V, c, u: with S[i] = sum of dpre over edges with dst i plus those
 * with src i, grad_V = S^T h and dh_final = dh_energy + S V; dz_out =
 * dh_final * (1 - h^2) (model.py:553) feeds the last message-passing layer. */
GFM_API size_t gfm_force_bwd_workspace_bytes(int H, int n_nodes, int dtype);
/* gfm_force_bwd in two stream-ordered halves sharing `workspace`: the edge
 * passes and grad_V / grad_c / grad_u (no dh_energy needed yet), then
 * dz_out = (dh_energy + S V) * (1 - h^2) -- so the energy-head backward
 * producing dh_energy can run concurrently with the first half. */
GFM_API int gfm_force_bwd_edges(const void* h, const void* P, int H, int n_nodes,
                                const int* rowptr, const int* col_src, const void* edge_dx,
                                const int* csc_ptr, const int* csc_eid, const int* csc_dst,
                                const void* V, const void* c, const void* u, const void* df,
                                void* grad_v, void* grad_c, void* grad_u, void* workspace,
                                int dtype, int flags, void* stream);
/* with grad_v == NULL, gfm_force_bwd_edges runs the edge passes only and
 * gfm_force_bwd_grads(…) then forms grad_V / grad_c / grad_u from the same
 * workspace (any stream ordered after the edge passes) */
GFM_API int gfm_force_bwd_grads(const void* h, int H, int n_nodes, void* grad_v, void* grad_c,
                                void* grad_u, void* workspace, int dtype, void* stream);
GFM_API int gfm_force_bwd_finish(const void* h, int H, int n_nodes, const void* V,
                                 const void* dh_energy, void* dz_out, void* workspace, int dtype,
                                 void* stream);
GFM_API int gfm_force_bwd(const void* h, const void* P, int H, int n_nodes, const int* rowptr,
                          const int* col_src, const void* edge_dx, const int* csc_ptr,
                          const int* csc_eid, const int* csc_dst, const void* V, const void* c,
                          const void* u, const void* df, const void* dh_energy, void* grad_v,
                          void* grad_c, void* grad_u, void* dz_out, void* workspace, int dtype,
                          int flags, void* stream);

/* ---- K6/K8: energy readout, loss, seeds (model.py:365-373, 437-462, 510-533) */
/* node_e = y a + c; e_pred = add.reduceat(node_e, node_offsets[:-1]) */
GFM_API int gfm_energy_readout(const void* y, int n_nodes, int G, const void* a, const void* c,
                       const int* node_offsets, int n_graphs, void* node_e, void* e_pred,
                       int dtype, void* stream);
/* loss = [total, energy_term, force_term]; de, df = backward seeds;
 * contrib (float32, optional) receives [total, 1.0] (train.py:257).
 * workspace (gfm_loss_workspace_bytes) must be ZERO-initialised once; the
 * kernel leaves it ready for the next call.  counts (device, optional) =
 * [B, N] true graph / node counts of a ragged batch held in n_graphs /
 * n_nodes capacity buffers: the means use the true counts and the capacity
 * tail gets zero seeds. */
GFM_API size_t gfm_loss_workspace_bytes(void);
GFM_API int gfm_loss_seeds(const void* e_pred, const void* e_true, const int* n_per, int n_graphs,
                   const void* f_pred, const void* f_true, int n_nodes, const int* counts,
                   double alpha_e, double alpha_f, void* loss, void* de, void* df,
                   float* contrib, void* workspace, int dtype, void* stream);
/* ds_i = de[g(i)]; dz = (ds_i a) * (1 - y^2)  (model.py:521-529).
 * ds is written as an [n_nodes][ld_ds] row-major column vector (column 0 =
 * ds, columns 1..ld_ds-1 = 0) so ld_ds = 4 keeps rows 16-byte aligned for the
 * TMA-fed weight-gradient GEMM that consumes it. */
GFM_API int gfm_energy_seed(const void* de, const int* gnode, int n_nodes, int G, const void* a,
                    const void* y, void* ds, int ld_ds, void* dz, int dtype, void* stream);

/* Deferred split-K: gfm_linear_bwd_weight without the final reduction; the
 * partials stay in `workspace` (which must then not be reused until reduced)
 * and `job` receives their descriptor.  gfm_splitk_reduce_batch reduces any
 * number of such jobs in one launch (fp64 sums in split order, fixed shape-
 * only grid: deterministic; float32 results equal the per-call reduction). */
typedef struct gfm_reduce_job {
  const void* ws;
  int splits, N, K1, K2, with_bias, trans;
  void* g1;
  void* g2;
  void* gb;
} gfm_reduce_job;
GFM_API int gfm_linear_bwd_weight_partials(const void* dY, int ldd, int M, const int* M_dev, int N,
                                           const void* X1, int ld1, int K1, const void* X2,
                                           int ld2, int K2, int with_bias, void* g1, void* g2,
                                           void* gb, void* workspace, gfm_reduce_job* job,
                                           int dtype, void* stream);
GFM_API int gfm_splitk_reduce_batch(const gfm_reduce_job* jobs, int n_jobs, int dtype, void* stream);

/* ---- K12: embedding gradient (model.py:564) --------------------------- */
/* grad[118][H] = onehot(z - 1)^T dh as a split-K GEMM (one-hot generated on
 * the fly, deterministic; absent elements exactly 0) */
GFM_API size_t gfm_embedding_grad_workspace_bytes(int n_nodes, int H, int dtype);
GFM_API int gfm_embedding_grad(const int* z, int n_nodes, const void* dh, int H, void* grad,
                       void* workspace, int dtype, void* stream);

/* ---- K13: optimiser and guard (train.py:96-108, 262-274) -------------- */
/* *flag |= any(!isfinite(v)) */
GFM_API int gfm_nonfinite_flag(const void* v, long long n, int dtype, int* flag, void* stream);
/* Adam on float64 master weights: grad = grad_sum / world; bias_corr (device)
 * = [1 - b1^t, 1 - b2^t]; skipped entirely when *skip_flag != 0; params32
 * (optional) receives the float32 working copy. */
GFM_API int gfm_adam_step(const void* grad_sum, int grad_dtype, long long n, double world, double* master,
                  double* m, double* v, const double* bias_corr, double lr, double beta1,
                  double beta2, double eps, const int* skip_flag, float* params32, void* stream);
/* device step counter: *step += 1, bias_corr = [1 - b1^step, 1 - b2^step]
 * (skipped when *skip_flag != 0) -- lets a CUDA-graph-captured step advance
 * Adam without host involvement.  bc_table (device, optional, [table_len][2])
 * holds the host-computed 1 - beta^t values (the reference's libm pow,
 * train.py:104-105); device pow is used only past its end.  bias_corr ==
 * NULL (SGD) advances the applied-step count only. */
GFM_API int gfm_adam_advance(long long* step, double beta1, double beta2, double* bias_corr,
                             const double* bc_table, long long table_len, const int* skip_flag,
                             void* stream);
/* gfm_nonfinite_flag + gfm_adam_advance in one launch: flag points at TWO
 * ints (flag[0] the non-finite flag, flag[1] a completion ticket that must
 * start at 0 and is left at 0); step / bias_corr are advanced after the
 * whole scan unless flag[0] is set (step == NULL: guard only) */
GFM_API int gfm_nonfinite_advance(const void* v, long long n, int dtype, int* flag,
                                  long long* step, double beta1, double beta2, double* bias_corr,
                                  const double* bc_table, long long table_len, void* stream);
GFM_API int gfm_sgd_step(const void* grad_sum, int grad_dtype, long long n, double world, double* master,
                 double lr, const int* skip_flag, float* params32, void* stream);
GFM_API int gfm_cast_f64_to_f32(const double* in, long long n, float* out, void* stream);

/* ---- C4: EGNN-style variant with autograd forces (oracle/egnn_oracle.py;
 * no reference implementation: SPEC.md:8, 352).  Reverse-over-forward
 * training: every "d" (tangent) pointer may be NULL for a primal-only call.
 * AB = h [wa; wb]^T ([n][2H] rows of stride ldab: A | B); x (n x 3).
 * Edge e = j -> i in CSR row i: m = tanh(A_i + B_j + wd |x_j - x_i|^2 + c),
 * agg_i = sum m, x'_i = x_i - sum (x_j - x_i)(m . ux) / max(deg_i, 1)
 * (coord_update != 0).  H in {32, 64, 128, 256, 512}. */
GFM_API int gfm_egnn_edge_fwd(const void* AB, int ldab, const void* ABd, const void* x,
                              const void* xd, int n_nodes, int H, const int* rowptr,
                              const int* col_src, const void* wd, const void* c, const void* ux,
                              int coord_update, void* agg, int ldg, void* aggd, void* x_out,
                              void* xd_out, int dtype, void* stream);
/* Edge adjoints: aggb/aggdb = dL/d agg (and tangent), xb_out/xdb_out =
 * dL/d x' (read when coord_update).  Writes dA at dAB and dB at dAB + H
 * (row stride ldd; tangent rows at dABd), per-edge dpre / dpredot (E x H,
 * CSR positions) and dr / drdot (E x 3) scratch, xb_in / xdb_in = dL/dx of
 * the layer input, part = per-node [d wd | d ux] partials (n x 2H).
 * Deterministic: dst sums in CSR order, src sums in CSC order. */
GFM_API int gfm_egnn_edge_bwd(const void* AB, int ldab, const void* ABd, const void* x,
                              const void* xd, int n_nodes, int H, const int* rowptr,
                              const int* col_src, const int* csc_ptr, const int* csc_eid,
                              const void* wd, const void* c, const void* ux, int coord_update,
                              const void* aggb, int ldgb, const void* aggdb, const void* xb_out,
                              const void* xdb_out, void* dAB, int ldd, void* dABd, void* preb,
                              void* predb, void* rb, void* rdb, void* xb_in, void* xdb_in,
                              void* part, int dtype, void* stream);
/* h = tanh(z + bias) (primal rows), hd = (1 - h^2) zd (tangent rows);
 * z == NULL: h is an input (tangent only) */
GFM_API int gfm_egnn_tanh_fwd(const void* z, const void* zd, int ldz, const void* bias, int n,
                              int H, void* h, void* hd, int ldh, int dtype, void* stream);
/* zb = (1 - h^2)(hb - 2 h zd hdb), zdb = (1 - h^2) hdb */
GFM_API int gfm_egnn_tanh_bwd(const void* h, int ldh, const void* zd, int ldzd, const void* hb,
                              const void* hdb, int ldhb, int n, int H, void* zb, void* zdb,
                              int ldzb, int dtype, void* stream);
/* node_e = y a + c (node_ed = yd a); e_pred / e_dot = per-graph sums */
GFM_API int gfm_egnn_energy(const void* y, const void* yd, int ldy, int n, int G, const void* a,
                            const void* c, const int* node_offsets, int n_graphs, void* node_e,
                            void* node_ed, void* e_pred, void* e_dot, int dtype, void* stream);
/* head seeds over `rows` (= n primal, or 2n with tangent) rows: s = de[g(i)]
 * (primal) or edot_seed (tangent), 0 for gnode < 0; ds = [s 0 0 0] rows,
 * yb = s a (row stride ldyb) */
GFM_API int gfm_egnn_head_seed(const void* de, const int* gnode, int n, int rows,
                               double edot_seed, const void* a, int G, void* ds, void* yb,
                               int ldyb, int dtype, void* stream);
/* out[c] (+)= sum_{r < rows} X[r][c] (row stride ld), fixed order (two
 * levels in one launch through a workspace of gfm_colsum_workspace_bytes:
 * float64 chunk partials, then per-slab tickets -- zero the workspace
 * before its first use; every call leaves the tickets at zero) */
GFM_API size_t gfm_colsum_workspace_bytes(int rows, int cols);
GFM_API int gfm_colsum(const void* X, int rows, int cols, int ld, void* out, int accumulate,
                       void* workspace, int dtype, void* stream);
/* y = alpha x */
GFM_API int gfm_scale(const void* x, long long n, double alpha, void* y, int dtype, void* stream);


/* ---- scoring and ensemble reductions (float64 in numpy's order) ------- */
/* evaluate's per-batch sums (train.py:178-183): acc[4] (device float64
 * [sum_e, n_graphs, sum_f, n_comp]) += [pairwise sum |(e - e_true) / n|, B,
 * pairwise sum |f - f_true| over 3N, 3N] */
GFM_API int gfm_eval_errors(const void* e_pred, const void* e_true, const int* n_per,
                            int n_graphs, const void* f_pred, const void* f_true, int n_nodes,
                            double* acc, int dtype, void* stream);
/* ensemble.py:121-130, 181: over the member axis of stack [K][n]: mean =
 * (sum in member order) / K, sigma = sqrt(sum (x - mean)^2 / K), 0 where the
 * members agree bitwise (mean / sigma may be NULL) */
GFM_API int gfm_member_stats(const void* stack, int n_members, long long n, void* mean,
                             void* sigma, int dtype, void* stream);
/* ensemble.py:133-148: per structure, the (n_g, 3) block of component
 * spreads -> how 0 max, 1 mean, 2 sqrt(mean of squares) */
GFM_API int gfm_force_sigma_reduce(const void* sigma_comp, const int* node_offsets, int n_graphs,
                                   int how, void* out, int dtype, void* stream);


/* ---- container ingest (records.py:126-183 payloads -> device arrays) --- */
/* one thread per payload (blob + offsets[r], lengths[r] bytes): header,
 * length and zlib CRC32 checks -> n_atoms[r], n_edges[r], status[r] (0 ok,
 * 1 truncated, 2 length mismatch, 3 checksum mismatch) */
GFM_API int gfm_record_scan(const void* blob, const long long* offsets, const long long* lengths,
                            int n_rec, int* n_atoms, int* n_edges, int* status, void* stream);
/* one warp per (checked) payload: z (int32), pos / forces (float64 [.,3]),
 * energy, record edges (int32 [.,2], record-local ids) at the records'
 * exclusive prefix sums atom_offsets / edge_offsets; deg (optional, zeroed
 * by the caller) += in-degree of every node (global ids); *bad (optional)
 * |= 1 when an edge endpoint is not below its record's atom count */
GFM_API int gfm_record_decode(const void* blob, const long long* offsets, int n_rec,
                              const long long* atom_offsets, const long long* edge_offsets, int* z,
                              double* pos, double* forces, double* energy, int* edges, int* deg,
                              int* bad, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* GFM_B200_H */
