/* rdist_b200.h — C ABI of the B200-native R-distance hot path.
 *
 * The reference (`rdist`, a pure numpy/scipy package) has no FFI of its own:
 * its only native crossing is numpy ufuncs and scipy's LAPACK wrappers. Each
 * entry point below replaces one of those call sites; the reference
 * file:line it stands in for is given beside it (paths relative to the
 * reference's pkg/src/rdist/).
 *
 * Conventions (all entry points):
 *   - every pointer argument is a DEVICE pointer unless stated otherwise;
 *     buffers are caller-owned (the Python host layer passes torch tensors'
 *     data_ptr()), the library allocates nothing persistent;
 *   - matrices are row-major float64 with leading dimension `ld` (elements);
 *     element [i][j] follows the reference orientation: weight / distance of
 *     the edge or path j -> i (graphs.py:1-8);
 *   - batched calls take `batch` matrices `stride` elements apart;
 *   - `stream` is a cudaStream_t passed as void*; every call is asynchronous
 *     on it (numerical status is written to device memory and read by the
 *     caller after a stream sync);
 *   - return value: RDB_OK or an RDB_E* code (argument / launch errors only).
 */
#ifndef RDIST_B200_H
#define RDIST_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RDB_ABI_VERSION 6
#define RDB_NB 128 /* Gauss-Jordan panel width; inverted matrices are padded to a multiple */

/* status codes */
#define RDB_OK 0
#define RDB_EINVAL 1    /* bad argument (shape, alignment, null pointer) */
#define RDB_ESINGULAR 2 /* reserved for callers: pivot below PIVOT_RTOL*scale (linalg.py:33-38) */
#define RDB_ENOTM 3     /* reserved for callers: no-pivot elimination not certified */
#define RDB_ECUDA 4     /* CUDA launch / runtime error */

/* Per-matrix pivot record written by the inversion kernels.
 * min_pivot = min |U_kk| over all elimination steps, i.e. the quantity the
 * reference thresholds at linalg.py:33-34; flags report why the
 * no-pivot certificate failed. */
typedef struct rdb_pivot_info {
  double min_pivot;
  int32_t min_index;
  int32_t flags;
} rdb_pivot_info;
#define RDB_PIV_NONPOS 1    /* a pivot <= 0 appeared: not a nonsingular M-matrix */
#define RDB_PIV_NONFINITE 2 /* a pivot was inf/nan */

/* build modes for rdb_build_m */
#define RDB_BUILD_X 0 /* out = gamma^W              (resolvent.py:90-98, build_x) */
#define RDB_BUILD_M 1 /* out = I - gamma^W, identity in the padding (resolvent.py:114-115) */

/* rdb_log_ceil counters, per matrix */
#define RDB_CNT_NEGATIVE 0  /* entries below NEGATIVE_ENTRY_TOL (resolvent.py:120) */
#define RDB_CNT_UNDERFLOW 1 /* exact zeros at reachable off-diagonal pairs (resolvent.py:121-124) */
#define RDB_CNT_D8_RANGE 2  /* uint8 D only: finite D outside [0, RDB_D8_MAX] (or NaN) */
#define RDB_NCOUNTERS 3

/* compact uint8 D (rdb_log_ceil_d8): 0..RDB_D8_MAX exact, RDB_D8_UNREACHABLE = +inf */
#define RDB_D8_MAX 254
#define RDB_D8_UNREACHABLE 255

const char* rdb_strerror(int code);
int rdb_abi_version(void);
/* cudaGetErrorString of the last CUDA error an entry point returned RDB_ECUDA for (this thread). */
const char* rdb_last_cuda_error(void);

/* ---- K1: X = gamma^W or M = I - gamma^W -------------------------------
 * Replaces np.power(gamma, W) (resolvent.py:98) and np.eye(n) - x
 * (resolvent.py:115). W entries: +inf = no edge (gamma^inf = 0); W == 1.0
 * maps to gamma exactly (the bitwise identity test_resolvent.py:72-75
 * pins). Output is n_pad x n_pad; for RDB_BUILD_M rows/cols >= n are the
 * identity (so the padded inverse is [[M^-1, 0], [0, I]]). Per-matrix gains
 * come from `gammas` (device, `batch` entries) or, when it is NULL, from the
 * scalar `gamma`. */
int rdb_build_m(const double* w, int64_t ldw, int64_t stride_w, int64_t n, int64_t n_pad,
                int64_t batch, const double* gammas, double gamma, int mode, double* out,
                int64_t ldo, int64_t stride_o, void* stream);

/* Same, from bit-packed adjacency: bit (j % 32) of word bits[b][i][j / 32]
 * set <=> edge j -> i (an unweighted graph, W == 1). words_per_row =
 * (n + 31) / 32; a graph is n * words_per_row words. */
int rdb_build_m_bits(const uint32_t* bits, int64_t n, int64_t n_pad, int64_t batch,
                     const double* gammas, double gamma, double* out, int64_t ldo,
                     int64_t stride_o, void* stream);

/* Identity in rows/cols [n, n_pad) of each matrix (embeds a generic matrix
 * for rdb_invert), zeros elsewhere in the padding. */
int rdb_pad_identity(double* a, int64_t n, int64_t n_pad, int64_t lda, int64_t stride,
                     int64_t batch, void* stream);

/* Statistics the reference checks before factorising / iterating
 * (linalg.py:27-29, :64-65): stats[0] = max |a_ij| over finite entries (the
 * `scale`), stats[1] = number of non-finite entries, stats[2] = number of
 * entries violating the Z-matrix sign pattern (off-diagonal > 0 or diagonal
 * <= 0), stats[3] = number of negative entries. Counts are exact doubles.
 * `stats` (4 doubles) must be zeroed by the caller. */
int rdb_matrix_stats(const double* a, int64_t n, int64_t lda, double* stats, void* stream);

/* ---- K2: blocked Gauss-Jordan inversion, FP64 DMMA, no pivoting --------
 * Replaces scipy.linalg.lu_factor + lu_solve(I) (linalg.py:32, :39).
 * In place: a <- a^-1. n_pad must be a multiple of RDB_NB, lda even.
 * Valid without pivoting for nonsingular M-matrices (every M = I - gamma^W
 * with gamma below the critical gain); `info` (device, batch entries)
 * records min |pivot| and RDB_PIV_* flags so the caller can apply the
 * reference's singularity rule and fall back to rdb_invert_pivoted when the
 * certificate fails. `work` must hold rdb_invert_workspace_bytes(n_pad,
 * batch) bytes. */
size_t rdb_invert_workspace_bytes(int64_t n_pad, int64_t batch);
int rdb_invert_batched(double* a, int64_t n_pad, int64_t lda, int64_t stride, int64_t batch,
                       void* work, rdb_pivot_info* info, void* stream);
/* Batched calls (batch > 1, n_pad <= 64 * RDB_NB) skip the tiles of
 * structurally zero 128 x 128 blocks: a symbolic Gauss-Jordan on the block
 * pattern (fill A_IJ |= A_Ip & A_pJ) lists, per step, the row-panel tiles
 * with a non-zero A_pJ and the update tiles with non-zero A_Ip and A_pJ. A
 * skipped tile would only add an exact zero, so results equal the dense
 * schedule's (up to the sign of zero entries). rdb_invert_batched finds the
 * pattern by scanning the matrices; rdb_invert_batched_bits takes it from
 * the bit-packed adjacency the matrices were built from (rdb_build_m_bits
 * format, n vertices; the rdb_apsp_bits_batched pipelines do the same).
 * Environment RDB_GJ_SKIP=0 runs the dense schedule. */
int rdb_invert_batched_bits(double* a, int64_t n_pad, int64_t lda, int64_t stride, int64_t batch,
                            const uint32_t* bits, int64_t n, void* work, rdb_pivot_info* info,
                            void* stream);
int rdb_invert(double* a, int64_t n_pad, int64_t lda, void* work, rdb_pivot_info* info,
               void* stream);

/* Building blocks of the distributed (2D block-cyclic) inversion, where each
 * rank holds a local matrix of NB x NB tiles and receives the panels by NCCL
 * broadcast (paper_2308_07403_b200/distributed.py):
 *   rdb_gj_panel_inverse: D = A^-1 in place for one NB x NB block (P1); pivot
 *     record as rdb_invert (first != 0 resets it; p0 = the block's global
 *     index for min_index);
 *   rdb_gemm_local: C (m x n) op= (negate ? -1 : 1) * A (m x k) * B (k x n),
 *     A, B, C row-major, m, n multiples of NB and k of 16; op is += (TMA
 *     reduce-add) when accumulate != 0, else =; row tile skip_row_tile and
 *     column tile skip_col_tile are left untouched (-1: none); column tile
 *     store_col_tile is always stored (=); at most max_ctas persistent CTAs
 *     (0: one per SM), so a look-ahead can keep SMs free for the panel work
 *     and the NCCL kernels of the next step. Same DMMA engine as rdb_invert. */
int rdb_gj_panel_inverse(double* a, int64_t lda, rdb_pivot_info* info, int first, int64_t p0,
                         void* stream);
int rdb_gemm_local(const double* a, int64_t lda, const double* b, int64_t ldb, double* c, int64_t ldc,
                   int64_t m, int64_t n, int64_t k, int64_t skip_row_tile, int64_t skip_col_tile,
                   int64_t store_col_tile, int accumulate, int negate, int64_t max_ctas, void* stream);

/* Gauss-Jordan with partial (row) pivoting, first-max pivot choice as
 * LAPACK idamax; in place, any n. For generic matrices handed to
 * lu_invert (linalg.py:18-39) that carry no M-matrix certificate.
 * `work` must hold rdb_invert_pivoted_workspace_bytes(n) bytes. */
size_t rdb_invert_pivoted_workspace_bytes(int64_t n);
int rdb_invert_pivoted(double* a, int64_t n, int64_t lda, void* work, rdb_pivot_info* info,
                       void* stream);

/* ---- K3: R = log Y / log gamma, D = ceil R ------------------------------
 * Replaces r_distance (resolvent.py:131-143) and rounded_r_distance
 * (resolvent.py:146-153): y > 0 -> log(y)/log(gamma), else +inf; diagonal
 * forced 0; D = ceil(R) without nudge. Near-integer quotients are refined
 * in double-double so exact powers give exact integers (test_resolvent.py:
 * 137-148). Any of r_out (fp64 R), dceil_out (fp64 D, +inf sentinel) and
 * d32_out (int32 D, INT32_MAX sentinel) may be NULL; they share ldo /
 * stride_o. `counters` (device, batch*RDB_NCOUNTERS, caller-zeroed) may be
 * NULL; `reachable` (uint8 n x n, ldm, one mask shared by the batch) may be
 * NULL, in which case the underflow counter is not updated. */
int rdb_log_ceil(const double* y, int64_t n, int64_t ldy, int64_t stride_y, int64_t batch,
                 const double* gammas, double gamma, double* r_out, double* dceil_out,
                 int32_t* d32_out, int64_t ldo, int64_t stride_o, const uint8_t* reachable,
                 int64_t ldm, unsigned long long* counters, void* stream);

/* K3 with a compact uint8 D (batch serving: 1/4 of the int32 bytes over
 * PCIe). Same D as rdb_log_ceil wherever 0 <= D <= RDB_D8_MAX, unreachable
 * pairs RDB_D8_UNREACHABLE. Entries outside that range are counted in
 * counters[b * RDB_NCOUNTERS + RDB_CNT_D8_RANGE] (counters required,
 * caller-zeroed); a matrix with a non-zero count must be redone in int32. */
int rdb_log_ceil_d8(const double* y, int64_t n, int64_t ldy, int64_t stride_y, int64_t batch,
                    const double* gammas, double gamma, uint8_t* d8_out, int64_t ldo,
                    int64_t stride_o, unsigned long long* counters, void* stream);

/* K3 over a rows x cols block of a larger Y (e.g. sampled columns, or a rank's
 * block-cyclic tiles): local row i is global row row0 + i, local column j is
 * global column gcol[j] (device int64, or col0 + j when gcol is NULL); the
 * forced-zero diagonal is where the two coincide. Outputs as rdb_log_ceil. */
int rdb_log_ceil_block(const double* y, int64_t rows, int64_t cols, int64_t ldy, int64_t row0,
                       int64_t col0, const int64_t* gcol, double gamma, double* r_out,
                       double* dceil_out, int32_t* d32_out, int64_t ldo,
                       unsigned long long* counters, void* stream);

/* ---- K5: inversion residual max |M Y - I| (resolvent.py:125-127) --------
 * n_pad a multiple of RDB_NB; *out_max (device) must be zeroed by caller. */
int rdb_residual(const double* m, int64_t ldm, const double* y, int64_t ldy, int64_t n_pad,
                 double* out_max, void* stream);

/* ---- K4: power iteration (linalg.py:57-94) ------------------------------
 * On a non-negative n x n matrix, or (indicator != 0) on the 0/1 pattern
 * isfinite(m) — adjacency_indicator (graphs.py:114-116) of a weight matrix,
 * as critical_gain uses it (resolvent.py:156-165). Same start vector,
 * estimate and stopping rule as the reference. result (device, 3 doubles):
 * value, converged (0/1), iterations. work: rdb_power_workspace_bytes(n). */
size_t rdb_power_workspace_bytes(int64_t n);
int rdb_power_iteration(const double* m, int64_t n, int64_t ldm, int indicator, double tol,
                        int64_t max_iter, void* work, double* result, void* stream);

/* ---- K6: greedy-descent next hop (navigation.py:63-67) -----------------
 * For each target t = targets[r] (device int32, n_targets) and every vertex
 * j: next[r][j] = the successor k of j (W[k][j] finite, ascending k) that
 * minimises W[k][j] + dist[r][k], first minimum on ties; -1 when j == t,
 * when j has no successor, or when the best score is not finite (the
 * reference's stop conditions, navigation.py:62-69). W is n x n; dist holds
 * one row per target (row r = the distances to targets[r], ldd), so the
 * full n x n distance matrix with targets = 0..n-1 is the table case;
 * next is n_targets x n (ldn). work: rdb_next_hop_workspace_bytes(n, nnz,
 * n_targets) where nnz = number of finite off-diagonal W entries
 * (rdb_count_edges). For n <= 4097 the successors of each column are sorted
 * by weight and each scan stops once no remaining successor can reach the
 * best score (exact: see csrc/next_hop.cu); larger n scan every successor. */
int rdb_count_edges(const double* w, int64_t n, int64_t ldw, unsigned long long* out_nnz,
                    void* stream);
size_t rdb_next_hop_workspace_bytes(int64_t n, int64_t nnz, int64_t n_targets);
int rdb_next_hop(const double* w, int64_t ldw, const double* dist, int64_t ldd, int64_t n,
                 int64_t nnz, const int32_t* targets, int64_t n_targets, int32_t* next,
                 int64_t ldn, void* work, void* stream);

/* ---- batched APSP (the config-2 workload in one call) -------------------
 * bits -> M (K1) -> in-place inverse (K2) -> int32 D (K3) for `batch`
 * unweighted graphs of n vertices with per-graph gains. `mwork` holds
 * batch * n_pad * n_pad doubles, `work` rdb_invert_workspace_bytes(n_pad,
 * batch) bytes; d32 is batch x n x n (ld n). */
int rdb_apsp_bits_batched(const uint32_t* bits, int64_t n, int64_t batch, const double* gammas,
                          double* mwork, void* work, rdb_pivot_info* info, int32_t* d32,
                          unsigned long long* counters, void* stream);

/* The same with uint8 D (rdb_log_ceil_d8 semantics; counters required). */
int rdb_apsp_bits_batched_d8(const uint32_t* bits, int64_t n, int64_t batch, const double* gammas,
                             double* mwork, void* work, rdb_pivot_info* info, uint8_t* d8,
                             unsigned long long* counters, void* stream);

/* Edge list (device int32 from/to, m edges; the caller has checked 0 <= id < n,
 * no self-loops, no duplicates as graph_from_edge_list does) -> bit-packed
 * adjacency, bit `from` of row `to` (the rdb_build_m_bits input format).
 * Zeroes `bits` (n x ceil(n/32) words) first. */
int rdb_edges_to_bits(const int32_t* src, const int32_t* dst, int64_t m, int64_t n, uint32_t* bits,
                      void* stream);

/* ---- K8: exact hop distances by all-source BFS (oracles.py:22-41) -------
 * Unweighted digraph in the rdb_build_m_bits row format (row i, bit j <=>
 * edge j -> i). dist[i][j] = hops from j to i, 0 on the diagonal,
 * unreachable INT32_MAX (dist_i32) or +inf (dist_f64): exactly one of the two
 * outputs is non-NULL. work: rdb_bfs_workspace_bytes(n). Synchronises the
 * stream once per level (early exit); *levels (host, may be NULL) receives
 * the deepest level reached. Replaces the reference's dense boolean matrix
 * products with a sparse-row x bit-matrix product per level. */
size_t rdb_bfs_workspace_bytes(int64_t n);
/* bit-packed adjacency pattern of a weight matrix (bit j of row i <=> W[i][j]
 * finite, i != j; adjacency_indicator, graphs.py:114-116); bits: n x ceil(n/32). */
int rdb_pattern_bits(const double* w, int64_t n, int64_t ldw, uint32_t* bits, void* stream);
int rdb_bfs_apsp(const uint32_t* bits, int64_t n, int32_t* dist_i32, double* dist_f64, int64_t ldd,
                 void* work, int64_t* levels, void* stream);

/* ---- K10: Floyd-Warshall exact weighted distances (oracles.py:44-50) ----
 * d (n x n, ldd) = W with a zero diagonal, then for k = 0..n-1:
 * d = min(d, d[:, k] + d[k, :]) — bit for bit the reference's loop (k-blocks
 * of 32 replay column / row k as they stood after step k-1). W: device fp64,
 * +inf = no edge, positive weights. work: rdb_floyd_workspace_bytes(n). */
size_t rdb_floyd_workspace_bytes(int64_t n);
int rdb_floyd_warshall(const double* w, int64_t ldw, int64_t n, double* d, int64_t ldd, void* work,
                       void* stream);

/* ---- K9: gamma-sweep accuracy counts (navigation.py:77-134) --------------
 * counts (device, 2 x u64, caller-zeroed, accumulated): {evaluated, hits}.
 * global: pairs i != j with finite exact; hit when est == exact
 * (global_accuracy, navigation.py:77-88).
 * local: (target t = targets[r], node i) with i != t, finite exact[t][i]
 * and a successor (finite W[k][i], k != i); hit when the estimate's chosen
 * successor j* = next_est[r][i] (K6 on the zero-weight pattern) has a
 * finite est[t][j*] and exact[t][j*] <= exact[t][next_exact[r][i]] + atol
 * (local_accuracy, navigation.py:91-134). est and exact are full n x n
 * matrices (row = target id); next_* have one row per target. work: n bytes. */
int rdb_global_accuracy(const double* est, int64_t lde, const double* exact, int64_t ldx, int64_t n,
                        unsigned long long* counts, void* stream);
int rdb_local_accuracy(const double* w, int64_t ldw, const int32_t* next_est, const int32_t* next_exact,
                       int64_t ldn, const double* est, int64_t lde, const double* exact, int64_t ldx,
                       const int32_t* targets, int64_t n_targets, int64_t n, double atol, void* work,
                       unsigned long long* counts, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RDIST_B200_H */
