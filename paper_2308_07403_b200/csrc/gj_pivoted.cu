// Gauss-Jordan inversion with partial (row) pivoting, for generic matrices
// handed to lu_invert (reference: pkg/src/rdist/linalg.py:18-39, which uses
// LAPACK getrf/getrs with partial pivoting). Pivot choice follows idamax:
// the first row of maximal |a_ik| among the not-yet-eliminated rows.
//
// This is NOT the R-distance hot path (M = I - gamma^W is an M-matrix and
// goes through the no-pivot DMMA kernel); it serves matrices without the
// M-matrix certificate (generic lu_invert, gamma past the critical gain).
//
// n >= 256: blocked, NB = 128 column panels. Panel p (columns P):
//   1. piv_panel_kernel (cooperative, one grid sync per column): Gauss-Jordan
//      with partial pivoting restricted to the n x 128 panel, every row
//      eliminated (rows swapped inside the panel as they are chosen); the
//      panel becomes D = A_pp^-1 in the pivot rows and C_I = -A_Ip D elsewhere;
//   2. piv_laswp_kernel: the panel's 128 row swaps, in order, on every other column;
//   3. A_IJ += C_I A_pJ for all I, J outside the panel (DMMA engine, TMA reduce-add);
//   4. A_pJ = D A_pJ (DMMA engine, in place).
// The per-column search, swap and rank-1 arithmetic inside the panel are the
// unblocked kernel's; the other columns receive the panel's rank-1 updates
// aggregated into one rank-128 product (rounding order differs, pivots are the
// same unless two candidates tie within rounding). n < 256: the unblocked
// kernel below (per column: one CTA selects the pivot, swaps rows, scales the
// pivot row and saves the pivot column; a grid kernel applies the rank-1
// update). The column permutation is undone at the end.
#include <cooperative_groups.h>

#include <cmath>

#include "common.cuh"

extern "C" int rdb_gemm_local(const double* a, int64_t lda, const double* b, int64_t ldb, double* c, int64_t ldc,
                              int64_t m, int64_t n, int64_t k, int64_t skip_row_tile, int64_t skip_col_tile,
                              int64_t store_col_tile, int accumulate, int negate, int64_t max_ctas, void* stream);

namespace rdb {

constexpr int PIV_THREADS = 1024;

__global__ void __launch_bounds__(PIV_THREADS)
    piv_select_kernel(double* __restrict__ a, int64_t n, int64_t lda, int64_t k,
                      double* __restrict__ colbuf, int32_t* __restrict__ perm,
                      rdb_pivot_info* __restrict__ info) {
  __shared__ double sval[PIV_THREADS / 32];
  __shared__ int64_t sidx[PIV_THREADS / 32];
  __shared__ int64_t piv_s;
  const int tid = threadIdx.x;
  // argmax |a[i][k]| over i >= k, first index on ties
  double best = -1.0;
  int64_t bi = INT64_MAX;
  for (int64_t i = k + tid; i < n; i += PIV_THREADS) {
    const double v = fabs(a[i * lda + k]);
    if (v > best || (v == best && i < bi)) {
      best = v;
      bi = i;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) {
      best = ov;
      bi = oi;
    }
  }
  if ((tid & 31) == 0) {
    sval[tid >> 5] = best;
    sidx[tid >> 5] = bi;
  }
  __syncthreads();
  if (tid < 32) {
    best = sval[tid];
    bi = sidx[tid];
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) {
        best = ov;
        bi = oi;
      }
    }
    if (tid == 0) piv_s = (bi == INT64_MAX) ? k : bi;
  }
  __syncthreads();
  const int64_t piv = piv_s;
  if (piv != k) {
    for (int64_t j = tid; j < n; j += PIV_THREADS) {
      const double t0 = a[k * lda + j];
      a[k * lda + j] = a[piv * lda + j];
      a[piv * lda + j] = t0;
    }
  }
  __syncthreads();
  const double p = a[k * lda + k];
  const double pinv = 1.0 / p;
  for (int64_t i = tid; i < n; i += PIV_THREADS) colbuf[i] = a[i * lda + k];
  __syncthreads();
  for (int64_t j = tid; j < n; j += PIV_THREADS) a[k * lda + j] = (j == k) ? pinv : a[k * lda + j] * pinv;
  if (tid == 0) {
    colbuf[n] = pinv;
    perm[k] = (int32_t)piv;
    const double ap = fabs(p);
    if (k == 0) {
      info->min_pivot = ap;
      info->min_index = 0;
      info->flags = 0;
    } else if (ap < info->min_pivot) {
      info->min_pivot = ap;
      info->min_index = (int32_t)k;
    }
    if (!(ap < INFINITY)) info->flags |= RDB_PIV_NONFINITE;
    if (!(p > 0.0)) info->flags |= RDB_PIV_NONPOS;
  }
}

__global__ void piv_update_kernel(double* __restrict__ a, int64_t n, int64_t lda, int64_t k,
                                  const double* __restrict__ colbuf) {
  const double pinv = colbuf[n];
  for (int64_t i = blockIdx.y; i < n; i += gridDim.y) {
    if (i == k) continue;
    const double f = colbuf[i];
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x) {
      double* p = a + i * lda + j;
      *p = (j == k) ? -f * pinv : fma(-f, a[k * lda + j], *p);
    }
  }
}

// idx[j] = source column of result column j after undoing the swaps
__global__ void piv_compose_kernel(const int32_t* __restrict__ perm, int32_t* __restrict__ idx,
                                   int64_t n) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int64_t j = 0; j < n; ++j) idx[j] = (int32_t)j;
  for (int64_t k = n - 1; k >= 0; --k) {
    const int32_t q = perm[k];
    const int32_t t = idx[k];
    idx[k] = idx[q];
    idx[q] = t;
  }
}

__global__ void piv_gather_kernel(double* __restrict__ a, int64_t n, int64_t lda,
                                  const int32_t* __restrict__ idx) {
  extern __shared__ double row[];
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) row[j] = a[i * lda + j];
    __syncthreads();
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) a[i * lda + j] = row[idx[j]];
    __syncthreads();
  }
}

// ------------------------------------------------------------------ blocked (n >= 256)
namespace cg = cooperative_groups;
constexpr int PP_THREADS = 256, PNB = 128;

struct PanelArgs {
  double* a;
  int64_t lda, n_pad, n_real, p0;
  int32_t* perm;
  rdb_pivot_info* info;
  double* cval;    // [2][grid] candidate |value|
  int64_t* cidx;   // [2][grid] candidate row
  double* crow;    // [2][grid][PNB] candidate rows (panel part)
  double* krow;    // [2][PNB] row k before the step
};

RDB_DEV bool better(double v, int64_t i, double bv, int64_t bi) { return v > bv || (v == bv && i < bi); }

// Every CTA keeps its rows of the panel in shared memory for the panel's 128
// steps; only the candidate rows, row k and the candidates go through global
// memory (double-buffered by step parity), with one grid sync per column.
__global__ void __launch_bounds__(PP_THREADS) piv_panel_kernel(PanelArgs A) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double S[];  // [own rows][PNB]
  __shared__ double prow[PNB];
  __shared__ double sval[PP_THREADS / 32];
  __shared__ int64_t sidx[PP_THREADS / 32];
  __shared__ int64_t s_piv;
  __shared__ double s_pv;
  __shared__ int s_src;
  const int G = gridDim.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t rows_per = (A.n_pad + G - 1) / G;
  const int64_t r_lo = (int64_t)blockIdx.x * rows_per;
  const int64_t r_hi = r_lo + rows_per < A.n_pad ? r_lo + rows_per : A.n_pad;
  const int nr = (int)(r_hi > r_lo ? r_hi - r_lo : 0);
  double* P = A.a + A.p0;  // panel: P[i * lda + c]
  for (int e = tid; e < nr * (PNB / 2); e += PP_THREADS) {
    const int r = e / (PNB / 2), j2 = e - r * (PNB / 2);
    *reinterpret_cast<double2*>(S + r * PNB + 2 * j2) =
        *reinterpret_cast<const double2*>(P + (r_lo + r) * A.lda + 2 * j2);
  }
  __syncthreads();
  for (int c = 0; c < PNB; ++c) {
    const int64_t k = A.p0 + c;
    const int par = c & 1;
    // 1. local candidate: first max |S[i][c]| over own rows i >= k
    double bv = -1.0;
    int64_t bi = INT64_MAX;
    for (int64_t i = (r_lo > k ? r_lo : k) + tid; i < r_hi; i += PP_THREADS) {
      const double v = fabs(S[(i - r_lo) * PNB + c]);
      if (better(v, i, bv, bi)) {
        bv = v;
        bi = i;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (better(ov, oi, bv, bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      sval[w] = bv;
      sidx[w] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      for (int q = 1; q < PP_THREADS / 32; ++q)
        if (better(sval[q], sidx[q], sval[0], sidx[0])) {
          sval[0] = sval[q];
          sidx[0] = sidx[q];
        }
      A.cval[par * G + blockIdx.x] = sval[0];
      A.cidx[par * G + blockIdx.x] = sidx[0];
    }
    __syncthreads();
    const int64_t mine = sidx[0];
    // copies of the candidate row and of row k, immutable for this step
    if (mine != INT64_MAX)
      for (int j = tid; j < PNB; j += PP_THREADS)
        A.crow[((int64_t)par * G + blockIdx.x) * PNB + j] = S[(mine - r_lo) * PNB + j];
    if (k >= r_lo && k < r_hi)
      for (int j = tid; j < PNB; j += PP_THREADS) A.krow[par * PNB + j] = S[(k - r_lo) * PNB + j];
    grid.sync();
    // 2. the pivot (every CTA reduces the candidates identically)
    if (w == 0) {
      double v = -1.0;
      int64_t i = INT64_MAX;
      int src = 0;
      for (int q = lane; q < G; q += 32) {
        const double qv = A.cval[par * G + q];
        const int64_t qi = A.cidx[par * G + q];
        if (better(qv, qi, v, i)) {
          v = qv;
          i = qi;
          src = q;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int64_t oi = __shfl_xor_sync(0xffffffffu, i, o);
        const int os = __shfl_xor_sync(0xffffffffu, src, o);
        if (better(ov, oi, v, i)) {
          v = ov;
          i = oi;
          src = os;
        }
      }
      if (lane == 0) {
        s_piv = (i == INT64_MAX) ? k : i;
        s_pv = (i == INT64_MAX) ? A.krow[par * PNB + c] : A.crow[((int64_t)par * G + src) * PNB + c];
        s_src = src;
      }
    }
    __syncthreads();
    const int64_t piv = s_piv;
    const double pv = s_pv;
    const double pinv = 1.0 / pv;
    const double* prow_src = (piv == k) ? A.krow + par * PNB : A.crow + ((int64_t)par * G + s_src) * PNB;
    for (int j = tid; j < PNB; j += PP_THREADS) prow[j] = (j == c) ? pinv : prow_src[j] * pinv;
    if (blockIdx.x == 0 && tid == 0) {
      A.perm[k] = (int32_t)piv;
      if (k < A.n_real) {
        const double ap = fabs(pv);
        if (k == 0) {
          A.info->min_pivot = ap;
          A.info->min_index = 0;
          A.info->flags = 0;
        } else if (ap < A.info->min_pivot) {
          A.info->min_pivot = ap;
          A.info->min_index = (int32_t)k;
        }
        if (!(ap < INFINITY)) A.info->flags |= RDB_PIV_NONFINITE;
        if (!(pv > 0.0)) A.info->flags |= RDB_PIV_NONPOS;
      }
    }
    __syncthreads();
    // 3. own rows: row k <- scaled pivot row; row piv <- old row k, eliminated; others eliminated
    const double* krow = A.krow + par * PNB;
    for (int r = w; r < nr; r += PP_THREADS / 32) {
      const int64_t i = r_lo + r;
      double* row = S + r * PNB;
      if (i == k) {
        for (int j = lane; j < PNB; j += 32) row[j] = prow[j];
        continue;
      }
      const bool swapped = (i == piv);
      const double f = swapped ? krow[c] : row[c];
      __syncwarp();
      for (int j = lane; j < PNB; j += 32) {
        const double old = swapped ? krow[j] : row[j];
        row[j] = (j == c) ? -f * pinv : fma(-f, prow[j], old);
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < nr * (PNB / 2); e += PP_THREADS) {
    const int r = e / (PNB / 2), j2 = e - r * (PNB / 2);
    *reinterpret_cast<double2*>(P + (r_lo + r) * A.lda + 2 * j2) =
        *reinterpret_cast<const double2*>(S + r * PNB + 2 * j2);
  }
}

// The panel's row swaps, in order, on the columns outside [p0, p0 + 128).
__global__ void piv_laswp_kernel(double* __restrict__ a, int64_t lda, int64_t n_pad, int64_t p0,
                                 const int32_t* __restrict__ perm) {
  __shared__ int32_t sp[PNB];
  for (int q = threadIdx.x; q < PNB; q += blockDim.x) sp[q] = perm[p0 + q];
  __syncthreads();
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_pad - PNB;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = j < p0 ? j : j + PNB;
    for (int q = 0; q < PNB; ++q) {
      const int64_t k = p0 + q, r = sp[q];
      if (r != k) {
        const double t = a[k * lda + col];
        a[k * lda + col] = a[r * lda + col];
        a[r * lda + col] = t;
      }
    }
  }
}

static int invert_pivoted_blocked(double* a, int64_t n_pad, int64_t lda, int64_t n_real, char* ws, int32_t* perm,
                                  rdb_pivot_info* info, cudaStream_t st) {
  int dev = 0, sms = 148, per_sm = 1;
  if (cudaGetDevice(&dev) != cudaSuccess) return RDB_ECUDA;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, piv_panel_kernel, PP_THREADS, 0) != cudaSuccess)
    return RDB_ECUDA;
  // grid of the cooperative panel kernel: one CTA per SM (measured fastest:
  // the per-step row work, not the grid sync, dominates; RDB_PIV_GRID overrides)
  int64_t G = sms;
  if (G > n_pad) G = n_pad;
  if (G < 1) G = 1;
  if (const char* e = getenv("RDB_PIV_GRID")) {
    const int64_t v = atoll(e);
    if (v > 0) G = v < sms ? v : sms;
  }
  if (G > 160) G = 160;
  const size_t smem = (size_t)((n_pad + G - 1) / G) * PNB * sizeof(double);  // own panel rows
  if (smem > 200 * 1024) return RDB_EINVAL;
  if (cudaFuncSetAttribute(piv_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) != cudaSuccess)
    return RDB_ECUDA;
  PanelArgs pa;
  pa.a = a;
  pa.lda = lda;
  pa.n_pad = n_pad;
  pa.n_real = n_real;
  pa.perm = perm;
  pa.info = info;
  pa.cval = reinterpret_cast<double*>(ws);
  pa.cidx = reinterpret_cast<int64_t*>(pa.cval + 2 * 160);
  pa.crow = reinterpret_cast<double*>(pa.cidx + 2 * 160);
  pa.krow = pa.crow + 2 * 160 * PNB;
  const int nt = (int)(n_pad / PNB);
  for (int p = 0; p < nt; ++p) {
    pa.p0 = (int64_t)p * PNB;
    void* args[] = {&pa};
    if (cudaLaunchCooperativeKernel((void*)piv_panel_kernel, dim3((unsigned)G), dim3(PP_THREADS), args, smem, st) !=
        cudaSuccess)
      return RDB_ECUDA;
    if (nt > 1) {
      const int64_t cols = n_pad - PNB;
      const unsigned g = (unsigned)((cols + 255) / 256);
      piv_laswp_kernel<<<g, 256, 0, st>>>(a, lda, n_pad, pa.p0, perm);
      const double* panel = a + pa.p0;
      double* rowp = a + pa.p0 * lda;
      int rc = rdb_gemm_local(panel, lda, rowp, lda, a, lda, n_pad, n_pad, PNB, p, p, -1, 1, 0, 0, st);
      if (rc) return rc;
      rc = rdb_gemm_local(a + pa.p0 * lda + pa.p0, lda, rowp, lda, rowp, lda, PNB, n_pad, PNB, -1, p, -1, 0, 0, 0, st);
      if (rc) return rc;
    }
  }
  return RDB_OK;
}

}  // namespace rdb

using namespace rdb;

static int64_t pad128(int64_t n) { return (n + 127) / 128 * 128; }
constexpr int64_t kBlockedMin = 256;
static size_t blocked_small_bytes() { return (size_t)(2 * 160 * 8 + 2 * 160 * 8 + 2 * 160 * 128 * 8 + 2 * 128 * 8 + 256); }

extern "C" size_t rdb_invert_pivoted_workspace_bytes(int64_t n) {
  if (n <= 0) return 0;
  const size_t base = (size_t)(n + 2) * sizeof(double) + 2 * (size_t)(pad128(n) + 2) * sizeof(int32_t) + 64;
  if (n < kBlockedMin) return base;
  const int64_t np = pad128(n);
  return base + blocked_small_bytes() + (np != n ? (size_t)np * np * sizeof(double) + 256 : 0);
}

// identity-padded np x np copy of the n x n input (the blocked path's operand)
__global__ void piv_pad_kernel(const double* __restrict__ src, int64_t n, int64_t ld_src, double* __restrict__ dst,
                               int64_t np) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < np * np; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / np, j = e - i * np;
    dst[e] = (i < n && j < n) ? src[i * ld_src + j] : (i == j ? 1.0 : 0.0);
  }
}

// the leading n x n block of the padded inverse back into the caller's matrix
__global__ void piv_unpad_kernel(const double* __restrict__ src, int64_t np, double* __restrict__ dst, int64_t n,
                                 int64_t ld_dst) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e - i * n;
    dst[i * ld_dst + j] = src[i * np + j];
  }
}

extern "C" int rdb_invert_pivoted(double* a, int64_t n, int64_t lda, void* work,
                                  rdb_pivot_info* info, void* stream) {
  if (!a || !work || !info || n <= 0 || lda < n) return RDB_EINVAL;
  const int64_t np = n < kBlockedMin ? n : pad128(n);
  if ((size_t)np * sizeof(double) > 200 * 1024) return RDB_EINVAL;  // row staging in smem
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* colbuf = static_cast<double*>(work);
  int32_t* perm = reinterpret_cast<int32_t*>(colbuf + n + 2);
  int32_t* idx = perm + np + 2;
  if (n >= kBlockedMin) {
    char* ws = reinterpret_cast<char*>(((uintptr_t)(idx + np + 2) + 255) & ~(uintptr_t)255);
    double* m = a;
    int64_t ldm = lda;
    if (np != n || (lda & 1) || ((uintptr_t)a & 15)) {  // padded (identity) copy in the workspace
      m = reinterpret_cast<double*>(ws + blocked_small_bytes());
      m = reinterpret_cast<double*>(((uintptr_t)m + 255) & ~(uintptr_t)255);
      ldm = np;
      piv_pad_kernel<<<1184, 256, 0, st>>>(a, n, lda, m, np);
    }
    int rc = invert_pivoted_blocked(m, np, ldm, n, ws, perm, info, st);
    if (rc) return rc;
    piv_compose_kernel<<<1, 32, 0, st>>>(perm, idx, np);
    const size_t smem = (size_t)np * sizeof(double);
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(piv_gather_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return RDB_ECUDA;
    piv_gather_kernel<<<(unsigned)(np < 1024 ? np : 1024), 256, smem, st>>>(m, np, ldm, idx);
    if (m != a) piv_unpad_kernel<<<1184, 256, 0, st>>>(m, np, a, n, lda);
    RDB_LAUNCH_CHECK();
    return RDB_OK;
  }
  int64_t gx = (n + 255) / 256;
  int64_t gy = n < 2048 ? n : 2048;
  for (int64_t k = 0; k < n; ++k) {
    piv_select_kernel<<<1, PIV_THREADS, 0, st>>>(a, n, lda, k, colbuf, perm, info);
    piv_update_kernel<<<dim3((unsigned)gx, (unsigned)gy), 256, 0, st>>>(a, n, lda, k, colbuf);
  }
  piv_compose_kernel<<<1, 32, 0, st>>>(perm, idx, n);
  const size_t smem = (size_t)n * sizeof(double);
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(piv_gather_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess)
    return RDB_ECUDA;
  piv_gather_kernel<<<(unsigned)(n < 1024 ? n : 1024), 256, smem, st>>>(a, n, lda, idx);
  RDB_LAUNCH_CHECK();
  return RDB_OK;
}
