// Gauss-Jordan inversion with partial (row) pivoting, for generic matrices
// handed to lu_invert (reference: pkg/src/rdist/linalg.py:18-39, which uses
// LAPACK getrf/getrs with partial pivoting). Pivot choice follows idamax:
// the first row of maximal |a_ik| among the not-yet-eliminated rows.
//
// This is NOT the R-distance hot path (M = I - gamma^W is an M-matrix and
// goes through the no-pivot DMMA kernel); it serves matrices without the
// M-matrix certificate. Per column k: one CTA selects the pivot, swaps rows,
// scales the pivot row and saves the pivot column; a grid kernel applies the
// rank-1 update. The column permutation is undone at the end.
#include <cmath>

#include "common.cuh"

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

}  // namespace rdb

using namespace rdb;

extern "C" size_t rdb_invert_pivoted_workspace_bytes(int64_t n) {
  if (n <= 0) return 0;
  return (size_t)(n + 2) * sizeof(double) + 2 * (size_t)(n + 2) * sizeof(int32_t) + 64;
}

extern "C" int rdb_invert_pivoted(double* a, int64_t n, int64_t lda, void* work,
                                  rdb_pivot_info* info, void* stream) {
  if (!a || !work || !info || n <= 0 || lda < n) return RDB_EINVAL;
  if ((size_t)n * sizeof(double) > 200 * 1024) return RDB_EINVAL;  // row staging in smem
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* colbuf = static_cast<double*>(work);
  int32_t* perm = reinterpret_cast<int32_t*>(colbuf + n + 2);
  int32_t* idx = perm + n + 2;
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
