// K4: power iteration for the dominant eigenvalue of a non-negative matrix,
// entirely on the device (one cooperative launch, grid-wide syncs between
// the GEMV and the normalisation). HBM-bound: 8 n^2 bytes per iteration.
//
// Follows pkg/src/rdist/linalg.py:57-94 step for step: v0 = ones/sqrt(n);
// w = m v; ratio = ||w||; ratio == 0 -> (0, converged); estimate = ratio on
// the first step, else sqrt(ratio * previous ratio); stop when successive
// estimates differ by < tol; else v = w / ratio; (est, False, max_iter) when
// the budget runs out. With indicator != 0 the matrix is isfinite(m) as
// 0/1, i.e. adjacency_indicator(g) (graphs.py:114-116) read straight from
// the weight matrix, as critical_gain needs it (resolvent.py:156-165).
#include <cooperative_groups.h>

#include <cmath>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace rdb {

constexpr int PI_THREADS = 512;

// matrix element as the GEMV reads it: the value, or isfinite(a) as 0/1
RDB_DEV double elem(double a, int indicator) {
  return indicator ? ((fabs(a) <= 1.7976931348623157e308) ? 1.0 : 0.0) : a;
}

__global__ void __launch_bounds__(PI_THREADS, 2)
    power_kernel(const double* __restrict__ m, int64_t n, int64_t ldm, int indicator, double tol,
                 int64_t max_iter, double* __restrict__ v, double* __restrict__ w,
                 double* __restrict__ partial, double* __restrict__ result) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[PI_THREADS / 32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t gwarp = (int64_t)blockIdx.x * (PI_THREADS / 32) + wib;
  const int64_t nwarps = (int64_t)gridDim.x * (PI_THREADS / 32);
  const int64_t gtid = (int64_t)blockIdx.x * PI_THREADS + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * PI_THREADS;

  // 16-byte row loads when every row start is 16-byte aligned (v is: workspace start)
  const bool vec = !(ldm & 1) && !((uintptr_t)m & 15);
  const int64_t n2 = n & ~(int64_t)1;
  const double v0 = 1.0 / sqrt((double)n);
  for (int64_t i = gtid; i < n; i += nthreads) v[i] = v0;
  grid.sync();

  bool have_prev = false;
  double prev_ratio = 0.0, prev_est = 0.0, est = 0.0;
  for (int64_t it = 1; it <= max_iter; ++it) {
    double sq = 0.0;
    for (int64_t i = gwarp; i < n; i += nwarps) {
      const double* row = m + i * ldm;
      double s = 0.0;
      if (vec) {
        // lane owns columns 2 lane + 64 k (16-byte loads), four loads in flight
        double s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int64_t j = 2 * lane;
        for (; j + 192 < n2; j += 256) {
          double2 a[4], x[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) a[u] = __ldcs(reinterpret_cast<const double2*>(row + j + 64 * u));
#pragma unroll
          for (int u = 0; u < 4; ++u) x[u] = *reinterpret_cast<const double2*>(v + j + 64 * u);
          s = fma(elem(a[0].x, indicator), x[0].x, fma(elem(a[0].y, indicator), x[0].y, s));
          s1 = fma(elem(a[1].x, indicator), x[1].x, fma(elem(a[1].y, indicator), x[1].y, s1));
          s2 = fma(elem(a[2].x, indicator), x[2].x, fma(elem(a[2].y, indicator), x[2].y, s2));
          s3 = fma(elem(a[3].x, indicator), x[3].x, fma(elem(a[3].y, indicator), x[3].y, s3));
        }
        for (; j < n2; j += 64) {
          const double2 a = __ldcs(reinterpret_cast<const double2*>(row + j));
          const double2 x = *reinterpret_cast<const double2*>(v + j);
          s = fma(elem(a.x, indicator), x.x, fma(elem(a.y, indicator), x.y, s));
        }
        s = (s + s1) + (s2 + s3);
        if (lane == 0 && n2 < n) s = fma(elem(row[n2], indicator), v[n2], s);
      } else {
        for (int64_t j = lane; j < n; j += 32) s = fma(elem(row[j], indicator), v[j], s);
      }
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) {
        w[i] = s;
        sq = fma(s, s, sq);
      }
    }
    if (lane == 0) red[wib] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int q = 0; q < PI_THREADS / 32; ++q) t += red[q];
      partial[blockIdx.x] = t;
    }
    grid.sync();
    // every thread reduces the per-block partials in the same order -> same ratio everywhere
    double tot = 0.0;
    for (int q = 0; q < (int)gridDim.x; ++q) tot += partial[q];
    const double ratio = sqrt(tot);
    if (ratio == 0.0) {
      if (gtid == 0) {
        result[0] = 0.0;
        result[1] = 1.0;
        result[2] = (double)it;
      }
      return;
    }
    est = have_prev ? sqrt(ratio * prev_ratio) : ratio;
    if (have_prev && fabs(est - prev_est) < tol) {
      if (gtid == 0) {
        result[0] = est;
        result[1] = 1.0;
        result[2] = (double)it;
      }
      return;
    }
    have_prev = true;
    prev_ratio = ratio;
    prev_est = est;
    for (int64_t i = gtid; i < n; i += nthreads) v[i] = w[i] / ratio;
    grid.sync();
  }
  if (gtid == 0) {
    result[0] = est;
    result[1] = 0.0;
    result[2] = (double)max_iter;
  }
}

}  // namespace rdb

using namespace rdb;

extern "C" size_t rdb_power_workspace_bytes(int64_t n) {
  if (n <= 0) return 0;
  return (size_t)(2 * n + 8192) * sizeof(double);
}

extern "C" int rdb_power_iteration(const double* m, int64_t n, int64_t ldm, int indicator, double tol,
                                   int64_t max_iter, void* work, double* result, void* stream) {
  if (!m || !work || !result || n <= 0 || ldm < n || max_iter < 0 || !(tol > 0.0))
    return RDB_EINVAL;
  int dev = 0, sms = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return RDB_ECUDA;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return RDB_ECUDA;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, power_kernel, PI_THREADS, 0) !=
      cudaSuccess)
    return RDB_ECUDA;
  int blocks = sms * (per_sm < 2 ? per_sm : 2);
  const int64_t need = (n + PI_THREADS / 32 - 1) / (PI_THREADS / 32);
  if (blocks > need) blocks = (int)need;
  if (blocks < 1) blocks = 1;
  double* v = static_cast<double*>(work);
  double* w = v + n;
  double* partial = w + n;
  int64_t nn = n, ld = ldm, mi = max_iter;
  int ind = indicator;
  double tl = tol;
  void* args[] = {(void*)&m, &nn, &ld, &ind, &tl, &mi, &v, &w, &partial, &result};
  if (cudaLaunchCooperativeKernel((const void*)power_kernel, dim3(blocks), dim3(PI_THREADS), args, 0,
                                  static_cast<cudaStream_t>(stream)) != cudaSuccess)
    return RDB_ECUDA;
  return RDB_OK;
}
