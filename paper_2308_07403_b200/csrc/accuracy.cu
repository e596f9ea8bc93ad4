// K9: the gamma sweep's accuracy counts on the device (reference:
// global_accuracy and local_accuracy, pkg/src/rdist/navigation.py:77-134, as
// _sweep_point calls them, experiments.py:138-167).
//
//  global: over ordered pairs i != j with exact[i][j] finite, count
//          estimate == exact (navigation.py:77-88).
//  local : over (goal t, node i) with i != t, exact[t][i] finite and i having
//          a successor, count predictions whose chosen successor j* (first
//          minimum of estimate[t][.] over successors, computed by K6 on the
//          zero-weight pattern) has a finite estimate and
//          exact[t][j*] <= min over successors of exact[t][.] + atol
//          (navigation.py:91-134).
#include "common.cuh"

namespace rdb {

__device__ __forceinline__ void warp_add(unsigned long long* out, unsigned long long v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(out, v);
}

__global__ void global_accuracy_kernel(const double* __restrict__ est, int64_t lde, const double* __restrict__ exact,
                                       int64_t ldx, int64_t n, unsigned long long* __restrict__ counts) {
  unsigned long long ev = 0, eq = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += stride) {
    const int64_t i = e / n, j = e - i * n;
    const double x = exact[i * ldx + j];
    if (i != j && isfinite(x)) {
      ++ev;
      eq += (est[i * lde + j] == x);
    }
  }
  warp_add(counts + 0, ev);
  warp_add(counts + 1, eq);
}

// has_succ[i] = any finite W[k][i], k != i (adj = isfinite(W), navigation.py:116-117)
__global__ void has_successor_kernel(const double* __restrict__ w, int64_t ldw, int64_t n,
                                     uint8_t* __restrict__ has_succ) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint8_t h = 0;
    for (int64_t k = 0; k < n && !h; ++k) h = (k != i) && isfinite(w[k * ldw + i]);
    has_succ[i] = h;
  }
}

__global__ void local_accuracy_kernel(const int32_t* __restrict__ next_est, const int32_t* __restrict__ next_exact,
                                      int64_t ldn, const double* __restrict__ est, int64_t lde,
                                      const double* __restrict__ exact, int64_t ldx,
                                      const int32_t* __restrict__ targets, int64_t n_targets, int64_t n,
                                      const uint8_t* __restrict__ has_succ, double atol,
                                      unsigned long long* __restrict__ counts) {
  unsigned long long ev = 0, ok = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n_targets * n; e += stride) {
    const int64_t r = e / n, i = e - r * n;
    const int64_t t = targets[r];
    const double* X = exact + t * ldx;
    if (i == t || !isfinite(X[i]) || !has_succ[i]) continue;
    ++ev;
    const int32_t js = next_est[r * ldn + i];
    const int32_t jb = next_exact[r * ldn + i];
    if (js >= 0 && isfinite(est[t * lde + js])) {
      const double best = jb >= 0 ? X[jb] : __longlong_as_double(0x7FF0000000000000LL);
      ok += (X[js] <= best + atol);
    }
  }
  warp_add(counts + 0, ev);
  warp_add(counts + 1, ok);
}

}  // namespace rdb

extern "C" int rdb_global_accuracy(const double* est, int64_t lde, const double* exact, int64_t ldx, int64_t n,
                                   unsigned long long* counts, void* stream) {
  if (!est || !exact || !counts || n <= 0 || lde < n || ldx < n) return RDB_EINVAL;
  const int64_t want = (n * n + 255) / 256;
  const unsigned blocks = (unsigned)(want < 148 * 8 ? want : 148 * 8);
  rdb::global_accuracy_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(est, lde, exact, ldx, n,
                                                                                       counts);
  RDB_LAUNCH_CHECK();
  return RDB_OK;
}

extern "C" int rdb_local_accuracy(const double* w, int64_t ldw, const int32_t* next_est,
                                  const int32_t* next_exact, int64_t ldn, const double* est, int64_t lde,
                                  const double* exact, int64_t ldx, const int32_t* targets, int64_t n_targets,
                                  int64_t n, double atol, void* work, unsigned long long* counts, void* stream) {
  if (!w || !next_est || !next_exact || !est || !exact || !targets || !work || !counts || n <= 0 ||
      n_targets <= 0 || ldw < n || ldn < n || lde < n || ldx < n)
    return RDB_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* has_succ = static_cast<uint8_t*>(work);
  rdb::has_successor_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(w, ldw, n, has_succ);
  RDB_LAUNCH_CHECK();
  const int64_t want = (n_targets * n + 255) / 256;
  const unsigned blocks = (unsigned)(want < 148 * 8 ? want : 148 * 8);
  rdb::local_accuracy_kernel<<<blocks, 256, 0, st>>>(next_est, next_exact, ldn, est, lde, exact, ldx, targets,
                                                     n_targets, n, has_succ, atol, counts);
  RDB_LAUNCH_CHECK();
  return RDB_OK;
}
