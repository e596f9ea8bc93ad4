// K6: greedy-descent next-hop table (reference: the step of
// pkg/src/rdist/navigation.py:62-69 applied to every (target, vertex) pair):
//   next[t][j] = argmin_{k in succ(j), ascending} W[k][j] + dist[t][k]
// first minimum on ties; -1 when j == t, j has no successor, or the best score
// is not finite (NaN scores stop the walk as numpy's argmin would pick them).
//
// W (dense, +inf = no edge) is compacted on the device into a CSC by source
// vertex j with ascending k (the successor order graphs.py:61-63 returns),
// segmented into k-blocks of NH_KB rows. The main kernel gives each thread one
// vertex j and NH_T targets: for every k-block, the NH_T dist rows are staged
// in shared memory and every (k, w) entry of column j is reused NH_T times.
// FP64 add/compare bound, not HBM bound.
#include <cmath>

#include "common.cuh"

namespace rdb {

constexpr int NH_T = 8;      // targets per CTA
constexpr int NH_KB = 1024;  // k-block (rows of dist staged per pass)
constexpr int NH_THREADS = 256;
constexpr int CSC_SPLIT = 8;  // row-range splits per column group when building the CSC

__global__ void count_edges_kernel(const double* __restrict__ w, int64_t n, int64_t ldw,
                                   unsigned long long* __restrict__ out) {
  unsigned cnt = 0;
  for (int64_t i = blockIdx.y; i < n; i += gridDim.y)
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x)
      cnt += (fabs(w[i * ldw + j]) <= 1.7976931348623157e308) ? 1u : 0u;
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(out, (unsigned long long)cnt);
}

// grid (ceil(n/32), CSC_SPLIT); warp 0 of each CTA: lane = column j0+lane,
// rows [split range). counts[(j * CSC_SPLIT) + split].
__global__ void csc_count_kernel(const double* __restrict__ w, int64_t n, int64_t ldw,
                                 int64_t* __restrict__ counts) {
  const int64_t j = (int64_t)blockIdx.x * 32 + threadIdx.x;
  const int64_t rows = (n + CSC_SPLIT - 1) / CSC_SPLIT;
  const int64_t r0 = blockIdx.y * rows, r1 = min(n, r0 + rows);
  int64_t c = 0;
  if (j < n)
    for (int64_t k = r0; k < r1; ++k) c += (fabs(w[k * ldw + j]) <= 1.7976931348623157e308);
  if (j < n) counts[j * CSC_SPLIT + blockIdx.y] = c;
}

// exclusive scan of counts (n * CSC_SPLIT entries) in one CTA; total -> ptr_end
__global__ void csc_scan_kernel(int64_t* __restrict__ counts, int64_t len) {
  __shared__ int64_t carry_s;
  __shared__ int64_t warp_sums[32];
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t base = 0; base < len; base += blockDim.x) {
    const int64_t idx = base + threadIdx.x;
    const int64_t x = idx < len ? counts[idx] : 0;
    int64_t incl = x;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) warp_sums[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      int64_t s = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
      }
      warp_sums[lane] = s;  // inclusive over warps
    }
    __syncthreads();
    const int64_t warp_off = wid ? warp_sums[wid - 1] : 0;
    const int64_t carry = carry_s;
    if (idx < len) counts[idx] = carry + warp_off + incl - x;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry_s = carry + warp_off + incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) counts[len] = carry_s;
}

__global__ void csc_fill_kernel(const double* __restrict__ w, int64_t n, int64_t ldw,
                                const int64_t* __restrict__ offs, int32_t* __restrict__ idx,
                                double* __restrict__ val) {
  const int64_t j = (int64_t)blockIdx.x * 32 + threadIdx.x;
  const int64_t rows = (n + CSC_SPLIT - 1) / CSC_SPLIT;
  const int64_t r0 = blockIdx.y * rows, r1 = min(n, r0 + rows);
  if (j >= n) return;
  int64_t o = offs[j * CSC_SPLIT + blockIdx.y];
  for (int64_t k = r0; k < r1; ++k) {
    const double x = w[k * ldw + j];
    if (fabs(x) <= 1.7976931348623157e308) {
      idx[o] = (int32_t)k;
      val[o] = x;
      ++o;
    }
  }
}

// seg[j * (nkb + 1) + q] = first entry of column j with k >= q * NH_KB
__global__ void csc_seg_kernel(const int64_t* __restrict__ offs, const int32_t* __restrict__ idx,
                               int64_t n, int64_t nkb, int64_t* __restrict__ seg) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int64_t beg = offs[j * CSC_SPLIT], end = offs[(j + 1) * CSC_SPLIT];
  int64_t e = beg;
  for (int64_t q = 0; q <= nkb; ++q) {
    const int64_t lim = q * NH_KB;
    while (e < end && idx[e] < lim) ++e;
    seg[j * (nkb + 1) + q] = e;
  }
}

__global__ void __launch_bounds__(NH_THREADS)
    next_hop_kernel(const int64_t* __restrict__ seg, const int32_t* __restrict__ idx,
                    const double* __restrict__ val, const double* __restrict__ dist, int64_t ldd,
                    int64_t n, int64_t nkb, const int32_t* __restrict__ targets, int64_t n_targets,
                    int32_t* __restrict__ next, int64_t ldn) {
  extern __shared__ double ds[];  // ds[k][q], NH_KB x NH_T
  const int64_t j = (int64_t)blockIdx.x * NH_THREADS + threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.y * NH_T;
  const int nq = (int)((n_targets - r0) < NH_T ? (n_targets - r0) : NH_T);
  double best[NH_T];
  int32_t bk[NH_T];
  bool nan_seen[NH_T];
#pragma unroll
  for (int q = 0; q < NH_T; ++q) {
    best[q] = INFINITY;
    bk[q] = -1;
    nan_seen[q] = false;
  }
  for (int64_t kb = 0; kb < nkb; ++kb) {
    const int64_t k0 = kb * NH_KB;
    const int kl = (int)((n - k0) < NH_KB ? (n - k0) : NH_KB);
    __syncthreads();
    for (int e = threadIdx.x; e < NH_KB * NH_T; e += NH_THREADS) {
      const int q = e / NH_KB, k = e % NH_KB;
      ds[k * NH_T + q] = (q < nq && k < kl) ? dist[(r0 + q) * ldd + k0 + k] : INFINITY;
    }
    __syncthreads();
    if (j < n) {
      const int64_t eb = seg[j * (nkb + 1) + kb], ee = seg[j * (nkb + 1) + kb + 1];
      for (int64_t e = eb; e < ee; ++e) {
        const int32_t k = idx[e];
        const double wv = val[e];
        const double* d = ds + (k - k0) * NH_T;
#pragma unroll
        for (int q = 0; q < NH_T; ++q) {
          const double s = wv + d[q];
          if (s < best[q]) {
            best[q] = s;
            bk[q] = k;
          }
          nan_seen[q] |= (s != s);
        }
      }
    }
  }
  if (j >= n) return;
#pragma unroll
  for (int q = 0; q < NH_T; ++q) {
    if (q < nq) {
      const int64_t t = targets[r0 + q];
      const bool stop = (t == j) || nan_seen[q] || !(best[q] < INFINITY);
      next[(r0 + q) * ldn + j] = stop ? -1 : bk[q];
    }
  }
}

struct NhWork {
  int64_t* offs;  // n*CSC_SPLIT + 1
  int64_t* seg;   // n*(nkb+1)
  int32_t* idx;   // nnz
  double* val;    // nnz
};

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

static NhWork carve(void* work, int64_t n, int64_t nnz) {
  const int64_t nkb = (n + NH_KB - 1) / NH_KB;
  char* p = static_cast<char*>(work);
  NhWork w;
  w.offs = reinterpret_cast<int64_t*>(p);
  p += align256((size_t)(n * CSC_SPLIT + 1) * 8);
  w.seg = reinterpret_cast<int64_t*>(p);
  p += align256((size_t)(n * (nkb + 1)) * 8);
  w.val = reinterpret_cast<double*>(p);
  p += align256((size_t)(nnz > 0 ? nnz : 1) * 8);
  w.idx = reinterpret_cast<int32_t*>(p);
  return w;
}

}  // namespace rdb

using namespace rdb;

extern "C" int rdb_count_edges(const double* w, int64_t n, int64_t ldw, unsigned long long* out_nnz,
                               void* stream) {
  if (!w || !out_nnz || n <= 0 || ldw < n) return RDB_EINVAL;
  int64_t gx = (n + 255) / 256, gy = n < 4096 ? n : 4096;
  count_edges_kernel<<<dim3((unsigned)gx, (unsigned)gy), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      w, n, ldw, out_nnz);
  RDB_LAUNCH_CHECK();
  return RDB_OK;
}

extern "C" size_t rdb_next_hop_workspace_bytes(int64_t n, int64_t nnz) {
  if (n <= 0 || nnz < 0) return 0;
  const int64_t nkb = (n + NH_KB - 1) / NH_KB;
  return align256((size_t)(n * CSC_SPLIT + 1) * 8) + align256((size_t)(n * (nkb + 1)) * 8) +
         align256((size_t)(nnz > 0 ? nnz : 1) * 8) + align256((size_t)(nnz > 0 ? nnz : 1) * 4);
}

extern "C" int rdb_next_hop(const double* w, int64_t ldw, const double* dist, int64_t ldd, int64_t n,
                            int64_t nnz, const int32_t* targets, int64_t n_targets, int32_t* next,
                            int64_t ldn, void* work, void* stream) {
  if (!w || !dist || !targets || !next || !work || n <= 0 || ldw < n || ldd < n || ldn < n ||
      n_targets <= 0 || nnz < 0 || n > 2147483647LL)
    return RDB_EINVAL;
  if ((n_targets + NH_T - 1) / NH_T > 65535) return RDB_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t nkb = (n + NH_KB - 1) / NH_KB;
  NhWork wk = carve(work, n, nnz);
  const dim3 cg((unsigned)((n + 31) / 32), CSC_SPLIT);
  csc_count_kernel<<<cg, 32, 0, st>>>(w, n, ldw, wk.offs);
  csc_scan_kernel<<<1, 1024, 0, st>>>(wk.offs, n * CSC_SPLIT);
  csc_fill_kernel<<<cg, 32, 0, st>>>(w, n, ldw, wk.offs, wk.idx, wk.val);
  csc_seg_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(wk.offs, wk.idx, n, nkb, wk.seg);
  const int smem = NH_KB * NH_T * (int)sizeof(double);
  if (cudaFuncSetAttribute(next_hop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
      cudaSuccess)
    return RDB_ECUDA;
  next_hop_kernel<<<dim3((unsigned)((n + NH_THREADS - 1) / NH_THREADS),
                         (unsigned)((n_targets + NH_T - 1) / NH_T)),
                    NH_THREADS, smem, st>>>(wk.seg, wk.idx, wk.val, dist, ldd, n, nkb, targets,
                                         n_targets, next, ldn);
  RDB_LAUNCH_CHECK();
  return RDB_OK;
}
