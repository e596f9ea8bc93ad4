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
constexpr int NH_KB = 128;   // k-block (rows of dist staged per pass)
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
                               int64_t n, int64_t nkb, int64_t* __restrict__ seg, const int* __restrict__ only_if) {
  if (only_if && *only_if == 0) return;  // pruned path: only needed by the NaN-exact kernel
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
                    int32_t* __restrict__ next, int64_t ldn, const int* __restrict__ only_if) {
  // the exact NaN-aware kernel; with only_if != nullptr it runs only when the
  // fast kernel flagged a NaN among the dist values
  if (only_if && *only_if == 0) return;
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

// Packed CSC entry: one 16-byte (uniform, broadcast) load per entry.
struct alignas(16) NhEnt {
  double w;
  int32_t k;
  int32_t pad;
};

__global__ void csc_pack_kernel(const int32_t* __restrict__ idx, const double* __restrict__ val, int64_t nnz,
                                NhEnt* __restrict__ pk) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x)
    pk[e] = NhEnt{val[e], idx[e], 0};
}

// Fast variant: 64 targets per CTA (2 per lane, adjacent in shared memory ->
// one LDS.128), 8 source vertices per warp, one 16-byte uniform load per CSC
// entry feeding 64 (target, successor) scores. NaN scores are not tracked per
// entry: a NaN among the staged dist values raises *nan_flag and the exact
// NaN-aware kernel (next_hop_kernel) then recomputes the table.
constexpr int NP_T = 64;
constexpr int NP_COLS = 8;
constexpr int NP_WARPS = 8;
constexpr int NP_ST = NP_T + 2;  // 66 doubles: 16-byte aligned rows

__global__ void __launch_bounds__(NP_WARPS * 32)
    next_hop_pair_kernel(const int64_t* __restrict__ seg, const NhEnt* __restrict__ pk,
                         const double* __restrict__ dist, int64_t ldd, int64_t n, int64_t nkb,
                         const int32_t* __restrict__ targets, int64_t n_targets, int32_t* __restrict__ next,
                         int64_t ldn, int* __restrict__ nan_flag) {
  extern __shared__ __align__(16) double dsP[];  // [NH_KB][NP_ST]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t t0 = (int64_t)blockIdx.y * NP_T;
  const int64_t j0 = (int64_t)blockIdx.x * (NP_COLS * NP_WARPS) + warp * NP_COLS;
  double b0[NP_COLS], b1[NP_COLS];
  int32_t k0v[NP_COLS], k1v[NP_COLS];
#pragma unroll
  for (int c = 0; c < NP_COLS; ++c) {
    b0[c] = b1[c] = INFINITY;
    k0v[c] = k1v[c] = -1;
  }
  bool nan_here = false;
  for (int64_t kb = 0; kb < nkb; ++kb) {
    const int64_t k0 = kb * NH_KB;
    const int kl = (int)((n - k0) < NH_KB ? (n - k0) : NH_KB);
    // this warp's CSC entries of the k-block, first 32 per column, loaded
    // cooperatively (one 16-byte load per lane) before the staging barrier
    int64_t eb[NP_COLS];
    int cnt[NP_COLS];
    NhEnt ent[NP_COLS];
#pragma unroll
    for (int c = 0; c < NP_COLS; ++c) {
      const int64_t j = j0 + c;
      eb[c] = 0;
      cnt[c] = 0;
      if (j < n) {
        eb[c] = seg[j * (nkb + 1) + kb];
        cnt[c] = (int)(seg[j * (nkb + 1) + kb + 1] - eb[c]);
      }
      if (lane < cnt[c]) ent[c] = pk[eb[c] + lane];
    }
    __syncthreads();
    constexpr int SU = 4;  // staging loads in flight per thread
    for (int e0 = threadIdx.x; e0 < NP_T * NH_KB; e0 += SU * NP_WARPS * 32) {
      double v[SU];
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        const int e = e0 + u * NP_WARPS * 32;
        const int q = e / NH_KB, k = e - (e / NH_KB) * NH_KB;
        v[u] = (e < NP_T * NH_KB && t0 + q < n_targets && k < kl) ? dist[(t0 + q) * ldd + k0 + k] : INFINITY;
      }
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        const int e = e0 + u * NP_WARPS * 32;
        if (e < NP_T * NH_KB) {
          const int q = e / NH_KB, k = e - (e / NH_KB) * NH_KB;
          nan_here |= (v[u] != v[u]);
          dsP[k * NP_ST + q] = v[u];
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < NP_COLS; ++c) {
      for (int base = 0; base < cnt[c]; base += 32) {
        NhEnt cur = ent[c];
        if (base > 0 && lane < cnt[c] - base) cur = pk[eb[c] + base + lane];
        const int m = (cnt[c] - base) < 32 ? (cnt[c] - base) : 32;
        for (int i = 0; i < m; ++i) {
          const double w = __shfl_sync(0xffffffffu, cur.w, i);
          const int32_t k = __shfl_sync(0xffffffffu, cur.k, i);
          const double2 d = *reinterpret_cast<const double2*>(&dsP[(k - k0) * NP_ST + 2 * lane]);
          const double s0 = w + d.x, s1 = w + d.y;
          if (s0 < b0[c]) {
            b0[c] = s0;
            k0v[c] = k;
          }
          if (s1 < b1[c]) {
            b1[c] = s1;
            k1v[c] = k;
          }
        }
      }
    }
  }
  if (__any_sync(0xffffffffu, nan_here) && lane == 0) atomicOr(nan_flag, 1);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t r = t0 + 2 * lane + h;
    if (r >= n_targets) break;
    const int64_t t = targets[r];
#pragma unroll
    for (int c = 0; c < NP_COLS; ++c) {
      const int64_t j = j0 + c;
      if (j >= n) break;
      const double b = h ? b1[c] : b0[c];
      const int32_t kk = h ? k1v[c] : k0v[c];
      next[r * ldn + j] = ((t == j) || !(b < INFINITY)) ? -1 : kk;
    }
  }
}

// ---------------------------------------------------------------------------
// Pruned variant (n <= SORT_MAX + 1, i.e. every column fits the in-smem sort):
// each column's successors sorted by weight (ties by k). For a target t the
// remaining candidates of a column score at least w + Rmin[t], where w is the
// current (smallest remaining) weight and Rmin[t] = min over k != t of
// dist[t][k]; once fl(w + Rmin[t]) > best[t] for every target of the warp no
// later candidate can win or tie (rounding is monotonic), so the scan stops.
// The successor k == t (dist[t][t], outside Rmin) is scored up front. Ties are
// broken by the lower k, which reproduces the first minimum over ascending k.
// dist is read transposed (RT[k][r]): one 512-byte coalesced load per entry
// gives the 64 targets of a warp.
constexpr int SORT_MAX = 4096;

constexpr int PR_T = 64;      // targets per warp (2 per lane)
constexpr int PR_WARPS = 8;   // warps per CTA: 8 consecutive columns
constexpr int PR_COLS = 4;    // columns per warp, one after the other
constexpr int PR_G = 4;  // entries (RT rows) in flight per step (8 measured slower: later bound checks)

RDB_DEV uint64_t order_key(double w) {  // total order of doubles as unsigned integers
  const uint64_t b = (uint64_t)__double_as_longlong(w);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}

// one CTA per column: bitonic sort of (weight key, k) in shared memory
__global__ void __launch_bounds__(256) csc_sort_kernel(const int64_t* __restrict__ offs,
                                                       const int32_t* __restrict__ idx,
                                                       const double* __restrict__ val, int64_t n,
                                                       NhEnt* __restrict__ srt) {
  extern __shared__ unsigned long long sk[];  // [P] keys, then [P] k (as 64-bit for alignment)
  const int64_t j = blockIdx.x;
  const int64_t beg = offs[j * CSC_SPLIT], end = offs[(j + 1) * CSC_SPLIT];
  const int m = (int)(end - beg);
  if (m == 0) return;
  int P = 1;
  while (P < m) P <<= 1;
  unsigned long long* kk = sk + P;
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    if (i < m) {
      sk[i] = order_key(val[beg + i]);
      kk[i] = (unsigned long long)idx[beg + i];
    } else {
      sk[i] = ~0ULL;
      kk[i] = ~0ULL;
    }
  }
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int l = i ^ stride;
        if (l > i) {
          const bool up = (i & size) == 0;
          const bool gt = sk[i] > sk[l] || (sk[i] == sk[l] && kk[i] > kk[l]);
          if (gt == up) {
            const unsigned long long a = sk[i], b = kk[i];
            sk[i] = sk[l];
            kk[i] = kk[l];
            sk[l] = a;
            kk[l] = b;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const unsigned long long key = sk[i];  // order_key is a bijection: decode the weight exactly
    const unsigned long long b = (key >> 63) ? (key & 0x7FFFFFFFFFFFFFFFULL) : ~key;
    srt[beg + i] = NhEnt{__longlong_as_double((long long)b), (int32_t)kk[i], 0};
  }
}

// RT[k][r] = dist[r][k] (32 x 32 tiles through shared memory)
__global__ void transpose_kernel(const double* __restrict__ dist, int64_t ldd, int64_t rows, int64_t cols,
                                 double* __restrict__ rt) {
  __shared__ double tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = r0 + i, c = c0 + threadIdx.x;
    tile[i][threadIdx.x] = (r < rows && c < cols) ? dist[r * ldd + c] : 0.0;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (c < cols && r < rows) rt[c * rows + r] = tile[threadIdx.x][i];
  }
}

// Rmin[r] = min over k != targets[r] of dist[r][k]; any NaN in the row raises *nan_flag
__global__ void rmin_kernel(const double* __restrict__ dist, int64_t ldd, int64_t n, const int32_t* __restrict__ targets,
                            int64_t n_targets, double* __restrict__ rmin, int* __restrict__ nan_flag) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n_targets; r += nwarps) {
    const int64_t t = targets[r];
    double m = INFINITY;
    bool nan = false;
    for (int64_t k = lane; k < n; k += 32) {
      const double v = dist[r * ldd + k];
      nan |= (v != v);
      if (k != t) m = fmin(m, v);
    }
    for (int o = 16; o > 0; o >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (__any_sync(0xffffffffu, nan) && lane == 0) atomicOr(nan_flag, 1);
    if (lane == 0) rmin[r] = m;
  }
}

__global__ void __launch_bounds__(PR_WARPS * 32)
    next_hop_pruned_kernel(const int64_t* __restrict__ offs, const NhEnt* __restrict__ srt,
                           const double* __restrict__ w, int64_t ldw, const double* __restrict__ rt, int64_t n,
                           const int32_t* __restrict__ targets, int64_t n_targets, const double* __restrict__ rmin,
                           int32_t* __restrict__ next, int64_t ldn, const int* __restrict__ nan_flag) {
  if (*nan_flag) return;  // the exact kernel handles NaN semantics
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r0 = (int64_t)blockIdx.y * PR_T + 2 * lane;  // this lane's two target rows r0, r0 + 1
  const bool v0 = r0 < n_targets, v1 = r0 + 1 < n_targets;
  const int64_t t0 = v0 ? targets[r0] : -1, t1 = v1 ? targets[r0 + 1] : -1;
  const double m0 = v0 ? rmin[r0] : INFINITY, m1 = v1 ? rmin[r0 + 1] : INFINITY;
  const bool vec = !(n_targets & 1);  // RT rows 16-byte aligned: one double2 per entry
  for (int c = 0; c < PR_COLS; ++c) {
    const int64_t j = ((int64_t)blockIdx.x * PR_WARPS + warp) * PR_COLS + c;
    if (j >= n) break;
    // the successor k == t (if any) first: W[t][j] + dist[t][t]
    double b0 = INFINITY, b1 = INFINITY;
    int32_t k0 = -1, k1 = -1;
    if (v0 && t0 != j) {
      const double wt = w[t0 * ldw + j];
      if (fabs(wt) <= 1.7976931348623157e308) {
        b0 = wt + rt[t0 * n_targets + r0];
        k0 = (int32_t)t0;
      }
    }
    if (v1 && t1 != j) {
      const double wt = w[t1 * ldw + j];
      if (fabs(wt) <= 1.7976931348623157e308) {
        b1 = wt + rt[t1 * n_targets + r0 + 1];
        k1 = (int32_t)t1;
      }
    }
    const int64_t beg = offs[j * CSC_SPLIT], end = offs[(j + 1) * CSC_SPLIT];
    // entries 32 at a time (one coalesced load), broadcast by shuffles; RT
    // rows of 4 entries in flight per step; the bound is checked once per 4
    // (with the smallest weight of the group)
    bool stop = false;
    for (int64_t base = beg; base < end && !stop; base += 32) {
      const int cnt = (int)((end - base) < 32 ? (end - base) : 32);
      NhEnt mine;
      mine.w = INFINITY;
      mine.k = 0;
      if (lane < cnt) mine = srt[base + lane];
      for (int i0 = 0; i0 < cnt; i0 += PR_G) {
        const double wf = __shfl_sync(0xffffffffu, mine.w, i0);
        const bool done = !(wf + m0 <= b0) && !(wf + m1 <= b1);
        if (__all_sync(0xffffffffu, done)) {
          stop = true;
          break;
        }

        double we[PR_G];
        int32_t ke[PR_G];
        double2 d[PR_G];
#pragma unroll
        for (int u = 0; u < PR_G; ++u) {
          we[u] = __shfl_sync(0xffffffffu, mine.w, i0 + u);
          ke[u] = __shfl_sync(0xffffffffu, mine.k, i0 + u);
          const bool live = i0 + u < cnt;
          const int64_t kr = (int64_t)(live ? ke[u] : 0) * n_targets + r0;
          if (vec && v1) {
            d[u] = *reinterpret_cast<const double2*>(rt + kr);
          } else {
            d[u].x = v0 ? rt[kr] : INFINITY;
            d[u].y = v1 ? rt[kr + 1] : INFINITY;
          }
          if (!live) we[u] = INFINITY;
        }
#pragma unroll
        for (int u = 0; u < PR_G; ++u) {
          const int32_t k = ke[u];
          const double s0 = we[u] + d[u].x, s1 = we[u] + d[u].y;
          if (k != t0 && (s0 < b0 || (s0 == b0 && k < k0))) {
            b0 = s0;
            k0 = k;
          }
          if (k != t1 && (s1 < b1 || (s1 == b1 && k < k1))) {
            b1 = s1;
            k1 = k;
          }
        }
      }
    }
    if (v0) next[r0 * ldn + j] = ((t0 == j) || !(b0 < INFINITY)) ? -1 : k0;
    if (v1) next[(r0 + 1) * ldn + j] = ((t1 == j) || !(b1 < INFINITY)) ? -1 : k1;
  }
}

struct NhWork {
  int64_t* offs;  // n*CSC_SPLIT + 1
  int64_t* seg;   // n*(nkb+1)
  int32_t* idx;   // nnz
  double* val;    // nnz
  NhEnt* pk;      // nnz
  int* nan_flag;  // 1
  NhEnt* srt;     // nnz, weight-sorted columns (pruned path)
  double* rt;     // n x n_targets, dist transposed (pruned path)
  double* rmin;   // n_targets (pruned path)
};

static bool pruned_path(int64_t n) {
  const char* e = getenv("RDB_NEXT_HOP_PRUNED");  // A-B switch: 0 selects the unpruned pair kernel
  return n <= SORT_MAX + 1 && !(e && e[0] == '0');
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

static NhWork carve(void* work, int64_t n, int64_t nnz, int64_t n_targets) {
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
  p += align256((size_t)(nnz > 0 ? nnz : 1) * 4);
  w.pk = reinterpret_cast<NhEnt*>(p);
  p += align256((size_t)(nnz > 0 ? nnz : 1) * sizeof(NhEnt));
  w.nan_flag = reinterpret_cast<int*>(p);
  p += 256;
  w.srt = nullptr;
  w.rt = nullptr;
  w.rmin = nullptr;
  if (pruned_path(n)) {
    w.srt = reinterpret_cast<NhEnt*>(p);
    p += align256((size_t)(nnz > 0 ? nnz : 1) * sizeof(NhEnt));
    w.rt = reinterpret_cast<double*>(p);
    p += align256((size_t)(n * n_targets) * 8);
    w.rmin = reinterpret_cast<double*>(p);
  }
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

extern "C" size_t rdb_next_hop_workspace_bytes(int64_t n, int64_t nnz, int64_t n_targets) {
  if (n <= 0 || nnz < 0 || n_targets < 0) return 0;
  const int64_t nkb = (n + NH_KB - 1) / NH_KB;
  size_t b = align256((size_t)(n * CSC_SPLIT + 1) * 8) + align256((size_t)(n * (nkb + 1)) * 8) +
             align256((size_t)(nnz > 0 ? nnz : 1) * 8) + align256((size_t)(nnz > 0 ? nnz : 1) * 4) +
             align256((size_t)(nnz > 0 ? nnz : 1) * sizeof(NhEnt)) + 256;
  if (pruned_path(n))
    b += align256((size_t)(nnz > 0 ? nnz : 1) * sizeof(NhEnt)) + align256((size_t)(n * n_targets) * 8) +
         align256((size_t)(n_targets > 0 ? n_targets : 1) * 8);
  return b;
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
  NhWork wk = carve(work, n, nnz, n_targets);
  const dim3 cg((unsigned)((n + 31) / 32), CSC_SPLIT);
  csc_count_kernel<<<cg, 32, 0, st>>>(w, n, ldw, wk.offs);
  csc_scan_kernel<<<1, 1024, 0, st>>>(wk.offs, n * CSC_SPLIT);
  csc_fill_kernel<<<cg, 32, 0, st>>>(w, n, ldw, wk.offs, wk.idx, wk.val);
  if (cudaMemsetAsync(wk.nan_flag, 0, sizeof(int), st) != cudaSuccess) return RDB_ECUDA;
  if (wk.srt && n_targets <= 65535LL * PR_T) {
    // pruned path: weight-sorted columns, dist transposed, per-target lower bounds
    const int sort_smem = 2 * SORT_MAX * (int)sizeof(unsigned long long);
    static DeviceFlags attr;
    const int attr_dev = current_device();
    if (!attr.get(attr_dev)) {
      if (cudaFuncSetAttribute(csc_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sort_smem) !=
          cudaSuccess)
        return RDB_ECUDA;
      attr.set(attr_dev);
    }
    csc_sort_kernel<<<(unsigned)n, 256, sort_smem, st>>>(wk.offs, wk.idx, wk.val, n, wk.srt);
    transpose_kernel<<<dim3((unsigned)((n + 31) / 32), (unsigned)((n_targets + 31) / 32)), dim3(32, 8), 0, st>>>(
        dist, ldd, n_targets, n, wk.rt);
    rmin_kernel<<<(unsigned)((n_targets + 7) / 8), 256, 0, st>>>(dist, ldd, n, targets, n_targets, wk.rmin,
                                                                 wk.nan_flag);
    next_hop_pruned_kernel<<<dim3((unsigned)((n + PR_WARPS * PR_COLS - 1) / (PR_WARPS * PR_COLS)),
                                  (unsigned)((n_targets + PR_T - 1) / PR_T)),
                             PR_WARPS * 32, 0, st>>>(wk.offs, wk.srt, w, ldw, wk.rt, n, targets, n_targets,
                                                     wk.rmin, next, ldn, wk.nan_flag);
    csc_seg_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(wk.offs, wk.idx, n, nkb, wk.seg, wk.nan_flag);
  } else {
  csc_seg_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(wk.offs, wk.idx, n, nkb, wk.seg, nullptr);
  csc_pack_kernel<<<592, 256, 0, st>>>(wk.idx, wk.val, nnz, wk.pk);
  const int smem = NH_KB * NP_ST * (int)sizeof(double);
  if (cudaFuncSetAttribute(next_hop_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
      cudaSuccess)
    return RDB_ECUDA;
  next_hop_pair_kernel<<<dim3((unsigned)((n + NP_COLS * NP_WARPS - 1) / (NP_COLS * NP_WARPS)),
                              (unsigned)((n_targets + NP_T - 1) / NP_T)),
                         NP_WARPS * 32, smem, st>>>(wk.seg, wk.pk, dist, ldd, n, nkb, targets, n_targets, next,
                                                    ldn, wk.nan_flag);
  }
  // exact NaN semantics (numpy argmin picks the first NaN and the walk stops):
  // recompute only when a NaN was seen; otherwise every CTA exits at once
  const int smem_exact = NH_KB * NH_T * (int)sizeof(double);
  next_hop_kernel<<<dim3((unsigned)((n + NH_THREADS - 1) / NH_THREADS), (unsigned)((n_targets + NH_T - 1) / NH_T)),
                    NH_THREADS, smem_exact, st>>>(wk.seg, wk.idx, wk.val, dist, ldd, n, nkb, targets, n_targets,
                                                  next, ldn, wk.nan_flag);
  RDB_LAUNCH_CHECK();
  return RDB_OK;
}
