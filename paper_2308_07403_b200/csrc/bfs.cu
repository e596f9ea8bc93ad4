// K8: exact all-pairs hop distances of an unweighted digraph by breadth-first
// search from every source at once (reference: bfs_apsp,
// pkg/src/rdist/oracles.py:22-41 — level-synchronous frontiers advanced with
// boolean matrix products). Used as the exact side of the gamma sweep's
// accuracy counts (experiments.py:138-211) and to verify D at sizes the CPU
// oracle cannot reach.
//
// Layout: the adjacency is the bit-packed row format of rdb_build_m_bits
// (row i, bit j set <=> edge j -> i). Frontier F, visited V: n rows x W words,
// bit j of row i = "source j reaches i". One level:
//     F'[i] = (OR over in-neighbours p of i of F[p]) & ~V[i];  V[i] |= F'[i]
// i.e. a sparse-row x bit-matrix product: row i ORs indeg(i) rows of F, read
// 128 bytes per warp instruction. Each new bit (i, j) writes dist[i][j] = level.
#include <algorithm>
#include <utility>

#include "common.cuh"

namespace rdb {
namespace bfs {

constexpr int SEGW = 8;  // words per lane per pass: a pass covers 32 * 8 words = 8192 sources

template <class T>
RDB_DEV T unreachable();
template <>
RDB_DEV int32_t unreachable<int32_t>() {
  return INT32_MAX;
}
template <>
RDB_DEV double unreachable<double>() {
  return __longlong_as_double(0x7FF0000000000000LL);
}

// F = V = identity, dist = 0 on the diagonal, unreachable elsewhere.
template <class T>
__global__ void init_kernel(int64_t n, int64_t W, uint32_t* __restrict__ F, uint32_t* __restrict__ V,
                            T* __restrict__ dist, int64_t ldd) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * W; e += stride) {
    const int64_t i = e / W, w = e - i * W;
    const uint32_t v = (i >> 5) == w ? (1u << (i & 31)) : 0u;
    F[e] = v;
    V[e] = v;
  }
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += stride) {
    const int64_t i = e / n, j = e - i * n;
    dist[i * ldd + j] = (i == j) ? T(0) : unreachable<T>();
  }
}

// One level. One warp per row i (grid-stride); lanes own words seg + lane + 32q.
template <class T>
__global__ void __launch_bounds__(256) level_kernel(const uint32_t* __restrict__ adj, int64_t n, int64_t W,
                                                    const uint32_t* __restrict__ F, uint32_t* __restrict__ Fn,
                                                    uint32_t* __restrict__ V, T* __restrict__ dist, int64_t ldd,
                                                    int level, int* __restrict__ grew) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  bool any = false;
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += nwarps) {
    const uint32_t* arow = adj + i * W;
    for (int64_t seg = 0; seg < W; seg += 32 * SEGW) {
      uint32_t acc[SEGW];
#pragma unroll
      for (int q = 0; q < SEGW; ++q) acc[q] = 0u;
      // in-neighbours p of i: scan the adjacency row 32 words at a time
      for (int64_t a0 = 0; a0 < W; a0 += 32) {
        const uint32_t mine = (a0 + lane < W) ? __ldg(arow + a0 + lane) : 0u;
        uint32_t live = __ballot_sync(0xffffffffu, mine != 0u);
        while (live) {
          const int src = __ffs(live) - 1;
          live &= live - 1;
          uint32_t word = __shfl_sync(0xffffffffu, mine, src);
          while (word) {
            const int b = __ffs(word) - 1;
            word &= word - 1;
            const uint32_t* frow = F + (32 * (a0 + src) + b) * W + seg + lane;
#pragma unroll
            for (int q = 0; q < SEGW; ++q)
              if (seg + lane + 32 * q < W) acc[q] |= __ldg(frow + 32 * q);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < SEGW; ++q) {
        const int64_t w = seg + lane + 32 * q;
        if (w < W) {
          const uint32_t vis = V[i * W + w];
          uint32_t fresh = acc[q] & ~vis;
          Fn[i * W + w] = fresh;
          if (fresh) {
            any = true;
            V[i * W + w] = vis | fresh;
            T* drow = dist + i * ldd + 32 * w;
            while (fresh) {
              const int b = __ffs(fresh) - 1;
              fresh &= fresh - 1;
              drow[b] = T(level);
            }
          }
        }
      }
    }
  }
  if (__any_sync(0xffffffffu, any) && lane == 0) *grew = 1;
}

// Adjacency pattern of a weight matrix in the bit-packed row format:
// bit j of row i <=> W[i][j] finite, i != j (adjacency_indicator, graphs.py:114-116).
__global__ void pattern_bits_kernel(const double* __restrict__ w, int64_t n, int64_t ldw, uint32_t* __restrict__ bits) {
  const int lane = threadIdx.x & 31;
  const int64_t W = (n + 31) / 32;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t e = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); e < n * W; e += nwarps) {
    const int64_t i = e / W, wd = e - i * W;
    const int64_t j = 32 * wd + lane;
    const bool on = j < n && j != i && isfinite(w[i * ldw + j]);
    const uint32_t word = __ballot_sync(0xffffffffu, on);
    if (lane == 0) bits[e] = word;
  }
}

size_t workspace_bytes(int64_t n) {
  if (n <= 0) return 0;
  const int64_t W = (n + 31) / 32;
  return (size_t)(3 * n * W * sizeof(uint32_t) + 256);
}

template <class T>
int run(const uint32_t* adj, int64_t n, T* dist, int64_t ldd, void* work, int64_t* levels_out, cudaStream_t st) {
  const int64_t W = (n + 31) / 32;
  uint32_t* F0 = static_cast<uint32_t*>(work);
  uint32_t* F1 = F0 + n * W;
  uint32_t* V = F1 + n * W;
  int* grew = reinterpret_cast<int*>(V + n * W);
  const unsigned iblocks = (unsigned)std::min<int64_t>((n * std::max<int64_t>(n, W) + 255) / 256, 148 * 32);
  init_kernel<T><<<iblocks, 256, 0, st>>>(n, W, F0, V, dist, ldd);
  RDB_LAUNCH_CHECK();
  const unsigned lblocks = (unsigned)std::min<int64_t>((n + 7) / 8, 148 * 16);
  int h_grew = 0;
  int64_t level = 0;
  for (level = 1; level < n; ++level) {
    if (cudaMemsetAsync(grew, 0, sizeof(int), st) != cudaSuccess) return RDB_ECUDA;
    level_kernel<T><<<lblocks, 256, 0, st>>>(adj, n, W, F0, F1, V, dist, ldd, (int)level, grew);
    RDB_LAUNCH_CHECK();
    if (cudaMemcpyAsync(&h_grew, grew, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return RDB_ECUDA;
    if (!h_grew) break;
    std::swap(F0, F1);
  }
  if (levels_out) *levels_out = level - 1;  // deepest level that found new vertices
  return RDB_OK;
}

}  // namespace bfs
}  // namespace rdb

extern "C" size_t rdb_bfs_workspace_bytes(int64_t n) { return rdb::bfs::workspace_bytes(n); }

extern "C" int rdb_bfs_apsp(const uint32_t* bits, int64_t n, int32_t* dist_i32, double* dist_f64, int64_t ldd,
                            void* work, int64_t* levels, void* stream) {
  if (!bits || !work || n <= 0 || ldd < n || (!dist_i32 == !dist_f64)) return RDB_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return dist_i32 ? rdb::bfs::run<int32_t>(bits, n, dist_i32, ldd, work, levels, st)
                  : rdb::bfs::run<double>(bits, n, dist_f64, ldd, work, levels, st);
}

extern "C" int rdb_pattern_bits(const double* w, int64_t n, int64_t ldw, uint32_t* bits, void* stream) {
  if (!w || !bits || n <= 0 || ldw < n) return RDB_EINVAL;
  const int64_t W = (n + 31) / 32;
  const int64_t want = (n * W + 7) / 8;
  const unsigned blocks = (unsigned)std::min<int64_t>(want, 148 * 16);
  rdb::bfs::pattern_bits_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(w, n, ldw, bits);
  RDB_LAUNCH_CHECK();
  return RDB_OK;
}
