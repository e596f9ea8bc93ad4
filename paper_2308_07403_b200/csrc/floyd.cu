// K10: Floyd–Warshall all-pairs shortest paths on the GPU, bit for bit the
// reference's floyd_warshall (pkg/src/rdist/oracles.py:44-50):
//   d = W, diag(d) = 0; for k = 0..n-1: d = min(d, d[:, k] + d[k, :])
// i.e. d_ij^(k) = min(d_ij^(k-1), d_ik^(k-1) + d_kj^(k-1)) in IEEE fp64.
//
// Blocked over KB = 32 consecutive k. The classic recurrence uses, at step k,
// column k and row k as they stood after step k-1; blocking must hand every
// (i, j) exactly those operands (the textbook blocked algorithm uses later
// values and rounds real-weight sums differently). Per k-block K:
//   fw_panel_kernel: every CTA replays the K x K block through the block's
//     steps (32^3 min/add, in shared memory), recording SK[k][k'] = d_kk'^(k-1)
//     and ET[k''][k] = d_k''k^(k-1); then either
//       S[k][j]  = d_kj^(k-1) for its column tile (rows K replayed per column), or
//       E[i][k]  = d_ik^(k-1) for its row tile (columns K replayed per row);
//   fw_update_kernel: d_ij = min(d_ij, E[i][k] + S[k][j]) for k in K in order,
//     over 64 x 128 tiles (E and S tiles staged in shared memory).
// Column k and row k do not change at step k (d_kk = 0, weights > 0), so the
// snapshots are the values the classic loop reads. Work: n^3 (add, min)
// pairs on the FP64 pipe; traffic 16 n^2 B per k-block.
#include <cmath>

#include "common.cuh"

namespace rdb {
namespace fw {

constexpr int KB = 32;
constexpr int TR = 64, TC = 128;  // update tile
constexpr int PT = 256;           // panel threads (one column / row each)

__global__ void init_kernel(const double* __restrict__ w, int64_t ldw, int64_t n, double* __restrict__ d,
                            int64_t ldd) {
  const int64_t total = n * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e - i * n;
    d[i * ldd + j] = (i == j) ? 0.0 : w[i * ldw + j];
  }
}

// Replay of the K x K block (kb <= KB) by one warp; SK / ET as above.
RDB_DEV void replay_block(const double* __restrict__ d, int64_t ldd, int64_t k0, int kb, double (*T)[KB + 1],
                          double (*SK)[KB + 1], double (*ET)[KB + 1]) {
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 32) {
    for (int c = 0; c < kb; ++c) T[lane][c] = (lane < kb) ? d[(k0 + lane) * ldd + k0 + c] : INFINITY;
    __syncwarp();
    for (int k = 0; k < kb; ++k) {
      if (lane < kb) {
        SK[k][lane] = T[k][lane];   // row k at step k-1 (unchanged at step k)
        ET[lane][k] = T[lane][k];   // column k at step k-1
      }
      __syncwarp();
      if (lane < kb) {
        const double dik = T[lane][k];
        for (int c = 0; c < kb; ++c) T[lane][c] = fmin(T[lane][c], dik + SK[k][c]);
      }
      __syncwarp();
    }
  }
  __syncthreads();
}

// blocks [0, ncol_tiles): S for columns j0 .. j0 + PT; then row tiles for E.
__global__ void __launch_bounds__(PT) panel_kernel(const double* __restrict__ d, int64_t ldd, int64_t n, int64_t k0,
                                                   int kb, int ncol_tiles, double* __restrict__ S,
                                                   double* __restrict__ E) {
  __shared__ double T[KB][KB + 1], SK[KB][KB + 1], ET[KB][KB + 1];
  replay_block(d, ldd, k0, kb, T, SK, ET);
  if ((int)blockIdx.x < ncol_tiles) {
    const int64_t j = (int64_t)blockIdx.x * PT + threadIdx.x;
    if (j >= n) return;
    double p[KB];
#pragma unroll
    for (int r = 0; r < KB; ++r) p[r] = (r < kb) ? d[(k0 + r) * ldd + j] : INFINITY;
#pragma unroll
    for (int k = 0; k < KB; ++k) {
      if (k >= kb) break;
      const double pk = p[k];
      S[(int64_t)k * n + j] = pk;
#pragma unroll
      for (int r = 0; r < KB; ++r) p[r] = fmin(p[r], ET[r][k] + pk);
    }
  } else {
    const int64_t i = (int64_t)(blockIdx.x - ncol_tiles) * PT + threadIdx.x;
    if (i >= n) return;
    double e[KB];
#pragma unroll
    for (int c = 0; c < KB; ++c) e[c] = (c < kb) ? d[i * ldd + k0 + c] : INFINITY;
#pragma unroll
    for (int k = 0; k < KB; ++k) {
      if (k >= kb) break;
      const double ek = e[k];
      E[(int64_t)k * n + i] = ek;  // E stored k-major (coalesced in the update kernel)
#pragma unroll
      for (int c = 0; c < KB; ++c) e[c] = fmin(e[c], ek + SK[k][c]);
    }
  }
}

// d_ij = min(d_ij, E[i][k] + S[k][j]) for k < kb in order; 256 threads, each
// 4 rows x 8 consecutive columns of a 64 x 128 tile.
__global__ void __launch_bounds__(256) update_kernel(double* __restrict__ d, int64_t ldd, int64_t n, int kb,
                                                     const double* __restrict__ S, const double* __restrict__ E) {
  __shared__ __align__(16) double Ss[KB][TC];
  __shared__ double Es[KB][TR];
  const int64_t i0 = (int64_t)blockIdx.y * TR, j0 = (int64_t)blockIdx.x * TC;
  for (int e = threadIdx.x; e < KB * TC; e += 256) {
    const int k = e / TC, c = e - k * TC;
    Ss[k][c] = (k < kb && j0 + c < n) ? S[(int64_t)k * n + j0 + c] : INFINITY;
  }
  for (int e = threadIdx.x; e < KB * TR; e += 256) {
    const int k = e / TR, r = e - k * TR;
    Es[k][r] = (k < kb && i0 + r < n) ? E[(int64_t)k * n + i0 + r] : INFINITY;
  }
  __syncthreads();
  const int cg = threadIdx.x & 15, rg = threadIdx.x >> 4;
  const int64_t jb = j0 + cg * 8;
  double acc[4][8];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t i = i0 + rg * 4 + r;
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = (i < n && jb + c < n) ? d[i * ldd + jb + c] : INFINITY;
  }
  for (int k = 0; k < kb; ++k) {
    double s[8], e[4];
#pragma unroll
    for (int c = 0; c < 8; c += 2) {
      const double2 v = *reinterpret_cast<const double2*>(&Ss[k][cg * 8 + c]);
      s[c] = v.x;
      s[c + 1] = v.y;
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) e[r] = Es[k][rg * 4 + r];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[r][c] = fmin(acc[r][c], e[r] + s[c]);
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t i = i0 + rg * 4 + r;
    if (i >= n) continue;
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (jb + c < n) d[i * ldd + jb + c] = acc[r][c];
  }
}

}  // namespace fw
}  // namespace rdb

using namespace rdb;

extern "C" size_t rdb_floyd_workspace_bytes(int64_t n) {
  return n <= 0 ? 0 : (size_t)2 * fw::KB * (size_t)n * sizeof(double);
}

extern "C" int rdb_floyd_warshall(const double* w, int64_t ldw, int64_t n, double* d, int64_t ldd, void* work,
                                  void* stream) {
  if (!w || !d || !work || n <= 0 || ldw < n || ldd < n || n > (int64_t)1 << 20) return RDB_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* S = static_cast<double*>(work);
  double* E = S + (int64_t)fw::KB * n;
  const int64_t total = n * n;
  fw::init_kernel<<<(unsigned)((total + 255) / 256 < 148 * 32 ? (total + 255) / 256 : 148 * 32), 256, 0, st>>>(
      w, ldw, n, d, ldd);
  const int tiles = (int)((n + fw::PT - 1) / fw::PT);
  const dim3 ugrid((unsigned)((n + fw::TC - 1) / fw::TC), (unsigned)((n + fw::TR - 1) / fw::TR));
  for (int64_t k0 = 0; k0 < n; k0 += fw::KB) {
    const int kb = (int)(n - k0 < fw::KB ? n - k0 : fw::KB);
    fw::panel_kernel<<<(unsigned)(2 * tiles), fw::PT, 0, st>>>(d, ldd, n, k0, kb, tiles, S, E);
    fw::update_kernel<<<ugrid, 256, 0, st>>>(d, ldd, n, kb, S, E);
  }
  RDB_LAUNCH_CHECK();
  return RDB_OK;
}
