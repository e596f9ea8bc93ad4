// FP64 DMMA tile engine: acc(128x64) = A(128xK) * B(Kx64), both operands
// row-major in global memory, staged into padded shared memory by the bulk-copy
// (TMA) engine through a 2-stage mbarrier pipeline.
//
// Used by the Gauss-Jordan row-panel product (D * A_p,J), the trailing
// rank-NB update (A_IJ -= Cw_I * B_J), and the inversion residual (M * Y).
//
// Layout choices:
//   * 8 warps as 4 (rows) x 2 (cols); a warp owns 32x32 = 4x4 DMMA tiles,
//     32 fp64 accumulators per lane.
//   * A stage: 128 rows x KC(32) k, row stride 36 doubles; B stage: KC x 64,
//     row stride 68 doubles. Both strides are 4 mod 16 doubles, which makes the
//     m8n8k4 fragment loads (lane -> [l/4][l%4]) bank-conflict free.
//   * One TMA bulk copy per smem row (256 B for A, 512 B for B); warp 0 issues
//     them, the stage's mbarrier counts the bytes.
#pragma once
#include "common.cuh"

namespace rdb {

constexpr int TM = 128;  // tile rows
constexpr int TN = 64;   // tile cols
constexpr int KC = 32;   // k per stage
constexpr int AST = KC + 4;   // 36
constexpr int BST = TN + 4;   // 68
constexpr int TILE_THREADS = 256;
constexpr uint32_t STAGE_BYTES = (TM * KC + KC * TN) * 8;  // 49152

struct TileSmem {
  alignas(128) double a[2][TM * AST];
  alignas(128) double b[2][KC * BST];
  alignas(8) uint64_t full[2];
};
constexpr size_t TILE_SMEM_BYTES = sizeof(TileSmem);

struct Acc {
  double v[4][4][2];
};

RDB_DEV void acc_zero(Acc& acc) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc.v[i][j][0] = acc.v[i][j][1] = 0.0;
}

// Issue the bulk copies of k-chunk `c` into stage `st`. Called by all 32 lanes of warp 0.
RDB_DEV void tile_issue(TileSmem& s, int st, int c, const double* A, int64_t lda, const double* B,
                        int64_t ldb, int lane) {
  if (lane == 0) mbar_arrive_expect_tx(&s.full[st], STAGE_BYTES);
  __syncwarp();
  const int k0 = c * KC;
#pragma unroll
  for (int q = 0; q < TM / 32; ++q) {
    const int i = lane + 32 * q;
    bulk_g2s(&s.a[st][i * AST], A + (int64_t)i * lda + k0, KC * 8, &s.full[st]);
  }
  bulk_g2s(&s.b[st][lane * BST], B + (int64_t)(k0 + lane) * ldb, TN * 8, &s.full[st]);
}

// acc += A[0:128, 0:K] * B[0:K, 0:64]; K a multiple of KC.
// Must be called by all 256 threads; ends with the smem free for reuse.
RDB_DEV void tile_mainloop(TileSmem& s, Acc& acc, const double* A, int64_t lda, const double* B,
                           int64_t ldb, int K) {
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wr = warp & 3, wc = warp >> 2;
  if (tid == 0) {
    mbar_init(&s.full[0], 1);
    mbar_init(&s.full[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int nchunks = K / KC;
  if (warp == 0) {
    tile_issue(s, 0, 0, A, lda, B, ldb, lane);
    if (nchunks > 1) tile_issue(s, 1, 1, A, lda, B, ldb, lane);
  }
  const int lr = lane >> 2, lk = lane & 3;
  for (int c = 0; c < nchunks; ++c) {
    const int st = c & 1;
    mbar_wait(&s.full[st], (c >> 1) & 1);
    const double* sa = s.a[st] + (wr * 32 + lr) * AST + lk;
    const double* sb = s.b[st] + lk * BST + wc * 32 + lr;
#pragma unroll
    for (int kk = 0; kk < KC; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) af[mi] = sa[mi * 8 * AST + kk];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) bf[ni] = sb[kk * BST + ni * 8];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma_8x8x4(acc.v[mi][ni][0], acc.v[mi][ni][1], af[mi], bf[ni]);
    }
    __syncthreads();
    if (warp == 0 && c + 2 < nchunks) tile_issue(s, st, c + 2, A, lda, B, ldb, lane);
  }
}

// Visit the accumulator elements: f(row, col, acc_pair) with col even; row/col
// relative to the tile origin.
template <class F>
RDB_DEV void tile_epilogue(Acc& acc, F&& f) {
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wr = warp & 3, wc = warp >> 2;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const int r = wr * 32 + mi * 8 + (lane >> 2);
      const int cc = wc * 32 + ni * 8 + 2 * (lane & 3);
      f(r, cc, acc.v[mi][ni][0], acc.v[mi][ni][1]);
    }
}

}  // namespace rdb
