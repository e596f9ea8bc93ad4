// P1 of the blocked Gauss-Jordan step: D = A_pp^-1 for the NB x NB diagonal
// block (NB = 128), in place.
//
// The block inverse is itself a blocked Gauss-Jordan with 32-wide sub-panels,
// entirely in shared memory (one CTA of 8 warps per matrix):
//   (i)   D32 = S_qq^-1        4 warps, unblocked, pivot row/column through smem
//                              (meanwhile the other 4 warps copy S_rq to T)
//   (ii)  S_qj = D32 * S_qj    j outside q                      (DMMA)
//   (iii) S_ij = [S_ij] - T_i * S_qj  for i outside q, all j    (DMMA; [.] = 0 for j in q)
// The pivots of (i) are the Schur-complement diagonals, i.e. LAPACK's diag(U)
// when no row swaps occur (linalg.py:33-34); their minimum and sign are
// recorded for the singularity rule and the no-pivot certificate.
#pragma once
#include "common.cuh"

namespace rdb {
namespace p1 {

constexpr int THREADS = 256;
constexpr int SQ = 32;        // sub-panel width
constexpr int SST = NB + 4;   // S row stride (132 = 4 mod 16: conflict-free fragments)
constexpr int TST = SQ + 4;   // T row stride (36 = 4 mod 16)

struct Smem {
  double S[NB * SST];
  double T[NB * TST];
  double prow[2][SQ];
  double pcol[2][SQ];
};
constexpr size_t SMEM_BYTES = sizeof(Smem);

RDB_DEV void named_bar(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

// (i): threads 0..127, thread (rg = t/32, j = t%32) holds rows 8rg..8rg+7 of column j.
RDB_DEV void inverse32(Smem& s, int q0, double& minp, int& mini, int& flags) {
  const int t = threadIdx.x;
  const int j = t & 31, rg = t >> 5;
  double v[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) v[e] = s.S[(q0 + 8 * rg + e) * SST + q0 + j];
  int b = 0;
#pragma unroll
  for (int kk = 0; kk < SQ; ++kk) {
    if (rg == (kk >> 3)) s.prow[b][j] = v[kk & 7];
    if (j == kk) {
#pragma unroll
      for (int e = 0; e < 8; ++e) s.pcol[b][8 * rg + e] = v[e];
    }
    named_bar(1, 128);
    const double p = s.prow[b][kk];
    const double pinv = rcp_nr(p);
    if (t == 0) {
      const double ap = fabs(p);
      if (!(ap < INFINITY)) flags |= RDB_PIV_NONFINITE;
      if (!(p > 0.0)) flags |= RDB_PIV_NONPOS;
      if (ap < minp || mini < 0) {
        minp = ap;
        mini = q0 + kk;
      }
    }
    const double u = (j == kk) ? pinv : s.prow[b][j] * pinv;
    if (j == kk) {
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] = 0.0;  // column kk becomes -f_i * pinv
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = fma(-s.pcol[b][8 * rg + e], u, v[e]);
    if (rg == (kk >> 3)) v[kk & 7] = u;
    b ^= 1;
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) s.S[(q0 + 8 * rg + e) * SST + q0 + j] = v[e];
}

// (ii): warp w updates column tiles 2w, 2w+1 (8 wide) of rows q, skipping q itself.
RDB_DEV void rowpanel32(Smem& s, int q0) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lr = lane >> 2, lk = lane & 3;
#pragma unroll
  for (int cc = 0; cc < 2; ++cc) {
    const int c0 = 8 * (2 * warp + cc);
    if (c0 >= q0 && c0 < q0 + SQ) continue;
    double acc[4][2];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) acc[mi][0] = acc[mi][1] = 0.0;
#pragma unroll
    for (int k = 0; k < SQ; k += 4) {
      const double bf = s.S[(q0 + k + lk) * SST + c0 + lr];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        const double af = s.S[(q0 + 8 * mi + lr) * SST + q0 + k + lk];
        dmma_8x8x4(acc[mi][0], acc[mi][1], af, bf);
      }
    }
    __syncwarp();
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
      double* o = &s.S[(q0 + 8 * mi + lr) * SST + c0 + 2 * lk];
      o[0] = acc[mi][0];
      o[1] = acc[mi][1];
    }
  }
}

// (iii): warp w owns columns [16w, 16w+16) of every row outside q.
RDB_DEV void update32(Smem& s, int q0) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lr = lane >> 2, lk = lane & 3;
  const int c0 = 16 * warp;
  const bool cq = (c0 >= q0 && c0 < q0 + SQ);
  double acc[12][2][2];
#pragma unroll
  for (int m = 0; m < 12; ++m) {
    const int r0 = 8 * m + (8 * m >= q0 ? SQ : 0);
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) {
      const double* c = &s.S[(r0 + lr) * SST + c0 + 8 * ni + 2 * lk];
      acc[m][ni][0] = cq ? 0.0 : c[0];
      acc[m][ni][1] = cq ? 0.0 : c[1];
    }
  }
#pragma unroll
  for (int k = 0; k < SQ; k += 4) {
    double bf[2];
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) bf[ni] = s.S[(q0 + k + lk) * SST + c0 + 8 * ni + lr];
#pragma unroll
    for (int m = 0; m < 12; ++m) {
      const int r0 = 8 * m + (8 * m >= q0 ? SQ : 0);
      const double af = -s.T[(r0 + lr) * TST + k + lk];
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) dmma_8x8x4(acc[m][ni][0], acc[m][ni][1], af, bf[ni]);
    }
  }
#pragma unroll
  for (int m = 0; m < 12; ++m) {
    const int r0 = 8 * m + (8 * m >= q0 ? SQ : 0);
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) {
      double* c = &s.S[(r0 + lr) * SST + c0 + 8 * ni + 2 * lk];
      c[0] = acc[m][ni][0];
      c[1] = acc[m][ni][1];
    }
  }
}

// The whole NB x NB inverse of A (global, row stride lda), in place.
RDB_DEV void panel_inverse(Smem& s, double* __restrict__ A, int64_t lda, int p0,
                           rdb_pivot_info* __restrict__ inf, int first) {
  const int t = threadIdx.x;
  for (int e = t; e < NB * NB / 2; e += THREADS) {
    const int r = e / (NB / 2), c2 = e % (NB / 2);
    *reinterpret_cast<double2*>(&s.S[r * SST + 2 * c2]) = ldg2(A + (int64_t)r * lda + 2 * c2);
  }
  __syncthreads();
  double minp = INFINITY;
  int mini = -1, flags = 0;
  for (int q0 = 0; q0 < NB; q0 += SQ) {
    if (t < 128) {
#ifndef RDB_EXP_P1_NOINV
      inverse32(s, q0, minp, mini, flags);
#endif
    } else {
      // copy the old S_rq (rows outside q) to T: the A operand of (iii)
      for (int e = t - 128; e < NB * SQ; e += THREADS - 128) {
        const int r = e / SQ, k = e % SQ;
        if (r < q0 || r >= q0 + SQ) s.T[r * TST + k] = s.S[r * SST + q0 + k];
      }
    }
    __syncthreads();
    rowpanel32(s, q0);
    __syncthreads();
#ifndef RDB_EXP_P1_NOUPD
    update32(s, q0);
#endif
    __syncthreads();
  }
  for (int e = t; e < NB * NB / 2; e += THREADS) {
    const int r = e / (NB / 2), c2 = e % (NB / 2);
    stg2(A + (int64_t)r * lda + 2 * c2, *reinterpret_cast<const double2*>(&s.S[r * SST + 2 * c2]));
  }
  if (t == 0) {
    if (first) {
      inf->min_pivot = minp;
      inf->min_index = p0 + mini;
      inf->flags = flags;
    } else {
      if (minp < inf->min_pivot) {
        inf->min_pivot = minp;
        inf->min_index = p0 + mini;
      }
      inf->flags |= flags;
    }
  }
}

}  // namespace p1
}  // namespace rdb
