// K2: blocked Gauss-Jordan inversion in FP64 on sm_100a, no pivoting.
//
// Replaces the reference's scipy.linalg.lu_factor + lu_solve(I)
// (pkg/src/rdist/linalg.py:32, :39). For M = I - gamma^W below the critical
// gain, M is a nonsingular M-matrix: elimination without pivoting is stable
// and every off-diagonal update accumulates same-signed terms, so Y = M^-1
// keeps componentwise relative accuracy (the tiny entries encode the long
// distances). LAPACK's partial pivoting performs no row swaps on these
// matrices, so the pivots recorded here are the
// reference's diag(U) (linalg.py:33-34).
//
// Per panel p = [k*NB, (k+1)*NB), r = all other indices, in place on A:
//   P1  D = A_pp^-1            (one CTA per matrix, unblocked GJ, pivots recorded)
//   P2  A_pr = D * A_pr        (DMMA tiles over the row panel)
//       Cw   = A_rp (copy)     (the update overwrites A_rp)
//   U   A_rr = A_rr - Cw * A_pr ;  A_rp = -Cw * D   (one DMMA tile kernel)
// After the last panel A = M^-1 (2n^3 flop in total).
#include <cmath>

#include "tile_mma.cuh"

namespace rdb {

// ------------------------------------------------------------------ P1
// Unblocked Gauss-Jordan inverse of the NB x NB diagonal block, in place.
// 512 threads; thread (rg = t/128, j = t%128) keeps column j, rows 32*rg..+32
// of the block in registers. Each step publishes the pivot row and column
// through shared memory (double-buffered) and applies a rank-1 update.
constexpr int P1_THREADS = 512;

__global__ void __launch_bounds__(P1_THREADS, 1)
    gj_panel_kernel(double* __restrict__ a, int64_t lda, int64_t stride, int p0,
                    rdb_pivot_info* __restrict__ info, int first) {
  __shared__ double prow[2][NB];
  __shared__ double pcol[2][NB];
  const int t = threadIdx.x;
  const int j = t & (NB - 1);
  const int rg = t >> 7;
  double* A = a + (int64_t)blockIdx.x * stride + (int64_t)p0 * lda + p0;
  double v[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) v[r] = A[(int64_t)(32 * rg + r) * lda + j];

  double minp = INFINITY;
  int mini = -1, flags = 0;

  int buf = 0;
#pragma unroll 1
  for (int q = 0; q < 4; ++q) {
#pragma unroll
    for (int s = 0; s < 32; ++s) {
      const int kk = 32 * q + s;
      // publish pivot row kk and pivot column kk
      if (rg == q) prow[buf][j] = v[s];
      if (j == kk) {
#pragma unroll
        for (int r = 0; r < 32; ++r) pcol[buf][32 * rg + r] = v[r];
      }
      __syncthreads();
      const double p = prow[buf][kk];
      const double pinv = 1.0 / p;
      if (t == 0) {
        const double ap = fabs(p);
        if (!(ap < INFINITY)) flags |= RDB_PIV_NONFINITE;
        if (!(p > 0.0)) flags |= RDB_PIV_NONPOS;
        if (ap < minp || mini < 0) {
          minp = ap;
          mini = kk;
        }
      }
      const double u = (j == kk) ? pinv : prow[buf][j] * pinv;
      if (j == kk) {
        // column kk of the result is -f_i * pinv: start from 0 so the common
        // fma(-f, u, v) below produces exactly that.
#pragma unroll
        for (int r = 0; r < 32; ++r) v[r] = 0.0;
      }
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        if (r == s && rg == q) {
          v[r] = u;
        } else {
          const double f = pcol[buf][32 * rg + r];
          v[r] = fma(-f, u, v[r]);
        }
      }
      buf ^= 1;
    }
  }
#pragma unroll
  for (int r = 0; r < 32; ++r) A[(int64_t)(32 * rg + r) * lda + j] = v[r];

  if (t == 0) {
    rdb_pivot_info* inf = info + blockIdx.x;
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

// ------------------------------------------------------------------ P2
// grid (n/TN, batch). Column tile J (TN wide):
//   * copy Cw[i][0:NB] = A[i][p0:p0+NB] for rows i in [J*TN, J*TN+TN) outside p;
//   * if J is outside p: A[p0:p0+NB][J] = D * A[p0:p0+NB][J] (DMMA tile, K = NB).
__global__ void __launch_bounds__(TILE_THREADS, 2)
    gj_rowpanel_kernel(double* __restrict__ a, int64_t n, int64_t lda, int64_t stride, int p0,
                       double* __restrict__ cw_all) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  TileSmem& s = *reinterpret_cast<TileSmem*>(smem_raw);
  const int J = blockIdx.x;
  const int64_t b = blockIdx.y;
  double* A = a + b * stride;
  double* cw = cw_all + b * n * NB;
  const int col0 = J * TN;
  const bool in_panel = (col0 >= p0) && (col0 < p0 + NB);

  // column-panel copy (rows col0 .. col0+TN; row-tile and column-tile index sets coincide)
  if (!in_panel) {
    const int tid = threadIdx.x;
    // TN rows x NB cols = TN * NB/2 double2
    for (int e = tid; e < TN * (NB / 2); e += TILE_THREADS) {
      const int r = e / (NB / 2), c2 = e % (NB / 2);
      const int64_t i = col0 + r;
      stg2(cw + i * NB + 2 * c2, ldg2(A + i * lda + p0 + 2 * c2));
    }
  }
  if (in_panel) return;

  Acc acc;
  acc_zero(acc);
  const double* D = A + (int64_t)p0 * lda + p0;
  const double* Bp = A + (int64_t)p0 * lda + col0;
  tile_mainloop(s, acc, D, lda, Bp, lda, NB);
  double* out = A + (int64_t)p0 * lda + col0;
  tile_epilogue(acc, [&](int r, int c, double x0, double x1) {
    stg2(out + (int64_t)r * lda + c, make_double2(x0, x1));
  });
}

// ------------------------------------------------------------------ U
// grid (n/TN, n/TM, batch). Tile (I, J), I != panel row tile:
//   A_IJ = (J in p ? 0 : A_IJ) - Cw_I * A_pJ.
__global__ void __launch_bounds__(TILE_THREADS, 2)
    gj_update_kernel(double* __restrict__ a, int64_t n, int64_t lda, int64_t stride, int p0,
                     const double* __restrict__ cw_all) {
  const int row0 = blockIdx.y * TM;
  if (row0 == p0) return;  // TM == NB: the panel row tile was written by P2
  extern __shared__ __align__(128) unsigned char smem_raw[];
  TileSmem& s = *reinterpret_cast<TileSmem*>(smem_raw);
  const int col0 = blockIdx.x * TN;
  const int64_t b = blockIdx.z;
  double* A = a + b * stride;
  const double* cw = cw_all + b * n * NB;
  const bool in_panel = (col0 >= p0) && (col0 < p0 + NB);

  Acc acc;
  acc_zero(acc);
  tile_mainloop(s, acc, cw + (int64_t)row0 * NB, NB, A + (int64_t)p0 * lda + col0, lda, NB);
  double* C = A + (int64_t)row0 * lda + col0;
  tile_epilogue(acc, [&](int r, int c, double x0, double x1) {
    double* p = C + (int64_t)r * lda + c;
    double2 o = in_panel ? make_double2(0.0, 0.0) : ldg2(p);
    o.x -= x0;
    o.y -= x1;
    stg2(p, o);
  });
}

static bool g_attr_set = false;

static int set_attrs() {
  if (g_attr_set) return RDB_OK;
  if (cudaFuncSetAttribute(gj_rowpanel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)TILE_SMEM_BYTES) != cudaSuccess)
    return RDB_ECUDA;
  if (cudaFuncSetAttribute(gj_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)TILE_SMEM_BYTES) != cudaSuccess)
    return RDB_ECUDA;
  g_attr_set = true;
  return RDB_OK;
}

int invert_batched(double* a, int64_t n, int64_t lda, int64_t stride, int64_t batch, void* work,
                   rdb_pivot_info* info, cudaStream_t st) {
  if (!a || !work || !info || n <= 0 || batch <= 0) return RDB_EINVAL;
  if (n % NB != 0 || lda < n || (lda & 1) || (batch > 1 && stride < n * lda)) return RDB_EINVAL;
  if (((uintptr_t)a & 15) || ((uintptr_t)work & 15)) return RDB_EINVAL;
  if (batch > 65535 || n / TN > 2147483647) return RDB_EINVAL;
  int rc = set_attrs();
  if (rc) return rc;
  double* cw = static_cast<double*>(work);
  const int nsteps = (int)(n / NB);
  for (int k = 0; k < nsteps; ++k) {
    const int p0 = k * NB;
    gj_panel_kernel<<<(unsigned)batch, P1_THREADS, 0, st>>>(a, lda, stride, p0, info, k == 0);
    gj_rowpanel_kernel<<<dim3((unsigned)(n / TN), (unsigned)batch), TILE_THREADS, TILE_SMEM_BYTES,
                         st>>>(a, n, lda, stride, p0, cw);
    gj_update_kernel<<<dim3((unsigned)(n / TN), (unsigned)(n / TM), (unsigned)batch), TILE_THREADS,
                       TILE_SMEM_BYTES, st>>>(a, n, lda, stride, p0, cw);
  }
  RDB_LAUNCH_CHECK();
  return RDB_OK;
}

// ------------------------------------------------------------------ K5 residual
// max |M Y - I| over the n_pad x n_pad product (resolvent.py:125-127). The
// padding is identity in both factors, so it contributes exact zeros.
__global__ void __launch_bounds__(TILE_THREADS, 2)
    residual_kernel(const double* __restrict__ m, int64_t ldm, const double* __restrict__ y,
                    int64_t ldy, int64_t n, double* __restrict__ out_max) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  TileSmem& s = *reinterpret_cast<TileSmem*>(smem_raw);
  const int row0 = blockIdx.y * TM, col0 = blockIdx.x * TN;
  Acc acc;
  acc_zero(acc);
  tile_mainloop(s, acc, m + (int64_t)row0 * ldm, ldm, y + col0, ldy, (int)n);
  double mx = 0.0;
  tile_epilogue(acc, [&](int r, int c, double x0, double x1) {
    const int gi = row0 + r, gj = col0 + c;
    const double e0 = fabs(x0 - (gi == gj ? 1.0 : 0.0));
    const double e1 = fabs(x1 - (gi == gj + 1 ? 1.0 : 0.0));
    // NaN must win the max, as numpy's max does
    mx = (e0 > mx || e0 != e0) ? e0 : mx;
    mx = (e1 > mx || e1 != e1) ? e1 : mx;
  });
  for (int o = 16; o > 0; o >>= 1) {
    const double other = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = (other > mx || other != other) ? other : mx;
  }
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(out_max, mx);
}

}  // namespace rdb

using namespace rdb;

extern "C" size_t rdb_invert_workspace_bytes(int64_t n_pad, int64_t batch) {
  if (n_pad <= 0 || batch <= 0) return 0;
  return (size_t)batch * (size_t)n_pad * NB * sizeof(double);
}

extern "C" int rdb_invert_batched(double* a, int64_t n_pad, int64_t lda, int64_t stride,
                                  int64_t batch, void* work, rdb_pivot_info* info, void* stream) {
  return invert_batched(a, n_pad, lda, stride, batch, work, info,
                        static_cast<cudaStream_t>(stream));
}

extern "C" int rdb_invert(double* a, int64_t n_pad, int64_t lda, void* work, rdb_pivot_info* info,
                          void* stream) {
  return invert_batched(a, n_pad, lda, n_pad * lda, 1, work, info,
                        static_cast<cudaStream_t>(stream));
}

extern "C" int rdb_residual(const double* m, int64_t ldm, const double* y, int64_t ldy,
                            int64_t n_pad, double* out_max, void* stream) {
  if (!m || !y || !out_max || n_pad <= 0 || n_pad % NB || (ldm & 1) || (ldy & 1) || ldm < n_pad ||
      ldy < n_pad)
    return RDB_EINVAL;
  if (cudaFuncSetAttribute(residual_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)TILE_SMEM_BYTES) != cudaSuccess)
    return RDB_ECUDA;
  residual_kernel<<<dim3((unsigned)(n_pad / TN), (unsigned)(n_pad / TM)), TILE_THREADS,
                    TILE_SMEM_BYTES, static_cast<cudaStream_t>(stream)>>>(m, ldm, y, ldy, n_pad,
                                                                           out_max);
  RDB_LAUNCH_CHECK();
  return RDB_OK;
}
