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
//   P1 (gj_panel_kernel, block x = 0)  D = A_pp^-1, pivots recorded; Dt = D^T
//   P1 (gj_panel_kernel, blocks x > 0) CwT = -(A_rp)^T   (the update overwrites A_rp)
//   P2 (engine, store)                 A_pJ = D * A_pJ             for J != p
//   U  (engine, reduce-add / store)    A_IJ += CwT^T * A_pJ        for I != p, J != p
//                                      A_Ip  = CwT^T * D           (= -A_Ip D)
// After the last panel A = M^-1 (2n^3 flop in total). P2 and U run on the
// persistent warp-specialised DMMA engine (dmma_engine.cuh).
#include <cmath>

#include "dmma_engine.cuh"
#include "gj_panel.cuh"

namespace rdb {

// ------------------------------------------------------------------ P1
// Block x = 0: D = A_pp^-1 in place (+ D^T, pivots), see gj_panel.cuh.
// Blocks x > 0: rows [128(x-1), 128x) of the column panel -> CwT = -(A_rp)^T.
__global__ void __launch_bounds__(p1::THREADS, 1)
    gj_panel_kernel(double* __restrict__ a, int64_t n, int64_t lda, int64_t stride, int p0,
                    rdb_pivot_info* __restrict__ info, int first, double* __restrict__ cwt_all,
                    double* __restrict__ dt_all) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int64_t b = blockIdx.y;
  double* A = a + b * stride;
  if (blockIdx.x == 0) {
    p1::panel_inverse(*reinterpret_cast<p1::Smem*>(smem_raw), A + (int64_t)p0 * lda + p0, lda, p0,
                      info + b, first, dt_all + b * NB * NB);
    return;
  }
  const int64_t i0 = (int64_t)(blockIdx.x - 1) * p1::CP_ROWS;
  if (i0 >= p0 && i0 < p0 + NB) return;  // the panel's own rows: not used by the update
  p1::panel_copy(reinterpret_cast<double*>(smem_raw), A, n, lda, p0, i0, cwt_all + b * NB * n);
}

// ------------------------------------------------------------------ schedulers
struct RowPanelSched {
  double* a;
  const double* dt_all;
  int64_t lda, stride;
  int nt, pt, batch;
  RDB_DEV int count() const { return batch * (nt - 1); }
  RDB_DEV eng::Tile tile(int t) const {
    const int g = t / (nt - 1);
    int J = t - g * (nt - 1);
    J += (J >= pt);
    double* A = a + (int64_t)g * stride;
    double* rowp = A + (int64_t)pt * NB * lda + (int64_t)J * NB;
    eng::Tile T;
    T.a = dt_all + (int64_t)g * NB * NB;
    T.lda = NB;
    T.b = rowp;
    T.ldb = lda;
    T.c = rowp;
    T.ldc = lda;
    T.nk = NB / eng::BK;
    T.mode = eng::EPI_STORE;
    return T;
  }
};

struct UpdateSched {
  double* a;
  const double* cwt_all;
  int64_t n, lda, stride;
  int nt, pt, batch;
  RDB_DEV int count() const { return batch * (nt - 1) * nt; }
  RDB_DEV eng::Tile tile(int t) const {
    const int per = (nt - 1) * nt;
    const int g = t / per;
    const int rem = t - g * per;
    int I = rem / nt;
    const int J = rem - I * nt;
    I += (I >= pt);
    double* A = a + (int64_t)g * stride;
    eng::Tile T;
    T.a = cwt_all + (int64_t)g * NB * n + (int64_t)I * NB;
    T.lda = n;
    T.b = A + (int64_t)pt * NB * lda + (int64_t)J * NB;
    T.ldb = lda;
    T.c = A + (int64_t)I * NB * lda + (int64_t)J * NB;
    T.ldc = lda;
    T.nk = NB / eng::BK;
    T.mode = (J == pt) ? eng::EPI_STORE : eng::EPI_REDUCE;
    return T;
  }
};

__global__ void __launch_bounds__(eng::THREADS, 1) gj_rowpanel_kernel(RowPanelSched sched) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  eng::run<true>(*reinterpret_cast<eng::Smem*>(smem_raw), sched);
}

__global__ void __launch_bounds__(eng::THREADS, 1) gj_update_kernel(UpdateSched sched) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  eng::run<true>(*reinterpret_cast<eng::Smem*>(smem_raw), sched);
}

static int g_sms = 0;

static int setup() {
  if (g_sms) return RDB_OK;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return RDB_ECUDA;
  if (cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return RDB_ECUDA;
  if (cudaFuncSetAttribute(gj_rowpanel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)eng::SMEM_BYTES) != cudaSuccess ||
      cudaFuncSetAttribute(gj_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)eng::SMEM_BYTES) != cudaSuccess ||
      cudaFuncSetAttribute(gj_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)p1::SMEM_BYTES) != cudaSuccess)
    return RDB_ECUDA;
  return RDB_OK;
}

int sm_count() {
  setup();
  return g_sms > 0 ? g_sms : 148;
}

static unsigned persistent_grid(int64_t tiles) {
  const int64_t sms = sm_count();
  return (unsigned)(tiles < sms ? tiles : sms);
}

int invert_batched(double* a, int64_t n, int64_t lda, int64_t stride, int64_t batch, void* work,
                   rdb_pivot_info* info, cudaStream_t st) {
  if (!a || !work || !info || n <= 0 || batch <= 0) return RDB_EINVAL;
  if (n % NB != 0 || lda < n || (lda & 1) || (batch > 1 && stride < n * lda)) return RDB_EINVAL;
  if (((uintptr_t)a & 15) || ((uintptr_t)work & 15)) return RDB_EINVAL;
  if (batch > 65535) return RDB_EINVAL;
  const int nt = (int)(n / NB);
  if ((int64_t)batch * nt * nt > 2147483647LL) return RDB_EINVAL;
  int rc = setup();
  if (rc) return rc;
  double* cwt = static_cast<double*>(work);
  double* dt = cwt + batch * NB * n;
  for (int k = 0; k < nt; ++k) {
    const int p0 = k * NB;
    gj_panel_kernel<<<dim3((unsigned)(1 + n / p1::CP_ROWS), (unsigned)batch), p1::THREADS, p1::SMEM_BYTES,
                      st>>>(
        a, n, lda, stride, p0, info, k == 0, cwt, dt);
    if (nt > 1) {
      RowPanelSched rp{a, dt, lda, stride, nt, k, (int)batch};
      gj_rowpanel_kernel<<<persistent_grid((int64_t)batch * (nt - 1)), eng::THREADS, eng::SMEM_BYTES,
                           st>>>(rp);
      UpdateSched up{a, cwt, n, lda, stride, nt, k, (int)batch};
      gj_update_kernel<<<persistent_grid((int64_t)batch * (nt - 1) * nt), eng::THREADS,
                         eng::SMEM_BYTES, st>>>(up);
    }
  }
  RDB_LAUNCH_CHECK();
  return RDB_OK;
}

// ------------------------------------------------------------------ K5 residual
// max |M Y - I| (resolvent.py:125-127) with M row-major as the A operand; the
// epilogue reduces |acc - delta_ij| instead of storing.
struct ResidualSched {
  const double* m;
  const double* y;
  int64_t ldm, ldy;
  int nt, nk;
  RDB_DEV int count() const { return nt * nt; }
  RDB_DEV eng::Tile tile(int t) const {
    const int I = t / nt, J = t - (t / nt) * nt;
    eng::Tile T;
    T.a = m + (int64_t)I * NB * ldm;
    T.lda = ldm;
    T.b = y + (int64_t)J * NB;
    T.ldb = ldy;
    T.c = nullptr;
    T.ldc = I;  // row tile index (the epilogue needs the origin only)
    T.nk = nk;
    T.mode = J;
    return T;
  }
};

struct ResidualEpi {
  double* out_max;
  RDB_DEV void operator()(const eng::Tile& T, double (&acc)[8][4][2], int wr, int wc, int lane,
                          double*) const {
    const int64_t row0 = T.ldc * NB + wr * 64, col0 = (int64_t)T.mode * NB + wc * 32;
    double mx = 0.0;
#pragma unroll
    for (int mi = 0; mi < 8; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        const int64_t gi = row0 + mi * 8 + (lane >> 2);
        const int64_t gj = col0 + ni * 8 + 2 * (lane & 3);
        const double e0 = fabs(acc[mi][ni][0] - (gi == gj ? 1.0 : 0.0));
        const double e1 = fabs(acc[mi][ni][1] - (gi == gj + 1 ? 1.0 : 0.0));
        mx = (e0 > mx || e0 != e0) ? e0 : mx;  // NaN wins, as in numpy's max
        mx = (e1 > mx || e1 != e1) ? e1 : mx;
      }
    for (int o = 16; o > 0; o >>= 1) {
      const double other = __shfl_xor_sync(0xffffffffu, mx, o);
      mx = (other > mx || other != other) ? other : mx;
    }
    if (lane == 0) atomic_max_nonneg(out_max, mx);
  }
};

__global__ void __launch_bounds__(eng::THREADS, 1) residual_kernel(ResidualSched sched, ResidualEpi epi) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  eng::run<false>(*reinterpret_cast<eng::Smem*>(smem_raw), sched, epi);
}

}  // namespace rdb

using namespace rdb;

extern "C" size_t rdb_invert_workspace_bytes(int64_t n_pad, int64_t batch) {
  if (n_pad <= 0 || batch <= 0) return 0;
  return (size_t)batch * ((size_t)n_pad * NB + (size_t)NB * NB) * sizeof(double);
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
                           (int)eng::SMEM_BYTES) != cudaSuccess)
    return RDB_ECUDA;
  const int nt = (int)(n_pad / NB);
  ResidualSched sched{m, y, ldm, ldy, nt, (int)(n_pad / eng::BK)};
  ResidualEpi epi{out_max};
  residual_kernel<<<persistent_grid((int64_t)nt * nt), eng::THREADS, eng::SMEM_BYTES,
                    static_cast<cudaStream_t>(stream)>>>(sched, epi);
  RDB_LAUNCH_CHECK();
  return RDB_OK;
}
