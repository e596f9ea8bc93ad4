// K3: R = log Y / log gamma and D = ceil R, fused with the resolvent health
// counters; HBM-bound (reference: r_distance / rounded_r_distance at
// pkg/src/rdist/resolvent.py:131-153, counters at resolvent.py:120-124).
//
// Exactness: ceil has no nudge (resolvent.py:146-153), so a quotient that
// should be an exact integer must come out exact. Both logs use the same
// device log, and any quotient within 1e-9 of an integer k is recomputed as
// k + log1p((y - gamma^k)/gamma^k)/log(gamma) with gamma^k in double-double:
// the result is then correctly rounded, so y == gamma^k (as in the lone-edge
// lattice case y == gamma) gives exactly k, and log(0.09)/log(0.3) gives 2.0
// (test_resolvent.py:137-148).
#include <algorithm>
#include <climits>
#include <cmath>

#include "common.cuh"

namespace rdb {

constexpr double NEGATIVE_ENTRY_TOL = -1e-12;  // resolvent.py:26

RDB_DEV double refine_near_integer(double y, double g, double lg, double r) {
  const double k = rint(r);
  if (!(fabs(r - k) <= 1e-9 * fmax(1.0, k)) || k < 1.0 || k > 4096.0) return r;
  // P = g^k as an unevaluated sum ph + pl (double-double)
  double ph = g, pl = 0.0;
  const int ik = (int)k;
  for (int e = 1; e < ik; ++e) {
    const double p = ph * g;
    double err = fma(ph, g, -p);
    err = fma(pl, g, err);
    ph = p + err;
    pl = err - (ph - p);
  }
  if (!(ph > 1e-280)) return r;
  const double d = (y - ph) - pl;  // y - ph is exact (Sterbenz): y/ph = g^(r-k) ~ 1
  const double t = d / ph;
  const double delta = fma(-0.5 * t, t, t) / lg;  // log1p(t) = t - t^2/2 + O(t^3), |t| < 1e-8
  return k + delta;
}

template <bool HAS_R, bool HAS_DC, bool HAS_D32>
__global__ void log_ceil_kernel(const double* __restrict__ y, int64_t n, int64_t ldy, int64_t stride_y,
                                const double* __restrict__ gammas, double gamma,
                                double* __restrict__ r_out, double* __restrict__ dc_out,
                                int32_t* __restrict__ d32_out, int64_t ldo, int64_t stride_o,
                                const uint8_t* __restrict__ reach, int64_t ldm,
                                unsigned long long* __restrict__ counters) {
  const int64_t b = blockIdx.z;
  const double g = gammas ? gammas[b] : gamma;
  const double lg = log(g);
  const double* Y = y + b * stride_y;
  unsigned neg = 0, under = 0;
  for (int64_t i = blockIdx.y; i < n; i += gridDim.y) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x) {
      const double v = Y[i * ldy + j];
      double r;
      if (i == j) {
        r = 0.0;
      } else if (v > 0.0) {
        r = refine_near_integer(v, g, lg, log(v) / lg);
      } else {
        r = INFINITY;
      }
      neg += (v < NEGATIVE_ENTRY_TOL);
      if (reach) under += (v == 0.0 && i != j && reach[i * ldm + j] != 0);
      const int64_t o = b * stride_o + i * ldo + j;
      if (HAS_R) r_out[o] = r;
      const double dcv = ceil(r);
      if (HAS_DC) dc_out[o] = dcv;
      if (HAS_D32) d32_out[o] = (dcv < 2147483647.0) ? (int32_t)dcv : INT_MAX;
    }
  }
  if (counters) {
    neg = __reduce_add_sync(0xffffffffu, neg);
    under = __reduce_add_sync(0xffffffffu, under);
    if ((threadIdx.x & 31) == 0) {
      if (neg) atomicAdd(&counters[b * RDB_NCOUNTERS + RDB_CNT_NEGATIVE], (unsigned long long)neg);
      if (under)
        atomicAdd(&counters[b * RDB_NCOUNTERS + RDB_CNT_UNDERFLOW], (unsigned long long)under);
    }
  }
}

template <bool A, bool B, bool C>
static void launch(dim3 grid, cudaStream_t st, const double* y, int64_t n, int64_t ldy,
                   int64_t stride_y, const double* gammas, double gamma, double* r, double* dc,
                   int32_t* d32, int64_t ldo, int64_t stride_o, const uint8_t* reach, int64_t ldm,
                   unsigned long long* counters) {
  log_ceil_kernel<A, B, C><<<grid, 256, 0, st>>>(y, n, ldy, stride_y, gammas, gamma, r, dc, d32, ldo,
                                                 stride_o, reach, ldm, counters);
}

int log_ceil(const double* y, int64_t n, int64_t ldy, int64_t stride_y, int64_t batch,
             const double* gammas, double gamma, double* r_out, double* dceil_out, int32_t* d32_out,
             int64_t ldo, int64_t stride_o, const uint8_t* reachable, int64_t ldm,
             unsigned long long* counters, cudaStream_t st) {
  if (!y || n <= 0 || ldy < n || batch <= 0 || batch > 65535) return RDB_EINVAL;
  if ((r_out || dceil_out || d32_out) && ldo < n) return RDB_EINVAL;
  if (reachable && ldm < n) return RDB_EINVAL;
  if (!gammas && !(gamma > 0.0 && gamma < 1.0)) return RDB_EINVAL;
  int64_t gx = (n + 255) / 256;
  int64_t gy = n;
  // aim for ~8 waves of 148 SMs in total
  const int64_t target = 148 * 16;
  int64_t total = gx * gy * batch;
  if (total > target * 64) gy = std::max<int64_t>(1, (target * 64) / (gx * batch));
  if (gy > 65535) gy = 65535;
  dim3 grid((unsigned)gx, (unsigned)gy, (unsigned)batch);
  const int key = (r_out ? 4 : 0) | (dceil_out ? 2 : 0) | (d32_out ? 1 : 0);
#define RDB_LC(K, A, B, C)                                                                      \
  case K:                                                                                       \
    launch<A, B, C>(grid, st, y, n, ldy, stride_y, gammas, gamma, r_out, dceil_out, d32_out, ldo, \
                    stride_o, reachable, ldm, counters);                                        \
    break;
  switch (key) {
    RDB_LC(0, false, false, false)
    RDB_LC(1, false, false, true)
    RDB_LC(2, false, true, false)
    RDB_LC(3, false, true, true)
    RDB_LC(4, true, false, false)
    RDB_LC(5, true, false, true)
    RDB_LC(6, true, true, false)
    RDB_LC(7, true, true, true)
  }
#undef RDB_LC
  RDB_LAUNCH_CHECK();
  return RDB_OK;
}

}  // namespace rdb

extern "C" int rdb_log_ceil(const double* y, int64_t n, int64_t ldy, int64_t stride_y, int64_t batch,
                            const double* gammas, double gamma, double* r_out, double* dceil_out,
                            int32_t* d32_out, int64_t ldo, int64_t stride_o,
                            const uint8_t* reachable, int64_t ldm, unsigned long long* counters,
                            void* stream) {
  return rdb::log_ceil(y, n, ldy, stride_y, batch, gammas, gamma, r_out, dceil_out, d32_out, ldo,
                       stride_o, reachable, ldm, counters, static_cast<cudaStream_t>(stream));
}
