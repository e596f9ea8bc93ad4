// K3: R = log Y / log gamma and D = ceil R, fused with the resolvent health
// counters; HBM-bound (reference: r_distance / rounded_r_distance at
// pkg/src/rdist/resolvent.py:131-153, counters at resolvent.py:120-124).
//
// Exactness: ceil has no nudge (resolvent.py:146-153), so a quotient that
// should be an exact integer must come out exact. R is first formed as
// log(y) * (1 / log gamma) (within a few ulp of the reference's quotient); any
// value within 1e-9 of an integer k is then recomputed as
// k + log1p((y - gamma^k)/gamma^k)/log(gamma) with gamma^k in double-double,
// which is correctly rounded: y == gamma^k (the lone-edge lattice case
// y == gamma) gives exactly k, and log(0.09)/log(0.3) gives 2.0
// (test_resolvent.py:137-148). Away from integers the ceil cannot change.
//
// Layout: one warp per matrix row, lane l handles columns 2l, 2l+1 of every
// 64-column chunk (16-byte loads of Y, 8-byte int32 pair stores).
#include <climits>
#include <cmath>

#include "common.cuh"
#include "log_table.cuh"

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

// Natural log of a positive finite double in ~18 FP64 operations (within ~1
// ulp): y = 2^e m, m in [1, 2); a 128-entry table (log_table.cuh, staged in
// shared memory) gives c ~ 1/m and L = -log c (double-double, folded with ln 2;
// c = 1 and 1/2 exactly in the two intervals around y = 1, so no term cancels
// there); log1p(m c - 1), |m c - 1| <= 2^-7, by its Taylor series to r^8.
// 16 copies of each entry, lane l reads copy l % 16: every half-warp touches 16
// distinct bank pairs whatever the (data-dependent) indices, so the lookups
// are conflict free (48 KB of shared memory per block).
struct LogTab {
  double c[128][16], hi[128][16], lo[128][16];
  RDB_DEV double C(int i) const { return c[i][threadIdx.x & 15]; }
  RDB_DEV double H(int i) const { return hi[i][threadIdx.x & 15]; }
  RDB_DEV double L(int i) const { return lo[i][threadIdx.x & 15]; }
};

// The same table read straight from constant memory: for kernels whose common
// path needs no table (the MUFU estimate), so the rare exact path costs no
// shared memory (full occupancy) and no per-block staging.
struct ConstTab {
  RDB_DEV double C(int i) const { return logtab::kC[i]; }
  RDB_DEV double H(int i) const { return logtab::kLhi[i]; }
  RDB_DEV double L(int i) const { return logtab::kLlo[i]; }
};

template <class Tab>
RDB_DEV double fast_log(double y, const Tab& T) {
  long long b = __double_as_longlong(y);
  int ex = (int)(b >> 52);
  int esub = 0;
  if (ex == 0) {  // subnormal: scale by 2^54
    b = __double_as_longlong(y * 18014398509481984.0);
    ex = (int)(b >> 52);
    esub = 54;
  }
  const int idx = (int)((b >> 45) & 127);
  const double m = __longlong_as_double((b & 0x000FFFFFFFFFFFFFLL) | 0x3FF0000000000000LL);
  const double e = (double)(ex - 1023 - esub + (idx >= 53 ? 1 : 0));
  const double r = fma(m, T.C(idx), -1.0);
  double p = fma(r, -0.125, 1.0 / 7.0);
  p = fma(r, p, -1.0 / 6.0);
  p = fma(r, p, 1.0 / 5.0);
  p = fma(r, p, -0.25);
  p = fma(r, p, 1.0 / 3.0);
  p = fma(r, p, -0.5);
  p = fma(r * r, p, r);
  const double a = e * logtab::LN2_HI;  // exact (LN2_HI has 21 significant bits)
  const double bh = T.H(idx);
  const double s = a + bh;
  // Fast2Sum error: valid as |a| >= ln2/2 > |bh| when e != 0, and exactly 0 when e == 0
  const double t = (a - s) + bh;
  return s + (t + fma(e, logtab::LN2_LO, T.L(idx)) + p);
}

template <class Tab>
RDB_DEV double rdist_value(double v, double g, double lg, double inv_lg, const Tab& T) {
  if (!(v > 0.0)) return INFINITY;
  if (!(v < INFINITY)) return -INFINITY;  // log(inf) / log(gamma), as numpy
  const double r = fast_log(v, T) * inv_lg;
  // only quotients within 1e-9 of an integer can change the ceil: refine those
  if (fabs(r - rint(r)) <= 1e-9 * fmax(1.0, r)) return refine_near_integer(v, g, lg, r);
  return r;
}

// D-only path: a value whose ceil equals ceil(rdist_value(v)). log2 y is first
// estimated as exponent + __log2f(mantissa) (absolute error < 4.1e-7: __log2f
// 2^-22 on [1, 2) plus 2^-23 / ln 2 for the 23-bit truncation, so the
// quotient's error is < 4.1e-7 / |log2 gamma| < thr / 7); only when the estimate
// lies within thr of an integer does the element take the full FP64 log and
// refinement. For the config-2 gains that is a tiny fraction of the entries.
RDB_DEV double dceil_value(double v, double g, double lg, double inv_lg, double inv_lg2, double thr,
                           const LogTab& T) {
  if (!(v > 0.0)) return INFINITY;
  if (!(v < INFINITY)) return -INFINITY;
  const long long b = __double_as_longlong(v);
  const int ex = (int)(b >> 52);
  if (ex != 0) {
    const float mf = (float)__longlong_as_double((b & 0x000FFFFFFFFFFFFFLL) | 0x3FF0000000000000LL);
    const double r = ((double)(ex - 1023) + (double)__log2f(mf)) * inv_lg2;
    if (fabs(r - rint(r)) > thr) return r;
  }
  return rdist_value(v, g, lg, inv_lg, T);
}

// The estimate alone; `need` is set when the element must take the full path
// (non-positive / non-finite / subnormal input, or within thr of an integer).
// The estimate uses the same table reduction as fast_log but only the first two
// Taylor terms (error < (2^-7)^3/3 < 1e-6 in log y) and no int/float
// conversions (the exponent becomes a double through the 2^52 magic number):
// ~10 FP64 ops. thr must exceed 1e-6 * |1/log gamma|.
RDB_DEV double dceil_estimate(double v, double inv_lg, double thr, const LogTab& T, bool& need) {
  const long long b = __double_as_longlong(v);
  const int ex = (int)(b >> 52);  // sign bit set (v <= -0) -> ex < 0 -> need
  const int idx = (int)((b >> 45) & 127);
  const double m = __longlong_as_double((b & 0x000FFFFFFFFFFFFFLL) | 0x3FF0000000000000LL);
  const long long eb = (long long)(ex - 1023 + (idx >= 53 ? 1 : 0) + (1 << 21));
  const double e = __longlong_as_double(0x4330000000000000LL + eb) - 4503599629467648.0;  // 2^52 + 2^21
  const double r = fma(m, T.C(idx), -1.0);
  const double lny = fma(e, 0.6931471805599453, T.H(idx) + fma(-0.5 * r, r, r));
  const double q = lny * inv_lg;
  need = (ex <= 0) | (ex >= 2047) | !(fabs(q - rint(q)) > thr);
  return q;
}

// Output kinds of D: none, int32 (INT32_MAX sentinel) or uint8 (compact,
// lossless while 0 <= D <= RDB_D8_MAX; RDB_D8_UNREACHABLE = +inf).
enum { DK_NONE = 0, DK_I32 = 1, DK_U8 = 2 };

template <bool HAS_R, bool HAS_DC, int DK>
struct Sink {
  double* r;
  double* dc;
  int32_t* d32;
  uint8_t* d8;
  // ceil to int32 in one saturating conversion: +inf -> INT_MAX (the sentinel)
  RDB_DEV static int32_t to_i32(double rv) { return __double2int_ru(rv); }
  // ceil to uint8; `bad` counts finite D outside [0, RDB_D8_MAX] (and NaN):
  // the caller must not use the uint8 D of such a matrix
  RDB_DEV static uint8_t to_u8(double rv, unsigned& bad) {
    if (rv == __longlong_as_double(0x7FF0000000000000LL)) return RDB_D8_UNREACHABLE;
    const double c = ceil(rv);
    const bool ok = c >= 0.0 && c <= (double)RDB_D8_MAX;  // false for NaN
    bad += !ok;
    return ok ? (uint8_t)(int)c : (uint8_t)RDB_D8_MAX;
  }
  // each returns the number of out-of-range uint8 entries written (0 otherwise)
  RDB_DEV unsigned put1(int64_t o, double rv) const {
    unsigned bad = 0;
    if (HAS_R) r[o] = rv;
    if (HAS_DC) dc[o] = ceil(rv);
    if (DK == DK_I32) d32[o] = to_i32(rv);
    if (DK == DK_U8) d8[o] = to_u8(rv, bad);
    return bad;
  }
  RDB_DEV unsigned put2(int64_t o, double r0, double r1) const {
    unsigned bad = 0;
    if (HAS_R) *reinterpret_cast<double2*>(r + o) = make_double2(r0, r1);
    if (HAS_DC) *reinterpret_cast<double2*>(dc + o) = make_double2(ceil(r0), ceil(r1));
    if (DK == DK_I32) *reinterpret_cast<int2*>(d32 + o) = make_int2(to_i32(r0), to_i32(r1));
    if (DK == DK_U8) {
      const uint8_t a = to_u8(r0, bad), b = to_u8(r1, bad);
      *reinterpret_cast<uchar2*>(d8 + o) = make_uchar2(a, b);
    }
    return bad;
  }
};

// rows x cols block of a larger matrix: global row of local row i is row0 + i,
// global column of local column j is gcol[j] (or col0 + j); the distance
// diagonal (forced 0) is where they coincide.
struct Shape {
  int64_t rows, cols, row0, col0;
  const int64_t* gcol;
  RDB_DEV int64_t gc(int64_t j) const { return gcol ? gcol[j] : col0 + j; }
};

template <bool HAS_R, bool HAS_DC, int DK, bool VEC>
__global__ void __launch_bounds__(256)
    log_ceil_kernel(const double* __restrict__ y, Shape sh, int64_t ldy, int64_t stride_y,
                    int64_t batch, const double* __restrict__ gammas, double gamma,
                    Sink<HAS_R, HAS_DC, DK> sink, int64_t ldo, int64_t stride_o,
                    const uint8_t* __restrict__ reach, int64_t ldm,
                    unsigned long long* __restrict__ counters) {
  __shared__ LogTab tab;
  for (int e = threadIdx.x; e < 128 * 16; e += blockDim.x) {
    const int i = e >> 4, k = e & 15;
    tab.c[i][k] = logtab::kC[i];
    tab.hi[i][k] = logtab::kLhi[i];
    tab.lo[i][k] = logtab::kLlo[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t n = sh.cols;
  const int64_t rows = sh.rows * batch;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < rows; w += nwarps) {
    const int64_t b = w / sh.rows, i = w - b * sh.rows;
    const int64_t gi = sh.row0 + i;
    const bool mapped = sh.gcol != nullptr;
    const int64_t dj = gi - sh.col0;  // local diagonal column when not mapped
    const double g = gammas ? gammas[b] : gamma;
    const double lg = log(g);
    const double inv_lg = 1.0 / lg;
    const double inv_lg2 = 0.6931471805599453 * inv_lg;  // 1 / log2(gamma)
    const float inv_lg2f = (float)inv_lg2, thr0 = (float)(1e-6 * fabs(inv_lg2));
    // 7x the MUFU estimate's error bound (4.1e-7 |1/log2 gamma| = 2.85e-7 |1/log gamma|)
    // and 12x the table estimate's (1.6e-7 |1/log gamma|). No cap: for gamma
    // near 1 the bound exceeds 1/2 and every element takes the exact path.
    const double thr = 2e-6 * fabs(inv_lg);
    auto val = [&](double v) -> double {
      return HAS_R ? rdist_value(v, g, lg, inv_lg, tab) : dceil_value(v, g, lg, inv_lg, inv_lg2, thr, tab);
    };
    const double* Y = y + b * stride_y + i * ldy;
    const int64_t orow = b * stride_o + i * ldo;
    const uint8_t* M = reach ? reach + i * ldm : nullptr;
    unsigned neg = 0, under = 0, bad = 0;
    int64_t jstart = 0;
    if (VEC) {
      // main body: 4 chunks of 64 columns per pass, all loads issued before any
      // math (memory-level parallelism for an HBM-bound row sweep)
      constexpr int U = 2;
      // software pipelining: the next block's loads are in flight while this
      // block computes
      double2 nxt[U];
      if (64 * U <= n) {
#pragma unroll
        for (int u = 0; u < U; ++u) nxt[u] = ldg2(Y + 64 * u + 2 * lane);
      }
      for (; jstart + 64 * U <= n; jstart += 64 * U) {
        double2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = nxt[u];
        if (jstart + 128 * U <= n) {
#pragma unroll
          for (int u = 0; u < U; ++u) nxt[u] = ldg2(Y + jstart + 64 * U + 64 * u + 2 * lane);
        }
        unsigned needbits = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t j = jstart + 64 * u + 2 * lane;
          const bool d0 = mapped ? gi == sh.gcol[j] : j == dj;
          const bool d1 = mapped ? gi == sh.gcol[j + 1] : j + 1 == dj;
          double r0, r1;
          if (HAS_R) {
            r0 = val(v[u].x);
            r1 = val(v[u].y);
          } else {
            // D only: cheap estimate now, exact path for the flagged few below
            bool n0, n1;
            r0 = dceil_estimate(v[u].x, inv_lg, thr, tab, n0);
            r1 = dceil_estimate(v[u].y, inv_lg, thr, tab, n1);
            needbits |= ((unsigned)(n0 && !d0) << (2 * u)) | ((unsigned)(n1 && !d1) << (2 * u + 1));
            // flagged entries are rewritten by the exact path below: store a
            // neutral provisional value (never counted as out of range)
            r0 = n0 ? 0.0 : r0;
            r1 = n1 ? 0.0 : r1;
          }
          r0 = d0 ? 0.0 : r0;
          r1 = d1 ? 0.0 : r1;
          bad += sink.put2(orow + j, r0, r1);
          neg += (v[u].x < NEGATIVE_ENTRY_TOL) + (v[u].y < NEGATIVE_ENTRY_TOL);
          if (M) under += (v[u].x == 0.0 && !d0 && M[j]) + (v[u].y == 0.0 && !d1 && M[j + 1]);
        }
        while (needbits) {  // rare: re-read the element (cache hit) and take the full path
          const int k = __ffs(needbits) - 1;
          needbits &= needbits - 1;
          const int64_t jj = jstart + 64 * (k >> 1) + 2 * lane + (k & 1);
          bad += sink.put1(orow + jj, rdist_value(Y[jj], g, lg, inv_lg, tab));
        }
      }
    }
    for (int64_t j0 = jstart; j0 < n; j0 += 64) {
      const int64_t j = j0 + 2 * lane;
      if (VEC && j + 1 < n) {
        const double2 v = ldg2(Y + j);
        const bool d0 = mapped ? gi == sh.gcol[j] : j == dj;
        const bool d1 = mapped ? gi == sh.gcol[j + 1] : j + 1 == dj;
        double r0 = val(v.x);
        double r1 = val(v.y);
        r0 = d0 ? 0.0 : r0;
        r1 = d1 ? 0.0 : r1;
        bad += sink.put2(orow + j, r0, r1);
        neg += (v.x < NEGATIVE_ENTRY_TOL) + (v.y < NEGATIVE_ENTRY_TOL);
        if (M) under += (v.x == 0.0 && !d0 && M[j]) + (v.y == 0.0 && !d1 && M[j + 1]);
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t jj = j + e;
          if (jj < n) {
            const double v = Y[jj];
            const bool dg = mapped ? gi == sh.gcol[jj] : jj == dj;
            bad += sink.put1(orow + jj, dg ? 0.0 : val(v));
            neg += (v < NEGATIVE_ENTRY_TOL);
            if (M) under += (v == 0.0 && !dg && M[jj]);
          }
        }
      }
    }
    if (counters) {
      neg = __reduce_add_sync(0xffffffffu, neg);
      under = __reduce_add_sync(0xffffffffu, under);
      if (DK == DK_U8) bad = __reduce_add_sync(0xffffffffu, bad);
      if (lane == 0) {
        if (neg) atomicAdd(&counters[b * RDB_NCOUNTERS + RDB_CNT_NEGATIVE], (unsigned long long)neg);
        if (under) atomicAdd(&counters[b * RDB_NCOUNTERS + RDB_CNT_UNDERFLOW], (unsigned long long)under);
        if (DK == DK_U8 && bad) atomicAdd(&counters[b * RDB_NCOUNTERS + RDB_CNT_D8_RANGE], (unsigned long long)bad);
      }
    }
  }
}

// Lean D-only estimate for the batch kernels: dceil_estimate in 32-bit integer
// arithmetic (high/low words instead of 64-bit shifts and adds), the table row
// given by a per-lane base pointer. Same value and same `need` rule.
struct LeanTab {
  const double* c;  // &tab.c[0][lane & 15]
  const double* h;  // &tab.hi[0][lane & 15]
};

RDB_DEV double dceil_estimate_lean(double v, double inv_lg, double thr, LeanTab T, bool& need) {
  const int hi = __double2hiint(v), lo = __double2loint(v);
  const int ex = hi >> 20;  // sign bit set (v <= -0) -> ex < 0 -> need
  const int idx = (hi >> 13) & 127;
  const double m = __hiloint2double((hi & 0x000FFFFF) | 0x3FF00000, lo);
  const int eb = ex - 1023 + (idx >= 53 ? 1 : 0);
  const double e = __hiloint2double(0x43300000, eb + 0x40000000) - 4503600701112320.0;  // 2^52 + 2^30
  const double r = fma(m, T.c[idx * 16], -1.0);
  const double lny = fma(e, 0.6931471805599453, T.h[idx * 16] + fma(-0.5 * r, r, r));
  const double q = lny * inv_lg;
  need = (ex <= 0) | (ex >= 2047) | !(fabs(q - rint(q)) > thr);
  return q;
}

// The same estimate with the mantissa's log2 from MUFU.LG2 on its leading 23
// bits (dceil_value's estimate: absolute error < 4.1e-7 in log2 y, so the
// quotient's error is < 4.1e-7 / |log2 gamma| < thr / 7 with thr as below): no
// table lookups. need as dceil_estimate_lean (non-positive, subnormal,
// non-finite, or within thr of an integer).
RDB_DEV double dceil_estimate_mufu(double v, double inv_lg2, double thr, bool& need) {
  const int hi = __double2hiint(v), lo = __double2loint(v);
  const int ex = hi >> 20;  // sign bit set (v <= -0) -> ex < 0 -> need
  const float mf = __int_as_float(((hi & 0x000FFFFF) << 3) | ((unsigned)lo >> 29) | 0x3F800000);
  const double q = ((double)(ex - 1023) + (double)__log2f(mf)) * inv_lg2;
  need = ((unsigned)(ex - 1) >= 2046u) | !(fabs(q - rint(q)) > thr);
  return q;
}

// The same decision in FP32 (the FP32 pipe issues twice the FP64 rate and the
// ceil is one F2I): s = (ex - 1023) + lg2(mantissa, 23 bits) rounded to float,
// q = s * (1 / log2 gamma) in float. Error of q against the true quotient:
// mantissa truncation (2^-23 / ln 2 = 1.72e-7) + MUFU.LG2 (2^-22 = 2.38e-7)
// < 4.1e-7 in log2 y, the float rounding of s < 6e-8 |s|, of 1/log2 gamma and
// of the product < 6e-8 |q| each, so |err| < 4.1e-7 |1/log2 gamma| +
// 1.8e-7 |q|. need unless q is more than thr0 + 4e-7 |q| (thr0 = 1e-6
// |1/log2 gamma|) from an integer, i.e. more than twice the bound (2.4x and
// 2.2x per term); the reference's own fp64 quotient is within ~1e-15 of the
// true one, so then both ceilings agree. q - rint(q) is exact in float.
RDB_DEV int dceil_estimate_f32(double v, float inv_lg2f, float thr0, bool& need) {
  const int hi = __double2hiint(v), lo = __double2loint(v);
  const int ex = hi >> 20;  // sign bit set (v <= -0) -> ex < 0 -> need
  const float mf = __int_as_float(((hi & 0x000FFFFF) << 3) | ((unsigned)lo >> 29) | 0x3F800000);
  // lg2.approx.ftz: mf is in [1, 2), never subnormal, so the flush-to-zero
  // form drops __log2f's subnormal guard (3 instructions per element); its
  // absolute error on [1, 2) is below 2^-22, the bound used above
  float lg2m;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg2m) : "f"(mf));
  const float q = ((float)(ex - 1023) + lg2m) * inv_lg2f;
  need = ((unsigned)(ex - 1) >= 2046u) | !(fabsf(q - rintf(q)) > fmaf(4e-7f, fabsf(q), thr0));
  return __float2int_ru(q);
}

// The lean kernel's exact path (rare): out of line by default, so its
// registers do not count against the streaming loop's.
#ifndef RDB_K3_NOINLINE
#define RDB_K3_NOINLINE 0
#endif
#if RDB_K3_NOINLINE
__device__ __noinline__
#else
RDB_DEV
#endif
double exact_value(double v, double g, double lg, double inv_lg) {
  return rdist_value(v, g, lg, inv_lg, ConstTab{});
}

// D-only K3 for whole n x n matrices, the batch path (no mask, no column map):
// one warp per row, each lane owns 4 consecutive columns of a 128-column block
// (two 16-byte loads; a warp stores 128 contiguous bytes of uint8 D or 512 of
// int32 D), two blocks in flight per lane. uint8 D: `bad` counts entries
// outside [0, RDB_D8_MAX] (RDB_CNT_D8_RANGE).
// one block of loads in flight ahead, main loop not unrolled, registers capped
// at 64 (4 blocks per SM; the common path needs no shared table): measured
// best of PF 1-2 x unroll 1-2 x 1/4/5/6 blocks per SM on the config-2 batch
// (tools/time_k3.py: uint8 D 0.56 -> 0.48 ms, int32 D 0.61 -> 0.53 ms)
#ifndef RDB_K3_MUFU
#define RDB_K3_MUFU 1
#endif
#ifndef RDB_K3_F32
#define RDB_K3_F32 1  // the MUFU estimate in FP32 (dceil_estimate_f32)
#endif
#ifndef LEAN_PF
#define LEAN_PF 1
#endif
#ifndef LEAN_UNROLL
#define LEAN_UNROLL 1
#endif
#ifndef LEAN_MINB
#define LEAN_MINB 4
#endif
#ifndef LEAN_GRID_PER_SM
#define LEAN_GRID_PER_SM 64  // uint8 D: 64 blocks per SM of grid (0.461 -> 0.456 ms vs 16; tools/time_k3.py)
#endif
constexpr int kLeanUnroll = LEAN_UNROLL;
template <int DK>
__global__ void __launch_bounds__(256, LEAN_MINB)
    log_ceil_lean_kernel(const double* __restrict__ y, int64_t n, int64_t ldy, int64_t stride_y, int64_t batch,
                         const double* __restrict__ gammas, double gamma, void* __restrict__ dout, int64_t ldo,
                         int64_t stride_o, unsigned long long* __restrict__ counters) {
  RDB_TRACE_SCOPE(50);
#if RDB_K3_MUFU
  const ConstTab tab;  // exact path only
  const int lane = threadIdx.x & 31;
#else
  __shared__ LogTab tab;
  for (int e = threadIdx.x; e < 128 * 16; e += blockDim.x) {
    const int i = e >> 4, k = e & 15;
    tab.c[i][k] = logtab::kC[i];
    tab.hi[i][k] = logtab::kLhi[i];
    tab.lo[i][k] = logtab::kLlo[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const LeanTab lt{&tab.c[0][lane & 15], &tab.hi[0][lane & 15]};
#endif
  const int64_t rows = n * batch;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int nfull = (int)(n & ~(int64_t)127);
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < rows; w += nwarps) {
    const int64_t b = w / n;
    const int i = (int)(w - b * n);
    const double g = gammas ? gammas[b] : gamma;
    const double lg = log(g);
    const double inv_lg = 1.0 / lg;
    const double thr = 2e-6 * fabs(inv_lg);  // as log_ceil_kernel's (no cap)
    const double* Y = y + b * stride_y + (int64_t)i * ldy;
    const int64_t orow = b * stride_o + (int64_t)i * ldo;
    unsigned neg = 0, bad = 0;
#if RDB_K3_MUFU
    const double inv_lg2 = 0.6931471805599453 * inv_lg;  // 1 / log2(gamma)
    const float inv_lg2f = (float)inv_lg2, thr0 = (float)(1e-6 * fabs(inv_lg2));
    // common path: the estimate, diagonal 0; D > RDB_D8_MAX or < 0 (u8) are
    // tracked by an unsigned max and counted below only when it exceeds the range
    unsigned dmax = 0;
#endif
    auto block = [&](int j, double2 p, double2 q) {
      const double v[4] = {p.x, p.y, q.x, q.y};
      int d[4];
#if RDB_K3_MUFU && RDB_K3_F32
      // The estimates' `need` flags stay predicates and the estimates are used
      // as they come: a block with a flag set (rare) resolves those elements
      // on the exact path; uint8 D leaves through a saturating pack (two
      // I2IP), so the common path has no per-element select, clamp or byte
      // permute. A common-path D outside 0 .. RDB_D8_MAX (stored saturated;
      // the matrix is redone in int32) is tracked by an unsigned max.
      bool nd[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) d[e] = dceil_estimate_f32(v[e], inv_lg2f, thr0, nd[e]);
      // (the block holding the diagonal, one in n / 4, goes the rare way too: D = 0 there)
      if (nd[0] | nd[1] | nd[2] | nd[3] | ((unsigned)(i - j) < 4u)) {  // rare (static indices keep v / d in registers)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (j + e == i) {
            d[e] = 0;
          } else if (nd[e]) {  // exact path
            const double r = exact_value(v[e], g, lg, inv_lg);
            d[e] = __double2int_ru(r);  // +inf -> INT32_MAX, the int32 sentinel
            neg += v[e] < NEGATIVE_ENTRY_TOL;  // a negative entry always takes this path (sign bit -> need)
            if (DK == DK_U8) {
              const bool unreachable = r == __longlong_as_double(0x7FF0000000000000LL);
              const bool ok = r == r && (unsigned)d[e] <= (unsigned)RDB_D8_MAX;  // NaN: out of range
              bad += !ok && !unreachable;
              d[e] = unreachable ? RDB_D8_UNREACHABLE : (ok ? d[e] : RDB_D8_MAX);
            }
          } else if (DK == DK_U8) {
            dmax = max(dmax, (unsigned)d[e]);
          }
        }
      } else if (DK == DK_U8) {
        dmax = max(max(dmax, max((unsigned)d[0], (unsigned)d[1])), max((unsigned)d[2], (unsigned)d[3]));
      }
      if (DK == DK_U8) {
        unsigned hi16, w;
        asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(hi16) : "r"(d[3]), "r"(d[2]), "r"(0));
        asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(w) : "r"(d[1]), "r"(d[0]), "r"(hi16));
        *reinterpret_cast<unsigned*>(static_cast<uint8_t*>(dout) + orow + j) = w;
      } else {
        *reinterpret_cast<int4*>(static_cast<int32_t*>(dout) + orow + j) = make_int4(d[0], d[1], d[2], d[3]);
      }
#else
      unsigned need = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        bool nd;
        const bool dg = j + e == i;
#if RDB_K3_MUFU
        const double r = dceil_estimate_mufu(v[e], inv_lg2, thr, nd);
#else
        const double r = dceil_estimate_lean(v[e], inv_lg, thr, lt, nd);
#endif
        need |= (unsigned)(nd && !dg) << e;
        d[e] = (dg || nd) ? 0 : __double2int_ru(r);
#if !RDB_K3_MUFU
        neg += v[e] < NEGATIVE_ENTRY_TOL;
#endif
      }
      if (need) {  // rare: exact path (static indices keep v / d in registers)
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (need & (1u << e)) {
            const double r = exact_value(v[e], g, lg, inv_lg);
            d[e] = __double2int_ru(r);  // +inf -> INT32_MAX, the int32 sentinel
            if (DK == DK_U8 && r == __longlong_as_double(0x7FF0000000000000LL)) d[e] = -2;  // unreachable
            if (DK == DK_U8 && r != r) d[e] = -1;  // NaN: out of range
#if RDB_K3_MUFU
            neg += v[e] < NEGATIVE_ENTRY_TOL;  // a negative entry always takes this path (sign bit -> need)
            if (DK == DK_U8) {  // resolve here: the common path below sees only 0 .. 254 or a range error
              const bool unreachable = d[e] == -2;
              const bool ok = (unsigned)d[e] <= (unsigned)RDB_D8_MAX;
              bad += !ok && !unreachable;
              d[e] = unreachable ? RDB_D8_UNREACHABLE : (ok ? d[e] : RDB_D8_MAX);
            }
#endif
          }
      }
#if RDB_K3_MUFU
      if (DK == DK_U8) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const unsigned u = (need >> e) & 1u ? 0u : (unsigned)d[e];  // exact-path values already resolved
          dmax = max(dmax, u);
          d[e] = (need >> e) & 1u ? d[e] : (int)min(u, (unsigned)RDB_D8_MAX);
        }
#else
      if (DK == DK_U8) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const bool unreachable = d[e] == -2;
          const bool ok = (unsigned)d[e] <= (unsigned)RDB_D8_MAX;
          bad += !ok && !unreachable;
          d[e] = unreachable ? RDB_D8_UNREACHABLE : (ok ? d[e] : RDB_D8_MAX);
        }
#endif
        *reinterpret_cast<uchar4*>(static_cast<uint8_t*>(dout) + orow + j) =
            make_uchar4((uint8_t)d[0], (uint8_t)d[1], (uint8_t)d[2], (uint8_t)d[3]);
      } else {
        *reinterpret_cast<int4*>(static_cast<int32_t*>(dout) + orow + j) = make_int4(d[0], d[1], d[2], d[3]);
      }
#endif
    };
    // LEAN_PF blocks of loads in flight ahead of the one being converted
    constexpr int PF = LEAN_PF;
    double2 pp[PF], qq[PF];
#pragma unroll
    for (int u = 0; u < PF; ++u)
      if (128 * (u + 1) <= nfull) {
        pp[u] = ldg2(Y + 128 * u + 4 * lane);
        qq[u] = ldg2(Y + 128 * u + 4 * lane + 2);
      }
    int j0 = 0;
#pragma unroll kLeanUnroll
    for (; j0 + 128 <= nfull; j0 += 128) {
      const double2 p0 = pp[0], q0 = qq[0];
#pragma unroll
      for (int u = 0; u + 1 < PF; ++u) {
        pp[u] = pp[u + 1];
        qq[u] = qq[u + 1];
      }
      if (j0 + 128 * (PF + 1) <= nfull) {
        pp[PF - 1] = ldg2(Y + j0 + 128 * PF + 4 * lane);
        qq[PF - 1] = ldg2(Y + j0 + 128 * PF + 4 * lane + 2);
      }
      block(j0 + 4 * lane, p0, q0);
    }
    for (int j = j0 + lane; j < n; j += 32) {  // ragged tail (n % 128)
      const double v = Y[j];
      const double r = (j == i) ? 0.0 : rdist_value(v, g, lg, inv_lg, tab);
      if (DK == DK_U8) {
        unsigned bb = 0;
        static_cast<uint8_t*>(dout)[orow + j] = Sink<false, false, DK_U8>::to_u8(r, bb);
        bad += bb;
      } else {
        static_cast<int32_t*>(dout)[orow + j] = __double2int_ru(r);
      }
      neg += v < NEGATIVE_ENTRY_TOL;
    }
#if RDB_K3_MUFU
    if (lane == 0 && i < nfull) neg += Y[i] < NEGATIVE_ENTRY_TOL;  // the diagonal (skips the exact path)
    if (DK == DK_U8 && __any_sync(0xffffffffu, dmax > (unsigned)RDB_D8_MAX)) {
      // rare: some common-path D left 0 .. 254; count them (the stored value is
      // already the clamp): re-derive the row's common-path D's
      for (int j = lane; j < nfull; j += 32) {
        bool nd;
#if RDB_K3_F32
        const int de = dceil_estimate_f32(Y[j], inv_lg2f, thr0, nd);
#else
        const int de = __double2int_ru(dceil_estimate_mufu(Y[j], inv_lg2, thr, nd));
#endif
        if (!nd && j != i) bad += (unsigned)de > (unsigned)RDB_D8_MAX;
      }
    }
#endif
    if (counters) {
      neg = __reduce_add_sync(0xffffffffu, neg);
      if (DK == DK_U8) bad = __reduce_add_sync(0xffffffffu, bad);
      if (lane == 0) {
        if (neg) atomicAdd(&counters[b * RDB_NCOUNTERS + RDB_CNT_NEGATIVE], (unsigned long long)neg);
        if (DK == DK_U8 && bad) atomicAdd(&counters[b * RDB_NCOUNTERS + RDB_CNT_D8_RANGE], (unsigned long long)bad);
      }
    }
  }
}

template <bool A, bool B, int C>
static void launch(bool vec, unsigned blocks, cudaStream_t st, const double* y, Shape n, int64_t ldy,
                   int64_t stride_y, int64_t batch, const double* gammas, double gamma, double* r,
                   double* dc, int32_t* d32, int64_t ldo, int64_t stride_o, const uint8_t* reach,
                   int64_t ldm, unsigned long long* counters, uint8_t* d8 = nullptr) {
  Sink<A, B, C> sink{r, dc, d32, d8};
  if (vec)
    log_ceil_kernel<A, B, C, true><<<blocks, 256, 0, st>>>(y, n, ldy, stride_y, batch, gammas, gamma, sink,
                                                           ldo, stride_o, reach, ldm, counters);
  else
    log_ceil_kernel<A, B, C, false><<<blocks, 256, 0, st>>>(y, n, ldy, stride_y, batch, gammas, gamma, sink,
                                                            ldo, stride_o, reach, ldm, counters);
}

int log_ceil_shaped(const double* y, Shape sh, int64_t ldy, int64_t stride_y, int64_t batch,
                    const double* gammas, double gamma, double* r_out, double* dceil_out,
                    int32_t* d32_out, int64_t ldo, int64_t stride_o, const uint8_t* reachable,
                    int64_t ldm, unsigned long long* counters, cudaStream_t st) {
  const int64_t n = sh.cols;
  if (!y || sh.rows <= 0 || n <= 0 || ldy < n || batch <= 0) return RDB_EINVAL;
  if ((r_out || dceil_out || d32_out) && ldo < n) return RDB_EINVAL;
  if (reachable && ldm < n) return RDB_EINVAL;
  if (!gammas && !(gamma > 0.0 && gamma < 1.0)) return RDB_EINVAL;
  auto al = [](const void* p, uintptr_t a) { return p == nullptr || ((uintptr_t)p % a) == 0; };
  const bool vec = !(ldy & 1) && !(stride_y & 1) && !(ldo & 1) && !(stride_o & 1) && al(y, 16) &&
                   al(r_out, 16) && al(dceil_out, 16) && al(d32_out, 8);
  const int64_t rows = sh.rows * batch;
  const int key = (r_out ? 4 : 0) | (dceil_out ? 2 : 0) | (d32_out ? 1 : 0);
  const int64_t want = (rows + 7) / 8;
  const unsigned blocks = (unsigned)(want < 148 * 16 ? want : 148 * 16);
  if (key == 1 && vec && !reachable && !sh.gcol && sh.row0 == 0 && sh.col0 == 0 && sh.rows == n &&
      !(ldo & 3) && !(stride_o & 3) && al(d32_out, 16) && n < (int64_t)1 << 31) {
    log_ceil_lean_kernel<DK_I32><<<blocks, 256, 0, st>>>(y, n, ldy, stride_y, batch, gammas, gamma, d32_out, ldo,
                                                         stride_o, counters);
    RDB_LAUNCH_CHECK();
    return RDB_OK;
  }
#define RDB_LC(K, A, B, C)                                                                       \
  case K:                                                                                        \
    launch<A, B, C>(vec, blocks, st, y, sh, ldy, stride_y, batch, gammas, gamma, r_out, dceil_out, \
                    d32_out, ldo, stride_o, reachable, ldm, counters);                           \
    break;
  switch (key) {
    RDB_LC(0, false, false, DK_NONE)
    RDB_LC(1, false, false, DK_I32)
    RDB_LC(2, false, true, DK_NONE)
    RDB_LC(3, false, true, DK_I32)
    RDB_LC(4, true, false, DK_NONE)
    RDB_LC(5, true, false, DK_I32)
    RDB_LC(6, true, true, DK_NONE)
    RDB_LC(7, true, true, DK_I32)
  }
#undef RDB_LC
  RDB_LAUNCH_CHECK();
  return RDB_OK;
}

int log_ceil(const double* y, int64_t n, int64_t ldy, int64_t stride_y, int64_t batch,
             const double* gammas, double gamma, double* r_out, double* dceil_out, int32_t* d32_out,
             int64_t ldo, int64_t stride_o, const uint8_t* reachable, int64_t ldm,
             unsigned long long* counters, cudaStream_t st) {
  return log_ceil_shaped(y, Shape{n, n, 0, 0, nullptr}, ldy, stride_y, batch, gammas, gamma, r_out,
                         dceil_out, d32_out, ldo, stride_o, reachable, ldm, counters, st);
}

int log_ceil_d8(const double* y, int64_t n, int64_t ldy, int64_t stride_y, int64_t batch,
                const double* gammas, double gamma, uint8_t* d8_out, int64_t ldo, int64_t stride_o,
                unsigned long long* counters, cudaStream_t st) {
  if (!y || !d8_out || !counters || n <= 0 || ldy < n || ldo < n || batch <= 0) return RDB_EINVAL;
  if (!gammas && !(gamma > 0.0 && gamma < 1.0)) return RDB_EINVAL;
  auto al = [](const void* p, uintptr_t a) { return ((uintptr_t)p % a) == 0; };
  const int64_t rows = n * batch;
  const int64_t want = (rows + 7) / 8;
  const unsigned blocks = (unsigned)(want < 148 * LEAN_GRID_PER_SM ? want : 148 * LEAN_GRID_PER_SM);
  if (!(ldy & 1) && !(stride_y & 1) && !(ldo & 3) && !(stride_o & 3) && al(y, 16) && al(d8_out, 4) &&
      n < (int64_t)1 << 31) {
    log_ceil_lean_kernel<DK_U8><<<blocks, 256, 0, st>>>(y, n, ldy, stride_y, batch, gammas, gamma, d8_out, ldo,
                                                        stride_o, counters);
  } else {
    launch<false, false, DK_U8>(false, blocks, st, y, Shape{n, n, 0, 0, nullptr}, ldy, stride_y, batch, gammas,
                                gamma, nullptr, nullptr, nullptr, ldo, stride_o, nullptr, 0, counters, d8_out);
  }
  RDB_LAUNCH_CHECK();
  return RDB_OK;
}

}  // namespace rdb

extern "C" int rdb_log_ceil_d8(const double* y, int64_t n, int64_t ldy, int64_t stride_y, int64_t batch,
                               const double* gammas, double gamma, uint8_t* d8_out, int64_t ldo,
                               int64_t stride_o, unsigned long long* counters, void* stream) {
  return rdb::log_ceil_d8(y, n, ldy, stride_y, batch, gammas, gamma, d8_out, ldo, stride_o, counters,
                          static_cast<cudaStream_t>(stream));
}

extern "C" int rdb_log_ceil_block(const double* y, int64_t rows, int64_t cols, int64_t ldy,
                                  int64_t row0, int64_t col0, const int64_t* gcol, double gamma,
                                  double* r_out, double* dceil_out, int32_t* d32_out, int64_t ldo,
                                  unsigned long long* counters, void* stream) {
  return rdb::log_ceil_shaped(y, rdb::Shape{rows, cols, row0, col0, gcol}, ldy, 0, 1, nullptr, gamma, r_out,
                              dceil_out, d32_out, ldo, 0, nullptr, 0, counters,
                              static_cast<cudaStream_t>(stream));
}

extern "C" int rdb_log_ceil(const double* y, int64_t n, int64_t ldy, int64_t stride_y, int64_t batch,
                            const double* gammas, double gamma, double* r_out, double* dceil_out,
                            int32_t* d32_out, int64_t ldo, int64_t stride_o,
                            const uint8_t* reachable, int64_t ldm, unsigned long long* counters,
                            void* stream) {
  return rdb::log_ceil(y, n, ldy, stride_y, batch, gammas, gamma, r_out, dceil_out, d32_out, ldo,
                       stride_o, reachable, ldm, counters, static_cast<cudaStream_t>(stream));
}

#ifdef RDB_TRACE
namespace rdb {
namespace k3 {
int trace_attach(void* buf, unsigned cap) { return trace::attach(buf, cap); }
}  // namespace k3
}  // namespace rdb
#endif
