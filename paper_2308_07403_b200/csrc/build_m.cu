// K1: X = gamma^W / M = I - gamma^W, elementwise and HBM-bound
// (reference: np.power(gamma, W) at pkg/src/rdist/resolvent.py:98 and
// np.eye(n) - x at resolvent.py:115), plus the matrix statistics the
// reference's lu_invert checks (linalg.py:27-29) and identity padding.
#include <cmath>

#include "common.cuh"

namespace rdb {

// gamma^w with the reference's special cases: w == 1 gives gamma exactly
// (IEEE pow(x, 1) == x; asserted bitwise by test_resolvent.py:72-75) and
// w == +inf gives 0 for 0 < gamma < 1.
RDB_DEV double gain_pow(double g, double w) {
  if (w == 1.0) return g;
  if (isinf(w) && w > 0) return 0.0;
  return pow(g, w);
}

// One thread per 2 columns of one row (grid-stride over rows).
__global__ void build_m_kernel(const double* __restrict__ w, int64_t ldw, int64_t stride_w, int64_t n,
                               int64_t n_pad, const double* __restrict__ gammas, double gamma,
                               int mode, double* __restrict__ out, int64_t ldo, int64_t stride_o) {
  const int64_t b = blockIdx.z;
  const double g = gammas ? gammas[b] : gamma;
  const double* W = w + b * stride_w;
  double* O = out + b * stride_o;
  const int64_t ncols = (mode == RDB_BUILD_M) ? n_pad : n;
  for (int64_t i = blockIdx.y; i < ncols; i += gridDim.y) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < ncols;
         j += (int64_t)gridDim.x * blockDim.x) {
      double v;
      if (i < n && j < n) {
        const double x = gain_pow(g, W[i * ldw + j]);
        v = (mode == RDB_BUILD_M) ? ((i == j ? 1.0 : 0.0) - x) : x;
      } else {
        v = (i == j) ? 1.0 : 0.0;
      }
      O[i * ldo + j] = v;
    }
  }
}

// Bit-packed adjacency -> M. Thread handles 2 adjacent columns (double2 store).
__global__ void build_m_bits_kernel(const uint32_t* __restrict__ bits, int64_t n, int64_t n_pad,
                                    int64_t batch, const double* __restrict__ gammas, double gamma,
                                    double* __restrict__ out, int64_t ldo, int64_t stride_o,
                                    const int* __restrict__ nonband, const int* __restrict__ s0bad, int s0_w) {
  RDB_TRACE_SCOPE(51);
  // one warp per output row (grid-stride over batch * n_pad rows); lane l
  // writes columns 2l, 2l+1 of every 64-column chunk: 512 B per store wave.
  // nonband (APSP pipelines): a matrix the banded inverse takes (nonband[b] ==
  // 0) gets only the 64-column chunks covering its 32-block tridiagonal band,
  // the blocks band_factor_kernel reads (the inverse overwrites the rest).
  const int lane = threadIdx.x & 31;
  const int64_t wpr = (n + 31) / 32;
  const int64_t rows = n_pad * batch;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < rows; w += nwarps) {
    const int64_t b = w / n_pad, i = w - b * n_pad;
    const double ng = -(gammas ? gammas[b] : gamma);
    const uint32_t* row = bits + (b * n + i) * wpr;
    double* O = out + b * stride_o + i * ldo;
    int64_t jb = 0, je = n_pad;
    // dense-wide matrix with a sparse first step (flags 2, s0bad bit 1 clear):
    // only the 256 x 256 block M_00 (the first band inverse); the step writes
    // the rest from the bits (gj_invert.cu dw_s0_*). Two-level path (s0_w =
    // W > 0): bit 2 clear = a sparse outer step, so only the leading W x W
    // block (with bit 1 clear: only its 256 x 256 block M_00).
    if (s0bad && nonband[b] == 2) {
      const int f = s0bad[b];
      int64_t lim = n_pad;
      if (s0_w > 0) {
        if (!(f & 2)) lim = (f & 1) ? s0_w : 2 * NB;
      } else if (!(f & 1)) {
        lim = 2 * NB;
      }
      if (i >= lim) continue;
      je = lim;
    }
    if (nonband && !nonband[b]) {
      const int64_t bi = i / 32;
      jb = bi > 0 ? ((32 * (bi - 1)) & ~(int64_t)63) : 0;
      je = ((32 * (bi + 2) + 63) & ~(int64_t)63) < n_pad ? ((32 * (bi + 2) + 63) & ~(int64_t)63) : n_pad;
    }
    for (int64_t j0 = jb; j0 < je; j0 += 64) {
      const int64_t j = j0 + 2 * lane;
      const int64_t wi = j0 >> 5;  // two words cover this 64-column chunk
      uint32_t w0 = 0, w1 = 0;
      if (i < n) {
        if (wi < wpr) w0 = __ldg(row + wi);
        if (wi + 1 < wpr) w1 = __ldg(row + wi + 1);
      }
      const uint32_t word = (lane < 16) ? w0 : w1;
      const int sh = (2 * lane) & 31;
      double v0 = ((word >> sh) & 1u) && (j < n) ? ng : 0.0;
      double v1 = ((word >> (sh + 1)) & 1u) && (j + 1 < n) ? ng : 0.0;
      if (j == i) v0 = 1.0;
      if (j + 1 == i) v1 = 1.0;
      stg2(O + j, make_double2(v0, v1));
    }
  }
}

__global__ void pad_identity_kernel(double* __restrict__ a, int64_t n, int64_t n_pad, int64_t lda,
                                    int64_t stride) {
  double* A = a + (int64_t)blockIdx.z * stride;
  for (int64_t i = blockIdx.y; i < n_pad; i += gridDim.y) {
    const int64_t j_begin = (i < n) ? n : 0;
    for (int64_t j = j_begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_pad;
         j += (int64_t)gridDim.x * blockDim.x)
      A[i * lda + j] = (i == j) ? 1.0 : 0.0;
  }
}

// stats[0] max|a| (atomic on the bit pattern), [1] non-finite count,
// [2] Z-pattern violations, [3] negative entries.
__global__ void matrix_stats_kernel(const double* __restrict__ a, int64_t n, int64_t lda,
                                    double* __restrict__ stats) {
  double mx = 0.0;
  unsigned nonfinite = 0, nonz = 0, neg = 0;
  for (int64_t i = blockIdx.y; i < n; i += gridDim.y) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x) {
      const double v = a[i * lda + j];
      const double av = fabs(v);
      if (!(av <= 1.7976931348623157e308)) {
        ++nonfinite;
      } else {
        mx = fmax(mx, av);
      }
      if (i == j ? !(v > 0.0) : (v > 0.0)) ++nonz;
      if (v < 0.0) ++neg;
    }
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  nonfinite = __reduce_add_sync(0xffffffffu, nonfinite);
  nonz = __reduce_add_sync(0xffffffffu, nonz);
  neg = __reduce_add_sync(0xffffffffu, neg);
  if ((threadIdx.x & 31) == 0) {
    atomic_max_nonneg(&stats[0], mx);
    // counts are kept as doubles (exact below 2^53)
    if (nonfinite) atomicAdd(&stats[1], (double)nonfinite);
    if (nonz) atomicAdd(&stats[2], (double)nonz);
    if (neg) atomicAdd(&stats[3], (double)neg);
  }
}

static dim3 grid2d(int64_t cols, int64_t rows, int64_t batch, int threads, int per_thread = 1) {
  int64_t gx = (cols + (int64_t)threads * per_thread - 1) / ((int64_t)threads * per_thread);
  if (gx < 1) gx = 1;
  if (gx > 1024) gx = 1024;
  int64_t gy = rows < 1 ? 1 : rows;
  if (gy > 65535) gy = 65535;
  return dim3((unsigned)gx, (unsigned)gy, (unsigned)batch);
}

}  // namespace rdb

using namespace rdb;

extern "C" int rdb_build_m(const double* w, int64_t ldw, int64_t stride_w, int64_t n, int64_t n_pad,
                           int64_t batch, const double* gammas, double gamma, int mode, double* out,
                           int64_t ldo, int64_t stride_o, void* stream) {
  if (!w || !out || n <= 0 || batch <= 0 || batch > 65535 || ldw < n) return RDB_EINVAL;
  if (mode != RDB_BUILD_X && mode != RDB_BUILD_M) return RDB_EINVAL;
  if (mode == RDB_BUILD_M && n_pad < n) return RDB_EINVAL;
  const int64_t cols = (mode == RDB_BUILD_M) ? n_pad : n;
  if (ldo < cols) return RDB_EINVAL;
  if (!gammas && !(gamma > 0.0 && gamma < 1.0)) return RDB_EINVAL;
  build_m_kernel<<<grid2d(cols, cols, batch, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      w, ldw, stride_w, n, n_pad, gammas, gamma, mode, out, ldo, stride_o);
  RDB_LAUNCH_CHECK();
  return RDB_OK;
}

extern "C" int rdb_build_m_bits(const uint32_t* bits, int64_t n, int64_t n_pad, int64_t batch,
                                const double* gammas, double gamma, double* out, int64_t ldo,
                                int64_t stride_o, void* stream) {
  if (!bits || !out || n <= 0 || n_pad < n || (n_pad & 1) || (ldo & 1) || ldo < n_pad ||
      batch <= 0 || batch > 65535 || ((uintptr_t)out & 15))
    return RDB_EINVAL;
  if (!gammas && !(gamma > 0.0 && gamma < 1.0)) return RDB_EINVAL;
  if (n_pad % 64) return RDB_EINVAL;
  const int64_t rows = n_pad * batch;
  const int64_t blocks = (rows + 7) / 8 < 148 * 32 ? (rows + 7) / 8 : 148 * 32;
  build_m_bits_kernel<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      bits, n, n_pad, batch, gammas, gamma, out, ldo, stride_o, nullptr, nullptr, 0);
  RDB_LAUNCH_CHECK();
  return RDB_OK;
}

namespace rdb {
// The APSP pipelines' K1 (apsp.cu): as rdb_build_m_bits (same checks), band
// rows only for the matrices the banded inverse takes, the block M_00 only
// for the dense-wide matrices whose first step is sparse (s0bad, may be null).
int build_m_bits_banded(const uint32_t* bits, int64_t n, int64_t n_pad, int64_t batch, const double* gammas,
                        double* out, int64_t stride_o, const int* nonband, cudaStream_t st, const int* s0bad,
                        int s0_w) {
  if (!nonband) return rdb_build_m_bits(bits, n, n_pad, batch, gammas, 0.0, out, n_pad, stride_o, st);
  if (!bits || !out || !gammas || n <= 0 || n_pad < n || n_pad % 64 || batch <= 0 || batch > 65535 ||
      ((uintptr_t)out & 15))
    return RDB_EINVAL;
  const int64_t rows = n_pad * batch;
  const int64_t blocks = (rows + 7) / 8 < 148 * 32 ? (rows + 7) / 8 : 148 * 32;
  build_m_bits_kernel<<<(unsigned)blocks, 256, 0, st>>>(bits, n, n_pad, batch, gammas, 0.0, out, n_pad, stride_o,
                                                        nonband, s0bad, s0_w);
  RDB_LAUNCH_CHECK();
  return RDB_OK;
}
}  // namespace rdb

extern "C" int rdb_pad_identity(double* a, int64_t n, int64_t n_pad, int64_t lda, int64_t stride,
                                int64_t batch, void* stream) {
  if (!a || n < 0 || n_pad < n || lda < n_pad || batch <= 0 || batch > 65535) return RDB_EINVAL;
  if (n_pad == n) return RDB_OK;
  pad_identity_kernel<<<grid2d(n_pad, n_pad, batch, 256), 256, 0,
                        static_cast<cudaStream_t>(stream)>>>(a, n, n_pad, lda, stride);
  RDB_LAUNCH_CHECK();
  return RDB_OK;
}

extern "C" int rdb_matrix_stats(const double* a, int64_t n, int64_t lda, double* stats,
                                void* stream) {
  if (!a || !stats || n <= 0 || lda < n) return RDB_EINVAL;
  int64_t gy = n < 4096 ? n : 4096;
  matrix_stats_kernel<<<grid2d(n, gy, 1, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      a, n, lda, stats);
  RDB_LAUNCH_CHECK();
  return RDB_OK;
}

// Edge list (from, to) -> bit-packed adjacency in the rdb_build_m_bits row
// format (row `to`, bit `from`): the wire format feeding K1 directly
// (graphs.py:99-111 builds the dense W the same way, w[to, from] = weight).
__global__ void edges_to_bits_kernel(const int32_t* __restrict__ src, const int32_t* __restrict__ dst, int64_t m,
                                     int64_t wpr, uint32_t* __restrict__ bits) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = src[e], d = dst[e];
    atomicOr(&bits[(int64_t)d * wpr + (s >> 5)], 1u << (s & 31));
  }
}

extern "C" int rdb_edges_to_bits(const int32_t* src, const int32_t* dst, int64_t m, int64_t n, uint32_t* bits,
                                 void* stream) {
  if (!bits || n <= 0 || m < 0 || (m > 0 && (!src || !dst))) return RDB_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t wpr = (n + 31) / 32;
  if (cudaMemsetAsync(bits, 0, (size_t)(n * wpr) * sizeof(uint32_t), st) != cudaSuccess) return RDB_ECUDA;
  if (m == 0) return RDB_OK;
  const int64_t want = (m + 255) / 256;
  edges_to_bits_kernel<<<(unsigned)(want < 148 * 32 ? want : 148 * 32), 256, 0, st>>>(src, dst, m, wpr, bits);
  RDB_LAUNCH_CHECK();
  return RDB_OK;
}

#ifdef RDB_TRACE
namespace rdb {
namespace k1 {
int trace_attach(void* buf, unsigned cap) { return trace::attach(buf, cap); }
}  // namespace k1
}  // namespace rdb
#endif
