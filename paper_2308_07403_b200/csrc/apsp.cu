// Library entry points that chain the kernels, and error strings.
//
// rdb_apsp_bits_batched is the config-2 workload in one call: the reference's
// per-graph run_rdist closure (pkg/src/rdist/experiments.py:305-310:
// resolvent(with_residual=False) -> r_distance -> ceil) for a whole batch of
// unweighted graphs, with per-graph gains.
#include <cstdlib>

#include "common.cuh"

namespace rdb {
int invert_batched(double* a, int64_t n, int64_t lda, int64_t stride, int64_t batch, void* work,
                   rdb_pivot_info* info, cudaStream_t st, const uint32_t* bits, int64_t n_bits, bool band_ready,
                   int phase, const double* m_gammas, int** s0bad_out, int* s0_levels_out);
int* band_flags(void* work, int64_t n, int64_t batch);
int band_detect(const uint32_t* bits, int64_t n, int64_t batch, int* nonband, cudaStream_t st);
int build_m_bits_banded(const uint32_t* bits, int64_t n, int64_t n_pad, int64_t batch, const double* gammas,
                        double* out, int64_t stride_o, const int* nonband, cudaStream_t st, const int* s0bad,
                        int s0_w);

// K1 and K2 of the pipelines: the matrices are classified from the bits
// first (banded, dense-wide with a sparse first step, other), so K1 writes
// only what K2 reads: the band of a banded matrix, the block M_00 of a
// sparse-first-step matrix (K2 writes the rest from the bits), else all of M.
static int build_and_invert(const uint32_t* bits, int64_t n, int64_t n_pad, int64_t batch, const double* gammas,
                            double* mwork, void* work, rdb_pivot_info* info, cudaStream_t st) {
  const int64_t stride = n_pad * n_pad;
  int* nonband = band_flags(work, n_pad, batch);
  int* s0bad = nullptr;
  const char* e = getenv("RDB_GJ_DW_SYNTH");  // A-B switch: 0 builds all of M and lets K2 read it
  if (nonband && e && e[0] == '0') {
    int rc = band_detect(bits, n, batch, nonband, st);
    if (rc) return rc;
    rc = build_m_bits_banded(bits, n, n_pad, batch, gammas, mwork, stride, nonband, st, nullptr, 0);
    if (rc) return rc;
    return invert_batched(mwork, n_pad, n_pad, stride, batch, work, info, st, bits, n, true, 0, nullptr, nullptr,
                          nullptr);
  }
  int levels = 1;
  if (nonband) {
    int rc = band_detect(bits, n, batch, nonband, st);
    if (rc) return rc;
    rc = invert_batched(mwork, n_pad, n_pad, stride, batch, work, info, st, bits, n, true, 1, gammas, &s0bad,
                        &levels);
    if (rc) return rc;
  }
  int rc = build_m_bits_banded(bits, n, n_pad, batch, gammas, mwork, stride, nonband, st, s0bad,
                               levels == 2 ? (int)(n_pad / 2) : 0);
  if (rc) return rc;
  return invert_batched(mwork, n_pad, n_pad, stride, batch, work, info, st, bits, n, nonband != nullptr,
                        nonband ? 2 : 0, gammas, nullptr, nullptr);
}
int log_ceil_d8(const double* y, int64_t n, int64_t ldy, int64_t stride_y, int64_t batch,
                const double* gammas, double gamma, uint8_t* d8_out, int64_t ldo, int64_t stride_o,
                unsigned long long* counters, cudaStream_t st);
int log_ceil(const double* y, int64_t n, int64_t ldy, int64_t stride_y, int64_t batch,
             const double* gammas, double gamma, double* r_out, double* dceil_out, int32_t* d32_out,
             int64_t ldo, int64_t stride_o, const uint8_t* reachable, int64_t ldm,
             unsigned long long* counters, cudaStream_t st);
}  // namespace rdb

extern "C" const char* rdb_strerror(int code) {
  switch (code) {
    case RDB_OK:
      return "ok";
    case RDB_EINVAL:
      return "invalid argument (shape, alignment or null pointer)";
    case RDB_ESINGULAR:
      return "singular to working precision";
    case RDB_ENOTM:
      return "no-pivot elimination not certified (not a nonsingular M-matrix)";
    case RDB_ECUDA:
      return "CUDA launch or runtime error";
    default:
      return "unknown error";
  }
}

extern "C" int rdb_abi_version(void) { return RDB_ABI_VERSION; }

namespace rdb {
static thread_local cudaError_t g_last_err = cudaSuccess;
void set_cuda_error(cudaError_t e) { g_last_err = e; }
}  // namespace rdb

extern "C" const char* rdb_last_cuda_error(void) { return cudaGetErrorString(rdb::g_last_err); }

extern "C" int rdb_apsp_bits_batched(const uint32_t* bits, int64_t n, int64_t batch,
                                     const double* gammas, double* mwork, void* work,
                                     rdb_pivot_info* info, int32_t* d32,
                                     unsigned long long* counters, void* stream) {
  if (!bits || !gammas || !mwork || !work || !info || !d32 || n <= 0 || batch <= 0)
    return RDB_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t n_pad = (n + RDB_NB - 1) / RDB_NB * RDB_NB;
  const int64_t stride = n_pad * n_pad;
  const int rc = rdb::build_and_invert(bits, n, n_pad, batch, gammas, mwork, work, info, st);
  if (rc) return rc;
  return rdb::log_ceil(mwork, n, n_pad, stride, batch, gammas, 0.0, nullptr, nullptr, d32, n, n * n,
                       nullptr, 0, counters, st);
}

extern "C" int rdb_apsp_bits_batched_d8(const uint32_t* bits, int64_t n, int64_t batch,
                                        const double* gammas, double* mwork, void* work,
                                        rdb_pivot_info* info, uint8_t* d8,
                                        unsigned long long* counters, void* stream) {
  if (!bits || !gammas || !mwork || !work || !info || !d8 || !counters || n <= 0 || batch <= 0)
    return RDB_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t n_pad = (n + RDB_NB - 1) / RDB_NB * RDB_NB;
  const int64_t stride = n_pad * n_pad;
  const int rc = rdb::build_and_invert(bits, n, n_pad, batch, gammas, mwork, work, info, st);
  if (rc) return rc;
  return rdb::log_ceil_d8(mwork, n, n_pad, stride, batch, gammas, 0.0, d8, n, n * n, counters, st);
}
