// Shared device helpers for the R-distance kernels (sm_100a).
//
// FP64 on sm_100a: the only FP64 tensor instruction is DMMA.8x8x4
// (PTX mma.sync.aligned.m8n8k4.row.col.f64); tcgen05.mma has no f64 kind,
// so the Blackwell-specific parts used here are the bulk-copy (TMA) engine
// (cp.async.bulk, SASS UBLKCP) and mbarrier transaction counting.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/rdist_b200.h"

#define RDB_DEV __device__ __forceinline__

namespace rdb {

constexpr int NB = RDB_NB;  // Gauss-Jordan panel width (128)

// ---------------------------------------------------------------- per-device host state
// Function attributes, SM counts and the library's internal streams / events
// are kept per CUDA device (the caller's current device), so one process may
// drive several GPUs.
constexpr int MAX_DEVICES = 64;
inline int current_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= MAX_DEVICES) return -1;
  return d;
}
// once-per-device flag for lazily applied settings (idempotent, so a benign race)
struct DeviceFlags {
  bool v[MAX_DEVICES] = {};
  bool get(int d) const { return d >= 0 && v[d]; }
  void set(int d) {
    if (d >= 0) v[d] = true;
  }
};

// ---------------------------------------------------------------- DMMA
// D(8x8) += A(8x4, row) * B(4x8, col). Lane l holds A[l/4][l%4], B[l%4][l/4],
// and C[l/4][2*(l%4) + {0,1}].
RDB_DEV void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// ---------------------------------------------------------------- mbarrier
RDB_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

RDB_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

RDB_DEV void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

RDB_DEV void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

RDB_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

RDB_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

RDB_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// 1-D bulk copy global -> shared through the TMA unit, completing on `bar`.
// dst/src 16-byte aligned, bytes a multiple of 16.
RDB_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Reciprocal without the IEEE-division slow-path call (whose ABI call site
// forces register spills in fully unrolled loops): MUFU.RCP64H seed and two
// Newton steps with FMA. Within 1 ulp (exact for powers of two) for normal p;
// 0 or non-finite p yield a non-finite result, which the callers flag.
RDB_DEV double rcp_nr(double p) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(p));
  double e = fma(-p, y, 1.0);
  y = fma(y, e, y);
  e = fma(-p, y, 1.0);
  return fma(y, e, y);
}

// ---------------------------------------------------------------- misc
RDB_DEV double2 ldg2(const double* p) { return *reinterpret_cast<const double2*>(p); }
RDB_DEV void stg2(double* p, double2 v) { *reinterpret_cast<double2*>(p) = v; }

// Monotone int64 key for non-negative doubles (IEEE ordering == integer ordering).
RDB_DEV void atomic_max_nonneg(double* addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(addr),
            static_cast<unsigned long long>(__double_as_longlong(v)));
}

}  // namespace rdb

// ---------------------------------------------------------------- SM timeline (diagnostic builds)
// Built with -DRDB_TRACE (tools/sm_timeline.py): every warp of a traced kernel
// appends {globaltimer at entry, at exit, SM id, kernel kind} to a device
// buffer, from which the tool rebuilds per-SM busy intervals of one call
// (where SMs sit idle between the launches of the concurrent streams).
// Off by default: RDB_TRACE_SCOPE expands to nothing.
#ifdef RDB_TRACE
namespace rdb {
namespace trace {
constexpr int SEGS = 192;  // per-SM segments of the buffer (SM ids < 192)
struct Rec {
  unsigned long long t0, t1;
  int sm, kind;
};
static __device__ Rec* g_buf;
static __device__ unsigned g_seg;        // records per segment
static __device__ unsigned g_n[SEGS];    // records per segment so far
RDB_DEV unsigned long long now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
struct Guard {
  int kind;
  unsigned long long t0;
  RDB_DEV explicit Guard(int k) : kind(k), t0(now()) {}
  RDB_DEV ~Guard() {
    if ((threadIdx.x & 31) != 0 || !g_buf) return;
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    if (sm >= (unsigned)SEGS) return;
    const unsigned i = atomicAdd(&g_n[sm], 1u);  // contention only within the SM
    if (i >= g_seg) return;
    g_buf[(size_t)sm * g_seg + i] = Rec{t0, now(), (int)sm, kind};
  }
};
// points this translation unit's copy at buf (cap records, SEGS segments), counts reset
static inline int attach(void* buf, unsigned cap) {
  unsigned zero[SEGS] = {};
  const unsigned seg = cap / SEGS;
  if (cudaMemcpyToSymbol(g_buf, &buf, sizeof(buf)) != cudaSuccess ||
      cudaMemcpyToSymbol(g_seg, &seg, sizeof(seg)) != cudaSuccess ||
      cudaMemcpyToSymbol(g_n, zero, sizeof(zero)) != cudaSuccess)
    return -1;
  return 0;
}
static inline unsigned count() {  // total records kept
  unsigned n[SEGS] = {}, seg = 0, tot = 0;
  cudaMemcpyFromSymbol(n, g_n, sizeof(n));
  cudaMemcpyFromSymbol(&seg, g_seg, sizeof(seg));
  for (int i = 0; i < SEGS; ++i) tot += n[i] < seg ? n[i] : seg;
  return tot;
}
}  // namespace trace
}  // namespace rdb
#define RDB_TRACE_SCOPE(kind) rdb::trace::Guard _rdb_trace_guard(kind)
#else
#define RDB_TRACE_SCOPE(kind) \
  do {                        \
  } while (0)
#endif

namespace rdb {
void set_cuda_error(cudaError_t e);  // remembered for rdb_last_cuda_error()
}

#define RDB_LAUNCH_CHECK()                                   \
  do {                                                       \
    cudaError_t _e = cudaGetLastError();                     \
    if (_e != cudaSuccess) {                                 \
      rdb::set_cuda_error(_e);                               \
      return RDB_ECUDA;                                      \
    }                                                        \
  } while (0)
