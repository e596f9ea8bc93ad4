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
//   P1 (gj_panel_kernel)             D = A_pp^-1, pivots recorded (gj_panel.cuh)
//   P2 (engine, store)               A_pJ = D * A_pJ                 for J != p
//   U  (engine, reduce-add / store)  A_IJ += -(A_Ip * A_pJ)          for I != p, J != p
//                                    A_Ip  = -(A_Ip * D)             (last in row block I)
// After the last panel A = M^-1 (2n^3 flop in total). P2 and U run on the
// persistent warp-specialised DMMA engine (dmma_engine.cuh). U reads the
// column panel A_Ip straight from A; the one tile per row block that
// overwrites it is enumerated last in that row block and holds its epilogue
// until the other tiles of the row block have their operands in shared
// memory (in-kernel counters, no copy of the panel).
#include <cudaTypedefs.h>

#include <cmath>
#include <mutex>

#include "dmma_engine.cuh"
#include "gj_panel.cuh"

namespace rdb {

using EC = eng::Default;  // engine warp layout

__global__ void __launch_bounds__(p1::THREADS, 1)
    gj_panel_kernel(double* __restrict__ a, int64_t lda, int64_t stride, int64_t off, int idx0,
                    rdb_pivot_info* __restrict__ info, int first, int64_t info_stride = 1,
                    const int* __restrict__ nonband = nullptr, int want = 1) {
  RDB_TRACE_SCOPE(want == 2 ? 1 : (want == 0 ? 5 : 0));
  // block at a + b*stride + off*(lda + 1); pivot indices recorded from idx0.
  // Per-matrix path flags (batched calls): 0 banded inverse, 1 block-sparse
  // Gauss-Jordan, 2 dense 256-wide Gauss-Jordan; only matrices whose flag is
  // `want` are processed.
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int64_t b = blockIdx.x;
  if (nonband && nonband[b * info_stride] != want) return;
#ifdef RDB_EXP_NO_NESTED_P1
  if (want == 2) return;  // timing experiment only (wrong results)
#endif
#ifdef RDB_EXP_NO_P1
  return;  // timing experiment only (tools/k2_split.py on a variant library): wrong results
#endif
  p1::panel_inverse(*reinterpret_cast<p1::Smem*>(smem_raw), a + b * stride + off * lda + off, lda, idx0,
                    info + b * info_stride, first);
}

// ------------------------------------------------------------------ schedulers
struct RowPanelSched {
  double* a;
  int64_t lda, stride;
  int nt, pt, batch;
  int* dyn = nullptr;  // dynamic tile counter (batched calls)
  // block-sparse plan (batched calls): tiles (g << 13 | first k-chunk << 10 |
  // k-chunks << 6 | J) of this step, *count_ptr of them
  const int* list = nullptr;
  const int* count_ptr = nullptr;
  RDB_DEV int count() const { return list ? *count_ptr : batch * (nt - 1); }
  RDB_DEV eng::Tile tile(int t) const {
    int g, J;
    int c0 = 0, nk = NB / eng::BK;
    if (list) {
      const int e = list[t];
      g = e >> 13;
      c0 = (e >> 10) & 7;
      nk = (e >> 6) & 15;
      J = e & 63;
    } else {
      g = t / (nt - 1);
      J = t - g * (nt - 1);
      J += (J >= pt);
    }
    double* A = a + (int64_t)g * stride;
    double* rowp = A + (int64_t)pt * NB * lda + (int64_t)J * NB;
    eng::Tile T;
    T.a_col = pt * NB + c0 * eng::BK;  // A operand: D = A_pp (columns of the k-chunks)
    T.a_row = pt * NB;
    T.a_mat = g;
    T.b = rowp + (int64_t)c0 * eng::BK * lda;  // the non-zero row strips of A_pJ
    T.ldb = lda;
    T.c_col = J * NB;
    T.c_row = pt * NB;
    T.c_mat = g;
    T.nk = nk;
    T.mode = eng::EPI_STORE;
    T.neg = 0;
    T.signal = nullptr;
    T.wait = nullptr;
    T.wait_target = 0;
    return T;
  }
};

struct UpdateSched {
  double* a;
  int* cnt;  // [batch][nt] row-block counters, zeroed before step 0
  int64_t lda, stride;
  int nt, pt, batch;
  // part 0: every tile. Single-matrix look-ahead (batch == 1): part 1 is the
  // next panel's diagonal tile (pt+1, pt+1) alone, part 2 every other tile;
  // or part 3 the whole row block pt+1 (the next P1 and row panel need it) and
  // part 4 every tile outside it
  int part;
  int* dyn = nullptr;  // dynamic tile counter (batched calls)
  // block-sparse plan (batched calls, part 0): entries {g << 12 | I << 6 | J,
  // wait target of the panel-column tile | first k-chunk << 16 | k-chunks << 20},
  // *count_ptr of them (gj_plan_walk)
  const int2* list = nullptr;
  const int* count_ptr = nullptr;
  RDB_DEV int count() const {
    if (list) return *count_ptr;
    return part == 0 ? batch * (nt - 1) * nt
                     : (part == 1 ? 1 : (part == 2 ? (nt - 1) * nt - 1 : (part == 3 ? nt : (nt - 2) * nt)));
  }
  RDB_DEV eng::Tile tile(int t) const {
    if (list) {
      const int2 e = list[t];
      eng::Tile T = make(e.x >> 12, (e.x >> 6) & 63, e.x & 63, e.y & 0xFFFF);
      const int c0 = (e.y >> 16) & 15, nk = e.y >> 20;  // the non-zero k-chunks of A_Ip
      T.a_col += c0 * eng::BK;
      T.b += (int64_t)c0 * eng::BK * T.ldb;
      T.nk = nk;
      return T;
    }
    // (g, row index I' over the rows other than pt, column index jj in the
    // order pt+1, ..., nt-1, 0, ..., pt: the panel column comes last)
    int g = 0, Ir, jj;
    if (part == 0) {
      const int per = (nt - 1) * nt;
      g = t / per;
      const int rem = t - g * per;
      Ir = rem / nt;
      jj = rem - Ir * nt;
    } else if (part == 1) {
      Ir = pt;  // row pt+1
      jj = 0;   // column pt+1
    } else if (part == 3) {
      Ir = pt;  // row pt+1, every column (the panel column last)
      jj = t;
    } else if (part == 4) {
      Ir = t / nt;  // rows other than pt+1
      jj = t - Ir * nt;
      Ir += (Ir >= pt) ? 1 : 0;
    } else {
      const int head = pt * nt;
      if (t < head) {
        Ir = t / nt;
        jj = t - Ir * nt;
      } else if (t - head < nt - 1) {
        Ir = pt;
        jj = t - head + 1;  // row pt+1 without its diagonal tile
      } else {
        const int r = t - head - (nt - 1);
        Ir = pt + 1 + r / nt;
        jj = r - (r / nt) * nt;
      }
    }
    const int I = Ir + (Ir >= pt);
    int J = pt + 1 + jj;
    if (J >= nt) J -= nt;
    // completed steps j < pt touched row block I unless j == I
    const int base = (pt - (I < pt ? 1 : 0)) * (nt - 1);
    return make(g, I, J, base + (nt - 1));
  }
  // tile (I, J) of matrix g; wait_target applies to the panel-column tile J == pt
  RDB_DEV eng::Tile make(int g, int I, int J, int wait_target) const {
    double* A = a + (int64_t)g * stride;
    eng::Tile T;
    T.a_col = pt * NB;  // A operand: A_Ip
    T.a_row = I * NB;
    T.a_mat = g;
    T.b = A + (int64_t)pt * NB * lda + (int64_t)J * NB;
    T.ldb = lda;
    T.c_col = J * NB;
    T.c_row = I * NB;
    T.c_mat = g;
    T.nk = NB / eng::BK;
    T.neg = 1;
    int* c = cnt + (int64_t)g * nt + I;
    if (J == pt) {
      T.mode = eng::EPI_STORE;
      T.signal = nullptr;
      T.wait = c;
      T.wait_target = wait_target;
    } else {
      T.mode = eng::EPI_REDUCE;
      T.signal = c;
      T.wait = nullptr;
      T.wait_target = 0;
    }
    return T;
  }
};

__global__ void __launch_bounds__(EC::THREADS, 1)
    gj_rowpanel_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap cmap,
                       RowPanelSched sched) {
  RDB_TRACE_SCOPE(2);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  eng::run<EC>(smem_raw, &amap, sched, eng::BulkEpilogue<EC>{&cmap});
}

__global__ void __launch_bounds__(EC::THREADS, 1)
    gj_update_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap cmap,
                     UpdateSched sched) {
  RDB_TRACE_SCOPE(3);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  eng::run<EC>(smem_raw, &amap, sched, eng::BulkEpilogue<EC>{&cmap});
}

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static int encode_map(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld,
                      int64_t stride, int64_t batch, int box_rows, int box_cols, CUtensorMapSwizzle swz) {
  if (!g_encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return RDB_ECUDA;
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  if (((uintptr_t)base & 15) || (ld & 1) || (stride & 1)) return RDB_EINVAL;
  const cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)batch};
  const cuuint64_t strides[2] = {(cuuint64_t)ld * 8, (cuuint64_t)stride * 8};
  const cuuint32_t box[3] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides,
                              box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? RDB_OK : RDB_EINVAL;
}

int make_a_map(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld,
               int64_t stride, int64_t batch) {
  return encode_map(map, base, rows, cols, ld, stride, batch, eng::BM, eng::BK, CU_TENSOR_MAP_SWIZZLE_128B);
}

int make_c_map(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld,
               int64_t stride, int64_t batch, int box_rows, int box_cols) {
  return encode_map(map, base, rows, cols, ld, stride, batch, box_rows, box_cols, CU_TENSOR_MAP_SWIZZLE_NONE);
}

static int make_ec_map(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld,
                       int64_t stride, int64_t batch) {
  return make_c_map(map, base, rows, cols, ld, stride, batch, EC::HROWS, EC::WCOLS);
}

static int g_sms[MAX_DEVICES] = {};

static int setup() {
  const int dev = current_device();
  if (dev < 0) return RDB_ECUDA;
  if (g_sms[dev]) return RDB_OK;
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return RDB_ECUDA;
  if (cudaFuncSetAttribute(gj_rowpanel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)EC::SMEM_BYTES) != cudaSuccess ||
      cudaFuncSetAttribute(gj_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)EC::SMEM_BYTES) != cudaSuccess ||
      cudaFuncSetAttribute(gj_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)p1::SMEM_BYTES) != cudaSuccess)
    return RDB_ECUDA;
  g_sms[dev] = sms;
  return RDB_OK;
}

// Internal streams and events, one set per device: the look-ahead side
// stream (single-matrix and wide paths) and the sub-batch streams of a split
// batch. Enqueueing is serialised by g_enqueue (invert_batched).
constexpr int MAX_PARTS = 4;
struct DevStreams {
  cudaStream_t side = nullptr;
  cudaEvent_t ev_a = nullptr, ev_p = nullptr, ev_b = nullptr;
  cudaStream_t part[MAX_PARTS] = {};
  cudaEvent_t fork = nullptr, join[MAX_PARTS] = {};
  // dense-wide look-ahead: one side stream + fork / join events per part
  cudaStream_t dw_side[MAX_PARTS] = {};
  cudaEvent_t dw_fork[MAX_PARTS] = {}, dw_join[MAX_PARTS] = {};
  cudaEvent_t s0_ready[MAX_PARTS] = {};  // sparse first step: the part's edge lists gathered
};
static DevStreams g_streams[MAX_DEVICES];

static DevStreams* dev_streams() {
  const int dev = current_device();
  if (dev < 0) return nullptr;
  DevStreams& d = g_streams[dev];
  if (!d.side) {
    if (cudaStreamCreateWithFlags(&d.side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&d.ev_a, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&d.ev_p, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&d.ev_b, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&d.fork, cudaEventDisableTiming) != cudaSuccess)
      return nullptr;
    for (int i = 0; i < MAX_PARTS; ++i)
      if (cudaStreamCreateWithFlags(&d.part[i], cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&d.join[i], cudaEventDisableTiming) != cudaSuccess ||
          cudaStreamCreateWithFlags(&d.dw_side[i], cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&d.dw_fork[i], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&d.dw_join[i], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&d.s0_ready[i], cudaEventDisableTiming) != cudaSuccess)
        return nullptr;
  }
  return &d;
}

int sm_count() {
  setup();
  const int dev = current_device();
  return dev >= 0 && g_sms[dev] > 0 ? g_sms[dev] : 148;
}

#define RDB_HOST_DEV __host__ __device__ __forceinline__

// ------------------------------------------------------------------ block-sparse plan (batched calls)
// Symbolic Gauss-Jordan on strip patterns: C[g][I][J] is an 8-bit mask of
// the 16-column strips (the engine's k-chunks) of block (I, J) of matrix g
// that may hold non-zeros, R[g][I][J] the same for its 16-row strips
// (supersets of the numerical patterns; 0 = the block is zero). Step p:
//   P2   A_pJ = D A_pJ            only where block (p, J) is non-zero, over
//        the k-chunks first..last non-zero row strip of A_pJ;
//   U    A_IJ += -(A_Ip A_pJ)     only where A_Ip and A_pJ are non-zero, and
//        A_Ip = -(A_Ip D)         only where A_Ip is, both over the k-chunks
//        [first, last] non-zero strip of A_Ip only;
// fill: C(A_IJ) |= C(A_pJ), R(A_IJ) |= R(A_Ip) (D A_pJ keeps A_pJ's zero
// columns and A_Ip D A_Ip's zero rows, D is invertible); D A_pJ has full rows,
// A_Ip D full columns and A_pp = D is full (D is treated as dense). A skipped
// tile or chunk would add exact zeros (C + -0 == C) or store them, so results
// are those of the dense schedule (up to the sign of zero entries). Banded
// matrices (the directed lattices of config 2: bandwidth = grid side 32) keep
// whole blocks zero until late steps, and the already-eliminated part of
// their column panels has non-zeros only in the strips that couple to the
// next grid rows: about 1/4 of the k-chunks of 1/2 of the tiles remain.
constexpr int PLAN_MAX_NT = 64;

RDB_HOST_DEV int pat_ld(int nt) { return (nt + 3) & ~3; }  // bytes per pattern row (32-bit atomics)

struct PlanPart {
  // strip masks of matrix g: C at pat + g * pat_stride + I * pat_ld(nt) + J, R
  // nt * pat_ld(nt) bytes after C
  unsigned char* pat;
  int64_t pat_stride;
  int* counts;  // [2][nt]: P2 tiles, update tiles per step
  int* offs;    // [2][nt][batch]: per-matrix tile counts, then list offsets
  int* rp;      // [nt][batch * (nt - 1)] P2 entries g << 13 | c0 << 10 | nk << 6 | J
  int2* up;     // [nt][batch * (nt - 1) * nt] update entries {g << 12 | I << 6 | J, wait | c0 << 16 | nk << 20}
  bool prebuilt = false;  // lists written by the caller (dense-wide nested inverse): no plan walk
};

// The plan in three launches, all parallel over matrices: gj_plan_walk<false>
// (a warp per matrix, lane = row block I and I + 32, the matrix's masks in
// shared memory) counts each step's P2 and update tiles per matrix;
// gj_plan_scan turns the counts into list offsets (matrix order) and totals;
// gj_plan_walk<true> repeats the walk and writes the entries (within a
// matrix: row blocks ascending, columns pt+1, ..., pt-1 and the panel column
// last, as in the dense order, so waits point only backwards).
RDB_DEV unsigned long long ballot64(bool lo, bool hi) {
  return (unsigned long long)__ballot_sync(0xffffffffu, lo) | ((unsigned long long)__ballot_sync(0xffffffffu, hi) << 32);
}

template <bool WRITE>
__global__ void __launch_bounds__(1024)
    gj_plan_walk(const unsigned char* __restrict__ pat, int64_t pat_stride, int batch, int nt,
                 int* __restrict__ offs, int* __restrict__ rp, int2* __restrict__ up) {
  RDB_TRACE_SCOPE(30);
  // offs: [2][nt][batch] per-matrix counts (WRITE = false) / exclusive offsets (WRITE = true)
  extern __shared__ __align__(16) unsigned char s_pat[];  // per warp: C then R, nt rows of ld bytes each
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = blockIdx.x * (blockDim.x >> 5) + wid;
  if (g >= batch) return;  // warp-uniform
  const int ld = pat_ld(nt);
  const int gbytes = 2 * nt * ld;
  unsigned char* C = s_pat + wid * gbytes;
  unsigned char* R = C + nt * ld;
  const unsigned char* src = pat + (int64_t)g * pat_stride;
  for (int q = lane; q < gbytes / 4; q += 32)
    reinterpret_cast<unsigned*>(C)[q] = reinterpret_cast<const unsigned*>(src)[q];
  __syncwarp();
  const int I0 = lane, I1 = lane + 32;
  if (I0 < nt) C[I0 * ld + I0] = R[I0 * ld + I0] = 0xFF;  // the diagonal blocks
  if (I1 < nt) C[I1 * ld + I1] = R[I1 * ld + I1] = 0xFF;
  const int64_t rp_cap = (int64_t)batch * (nt - 1), up_cap = (int64_t)batch * (nt - 1) * nt;
  int cum0 = 0, cum1 = 0;  // signals row blocks I0, I1 have received (their in-kernel counters)
  for (int k = 0; k < nt; ++k) {
    __syncwarp();
    const unsigned long long rowp =
        ballot64(I0 < nt && I0 != k && C[k * ld + I0], I1 < nt && I1 != k && C[k * ld + I1]);
    const unsigned long long colp =
        ballot64(I0 < nt && I0 != k && C[I0 * ld + k], I1 < nt && I1 != k && C[I1 * ld + k]);
    const int nrp = __popcll(rowp);
    if (!WRITE) {
      if (lane == 0) {
        offs[(int64_t)k * batch + g] = nrp;
        offs[((int64_t)nt + k) * batch + g] = __popcll(colp) * (nrp + 1);
      }
    } else {
      // P2 tiles: lane J (J in rowp) over A_pJ's non-zero row strips
      const int rbase = offs[(int64_t)k * batch + g];
      const int ubase = offs[((int64_t)nt + k) * batch + g];
      for (int h = 0; h < 2; ++h) {
        const int J = h ? I1 : I0;
        if (J < nt && ((rowp >> J) & 1ull)) {
          const unsigned m = R[k * ld + J];
          const int c0 = __ffs(m) - 1, nk = 32 - __clz(m) - c0;
          rp[k * rp_cap + rbase + __popcll(rowp & ((1ull << J) - 1))] = (g << 13) | (c0 << 10) | (nk << 6) | J;
        }
      }
      // update tiles: lane I (I in colp) writes its row's nrp + 1 entries
      for (int h = 0; h < 2; ++h) {
        const int I = h ? I1 : I0;
        if (I < nt && ((colp >> I) & 1ull)) {
          int2* upl = up + k * up_cap + ubase + __popcll(colp & ((1ull << I) - 1)) * (nrp + 1);
          const unsigned m = C[I * ld + k];  // non-zero k-chunks of A_Ip
          const int c0 = __ffs(m) - 1, nk = 32 - __clz(m) - c0;
          const int kr = (c0 << 16) | (nk << 20);
          int& cum = h ? cum1 : cum0;
          int c = 0;
          for (int jj = 0; jj < nt; ++jj) {
            int J = k + 1 + jj;
            if (J >= nt) J -= nt;
            if (J == k) {
              upl[c++] = make_int2((g << 12) | (I << 6) | J, cum | kr);
            } else if ((rowp >> J) & 1ull) {
              ++cum;
              upl[c++] = make_int2((g << 12) | (I << 6) | J, kr);
            }
          }
        }
      }
    }
    __syncwarp();
    // fill (rows I != k read only row k's C and their own R[I][k])
    for (int h = 0; h < 2; ++h) {
      const int I = h ? I1 : I0;
      if (I < nt && ((colp >> I) & 1ull)) {
        const unsigned char rik = R[I * ld + k];
        for (int J = 0; J < nt; ++J)
          if ((rowp >> J) & 1ull) {
            C[I * ld + J] |= C[k * ld + J];
            R[I * ld + J] |= rik;
          }
        C[I * ld + k] = 0xFF;  // A_Ip = -(A_Ip D)
      }
    }
    __syncwarp();
    for (int h = 0; h < 2; ++h) {  // D A_pJ
      const int J = h ? I1 : I0;
      if (J < nt && ((rowp >> J) & 1ull)) R[k * ld + J] = 0xFF;
    }
  }
}

// One CTA: exclusive prefix sums of the 2 nt per-matrix count rows in place
// (a warp per row); the totals go to counts[0 .. 2 nt).
__global__ void __launch_bounds__(1024)
    gj_plan_scan(int* __restrict__ offs, int batch, int nt, int* __restrict__ counts) {
  RDB_TRACE_SCOPE(31);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (int)(blockDim.x >> 5);
  for (int row = wid; row < 2 * nt; row += nw) {
    int* v = offs + (int64_t)row * batch;
    int carry = 0;
    for (int g0 = 0; g0 < batch; g0 += 32) {
      const int g = g0 + lane;
      const int x = g < batch ? v[g] : 0;
      int y = x;
      for (int o = 1; o < 32; o <<= 1) {
        const int z = __shfl_up_sync(0xffffffffu, y, o);
        if (lane >= o) y += z;
      }
      if (g < batch) v[g] = carry + y - x;
      carry += __shfl_sync(0xffffffffu, y, 31);
    }
    if (lane == 0) counts[row] = carry;
  }
}

// Host: warps per CTA of gj_plan_walk (shared memory holds one matrix's masks per warp).
static int plan_warps(int nt) {
  const int bytes = 2 * nt * pat_ld(nt);
  int w = (48 * 1024) / bytes;
  return w < 1 ? 1 : (w > 8 ? 8 : w);
}

static void launch_plan(const PlanPart& pp, int batch, int nt, cudaStream_t st) {
  const int w = plan_warps(nt);
  const unsigned grid = (unsigned)((batch + w - 1) / w);
  const size_t smem = (size_t)w * 2 * nt * pat_ld(nt);
  gj_plan_walk<false><<<grid, 32 * w, smem, st>>>(pp.pat, pp.pat_stride, batch, nt, pp.offs, pp.rp, pp.up);
  gj_plan_scan<<<1, 32 * (2 * nt < 32 ? 2 * nt : 32), 0, st>>>(pp.offs, batch, nt, pp.counts);
  gj_plan_walk<true><<<grid, 32 * w, smem, st>>>(pp.pat, pp.pat_stride, batch, nt, pp.offs, pp.rp, pp.up);
}

// Strip patterns from bit-packed adjacency (the rdb_build_m_bits input): a
// warp per 16-row strip (ORed in registers, then one atomic per mask word).
// Column strips: word q covers strips 2q, 2q + 1 of block q / 4; masks of four
// consecutive blocks share a 32-bit word (pat_ld pads rows to 4 bytes). Row
// strips: bit (i % NB) / 16 in every block the strip's rows touch.
__global__ void strip_pattern_bits_kernel(const uint32_t* __restrict__ bits, int64_t n, int64_t batch, int nt,
                                          unsigned char* __restrict__ pat, const int* __restrict__ nonband) {
  const int lane = threadIdx.x & 31;
  const int ld = pat_ld(nt);
  const int64_t wpr = (n + 31) / 32;
  const int64_t strips = (n + 15) / 16;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < batch * strips; w += nwarps) {
    const int64_t b = w / strips, s16 = w - b * strips;
    if (nonband && !nonband[b]) continue;  // banded path: the pattern stays zero, no GJ tiles
    const int64_t i0 = s16 * 16, i1 = i0 + 16 < n ? i0 + 16 : n;
    unsigned char* Pc = pat + b * 2 * nt * ld;
    unsigned* dst = reinterpret_cast<unsigned*>(Pc + (i0 / NB) * ld);
    unsigned* rdst = reinterpret_cast<unsigned*>(Pc + (nt + i0 / NB) * ld);
    const unsigned rbit = 1u << ((i0 % NB) / 16);
    for (int64_t q0 = 0; q0 < wpr; q0 += 32) {
      const int64_t q = q0 + lane;
      uint32_t v = 0;
      if (q < wpr)
        for (int64_t i = i0; i < i1; ++i) v |= __ldg(bits + (b * n + i) * wpr + q);
      // block J = q / 4 gets bits 2 (q % 4) + {0, 1}; 16 words (4 blocks) per 32-bit mask word
      unsigned m = ((v & 0xFFFFu) ? 1u : 0u) | ((v >> 16) ? 2u : 0u);
      m <<= 2 * (q & 3) + 8 * ((q >> 2) & 3);
      for (int o = 1; o < 16; o <<= 1) m |= __shfl_xor_sync(0xffffffffu, m, o);
      if ((lane & 15) == 0 && m) {
        atomicOr(dst + (q >> 4), m);
        unsigned r = 0;  // the row strip in each of the (up to 4) blocks this word touches
        for (int j = 0; j < 4; ++j)
          if ((m >> (8 * j)) & 0xFFu) r |= rbit << (8 * j);
        atomicOr(rdst + (q >> 4), r);
      }
    }
  }
}

// Strip patterns by scanning the matrices (generic batched calls): a warp per
// block, rows in order (lane l covers columns 4l .. 4l + 3 = strip l / 4),
// stopping once all 8 column strips are non-zero (a dense block costs a row
// or two; zero blocks are read in full). Row strips are not resolved: a
// non-zero block gets all 8. NaN counts as non-zero.
__global__ void strip_pattern_m_kernel(const double* __restrict__ a, int64_t lda, int64_t stride, int64_t batch,
                                       int nt, unsigned char* __restrict__ pat) {
  const int lane = threadIdx.x & 31;
  const int ld = pat_ld(nt);
  const int64_t blocks = batch * nt * nt;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < blocks; w += nwarps) {
    const int64_t b = w / (nt * nt);
    const int I = (int)((w / nt) % nt), J = (int)(w % nt);
    const double* p = a + b * stride + (int64_t)I * NB * lda + (int64_t)J * NB + 4 * lane;
    unsigned m = 0;
    for (int r = 0; r < NB && m != 0xFFu; ++r) {
      const double2 u = ldg2(p + (int64_t)r * lda), v = ldg2(p + (int64_t)r * lda + 2);
      const bool nz = u.x != 0.0 || u.y != 0.0 || v.x != 0.0 || v.y != 0.0;
      m |= __reduce_or_sync(0xffffffffu, nz ? 1u << (lane >> 2) : 0u);
    }
    if (lane == 0) {
      pat[(b * 2 * nt + I) * ld + J] = (unsigned char)m;
      pat[(b * 2 * nt + nt + I) * ld + J] = m ? 0xFF : 0;
    }
  }
}

static unsigned persistent_grid(int64_t tiles) {
  const int64_t sms = sm_count();
  return (unsigned)(tiles < sms ? tiles : sms);
}

static int invert_wide(double* a, int64_t n, int64_t lda, void* work, rdb_pivot_info* info, cudaStream_t st);
static int64_t wide_min_n();

// SMs the single-matrix row look-ahead gives the side stream (0: the older
// diagonal-tile look-ahead with a one-round row-panel launch per step)
static int la_side_sms() {
  const char* e = getenv("RDB_GJ_LA_SIDE");
  const int v = e ? atoi(e) : 16;
  return v < 0 ? 0 : v;
}

// Blocked Gauss-Jordan with NB = 128 panels. `first` resets the pivot record
// (step 0); idx_base offsets the reported pivot indices (a diagonal sub-block
// inverted as part of a larger matrix).
static int invert_core(double* a, int64_t n, int64_t lda, int64_t stride, int64_t batch, void* work,
                       rdb_pivot_info* info, cudaStream_t st, int first, int64_t idx_base, int* dyn = nullptr,
                       const PlanPart* plan = nullptr, int64_t info_stride = 1, const int* nonband = nullptr,
                       int grid_cap = 0, int want = 1) {
  if (!a || !work || !info || n <= 0 || batch <= 0) return RDB_EINVAL;
  if (n % NB != 0 || lda < n || (lda & 1) || (batch > 1 && stride < n * lda)) return RDB_EINVAL;
  if (((uintptr_t)a & 15) || ((uintptr_t)work & 15)) return RDB_EINVAL;
  if (batch > 65535) return RDB_EINVAL;
  const int nt = (int)(n / NB);
  if ((int64_t)batch * nt * nt > 2147483647LL) return RDB_EINVAL;
  int rc = setup();
  if (rc) return rc;
  int* cnt = static_cast<int*>(work);
  CUtensorMap amap, cmap;
  rc = make_a_map(&amap, a, n, n, lda, batch > 1 ? stride : n * lda, batch);
  if (rc) return rc;
  rc = make_ec_map(&cmap, a, n, n, lda, batch > 1 ? stride : n * lda, batch);
  if (rc) return rc;
  if (cudaMemsetAsync(cnt, 0, sizeof(int) * (size_t)batch * nt, st) != cudaSuccess) return RDB_ECUDA;
  if (plan && (batch == 1 || nt > PLAN_MAX_NT)) plan = nullptr;
  if (plan && !plan->prebuilt)
    launch_plan(*plan, (int)batch, nt, st);
  // Single matrix: look-ahead. The next panel's column block is updated first
  // (part 1); the next P1 (one CTA, latency-bound) then runs on a side stream
  // on one SM while the rest of the update (part 2) uses the other SMs.
  const bool lookahead = (batch == 1 && nt >= 3);
  DevStreams* ds = lookahead ? dev_streams() : nullptr;
  if (lookahead && !ds) return RDB_ECUDA;
  cudaStream_t side = ds ? ds->side : nullptr;
  gj_panel_kernel<<<(unsigned)batch, p1::THREADS, p1::SMEM_BYTES, st>>>(a, lda, stride, 0, idx_base, info, first,
                                                                       info_stride, nonband, want);
  // Row look-ahead (single matrix, RDB_GJ_LA_SIDE SMs, default 16): the side
  // stream updates the whole next row block, inverts its diagonal tile and
  // forms its row panel while the rest of the update runs on the other SMs,
  // so the next step starts with its row panel done (no one-round P2 launch).
  const int la_side = lookahead ? la_side_sms() : 0;
  for (int k = 0; k < nt; ++k) {
    const int p0 = k * NB;
    if (k > 0 && !lookahead)
      gj_panel_kernel<<<(unsigned)batch, p1::THREADS, p1::SMEM_BYTES, st>>>(a, lda, stride, p0, idx_base + p0,
                                                                           info, 0, info_stride, nonband, want);
    if (nt == 1) break;
    RowPanelSched rp{a, lda, stride, nt, k, (int)batch, batch > 1 ? dyn : nullptr};
    if (plan) {
      rp.list = plan->rp + (int64_t)k * batch * (nt - 1);
      rp.count_ptr = plan->counts + k;
    }
    if (!(la_side > 0 && k > 0))  // with the row look-ahead, step k's row panel was formed on the side stream
      gj_rowpanel_kernel<<<persistent_grid((int64_t)batch * (nt - 1)), EC::THREADS, EC::SMEM_BYTES, st>>>(
          amap, cmap, rp);
    if (la_side > 0 && k + 1 < nt) {
      cudaEventRecord(ds->ev_a, st);
      cudaStreamWaitEvent(side, ds->ev_a, 0);
      UpdateSched ua{a, cnt, lda, stride, nt, k, 1, 3, dyn ? dyn + 3 : nullptr};
      gj_update_kernel<<<(unsigned)(nt < la_side ? nt : la_side), EC::THREADS, EC::SMEM_BYTES, side>>>(amap, cmap, ua);
      const int p1n = (k + 1) * NB;
      gj_panel_kernel<<<1, p1::THREADS, p1::SMEM_BYTES, side>>>(a, lda, stride, p1n, idx_base + p1n, info, 0);
      RowPanelSched rn{a, lda, stride, nt, k + 1, 1, nullptr};
      gj_rowpanel_kernel<<<(unsigned)(nt - 1 < la_side ? nt - 1 : la_side), EC::THREADS, EC::SMEM_BYTES, side>>>(
          amap, cmap, rn);
      cudaEventRecord(ds->ev_p, side);
      UpdateSched ub{a, cnt, lda, stride, nt, k, 1, 4, dyn ? dyn + 1 : nullptr};
      const int64_t tiles = (int64_t)(nt - 2) * nt;
      const int main_grid = sm_count() - la_side;
      gj_update_kernel<<<(unsigned)(tiles < main_grid ? tiles : main_grid), EC::THREADS, EC::SMEM_BYTES, st>>>(
          amap, cmap, ub);
      cudaStreamWaitEvent(st, ds->ev_p, 0);
    } else if (lookahead && k + 1 < nt) {
      // side stream, one SM: the next diagonal tile, then its inverse (P1);
      // main stream, the other SMs: every other tile of this update
      cudaEventRecord(ds->ev_a, st);
      cudaStreamWaitEvent(side, ds->ev_a, 0);
      UpdateSched ua{a, cnt, lda, stride, nt, k, 1, 1};
      gj_update_kernel<<<1, EC::THREADS, EC::SMEM_BYTES, side>>>(amap, cmap, ua);
      const int p1n = (k + 1) * NB;
      gj_panel_kernel<<<1, p1::THREADS, p1::SMEM_BYTES, side>>>(a, lda, stride, p1n, idx_base + p1n, info, 0);
      cudaEventRecord(ds->ev_p, side);
      UpdateSched ub{a, cnt, lda, stride, nt, k, 1, 2, dyn ? dyn + 1 : nullptr};
      const int64_t tiles = (int64_t)(nt - 1) * nt - 1;
      const unsigned grid = (unsigned)(tiles < sm_count() - 1 ? tiles : sm_count() - 1);
      gj_update_kernel<<<grid, EC::THREADS, EC::SMEM_BYTES, st>>>(amap, cmap, ub);
      cudaStreamWaitEvent(st, ds->ev_p, 0);
    } else {
      UpdateSched up{a, cnt, lda, stride, nt, k, (int)batch, 0, dyn ? dyn + 1 : nullptr};
      if (plan) {
        up.list = plan->up + (int64_t)k * batch * (nt - 1) * nt;
        up.count_ptr = plan->counts + nt + k;
      }
      unsigned grid = persistent_grid((int64_t)batch * (nt - 1) * nt);
      if (grid_cap > 0 && grid > (unsigned)grid_cap) grid = (unsigned)grid_cap;
      gj_update_kernel<<<grid, EC::THREADS, EC::SMEM_BYTES, st>>>(amap, cmap, up);
    }
  }
  RDB_LAUNCH_CHECK();
  return RDB_OK;
}

// ------------------------------------------------------------------ dense 256-wide batched path (DW)
// Batched matrices whose strip pattern has no zero strip anywhere off the
// diagonal (the Erdos-Renyi half of config 2: the block-sparse plan would run
// every k-chunk anyway) take 256-wide Gauss-Jordan steps: every update tile
// then runs 16 k-chunks per epilogue instead of 8, halving the engine's
// per-tile switch + epilogue cost per flop (~2.4 us against 2.12 us per
// k-chunk). Step p, band B = block rows/columns 2p, 2p+1, for every listed matrix:
//   1. A_BB = A_BB^-1 in place: the NB = 128 Gauss-Jordan on the 256 x 256
//      block (invert_core on the sub-blocks, P1 via the path flag `want` = 2,
//      row panel / update tiles from prebuilt lists);
//   2. A_BJ = A_BB A_BJ (J outside B), in place: tiles (r, J), r = 0, 1, K = 256.
//      Both overwrite the B operand A_BJ they share: each signals when its
//      operands have landed and stores only when both have (column counters);
//   3. A_IJ += -(A_IB A_BJ) (I, J outside B, TMA reduce-add) and
//      A_I,B = -(A_IB A_BB) (the two band tiles, store): the band tiles
//      overwrite A_IB, every tile's A operand in row block I, so they store
//      only when all nt tiles of that row have loaded it (row counters).
// Same algebra as the NB = 128 steps (the nested inverse is their first two
// steps on the band); rounding order differs, so the inverse agrees to
// ~1e-15 relative and D is unchanged (tests compare with the reference).
// Waits point to tiles of smaller index or to the tile's own dependency group
// (dmma_engine.cuh, Tile::wait: the producer gates on them, the MMA warps never block).
struct WBRowSched {
  double* a;
  int64_t lda, stride;
  int nt, p0t, step;
  const int* list;        // listed matrices (indices within the strided batch)
  const int* list_count;  // device count
  int* colcnt;            // [g][nt] cumulative column counters
  int* dyn;
  RDB_DEV int count() const { return *list_count * (nt - 2) * 2; }
  RDB_DEV eng::Tile tile(int t) const {
    const int r = t & 1, q = t >> 1;
    const int li = q / (nt - 2), jj = q - li * (nt - 2);
    const int J = jj + (jj >= p0t ? 2 : 0);
    const int g = list[li];
    double* A = a + (int64_t)g * stride;
    eng::Tile T;
    T.a_col = p0t * NB;  // A operand: D rows r (128 x 256)
    T.a_row = (p0t + r) * NB;
    T.a_mat = g;
    T.b = A + (int64_t)p0t * NB * lda + (int64_t)J * NB;  // A_BJ, 256 x 128
    T.ldb = lda;
    T.c_col = J * NB;
    T.c_row = (p0t + r) * NB;
    T.c_mat = g;
    T.nk = 2 * NB / eng::BK;
    T.mode = eng::EPI_STORE;
    T.neg = 0;
    int* c = colcnt + (int64_t)g * nt + J;
    T.signal = c;
    T.wait = c;
    T.wait_target = 2 * (step - ((J >> 1) < step ? 1 : 0) + 1);
    return T;
  }
};

struct WBUpdateSched {
  double* a;
  int64_t lda, stride;
  int nt, p0t, step;
  const int* list;
  const int* list_count;
  int* rowcnt;  // [g][nt] cumulative row counters
  int* dyn;
  // part 0: every tile; 1: the next band's 2 x 2 diagonal tiles only (look-ahead:
  // the next band inverse can start); 2: every tile except those
  int part = 0;
  int dyn_ctas = 0;  // > 0: CTAs of the main and the helper launch sharing dyn
  RDB_DEV int per() const { return part == 1 ? 4 : (nt - 2) * nt - (part == 2 ? 4 : 0); }
  RDB_DEV int count() const { return *list_count * per(); }
  RDB_DEV eng::Tile tile(int t) const {
    const int pm = per();
    const int li = t / pm;
    int rem = t - li * pm;
    int ri, jj;
    if (part == 1) {  // rows / columns p0t + 2, p0t + 3 = index p0t, p0t + 1 outside the band
      ri = p0t + (rem >> 1);
      jj = p0t + (rem & 1);
    } else if (part == 0 || rem < p0t * nt) {
      ri = rem / nt;
      jj = rem - ri * nt;
    } else if ((rem -= p0t * nt) < 2 * (nt - 2)) {  // the next band's rows without its two columns
      ri = p0t + rem / (nt - 2);
      jj = rem - (ri - p0t) * (nt - 2);
      jj += (jj >= p0t) ? 2 : 0;
    } else {
      rem -= 2 * (nt - 2);
      ri = p0t + 2 + rem / nt;
      jj = rem - (ri - p0t - 2) * nt;
    }
    const int I = ri + (ri >= p0t ? 2 : 0);
    const int g = list[li];
    double* A = a + (int64_t)g * stride;
    eng::Tile T;
    T.a_col = p0t * NB;  // A operand: A_IB, 128 x 256
    T.a_row = I * NB;
    T.a_mat = g;
    T.c_row = I * NB;
    T.c_mat = g;
    T.nk = 2 * NB / eng::BK;
    T.neg = 1;
    T.ldb = lda;
    int* c = rowcnt + (int64_t)g * nt + I;
    T.signal = c;
    if (jj < nt - 2) {
      const int J = jj + (jj >= p0t ? 2 : 0);
      T.b = A + (int64_t)p0t * NB * lda + (int64_t)J * NB;  // the new row panel A_BJ
      T.c_col = J * NB;
      T.mode = eng::EPI_REDUCE;
      T.wait = nullptr;
      T.wait_target = 0;
    } else {
      const int h = jj - (nt - 2);
      T.b = A + (int64_t)p0t * NB * lda + (int64_t)(p0t + h) * NB;  // columns h of A_BB (= its inverse)
      T.c_col = (p0t + h) * NB;
      T.mode = eng::EPI_STORE;
      T.wait = c;
      T.wait_target = nt * (step - ((I >> 1) < step ? 1 : 0) + 1);
    }
    return T;
  }
};

__global__ void __launch_bounds__(EC::THREADS, 1)
    gj_wb_row_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap cmap,
                     WBRowSched sched) {
  RDB_TRACE_SCOPE(4);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  eng::run<EC>(smem_raw, &amap, sched, eng::BulkEpilogue<EC>{&cmap});
}

__global__ void __launch_bounds__(EC::THREADS, 1)
    gj_wb_update_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap cmap,
                        WBUpdateSched sched) {
  RDB_TRACE_SCOPE(10 + sched.part);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  eng::run<EC>(smem_raw, &amap, sched, eng::BulkEpilogue<EC>{&cmap});
}

// ---- two-level dense-wide path (n = 1024): two outer steps of width W = n/2
// (bt = W / 128 tiles), their band inverses W x W dense-wide inversions
// (dw_part on the sub-block). Outer step p, band B = tiles [b0t, b0t + bt):
//   row panel: A_BJ = D A_BJ (J outside B), tiles (r, J), K = W, in place on
//     the B operand they share: each signals when its operands have landed,
//     stores when all bt have (column counters, target bt);
//   update: A_IJ += -(A_IB A_BJ) (J outside B, reduce) and A_IB = -(A_IB D)
//     (store, after all nt tiles of row I have loaded A_IB: row counters,
//     target nt).
// Each column / row block takes part in one outer row panel / update, so the
// counters (zeroed before each step) need no step arithmetic.
struct W2RowSched {
  double* a;
  int64_t lda, stride;
  int nt, b0t, bt;
  const int* list;
  const int* list_count;
  int* colcnt;
  int* dyn;
  RDB_DEV int count() const { return *list_count * (nt - bt) * bt; }
  RDB_DEV eng::Tile tile(int t) const {
    const int r = t % bt, q = t / bt;
    const int li = q / (nt - bt), jj = q - li * (nt - bt);
    const int J = jj + (jj >= b0t ? bt : 0);
    const int g = list[li];
    double* A = a + (int64_t)g * stride;
    eng::Tile T;
    T.a_col = b0t * NB;  // A operand: D rows r (128 x W)
    T.a_row = (b0t + r) * NB;
    T.a_mat = g;
    T.b = A + (int64_t)b0t * NB * lda + (int64_t)J * NB;  // A_BJ, W x 128
    T.ldb = lda;
    T.c_col = J * NB;
    T.c_row = (b0t + r) * NB;
    T.c_mat = g;
    T.nk = bt * NB / eng::BK;
    T.mode = eng::EPI_STORE;
    T.neg = 0;
    int* c = colcnt + (int64_t)g * nt + J;
    T.signal = c;
    T.wait = c;
    T.wait_target = bt;
    return T;
  }
};

struct W2UpdateSched {
  double* a;
  int64_t lda, stride;
  int nt, b0t, bt;
  const int* list;
  const int* list_count;
  int* rowcnt;
  int* dyn;
  int dyn_ctas = 0;
  RDB_DEV int count() const { return *list_count * (nt - bt) * nt; }
  RDB_DEV eng::Tile tile(int t) const {
    const int pm = (nt - bt) * nt;
    const int li = t / pm, rem = t - li * pm;
    const int ri = rem / nt, jj = rem - ri * nt;
    const int I = ri + (ri >= b0t ? bt : 0);
    const int g = list[li];
    double* A = a + (int64_t)g * stride;
    eng::Tile T;
    T.a_col = b0t * NB;  // A operand: A_IB, 128 x W
    T.a_row = I * NB;
    T.a_mat = g;
    T.c_row = I * NB;
    T.c_mat = g;
    T.nk = bt * NB / eng::BK;
    T.neg = 1;
    T.ldb = lda;
    int* c = rowcnt + (int64_t)g * nt + I;
    T.signal = c;
    if (jj < nt - bt) {
      const int J = jj + (jj >= b0t ? bt : 0);
      T.b = A + (int64_t)b0t * NB * lda + (int64_t)J * NB;  // the new row panel A_BJ
      T.c_col = J * NB;
      T.mode = eng::EPI_REDUCE;
      T.wait = nullptr;
      T.wait_target = 0;
    } else {
      const int h = jj - (nt - bt);
      T.b = A + (int64_t)b0t * NB * lda + (int64_t)(b0t + h) * NB;  // columns h of D
      T.c_col = (b0t + h) * NB;
      T.mode = eng::EPI_STORE;
      T.wait = c;
      T.wait_target = nt;
    }
    return T;
  }
};

__global__ void __launch_bounds__(EC::THREADS, 1)
    gj_w2_row_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap cmap,
                     W2RowSched sched) {
  RDB_TRACE_SCOPE(14);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  eng::run<EC>(smem_raw, &amap, sched, eng::BulkEpilogue<EC>{&cmap});
}

__global__ void __launch_bounds__(EC::THREADS, 1)
    gj_w2_update_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap cmap,
                        W2UpdateSched sched) {
  RDB_TRACE_SCOPE(15);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  eng::run<EC>(smem_raw, &amap, sched, eng::BulkEpilogue<EC>{&cmap});
}

// Per-part device state of the DW path (inside the batched workspace).
struct DwPart {
  int* list;    // [cnt] local indices of the part's DW matrices
  int* count;   // 1 int
  int* ncounts; // nested plan counts [2][2]
  int* nrp;     // nested row-panel entries [2][cnt]
  int2* nup;    // nested update entries [2][2 cnt]
  int* ncnt;    // nested row-block counters (invert_core work, 16-byte aligned)
  int* colcnt;  // [cnt][nt]
  int* rowcnt;  // [cnt][nt]
  int* list_s;  // [cnt] listed matrices whose first step is sparse (count[1]), in list order
  int* list_d;  // [cnt] the others (count[2]): their first step runs the dense tiles
};

// One CTA per part: classify the part's matrices (flag 1 -> 2 when every
// off-diagonal block has all 8 column and all 8 row strips), zero their strip
// patterns (the block-sparse plan then lists no tiles for them), and write the
// part's list plus the nested-inverse plan lists, in matrix order.
struct DwClassifyArgs {
  unsigned char* pat;
  int* flags;
  int64_t batch;
  int nt, parts;
  DwPart part[4];
};

__global__ void __launch_bounds__(1024) dw_classify_kernel(DwClassifyArgs arg) {
  RDB_TRACE_SCOPE(32);
  const int i = blockIdx.x;
  const int nt = arg.nt, ld = pat_ld(nt), wpm = 2 * nt * ld / 4;  // pattern words per matrix
  const int64_t cnt = (arg.batch - i + arg.parts - 1) / arg.parts;
  const DwPart& d = arg.part[i];
  __shared__ int warp_tot[32];
  __shared__ int base;
  __shared__ unsigned char dense_s[1024];
  if (threadIdx.x == 0) base = 0;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t l0 = 0; l0 < cnt; l0 += 1024) {
    const int64_t nl = cnt - l0 < 1024 ? cnt - l0 : 1024;
    __syncthreads();
    {
      const int64_t l = l0 + threadIdx.x;
      dense_s[threadIdx.x] = l < cnt && arg.flags[i + (int64_t)arg.parts * l] == 1;
    }
    __syncthreads();
    // every (matrix, pattern word) of the chunk across the CTA: a zero strip
    // off the diagonal clears the matrix's flag
    for (int64_t e = threadIdx.x; e < nl * wpm; e += 1024) {
      const int64_t ll = e / wpm;
      const int wi = (int)(e - ll * wpm);
      if (!dense_s[ll]) continue;
      const int64_t m = i + (int64_t)arg.parts * (l0 + ll);
      const uint32_t v = reinterpret_cast<const uint32_t*>(arg.pat + m * 2 * nt * ld)[wi];
      const int I = (wi / (ld / 4)) % nt, J0 = 4 * (wi % (ld / 4));
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int J = J0 + b;
        if (J < nt && J != I && ((v >> (8 * b)) & 0xFFu) != 0xFFu) dense_s[ll] = 0;
      }
    }
    __syncthreads();
    // ordered compaction (block scan of the dense flags)
    const int64_t l = l0 + threadIdx.x;
    const int64_t m = i + (int64_t)arg.parts * l;
    const bool dense = threadIdx.x < nl && dense_s[threadIdx.x];
    const unsigned bal = __ballot_sync(0xffffffffu, dense);
    if (lane == 0) warp_tot[w] = __popc(bal);
    __syncthreads();
    int off = base;
    for (int k = 0; k < w; ++k) off += warp_tot[k];
    const int pos = off + __popc(bal & ((1u << lane) - 1));
    if (dense) {
      arg.flags[m] = 2;
      uint32_t* P = reinterpret_cast<uint32_t*>(arg.pat + m * 2 * nt * ld);
      for (int e = 0; e < wpm; ++e) P[e] = 0u;
      d.list[pos] = (int)l;
      d.list_d[pos] = (int)l;  // (the sparse-first-step split refines list_s / list_d)
      for (int k = 0; k < 2; ++k) {
        d.nrp[k * cnt + pos] = (int)(l << 13) | (8 << 6) | (1 - k);
        d.nup[k * 2 * cnt + 2 * pos] = make_int2((int)(l << 12) | ((1 - k) << 6) | (1 - k), 1 | (8 << 20));
        d.nup[k * 2 * cnt + 2 * pos + 1] = make_int2((int)(l << 12) | ((1 - k) << 6) | k, 1 | (8 << 20));
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int k = 0; k < 32; ++k) tot += warp_tot[k];
      base += tot;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    d.count[0] = base;
    d.count[1] = 0;
    d.count[2] = base;
    // the two-level path's inner level reads its counts at count + 4: the
    // sparse-first-step split refines them; without it (RDB_GJ_DW_S0=0, or a
    // generic call whose split never runs) they are the classification's
    d.count[4] = base;
    d.count[5] = 0;
    d.count[6] = base;
    d.ncounts[0] = d.ncounts[1] = base;          // nested row panels, steps 0 and 1
    d.ncounts[2] = d.ncounts[3] = 2 * base;      // nested update tiles
  }
}

// ---- sparse first step of the DW path (matrices built from bit-packed adjacency)
// Step 0 reads the input M = I - gamma W itself: its block row 0 (A_0J, J
// outside the band) and block column 0 (A_I0) hold only the graph's edges
// (config 2's Erdos-Renyi graphs: ~5 per row / column of a 256-wide block), so
// the step's rank-256 products are sparse:
//   A_0J = D A_0J                   (D = A_00^-1 from the nested inverse)
//   A_iJ = A_iJ - sum_k a_ik A_kJ   (i outside the band, k over the edges of
//   A_i0 = -sum_k a_ik D_k,:         row i into block 0, in increasing k)
// — the same algebra as the dense tiles of step 0 (a zero a_ik contributes an
// exact zero), summed in a different order (the inverse agrees to rounding,
// D is unchanged; tests compare with the reference). The dense step-0 tiles
// (1/4 of the matrix's flop at n = 1024) are skipped; what is left is one
// pass over the matrix in HBM (read M_i, write A_i).
//   dw_s0_gather_kernel: the edges of block column 0 (per row i) and block
//     row 0 (per column j), with their values, into compact lists (a snapshot:
//     the step overwrites them in place), in increasing k; a matrix with more
//     than S0_CAP edges in any such row or column keeps the dense step;
//   dw_s0_row_kernel: A_0J = D A_0J, 16 rows of D (transposed) in shared
//     memory per CTA, a half-warp per output column;
//   dw_s0_update_kernel: the rows outside the band, a warp per row, block
//     row 0 (as updated) read from L2.
// The lists live in the matrix's slice of the banded path's scratch, which
// the banded inverse uses only for banded matrices (never dense-wide ones).
// Edges kept per row / column of the step-0 blocks: B0 = 256 (one-level
// steps, ~5 per row for config 2) or 512 (the two-level path's outer step,
// ~10 per row); a matrix with more in any row or column keeps the dense step.
template <int B0>
struct S0 {
  static constexpr int CAP = B0 == 256 ? 24 : 32;
};
constexpr int S0_CAP = S0<256>::CAP;  // (host restatement: batch.py S0_CAP)

// List layout inside a matrix's slice (R = n - B0 rows / columns outside the
// band): row and column lists both row-major (a half-warp reads one row's /
// column's entries in one pass, two 16-bit indices per lane):
// vals_r [R][CAP] double | vals_c [R][CAP] double | idx_r [R][CAP] u16 |
// idx_c [R][CAP] u16 | cnt_r [R] u8 | cnt_c [R] u8.
struct S0Lists {
  double *vr, *vc;
  unsigned short *ir, *ic;
  unsigned char *nr, *nc;
  RDB_HOST_DEV S0Lists(void* base, int R, int cap) {
    vr = static_cast<double*>(base);
    vc = vr + (size_t)cap * R;
    ir = reinterpret_cast<unsigned short*>(vc + (size_t)cap * R);
    ic = ir + (size_t)cap * R;
    nr = reinterpret_cast<unsigned char*>(ic + (size_t)cap * R);
    nc = nr + R;
  }
  static size_t bytes(int R, int cap) { return (size_t)R * cap * (2 * sizeof(double) + 4) + 2 * (size_t)R; }
};

struct S0Args {
  double* a;              // the (sub)problem: matrix l at a + l * pstride, n x n, row pitch lda
  int64_t lda, pstride;
  char* lists;            // part-local matrix l's lists at lists + l * lstride
  int64_t lstride;
  int n;                  // the problem's size (multiple of 256)
  const int* list;        // list_s
  const int* count;       // count[1] = entries of list_s
  int* colcnt;            // one-level path: the step-0 counts of the dense tiles (nullptr: none)
  int* rowcnt;
  // gather / split (dw_s0_gather_kernel, dw_s0_split_kernel)
  const uint32_t* bits;   // part-local matrix l at bits + l * bstride (rows of wpr words)
  int64_t bstride, wpr, n_bits;  // n_bits: vertices inside the problem (<= n)
  int* bad;               // part-local matrix l's flags at bad[l * bad_stride] (bit bad_bit: dense step)
  int64_t bad_stride;
  int bad_bit;
  const int* n_list;      // entries of the part's dense-wide list
  const int* dw_list;     // the part's dense-wide list
  int* list_s;
  int* list_d;
  int* counts;            // counts[0..2] written by the split (list, list_s, list_d entries)
  // M built from the adjacency bits (the APSP pipelines): part-local matrix l
  // is I - gam[l * gam_stride] A; the gather then takes the edge values from
  // the gain, and the sparse step writes rows outside the band from the bits
  // (K1 built only what the first band inverse reads). nullptr: M is the
  // caller's, read from memory.
  const double* gam;
  int64_t gam_stride;
};

// The edges of row or column B0 + t (thread's role) into / out of block 0, in
// increasing k, into ps (at most CAP kept); returns the total count.
template <int B0>
RDB_DEV int s0_positions(const uint32_t* bm, int64_t wpr, int64_t n_bits, int nb0, bool col, int t, int tl,
                         const uint32_t (*sw)[9], unsigned short* ps) {
  constexpr int CAP = S0<B0>::CAP;
  const int w0 = (nb0 + 31) / 32;
  int c = 0;
  if (!col) {  // row i = B0 + t: edges k < nb0 (the row's words loaded together)
    const int64_t i = B0 + t;
    uint32_t wr[B0 / 32];
#pragma unroll
    for (int q = 0; q < B0 / 32; ++q) wr[q] = (q < w0 && i < n_bits) ? bm[i * wpr + q] : 0u;
#pragma unroll
    for (int q = 0; q < B0 / 32; ++q) {
      uint32_t w = wr[q];
      while (w) {
        const int k = 32 * q + __ffs(w) - 1;
        w &= w - 1;
        if (ps && c < CAP) ps[c] = (unsigned short)k;
        ++c;
      }
    }
  } else {  // column j = B0 + t: edges k < nb0 (sw: the chunk's words of rows k)
    const int q = tl >> 5, b = tl & 31;
    for (int k = 0; k < nb0; ++k)
      if ((sw[k][q] >> b) & 1) {
        if (ps && c < CAP) ps[c] = (unsigned short)k;
        ++c;
      }
  }
  return c;
}

// bits words of rows k < nb0 for the 256-column chunk x (columns B0 + 256 x ..)
template <int B0>
RDB_DEV void s0_stage_words(const uint32_t* bm, int64_t wpr, int nb0, uint32_t (*sw)[9], int x) {
  const int64_t q0 = (B0 + (int64_t)x * 256) / 32;
  for (int e = threadIdx.x; e < nb0 * 8; e += blockDim.x) {
    const int k = e >> 3, q = e & 7;
    sw[k][q] = q0 + q < wpr ? bm[k * wpr + q0 + q] : 0u;
  }
}

// Before K1 (APSP pipelines, M from bits): grid (2 ceil(R / 256), batch), 256
// threads (x even: rows, odd: columns of chunk x / 2), dense-wide matrices
// (flags == 2), the problem = the leading n x n block: bad[m] |= bit when a
// row of block column 0 or a column of block row 0 (B0 wide) has more than
// CAP edges.
template <int B0>
__global__ void __launch_bounds__(256) dw_s0_count_kernel(const uint32_t* __restrict__ bits, int64_t n_bits,
                                                          int n, const int* __restrict__ flags, int* __restrict__ bad,
                                                          int bit) {
  const int64_t m = blockIdx.y;
  if (flags[m] != 2) return;
  const int R = n - B0;
  const int64_t wpr = (n_bits + 31) / 32;
  const uint32_t* bm = bits + m * n_bits * wpr;
  const int64_t nb = n_bits < n ? n_bits : n;
  const int nb0 = (int)(nb < B0 ? nb : B0);
  const bool col = blockIdx.x & 1;
  const int x = blockIdx.x >> 1, tl = threadIdx.x, t = x * 256 + tl;
  __shared__ uint32_t sw[B0][9];
  if (col) s0_stage_words<B0>(bm, wpr, nb0, sw, x);
  __syncthreads();
  if (t >= R) return;
  // (columns past the problem's n are outside: the chunk covers B0 + 256 x + [0, 256) < n)
  if (s0_positions<B0>(bm, wpr, nb, nb0, col, t, tl, sw, nullptr) > S0<B0>::CAP) atomicOr(bad + m, bit);
}

// grid (2 ceil(R / 256), list capacity), 256 threads, for the part's
// dense-wide matrices: x even, thread t gathers row B0 + 256 (x / 2) + t; x
// odd, column B0 + 256 (x / 2) + t; bad |= bit when one has more than CAP
// edges. Runs on the part's side stream beside the first band inverse.
template <int B0>
__global__ void __launch_bounds__(256, 4) dw_s0_gather_kernel(S0Args g) {
  RDB_TRACE_SCOPE(33);
  constexpr int CAP = S0<B0>::CAP;
  if ((int)blockIdx.y >= *g.n_list) return;
  const int l = g.dw_list[blockIdx.y];
  const int n = g.n;
  const int64_t n_bits = g.n_bits, lda = g.lda, wpr = g.wpr;
  const int R = n - B0;
  const uint32_t* bm = g.bits + (int64_t)l * g.bstride;
  const double* A = g.a + (int64_t)l * g.pstride;
  const S0Lists L(g.lists + (int64_t)l * g.lstride, R, CAP);
  const int nb0 = (int)(n_bits < B0 ? n_bits : B0);
  const bool col = blockIdx.x & 1;
  const int x = blockIdx.x >> 1, tl = threadIdx.x;
  const int t = x * 256 + tl;               // row / column index - B0
  __shared__ uint32_t sw[B0][9];            // the chunk's 8 words of rows k < nb0 (padded)
  __shared__ unsigned short pos[256][CAP];  // edge positions, then one batch of value loads
  if (col) s0_stage_words<B0>(bm, wpr, nb0, sw, x);
  __syncthreads();
  if (t >= R) return;
  unsigned short* ps = pos[threadIdx.x];
  const int c = s0_positions<B0>(bm, wpr, n_bits, nb0, col, t, tl, sw, ps);
  const int nc = c < CAP ? c : CAP;
  const double* src = col ? A + B0 + t : A + (int64_t)(B0 + t) * lda;  // column: row k at src + k lda
  const int64_t step = col ? lda : 1;
  const double ng = g.gam ? -g.gam[(int64_t)l * g.gam_stride] : 0.0;  // M from bits: every edge is -gamma
  constexpr int H = 12;
  for (int e0 = 0; e0 < nc; e0 += H) {  // H independent loads at a time (one batch for most)
    double v[H];
#pragma unroll
    for (int e = 0; e < H; ++e) v[e] = e0 + e < nc ? (g.gam ? ng : src[ps[e0 + e] * step]) : 0.0;
#pragma unroll
    for (int e = 0; e < H; ++e)
      if (e0 + e < nc) {
        if (!col) {
          L.ir[(size_t)t * CAP + e0 + e] = ps[e0 + e];
          L.vr[(size_t)t * CAP + e0 + e] = v[e];
        } else {
          L.ic[(size_t)t * CAP + e0 + e] = ps[e0 + e];
          L.vc[(size_t)t * CAP + e0 + e] = v[e];
        }
      }
  }
  (col ? L.nc : L.nr)[t] = (unsigned char)nc;
  if (!g.gam && c > CAP) atomicOr(g.bad + (int64_t)l * g.bad_stride, g.bad_bit);  // (M from bits: counted before K1)
}

// One CTA: the part's dense-wide list split by the flags' bit into list_s
// (sparse first step) and list_d, both in list order.
__global__ void __launch_bounds__(1024) dw_s0_split_kernel(S0Args g) {
  __shared__ int wt[32], ws[32];
  __shared__ int base, base_s;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) base = base_s = 0;
  __syncthreads();
  const int cnt = *g.n_list;
  for (int p0 = 0; p0 < cnt; p0 += 1024) {
    const int p = p0 + threadIdx.x;
    const int l = p < cnt ? g.dw_list[p] : 0;
    const bool in = p < cnt, sp = in && !(g.bad[(int64_t)l * g.bad_stride] & g.bad_bit);
    const unsigned bi = __ballot_sync(0xffffffffu, in), bs = __ballot_sync(0xffffffffu, sp);
    if (lane == 0) {
      wt[w] = __popc(bi);
      ws[w] = __popc(bs);
    }
    __syncthreads();
    int off = base, off_s = base_s;
    for (int k = 0; k < w; ++k) {
      off += wt[k];
      off_s += ws[k];
    }
    const int pos = off + __popc(bi & ((1u << lane) - 1)), pos_s = off_s + __popc(bs & ((1u << lane) - 1));
    if (sp) g.list_s[pos_s] = l;
    else if (in) g.list_d[pos - pos_s] = l;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int k = 0; k < 32; ++k) {
        base += wt[k];
        base_s += ws[k];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    g.counts[0] = base;
    g.counts[1] = base_s;
    g.counts[2] = base - base_s;
  }
}

// The row panel's sparse products, one half-warp (16 lanes, lane c) per
// output column: o += sum_e a_e * S[idx_e][c] over the column's edge list, in
// list order (increasing k: the same sums, bit for bit, as a lane-per-column
// kernel would form). S is a 16-row strip of the dense operand in shared
// memory, transposed, so every edge costs one conflict-free 128-byte read
// per half-warp; the list (CAP 16-bit indices, row-major) sits in the
// half-warp's registers, two entries per lane, and is broadcast a pair at a
// time by one shuffle. CONSTV: every edge value is the same (M built from
// adjacency bits: -gamma); otherwise lane c also holds the values of entries
// 2c and 2c + 1. The lists are loaded without looking at their counts first
// (the slots past a count are allocated, never used), so no load depends on
// another.
RDB_DEV double s0_fma(double a, double s, double o) { return fma(a, s, o); }
// shared-memory reads by 32-bit shared address (the strip's base is converted
// once per thread; through a generic pointer the compiler rebuilt the shared
// window base at every read)
RDB_DEV void s0_lds(unsigned addr, double& v) { asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr)); }

// sbase: shared address of S[0][c]; PITCHB: bytes per row of S. S has one
// more row than the operand, all zeros (row ZROW): s0_fix points every list
// slot at or past the row's count there (and zeroes its value), so the loop
// body has no predicate — such a slot adds cv * 0 = 0 to an accumulator that
// is never -0 (it starts from +0, 1 or an edge value), i.e. nothing.
template <int ZROW>
RDB_DEV void s0_fix(unsigned& pk, double& v0, double& v1, int c, int cnt) {
  if (2 * c + 1 >= cnt) {
    pk = (pk & 0xFFFFu) | ((unsigned)ZROW << 16);
    v1 = 0.0;
  }
  if (2 * c >= cnt) {
    pk = (unsigned)ZROW | ((unsigned)ZROW << 16);
    v0 = 0.0;
  }
}

// Two independent lists at once (two output columns of the half-warp): twice
// the loads in flight per warp; the trip count covers the longest of the
// four lists of the warp (shorter ones run on into the zero row).
template <int PITCHB, bool CONSTV, class T>
RDB_DEV void s0_accumulate2(T& oa, T& ob, unsigned sbase, int cmax, unsigned packed_a, unsigned packed_b, double va0,
                            double va1, double vb0, double vb1, double cv) {
#pragma unroll 2
  for (int p = 0; 2 * p < cmax; ++p) {
    const unsigned pa = __shfl_sync(0xffffffffu, packed_a, p, 16);
    const unsigned pb = __shfl_sync(0xffffffffu, packed_b, p, 16);
    double a0 = cv, a1 = cv, b0 = cv, b1 = cv;
    if (!CONSTV) {
      a0 = __shfl_sync(0xffffffffu, va0, p, 16);
      a1 = __shfl_sync(0xffffffffu, va1, p, 16);
      b0 = __shfl_sync(0xffffffffu, vb0, p, 16);
      b1 = __shfl_sync(0xffffffffu, vb1, p, 16);
    }
    T sa0, sa1, sb0, sb1;
    s0_lds(sbase + (pa & 0xFFFFu) * PITCHB, sa0);
    s0_lds(sbase + (pb & 0xFFFFu) * PITCHB, sb0);
    s0_lds(sbase + (pa >> 16) * PITCHB, sa1);
    s0_lds(sbase + (pb >> 16) * PITCHB, sb1);
    oa = s0_fma(a0, sa0, oa);
    ob = s0_fma(b0, sb0, ob);
    oa = s0_fma(a1, sa1, oa);
    ob = s0_fma(b1, sb1, ob);
  }
}

// A_0J = D A_0J: rows k0 .. k0 + 15 of block row 0 per CTA (k0 = 16
// blockIdx.x). D's 16 rows sit transposed in shared memory (S[m][kk] =
// D[k0 + kk][m], pitch 17: conflict-free both ways), so column j of the
// result is the combination of the rows S[m] its edges m -> j select: a
// half-warp per column, CB = 8 columns per batch (their lists loaded QB
// columns at a time, all loads in flight together), staged through a private
// 16 x 8 tile so the stores are 64-byte row segments. grid (B0 / 16, list
// capacity), 512 threads; 107 KB (B0 = 512: two CTAs, 32 warps per SM) or
// 72 KB (B0 = 256: three CTAs) of shared memory.
#ifndef RDB_S0_ROW_THREADS
#define RDB_S0_ROW_THREADS 512
#endif
template <int B0>
struct S0Row {
  static constexpr int P = 17, THREADS = RDB_S0_ROW_THREADS, NH = THREADS / 16, CB = 8, PO = CB + 1;
  static constexpr size_t SMEM = ((size_t)(B0 + 1) * P + NH * 16 * PO) * sizeof(double);  // + the zero row
};

template <int B0, bool CONSTV>
RDB_DEV void s0_row_columns(const S0Args& g, const S0Lists& L, double* A, unsigned sbase, double* O, int R, int k0,
                            int hw, int c, double cv) {
  using K = S0Row<B0>;
  constexpr int CAP = S0<B0>::CAP, P = K::P, CB = K::CB, PO = K::PO, QB = CONSTV ? CB : 4;
  for (int t0 = hw * CB; t0 < R; t0 += K::NH * CB) {  // this half-warp's CB columns B0 + t0 ..
    const int cnts = (c < CB && t0 + c < R) ? L.nc[t0 + c] : 0;
#pragma unroll 1
    for (int q0 = 0; q0 < CB; q0 += QB) {
      unsigned pk[QB];
      double v0[QB], v1[QB];
#pragma unroll
      for (int q = 0; q < QB; ++q) {
        const size_t t = (size_t)min(t0 + q0 + q, R - 1);
        pk[q] = *reinterpret_cast<const unsigned*>(L.ic + t * CAP + 2 * c);
        v0[q] = v1[q] = 0.0;
        if (!CONSTV) {
          v0[q] = L.vc[t * CAP + 2 * c];
          v1[q] = L.vc[t * CAP + 2 * c + 1];
        }
      }
#pragma unroll
      for (int q = 0; q < QB; q += 2) {
        const int cnt_a = __shfl_sync(0xffffffffu, cnts, q0 + q, 16);
        const int cnt_b = __shfl_sync(0xffffffffu, cnts, q0 + q + 1, 16);
        const int cm = max(cnt_a, cnt_b);
        const int cmax = max(cm, __shfl_xor_sync(0xffffffffu, cm, 16));
        s0_fix<B0>(pk[q], v0[q], v1[q], c, cnt_a);
        s0_fix<B0>(pk[q + 1], v0[q + 1], v1[q + 1], c, cnt_b);
        double oa = 0.0, ob = 0.0;
        s0_accumulate2<P * 8, CONSTV, double>(oa, ob, sbase, cmax, pk[q], pk[q + 1], v0[q], v1[q], v0[q + 1],
                                              v1[q + 1], cv);
        O[c * PO + q0 + q] = oa;
        O[c * PO + q0 + q + 1] = ob;
      }
    }
    __syncwarp();
    const int cc = c & (CB - 1), rr = c / CB;  // two rows of the tile per pass
    if (t0 + cc < R) {
#pragma unroll 4
      for (int r = rr; r < 16; r += 16 / CB) A[(int64_t)(k0 + r) * g.lda + B0 + t0 + cc] = O[r * PO + cc];
    }
    __syncwarp();
  }
}

template <int B0>
__global__ void __launch_bounds__(S0Row<B0>::THREADS) dw_s0_row_kernel(S0Args g) {
  RDB_TRACE_SCOPE(6);
  using K = S0Row<B0>;
  constexpr int CAP = S0<B0>::CAP, P = K::P;
  if ((int)blockIdx.y >= g.count[1]) return;
  const int l = g.list[blockIdx.y];
  double* A = g.a + (int64_t)l * g.pstride;
  const int R = g.n - B0;
  const S0Lists L(g.lists + (int64_t)l * g.lstride, R, CAP);
  const int tid = threadIdx.x, k0 = (int)blockIdx.x * 16;
  const int nt = g.n / NB;
  if (g.colcnt && blockIdx.x == 0 && tid < nt) {  // the step-0 counts the dense tiles would have signalled
    g.colcnt[(int64_t)l * nt + tid] = tid >= 2 ? 2 : 0;
    g.rowcnt[(int64_t)l * nt + tid] = tid >= 2 ? nt : 0;
  }
  extern __shared__ __align__(16) double s0_smem[];
  double* S = s0_smem;
  for (int e = tid; e < 16 * B0; e += K::THREADS)
    S[(e % B0) * P + e / B0] = A[(int64_t)(k0 + e / B0) * g.lda + e % B0];
  if (tid < P) S[B0 * P + tid] = 0.0;
  __syncthreads();
  const int hw = tid >> 4, c = tid & 15;
  double* O = s0_smem + (size_t)(B0 + 1) * P + hw * 16 * K::PO;
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(S + c);
  if (g.gam)  // a_mj = -gamma
    s0_row_columns<B0, true>(g, L, A, sbase, O, R, k0, hw, c, -g.gam[(int64_t)l * g.gam_stride]);
  else
    s0_row_columns<B0, false>(g, L, A, sbase, O, R, k0, hw, c, 0.0);
}

// Rows [r0, r1) outside the band: A_i = M'_i - sum_k a_ik A_k (block row 0
// as updated, read from L2), M' = M with block column 0 zeroed. A warp per
// row: its edge list in one load (lane e holds entry e), then passes over
// 256 columns (4 16-byte chunks per lane). Low register count: 4 CTAs per SM
// keep enough loads in flight. grid ((r1 - r0) / 8, list capacity).
template <int B0>
__global__ void __launch_bounds__(256, 4) dw_s0_update_kernel(S0Args g, int r0, int r1) {
  RDB_TRACE_SCOPE(7);
  constexpr int CAP = S0<B0>::CAP;
  if ((int)blockIdx.y >= g.count[1]) return;
  const int l = g.list[blockIdx.y];
  double* A = g.a + (int64_t)l * g.pstride;
  const int R = g.n - B0;
  const S0Lists L(g.lists + (int64_t)l * g.lstride, R, CAP);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = r0 + (int)blockIdx.x * 8 + warp;
  if (i >= r1) return;
  const int t = i - B0;
  const int cnt = L.nr[t];
  int kl = 0;
  double vl = 0.0;
  if (lane < cnt) {
    kl = L.ir[(size_t)t * CAP + lane];
    vl = L.vr[(size_t)t * CAP + lane];
  }
  double* Ai = A + (int64_t)i * g.lda;
  // M from bits: M'_ij = [i == j] - gamma [edge i -> j] (j >= B0), no read of M
  const uint32_t* brow = g.bits + (int64_t)l * g.bstride + (int64_t)i * g.wpr;
  const double ng = g.gam ? -g.gam[(int64_t)l * g.gam_stride] : 0.0;
  for (int jb = 2 * lane; jb < g.n; jb += 256) {  // n % 256 == 0
    double2 o[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = jb + 64 * u;
      if (j < B0) {
        o[u] = make_double2(0.0, 0.0);
      } else if (g.gam) {
        const uint32_t wd = (i < g.n_bits && j < g.n_bits) ? __ldg(brow + (j >> 5)) : 0u;
        o[u].x = ((wd >> (j & 31)) & 1u) && j < g.n_bits ? ng : 0.0;
        o[u].y = ((wd >> ((j + 1) & 31)) & 1u) && j + 1 < g.n_bits ? ng : 0.0;
        if (j == i) o[u].x = 1.0;
        if (j + 1 == i) o[u].y = 1.0;
      } else {
        o[u] = ldg2(Ai + j);
      }
    }
    for (int e = 0; e < cnt; ++e) {
      const int k = __shfl_sync(0xffffffffu, kl, e);
      const double mk = -__shfl_sync(0xffffffffu, vl, e);
      const double2* pr = reinterpret_cast<const double2*>(A + (int64_t)k * g.lda + jb);
      double2 pk[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) pk[u] = __ldg(pr + 32 * u);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        o[u].x = fma(mk, pk[u].x, o[u].x);
        o[u].y = fma(mk, pk[u].y, o[u].y);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) stg2(Ai + jb + 64 * u, o[u]);
  }
}

template <int B0>
static void launch_s0_gather(const S0Args& g, int64_t pcnt, cudaStream_t st) {
  dw_s0_gather_kernel<B0><<<dim3((unsigned)(2 * ((g.n - B0 + 255) / 256)), (unsigned)pcnt), 256, 0, st>>>(g);
  dw_s0_split_kernel<<<1, 1024, 0, st>>>(g);
}

// (dynamic shared memory above 48 KB: opted in once per device)
template <int B0>
static void s0_attrs() {
  static DeviceFlags attrs;
  const int dev = current_device();
  if (attrs.get(dev)) return;
  cudaFuncSetAttribute(dw_s0_row_kernel<B0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S0Row<B0>::SMEM);
  attrs.set(dev);
}

template <int B0>
static void launch_s0_row(const S0Args& g, int64_t pcnt, cudaStream_t st) {
  s0_attrs<B0>();
  dw_s0_row_kernel<B0><<<dim3(B0 / 16, (unsigned)pcnt), S0Row<B0>::THREADS, S0Row<B0>::SMEM, st>>>(g);
}

template <int B0>
static void launch_s0_update(const S0Args& g, int r0, int r1, int64_t pcnt, cudaStream_t st) {
  if (r1 > r0) dw_s0_update_kernel<B0><<<dim3((unsigned)((r1 - r0) / 8), (unsigned)pcnt), 256, 0, st>>>(g, r0, r1);
}

static bool dw_helper();

// The DW steps for one part (its matrices a + l * pstride, l < pcnt).
static int dw_part(double* a, int64_t n, int64_t lda, int64_t pstride, int64_t pcnt, const DwPart& d,
                   rdb_pivot_info* info, int64_t info_stride, const int* flags, int* dyn, cudaStream_t st,
                   cudaStream_t side = nullptr, cudaEvent_t ev_fork = nullptr, cudaEvent_t ev_join = nullptr,
                   int* side_dyn = nullptr, const S0Args* s0 = nullptr, cudaEvent_t s0_ready = nullptr,
                   int first_rec = 1, int64_t idx_off = 0) {
  const int nt = (int)(n / NB);
  if (cudaMemsetAsync(d.colcnt, 0, sizeof(int) * (size_t)pcnt * nt, st) != cudaSuccess ||
      cudaMemsetAsync(d.rowcnt, 0, sizeof(int) * (size_t)pcnt * nt, st) != cudaSuccess)
    return RDB_ECUDA;
  static DeviceFlags attrs;
  const int attrs_dev = current_device();
  if (!attrs.get(attrs_dev)) {
    if (cudaFuncSetAttribute(gj_wb_row_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)EC::SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(gj_wb_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)EC::SMEM_BYTES) != cudaSuccess)
      return RDB_ECUDA;
    attrs.set(attrs_dev);
  }
  CUtensorMap amap, cmap;
  int rc = make_a_map(&amap, a, n, n, lda, pstride, pcnt);
  if (rc) return rc;
  rc = make_ec_map(&cmap, a, n, n, lda, pstride, pcnt);
  if (rc) return rc;
  PlanPart np;
  np.pat = nullptr;
  np.pat_stride = 0;
  np.offs = nullptr;
  np.counts = d.ncounts;
  np.rp = d.nrp;
  np.up = d.nup;
  np.prebuilt = true;
  // Look-ahead: the next band's 2 x 2 diagonal tiles are updated first; its
  // 256-block inverse then runs on the part's side stream (own ticket
  // counters) while the rest of the update runs here. No tile of the rest
  // reads or writes that block.
  // sparse first step: the edge lists are gathered (and the list split) on the
  // side stream while the first band inverse runs here (already enqueued by
  // the caller when s0_ready is given)
  if (s0 && !s0_ready) {
    cudaStream_t gs = side ? side : st;
    if (side) {
      cudaEventRecord(ev_fork, st);
      cudaStreamWaitEvent(side, ev_fork, 0);
    }
    launch_s0_gather<2 * NB>(*s0, pcnt, gs);
    if (side) cudaEventRecord(ev_join, side);
  }
#ifndef RDB_EXP_NO_NESTED
  rc = invert_core(a, 2 * NB, lda, pstride, pcnt, d.ncnt, info, st, first_rec, idx_off, dyn, &np, info_stride, flags,
                   0, 2);
  if (rc) return rc;
#endif
  if (s0 && (side || s0_ready)) cudaStreamWaitEvent(st, s0_ready ? s0_ready : ev_join, 0);
  for (int p = 0; p < nt / 2; ++p) {
    const int p0t = 2 * p;
    const bool ahead = side && p + 1 < nt / 2;
    // step 0 of the sparse-first-step matrices: their own kernels; the dense
    // tiles of step 0 take the other listed matrices (list_d, count[2])
    const bool sp = s0 && p == 0;
    const int* list = sp ? d.list_d : d.list;
    const int* list_count = sp ? d.count + 2 : d.count;
    if (sp) launch_s0_row<2 * NB>(*s0, pcnt, st);
    WBRowSched rs{a, lda, pstride, nt, p0t, p, list, list_count, d.colcnt, dyn};
#ifndef RDB_EXP_NO_WBROW  // timing experiments only (wrong results)
    gj_wb_row_kernel<<<persistent_grid(pcnt * (nt - 2) * 2), EC::THREADS, EC::SMEM_BYTES, st>>>(amap, cmap, rs);
#endif
    // sparse step 0, rows of the next band first (its inverse can then start)
    if (sp) launch_s0_update<2 * NB>(*s0, 2 * NB, 4 * NB, pcnt, st);
    if (sp && !ahead) launch_s0_update<2 * NB>(*s0, 4 * NB, (int)n, pcnt, st);
    WBUpdateSched us{a, lda, pstride, nt, p0t, p, list, list_count, d.rowcnt, dyn ? dyn + 1 : nullptr};
    if (ahead) {
      us.part = 1;
      gj_wb_update_kernel<<<persistent_grid(pcnt * 4), EC::THREADS, EC::SMEM_BYTES, st>>>(amap, cmap, us);
      cudaEventRecord(ev_fork, st);
      cudaStreamWaitEvent(side, ev_fork, 0);
      const int64_t q0 = (int64_t)(p0t + 2) * NB;
#ifndef RDB_EXP_NO_NESTED  // timing experiments only (wrong results)
      rc = invert_core(a + q0 * lda + q0, 2 * NB, lda, pstride, pcnt, d.ncnt, info, side, 0, idx_off + q0, side_dyn,
                       &np, info_stride, flags, 0, 2);
      if (rc) return rc;
#endif
      cudaEventRecord(ev_join, side);
      us.part = 2;
      if (sp && n > 4 * NB)  // the other rows of the sparse step, beside the next band's inverse
        launch_s0_update<2 * NB>(*s0, 4 * NB, (int)n, pcnt, st);
    }
    const unsigned full = persistent_grid(pcnt * (nt - 2) * nt);
    unsigned ugrid = full, helper = 0;
    if (ahead) {
      // leave SMs to the side stream's band inverse (P1 needs one CTA per
      // matrix): the rest of the update on sm_count - 64 CTAs (RDB_GJ_DW_LA_RESERVE
      // overrides). Config 2 K2: 9.32 ms with no reserve, 9.09 ms with 48-80
      // (plateau), 10.7 ms with 100 (profiles/r02_dw_la_reserve.json). Once
      // the band inverse is done, a helper launch on the side stream takes
      // the reserved SMs back: it draws tickets from the same counter, so the
      // rest of the update runs on every SM (the SM timeline showed the
      // reserve idle for ~0.9 ms of the last look-ahead step otherwise,
      // profiles/r02_sm_timeline_k2.json).
      const char* e = getenv("RDB_GJ_DW_LA_RESERVE");
      const int res = e ? atoi(e) : (sm_count() * 7) / 16;
      // (never below 8 CTAs: a launch must be able to hold a whole dependency group, dmma_engine.cuh)
      const int keep = sm_count() - res > 8 ? sm_count() - res : 8;
      if (res > 0 && (int)ugrid > keep) ugrid = (unsigned)keep;
      if (dyn && dw_helper() && full > ugrid) helper = full - ugrid;
      if (helper) us.dyn_ctas = (int)(ugrid + helper);
    }
    gj_wb_update_kernel<<<ugrid, EC::THREADS, EC::SMEM_BYTES, st>>>(amap, cmap, us);
    if (ahead) {
      if (helper) {
        gj_wb_update_kernel<<<helper, EC::THREADS, EC::SMEM_BYTES, side>>>(amap, cmap, us);
        cudaEventRecord(ev_join, side);
      }
      cudaStreamWaitEvent(st, ev_join, 0);
    } else if (p + 1 < nt / 2) {
      const int64_t q0 = (int64_t)(p0t + 2) * NB;
      rc = invert_core(a + q0 * lda + q0, 2 * NB, lda, pstride, pcnt, d.ncnt, info, st, 0, idx_off + q0, dyn, &np,
                       info_stride, flags, 0, 2);
      if (rc) return rc;
    }
  }
  RDB_LAUNCH_CHECK();
  return RDB_OK;
}

// The two-level DW steps for one part (n = 2 W): D0 = the leading W x W
// block's inverse (dw_part on it, with its own sparse first step), the outer
// step 0 (sparse for the matrices listed in s_out, dense tiles for the
// others), D1 = the trailing block's inverse (dw_part, dense), the outer
// step 1 (dense). The gathers of both levels are queued by the caller before
// s0_ready (or here, inline, when it is null). Against the one-level steps
// this replaces the dense 256-wide steps 1..3 of an n = 1024 matrix (3/4 of
// its flop) by one 512-wide step plus two 512 x 512 inversions (62% of it).
static int dw2_part(double* a, int64_t n, int64_t lda, int64_t pstride, int64_t pcnt, const DwPart& d,
                    const DwPart& din, rdb_pivot_info* info, int64_t info_stride, const int* flags, int* dyn,
                    cudaStream_t st, cudaStream_t side, cudaEvent_t ev_fork, cudaEvent_t ev_join, int* side_dyn,
                    const S0Args* s_in, const S0Args* s_out, cudaEvent_t s0_ready) {
  const int64_t W = n / 2;
  const int nt = (int)(n / NB), bt = (int)(W / NB);
  static DeviceFlags attrs;
  const int attrs_dev = current_device();
  if (!attrs.get(attrs_dev)) {
    if (cudaFuncSetAttribute(gj_w2_row_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)EC::SMEM_BYTES) !=
            cudaSuccess ||
        cudaFuncSetAttribute(gj_w2_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)EC::SMEM_BYTES) != cudaSuccess)
      return RDB_ECUDA;
    attrs.set(attrs_dev);
  }
  CUtensorMap amap, cmap;
  int rc = make_a_map(&amap, a, n, n, lda, pstride, pcnt);
  if (rc) return rc;
  rc = make_ec_map(&cmap, a, n, n, lda, pstride, pcnt);
  if (rc) return rc;
  if ((s_in || s_out) && !s0_ready) {  // gathers inline, ahead of everything else here
    if (s_in) launch_s0_gather<2 * NB>(*s_in, pcnt, st);
    if (s_out) launch_s0_gather<4 * NB>(*s_out, pcnt, st);
    cudaEventRecord(ev_join, st);
    s0_ready = ev_join;
  }
  // A: D0 = A_00^-1 (W x W)
  rc = dw_part(a, W, lda, pstride, pcnt, din, info, info_stride, flags, dyn, st, side, ev_fork, ev_join, side_dyn,
               s_in, s_in ? s0_ready : nullptr, 1, 0);
  if (rc) return rc;
  if (s_out && s0_ready) cudaStreamWaitEvent(st, s0_ready, 0);
  // B: outer step 0 (band 0)
  auto outer_step = [&](int b0t, const int* list, const int* list_count) {
    if (cudaMemsetAsync(d.colcnt, 0, sizeof(int) * (size_t)pcnt * nt, st) != cudaSuccess ||
        cudaMemsetAsync(d.rowcnt, 0, sizeof(int) * (size_t)pcnt * nt, st) != cudaSuccess)
      return RDB_ECUDA;
    W2RowSched rs{a, lda, pstride, nt, b0t, bt, list, list_count, d.colcnt, dyn};
    gj_w2_row_kernel<<<persistent_grid(pcnt * (nt - bt) * bt), EC::THREADS, EC::SMEM_BYTES, st>>>(amap, cmap, rs);
    if (b0t == 0 && s_out)  // the sparse outer step's rows (their own matrices) before the dense tiles
      launch_s0_update<4 * NB>(*s_out, (int)W, (int)n, pcnt, st);
    W2UpdateSched us{a, lda, pstride, nt, b0t, bt, list, list_count, d.rowcnt, dyn ? dyn + 1 : nullptr};
    gj_w2_update_kernel<<<persistent_grid(pcnt * (nt - bt) * nt), EC::THREADS, EC::SMEM_BYTES, st>>>(amap, cmap,
                                                                                                      us);
    return RDB_OK;
  };
  if (s_out) launch_s0_row<4 * NB>(*s_out, pcnt, st);
  rc = outer_step(0, s_out ? d.list_d : d.list, s_out ? d.count + 2 : d.count);
  if (rc) return rc;
  // C: D1 = (Schur complement)^-1, the trailing W x W block (dense); its
  // pivots continue the record of A (indices from W)
  DwPart dc = din;
  dc.list = d.list;
  dc.count = d.count;
  rc = dw_part(a + W * lda + W, W, lda, pstride, pcnt, dc, info, info_stride, flags, dyn, st, side, ev_fork, ev_join,
               side_dyn, nullptr, nullptr, 0, W);
  if (rc) return rc;
  // D: outer step 1 (band 1), every listed matrix
  rc = outer_step(bt, d.list, d.count);
  if (rc) return rc;
  RDB_LAUNCH_CHECK();
  return RDB_OK;
}

// Sub-batches of a large batch on their own streams (default two halves):
// each part's kernels fill the others' tails (the last partial round of every persistent launch, the
// second wave of the one-CTA-per-matrix panel inverses). Measured on config 2:
// 18.44 -> 18.03 ms for 256 graphs (tools/two_stream.py).

static size_t counter_bytes(int64_t n_pad, int64_t batch) {
  const size_t nt = (size_t)((n_pad + NB - 1) / NB);
  return ((size_t)batch * nt * sizeof(int) + 64 + 255) & ~(size_t)255;  // + 16-byte alignment of the parts
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// Batched workspace: row-block counters | dynamic tile counters (256 B) |
// block-sparse plan (batch > 1 and nt <= PLAN_MAX_NT): pattern, per-part
// counts, P2 lists, update lists | banded path: per-matrix flags, G/H/D blocks
// (gj_band.cu).
namespace band {
size_t ws_doubles(int64_t n_pad);
}
int band_detect(const uint32_t* bits, int64_t n, int64_t batch, int* nonband, cudaStream_t st);
int band_invert(double* a, int64_t n_pad, int64_t lda, int64_t stride, int64_t batch, const int* nonband,
                double* ws, rdb_pivot_info* info, cudaStream_t st);

struct BatchWs {
  size_t cnt, dyn, blk, counts, rp, up, offs, band, band_ws, dwl, dwc, dwnc, dwrp, dwup, dwcnt, dwcol, dwrow, dws0,
      dwls, dwld, dwls2, dwld2, total;
  BatchWs(int64_t n_pad, int64_t batch) {
    const size_t nt = (size_t)(n_pad / NB), b = (size_t)batch;
    cnt = 0;
    dyn = counter_bytes(n_pad, batch);
    blk = dyn + 256;  // dynamic tile counters (2 per sub-batch part)
    if (batch > 1 && nt <= (size_t)PLAN_MAX_NT && n_pad % NB == 0) {
      counts = blk + align256(b * 2 * nt * (size_t)pat_ld((int)nt));  // column + row strip masks
      rp = counts + align256((size_t)MAX_PARTS * 2 * nt * sizeof(int));
      up = rp + align256(b * nt * (nt - 1) * sizeof(int));
      offs = up + align256(b * nt * nt * (nt - 1) * sizeof(int2));
      band = offs + align256(b * 2 * nt * sizeof(int));
      band_ws = band + align256(b * sizeof(int));
      dwl = band_ws + align256(b * band::ws_doubles(n_pad) * sizeof(double));  // dense-wide path
      dwc = dwl + align256(b * sizeof(int));
      dwnc = dwc + align256((size_t)MAX_PARTS * 16 * sizeof(int));
      dwrp = dwnc + align256((size_t)MAX_PARTS * 16 * sizeof(int));
      dwup = dwrp + align256(2 * b * sizeof(int));
      dwcnt = dwup + align256(4 * b * sizeof(int2));
      dwcol = dwcnt + align256((2 * b + 4 * MAX_PARTS) * sizeof(int));
      dwrow = dwcol + align256(b * nt * sizeof(int));
      dws0 = dwrow + align256(b * nt * sizeof(int));  // sparse first step: bad flags, list_s, list_d
      dwls = dws0 + align256(b * sizeof(int));
      dwld = dwls + align256(b * sizeof(int));
      dwls2 = dwld + align256(b * sizeof(int));  // two-level path: the outer step's list_s, list_d
      dwld2 = dwls2 + align256(b * sizeof(int));
      total = dwld2 + align256(b * sizeof(int));
    } else {
      counts = rp = up = offs = band = band_ws = dwl = dwc = dwnc = dwrp = dwup = dwcnt = dwcol = dwrow = dws0 = dwls =
          dwld = dwls2 = dwld2 = total = blk;
    }
  }
  bool has_plan() const { return total > blk; }
  // the dense-wide state of part i of `parts` (matrices i, i + parts, ...; lo before it)
  DwPart dw_part(char* wb, int i, int64_t lo, int nt) const {
    DwPart d;
    d.list = reinterpret_cast<int*>(wb + dwl) + lo;
    d.count = reinterpret_cast<int*>(wb + dwc) + 16 * i;
    d.ncounts = reinterpret_cast<int*>(wb + dwnc) + 16 * i;
    d.nrp = reinterpret_cast<int*>(wb + dwrp) + 2 * lo;
    d.nup = reinterpret_cast<int2*>(wb + dwup) + 4 * lo;
    d.ncnt = reinterpret_cast<int*>(wb + dwcnt + ((2 * (size_t)lo * sizeof(int) + 15) & ~(size_t)15));
    d.colcnt = reinterpret_cast<int*>(wb + dwcol) + lo * nt;
    d.rowcnt = reinterpret_cast<int*>(wb + dwrow) + lo * nt;
    d.list_s = reinterpret_cast<int*>(wb + dwls) + lo;
    d.list_d = reinterpret_cast<int*>(wb + dwld) + lo;
    return d;
  }
  // two-level path: the outer level (its own sparse-step lists) and the inner
  // level (the W x W inversions: the one-level lists, counts at count + 4)
  DwPart dw2_outer(char* wb, int i, int64_t lo, int nt) const {
    DwPart d = dw_part(wb, i, lo, nt);
    d.list_s = reinterpret_cast<int*>(wb + dwls2) + lo;
    d.list_d = reinterpret_cast<int*>(wb + dwld2) + lo;
    return d;
  }
  DwPart dw2_inner(char* wb, int i, int64_t lo, int nt) const {
    DwPart d = dw_part(wb, i, lo, nt);
    d.count += 4;
    return d;
  }
};

// Two-level dense-wide steps for n = 1024 (A-B switch RDB_GJ_DW2=0).
static bool dw2_enabled() {
  const char* e = getenv("RDB_GJ_DW2");
  return !(e && e[0] == '0');
}

// Sparse first step of the dense-wide path (A-B switch RDB_GJ_DW_S0=0).
static bool dw_s0_enabled() {
  const char* e = getenv("RDB_GJ_DW_S0");
  return !(e && e[0] == '0');
}

// Dense-wide look-ahead of the next band inverse on a side stream (A-B switch RDB_GJ_DW_LA=0).
static bool dw_helper() {  // RDB_GJ_DW_HELPER=0: no helper launch (A/B)
  const char* e = getenv("RDB_GJ_DW_HELPER");
  return !(e && e[0] == '0');
}

static bool dw_lookahead() {
  const char* e = getenv("RDB_GJ_DW_LA");
  return !(e && e[0] == '0');
}

// Dense 256-wide steps for fully dense batched matrices (A-B switch RDB_GJ_DW=0).
static bool dw_enabled() {
  const char* e = getenv("RDB_GJ_DW");
  return !(e && e[0] == '0');
}

static bool skip_enabled() {
  const char* e = getenv("RDB_GJ_SKIP");  // A-B switch: 0 runs the dense schedule
  return !(e && e[0] == '0');
}

// Update tiles are taken by atomic ticket (a global counter per launch) by
// default: the forward-progress argument for the in-kernel waits then needs
// no co-residency of the whole grid (a tile's dependencies are taken by running
// CTAs in index order and the producer gates on open waits: dmma_engine.cuh,
// Tile::wait), whatever else shares the GPU. Measured equal to the static
// stride on config 2 (9.498 vs 9.497 ms per K2 call, profiles/r02_k2_modes.json).
// Block-tridiagonal matrices (every edge within the 32-block band, from the
// adjacency bits) skip Gauss-Jordan and run the banded inverse (gj_band.cu).
static bool band_enabled() {
  const char* e = getenv("RDB_GJ_BAND");  // A-B switch: 0 sends every matrix through Gauss-Jordan
  return !(e && e[0] == '0');
}

static bool dyn_sched() {
  const char* e = getenv("RDB_GJ_DYNAMIC");  // A-B switch: 0 takes tiles by static stride
  return !(e && e[0] == '0');
}

// Forward progress of the update kernel's in-kernel waits (the panel-column
// tile of a row block waits for that row's other tiles, which have smaller
// indices): with the static tile stride a waiting CTA needs every CTA of its
// own grid resident. When the sub-batches' update kernels run concurrently on
// their own streams, that holds if their grids together fit one CTA per SM
// (every other kernel in flight — panel inverses, row panels, the banded
// path — never waits, so it frees its SM): each part's update grid is capped
// at sm_count / parts when the static stride is selected (RDB_GJ_DYNAMIC=0);
// RDB_GJ_COSCHED=0 lifts that cap (A-B timing only). The default ticket order
// is sound without it.
static bool cosched_cap() {
  const char* e = getenv("RDB_GJ_COSCHED");
  return !(e && e[0] == '0');
}

static int split_min_batch() {
  const char* e = getenv("RDB_GJ_SPLIT_MIN");  // A-B switch; 0 disables the split
  const int v = e ? atoi(e) : 64;
  return v <= 0 ? 1 << 30 : v;
}

static int split_parts() {
  const char* e = getenv("RDB_GJ_SPLIT_PARTS");  // tuning: sub-batches on their own streams (2..4)
  const int v = e ? atoi(e) : 2;
  return v < 2 ? 2 : (v > MAX_PARTS ? MAX_PARTS : v);
}

// The internal streams and events (look-ahead side stream, sub-batch streams)
// are process-wide: host threads enqueueing inversions concurrently are
// serialised here (enqueue only; the calls stay asynchronous).
static std::mutex g_enqueue;

// Batched calls (batch > 1, n <= 64 NB) run the block-sparse plan: the
// pattern comes from the bit-packed adjacency when the caller has it (`bits`,
// n_bits vertices: the rdb_apsp_bits_batched pipelines), else from a scan of
// the matrices.
// The banded path's per-matrix flags in a batched workspace, or nullptr when
// invert_batched will not use the banded path for (n, batch). The APSP
// pipelines fill them before K1 (band_detect) and pass band_ready.
int* band_flags(void* work, int64_t n, int64_t batch) {
  const BatchWs ws(n, batch);
  if (!work || batch <= 1 || n % NB || !ws.has_plan() || !skip_enabled() || !band_enabled()) return nullptr;
  return reinterpret_cast<int*>(static_cast<char*>(work) + ws.band);
}

// phase (the APSP pipelines, M built from bits as I - gamma A): 1 = classify
// only, before K1 (patterns, dense-wide lists, sparse-first-step counts; the
// matrices whose first step is sparse are returned in *s0bad_out as
// s0bad[m] == 0 with flags[m] == 2, and K1 builds only their block M_00);
// 2 = the inversion after K1 (classification skipped); 0 = both, M given.
// m_gammas: the gains of M = I - gamma A (phases 1 and 2), else nullptr.
int invert_batched(double* a, int64_t n, int64_t lda, int64_t stride, int64_t batch, void* work,
                   rdb_pivot_info* info, cudaStream_t st, const uint32_t* bits = nullptr, int64_t n_bits = 0,
                   bool band_ready = false, int phase = 0, const double* m_gammas = nullptr,
                   int** s0bad_out = nullptr, int* s0_levels_out = nullptr) {
  std::lock_guard<std::mutex> guard(g_enqueue);
  if (s0bad_out) *s0bad_out = nullptr;
  if (batch == 1 && n >= wide_min_n() && n % (2 * NB) == 0 && a && work && info && lda >= n && !(lda & 1) &&
      !((uintptr_t)a & 15) && !((uintptr_t)work & 15))
    return phase == 1 ? RDB_OK : invert_wide(a, n, lda, work, info, st);
  const BatchWs ws(n, batch);
  char* const wb = static_cast<char*>(work);
  const bool use_plan = batch > 1 && ws.has_plan() && skip_enabled() && a && work && n % NB == 0 &&
                        batch <= (1 << 19) && stride >= n * lda;
  const int64_t ntl = n / NB;
  const int64_t pld = pat_ld((int)ntl);
  unsigned char* pat = use_plan ? reinterpret_cast<unsigned char*>(wb + ws.blk) : nullptr;
  const bool use_band = use_plan && bits && (band_ready || band_enabled()) && info && lda >= n;
  if (band_ready && !use_band) return RDB_EINVAL;  // K1 has skipped the off-band blocks: must not run GJ on them
  int* nonband = use_band ? reinterpret_cast<int*>(wb + ws.band) : nullptr;
  double* band_ws = use_band ? reinterpret_cast<double*>(wb + ws.band_ws) : nullptr;
  if (use_plan && phase != 2) {
    if (cudaMemsetAsync(pat, 0, (size_t)(batch * 2 * ntl * pld), st) != cudaSuccess) return RDB_ECUDA;
    if (use_band && !band_ready) {
      const int rc = band_detect(bits, n_bits, batch, nonband, st);
      if (rc) return rc;
    }
    if (bits) {
      const int64_t want = (batch * ((n_bits + 15) / 16) + 7) / 8;
      strip_pattern_bits_kernel<<<(unsigned)(want < 148 * 16 ? want : 148 * 16), 256, 0, st>>>(
          bits, n_bits, batch, (int)ntl, pat, nonband);
    } else {
      const int64_t want = (batch * ntl * ntl + 7) / 8;
      strip_pattern_m_kernel<<<(unsigned)(want < 148 * 16 ? want : 148 * 16), 256, 0, st>>>(
          a, lda, stride, batch, (int)ntl, pat);
    }
  }
  // part i of `parts` = matrices i, i + parts, i + 2 parts, ... (interleaved:
  // the parts get similar mixes of dense and block-sparse matrices whatever
  // the batch order); lo = matrices in the parts before it (workspace slices)
  auto part_plan = [&](int i, int parts_, int64_t lo) {
    PlanPart pp;
    pp.pat = pat + i * 2 * ntl * pld;
    pp.pat_stride = parts_ * 2 * ntl * pld;
    pp.counts = reinterpret_cast<int*>(wb + ws.counts) + 2 * ntl * i;
    pp.rp = reinterpret_cast<int*>(wb + ws.rp) + lo * ntl * (ntl - 1);
    pp.up = reinterpret_cast<int2*>(wb + ws.up) + lo * ntl * ntl * (ntl - 1);
    pp.offs = reinterpret_cast<int*>(wb + ws.offs) + lo * 2 * ntl;
    return pp;
  };
  const int parts = split_parts();
  const bool split =
      batch >= split_min_batch() && batch >= 4 * parts && a && work && info && n % NB == 0 && stride >= n * lda;
  // dense-wide path: classify (flags 1 -> 2, patterns zeroed, per-part lists) before the fork
  const bool use_dw = use_band && dw_enabled() && ntl >= 4 && ntl % 2 == 0 && batch >= 2 * (split ? parts : 1);
  DwPart dwp[MAX_PARTS];
  const bool use_s0 = use_dw && dw_s0_enabled();
  int* s0flags = use_s0 ? reinterpret_cast<int*>(wb + ws.dws0) : nullptr;
  const bool synth = use_s0 && m_gammas && bits;  // M = I - gamma A: the sparse step reads the bits, not M
  const int64_t lstride = (int64_t)(band::ws_doubles(n) * sizeof(double));  // lists in the banded scratch
  const int64_t wpr = (n_bits + 31) / 32;
  // two-level path (n = 1024): outer steps of width W = n / 2 = 512
  const bool use_dw2 = use_dw && n == 4 * 2 * NB && dw2_enabled();
  // the sparse first step of a problem (the leading pn x pn block; one-level:
  // the matrix, bit 1; two-level: inner = the leading W block, bit 1, outer =
  // the matrix, bit 2, lists past the inner ones in the matrix's slice)
  auto s0_args = [&](const DwPart& d, int i, int parts_, int64_t pn, int bit, const int* n_list) {
    S0Args g;
    g.a = a + i * stride;
    g.lda = lda;
    g.pstride = parts_ * stride;
    g.lists = wb + ws.band_ws + i * lstride + (bit == 2 ? (int64_t)256 * 1024 : 0);
    g.lstride = parts_ * lstride;
    g.n = (int)pn;
    g.list = d.list_s;
    g.count = d.count;
    g.colcnt = bit == 2 ? nullptr : d.colcnt;
    g.rowcnt = bit == 2 ? nullptr : d.rowcnt;
    g.bits = bits + (int64_t)i * n_bits * wpr;
    g.bstride = parts_ * n_bits * wpr;
    g.wpr = wpr;
    g.n_bits = n_bits < pn ? n_bits : pn;
    g.bad = s0flags + i;
    g.bad_stride = parts_;
    g.bad_bit = bit;
    g.n_list = n_list;
    g.dw_list = d.list;
    g.list_s = d.list_s;
    g.list_d = d.list_d;
    g.counts = d.count;
    g.gam = synth ? m_gammas + i : nullptr;
    g.gam_stride = parts_;
    return g;
  };
  if (use_dw && phase != 2) {
    if (use_s0 && cudaMemsetAsync(s0flags, 0, (size_t)batch * sizeof(int), st) != cudaSuccess) return RDB_ECUDA;
    DwClassifyArgs ca;
    ca.pat = pat;
    ca.flags = nonband;
    ca.batch = batch;
    ca.nt = (int)ntl;
    ca.parts = split ? parts : 1;
    int64_t lo = 0;
    for (int i = 0; i < ca.parts; ++i) {
      dwp[i] = ws.dw_part(wb, i, lo, (int)ntl);
      ca.part[i] = dwp[i];
      lo += (batch - i + ca.parts - 1) / ca.parts;
    }
    dw_classify_kernel<<<(unsigned)ca.parts, 1024, 0, st>>>(ca);
    if (synth && !use_dw2)  // counted now: K1 builds only M_00 of the matrices whose first step is sparse
      dw_s0_count_kernel<2 * NB><<<dim3((unsigned)(2 * ((n - 2 * NB + 255) / 256)), (unsigned)batch), 256, 0, st>>>(
          bits, n_bits, (int)n, nonband, s0flags, 1);
    if (synth && use_dw2) {  // both levels: the leading 512 block (bit 1) and the matrix (bit 2)
      dw_s0_count_kernel<2 * NB><<<dim3((unsigned)(2 * ((n / 2 - 2 * NB + 255) / 256)), (unsigned)batch), 256, 0,
                                   st>>>(bits, n_bits, (int)(n / 2), nonband, s0flags, 1);
      dw_s0_count_kernel<4 * NB><<<dim3((unsigned)(2 * ((n - 4 * NB + 255) / 256)), (unsigned)batch), 256, 0, st>>>(
          bits, n_bits, (int)n, nonband, s0flags, 2);
    }
  } else if (use_dw) {
    int64_t lo = 0;
    for (int i = 0; i < (split ? parts : 1); ++i) {
      dwp[i] = ws.dw_part(wb, i, lo, (int)ntl);
      lo += (batch - i + (split ? parts : 1) - 1) / (split ? parts : 1);
    }
    if (use_s0 && !synth && cudaMemsetAsync(s0flags, 0, (size_t)batch * sizeof(int), st) != cudaSuccess)
      return RDB_ECUDA;
  }
  if (phase == 1) {
    if (s0bad_out && synth) *s0bad_out = s0flags;
    if (s0_levels_out) *s0_levels_out = use_dw2 ? 2 : 1;
    RDB_LAUNCH_CHECK();
    return RDB_OK;
  }
  if (split) {
    DevStreams* ds = dev_streams();
    if (!ds) return RDB_ECUDA;
    int* dyn = reinterpret_cast<int*>(wb + ws.dyn);
    if (cudaMemsetAsync(dyn, 0, 4 * MAX_PARTS * sizeof(int), st) != cudaSuccess) return RDB_ECUDA;
    cudaEventRecord(ds->fork, st);
    // the banded matrices on this stream, concurrently with the sub-batches
    int rc = use_band ? band_invert(a, n, lda, stride, batch, nonband, band_ws, info, st) : RDB_OK;
    int64_t lo = 0;
    for (int i = 0; i < parts && rc == RDB_OK; ++i) {
      const int64_t cnt = (batch - i + parts - 1) / parts;
      cudaStreamWaitEvent(ds->part[i], ds->fork, 0);
      const PlanPart pp = part_plan(i, parts, lo);
      // row-block counters of the part, 16-byte aligned (counter_bytes has the slack)
      char* cw = wb + (((size_t)lo * ntl * sizeof(int) + 15) & ~(size_t)15);
      const bool dyn_on = dyn_sched();
      // With the dense-wide path the part's block-sparse plan (its other
      // matrices; for config 2 an empty schedule) runs on the part's side
      // stream, concurrently with the dense-wide steps (disjoint matrices, own
      // ticket counters), ahead of the look-ahead work queued there later.
      const bool plan_aside = use_dw && dw_lookahead();
      cudaStream_t plan_st = plan_aside ? ds->dw_side[i] : ds->part[i];
      if (plan_aside) {
        cudaEventRecord(ds->dw_fork[i], ds->part[i]);
        cudaStreamWaitEvent(plan_st, ds->dw_fork[i], 0);
      }
      // sparse first step: gather the part's edge lists on the side stream
      // first (ahead of the plan), beside the part's first band inverse
      const DwPart d2o = use_dw2 ? ws.dw2_outer(wb, i, lo, (int)ntl) : DwPart{};
      const DwPart d2i = use_dw2 ? ws.dw2_inner(wb, i, lo, (int)ntl) : DwPart{};
      const S0Args g0 = !use_s0 ? S0Args{}
                        : use_dw2 ? s0_args(d2i, i, parts, n / 2, 1, dwp[i].count)
                                  : s0_args(dwp[i], i, parts, n, 1, dwp[i].count);
      const S0Args g2 = use_s0 && use_dw2 ? s0_args(d2o, i, parts, n, 2, dwp[i].count) : S0Args{};
      const bool s0_aside = use_s0 && plan_aside;
      if (s0_aside) {
        launch_s0_gather<2 * NB>(g0, cnt, plan_st);
        if (use_dw2) launch_s0_gather<4 * NB>(g2, cnt, plan_st);
        cudaEventRecord(ds->s0_ready[i], plan_st);
      }
      rc = invert_core(a + i * stride, n, lda, parts * stride, cnt, cw, info + i, plan_st, 1, 0,
                       dyn_on ? (plan_aside ? dyn + 2 * MAX_PARTS + 2 * i : dyn + 2 * i) : nullptr,
                       use_plan ? &pp : nullptr, parts, nonband ? nonband + i : nullptr,
                       (!dyn_on && cosched_cap()) ? sm_count() / parts : 0);
      if (rc) break;
      if (use_dw2) {
        rc = dw2_part(a + i * stride, n, lda, parts * stride, cnt, d2o, d2i, info + i, parts, nonband + i,
                      dyn_on ? dyn + 2 * i : nullptr, ds->part[i], dw_lookahead() ? ds->dw_side[i] : nullptr,
                      ds->dw_fork[i], ds->dw_join[i], dyn_on ? dyn + 2 * MAX_PARTS + 2 * i : nullptr,
                      use_s0 ? &g0 : nullptr, use_s0 ? &g2 : nullptr, s0_aside ? ds->s0_ready[i] : nullptr);
        if (rc) break;
      } else if (use_dw) {
        rc = dw_part(a + i * stride, n, lda, parts * stride, cnt, dwp[i], info + i, parts, nonband + i,
                     dyn_on ? dyn + 2 * i : nullptr, ds->part[i], dw_lookahead() ? ds->dw_side[i] : nullptr,
                     ds->dw_fork[i], ds->dw_join[i], dyn_on ? dyn + 2 * MAX_PARTS + 2 * i : nullptr,
                     use_s0 ? &g0 : nullptr, s0_aside ? ds->s0_ready[i] : nullptr);
        if (rc) break;
      }
      if (plan_aside) {  // the side stream's last work (plan, then look-ahead) joins the part
        cudaEventRecord(ds->dw_join[i], plan_st);
        cudaStreamWaitEvent(ds->part[i], ds->dw_join[i], 0);
      }
      cudaEventRecord(ds->join[i], ds->part[i]);
      lo += cnt;
    }
    for (int i = 0; i < parts; ++i) cudaStreamWaitEvent(st, ds->join[i], 0);
    return rc;
  }
  const PlanPart pp = part_plan(0, 1, 0);
  if (use_band) {
    const int rc = band_invert(a, n, lda, stride, batch, nonband, band_ws, info, st);
    if (rc) return rc;
  }
  if (!a || !work || !info || n <= 0 || n % NB != 0 || lda < n || batch <= 0 || ((uintptr_t)work & 15))
    return RDB_EINVAL;  // (validated before the first CUDA call)
  int* dyn = nullptr;
  if (dyn_sched()) {
    dyn = reinterpret_cast<int*>(wb + ws.dyn);
    if (cudaMemsetAsync(dyn, 0, 4 * MAX_PARTS * sizeof(int), st) != cudaSuccess) return RDB_ECUDA;
  }
  if (use_dw2) {
    // (the events order the inline gathers too: needed with or without the look-ahead's side stream)
    DevStreams* ds = dev_streams();
    if (!ds) return RDB_ECUDA;
    const DwPart d2o = ws.dw2_outer(wb, 0, 0, (int)ntl), d2i = ws.dw2_inner(wb, 0, 0, (int)ntl);
    const S0Args g0 = use_s0 ? s0_args(d2i, 0, 1, n / 2, 1, dwp[0].count) : S0Args{};
    const S0Args g2 = use_s0 ? s0_args(d2o, 0, 1, n, 2, dwp[0].count) : S0Args{};
    const int rc = dw2_part(a, n, lda, stride, batch, d2o, d2i, info, 1, nonband, dyn, st,
                            dw_lookahead() ? ds->dw_side[0] : nullptr, ds->dw_fork[0], ds->dw_join[0],
                            dyn ? dyn + 2 * MAX_PARTS : nullptr,
                            use_s0 ? &g0 : nullptr, use_s0 ? &g2 : nullptr, nullptr);
    if (rc) return rc;
  } else if (use_dw) {
    DevStreams* ds = dw_lookahead() ? dev_streams() : nullptr;
    const S0Args g0 = use_s0 ? s0_args(dwp[0], 0, 1, n, 1, dwp[0].count) : S0Args{};
    const int rc = dw_part(a, n, lda, stride, batch, dwp[0], info, 1, nonband, dyn, st, ds ? ds->dw_side[0] : nullptr,
                           ds ? ds->dw_fork[0] : nullptr, ds ? ds->dw_join[0] : nullptr,
                           dyn ? dyn + 2 * MAX_PARTS : nullptr, use_s0 ? &g0 : nullptr);
    if (rc) return rc;
  }
  return invert_core(a, n, lda, stride, batch, work, info, st, 1, 0, dyn, use_plan ? &pp : nullptr, 1,
                     nonband);
}

// ------------------------------------------------------------------ wide (NB = 256) single matrix
// One large matrix (configs 3 and 5; n >= 8192 by default) in 256-wide steps: every rank-256 update
// tile runs 16 k-chunks per epilogue instead of 8, halving the engine's
// per-tile cost per flop (tools/tile_overhead.py: 32.0 -> 34.1 TFLOP/s). Step p
// (band = rows/cols p0 .. p0+255):
//   1. D = A_pp^-1 in place: the NB = 128 Gauss-Jordan on the 256 x 256 block;
//   2. R = D A_pJ (J outside the band) into a 256 x n scratch;
//   3. A_IJ += -(A_Ip R_J) (I, J outside the band, reduce-add) and
//      C_I = -(A_Ip D) into an n x 256 scratch (I outside the band), in one
//      launch with two output maps;
//   4. the scratches are copied into the band rows / columns.
// The scratches remove every in-kernel dependency (no tile overwrites another
// tile's operand). Same algebra as the NB = 128 path, different rounding
// order: the inverse agrees to ~1e-15 relative, D is unchanged (tests).
constexpr int WB = 2 * NB;

struct WideRowSched {  // R[r][J] = D[r rows] * A_pJ, r in {0, 1}, J outside the band
  const double* a;
  int64_t lda;
  int nt, p0t;  // tiles of 128; band = tiles p0t, p0t + 1
  RDB_DEV int count() const { return 2 * (nt - 2); }
  RDB_DEV eng::Tile tile(int t) const {
    const int r = t / (nt - 2);
    int J = t - r * (nt - 2);
    J += (J >= p0t) ? 2 : 0;
    eng::Tile T;
    T.a_col = p0t * NB;
    T.a_row = (p0t + r) * NB;
    T.a_mat = 0;
    T.b = a + (int64_t)p0t * NB * lda + (int64_t)J * NB;
    T.ldb = lda;
    T.c_col = J * NB;
    T.c_row = r * NB;
    T.c_mat = 0;
    T.nk = WB / eng::BK;
    T.mode = eng::EPI_STORE;
    T.neg = 0;
    T.signal = nullptr;
    T.wait = nullptr;
    T.wait_target = 0;
    return T;
  }
};

struct WideUpdateSched {  // rows I outside the band; J outside -> reduce into A, J in band -> column scratch
  const double* a;
  const double* rows;  // the 256 x n row scratch R
  int64_t lda, ldr;
  int nt, p0t;
  // part 0: every tile; 1: only the next band's 2 x 2 diagonal tiles (look-ahead:
  // the next 256-block inverse can start); 2: every tile except those
  int part;
  RDB_DEV int count() const { return part == 1 ? 4 : (nt - 2) * nt - (part == 2 ? 4 : 0); }
  // (ri, jj): ri-th row tile outside the band, jj-th column in the order
  // [nt - 2 reduce columns outside the band, then the 2 band columns]
  RDB_DEV eng::Tile make(int ri, int jj) const {
    const int I = ri + ((ri >= p0t) ? 2 : 0);
    eng::Tile T;
    T.a_col = p0t * NB;  // A operand: A_Ip, 128 x 256
    T.a_row = I * NB;
    T.a_mat = 0;
    T.c_row = I * NB;
    T.c_mat = 0;
    T.nk = WB / eng::BK;
    T.neg = 1;
    T.signal = nullptr;
    T.wait = nullptr;
    T.wait_target = 0;
    if (jj < nt - 2) {
      const int J = jj + ((jj >= p0t) ? 2 : 0);
      T.b = rows + (int64_t)J * NB;
      T.ldb = ldr;
      T.c_col = J * NB;
      T.mode = eng::EPI_REDUCE;
    } else {
      const int h = jj - (nt - 2);
      T.b = a + (int64_t)p0t * NB * lda + (int64_t)(p0t + h) * NB;  // D columns
      T.ldb = lda;
      T.c_col = h * NB;
      T.c_sel = 1;
      T.mode = eng::EPI_STORE;
    }
    return T;
  }
  RDB_DEV eng::Tile tile(int t) const {
    // the next band (tiles p0t + 2, p0t + 3) is row / column index p0t, p0t + 1 here
    if (part == 1) return make(p0t + (t >> 1), p0t + (t & 1));
    if (part == 0) return make(t / nt, t - (t / nt) * nt);
    const int head = p0t * nt;  // rows before the next band: all columns
    if (t < head) return make(t / nt, t - (t / nt) * nt);
    t -= head;
    if (t < 2 * (nt - 2)) {  // the next band's two rows, its two columns skipped
      const int r = t / (nt - 2), jr = t - r * (nt - 2);
      return make(p0t + r, jr < p0t ? jr : jr + 2);
    }
    t -= 2 * (nt - 2);
    return make(p0t + 2 + t / nt, t - (t / nt) * nt);
  }
};

__global__ void __launch_bounds__(EC::THREADS, 1)
    gj_wide_row_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap rmap,
                       WideRowSched sched) {
  RDB_TRACE_SCOPE(8);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  eng::run<EC>(smem_raw, &amap, sched, eng::BulkEpilogue<EC>{&rmap});
}

__global__ void __launch_bounds__(EC::THREADS, 1)
    gj_wide_update_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap cmap,
                          const __grid_constant__ CUtensorMap smap, WideUpdateSched sched) {
  RDB_TRACE_SCOPE(9);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  eng::run<EC>(smem_raw, &amap, sched, eng::BulkEpilogue<EC>{&cmap, &smap});
}

static int64_t wide_min_n() {
  const char* e = getenv("RDB_GJ_WIDE_MIN");  // tuning / A-B switch (read per call); 0 disables the wide path
  const int64_t v = e ? atoll(e) : 8192;  // measured (tools/wide_check.py): +8% at 8192, +5.6% at 16384, +6.9% at 32768, even at 4096
  return v == 0 ? INT64_MAX : v;
}

static bool wide_lookahead() {
  const char* e = getenv("RDB_GJ_WIDE_LA");  // debugging switch: 0 runs the wide steps without look-ahead
  return !(e && e[0] == '0');
}

static size_t wide_scratch_bytes(int64_t n) { return (size_t)2 * WB * n * sizeof(double); }

static int invert_wide(double* a, int64_t n, int64_t lda, void* work, rdb_pivot_info* info, cudaStream_t st) {
  int rc = setup();
  if (rc) return rc;
  static DeviceFlags attrs;
  const int attrs_dev = current_device();
  if (!attrs.get(attrs_dev)) {
    if (cudaFuncSetAttribute(gj_wide_row_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)EC::SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(gj_wide_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)EC::SMEM_BYTES) != cudaSuccess)
      return RDB_ECUDA;
    attrs.set(attrs_dev);
  }
  const int nt = (int)(n / NB);
  // workspace: [counters of the nested 256-block inverse | R (256 x n) | C (n x 256)]
  char* base = static_cast<char*>(work);
  int* cnt = reinterpret_cast<int*>(base);
  double* R = reinterpret_cast<double*>(base + 256);
  double* Cs = R + (int64_t)WB * n;
  CUtensorMap amap, cmap, rmap, smap;
  if ((rc = make_a_map(&amap, a, n, n, lda, n * lda, 1)) || (rc = make_ec_map(&cmap, a, n, n, lda, n * lda, 1)) ||
      (rc = make_ec_map(&rmap, R, WB, n, n, (int64_t)WB * n, 1)) ||
      (rc = make_ec_map(&smap, Cs, n, WB, WB, (int64_t)WB * n, 1)))
    return rc;
  DevStreams* ds = dev_streams();
  if (!ds) return RDB_ECUDA;
  cudaStream_t side = ds->side;
  // 1. (step 0) D = A_00^-1: the NB = 128 Gauss-Jordan on the 256 x 256 block
  rc = invert_core(a, WB, lda, 0, 1, cnt, info, st, 1, 0);
  if (rc) return rc;
  for (int p = 0; p < nt / 2; ++p) {
    const int p0t = 2 * p;
    const int64_t p0 = (int64_t)p0t * NB;
    const bool ahead = p + 1 < nt / 2 && wide_lookahead();
    // 2. R = D A_pJ
    WideRowSched rs{a, lda, nt, p0t};
    gj_wide_row_kernel<<<persistent_grid(2 * (nt - 2)), EC::THREADS, EC::SMEM_BYTES, st>>>(amap, rmap, rs);
    // 3. trailing update + new column panel. Look-ahead: the next band's
    // diagonal block is updated first and inverted (1.) on a side stream, one
    // SM, while the rest of the update runs on the other SMs
    if (ahead) {
      cudaEventRecord(ds->ev_a, st);
      cudaStreamWaitEvent(side, ds->ev_a, 0);
      WideUpdateSched u1{a, R, lda, n, nt, p0t, 1};
      gj_wide_update_kernel<<<1, EC::THREADS, EC::SMEM_BYTES, side>>>(amap, cmap, smap, u1);
      cudaEventRecord(ds->ev_b, side);  // u1 has read the old column panel (the copy-back below overwrites it)
      const int64_t q0 = p0 + WB;
      rc = invert_core(a + q0 * lda + q0, WB, lda, 0, 1, cnt, info, side, 0, q0);
      if (rc) return rc;
      cudaEventRecord(ds->ev_p, side);
      WideUpdateSched u2{a, R, lda, n, nt, p0t, 2};
      const int64_t tiles = (int64_t)(nt - 2) * nt - 4;
      const unsigned grid = (unsigned)(tiles < sm_count() - 1 ? tiles : sm_count() - 1);
      gj_wide_update_kernel<<<grid, EC::THREADS, EC::SMEM_BYTES, st>>>(amap, cmap, smap, u2);
    } else {
      WideUpdateSched us{a, R, lda, n, nt, p0t, 0};
      gj_wide_update_kernel<<<persistent_grid((int64_t)(nt - 2) * nt), EC::THREADS, EC::SMEM_BYTES, st>>>(
          amap, cmap, smap, us);
    }
    // 4. scratches -> band rows (R, columns outside the band) and band columns (C, rows outside)
    if (ahead) cudaStreamWaitEvent(st, ds->ev_b, 0);
    const int64_t right = n - p0 - WB;
    if (p0 > 0 &&
        (cudaMemcpy2DAsync(a + p0 * lda, lda * 8, R, n * 8, p0 * 8, WB, cudaMemcpyDeviceToDevice, st) ||
         cudaMemcpy2DAsync(a + p0, lda * 8, Cs, WB * 8, WB * 8, p0, cudaMemcpyDeviceToDevice, st)))
      return RDB_ECUDA;
    if (right > 0 &&
        (cudaMemcpy2DAsync(a + p0 * lda + p0 + WB, lda * 8, R + p0 + WB, n * 8, right * 8, WB,
                           cudaMemcpyDeviceToDevice, st) ||
         cudaMemcpy2DAsync(a + (p0 + WB) * lda + p0, lda * 8, Cs + (p0 + WB) * WB, WB * 8, WB * 8, right,
                           cudaMemcpyDeviceToDevice, st)))
      return RDB_ECUDA;
    if (ahead) {
      cudaStreamWaitEvent(st, ds->ev_p, 0);
    } else if (p + 1 < nt / 2) {  // no look-ahead: the next 256-block inverse here
      const int64_t q0 = p0 + WB;
      rc = invert_core(a + q0 * lda + q0, WB, lda, 0, 1, cnt, info, st, 0, q0);
      if (rc) return rc;
    }
  }
  RDB_LAUNCH_CHECK();
  return RDB_OK;
}

// ------------------------------------------------------------------ local GEMM (distributed GJ)
// C (m x n tiles of 128) op= sign * A (m x K) * B (K x n) for a rank's local
// tiles of the 2D block-cyclic inversion: A = the received column panel, B =
// the received row panel (or D and the local row block for the row-panel
// product). Row tile skip_row and column tile skip_col are left out; column
// tile store_col is stored instead of accumulated.
struct LocalSched {
  const double* b;
  int64_t ldb;
  int mt, nt, nk, skip_row, skip_col, store_col, mode, neg;
  RDB_DEV int rows() const { return mt - (skip_row >= 0 ? 1 : 0); }
  RDB_DEV int cols() const { return nt - (skip_col >= 0 ? 1 : 0); }
  RDB_DEV int count() const { return rows() * cols(); }
  RDB_DEV eng::Tile tile(int t) const {
    const int nc = cols();
    int I = t / nc, J = t - (t / nc) * nc;
    if (skip_row >= 0 && I >= skip_row) ++I;
    if (skip_col >= 0 && J >= skip_col) ++J;
    eng::Tile T;
    T.a_col = 0;
    T.a_row = I * NB;
    T.a_mat = 0;
    T.b = b + (int64_t)J * NB;
    T.ldb = ldb;
    T.c_col = J * NB;
    T.c_row = I * NB;
    T.c_mat = 0;
    T.nk = nk;
    T.mode = (J == store_col) ? eng::EPI_STORE : mode;
    T.neg = neg;
    T.signal = nullptr;
    T.wait = nullptr;
    T.wait_target = 0;
    return T;
  }
};

__global__ void __launch_bounds__(EC::THREADS, 1)
    local_gemm_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap cmap,
                      LocalSched sched) {
  RDB_TRACE_SCOPE(20);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  eng::run<EC>(smem_raw, &amap, sched, eng::BulkEpilogue<EC>{&cmap});
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
    T.a_col = 0;  // A operand: M rows I
    T.a_row = I * NB;
    T.a_mat = 0;
    T.b = y + (int64_t)J * NB;
    T.ldb = ldy;
    T.c_col = J * NB;  // the epilogue needs the tile origin only
    T.c_row = I * NB;
    T.c_mat = 0;
    T.nk = nk;
    T.mode = eng::EPI_STORE;
    T.neg = 0;
    T.signal = nullptr;
    T.wait = nullptr;
    T.wait_target = 0;
    return T;
  }
};

struct ResidualEpi {
  double* out_max;
  RDB_DEV void operator()(eng::Tile T, double (&acc)[EC::MI][EC::NI][2], int wr, int wc, int lane,
                          double*) const {
    const int64_t row0 = T.c_row + wr * EC::MI * 8, col0 = (int64_t)T.c_col + wc * EC::WCOLS;
    double mx = 0.0;
#pragma unroll
    for (int mi = 0; mi < EC::MI; ++mi)
#pragma unroll
      for (int ni = 0; ni < EC::NI; ++ni) {
        const int64_t gi = row0 + mi * 8 + eng::pi_row(lane >> 2);
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

__global__ void __launch_bounds__(EC::THREADS, 1)
    residual_kernel(const __grid_constant__ CUtensorMap amap, ResidualSched sched, ResidualEpi epi) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  eng::run<EC>(smem_raw, &amap, sched, epi);
}

}  // namespace rdb

using namespace rdb;

extern "C" size_t rdb_invert_workspace_bytes(int64_t n_pad, int64_t batch) {
  if (n_pad <= 0 || batch <= 0) return 0;
  const size_t counters = rdb::counter_bytes(n_pad, batch);
  if (batch == 1 && n_pad >= rdb::wide_min_n() && n_pad % rdb::WB == 0)
    return (counters > 256 ? counters : 256) + rdb::wide_scratch_bytes(n_pad);  // counters | R | C
  return rdb::BatchWs(n_pad, batch).total;  // counters | dynamic tile counters | block-sparse plan
}

extern "C" int rdb_invert_batched(double* a, int64_t n_pad, int64_t lda, int64_t stride,
                                  int64_t batch, void* work, rdb_pivot_info* info, void* stream) {
  return invert_batched(a, n_pad, lda, stride, batch, work, info,
                        static_cast<cudaStream_t>(stream));
}

extern "C" int rdb_invert_batched_bits(double* a, int64_t n_pad, int64_t lda, int64_t stride, int64_t batch,
                                       const uint32_t* bits, int64_t n, void* work, rdb_pivot_info* info,
                                       void* stream) {
  if (!bits || n <= 0 || n > n_pad) return RDB_EINVAL;
  return invert_batched(a, n_pad, lda, stride, batch, work, info, static_cast<cudaStream_t>(stream), bits, n);
}

extern "C" int rdb_invert(double* a, int64_t n_pad, int64_t lda, void* work, rdb_pivot_info* info,
                          void* stream) {
  return invert_batched(a, n_pad, lda, n_pad * lda, 1, work, info,
                        static_cast<cudaStream_t>(stream));
}

extern "C" int rdb_gj_panel_inverse(double* a, int64_t lda, rdb_pivot_info* info, int first, int64_t p0,
                                    void* stream) {
  if (!a || !info || lda < NB || (lda & 1) || ((uintptr_t)a & 15)) return RDB_EINVAL;
  int rc = setup();
  if (rc) return rc;
  // the block is at `a`; p0 is its global index, used only for the recorded pivot index
  gj_panel_kernel<<<1, p1::THREADS, p1::SMEM_BYTES, static_cast<cudaStream_t>(stream)>>>(a, lda, 0, 0, (int)p0,
                                                                                         info, first);
  RDB_LAUNCH_CHECK();
  return RDB_OK;
}

extern "C" int rdb_gemm_local(const double* a, int64_t lda, const double* b, int64_t ldb, double* c,
                              int64_t ldc, int64_t m, int64_t n, int64_t k, int64_t skip_row_tile,
                              int64_t skip_col_tile, int64_t store_col_tile, int accumulate, int negate,
                              int64_t max_ctas, void* stream) {
  if (!a || !b || !c || m <= 0 || n <= 0 || k <= 0 || m % NB || n % NB || k % eng::BK) return RDB_EINVAL;
  if ((lda & 1) || (ldb & 1) || (ldc & 1) || lda < k || ldb < n || ldc < n) return RDB_EINVAL;
  if (((uintptr_t)b & 15) || ((uintptr_t)c & 15)) return RDB_EINVAL;
  int rc = setup();
  if (rc) return rc;
  static DeviceFlags attr;
  const int attr_dev = current_device();
  if (!attr.get(attr_dev)) {
    if (cudaFuncSetAttribute(local_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)EC::SMEM_BYTES) != cudaSuccess)
      return RDB_ECUDA;
    attr.set(attr_dev);
  }
  CUtensorMap amap;
  rc = make_a_map(&amap, a, m, k, lda, m * lda, 1);
  if (rc) return rc;
  const int mt = (int)(m / NB), nt = (int)(n / NB);
  CUtensorMap cmap;
  rc = make_ec_map(&cmap, c, m, n, ldc, m * ldc, 1);
  if (rc) return rc;
  LocalSched sched{b, ldb, mt, nt, (int)(k / eng::BK),
                   (int)(skip_row_tile >= 0 && skip_row_tile < mt ? skip_row_tile : -1),
                   (int)(skip_col_tile >= 0 && skip_col_tile < nt ? skip_col_tile : -1),
                   (int)(store_col_tile >= 0 && store_col_tile < nt ? store_col_tile : -1),
                   accumulate ? eng::EPI_REDUCE : eng::EPI_STORE, negate ? 1 : 0};
  const int64_t tiles = (int64_t)(mt - (sched.skip_row >= 0)) * (nt - (sched.skip_col >= 0));
  if (tiles <= 0) return RDB_OK;
  unsigned grid = persistent_grid(tiles);
  if (max_ctas > 0 && grid > (unsigned)max_ctas) grid = (unsigned)max_ctas;
  local_gemm_kernel<<<grid, EC::THREADS, EC::SMEM_BYTES, static_cast<cudaStream_t>(stream)>>>(amap, cmap, sched);
  RDB_LAUNCH_CHECK();
  return RDB_OK;
}

extern "C" int rdb_residual(const double* m, int64_t ldm, const double* y, int64_t ldy,
                            int64_t n_pad, double* out_max, void* stream) {
  if (!m || !y || !out_max || n_pad <= 0 || n_pad % NB || (ldm & 1) || (ldy & 1) || ldm < n_pad ||
      ldy < n_pad)
    return RDB_EINVAL;
  if (cudaFuncSetAttribute(residual_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)EC::SMEM_BYTES) != cudaSuccess)
    return RDB_ECUDA;
  const int nt = (int)(n_pad / NB);
  ResidualSched sched{m, y, ldm, ldy, nt, (int)(n_pad / eng::BK)};
  ResidualEpi epi{out_max};
  CUtensorMap amap;
  int rc = make_a_map(&amap, m, n_pad, n_pad, ldm, n_pad * ldm, 1);
  if (rc) return rc;
  residual_kernel<<<persistent_grid((int64_t)nt * nt), EC::THREADS, EC::SMEM_BYTES,
                    static_cast<cudaStream_t>(stream)>>>(amap, sched, epi);
  RDB_LAUNCH_CHECK();
  return RDB_OK;
}


#ifdef RDB_TRACE
// Diagnostic builds only (tools/sm_timeline.py): records go to buf[0, cap/2)
// from this file's kernels and to buf[cap/2, cap) from the banded path's.
namespace rdb {
namespace band {
int trace_attach(void* buf, unsigned cap);
unsigned trace_count();
}  // namespace band
}  // namespace rdb
namespace rdb {
namespace k1 {
int trace_attach(void* buf, unsigned cap);
}
namespace k3 {
int trace_attach(void* buf, unsigned cap);
}
}  // namespace rdb
extern "C" int rdb_trace_attach(void* buf, unsigned cap) {  // four quarters: K2, banded path, K1, K3
  const unsigned q = cap / 4;
  trace::Rec* r = static_cast<trace::Rec*>(buf);
  if (trace::attach(buf, q) || band::trace_attach(buf ? r + q : nullptr, q) ||
      k1::trace_attach(buf ? r + 2 * q : nullptr, q) || k3::trace_attach(buf ? r + 3 * q : nullptr, q))
    return RDB_ECUDA;
  return RDB_OK;
}
extern "C" void rdb_trace_counts(unsigned* out) {
  out[0] = trace::count();
  out[1] = band::trace_count();
}
#endif
