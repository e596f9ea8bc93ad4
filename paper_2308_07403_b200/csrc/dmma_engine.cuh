// Persistent, warp-specialised FP64 DMMA GEMM engine for sm_100a.
//
//   for every tile t assigned to this CTA (t = blockIdx.x, += gridDim.x):
//     acc(128x128) = sum_k A(rows, k) * B(k, cols)          (DMMA.8x8x4)
//     C(rows, cols)  = acc   (EPI_STORE)   or   C += acc (EPI_REDUCE)
//
// * warps 0-7 (MMA): 2 x 4 grid of 64x32 warp tiles, 64 fp64 accumulators per
//   lane; fragments from padded shared memory (bank-conflict free for the
//   m8n8k4 lane layout).
// * warp 8 (producer): streams BK=16-deep k-chunks of A and B into a
//   STAGES-deep ring with 1-D bulk copies (TMA engine, cp.async.bulk), one
//   full/empty mbarrier pair per stage; it runs ahead across tile boundaries,
//   so the next tile's operands arrive while the MMA warps drain the epilogue.
// * epilogue: each MMA warp stages 32x32 sub-tiles in shared memory and
//   writes them back with bulk stores or bulk reduce-adds
//   (cp.reduce.async.bulk .add.f64, SASS UBLKRED.ADD.F64.RN): C is never read
//   by the SM, the L2 applies C + acc with one IEEE rounding.
//
// A is either k-major in memory (A^T row-major: element (i,k) at A[k*lda+i];
// 16 bulk copies of 1 KB per chunk) or row-major (element (i,k) at
// A[i*lda+k]; 128 copies of 128 B). B is row-major (element (k,j) at
// B[k*ldb+j]).
#pragma once
#include "common.cuh"

namespace rdb {
namespace eng {

constexpr int BM = 128, BN = 128, BK = 16, STAGES = 3;
constexpr int AST_K = BM + 4;  // k-major A row stride (132 = 4 mod 16)
constexpr int AST_R = BK + 4;  // row-major A row stride (20 = 4 mod 16)
constexpr int BST = BN + 4;    // B row stride (132)
constexpr int OST = 40;        // epilogue staging row stride (STS.128 conflict free)
constexpr int MMA_WARPS = 8;
constexpr int THREADS = (MMA_WARPS + 1) * 32;
constexpr uint32_t STAGE_BYTES = (BM * BK + BK * BN) * 8;
constexpr int A_STAGE_DOUBLES = (BM * AST_R > BK * AST_K) ? BM * AST_R : BK * AST_K;

enum { EPI_STORE = 0, EPI_REDUCE = 1 };

struct Smem {
  alignas(128) double a[STAGES][A_STAGE_DOUBLES];
  alignas(128) double b[STAGES][BK * BST];
  alignas(128) double out[MMA_WARPS][32 * OST];
  alignas(8) uint64_t full[STAGES];
  alignas(8) uint64_t empty[STAGES];
};
constexpr size_t SMEM_BYTES = sizeof(Smem);

// A tile job produced by a scheduler: operand origins for this tile, K, output.
struct Tile {
  const double* a;  // k-major: &A^T[0][row0]; row-major: &A[row0][0]
  int64_t lda;
  const double* b;  // &B[0][col0]
  int64_t ldb;
  double* c;        // &C[row0][col0]
  int64_t ldc;
  int nk;           // number of BK chunks
  int mode;         // EPI_STORE / EPI_REDUCE
};

RDB_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

RDB_DEV void bulk_s2g(double* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}

RDB_DEV void bulk_s2g_add(double* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;\n" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}

RDB_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
RDB_DEV void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
RDB_DEV void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }

// Default epilogue: C = acc (EPI_STORE) or C += acc (EPI_REDUCE) through two
// 32x32 halves of the per-warp staging buffer and bulk stores / reduce-adds.
struct BulkEpilogue {
  RDB_DEV void operator()(const Tile& T, double (&acc)[8][4][2], int wr, int wc, int lane,
                          double* stage_out) const {
    const int lr = lane >> 2, lk = lane & 3;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      bulk_wait_read0();  // this lane's previous bulk op has finished reading staging
      __syncwarp();
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
          const int row = m * 8 + lr;
          const int col = ni * 8 + 2 * lk;
          *reinterpret_cast<double2*>(&stage_out[row * OST + col]) =
              make_double2(acc[4 * h + m][ni][0], acc[4 * h + m][ni][1]);
        }
      fence_proxy_async();
      __syncwarp();
      double* dst = T.c + (int64_t)(wr * 64 + 32 * h + lane) * T.ldc + wc * 32;
      if (T.mode == EPI_REDUCE)
        bulk_s2g_add(dst, &stage_out[lane * OST], 32 * 8);
      else
        bulk_s2g(dst, &stage_out[lane * OST], 32 * 8);
      bulk_commit();
    }
  }
};

// Sched must provide: int count() and Tile tile(int t) (identical in every warp).
// Epi: callable (Tile, acc, wr, wc, lane, staging) run by each MMA warp per tile.
template <bool A_KMAJOR, class Sched, class Epi = BulkEpilogue>
__device__ __forceinline__ void run(Smem& s, const Sched& sched, const Epi& epi = Epi()) {
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&s.full[i], 1);
      mbar_init(&s.empty[i], MMA_WARPS);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int ntiles = sched.count();

  if (warp == MMA_WARPS) {
    // ------------------------------------------------------------ producer
    int st = 0;
    uint32_t ph = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const Tile T = sched.tile(t);
      for (int c = 0; c < T.nk; ++c) {
        mbar_wait(&s.empty[st], ph ^ 1);
        if (lane == 0) mbar_arrive_expect_tx(&s.full[st], STAGE_BYTES);
        __syncwarp();
        const int k0 = c * BK;
        if (A_KMAJOR) {
          if (lane < BK)
            bulk_g2s(&s.a[st][lane * AST_K], T.a + (int64_t)(k0 + lane) * T.lda, BM * 8, &s.full[st]);
        } else {
#pragma unroll
          for (int q = 0; q < BM / 32; ++q) {
            const int i = lane + 32 * q;
            bulk_g2s(&s.a[st][i * AST_R], T.a + (int64_t)i * T.lda + k0, BK * 8, &s.full[st]);
          }
        }
        if (lane >= 32 - BK) {
          const int kk = lane - (32 - BK);
          bulk_g2s(&s.b[st][kk * BST], T.b + (int64_t)(k0 + kk) * T.ldb, BN * 8, &s.full[st]);
        }
        if (++st == STAGES) {
          st = 0;
          ph ^= 1;
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- MMA warps
  const int wr = warp >> 2;  // 0..1 : rows 64*wr
  const int wc = warp & 3;   // 0..3 : cols 32*wc
  const int lr = lane >> 2, lk = lane & 3;
  double* stage_out = s.out[warp];
  int st = 0;
  uint32_t ph = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const Tile T = sched.tile(t);
    double acc[8][4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int c = 0; c < T.nk; ++c) {
      mbar_wait(&s.full[st], ph);
      const double* sa = s.a[st];
      const double* sb = s.b[st] + lk * BST + wc * 32 + lr;
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        double af[8], bf[4];
#pragma unroll
        for (int mi = 0; mi < 8; ++mi) {
          const int r = wr * 64 + mi * 8 + lr;
          af[mi] = A_KMAJOR ? sa[(kk + lk) * AST_K + r] : sa[r * AST_R + kk + lk];
        }
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) bf[ni] = sb[kk * BST + ni * 8];
#pragma unroll
        for (int mi = 0; mi < 8; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&s.empty[st]);
      if (++st == STAGES) {
        st = 0;
        ph ^= 1;
      }
    }

    epi(T, acc, wr, wc, lane, stage_out);
  }
  bulk_wait0();
}

}  // namespace eng
}  // namespace rdb
