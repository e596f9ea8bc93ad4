// Persistent, warp-specialised FP64 DMMA GEMM engine for sm_100a.
//
//   for every tile t assigned to this CTA (t = blockIdx.x, += gridDim.x):
//     acc(128x128) = sum_k A(rows, k) * B(k, cols)          (DMMA.8x8x4)
//     C(rows, cols)  = +-acc (EPI_STORE)   or   C += +-acc (EPI_REDUCE)
//
// * MMA warps: a WGM x WGN grid of warp tiles ((128/WGM) x (128/WGN)),
//   accumulators in registers (Cfg below).
// * one producer warp: streams BK=16-deep k-chunks into a STAGES-deep ring,
//   one full/empty mbarrier pair per stage, running ahead across tile
//   boundaries so the next tile's operands arrive during the epilogue.
//   - A (row-major in global memory) arrives as ONE 3-D TMA tensor tile
//     (cp.async.bulk.tensor, SASS UTMALDG): 128 rows x 16 doubles, 128-byte
//     swizzle. The MMA row -> smem row map pi(r) = 2(r%4) + (r%8)/4 (within
//     each 8-row group) makes the m8n8k4 A-fragment loads bank-conflict free
//     under that swizzle; the epilogue writes accumulator row r to C row pi(r).
//   - B (row-major) arrives as 16 one-dimensional bulk copies of 1 KB into a
//     padded layout (row stride 132 doubles, conflict free).
// * epilogue: each MMA warp stages its 32 x 32 tile in shared memory and
//   writes it back with ONE TMA tensor store or tensor reduce-add
//   (cp.reduce.async.bulk.tensor .add, SASS UTMAREDG.ADD on an FP64 tensor
//   map): C is never read by the SM; the L2 applies C + acc with one IEEE
//   rounding. The TMA op is issued a few chunks into the next tile
//   (deferred), so the epilogue itself is only the staging stores.
// * in-kernel dependencies (tiles that overwrite an operand other tiles read):
//   the producer signals a tile's counter from the full barrier of its last
//   chunk and holds the next tile until this tile's own wait is satisfied;
//   the MMA warps never spin inside a tile (Tile::wait below).
// * STAGES = 3 with whole-tile staging measured 1% faster on the config-2
//   batch and the N = 16384 inversion than 4 stages + half-tile staging
//   (tools/time_k2.py); conflict-free (shuffle-paired) staging, an L2
//   prefetch of C and a two-group warp stagger measured no gain.
#pragma once
#include <cuda.h>

#include "common.cuh"

namespace rdb {
namespace eng {

#ifndef RDB_ENG_STAGES
#define RDB_ENG_STAGES 3
#endif
#ifndef RDB_ENG_PIECES
#define RDB_ENG_PIECES 1
#endif
#ifndef RDB_ENG_DEFER
#define RDB_ENG_DEFER 1
#endif
// deferred epilogue: warp w issues its TMA write at chunk w * min(nk, SPAN) / 16
// (SPAN 4: all issued in the first quarter of a K = 256 tile, so the staging
// buffer is free again by the epilogue; measured 9.47 -> 9.41 ms per config-2
// K2 call and +1% at N = 16384 against spreading over the whole tile)
#ifndef RDB_ENG_ISSUE_SPAN
#define RDB_ENG_ISSUE_SPAN 4
#endif
constexpr int BM = 128, BN = 128, BK = 16, STAGES = RDB_ENG_STAGES;
constexpr int BST = BN + 4;  // B row stride (132 = 4 mod 16)
constexpr uint32_t STAGE_BYTES = (BM * BK + BK * BN) * 8;

// Warp layout: WGM x WGN MMA warps, warp tile (8*MI) x (8*NI).
template <int WGM_, int WGN_>
struct Cfg {
  static constexpr int WGM = WGM_, WGN = WGN_;
  static constexpr int MMA_WARPS = WGM * WGN;
  static constexpr int THREADS = (MMA_WARPS + 1) * 32;
  static constexpr int MI = BM / WGM / 8;   // 8-row groups per warp
  static constexpr int NI = BN / WGN / 8;   // 8-col groups per warp
  static constexpr int WCOLS = NI * 8;      // warp tile width (doubles)
  static constexpr int PIECES = RDB_ENG_PIECES;    // staging pieces per warp tile
  static constexpr int HROWS = MI * 8 / PIECES;  // staging piece height
  struct Smem {
    alignas(1024) double a[STAGES][BM * BK];
    alignas(128) double b[STAGES][BK * BST];
    alignas(128) double out[MMA_WARPS][HROWS * WCOLS];  // dense HROWS x WCOLS TMA box per warp
    alignas(8) uint64_t full[STAGES];
    alignas(8) uint64_t empty[STAGES];
    int tile_of[STAGES];  // dynamic scheduling: tile index of the stage's first chunk (-1: done)
  };
  static constexpr size_t SMEM_BYTES = sizeof(Smem) + 1024;  // + alignment slack
};

using Default = Cfg<4, 4>;  // 16 MMA warps, 32x32 warp tiles

enum { EPI_STORE = 0, EPI_REDUCE = 1 };

// A tile job produced by a scheduler.
struct Tile {
  int a_col, a_row, a_mat;  // TMA coordinates of A(row0, k=0): column, row, matrix (batch) index
  const double* b;          // &B[0][col0]
  int64_t ldb;
  int c_col, c_row, c_mat;  // TMA coordinates of C(row0, col0) in the C tensor map
  int c_sel = 0;            // 1: write through the epilogue's second C map (cmap2)
  int nk;                   // number of BK chunks
  int mode;                 // EPI_STORE / EPI_REDUCE
  int neg;                  // write -acc instead of acc
  // Optional in-kernel dependency (tiles that overwrite another tile's
  // operand): after its last k-chunk has landed in shared memory a tile
  // increments *signal (the producer warp does, from the stage's full
  // barrier); a tile with wait != nullptr holds its write until *wait >=
  // wait_target. The awaited tiles are the tile's dependency group: tiles of
  // smaller index, or the few tiles next to it in index order that share its
  // operand (the G tiles of a row-panel column, the band tiles at the end of
  // an update row; G <= 4). Forward progress: a CTA's producer takes no new
  // tile while the last one's wait is open (its MMA warps never block inside
  // a tile, so every taken tile is loaded and signalled); tiles are handed
  // out in index order, so the lowest group with untaken tiles is held by at
  // most G - 1 CTAs and every other CTA of the launch is released by groups
  // that are fully taken, then takes the missing tiles. A launch therefore
  // progresses whenever G of its CTAs can be resident, whatever else shares
  // the GPU (its grid is never smaller than a group).
  int* signal;
  const int* wait;
  int wait_target;
};

RDB_DEV int pi_row(int r) { return 2 * (r & 3) + ((r >> 2) & 1); }

RDB_DEV void signal_done(int* cnt) {
  fence_proxy_async();
  __threadfence();
  atomicAdd(cnt, 1);
}

RDB_DEV void wait_count(const int* cnt, int target) {
  int v;
  do {
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(cnt) : "memory");
  } while (v < target);
  fence_proxy_async();
}

RDB_DEV void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
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

// Default epilogue: C = +-acc (EPI_STORE) or C += +-acc (EPI_REDUCE), the warp
// tile staged in two HROWS x WCOLS halves through the per-warp staging buffer
// (dense, the TMA box layout), each written back by ONE tensor store / tensor
// reduce-add (SASS UTMASTG / UTMAREDG.ADD) issued by lane 0.
RDB_DEV void tma_store_3d(const CUtensorMap* map, int c0, int c1, int c2, const void* src) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src))
               : "memory");
}

RDB_DEV void tma_reduce_add_3d(const CUtensorMap* map, int c0, int c1, int c2, const void* src) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src))
      : "memory");
}


template <class C>
struct BulkEpilogue {
  const CUtensorMap* cmap;            // box HROWS x WCOLS over the output matrices
  const CUtensorMap* cmap2 = nullptr;  // optional second output (tiles with c_sel = 1)
  // With the whole warp tile staged (PIECES == 1, the default) the TMA store /
  // reduce-add is not issued in the epilogue but a few k-chunks into the NEXT
  // tile (warp w at chunk w*nk/16, see run()): the 128 KB of C traffic per
  // tile leaves the SM spread over the main loop instead of as one burst
  // queued in front of the next tile's operand loads, and the epilogue is
  // just staging + fence.
  static constexpr bool kDeferred = (C::PIECES == 1) && (RDB_ENG_DEFER != 0);

  // piece h (HROWS rows) of the warp tile -> dense staging box, fenced for TMA
  RDB_DEV void write_piece(const Tile& T, double (&acc)[C::MI][C::NI][2], int h, int lane, double* stage_out) const {
    const int lr = lane >> 2, lk = lane & 3;
    const int pr = pi_row(lr);
#pragma unroll
    for (int m = 0; m < C::MI / C::PIECES; ++m)
#pragma unroll
      for (int ni = 0; ni < C::NI; ++ni) {
        const int row = m * 8 + pr;
        const int col = ni * 8 + 2 * lk;
        const double x0 = acc[(C::MI / C::PIECES) * h + m][ni][0], x1 = acc[(C::MI / C::PIECES) * h + m][ni][1];
        *reinterpret_cast<double2*>(&stage_out[row * C::WCOLS + col]) =
            T.neg ? make_double2(-x0, -x1) : make_double2(x0, x1);
      }
    fence_proxy_async();
    __syncwarp();
  }

  // lane 0: write piece h of tile T from the staging buffer, after T.wait
  // when `wait` is set (the deferred form honours the dependency here)
  RDB_DEV void issue(const Tile& T, int wr, int wc, int h, int lane, bool wait, const double* stage_out) const {
    if (lane == 0) {
      if (wait && T.wait) wait_count(T.wait, T.wait_target);
      const int c0 = T.c_col + wc * C::WCOLS;
      const int c1 = T.c_row + wr * C::MI * 8 + C::HROWS * h;
      const CUtensorMap* map = (T.c_sel && cmap2) ? cmap2 : cmap;
      if (T.mode == EPI_REDUCE)
        tma_reduce_add_3d(map, c0, c1, T.c_mat, stage_out);
      else
        tma_store_3d(map, c0, c1, T.c_mat, stage_out);
      bulk_commit();
    }
  }

  // deferred form, part 1: stage the warp tile (issue() follows later)
  RDB_DEV void stage(const Tile& T, double (&acc)[C::MI][C::NI][2], int lane, double* stage_out) const {
    if (lane == 0) bulk_wait_read0();  // the previous tile's write has left the staging buffer
    __syncwarp();
    write_piece(T, acc, 0, lane, stage_out);
  }

  // immediate form (the run loop has already honoured T.wait)
  RDB_DEV void operator()(Tile T, double (&acc)[C::MI][C::NI][2], int wr, int wc, int lane,
                          double* stage_out) const {
#pragma unroll
    for (int h = 0; h < C::PIECES; ++h) {
      if (lane == 0) bulk_wait_read0();  // the previous piece has left the staging buffer
      __syncwarp();
      write_piece(T, acc, h, lane, stage_out);
      issue(T, wr, wc, h, lane, false, stage_out);
    }
  }
};

// Sched::dyn (when present and non-null): a global tile counter. CTAs then take
// tiles in arrival order (atomicAdd) instead of the static blockIdx + k*gridDim
// stride, so a launch that shares the GPU with another stream's kernels
// balances itself; each CTA still sees increasing tile indices (the in-kernel
// dependency argument holds). The last grab (value ntiles + gridDim - 1)
// resets the counter to 0 for the next launch.
template <class S, class = void>
struct DynOf {
  RDB_DEV static int* get(const S&) { return nullptr; }
};
template <class S>
struct DynOf<S, decltype((void)S::dyn)> {
  RDB_DEV static int* get(const S& s) { return s.dyn; }
};

// Sched::dyn_ctas (when present and > 0): the CTAs of every launch sharing the
// counter (a helper launch on another stream joins the same tile list; the
// reset then waits for all of their final grabs); else this grid's.
template <class S, class = void>
struct DynCtasOf {
  RDB_DEV static int get(const S&) { return (int)gridDim.x; }
};
template <class S>
struct DynCtasOf<S, decltype((void)S::dyn_ctas)> {
  RDB_DEV static int get(const S& s) { return s.dyn_ctas > 0 ? s.dyn_ctas : (int)gridDim.x; }
};

RDB_DEV int grab_tile(int* dyn, int ntiles, int ctas, int lane) {
  int v = 0;
  if (lane == 0) {
    v = atomicAdd(dyn, 1);
    if (v == ntiles + ctas - 1) atomicExch(dyn, 0);
  }
  return __shfl_sync(0xffffffffu, v, 0);
}

// Epi::kDeferred (when present) selects the stage()/issue() protocol.
template <class E, class = void>
struct Defers {
  static constexpr bool value = false;
};
template <class E>
struct Defers<E, decltype((void)E::kDeferred)> {
  static constexpr bool value = E::kDeferred;
};

// Sched must provide: int count() and Tile tile(int t) (identical in every warp).
// Epi: callable (Tile, acc, wr, wc, lane, staging) run by each MMA warp per
// tile, or a deferred epilogue (BulkEpilogue with kDeferred).
template <class C, class Sched, class Epi>
__device__ __forceinline__ void run(unsigned char* smem_raw, const CUtensorMap* amap, const Sched& sched,
                                    const Epi& epi) {
  using Smem = typename C::Smem;
  // the 128-byte TMA swizzle atom needs a 1024-byte aligned destination: align
  // the dynamic shared memory base (pointer arithmetic keeps the shared space)
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  Smem& s = *reinterpret_cast<Smem*>(smem_raw + pad);
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&s.full[i], 1);
      mbar_init(&s.empty[i], C::MMA_WARPS);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int ntiles = sched.count();

  if (warp == C::MMA_WARPS) {
    // ------------------------------------------------------------ producer
    if (lane == 0) asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(amap)) : "memory");
    int st = 0;
    uint32_t ph = 0;
    int* const dyn = DynOf<Sched>::get(sched);
    const int ctas = DynCtasOf<Sched>::get(sched);
    for (int t = dyn ? grab_tile(dyn, ntiles, ctas, lane) : (int)blockIdx.x;;
         t = dyn ? grab_tile(dyn, ntiles, ctas, lane) : t + (int)gridDim.x) {
      if (t >= ntiles) {
        if (dyn) {  // tell the MMA warps: no more tiles
          mbar_wait(&s.empty[st], ph ^ 1);
          if (lane == 0) {
            s.tile_of[st] = -1;
            mbar_arrive(&s.full[st]);
          }
        }
        break;
      }
      const Tile T = sched.tile(t);
      int st_last = 0;
      uint32_t ph_last = 0;
      for (int c = 0; c < T.nk; ++c) {
        mbar_wait(&s.empty[st], ph ^ 1);
        const int k0 = c * BK;
        if (lane == 0) {
          if (c == 0) s.tile_of[st] = t;  // published by the full barrier's completion
          mbar_arrive_expect_tx(&s.full[st], STAGE_BYTES);
          tma_load_3d(s.a[st], amap, T.a_col + k0, T.a_row, T.a_mat, &s.full[st]);
        }
        __syncwarp();
        if (lane < BK)
          bulk_g2s(&s.b[st][lane * BST], T.b + (int64_t)(k0 + lane) * T.ldb, BN * 8, &s.full[st]);
        st_last = st;
        ph_last = ph;
        if (++st == STAGES) {
          st = 0;
          ph ^= 1;
        }
      }
      // Dependency groups (see Tile::wait). The producer signals as soon as the
      // tile's last chunk has landed (this stage's full barrier: it cannot be
      // re-armed before the producer itself refills it), and takes no further
      // tile until this tile's own wait is satisfied: the MMA warps then never
      // spin on a counter in the middle of a tile, so the CTA never holds a
      // tile it cannot finish while sitting on another one the same group
      // needs (a CTA that drew two tiles of a group deadlocked otherwise).
      if (T.signal || T.wait) {
        if (lane == 0) {
          if (T.signal) {
            mbar_wait(&s.full[st_last], ph_last);
            signal_done(T.signal);
          }
          if (T.wait) wait_count(T.wait, T.wait_target);
        }
        __syncwarp();
      }
    }
    return;
  }

  // -------------------------------------------------------------- MMA warps
  const int wr = warp / C::WGN;
  const int wc = warp % C::WGN;
  const int lr = lane >> 2, lk = lane & 3;
  // A fragment byte offsets within a stage for (mi, kk): physical row
  // pr = 8*MI*wr + 8mi + pi(lr); 16-byte chunk ((kk+lk)/2) ^ (pr%8); +8 if odd k.
  const int prow = wr * C::MI * 8 + pi_row(lr);
  const int psw = pi_row(lr);  // == prow % 8
  double* stage_out = s.out[warp];
  constexpr bool kDefer = Defers<Epi>::value;
  int pend_t = -1;  // tile whose staged write is not yet issued (deferred epilogue)
  int st = 0;
  uint32_t ph = 0;
  const bool dyn = DynOf<Sched>::get(sched) != nullptr;
  for (int t = blockIdx.x;; t += gridDim.x) {
    if (dyn) {
      mbar_wait(&s.full[st], ph);  // the tile's first chunk (or the end marker)
      t = s.tile_of[st];
      if (t < 0) break;
    } else if (t >= ntiles) {
      break;
    }
    const Tile T = sched.tile(t);
    const int issue_at = kDefer ? (warp * (T.nk < RDB_ENG_ISSUE_SPAN ? T.nk : RDB_ENG_ISSUE_SPAN)) / C::MMA_WARPS : 0;
    double acc[C::MI][C::NI][2];
#pragma unroll
    for (int i = 0; i < C::MI; ++i)
#pragma unroll
      for (int j = 0; j < C::NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int c = 0; c < T.nk; ++c) {
      if (!dyn || c > 0) mbar_wait(&s.full[st], ph);
      if constexpr (kDefer) {
        if (pend_t >= 0 && c == issue_at) {
          epi.issue(sched.tile(pend_t), wr, wc, 0, lane, true, stage_out);
          pend_t = -1;
        }
      }
      const char* sa = reinterpret_cast<const char*>(s.a[st]);
      const double* sb = s.b[st] + lk * BST + wc * C::WCOLS + lr;
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        double af[C::MI], bf[C::NI];
        const int kq = kk + lk;
        const int off = (((kq >> 1) ^ psw) << 4) + ((kq & 1) << 3);
#pragma unroll
        for (int mi = 0; mi < C::MI; ++mi)
          af[mi] = *reinterpret_cast<const double*>(sa + (prow + mi * 8) * 128 + off);
#pragma unroll
        for (int ni = 0; ni < C::NI; ++ni) bf[ni] = sb[kk * BST + ni * 8];
#pragma unroll
        for (int mi = 0; mi < C::MI; ++mi)
#pragma unroll
          for (int ni = 0; ni < C::NI; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&s.empty[st]);
      if (++st == STAGES) {
        st = 0;
        ph ^= 1;
      }
    }

    if constexpr (kDefer) {
      if (pend_t >= 0) epi.issue(sched.tile(pend_t), wr, wc, 0, lane, true, stage_out);  // nk <= issue_at
      epi.stage(T, acc, lane, stage_out);
      pend_t = t;
    } else {
      if (T.wait) {
        if (lane == 0) wait_count(T.wait, T.wait_target);
        __syncwarp();
      }
      epi(T, acc, wr, wc, lane, stage_out);
    }
  }
  if constexpr (kDefer) {
    if (pend_t >= 0) epi.issue(sched.tile(pend_t), wr, wc, 0, lane, true, stage_out);
  }
  bulk_wait0();
}

}  // namespace eng

// Host: a 3-D tensor map over `batch` row-major fp64 matrices (rows x cols,
// row stride ld, matrix stride `stride` elements) with 128 x 16 boxes and
// 128-byte swizzle — the engine's A operand. Returns RDB_OK or an error.
int make_a_map(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld,
               int64_t stride, int64_t batch);
// Host: the epilogue's C map over the same kind of 3-D layout, box
// box_rows x box_cols, no swizzle (the staging buffer is the dense box).
int make_c_map(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld,
               int64_t stride, int64_t batch, int box_rows, int box_cols);

}  // namespace rdb
