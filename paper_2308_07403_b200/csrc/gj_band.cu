// K2b: inverse of block-tridiagonal M-matrices (bandwidth <= 32) in a batch.
//
// Part of rdb_invert_batched_bits / the rdb_apsp_bits_batched pipelines
// (replacing scipy.linalg.lu_factor + lu_solve(I), pkg/src/rdist/linalg.py:32,
// :39, like K2). A matrix whose adjacency has every edge j -> i within
// |i / 32 - j / 32| <= 1 (any bandwidth-32 graph in its vertex order, e.g. the
// directed 32 x 32 lattices of config 2) is block tridiagonal in 32 x 32
// blocks: M = tridiag(L_r, T_r, U_r), r = 0 .. nb-1. Its inverse follows from
// two block-Schur sweeps instead of Gauss-Jordan on the whole matrix:
//   forward   D_0 = T_0,       D_r = T_r + L_r G_{r-1},  G_r = -D_r^-1 U_r
//   backward  S_last = T_last,  S_r = T_r + U_r H_{r+1},  H_r = -S_r^-1 L_r
//   diagonal  Y_rr = (D_r + K_r)^-1,  K_r = U_r H_{r+1}
//   chains    Y_ij = G_i Y_{i+1,j} (i < j),   Y_ij = H_i Y_{i-1,j} (i > j)
// (block row i of M Y = I for i < j reads L_i Y_{i-1,j} + T_i Y_ij + U_i
// Y_{i+1,j} = 0; eliminating downwards gives D_i Y_ij = -U_i Y_{i+1,j}.)
// 2 32^3 ((nb - 1)(nb + 5) + 3 nb) flop against GJ's 2 n^3 (n = 1024: 8.1e7
// vs 2.1e9).
//
// Numerics: for a nonsingular M-matrix every D_r, S_r and diagonal Schur
// complement is again an M-matrix (inverse >= 0), G_r, H_r >= 0 and every
// chain product multiplies non-negative matrices: no cancellation, so the
// tiny entries keep componentwise relative accuracy as in K2. The D_r are
// the Schur complements of the natural elimination order, so their
// Gauss-Jordan pivots are LAPACK's diag(U) without row swaps
// (linalg.py:33-34): they give the pivot record; any pivot <= 0 in any of the
// inversions sets RDB_PIV_NONPOS. The chain kernel has then overwritten M,
// so the batch API (batch.redo_pivoted) rebuilds that graph's M from its
// adjacency and inverts it with the partial-pivoting kernel, which decides
// singularity as the reference's LAPACK path does.
//
// Kernels: band_detect_bits_kernel (flag per matrix from the adjacency bits),
// band_factor_kernel (two matrices per CTA, a 4-warp group per sweep, all
// four sweeps concurrent; the backward sweep also keeps K_r = U_r H_{r+1}),
// band_chain_kernel (a warp per block column j: Y_jj = (D_j + K_j)^-1 by a
// register-resident warp Gauss-Jordan, then nb - 1 chained 32 x 32 x 32 DMMA
// products, the operator G_i / H_i prefetched into registers one step ahead,
// the running block in shared memory, every block stored to its place in M).
#include "common.cuh"

namespace rdb {
namespace band {

constexpr int S = 32;          // block size (= the bandwidth bound)
constexpr int LD = 36;         // shared-memory row stride: conflict-free m8n8k4 fragment loads
constexpr int BLK = S * S;     // doubles per block in the workspace
constexpr int SBUF = S * LD;   // doubles per shared-memory block
constexpr int CW = 4;          // warps (block columns) per chain CTA

// Workspace per matrix: G[nb] and H[nb] in A-fragment order, D[nb] and K[nb] row-major.
size_t ws_doubles(int64_t n_pad) { return (size_t)4 * (size_t)(n_pad / S) * BLK; }
#ifndef RDB_BAND_GPC
#define RDB_BAND_GPC 2
#endif
constexpr int GPC = RDB_BAND_GPC;  // matrices per factor CTA

RDB_DEV void gbar(int id) { asm volatile("bar.sync %0, 128;\n" ::"r"(id) : "memory"); }

// A-fragment order of a 32 x 32 left operand: mma.m8n8k4 lane l holds
// A[8 mi + l / 4][4 ks + l % 4]; element e = ((ks * 2 + h) * 32 + l) * 2 + b
// is row tile mi = 2 h + b, so lane l loads tiles 2h, 2h + 1 of k-step ks as
// one coalesced double2.
RDB_DEV void frag_rc(int e, int& row, int& col) {
  const int b = e & 1, lane = (e >> 1) & 31, kh = e >> 6;
  row = 8 * (2 * (kh & 1) + b) + (lane >> 2);
  col = 4 * (kh >> 1) + (lane & 3);
}

struct Group {  // one 4-warp group's shared memory
  double X[SBUF], A[SBUF], P[SBUF];
  double prow[2][S], pcol[2][S];
};
struct FactorSmem {
  Group g[2 * GPC];
  int flags[2 * GPC];
};

// 128 threads: global row-major block (ld) <-> shared block
RDB_DEV void load_block(double* dst, const double* __restrict__ src, int64_t ld, int t) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int e = t + 128 * q, r = e >> 4, c2 = e & 15;
    *reinterpret_cast<double2*>(dst + r * LD + 2 * c2) = ldg2(src + (int64_t)r * ld + 2 * c2);
  }
}
RDB_DEV void store_block(double* __restrict__ dst, int64_t ld, const double* src, int t) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int e = t + 128 * q, r = e >> 4, c2 = e & 15;
    stg2(dst + (int64_t)r * ld + 2 * c2, *reinterpret_cast<const double2*>(src + r * LD + 2 * c2));
  }
}
RDB_DEV void store_frag(double* __restrict__ dst, const double* src, int t) {
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int e = t + 128 * q;
    int r, c;
    frag_rc(e, r, c);
    dst[e] = src[r * LD + c];
  }
}
RDB_DEV void load_frag(double* dst, const double* __restrict__ src, int t) {
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int e = t + 128 * q;
    int r, c;
    frag_rc(e, r, c);
    dst[r * LD + c] = src[e];
  }
}

// out = [init] + (neg ? -1 : 1) A B, all 32 x 32 in shared memory; warp w of
// the group computes rows 8w .. 8w + 7. out may alias init, A or B.
RDB_DEV void gemm(double* out, const double* init, const double* A, const double* B, bool neg, int t, int id) {
  const int w = t >> 5, lane = t & 31, lr = lane >> 2, lk = lane & 3, r0 = 8 * w;
  double acc[4][2];
#pragma unroll
  for (int ni = 0; ni < 4; ++ni) {
    acc[ni][0] = init ? init[(r0 + lr) * LD + 8 * ni + 2 * lk] : 0.0;
    acc[ni][1] = init ? init[(r0 + lr) * LD + 8 * ni + 2 * lk + 1] : 0.0;
  }
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
    double af = A[(r0 + lr) * LD + 4 * ks + lk];
    if (neg) af = -af;
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) dmma_8x8x4(acc[ni][0], acc[ni][1], af, B[(4 * ks + lk) * LD + 8 * ni + lr]);
  }
  gbar(id);
#pragma unroll
  for (int ni = 0; ni < 4; ++ni)
    *reinterpret_cast<double2*>(&out[(r0 + lr) * LD + 8 * ni + 2 * lk]) = make_double2(acc[ni][0], acc[ni][1]);
  gbar(id);
}

// X <- X^-1 in place, Gauss-Jordan without pivoting; thread (rg = t / 32,
// j = t % 32) holds rows 8 rg .. 8 rg + 7 of column j. Pivots: flags always,
// the minimum |pivot| (index base + k) when `rec`.
RDB_DEV void inverse(Group& g, double* X, int id, int t, bool rec, int base, double& minp, int& mini,
                     int& flags) {
  const int j = t & 31, rg = t >> 5;
  double v[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) v[e] = X[(8 * rg + e) * LD + j];
  int b = 0;
#pragma unroll
  for (int kk = 0; kk < S; ++kk) {
    if (rg == (kk >> 3)) g.prow[b][j] = v[kk & 7];
    if (j == kk) {
#pragma unroll
      for (int e = 0; e < 8; ++e) g.pcol[b][8 * rg + e] = v[e];
    }
    gbar(id);
    const double p = g.prow[b][kk];
    const double pinv = rcp_nr(p);
    if (t == 0) {
      const double ap = fabs(p);
      if (!(ap < INFINITY)) flags |= RDB_PIV_NONFINITE;
      if (!(p > 0.0)) flags |= RDB_PIV_NONPOS;
      if (rec && (ap < minp || mini < 0)) {
        minp = ap;
        mini = base + kk;
      }
    }
    const double u = (j == kk) ? pinv : g.prow[b][j] * pinv;
    if (j == kk) {
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] = 0.0;
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = fma(-g.pcol[b][8 * rg + e], u, v[e]);
    if (rg == (kk >> 3)) v[kk & 7] = u;
    b ^= 1;
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) X[(8 * rg + e) * LD + j] = v[e];
  gbar(id);
}

// Warp-level Gauss-Jordan inverse without pivoting, lane j holding column j
// in v (the same operations as inverse(): the pivot column's entries reach
// the other lanes by shuffles).
RDB_DEV void warp_inverse(double (&v)[S], int lane, int& flags) {
#pragma unroll
  for (int kk = 0; kk < S; ++kk) {
    const double p = __shfl_sync(0xffffffffu, v[kk], kk);
    const double pinv = rcp_nr(p);
    if (!(fabs(p) < INFINITY)) flags |= RDB_PIV_NONFINITE;
    if (!(p > 0.0)) flags |= RDB_PIV_NONPOS;
    const bool piv = (lane == kk);
    const double u = piv ? pinv : v[kk] * pinv;
#pragma unroll
    for (int i = 0; i < S; ++i) {
      if (i == kk) continue;
      const double f = __shfl_sync(0xffffffffu, v[i], kk);
      v[i] = fma(-f, u, piv ? 0.0 : v[i]);
    }
    v[kk] = u;
  }
}

}  // namespace band

using namespace band;

// nonband[b] = 1 unless every edge of graph b lies in the 32-block tridiagonal
// band (word q of row i non-zero only for |q - i / 32| <= 1). A thread per
// 16-byte group of words (coalesced over the whole batch); the caller zeroes
// nonband first. Rows whose word count is not a multiple of 4 take the
// word-by-word loop.
__global__ void band_detect_bits_kernel(const uint32_t* __restrict__ bits, int64_t n, int64_t batch,
                                        int* __restrict__ nonband) {
  RDB_TRACE_SCOPE(42);
  const int64_t wpr = (n + 31) / 32;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if ((wpr & 3) == 0 && !((uintptr_t)bits & 15)) {
    const int64_t q4r = wpr / 4;  // uint4 per row
    const uint4* b4 = reinterpret_cast<const uint4*>(bits);
    for (int64_t e = t0; e < batch * n * q4r; e += nthreads) {
      const int64_t row = e / q4r, q0 = 4 * (e - row * q4r);
      const int64_t b = row / n, bi = (row - b * n) / 32;
      if (q0 + 3 >= bi - 1 && q0 <= bi + 1) {  // the group touches the band: check its outside words
        const uint4 v = __ldg(b4 + e);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
        bool bad = false;
#pragma unroll
        for (int k = 0; k < 4; ++k) bad |= (q0 + k < bi - 1 || q0 + k > bi + 1) && w[k];
        if (bad) nonband[b] = 1;
      } else {
        const uint4 v = __ldg(b4 + e);
        if (v.x | v.y | v.z | v.w) nonband[b] = 1;
      }
    }
  } else {
    for (int64_t e = t0; e < batch * n * wpr; e += nthreads) {
      const int64_t row = e / wpr, q = e - row * wpr;
      const int64_t b = row / n, bi = (row - b * n) / 32;
      if ((q < bi - 1 || q > bi + 1) && __ldg(bits + e)) nonband[b] = 1;
    }
  }
}

// Both block-Schur sweeps of GPC matrices per CTA (a 4-warp group per sweep,
// 128 * 2 * GPC threads). Writes G, H, D, K to the workspace and the pivot
// record (forward pivots = LAPACK's diag(U); flags from every inverse).
__global__ void __launch_bounds__(256 * GPC, 1)
    band_factor_kernel(const double* __restrict__ a, int64_t lda, int64_t stride, int nb, int64_t batch,
                       const int* __restrict__ nonband, double* __restrict__ ws, rdb_pivot_info* __restrict__ info) {
  RDB_TRACE_SCOPE(40);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  FactorSmem& s = *reinterpret_cast<FactorSmem*>(smem_raw);
  const int grp = threadIdx.x >> 7, t = threadIdx.x & 127, id = 1 + grp;
  const int64_t m = (int64_t)blockIdx.x * GPC + (grp >> 1);
  const bool active = m < batch && !nonband[m];  // uniform per group (named barriers are per group)
  double minp = INFINITY;
  int mini = -1, flags = 0;
  if (active) {
    const double* A = a + m * stride;
    double* G = ws + m * 4 * (int64_t)nb * BLK;
    double* H = G + (int64_t)nb * BLK;
    double* Dl = H + (int64_t)nb * BLK;
    double* K = Dl + (int64_t)nb * BLK;
    Group& g = s.g[grp];
    auto blk = [&](int r, int c) { return A + (int64_t)(S * r) * lda + S * c; };
    if ((grp & 1) == 0) {
      for (int r = 0; r < nb; ++r) {  // D_r = T_r + L_r G_{r-1}; G_r = -D_r^-1 U_r
        load_block(g.X, blk(r, r), lda, t);
        if (r > 0) {
          load_block(g.A, blk(r, r - 1), lda, t);
          gbar(id);
          gemm(g.X, g.X, g.A, g.P, false, t, id);
        } else {
          gbar(id);
        }
        store_block(Dl + (int64_t)r * BLK, S, g.X, t);
        inverse(g, g.X, id, t, true, S * r, minp, mini, flags);
        if (r < nb - 1) {
          load_block(g.A, blk(r, r + 1), lda, t);
          gbar(id);
          gemm(g.P, nullptr, g.X, g.A, true, t, id);
          store_frag(G + (int64_t)r * BLK, g.P, t);
        }
      }
    } else {
      for (int r = nb - 1; r >= 0; --r) {  // K_r = U_r H_{r+1}; S_r = T_r + K_r; H_r = -S_r^-1 L_r
        load_block(g.X, blk(r, r), lda, t);
        if (r < nb - 1) {
          load_block(g.A, blk(r, r + 1), lda, t);
          gbar(id);
          gemm(g.A, nullptr, g.A, g.P, false, t, id);
          store_block(K + (int64_t)r * BLK, S, g.A, t);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int e = t + 128 * q, rr = e >> 5, cc = e & 31;
            g.X[rr * LD + cc] += g.A[rr * LD + cc];
          }
        } else {
          const int e0 = t;
          for (int e = e0; e < BLK; e += 128) K[(int64_t)r * BLK + e] = 0.0;
        }
        gbar(id);
        inverse(g, g.X, id, t, false, 0, minp, mini, flags);
        if (r > 0) {
          load_block(g.A, blk(r, r - 1), lda, t);
          gbar(id);
          gemm(g.P, nullptr, g.X, g.A, true, t, id);
          store_frag(H + (int64_t)r * BLK, g.P, t);
        }
      }
    }
  }
  if (t == 0) s.flags[grp] = flags;
  __syncthreads();
  if (active && (grp & 1) == 0 && t == 0) {
    rdb_pivot_info* inf = info + m;
    inf->min_pivot = minp;
    inf->min_index = mini;
    inf->flags = flags | s.flags[grp + 1];
  }
}

// Block column j per warp: Y_jj = (D_j + K_j)^-1 (warp Gauss-Jordan, flags
// ORed into the pivot record), then up the column (Y_ij = G_i Y_{i+1,j},
// i = j-1 .. 0) and down (Y_ij = H_i Y_{i-1,j}, i = j+1 .. nb-1): nb - 1
// products per warp. The operator G_i / H_i of the next product streams into
// a second shared-memory buffer (cp.async, each lane copies the 16-byte
// fragment pairs it reads itself) while the current one multiplies. Reads only
// the workspace (and its own Y_jj), writes every block of M.
constexpr size_t CHAIN_SMEM = (size_t)CW * (SBUF + 2 * BLK) * sizeof(double);

RDB_DEV void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
RDB_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
RDB_DEV void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

__global__ void __launch_bounds__(CW * 32, 2)
    band_chain_kernel(double* __restrict__ a, int64_t lda, int64_t stride, int nb, const int* __restrict__ nonband,
                      const double* __restrict__ ws, rdb_pivot_info* __restrict__ info) {
  RDB_TRACE_SCOPE(41);
  const int64_t m = blockIdx.y;
  if (nonband[m]) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x * CW + warp;
  if (j >= nb) return;  // warp-uniform; only warp-level synchronisation below
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* B = reinterpret_cast<double*>(smem_raw) + warp * (SBUF + 2 * BLK);  // the running block (B operand)
  double2* Abuf = reinterpret_cast<double2*>(B + SBUF);                      // 2 x BLK: operators, fragment order
  double* A = a + m * stride;
  const double* G = ws + m * 4 * (int64_t)nb * BLK;
  const double* H = G + (int64_t)nb * BLK;
  const double* Dl = H + (int64_t)nb * BLK + (int64_t)j * BLK;
  const double* K = Dl + (int64_t)nb * BLK;
  double* diag = A + (int64_t)(S * j) * lda + S * j;
  const int lr = lane >> 2, lk = lane & 3;
  auto op_of = [&](int st) -> const double2* {
    return reinterpret_cast<const double2*>(st < j ? G + (int64_t)(j - 1 - st) * BLK : H + (int64_t)(st + 1) * BLK);
  };
  auto fetch = [&](int st) {  // this lane's 16 fragment pairs of operator st into buffer st & 1
    const double2* src = op_of(st);
    double2* dst = Abuf + (st & 1) * (BLK / 2);
#pragma unroll
    for (int q = 0; q < 16; ++q) cp_async16(dst + q * 32 + lane, src + q * 32 + lane);
    cp_async_commit();
  };
  const int steps = nb - 1;
  fetch(0);
  {
    double v[S];
#pragma unroll
    for (int i = 0; i < S; ++i) v[i] = Dl[i * S + lane] + K[i * S + lane];
    int flags = 0;
    warp_inverse(v, lane, flags);
#pragma unroll
    for (int i = 0; i < S; ++i) {
      B[i * LD + lane] = v[i];
      diag[(int64_t)i * lda + lane] = v[i];
    }
    flags = __reduce_or_sync(0xffffffffu, flags);
    if (flags && lane == 0) atomicOr(&info[m].flags, flags);
    __syncwarp();
  }
  for (int st = 0; st < steps; ++st) {
    if (st + 1 < steps) fetch(st + 1);
    else cp_async_commit();  // empty group: wait_group 1 below still retires operator st
    if (st == j && j > 0) {  // the downward chain starts again from Y_jj (written above by this warp)
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int e = lane + 32 * q, r = e >> 4, c2 = e & 15;
        *reinterpret_cast<double2*>(B + r * LD + 2 * c2) = *reinterpret_cast<const double2*>(diag + (int64_t)r * lda + 2 * c2);
      }
      __syncwarp();
    }
    cp_async_wait1();
    const double2* As = Abuf + (st & 1) * (BLK / 2);
    const int i = st < j ? j - 1 - st : st + 1;
    double acc[4][4][2];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      double bf[4];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) bf[ni] = B[(4 * ks + lk) * LD + 8 * ni + lr];
      const double2 a01 = As[(2 * ks) * 32 + lane], a23 = As[(2 * ks + 1) * 32 + lane];
      const double af[4] = {a01.x, a01.y, a23.x, a23.y};
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
    }
    __syncwarp();
    double* out = A + (int64_t)(S * i) * lda + S * j;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        const int row = 8 * mi + lr, col = 8 * ni + 2 * lk;
        const double2 v = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
        *reinterpret_cast<double2*>(B + row * LD + col) = v;
        stg2(out + (int64_t)row * lda + col, v);
      }
    __syncwarp();
  }
}

// Host: detection, then both kernels, on `st`. n_pad % 32 == 0; ws holds
// ws_doubles(n_pad) per matrix; nonband (batch ints) filled by band_detect().
int band_detect(const uint32_t* bits, int64_t n, int64_t batch, int* nonband, cudaStream_t st) {
  if (cudaMemsetAsync(nonband, 0, sizeof(int) * (size_t)batch, st) != cudaSuccess) return RDB_ECUDA;
  const int64_t want = (batch * n * ((n + 31) / 32) / 4 + 255) / 256;
  band_detect_bits_kernel<<<(unsigned)(want < 148 * 8 ? (want > 0 ? want : 1) : 148 * 8), 256, 0, st>>>(bits, n, batch,
                                                                                                    nonband);
  RDB_LAUNCH_CHECK();
  return RDB_OK;
}

int band_invert(double* a, int64_t n_pad, int64_t lda, int64_t stride, int64_t batch, const int* nonband,
                double* ws, rdb_pivot_info* info, cudaStream_t st) {
  if (n_pad % S || n_pad / S < 2) return RDB_EINVAL;
  static DeviceFlags attr;
  const int attr_dev = current_device();
  if (!attr.get(attr_dev)) {
    if (cudaFuncSetAttribute(band_factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(FactorSmem)) != cudaSuccess ||
        cudaFuncSetAttribute(band_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CHAIN_SMEM) !=
            cudaSuccess)
      return RDB_ECUDA;
    attr.set(attr_dev);
  }
  const int nb = (int)(n_pad / S);
  band_factor_kernel<<<(unsigned)((batch + GPC - 1) / GPC), 256 * GPC, sizeof(FactorSmem), st>>>(
      a, lda, stride, nb, batch, nonband, ws, info);
  band_chain_kernel<<<dim3((unsigned)((nb + CW - 1) / CW), (unsigned)batch), CW * 32, CHAIN_SMEM, st>>>(a, lda, stride, nb,
                                                                                            nonband, ws, info);
  RDB_LAUNCH_CHECK();
  return RDB_OK;
}

}  // namespace rdb

#ifdef RDB_TRACE
namespace rdb {
namespace band {
int trace_attach(void* buf, unsigned cap) { return trace::attach(buf, cap); }
unsigned trace_count() { return trace::count(); }
}  // namespace band
}  // namespace rdb
#endif
