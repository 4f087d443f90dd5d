// Factor packing (G7) and the matvec hot path (S7-S10).
//
// HBM layout:
//   U leaf panel (level l, served leaf L, level-l ancestor X): column-major mLp x R_X, the
//                                     rows of L of [U_b1 | U_b2 | ...] over the blocks (X, Y),
//                                     Y in I_X ascending; mLp = |L| rounded up to even.  One
//                                     contiguous 16-byte aligned range per (leaf, level).
//   V panel of column box Y         : row-major n_Y x RVp_Y, the columns of the blocks
//                                     (X, Y), X in I_Y ascending (RVp_Y = RV_Y rounded up to
//                                     even).  Row i holds the RV_Y values that multiply x_i.
//   t                               : one value per (block, rank index) in U-column order
//                                     (a row box's t is contiguous); stage A writes it through
//                                     vdst (V-panel column -> t position).
// Matvec (Alg. 2; stage order is free, R18):
//   stage A  t = V^T x          persistent, bulk-TMA pipelined, one work item per
//                               (column box, row chunk), multi-chunk boxes reduced by the
//                               last chunk to finish                  (high-priority stream)
//   stage B  yfar_L = sum_l U_{X_l}[rows of L, :] t_{X_l}
//                               persistent, bulk-TMA pipelined, one item per leaf (row block)
//   p2p      ynear = K_near x   three deterministic slots             (low-priority stream,
//                               co-resident with A and B: they leave it registers and smem)
//   combine  y = yfar + scale * ynear + shift * x, permuted to the caller's order.
#include <algorithm>
#include <cstdlib>
#include <numeric>
#include <type_traits>

#include "h2d_internal.cuh"
#include "stages.cuh"
#include "pairs.cuh"

namespace h2d {
namespace {

constexpr int64_t kATargetDefault = 1048576;  // stage-A elements per work item (8 MB)
constexpr int kAMaxRows = 16384;     // rows per stage-A item
constexpr int kBRows = 224;          // rows per stage-B item (leaf row block) <= kCons
constexpr int kT1Max = kT1Smem;      // symmetric stage B': widest first-side panel (its t1 rides in the slot)
// stage B' ring: 2 x 44 KB slots.  The fused column-sum + row-dot pass is issue-bound, not
// latency-bound (the second CTA on the SM hides the copy latency), so fewer, larger stages
// win by amortising the per-stage overhead: A'+B' 2.20 ms (5 x 16 KB) -> 1.76 ms (C3).
#ifndef H2D_NS_DUAL
#define H2D_NS_DUAL 2
#define H2D_SD_DUAL 5632
#endif
constexpr int kNSDual = H2D_NS_DUAL, kSDDual = H2D_SD_DUAL;   // (4 x 2816 / 3 x 4096 / 3 x 3584 measured slower: C3 symmetric 406 -> 390 / 402 / 400 per s)

struct UCopyItem {
  const double* src;   // column-major, leading dimension ld_src
  double* dst;         // column-major, leading dimension ld_dst
  int32_t ld_src, ld_dst, rows, cols;
};
__global__ void ucopy_kernel(const UCopyItem* __restrict__ items) {
  const UCopyItem it = items[blockIdx.x];
  const int64_t tot = (int64_t)it.rows * it.cols;
  for (int64_t e = threadIdx.x; e < tot; e += blockDim.x) {
    const int64_t c = e / it.rows, i = e - c * it.rows;
    it.dst[c * it.ld_dst + i] = it.src[c * it.ld_src + i];
  }
}

struct VPackItem {
  const double* src;  // column-major n x r
  double* dst;        // row-major panel, first column of the block
  int32_t n, r, ld;
  int32_t pad;
};
__global__ void vpack_kernel(const VPackItem* __restrict__ items) {
  const VPackItem it = items[blockIdx.x];
  const int64_t tot = (int64_t)it.n * it.r;
  for (int64_t e = threadIdx.x; e < tot; e += blockDim.x) {
    int64_t j = e / it.r, q = e - j * it.r;
    it.dst[j * it.ld + q] = it.src[j + q * it.n];
  }
}

template <class T>
T* upload_tmp(const std::vector<T>& v, cudaStream_t s) {
  T* p = nullptr;
  H2D_CUDA(cudaMallocAsync(&p, std::max<size_t>(1, v.size()) * sizeof(T), s));
  if (!v.empty())
    H2D_CUDA(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  return p;
}

// ---------------------------------------------------------------- near-field P2P (symmetric)
// Alg. 2 l.4 and l.7: y_X += K(X, X) x_X + sum_{Y in E_X} K(X, Y) x_Y.
// Every configured kernel is symmetric, so each unordered leaf pair is evaluated
// once: the CTA of leaf X evaluates its self block (i < j, plus the diagonal) and the
// blocks with its +x and +y edge neighbours (Morton codes grow with each coordinate, so
// those are the higher-numbered sharers).  Contributions land in three slots per row,
// each row slot having exactly one writer CTA (deterministic, no atomics):
//   s0[r] : row r's own CTA (self block + its +x/+y blocks, both orientations of self)
//   sL[r] : written by the -x neighbour's CTA (K(X_left, X)^T x_left)
//   sD[r] : written by the -y neighbour's CTA
// Stage B adds shift x + scale (s0 + sL + sD).  Neighbours outside the rank's served
// leaves are evaluated one-sidedly by the served leaf (rows only).
// Thread (ti, tj) of a 16 x 16 grid owns the 4 x 4 micro-tile rows ti + 16a, columns
// tj + 16b of a 64 x 64 super-tile: 16 independent kernel evaluations per super-tile with
// the 8 point coordinates and x values held in registers.
constexpr int kSymRowsOnly = 0, kSymBoth = 1, kSymSelf = 2;

template <int KID>
__device__ __forceinline__ double p2p_eval(const KernelParams& kp, const double2* tab, double px,
                                           double py, double qx, double qy) {
  if (KID == H2D_KERNEL_LOG || KID == kLogSafe || KID == kLogNoSel || KID == kLogNoSelRepl) {
    const double dx = px - qx, dy = py - qy;
    const double r2 = fma(dx, dx, dy * dy);
    return r2 > 0.0 ? hlog_r2<KID == kLogSafe, KID == kLogNoSelRepl>(r2, tab) : 0.0;
  }
  return kernel_eval_t<KID>(kp, px, py, qx, qy);
}

// Fast tile (distance kernels, both tiles <= 96 points, already in shared memory as
// [px | py | x] x 96): thread (ti, tj) of the 16 x 16 grid owns rows ti + 16 a and columns
// tj + 16 b; its columns live in registers, rows are read from smem once per row.  Every
// pair is evaluated branch-free; rows / columns beyond the tile carry zero weights.  DIAG:
// the self block, pairs i < j only (both orientations) plus K0 x_i on the diagonal.
template <int KID, bool DIAG>
__device__ __forceinline__ void tile_fast(int mt, int nt, const double* __restrict__ sa,
                                          const double* __restrict__ sb, const double2* __restrict__ tab,
                                          const KernelParams& kp, double k0, double* srow,
                                          double (*scol)[kSymTile + 1]) {
  const int tid = threadIdx.x, ti = tid >> 4, tj = tid & 15;
  const int A = (mt + 15) >> 4, B = (nt + 15) >> 4;
  double cpx[kSymMaxB], cpy[kSymMaxB], cxv[kSymMaxB], cacc[kSymMaxB];
#pragma unroll
  for (int bb = 0; bb < kSymMaxB; ++bb) {
    const int j = tj + 16 * bb;
    const bool vj = j < nt;
    cpx[bb] = vj ? sb[j] : 0.0;
    cpy[bb] = vj ? sb[kSymTile + j] : 0.0;
    cxv[bb] = vj ? sb[2 * kSymTile + j] : 0.0;
    cacc[bb] = 0.0;
  }
  for (int aa = 0; aa < A; ++aa) {
    const int i = ti + 16 * aa;
    const bool vi = i < mt;
    const double rpx = vi ? sa[i] : 0.0, rpy = vi ? sa[kSymTile + i] : 0.0;
    const double rx = vi ? sa[2 * kSymTile + i] : 0.0;
    double racc = 0.0;
#pragma unroll
    for (int bb = 0; bb < kSymMaxB; ++bb) {
      if (bb < B) {
        const double dx = rpx - cpx[bb], dy = rpy - cpy[bb];
        double k = kfast<KID>(fma(dx, dx, dy * dy), tab, kp);
        if (DIAG) k = i < tj + 16 * bb ? k : 0.0;
        racc = fma(k, cxv[bb], racc);
        cacc[bb] = fma(k, rx, cacc[bb]);
      }
    }
    if (DIAG && tj == 0) racc = fma(k0, rx, racc);
    racc += __shfl_xor_sync(0xffffffffu, racc, 8);
    racc += __shfl_xor_sync(0xffffffffu, racc, 4);
    racc += __shfl_xor_sync(0xffffffffu, racc, 2);
    racc += __shfl_xor_sync(0xffffffffu, racc, 1);
    if (tj == 0 && vi) srow[i] = racc;
  }
#pragma unroll
  for (int bb = 0; bb < kSymMaxB; ++bb)
    if (bb < B) scol[ti][tj + 16 * bb] = cacc[bb];
}

// Fold a fast tile's row sums into row_dst and (unless null) its column sums into col_dst.
__device__ __forceinline__ void tile_flush(int mt, int nt, double* row_dst, double* col_dst,
                                           const double* srow, double (*scol)[kSymTile + 1]) {
  const int tid = threadIdx.x;
  __syncthreads();
  if (tid < mt) row_dst[tid] += srow[tid];
  if (col_dst && tid < nt) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += scol[k][tid];
    col_dst[tid] += s;
  }
  __syncthreads();
}

// One leaf-pair block on a 16 x 16 thread grid: thread (ti, tj) owns rows ti + 16a
// (a < A = ceil(m/16)) and columns tj + 16b (b < B = ceil(n/16)) of a super-tile of up to
// 96 x 96 points (a leaf of the configs fits one super-tile; larger blocks loop).  Row
// points live in registers one row at a time, column points are read from shared memory,
// column sums stay in registers (cacc[b]), row sums are reduced over tj by shuffles.
template <int KID>
__device__ __noinline__ void sym_block(int mode, int64_t a0, int m, int64_t b0, int n, double* row_dst,
                          double* col_dst, const double* __restrict__ px,
                          const double* __restrict__ py, const double* __restrict__ x,
                          const KernelParams& kp, const double2* tab, double* s_a, double* s_b,
                          double (*scol)[kSymTile + 1], double* srow) {
  const int tid = threadIdx.x, ti = tid >> 4, tj = tid & 15;
  for (int ra = 0; ra < m; ra += kSymTile) {
    const int mt = min(kSymTile, m - ra);
    const int A = (mt + 15) >> 4;
    const int cstart = mode == kSymSelf ? ra : 0;
    for (int cb = cstart; cb < n; cb += kSymTile) {
      const int nt = min(kSymTile, n - cb);
      const int B = (nt + 15) >> 4;
      __syncthreads();
      for (int e = tid; e < mt; e += 256) {
        s_a[e] = px[a0 + ra + e];
        s_a[kSymTile + e] = py[a0 + ra + e];
        s_a[2 * kSymTile + e] = x[a0 + ra + e];
      }
      for (int e = tid; e < nt; e += 256) {
        s_b[e] = px[b0 + cb + e];
        s_b[kSymTile + e] = py[b0 + cb + e];
        s_b[2 * kSymTile + e] = x[b0 + cb + e];
      }
      __syncthreads();
      const bool diag_tile = mode == kSymSelf && cb == ra;
      // this thread's columns tj + 16 bb live in registers for the whole tile
      double cpx[kSymMaxB], cpy[kSymMaxB], cxv[kSymMaxB], cacc[kSymMaxB];
#pragma unroll
      for (int bb = 0; bb < kSymMaxB; ++bb) {
        const int j = tj + 16 * bb;
        const bool vj = bb < B && j < nt;
        cpx[bb] = vj ? s_b[j] : 0.0;
        cpy[bb] = vj ? s_b[kSymTile + j] : 0.0;
        cxv[bb] = vj ? s_b[2 * kSymTile + j] : 0.0;
        cacc[bb] = 0.0;
      }
      for (int aa = 0; aa < A; ++aa) {
        const int i = ti + 16 * aa;
        const bool vi = i < mt;
        const double rpx = s_a[i], rpy = s_a[kSymTile + i], rx = vi ? s_a[2 * kSymTile + i] : 0.0;
        double racc = 0.0;
#pragma unroll
        for (int bb = 0; bb < kSymMaxB; ++bb) {
          const int j = tj + 16 * bb;
          if (bb < B) {
            bool ok = vi && j < nt;
            if (diag_tile) ok = ok && i <= j;
            if (ok) {
              const double k = p2p_eval<KID>(kp, tab, rpx, rpy, cpx[bb], cpy[bb]);
              racc = fma(k, cxv[bb], racc);
              if (!(diag_tile && i == j)) cacc[bb] = fma(k, rx, cacc[bb]);
            }
          }
        }
        racc += __shfl_xor_sync(0xffffffffu, racc, 8);
        racc += __shfl_xor_sync(0xffffffffu, racc, 4);
        racc += __shfl_xor_sync(0xffffffffu, racc, 2);
        racc += __shfl_xor_sync(0xffffffffu, racc, 1);
        if (tj == 0 && vi) srow[i] = racc;
      }
      if (mode != kSymRowsOnly) {
#pragma unroll
        for (int bb = 0; bb < kSymMaxB; ++bb)
          if (bb < B) scol[ti][tj + 16 * bb] = cacc[bb];
      }
      __syncthreads();
      if (tid < mt) row_dst[ra + tid] += srow[tid];
      if (mode != kSymRowsOnly) {
        __syncthreads();   // self blocks: row and column targets may coincide
        if (tid < nt) {
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < 16; ++k) s += scol[k][tid];
          col_dst[cb + tid] += s;
        }
      }
    }
  }
}

template <int KID>
__global__ void __launch_bounds__(256, 3)
p2p_sym_kernel(int kappa, int64_t leaf_begin, int64_t leaf_end, const int32_t* __restrict__ leaves,
               const int32_t* __restrict__ leaf_start, const double* __restrict__ px,
               const double* __restrict__ py, const double* __restrict__ x, KernelParams kp,
               double* __restrict__ s0, double* __restrict__ sL, double* __restrict__ sD) {
  __shared__ double s_a[3 * kSymTile], s_b[3 * kSymTile], s_c[3 * kSymTile], srow[kSymTile];
  __shared__ double scol[16][kSymTile + 1];
  __shared__ double2 s_logtab[kHlogBins];
  const int64_t X = leaves[blockIdx.x];
  const int tid = threadIdx.x;
  if (kNeedsLogTable<KID>) hlog_table<KID>(s_logtab);
  const uint32_t cx = p2p_compact((uint32_t)X), cy = p2p_compact((uint32_t)X >> 1);
  const uint32_t side = 1u << kappa;
  const int64_t xs = leaf_start[X];
  const int m = leaf_start[X + 1] - (int)xs;
  auto served = [&](int64_t Y) { return Y >= leaf_begin && Y < leaf_end; };
  const bool has_r = cx + 1 < side, has_u = cy + 1 < side, has_l = cx > 0, has_d = cy > 0;
  const int64_t Rn = has_r ? (int64_t)(p2p_spread(cx + 1) | (p2p_spread(cy) << 1)) : -1;
  const int64_t Un = has_u ? (int64_t)(p2p_spread(cx) | (p2p_spread(cy + 1) << 1)) : -1;
  const int64_t Ln = has_l ? (int64_t)(p2p_spread(cx - 1) | (p2p_spread(cy) << 1)) : -1;
  const int64_t Dn = has_d ? (int64_t)(p2p_spread(cx) | (p2p_spread(cy - 1) << 1)) : -1;
  const bool do_r = has_r && served(Rn), do_u = has_u && served(Un);
  const bool own_l = !has_l || !served(Ln), own_d = !has_d || !served(Dn);
  int64_t rs = 0, us = 0;
  int rn = 0, un = 0;
  if (has_r) { rs = leaf_start[Rn]; rn = leaf_start[Rn + 1] - (int)rs; }
  if (has_u) { us = leaf_start[Un]; un = leaf_start[Un + 1] - (int)us; }
  // phase 0: zero every slot row this CTA is the writer of
  for (int i = tid; i < m; i += 256) {
    s0[xs + i] = 0.0;
    if (own_l) sL[xs + i] = 0.0;
    if (own_d) sD[xs + i] = 0.0;
  }
  if (do_r)
    for (int i = tid; i < rn; i += 256) sL[rs + i] = 0.0;
  if (do_u)
    for (int i = tid; i < un; i += 256) sD[us + i] = 0.0;
  if (m == 0) return;
  constexpr bool kDist = kDistKernel<KID>;
  int first_task = 0;
  if (kDist && m <= kSymTile && rn <= kSymTile && un <= kSymTile) {
    // fast path: the self, +x and +y tiles are loaded together (one memory latency), then
    // evaluated branch-free; only rows-only partners (rank boundaries) take the generic path
    for (int e = tid; e < 3 * kSymTile; e += 256) {
      const int a = e / kSymTile, i = e - a * kSymTile;
      const double* src = a == 0 ? px : a == 1 ? py : x;
      if (i < m) s_a[e] = src[xs + i];
      if (i < rn) s_b[e] = src[rs + i];
      if (i < un) s_c[e] = src[us + i];
    }
    __syncthreads();
    const double k0 = KID == H2D_KERNEL_IMQ ? 1.0 : 0.0;
    tile_fast<KID, true>(m, m, s_a, s_a, s_logtab, kp, k0, srow, scol);
    tile_flush(m, m, s0 + xs, s0 + xs, srow, scol);
    if (has_r) {
      tile_fast<KID, false>(m, rn, s_a, s_b, s_logtab, kp, k0, srow, scol);
      tile_flush(m, rn, s0 + xs, do_r ? sL + rs : nullptr, srow, scol);
    }
    if (has_u) {
      tile_fast<KID, false>(m, un, s_a, s_c, s_logtab, kp, k0, srow, scol);
      tile_flush(m, un, s0 + xs, do_u ? sD + us : nullptr, srow, scol);
    }
    first_task = 3;
  }
  // generic path: blocks in a fixed order (one code instance: keeps the I-cache small)
  for (int task = first_task; task < 5; ++task) {
    int mode = kSymRowsOnly, n = 0;
    int64_t b0 = 0;
    double *rdst = s0 + xs, *cdst = nullptr;
    if (task == 0) { mode = kSymSelf; b0 = xs; n = m; cdst = s0 + xs; }
    else if (task == 1) {
      if (!has_r) continue;
      mode = do_r ? kSymBoth : kSymRowsOnly; b0 = rs; n = rn; cdst = sL + rs;
    } else if (task == 2) {
      if (!has_u) continue;
      mode = do_u ? kSymBoth : kSymRowsOnly; b0 = us; n = un; cdst = sD + us;
    } else if (task == 3) {
      if (!(has_l && own_l)) continue;
      b0 = leaf_start[Ln]; n = leaf_start[Ln + 1] - (int)b0; rdst = sL + xs;
    } else {
      if (!(has_d && own_d)) continue;
      b0 = leaf_start[Dn]; n = leaf_start[Dn + 1] - (int)b0; rdst = sD + xs;
    }
    sym_block<KID>(mode, xs, m, b0, n, rdst, cdst, px, py, x, kp, s_logtab, s_a, s_b, scol, srow);
  }
}

// ---------------------------------------------------------------- persistent fast P2P
// The same slot protocol as p2p_sym_kernel for the leaves whose whole near field is served
// by this handle and fits the fast tile (self, +x and +y neighbour <= 96 points; distance
// kernels).  One CTA per SM loops over its leaves (atomic counter); the next leaf's three
// tiles are prefetched with cp.async while the current one is evaluated, the leaf's own
// rows are accumulated in shared memory and every slot row is written exactly once (no
// global read-modify-write): s0[X] = self + (+x rows) + (+y rows), sL[R] and sD[U] = the
// neighbour columns, sL[X] / sD[X] = 0 on the domain boundary.
struct P2PMeta {
  int64_t xs, rs, us;
  int m, rn, un;
  int has_r, has_u, has_l, has_d;
};

__device__ __forceinline__ P2PMeta p2p_meta(int kappa, int64_t X, const int32_t* __restrict__ leaf_start) {
  P2PMeta M{};
  const uint32_t cx = p2p_compact((uint32_t)X), cy = p2p_compact((uint32_t)X >> 1);
  const uint32_t side = 1u << kappa;
  M.has_r = cx + 1 < side;
  M.has_u = cy + 1 < side;
  M.has_l = cx > 0;
  M.has_d = cy > 0;
  M.xs = leaf_start[X];
  M.m = leaf_start[X + 1] - (int)M.xs;
  if (M.has_r) {
    const int64_t Rn = (int64_t)(p2p_spread(cx + 1) | (p2p_spread(cy) << 1));
    M.rs = leaf_start[Rn];
    M.rn = leaf_start[Rn + 1] - (int)M.rs;
  }
  if (M.has_u) {
    const int64_t Un = (int64_t)(p2p_spread(cx) | (p2p_spread(cy + 1) << 1));
    M.us = leaf_start[Un];
    M.un = leaf_start[Un + 1] - (int)M.us;
  }
  return M;
}

__device__ __forceinline__ void p2p_prefetch(const P2PMeta& M, double (*T)[3 * kSymTile],
                                             const double* __restrict__ px, const double* __restrict__ py,
                                             const double* __restrict__ x) {
  for (int e = threadIdx.x; e < 3 * kSymTile; e += blockDim.x) {
    const int a = e / kSymTile, i = e - a * kSymTile;
    const double* src = a == 0 ? px : a == 1 ? py : x;
    if (i < M.m) cp_async8(&T[0][e], src + M.xs + i);
    if (i < M.rn) cp_async8(&T[1][e], src + M.rs + i);
    if (i < M.un) cp_async8(&T[2][e], src + M.us + i);
  }
}

// tile_fast with the column sums reduced over the warp's two thread rows by a shuffle and
// stored per warp: scol8[w][j].
template <int KID, bool DIAG>
__device__ __forceinline__ void tile_fast8(int mt, int nt, const double* __restrict__ sa,
                                           const double* __restrict__ sb, const double2* __restrict__ tab,
                                           const KernelParams& kp, double k0, double* srow,
                                           double (*scol8)[kSymTile + 1]) {
  const int tid = threadIdx.x, ti = tid >> 4, tj = tid & 15;
  const int A = (mt + 15) >> 4, B = (nt + 15) >> 4;
  double cpx[kSymMaxB], cpy[kSymMaxB], cxv[kSymMaxB], cacc[kSymMaxB];
#pragma unroll
  for (int bb = 0; bb < kSymMaxB; ++bb) {
    const int j = tj + 16 * bb;
    const bool vj = j < nt;
    cpx[bb] = vj ? sb[j] : 0.0;
    cpy[bb] = vj ? sb[kSymTile + j] : 0.0;
    cxv[bb] = vj ? sb[2 * kSymTile + j] : 0.0;
    cacc[bb] = 0.0;
  }
  // two rows (i, i + 16) per pass: 2 B independent evaluations in flight per thread (the
  // kernel runs at 8 warps per SM beside the streaming CTAs, so ILP is its latency cover)
  for (int aa = 0; aa < A; aa += 2) {
    const int i0 = ti + 16 * aa, i1 = i0 + 16;
    const bool v0 = i0 < mt, v1 = i1 < mt && aa + 1 < A;
    const double px0 = v0 ? sa[i0] : 0.0, py0 = v0 ? sa[kSymTile + i0] : 0.0, x0 = v0 ? sa[2 * kSymTile + i0] : 0.0;
    const double px1 = v1 ? sa[i1] : 0.0, py1 = v1 ? sa[kSymTile + i1] : 0.0, x1 = v1 ? sa[2 * kSymTile + i1] : 0.0;
    double r0 = 0.0, r1 = 0.0;
#pragma unroll
    for (int bb = 0; bb < kSymMaxB; ++bb) {
      // self block: column block bb < aa lies wholly below the diagonal (i >= 16 aa > j), as
      // does bb = aa for the second row (warp-uniform skips, no evaluation)
      if (bb < B && (!DIAG || bb >= aa)) {
        const double dx0 = px0 - cpx[bb], dy0 = py0 - cpy[bb];
        double k0v = kfast<KID>(fma(dx0, dx0, dy0 * dy0), tab, kp);
        if (DIAG) k0v = i0 < tj + 16 * bb ? k0v : 0.0;
        r0 = fma(k0v, cxv[bb], r0);
        cacc[bb] = fma(k0v, x0, cacc[bb]);
        if (!DIAG || bb > aa) {
          const double dx1 = px1 - cpx[bb], dy1 = py1 - cpy[bb];
          double k1v = kfast<KID>(fma(dx1, dx1, dy1 * dy1), tab, kp);
          if (DIAG) k1v = i1 < tj + 16 * bb ? k1v : 0.0;
          r1 = fma(k1v, cxv[bb], r1);
          cacc[bb] = fma(k1v, x1, cacc[bb]);
        }
      }
    }
    if (DIAG && tj == 0) {
      r0 = fma(k0, x0, r0);
      r1 = fma(k0, x1, r1);
    }
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) {
      r0 += __shfl_xor_sync(0xffffffffu, r0, o);
      r1 += __shfl_xor_sync(0xffffffffu, r1, o);
    }
    if (tj == 0 && v0) srow[i0] = r0;
    if (tj == 0 && v1) srow[i1] = r1;
  }
  const int w = tid >> 5;
#pragma unroll
  for (int bb = 0; bb < kSymMaxB; ++bb) {
    if (bb < B) {
      const double v = cacc[bb] + __shfl_xor_sync(0xffffffffu, cacc[bb], 16);
      if ((tid & 16) == 0) scol8[w][tj + 16 * bb] = v;
    }
  }
}

__device__ __forceinline__ double colsum8(double (*scol8)[kSymTile + 1], int j) {
  return ((scol8[0][j] + scol8[1][j]) + (scol8[2][j] + scol8[3][j])) +
         ((scol8[4][j] + scol8[5][j]) + (scol8[6][j] + scol8[7][j]));
}

template <int KID>
__global__ void __launch_bounds__(256, 3)
p2p_fast_kernel(int kappa, const int32_t* __restrict__ leaves, int n_leaves, int32_t* counter,
                const int32_t* __restrict__ leaf_start, const double* __restrict__ px,
                const double* __restrict__ py, const double* __restrict__ x, KernelParams kp,
                double* __restrict__ s0, double* __restrict__ sL, double* __restrict__ sD) {
  __shared__ double tiles[2][3][3 * kSymTile];   // [buffer][X, +x, +y][px | py | x]
  __shared__ double acc[kSymTile], srow[kSymTile];
  __shared__ double scol8[8][kSymTile + 1];
  __shared__ double2 tab[kHlogBins];
  __shared__ int s_next;
  const int tid = threadIdx.x;
  const double k0 = KID == H2D_KERNEL_IMQ ? 1.0 : 0.0;
  if (kNeedsLogTable<KID>) hlog_table<KID>(tab);
  if (tid == 0) s_next = atomicAdd(counter, 1);
  __syncthreads();
  int cur = s_next;
  P2PMeta Mc{};
  if (cur < n_leaves) {
    Mc = p2p_meta(kappa, leaves[cur], leaf_start);
    p2p_prefetch(Mc, tiles[0], px, py, x);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  int b = 0;
  while (cur < n_leaves) {
    __syncthreads();                      // s_next consumed, buffer b ^ 1 free
    if (tid == 0) s_next = atomicAdd(counter, 1);
    __syncthreads();
    const int nxt = s_next;
    P2PMeta Mn{};
    if (nxt < n_leaves) {
      Mn = p2p_meta(kappa, leaves[nxt], leaf_start);
      p2p_prefetch(Mn, tiles[b ^ 1], px, py, x);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");   // this leaf's tiles have landed
    __syncthreads();
    const double* TX = tiles[b][0];
    const int m = Mc.m;
    // self block
    tile_fast8<KID, true>(m, m, TX, TX, tab, kp, k0, srow, scol8);
    __syncthreads();
    if (tid < m) acc[tid] = srow[tid] + colsum8(scol8, tid);
    __syncthreads();
    if (Mc.has_r) {
      tile_fast8<KID, false>(m, Mc.rn, TX, tiles[b][1], tab, kp, k0, srow, scol8);
      __syncthreads();
      if (tid < m) acc[tid] += srow[tid];
      if (tid < Mc.rn) sL[Mc.rs + tid] = colsum8(scol8, tid);
      __syncthreads();
    }
    if (Mc.has_u) {
      tile_fast8<KID, false>(m, Mc.un, TX, tiles[b][2], tab, kp, k0, srow, scol8);
      __syncthreads();
      if (tid < m) acc[tid] += srow[tid];
      if (tid < Mc.un) sD[Mc.us + tid] = colsum8(scol8, tid);
    }
    if (tid < m) {
      s0[Mc.xs + tid] = acc[tid];
      if (!Mc.has_l) sL[Mc.xs + tid] = 0.0;
      if (!Mc.has_d) sD[Mc.xs + tid] = 0.0;
    }
    Mc = Mn;
    cur = nxt;
    b ^= 1;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// Warp-per-leaf near field for leaves of <= 96 points: one warp per leaf (atomic counter),
// lane owns rows lane + 32 r (r < RPL = ceil(m / 32)); no block barriers, so 8 leaves per
// CTA proceed independently (the CTA kernel's six barriers per leaf made it latency-bound:
// C3 P2P 1.21 -> 0.64 ms standalone, FP64 fraction 0.14 -> 0.26).  The leaf's points are
// staged in the warp's smem.  Self block: row sums over all m x m pairs (a third more
// evaluations than the symmetric CTA kernel, no column sums).  +x / +y neighbour (any size,
// 32-point chunks, 8 columns at a time): row sums in registers, the 8 column sums of the
// group (over all RPL rows) by a transposed butterfly (9 double shuffles; lane 4t ends up
// holding column t).  Same slots as p2p_fast_kernel: s0 (own rows), sL / sD (the
// neighbour's rows), one writer per value.
// Adaptive near field (R24): warp per (leaf, 64-row pass); the leaf's dense column ranges
// (its own blocks and its subdivided ancestors' blocks against leaf neighbours) stream through
// a per-warp shared-memory tile of 32 points; lane owns rows lane and lane + 32; one writer
// per row (slot s0), no atomics.  item = (leaf << 8) | pass.
template <int KID>
__global__ void __launch_bounds__(256, 3)
p2p_list_kernel(const int64_t* __restrict__ items, int n_items, int32_t* counter,
                const int32_t* __restrict__ lf_start, const int64_t* __restrict__ nf_off,
                const int64_t* __restrict__ nf_rng, const double* __restrict__ px,
                const double* __restrict__ py, const double* __restrict__ x, KernelParams kp,
                double* __restrict__ s0) {
  __shared__ double2 sq[8][32];
  __shared__ double sxv[8][32];
  __shared__ double2 tab[kHlogBins];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (kNeedsLogTable<KID>) hlog_table<KID>(tab);
  __syncthreads();
  for (;;) {
    int idx = 0;
    if (lane == 0) idx = atomicAdd(counter, 1);
    idx = __shfl_sync(0xffffffffu, idx, 0);
    if (idx >= n_items) break;
    const int64_t it = items[idx];
    const int64_t lf = it >> 8;
    const int64_t xs = (int64_t)lf_start[lf] + 64 * (it & 255);
    const int m = (int)min((int64_t)64, (int64_t)lf_start[lf + 1] - xs);
    if (m <= 32) {
      // small pass (the adaptive tree's typical leaf): G = 32 / S column groups of S >= m
      // lanes, lane = (group g, row i); the groups take every G-th column of a tile and
      // their row sums meet by xor shuffles (the two-row mapping evaluated 64 rows per pass)
      const int S = m <= 8 ? 8 : m <= 16 ? 16 : 32;
      const int G = 32 / S, g = lane / S, i = lane - g * S;
      const double pr = i < m ? px[xs + i] : 0.0, qr = i < m ? py[xs + i] : 0.0;
      double a = 0.0;
      for (int64_t e = nf_off[lf]; e < nf_off[lf + 1]; ++e) {
        const int64_t c0 = nf_rng[2 * e], cnt = nf_rng[2 * e + 1];
        for (int64_t t = 0; t < cnt; t += 32) {
          const int64_t j = t + lane;
          __syncwarp();
          sq[w][lane] = j < cnt ? make_double2(px[c0 + j], py[c0 + j]) : make_double2(0.0, 0.0);
          sxv[w][lane] = j < cnt ? x[c0 + j] : 0.0;
          __syncwarp();
          const int nt = (int)min((int64_t)32, cnt - t);
          for (int jj = g; jj < nt; jj += G) {
            const double2 q = sq[w][jj];
            double k;
            if constexpr (kDistKernel<KID>) {
              const double dx = pr - q.x, dy = qr - q.y;
              k = kfast<KID>(fma(dx, dx, dy * dy), tab, kp);
            } else {
              k = kernel_eval_t<KID>(kp, pr, qr, q.x, q.y);
            }
            a = fma(k, sxv[w][jj], a);
          }
        }
      }
      if (G >= 4) a += __shfl_xor_sync(0xffffffffu, a, 8);
      if (G >= 2) a += __shfl_xor_sync(0xffffffffu, a, 16);
      if (g == 0 && i < m) s0[xs + i] = a;
      continue;
    }
    double pi[2], qi[2], acc[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int i = lane + 32 * r;
      pi[r] = i < m ? px[xs + i] : 0.0;
      qi[r] = i < m ? py[xs + i] : 0.0;
      acc[r] = 0.0;
    }
    for (int64_t e = nf_off[lf]; e < nf_off[lf + 1]; ++e) {
      const int64_t c0 = nf_rng[2 * e], cnt = nf_rng[2 * e + 1];
      for (int64_t t = 0; t < cnt; t += 32) {
        const int64_t j = t + lane;
        __syncwarp();
        sq[w][lane] = j < cnt ? make_double2(px[c0 + j], py[c0 + j]) : make_double2(0.0, 0.0);
        sxv[w][lane] = j < cnt ? x[c0 + j] : 0.0;
        __syncwarp();
        const int nt = (int)min((int64_t)32, cnt - t);
        for (int jj = 0; jj < nt; ++jj) {
          const double2 q = sq[w][jj];
          const double xj = sxv[w][jj];
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            double k;
            if constexpr (kDistKernel<KID>) {
              const double dx = pi[r] - q.x, dy = qi[r] - q.y;
              k = kfast<KID>(fma(dx, dx, dy * dy), tab, kp);
            } else {
              k = kernel_eval_t<KID>(kp, pi[r], qi[r], q.x, q.y);
            }
            acc[r] = fma(k, xj, acc[r]);
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r)
      if (lane + 32 * r < m) s0[xs + lane + 32 * r] = acc[r];
  }
}

// Near-field pairs of distinct points with a subnormal r^2 (closer than ~1.5e-154): sets
// *flag, and the handle's near field then runs the subnormal-safe table log (kLogSafe).  A
// CTA per leaf (grid-stride), every (row, column) of the leaf's dense column ranges: the
// self leaf and the edge neighbours (balanced), or the adaptive ranges (nf_off != nullptr).
__global__ void subnormal_check_kernel(int kappa, int64_t nleaf, const int32_t* __restrict__ lstart,
                                       const int64_t* __restrict__ nf_off, const int64_t* __restrict__ nf_rng,
                                       const double* __restrict__ px, const double* __restrict__ py, int* flag) {
  __shared__ int64_t rb[5], rc[5];
  __shared__ int nr;
  for (int64_t L = blockIdx.x; L < nleaf; L += gridDim.x) {
    if (threadIdx.x == 0) {
      nr = 0;
      if (nf_off) {
        for (int64_t e = nf_off[L]; e < nf_off[L + 1] && nr < 5; ++e) { rb[nr] = nf_rng[2 * e]; rc[nr] = nf_rng[2 * e + 1]; ++nr; }
      } else {
        const uint32_t cx = p2p_compact((uint32_t)L), cy = p2p_compact((uint32_t)L >> 1), side = 1u << kappa;
        const int dxs[5] = {0, 1, -1, 0, 0}, dys[5] = {0, 0, 0, 1, -1};
        for (int k = 0; k < 5; ++k) {
          const int64_t qx = (int64_t)cx + dxs[k], qy = (int64_t)cy + dys[k];
          if (qx < 0 || qy < 0 || qx >= side || qy >= side) continue;
          const int64_t Y = (int64_t)(p2p_spread((uint32_t)qx) | (p2p_spread((uint32_t)qy) << 1));
          rb[nr] = lstart[Y];
          rc[nr] = lstart[Y + 1] - lstart[Y];
          ++nr;
        }
      }
    }
    __syncthreads();
    const int64_t s0 = nf_off ? lstart[L] : lstart[L];
    const int64_t m = lstart[L + 1] - s0;
    bool bad = false, same = false;
    for (int64_t i = s0 + threadIdx.x; i < s0 + m; i += blockDim.x) {
      const double xi = px[i], yi = py[i];
      for (int k = 0; k < nr; ++k)
        for (int64_t j = rb[k]; j < rb[k] + rc[k]; ++j) {
          const double dx = xi - px[j], dy = yi - py[j];
          const double r2 = fma(dx, dx, dy * dy);
          bad |= r2 > 0.0 && r2 < 0x1p-1022;
          same |= r2 == 0.0 && j != i;
        }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
    if (__syncthreads_or(same) && threadIdx.x == 0) atomicOr(flag, 2);
  }
}

constexpr int kWarpLeaf = 96;      // rows per lane RPL = ceil(m / 32) <= 3 (leaves <= 96 points)

template <int KID, int RPL>
__device__ __forceinline__ void warp_nbr(int lane, const double (&pi)[RPL], const double (&qi)[RPL],
                                         const double (&xi)[RPL], int n, int64_t nb0, const double* __restrict__ px,
                                         const double* __restrict__ py, const double* __restrict__ x,
                                         double2* __restrict__ spq, double* __restrict__ sx,
                                         const double2* __restrict__ tab, const KernelParams& kp,
                                         double (&acc)[RPL], double* __restrict__ out) {
  for (int cb = 0; cb < n; cb += 32) {
    const int nc = min(32, n - cb);
    __syncwarp();
    // slots past the chunk hold a far dummy point with zero weight, so every group of 8
    // columns runs branch-free (its row sums gain K * 0; its column sums are never written)
    const bool vj = lane < nc;
    spq[lane] = vj ? make_double2(px[nb0 + cb + lane], py[nb0 + cb + lane]) : make_double2(1e30, 1e30);
    sx[lane] = vj ? x[nb0 + cb + lane] : 0.0;
    __syncwarp();
    for (int g = 0; g < nc; g += 8) {
      double c[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int j = g + t;
        c[t] = 0.0;
        const double2 q = spq[j];
        const double xj = sx[j];
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
          const double dx = pi[r] - q.x, dy = qi[r] - q.y;
          const double v = kfast<KID>(fma(dx, dx, dy * dy), tab, kp);
          acc[r] = fma(v, xj, acc[r]);
          c[t] = fma(v, xi[r], c[t]);   // xi = 0 on rows past the leaf
        }
      }
      const double v = warp_transpose_sum8(c, lane);
      const int col = g + (lane >> 2);
      if ((lane & 3) == 0 && col < nc) out[cb + col] = v;
    }
  }
}

#ifndef H2D_P2P_WARP_MINB
#define H2D_P2P_WARP_MINB 3
#endif
template <int KID, int RPL>
__global__ void __launch_bounds__(256, H2D_P2P_WARP_MINB)
p2p_warp_kernel(int kappa, const int32_t* __restrict__ leaves, int n_leaves, int32_t* counter,
                const int32_t* __restrict__ leaf_start, const double* __restrict__ px,
                const double* __restrict__ py, const double* __restrict__ x, KernelParams kp,
                double* __restrict__ s0, double* __restrict__ sL, double* __restrict__ sD) {
  __shared__ double2 sself[8][32 * RPL], snb[8][32];
  __shared__ double xself[8][32 * RPL], xnb[8][32];
  __shared__ double2 tab[kHlogBins];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (kNeedsLogTable<KID>) hlog_table<KID>(tab);
  __syncthreads();
  for (;;) {
    int idx = 0;
    if (lane == 0) idx = atomicAdd(counter, 1);
    idx = __shfl_sync(0xffffffffu, idx, 0);
    if (idx >= n_leaves) break;
    const P2PMeta M = p2p_meta(kappa, leaves[idx], leaf_start);
    double pi[RPL], qi[RPL], xi[RPL], acc[RPL];
    __syncwarp();
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = lane + 32 * r;
      const bool vi = i < M.m;
      pi[r] = vi ? px[M.xs + i] : 0.0;
      qi[r] = vi ? py[M.xs + i] : 0.0;
      xi[r] = vi ? x[M.xs + i] : 0.0;
      acc[r] = 0.0;
      sself[w][i] = make_double2(pi[r], qi[r]);
      xself[w][i] = xi[r];
    }
    __syncwarp();
    for (int j = 0; j < M.m; ++j) {   // self block (K(0) by kfast's r2 = 0 branch)
      const double2 q = sself[w][j];
      const double xj = xself[w][j];
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        const double dx = pi[r] - q.x, dy = qi[r] - q.y;
        acc[r] = fma(kfast<KID>(fma(dx, dx, dy * dy), tab, kp), xj, acc[r]);
      }
    }
    if (KID == kLogNoSel || KID == kLogNoSelRepl) {   // the diagonal (r2 = 0) was evaluated as hlog_r2(0): take it out
      const double g = hlog_r2<false, KID == kLogNoSelRepl>(0.0, tab);
#pragma unroll
      for (int r = 0; r < RPL; ++r) acc[r] = fma(-g, xi[r], acc[r]);
    }
    if (M.has_r)
      warp_nbr<KID, RPL>(lane, pi, qi, xi, M.rn, M.rs, px, py, x, snb[w], xnb[w], tab, kp, acc, sL + M.rs);
    if (M.has_u)
      warp_nbr<KID, RPL>(lane, pi, qi, xi, M.un, M.us, px, py, x, snb[w], xnb[w], tab, kp, acc, sD + M.us);
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = lane + 32 * r;
      if (i < M.m) {
        s0[M.xs + i] = acc[r];
        if (!M.has_l) sL[M.xs + i] = 0.0;
        if (!M.has_d) sD[M.xs + i] = 0.0;
      }
    }
  }
}

// y = yfar + scale (s0 + sL + sD) + shift x over the served rows, in the caller's order.
__global__ void combine_kernel(int64_t row_begin, int64_t rows, const double* __restrict__ yfar,
                               const double* __restrict__ ynear, int64_t n, const double* __restrict__ x,
                               double scale, double shift, double* __restrict__ y,
                               const int32_t* __restrict__ perm, int order_out, int64_t y_row0) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < rows;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = row_begin + k;
    const double s = yfar[k] + fma(scale, (ynear[r] + ynear[n + r]) + ynear[2 * n + r], shift * x[r]);
    if (order_out == H2D_ORDER_ORIGINAL) y[perm[r]] = s;
    else y[r - y_row0] = s;
  }
}

// symmetric apply: y = yfar (C') + sum_l y1[l] (B') + scale ynear + shift x over the served
// rows row_begin + k (yfar is indexed by served row, y1 / ynear / x by TREE row)
__global__ void combine_sym_kernel(int64_t row_begin, int64_t rows, int kappa, const double* __restrict__ yfar,
                                   const double* __restrict__ y1, const double* __restrict__ ynear, int64_t n,
                                   const double* __restrict__ x, double scale, double shift, double* __restrict__ y,
                                   const int32_t* __restrict__ perm, int order_out, int64_t y_row0) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < rows; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = row_begin + k;
    double v = yfar[k];
    for (int l = 0; l < kappa; ++l) v += y1[(int64_t)l * n + r];
    v += fma(scale, (ynear[r] + ynear[n + r]) + ynear[2 * n + r], shift * x[r]);
    if (order_out == H2D_ORDER_ORIGINAL) y[perm[r]] = v;
    else y[r - y_row0] = v;
  }
}

__global__ void permute_in_kernel(const double* __restrict__ x, const int32_t* __restrict__ perm,
                                  int64_t n, double* __restrict__ xt) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n;
       s += (int64_t)gridDim.x * blockDim.x)
    xt[s] = x[perm[s]];
}

// x_tree[s] = xg[r * stride + (s - rows[r])] for the rank r owning TREE row s.
__global__ void unpad_kernel(const double* __restrict__ xg, const int64_t* __restrict__ rows,
                             int world, int64_t stride, int64_t n, double* __restrict__ xt) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n;
       s += (int64_t)gridDim.x * blockDim.x) {
    int r = 0;
    while (r + 1 < world && rows[r + 1] <= s) ++r;
    xt[s] = xg[r * stride + (s - rows[r])];
  }
}

}  // namespace

void unpad_gathered(Handle& h, const double* d_xg, double* d_xtree) {
  int blocks = (int)std::min<int64_t>((h.n + 255) / 256, 148 * 16);
  unpad_kernel<<<blocks, 256, 0, h.stream>>>(d_xg, h.d_rank_rows, h.opts.world, h.gather_stride, h.n,
                                             d_xtree);
  H2D_LAUNCH_CHECK();
}

// Pack one level's factors (per-block sources, column-major U_b m x r and V_b n x r) into
// the U leaf panels and V panels and fill the level's panel metadata.
void pack_level(Handle& h, Level& L, const std::vector<const double*>& srcU,
                const std::vector<const double*>& srcV) {
  cudaStream_t s = h.stream;
  const int l = L.l;
  const int64_t nbox = L.nbox;
  const int sh = 2 * (h.kappa - l);
  // symmetric apply: U leaf panels hold the second-side blocks (row > column box), V box
  // panels the first-side blocks (row < column box); the first-side U factors go to the
  // row-major U box panels Ub below
  const bool sym = h.symapply;
  std::vector<int32_t> rowbox;
  if (sym) {
    rowbox.resize((size_t)L.nblocks);
    for (int64_t X = 0; X < nbox; ++X)
      for (int32_t e = L.off[(size_t)X]; e < L.off[(size_t)X + 1]; ++e) rowbox[(size_t)e] = (int32_t)X;
  }
  auto rank_all = [&](int64_t e) { return std::max<int32_t>(0, L.rank[(size_t)e]); };
  auto rankU = [&](int64_t e) { return sym && rowbox[(size_t)e] < L.col[(size_t)e] ? 0 : rank_all(e); };
  // (a multi-rank symmetric handle also drops the first-side V of pairs whose row box X has
  // no served row: their t1 = V^T x_Y only feeds y_X; B' still needs their U for t2)
  auto rankV = [&](int64_t e) {
    if (!sym) return rank_all(e);
    const int32_t X = rowbox[(size_t)e];
    return X > L.col[(size_t)e] || !h.row_box_active(l, X) ? 0 : rank_all(e);
  };
  auto up16 = [](int64_t v) { return (v + 15) & ~(int64_t)15; };
  L.ucol.assign((size_t)L.nblocks, 0);
  L.vcol.assign((size_t)L.nblocks, 0);
  L.vpan_off.assign((size_t)nbox, 0);
  L.ucolbase.assign((size_t)nbox + 1, 0);
  L.vR.assign((size_t)nbox, 0);
  int64_t vo = 0, vvals = 0;
  int32_t cb = 0;
  for (int64_t X = 0; X < nbox; ++X) {
    const int64_t m = h.box_end(l, X) - h.box_begin(l, X);
    int32_t R = 0;
    for (int32_t e = L.off[(size_t)X]; e < L.off[(size_t)X + 1]; ++e) {
      L.ucol[(size_t)e] = R;
      R += rankU(e);
    }
    L.ucolbase[(size_t)X] = cb;
    cb += R;
    // V panel of column box X: blocks (Z, X) for Z in I_X ascending
    int32_t RV = 0;
    for (int32_t e2 = L.off[(size_t)X]; e2 < L.off[(size_t)X + 1]; ++e2) {
      const int32_t b = L.trans[(size_t)e2];
      L.vcol[(size_t)b] = RV;
      RV += rankV(b);
    }
    if (RV > 2048) throw Error{H2D_EINVAL, "V panel wider than 2048 columns (lower max_rank)"};
    L.vR[(size_t)X] = RV;
    L.vpan_off[(size_t)X] = vo;
    vo = up16(vo + m * ((RV + 1) & ~1));
    vvals += m * RV;
  }
  L.ucolbase[(size_t)nbox] = cb;
  // U leaf panels of the served leaves
  const int64_t nserved = h.leaf_end - h.leaf_begin;
  L.uoff.assign((size_t)std::max<int64_t>(nserved, 0), 0);
  int64_t uo = 0, uvals = 0;
  for (int64_t lf = h.leaf_begin; lf < h.leaf_end; ++lf) {
    const int64_t X = h.leaf_code(lf) >> sh;   // (adaptive: levels below the leaf have no columns)
    const int64_t R = L.ucolbase[(size_t)X + 1] - L.ucolbase[(size_t)X];
    const int64_t mL = h.leaf_e(lf) - h.leaf_s(lf);
    L.uoff[(size_t)(lf - h.leaf_begin)] = uo;
    uo = up16(uo + ((mL + 1) & ~1) * R);
    uvals += mL * R;
  }
  L.u_values = uvals;
  L.v_values = vvals;
  L.u_alloc = uo;
  L.v_alloc = vo;
  L.U = h.alloc<double>(uo);
  L.V = h.alloc<double>(vo);
  H2D_CUDA(cudaMemsetAsync(L.U, 0, std::max<int64_t>(1, uo) * sizeof(double), s));
  H2D_CUDA(cudaMemsetAsync(L.V, 0, std::max<int64_t>(1, vo) * sizeof(double), s));
  std::vector<UCopyItem> uitems;
  std::vector<VPackItem> vitems;
  for (int64_t lf = h.leaf_begin; lf < h.leaf_end; ++lf) {
    const int64_t X = h.leaf_code(lf) >> sh;
    const int64_t bx0 = h.box_begin(l, X), mX = h.box_end(l, X) - bx0;
    const int64_t s0 = h.leaf_s(lf);
    const int32_t mL = (int32_t)(h.leaf_e(lf) - s0);
    if (mL == 0) continue;
    double* base = L.U + L.uoff[(size_t)(lf - h.leaf_begin)];
    for (int32_t e = L.off[(size_t)X]; e < L.off[(size_t)X + 1]; ++e) {
      const int r = rankU(e);
      if (r == 0) continue;
      uitems.push_back(UCopyItem{srcU[(size_t)e] + (s0 - bx0), base + (int64_t)L.ucol[(size_t)e] * ((mL + 1) & ~1),
                                 (int32_t)mX, (mL + 1) & ~1, mL, r});
    }
  }
  for (int64_t X = 0; X < nbox; ++X) {
    for (int32_t e = L.off[(size_t)X]; e < L.off[(size_t)X + 1]; ++e) {
      const int r = rankV(e);
      if (r == 0) continue;
      const int64_t Y = L.col[(size_t)e];
      const int64_t nY = h.box_end(l, Y) - h.box_begin(l, Y);
      if (nY * r > 0)
        vitems.push_back(VPackItem{srcV[(size_t)e], L.V + L.vpan_off[(size_t)Y] + L.vcol[(size_t)e],
                                   (int32_t)nY, r, (L.vR[(size_t)Y] + 1) & ~1, 0});
    }
  }
  if (sym) {
    // first-side U factors (X, Y), X < Y, as row-major box panels of X (stage B'); t1 layout
    L.ub_off.assign((size_t)nbox, 0);
    L.ubR.assign((size_t)nbox, 0);
    L.ubcol.assign((size_t)L.nblocks, 0);
    L.t1base.assign((size_t)nbox + 1, 0);
    int64_t bo = 0, bvals = 0;
    int32_t tb = 0;
    for (int64_t X = 0; X < nbox; ++X) {
      const int64_t m = h.box_end(l, X) - h.box_begin(l, X);
      int32_t R = 0;
      for (int32_t e = L.off[(size_t)X]; e < L.off[(size_t)X + 1]; ++e) {
        if (L.col[(size_t)e] < X) continue;
        L.ubcol[(size_t)e] = R;
        R += rank_all(e);
      }
      if (R > kT1Max) throw Error{H2D_EINVAL, "symmetric apply: first-side panel wider than 1024 columns"};
      L.ubR[(size_t)X] = R;
      L.t1base[(size_t)X] = tb;
      tb += R;
      L.ub_off[(size_t)X] = bo;
      bo = up16(bo + m * ((R + 1) & ~1));
      bvals += m * R;
    }
    L.t1base[(size_t)nbox] = tb;
    L.ub_values = bvals;
    L.ub_alloc = bo;
    L.Ub = h.alloc<double>(bo);
    H2D_CUDA(cudaMemsetAsync(L.Ub, 0, std::max<int64_t>(1, bo) * sizeof(double), s));
    for (int64_t X = 0; X < nbox; ++X) {
      const int64_t m = h.box_end(l, X) - h.box_begin(l, X);
      for (int32_t e = L.off[(size_t)X]; e < L.off[(size_t)X + 1]; ++e) {
        const int r = rank_all(e);
        if (L.col[(size_t)e] < X || r == 0 || m == 0) continue;
        vitems.push_back(VPackItem{srcU[(size_t)e], L.Ub + L.ub_off[(size_t)X] + L.ubcol[(size_t)e], (int32_t)m, r,
                                   (L.ubR[(size_t)X] + 1) & ~1, 0});
      }
    }
  }
  if (h.pair_wanted && !h.pair_failed) {
    for (int64_t e = 0; e < L.nblocks; ++e)
      if (rank_all(e) > kPMaxR) h.pair_failed = true;
    if (h.pair_failed)   // ranks above kPMaxR: the pair apply is off for these factors
      for (auto& Lv : h.levels) { h.release(Lv.Pr); Lv.Pr = nullptr; Lv.pairs.clear(); }
  }
  if (h.pair_wanted && !h.pair_failed) {
    // pair apply (pairs.cuh): per pair {X, Y}, X < Y, V_XY (n_Y x r) then U_XY (m_X x r),
    // column-major as the ACA stores them; pairs in CSR order of their first side X
    h.release(L.Pr);
    L.Pr = nullptr;
    L.pairs.clear();
    int64_t po = 0, pvals = 0;
    for (int64_t X = 0; X < nbox; ++X) {
      const int64_t m = h.box_end(l, X) - h.box_begin(l, X);
      for (int32_t e = L.off[(size_t)X]; e < L.off[(size_t)X + 1]; ++e) {
        const int64_t Y = L.col[(size_t)e];
        const int r = rank_all(e);
        const int64_t n = h.box_end(l, Y) - h.box_begin(l, Y);
        if (Y < X || r == 0 || m == 0 || n == 0) continue;
        Level::PairDesc d{po, po + n * r, (int32_t)h.box_begin(l, Y), (int32_t)h.box_begin(l, X), (int32_t)n,
                          (int32_t)m, r, r};
        L.pairs.push_back(d);
        po += (n + m) * r;
        pvals += (n + m) * r;
        uitems.push_back(UCopyItem{srcV[(size_t)e], nullptr, (int32_t)n, (int32_t)n, (int32_t)n, r});
        uitems.push_back(UCopyItem{srcU[(size_t)e], nullptr, (int32_t)m, (int32_t)m, (int32_t)m, r});
      }
    }
    L.pr_alloc = po;
    L.pr_values = pvals;
    L.Pr = h.alloc<double>(po);
    // destinations now that the array exists (the last 2 x pairs items are the pair copies)
    size_t k0 = uitems.size() - 2 * L.pairs.size();
    for (const auto& d : L.pairs) {
      uitems[k0++].dst = L.Pr + d.v_off;
      uitems[k0++].dst = L.Pr + d.u_off;
    }
  }
  const size_t CH = 1 << 20;
  for (size_t c0 = 0; c0 < uitems.size(); c0 += CH) {
    std::vector<UCopyItem> part(uitems.begin() + c0, uitems.begin() + std::min(uitems.size(), c0 + CH));
    UCopyItem* d = upload_tmp(part, s);
    ucopy_kernel<<<(int)part.size(), 256, 0, s>>>(d);
    H2D_LAUNCH_CHECK();
    H2D_CUDA(cudaFreeAsync(d, s));
  }
  for (size_t c0 = 0; c0 < vitems.size(); c0 += CH) {
    std::vector<VPackItem> part(vitems.begin() + c0, vitems.begin() + std::min(vitems.size(), c0 + CH));
    VPackItem* d = upload_tmp(part, s);
    vpack_kernel<<<(int)part.size(), 256, 0, s>>>(d);
    H2D_LAUNCH_CHECK();
    H2D_CUDA(cudaFreeAsync(d, s));
  }
  H2D_CUDA(cudaStreamSynchronize(s));
}

// Copy block e of level l out of the panels: U (m x r col-major), V (n x r col-major),
// host arrays.  U needs every leaf of the row box to be served by this handle.
void unpack_block(Handle& h, int l, int64_t e, int* m, int* n, int* r, double* U, double* V) {
  Level& L = h.levels[(size_t)l];
  const int64_t X = (int64_t)(std::upper_bound(L.off.begin(), L.off.end(), (int32_t)e) - L.off.begin()) - 1;
  const int64_t Y = L.col[(size_t)e];
  const int64_t bx0 = h.box_begin(l, X);
  const int64_t mm = h.box_end(l, X) - bx0;
  const int64_t nn = h.box_end(l, Y) - h.box_begin(l, Y);
  const int rr = std::max<int32_t>(0, L.rank[(size_t)e]);
  *m = (int)mm; *n = (int)nn; *r = rr;
  if (rr == 0) return;
  // a row-major box panel (ld doubles per row, first column c0) -> column-major rows x rr
  auto from_rowmajor = [&](double* dst, const double* panel, int64_t ld, int64_t c0, int64_t rows) {
    std::vector<double> rm((size_t)(rows * rr));
    if (rows > 0)
      H2D_CUDA(cudaMemcpy2D(rm.data(), rr * 8, panel + c0, (size_t)ld * 8, rr * 8, rows, cudaMemcpyDeviceToHost));
    for (int64_t j = 0; j < rows; ++j)
      for (int q = 0; q < rr; ++q) dst[j + (int64_t)q * rows] = rm[(size_t)(j * rr + q)];
  };
  if (h.symapply) {
    // first side (X < Y): U in the Ub box panel of X, V in the V box panel of Y;
    // second side (X > Y): U in the leaf panels (handled below), V = U of the pair (Y, X)
    if (X < Y) {
      if (V && !h.row_box_active(l, X))
        throw Error{H2D_EINVAL, "block row box not served by this handle (symmetric: V not stored)"};
      if (U) from_rowmajor(U, L.Ub + L.ub_off[(size_t)X], (L.ubR[(size_t)X] + 1) & ~1, L.ubcol[(size_t)e], mm);
      if (V) from_rowmajor(V, L.V + L.vpan_off[(size_t)Y], (L.vR[(size_t)Y] + 1) & ~1, L.vcol[(size_t)e], nn);
      return;
    }
    if (V) {
      const int32_t t = L.trans[(size_t)e];
      from_rowmajor(V, L.Ub + L.ub_off[(size_t)Y], (L.ubR[(size_t)Y] + 1) & ~1, L.ubcol[(size_t)t], nn);
      V = nullptr;
    }
  }
  if (U) {
    const int sh = 2 * (h.kappa - l);
    int64_t lf0 = X << sh, lf1 = (X + 1) << sh;
    if (h.adaptive) {   // the adaptive leaves inside box X (a contiguous run in Morton order)
      lf0 = std::lower_bound(h.lf_code.begin(), h.lf_code.end(), X << sh) - h.lf_code.begin();
      lf1 = std::lower_bound(h.lf_code.begin(), h.lf_code.end(), (X + 1) << sh) - h.lf_code.begin();
    }
    if (lf0 < h.leaf_begin || lf1 > h.leaf_end)
      throw Error{H2D_EINVAL, "block row box not fully served by this handle"};
    for (int64_t lf = lf0; lf < lf1; ++lf) {
      const int64_t s0 = h.leaf_s(lf);
      const int64_t mL = h.leaf_e(lf) - s0;
      if (mL == 0) continue;
      const int64_t mLp = (mL + 1) & ~1;
      H2D_CUDA(cudaMemcpy2D(U + (s0 - bx0), mm * 8,
                            L.U + L.uoff[(size_t)(lf - h.leaf_begin)] + (int64_t)L.ucol[(size_t)e] * mLp,
                            mLp * 8, mL * 8, rr, cudaMemcpyDeviceToHost));
    }
  }
  if (V) {
    const int64_t Rp = (L.vR[(size_t)Y] + 1) & ~1;
    std::vector<double> rm((size_t)(nn * rr));
    if (nn > 0)
      H2D_CUDA(cudaMemcpy2D(rm.data(), rr * 8, L.V + L.vpan_off[(size_t)Y] + L.vcol[(size_t)e],
                            (size_t)Rp * 8, rr * 8, nn, cudaMemcpyDeviceToHost));
    for (int64_t j = 0; j < nn; ++j)
      for (int q = 0; q < rr; ++q) V[j + (int64_t)q * nn] = rm[(size_t)(j * rr + q)];
  }
}

template <int NS>
static void set_pipe_attrs() {
  const int smem = (int)sizeof(PipeSmem<NS>);
  H2D_CUDA(cudaFuncSetAttribute(stageA_tma_kernel<NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  H2D_CUDA(cudaFuncSetAttribute(stageA_tma_kernel<NS>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                cudaSharedmemCarveoutMaxShared));
}

// Build the stage-A / reduce schedule, the t layout (U-column order), the stage-B items
// and the per-level device tables.
// The warp-per-leaf near-field classes with kernel KID, run alone (4 CTAs per SM) on st.
template <int KID>
static void warp_classes_alone(Handle& h, const double* x, cudaStream_t st) {
  int64_t off = 0;
  for (int r = 0; r < 3; ++r) {
    const int64_t cnt = h.n_p2p_warp_rpl[r];
    if (cnt <= 0) continue;
    auto* kfn = r == 0 ? p2p_warp_kernel<KID, 1> : r == 1 ? p2p_warp_kernel<KID, 2> : p2p_warp_kernel<KID, 3>;
    const int grid = (int)std::min<int64_t>(4 * (int64_t)h.num_sms, (cnt + 7) / 8);
    H2D_CUDA(cudaMemsetAsync(h.d_counters + 4 + r, 0, sizeof(int32_t), st));
    kfn<<<grid, 256, 0, st>>>(h.kappa, h.d_p2p_warp + off, (int)cnt, h.d_counters + 4 + r, h.d_leaf_start, h.d_px,
                              h.d_py, x, h.kp, h.d_ynear, h.d_ynear + h.n, h.d_ynear + 2 * h.n);
    H2D_LAUNCH_CHECK();
    off += cnt;
  }
}

// Log table of the warp-per-leaf near field (kLogNoSel handles): the 512-bin table or the
// replicated 64-bin one (kLogNoSelRepl, pipe.cuh).  Which is faster depends on how the
// near field's r^2 mantissas spread over the shared-memory banks (a regular grid: few
// distinct values, many conflicts), so the build times both on this handle's leaves (a
// warm-up and the best of three each, x = 0: the time does not depend on x) and keeps the
// replicated table only when it is at least 10 % faster (so that handles of the same points
// do not flip between the two on timing noise).  The two differ by rounding only (<= 1e-16
// absolute per evaluation).
// H2D_P2P_TABLE=0 / 1 forces the 512-bin / replicated table.
static void pick_log_table(Handle& h, cudaStream_t s) {
  const char* env = getenv("H2D_P2P_TABLE");
  if (env) {
    if (atoi(env) == 1) h.p2p_kid = kLogNoSelRepl;
    return;
  }
  double* x0 = nullptr;
  H2D_CUDA(cudaMallocAsync(&x0, h.n * sizeof(double), s));
  H2D_CUDA(cudaMemsetAsync(x0, 0, h.n * sizeof(double), s));
  cudaEvent_t e0, e1;
  H2D_CUDA(cudaEventCreate(&e0));
  H2D_CUDA(cudaEventCreate(&e1));
  float best[2] = {1e30f, 1e30f};
  for (int rep = 0; rep < 4; ++rep)
    for (int v = 0; v < 2; ++v) {
      H2D_CUDA(cudaEventRecord(e0, s));
      if (v == 0) warp_classes_alone<kLogNoSel>(h, x0, s);
      else warp_classes_alone<kLogNoSelRepl>(h, x0, s);
      H2D_CUDA(cudaEventRecord(e1, s));
      H2D_CUDA(cudaEventSynchronize(e1));
      float ms = 0.f;
      H2D_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      if (rep > 0) best[v] = std::min(best[v], ms);
    }
  H2D_CUDA(cudaEventDestroy(e0));
  H2D_CUDA(cudaEventDestroy(e1));
  H2D_CUDA(cudaFreeAsync(x0, s));
  const bool repl = best[1] < 0.9f * best[0];
  if (repl) h.p2p_kid = kLogNoSelRepl;
  if (getenv("H2D_VERBOSE"))
    fprintf(stderr, "[h2d] near-field log table: %s (512 bins %.4f ms, replicated 64 bins %.4f ms alone)\n",
            repl ? "replicated" : "512 bins", best[0], best[1]);
}

// The adaptive list near field with kernel KID, run alone (3 CTAs per SM, as p2p_serial) on st.
template <int KID>
static void list_alone(Handle& h, const double* x, cudaStream_t st) {
  const int grid = (int)std::min<int64_t>((int64_t)h.num_sms * 3, (h.n_p2p_list + 7) / 8);
  H2D_CUDA(cudaMemsetAsync(h.d_counters + 4, 0, sizeof(int32_t), st));
  p2p_list_kernel<KID><<<grid, 256, 0, st>>>(h.d_p2p_list, (int)h.n_p2p_list, h.d_counters + 4, h.d_lf_start,
                                             h.d_ad_nf_off, h.d_ad_nf_rng, h.d_px, h.d_py, x, h.kp, h.d_ynear);
  H2D_LAUNCH_CHECK();
}

// pick_log_table for the adaptive list near field (log and RBF phi_1 kernels): the same
// timing and 10 % margin; H2D_P2P_TABLE=0 / 1 forces either.
static void pick_list_table(Handle& h, cudaStream_t s) {
  const char* env = getenv("H2D_P2P_TABLE");
  if (env) {
    h.list_repl = atoi(env) == 1;
    return;
  }
  const bool phi1 = h.kp.id == H2D_KERNEL_RBF_PHI1;
  double* x0 = nullptr;
  H2D_CUDA(cudaMallocAsync(&x0, h.n * sizeof(double), s));
  H2D_CUDA(cudaMemsetAsync(x0, 0, h.n * sizeof(double), s));
  cudaEvent_t e0, e1;
  H2D_CUDA(cudaEventCreate(&e0));
  H2D_CUDA(cudaEventCreate(&e1));
  float best[2] = {1e30f, 1e30f};
  for (int rep = 0; rep < 4; ++rep)
    for (int v = 0; v < 2; ++v) {
      H2D_CUDA(cudaEventRecord(e0, s));
      if (phi1) {
        if (v == 0) list_alone<H2D_KERNEL_RBF_PHI1>(h, x0, s);
        else list_alone<kPhi1Repl>(h, x0, s);
      } else {
        if (v == 0) list_alone<H2D_KERNEL_LOG>(h, x0, s);
        else list_alone<kLogRepl>(h, x0, s);
      }
      H2D_CUDA(cudaEventRecord(e1, s));
      H2D_CUDA(cudaEventSynchronize(e1));
      float ms = 0.f;
      H2D_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      if (rep > 0) best[v] = std::min(best[v], ms);
    }
  H2D_CUDA(cudaEventDestroy(e0));
  H2D_CUDA(cudaEventDestroy(e1));
  H2D_CUDA(cudaFreeAsync(x0, s));
  h.list_repl = best[1] < 0.9f * best[0];
  if (getenv("H2D_VERBOSE"))
    fprintf(stderr, "[h2d] adaptive near-field log table: %s (512 bins %.4f ms, replicated 64 bins %.4f ms alone)\n",
            h.list_repl ? "replicated" : "512 bins", best[0], best[1]);
}

void finalize_schedule(Handle& h) {
  cudaStream_t s = h.stream;
  int64_t t_len = 0, tpart_len = 0;
  // stage-A item size: large items amortise the per-item epilogue (measured: 32K -> 1M
  // elements takes C3's stage A from 1.60 to 1.44 ms), but at least ~4 items per CTA keep
  // the dynamic schedule balanced on small operators
  int64_t a_elems = 0;
  for (int l = 1; l <= h.kappa; ++l) {
    const Level& L = h.levels[(size_t)l];
    for (int64_t Y = 0; Y < L.nbox; ++Y)
      a_elems += (h.box_end(l, Y) - h.box_begin(l, Y)) * ((L.vR[(size_t)Y] + 1) & ~1);
  }
  if (!h.num_sms) H2D_CUDA(cudaDeviceGetAttribute(&h.num_sms, cudaDevAttrMultiProcessorCount, h.device));
  if (!h.persist_ctas) h.persist_ctas = 2 * h.num_sms;
  const char* env_at = getenv("H2D_A_TARGET");    // diagnostics override (elements)
  const int64_t kATarget = env_at && atoll(env_at) >= 2048
                               ? atoll(env_at)
                               : std::min<int64_t>(kATargetDefault,
                                                   std::max<int64_t>(32768, a_elems / (4 * (int64_t)h.persist_ctas)));
  std::vector<AItem> aitems;
  std::vector<RItem> ritems;
  for (int l = 1; l <= h.kappa; ++l) {
    Level& L = h.levels[(size_t)l];
    L.tu_base = t_len;
    t_len += L.ucolbase[(size_t)L.nbox];
  }
  if (t_len > INT32_MAX) throw Error{H2D_EINVAL, "t vector exceeds 2^31 entries"};
  // symmetric apply: stage A' writes t1 (first-side blocks, U-box column order), the
  // directed t above is t2 (second-side blocks, U-leaf column order)
  const bool sym = h.symapply;
  int64_t t1_len = 0;
  if (sym)
    for (int l = 1; l <= h.kappa; ++l) {
      Level& L = h.levels[(size_t)l];
      L.t1_base = t1_len;
      t1_len += L.t1base[(size_t)L.nbox];
    }
  // vdst: V-panel columns in column-box order (per level, box, column) -> t (t1) index
  // (a multi-rank symmetric handle has more first-side than second-side columns: t1 holds
  // every pair touching its rows, t2 only the second-side blocks of its served rows)
  std::vector<int32_t> vdst((size_t)std::max<int64_t>(1, sym ? t1_len : t_len));
  int64_t vpos = 0;
  for (int l = 1; l <= h.kappa; ++l) {
    Level& L = h.levels[(size_t)l];
    L.t_off.assign((size_t)L.nbox, 0);
    for (int64_t Y = 0; Y < L.nbox; ++Y) {
      L.t_off[(size_t)Y] = vpos;
      for (int32_t e2 = L.off[(size_t)Y]; e2 < L.off[(size_t)Y + 1]; ++e2) {
        const int32_t b = L.trans[(size_t)e2];           // block (X, Y)
        const int64_t X = L.col[(size_t)e2];
        const int r = sym && (X > Y || !h.row_box_active(l, X)) ? 0 : std::max<int32_t>(0, L.rank[(size_t)b]);
        if (r == 0) continue;
        const int64_t base = sym ? L.t1_base + L.t1base[(size_t)X] + L.ubcol[(size_t)b]
                                 : L.tu_base + L.ucolbase[(size_t)X] + L.ucol[(size_t)b];
        for (int q = 0; q < r; ++q) vdst[(size_t)(vpos + L.vcol[(size_t)b] + q)] = (int32_t)(base + q);
      }
      vpos += L.vR[(size_t)Y];
    }
  }
  // (multi-rank symmetric: A' skips the pairs whose row box has no served row)
  const bool all_rows = h.row_begin == 0 && h.row_end == h.n;
  if (sym ? (vpos > t1_len || (all_rows && vpos != t1_len)) : vpos != t_len)
    throw Error{H2D_ECUDA, "t layout mismatch"};
  h.t_len = t_len;
  // symmetric: one extra entry at t_len takes B''s t2 writes whose mirrored block (Y, X)
  // has no row served here (multi-rank handles; never read)
  h.d_t = h.alloc<double>(t_len + (sym ? 1 : 0));
  h.d_vdst = h.alloc<int32_t>(vdst.size());
  H2D_CUDA(cudaMemcpyAsync(h.d_vdst, vdst.data(), vdst.size() * 4, cudaMemcpyHostToDevice, s));
  for (int l = 1; l <= h.kappa; ++l) {
    Level& L = h.levels[(size_t)l];
    L.d_ucolbase = h.alloc<int32_t>(L.ucolbase.size());
    L.d_uoff = h.alloc<int64_t>(L.uoff.size());
    H2D_CUDA(cudaMemcpyAsync(L.d_ucolbase, L.ucolbase.data(), L.ucolbase.size() * 4,
                             cudaMemcpyHostToDevice, s));
    if (!L.uoff.empty())
      H2D_CUDA(cudaMemcpyAsync(L.d_uoff, L.uoff.data(), L.uoff.size() * 8, cudaMemcpyHostToDevice, s));
    H2D_CUDA(cudaStreamSynchronize(s));
    h.lp.U[l] = L.U;
    h.lp.V[l] = L.V;
    h.lp.ucolbase[l] = L.d_ucolbase;
    h.lp.uoff[l] = L.d_uoff;
    h.lp.tu[l] = h.d_t + L.tu_base;
    h.lp.Ub[l] = L.Ub;
    // stage-A items: chunks of <= kATarget elements and <= kAMaxRows rows
    for (int64_t Y = 0; Y < L.nbox; ++Y) {
      const int R = L.vR[(size_t)Y], Rp = (R + 1) & ~1;
      const int64_t y0 = h.box_begin(l, Y);
      const int64_t nY = h.box_end(l, Y) - y0;
      if (R == 0 || nY == 0) continue;
      int64_t nch = std::max<int64_t>((nY * Rp + kATarget - 1) / kATarget, (nY + kAMaxRows - 1) / kAMaxRows);
      nch = std::min<int64_t>(nY, std::max<int64_t>(1, nch));
      const int64_t rows = (nY + nch - 1) / nch;
      nch = (nY + rows - 1) / rows;
      const int32_t vp = (int32_t)L.t_off[(size_t)Y];
      if (nch == 1) {
        aitems.push_back(AItem{L.vpan_off[(size_t)Y], y0, (int32_t)nY, R, vp, l, -1, Rp});
      } else {
        if (tpart_len + nch * R > INT32_MAX) throw Error{H2D_EINVAL, "partial buffer too large"};
        ritems.push_back(RItem{vp, (int32_t)tpart_len, R, (int32_t)nch});
        for (int64_t c = 0; c < nch; ++c) {
          const int64_t r0 = c * rows, nr = std::min(rows, nY - r0);
          aitems.push_back(AItem{L.vpan_off[(size_t)Y] + r0 * Rp, y0 + r0, (int32_t)nr, R,
                                 (int32_t)(-(tpart_len + c * R) - 1), l,
                                 (int32_t)(ritems.size() - 1), Rp});
        }
        tpart_len += nch * R;
      }
    }
  }
  // single-chunk boxes of <= kSmallARows rows go to the warp-per-item kernel (tail of the
  // list, H2D_SMALL_ITEMS=0 keeps them in the ring); the ring's items largest first: the
  // dynamic (atomic-counter) schedule then ends with small items
  // (only when there are enough of them to fill the GPU: a handful stay in the ring)
  const bool small_items = !(getenv("H2D_SMALL_ITEMS") && atoi(getenv("H2D_SMALL_ITEMS")) == 0);
  // H2D_SMALL_MIN (tests): the minimum count (default 4 per SM)
  const int64_t small_min = getenv("H2D_SMALL_MIN") ? atoll(getenv("H2D_SMALL_MIN")) : 4 * (int64_t)h.num_sms;
  auto a_small = [](const AItem& a) { return a.nrows <= kSmallARows && a.ritem < 0 && a.out >= 0; };
  // H2D_SMALL_A=0 / 1 (diagnostics): stage A's small items only
  const bool small_a = getenv("H2D_SMALL_A") ? atoi(getenv("H2D_SMALL_A")) != 0 : small_items;
  const bool a_split = small_a && std::count_if(aitems.begin(), aitems.end(), a_small) >= small_min;
  // the small stage-A kernel before the ring (balanced trees) or after it (adaptive trees):
  // measured on the 1000^2 Chebyshev phi_1 system (profiles/r02q): adaptive symmetric 3.80 ->
  // 3.62 ms, directed 4.49 -> 4.25 with it after; balanced (N_max 500) 7.41 -> 7.58 and 7.29 ->
  // 8.54 ms (H2D_SMALL_A_AFTER=0 / 1 overrides)
  h.small_a_after = getenv("H2D_SMALL_A_AFTER") ? atoi(getenv("H2D_SMALL_A_AFTER")) == 1 : h.adaptive;
  h.p2p_after_b1 = getenv("H2D_P2P_AFTER_B1") && atoi(getenv("H2D_P2P_AFTER_B1")) == 1;
  const auto amid = std::stable_partition(aitems.begin(), aitems.end(),
                                          [&](const AItem& a) { return !(a_split && a_small(a)); });
  h.n_abig = amid - aitems.begin();
  std::stable_sort(aitems.begin(), amid, [](const AItem& a, const AItem& b) {
    return (int64_t)a.nrows * a.Rp > (int64_t)b.nrows * b.Rp;
  });
  // H2D_ORDER_LOCAL (a communicator with several ranks): items whose rows lie in the served
  // range first (each part keeps its order), so they can run while x is being gathered
  if (h.comm && h.opts.world > 1) {
    auto local = [&](const AItem& a) { return a.x_off >= h.row_begin && a.x_off + a.nrows <= h.row_end; };
    h.n_abig_loc = std::stable_partition(aitems.begin(), amid, local) - aitems.begin();
    h.n_asmall_loc = std::stable_partition(amid, aitems.end(), local) - amid;
  } else {
    h.n_abig_loc = h.n_abig;
    h.n_asmall_loc = (int64_t)aitems.size() - h.n_abig;
  }
  // symmetric stage B' items over the first-side U box panels (same chunking as stage A);
  // udst maps a U-box column (block (X, Y), X < Y, column q) to the t2 index of (Y, X)
  std::vector<AItem> b1items;
  std::vector<RItem> b1ritems;
  int64_t b1part_len = 0;
  if (sym) {
    std::vector<int32_t> udst((size_t)std::max<int64_t>(1, t1_len));
    int64_t upos = 0;
    for (int l = 1; l <= h.kappa; ++l) {
      Level& L = h.levels[(size_t)l];
      for (int64_t X = 0; X < L.nbox; ++X) {
        const int R = L.ubR[(size_t)X], Rp = (R + 1) & ~1;
        for (int32_t e = L.off[(size_t)X]; e < L.off[(size_t)X + 1]; ++e) {
          const int64_t Y = L.col[(size_t)e];
          const int r = std::max<int32_t>(0, L.rank[(size_t)e]);
          if (Y < X || r == 0) continue;
          const int32_t t = L.trans[(size_t)e];
          const bool served = L.rank[(size_t)t] >= 0;   // (Y, X) mirrored: Y's rows served here
          for (int q = 0; q < r; ++q)
            udst[(size_t)(upos + L.ubcol[(size_t)e] + q)] =
                served ? (int32_t)(L.tu_base + L.ucolbase[(size_t)Y] + L.ucol[(size_t)t] + q) : (int32_t)t_len;
        }
        const int64_t x0 = h.box_begin(l, X), nX = h.box_end(l, X) - x0;
        if (R > 0 && nX > 0) {
          const int64_t t1o = L.t1_base + L.t1base[(size_t)X];
          int64_t nch = std::max<int64_t>((nX * Rp + kATarget - 1) / kATarget, (nX + kAMaxRows - 1) / kAMaxRows);
          nch = std::min<int64_t>(nX, std::max<int64_t>(1, nch));
          const int64_t rows = (nX + nch - 1) / nch;
          nch = (nX + rows - 1) / rows;
          if (nch == 1) {
            b1items.push_back(AItem{L.ub_off[(size_t)X], x0, (int32_t)nX, R, (int32_t)upos, l, -1, Rp, t1o});
          } else {
            if (b1part_len + nch * R > INT32_MAX) throw Error{H2D_EINVAL, "partial buffer too large"};
            b1ritems.push_back(RItem{(int32_t)upos, (int32_t)b1part_len, R, (int32_t)nch});
            for (int64_t c = 0; c < nch; ++c) {
              const int64_t r0 = c * rows, nr = std::min(rows, nX - r0);
              b1items.push_back(AItem{L.ub_off[(size_t)X] + r0 * Rp, x0 + r0, (int32_t)nr, R,
                                      (int32_t)(-(b1part_len + c * R) - 1), l, (int32_t)(b1ritems.size() - 1),
                                      Rp, t1o});
            }
            b1part_len += nch * R;
          }
        }
        upos += R;
      }
    }
    if (upos != t1_len) throw Error{H2D_ECUDA, "symmetric U-box layout mismatch"};
    // small single-chunk boxes: the warp-per-item B' kernel after the ring (H2D_SMALL_B1=0:
    // all in the ring); the ring's items largest first
    const bool small_b1 = getenv("H2D_SMALL_B1") ? atoi(getenv("H2D_SMALL_B1")) != 0 : small_items;
    const bool b1_split = small_b1 && std::count_if(b1items.begin(), b1items.end(), a_small) >= small_min;
    const auto b1mid = std::stable_partition(b1items.begin(), b1items.end(),
                                             [&](const AItem& a) { return !(b1_split && a_small(a)); });
    h.n_b1big = b1mid - b1items.begin();
    std::stable_sort(b1items.begin(), b1mid, [](const AItem& a, const AItem& b) {
      return (int64_t)a.nrows * a.Rp > (int64_t)b.nrows * b.Rp;
    });
    if (getenv("H2D_VERBOSE")) {   // diagnostics: share of B' elements on the two-pass (wide) path
      double tot = 0, wide = 0;
      for (const AItem& it : b1items) {
        const double e = (double)it.nrows * it.Rp;
        tot += e;
        if (it.Rp / 2 > 32 * kDualMaxC) wide += e;
      }
      fprintf(stderr, "[h2d] B' items %zu, elements %.0f, wide (R > %d) share %.4f\n", b1items.size(), tot,
              64 * kDualMaxC, tot > 0 ? wide / tot : 0.0);
      for (int sd : {2048, 3072, 4096}) {   // stages per slot size (doubles)
        double st = 0;
        for (const AItem& it : b1items) {
          const int rs = std::min(kStageVec, (sd - ((it.R + 1) & ~1)) / it.Rp);
          st += (it.nrows + rs - 1) / rs;
        }
        fprintf(stderr, "[h2d]   slot %d doubles: %.0f stages, fill %.3f\n", sd, st, tot / (st * sd));
      }
      double sa = 0, ea = 0;
      for (const AItem& it : aitems) {
        const int rs = std::min(kStageVec, kStageDbl / it.Rp);
        sa += (it.nrows + rs - 1) / rs;
        ea += (double)it.nrows * it.Rp;
      }
      fprintf(stderr, "[h2d] A' items %zu: %.0f stages, fill %.3f\n", aitems.size(), sa, ea / (sa * kStageDbl));
    }
    h.t1_len = t1_len;
    h.d_t1 = h.alloc<double>(t1_len);
    // (entries A' never writes: pairs whose row box has no served row; B' reads them as 0)
    H2D_CUDA(cudaMemsetAsync(h.d_t1, 0, std::max<int64_t>(1, t1_len) * sizeof(double), s));
    h.d_udst = h.alloc<int32_t>(udst.size());
    H2D_CUDA(cudaMemcpyAsync(h.d_udst, udst.data(), udst.size() * 4, cudaMemcpyHostToDevice, s));
    h.n_b1items = (int64_t)b1items.size();
    h.d_b1items = h.alloc<AItem>(b1items.size());
    h.d_b1ritems = h.alloc<RItem>(b1ritems.size());
    h.d_b1rcount = h.alloc<int32_t>(b1ritems.size());
    h.d_b1tpart = h.alloc<double>(b1part_len);
    H2D_CUDA(cudaMemsetAsync(h.d_b1rcount, 0, std::max<size_t>(1, b1ritems.size()) * sizeof(int32_t), s));
    if (!b1items.empty())
      H2D_CUDA(cudaMemcpyAsync(h.d_b1items, b1items.data(), b1items.size() * sizeof(AItem), cudaMemcpyHostToDevice, s));
    if (!b1ritems.empty())
      H2D_CUDA(cudaMemcpyAsync(h.d_b1ritems, b1ritems.data(), b1ritems.size() * sizeof(RItem),
                               cudaMemcpyHostToDevice, s));
    // entries of rows without a first-side panel at a level are never written by B': zeroed
    // here, at every (re)schedule, not per matvec
    if (!h.d_y1) h.d_y1 = h.alloc<double>((size_t)h.kappa * h.n);
    H2D_CUDA(cudaMemsetAsync(h.d_y1, 0, (size_t)h.kappa * h.n * sizeof(double), s));
  }
  // stage-B items: served leaves in row blocks of <= kBRows rows, largest cost first, with
  // the per-level metadata of each item precomputed (one dependent load in the producer)
  std::vector<BItem> bitems;
  std::vector<int64_t> bcost, bleaf;
  for (int64_t lf = h.leaf_begin; lf < h.leaf_end; ++lf) {
    const int32_t s0 = (int32_t)h.leaf_s(lf);
    const int32_t mL = (int32_t)h.leaf_e(lf) - s0;
    int64_t RL = 0;
    for (int l = 1; l <= h.kappa; ++l) {
      const Level& L = h.levels[(size_t)l];
      const int64_t X = h.leaf_code(lf) >> (2 * (h.kappa - l));
      RL += L.ucolbase[(size_t)X + 1] - L.ucolbase[(size_t)X];
    }
    for (int32_t r0 = 0; r0 < mL; r0 += kBRows) {
      const int32_t rows = std::min(kBRows, mL - r0);
      bitems.push_back(BItem{r0, rows, mL, (int32_t)(s0 + r0 - h.row_begin)});
      bcost.push_back((int64_t)((rows + 1) & ~1) * RL + 512);
      bleaf.push_back(lf);
    }
  }
  if (getenv("H2D_VERBOSE")) {   // diagnostics: stage A / B items, stages and bytes by size
    const int edges[6] = {0, 8, 32, 96, 224, 1 << 30};
    double cnt[5] = {0}, el[5] = {0}, st[5] = {0};
    for (size_t k = 0; k < bitems.size(); ++k) {
      const int rows = bitems[k].rows, rowsp = (rows + 1) & ~1;
      int b = 0;
      while (rows > edges[b + 1]) ++b;
      const int64_t lf = bleaf[k];
      const int cols_s = std::min(kStageVec, kStageDbl / rowsp);
      for (int l = 1; l <= h.kappa; ++l) {
        const Level& L = h.levels[(size_t)l];
        const int64_t X = h.leaf_code(lf) >> (2 * (h.kappa - l));
        const int R = L.ucolbase[(size_t)X + 1] - L.ucolbase[(size_t)X];
        el[b] += (double)rowsp * R;
        st[b] += (R + cols_s - 1) / cols_s;
      }
      cnt[b] += 1;
    }
    for (int b = 0; b < 5; ++b)
      fprintf(stderr, "[h2d] B items rows (%d, %d]: %.0f items, %.0f stages, %.3f GB\n", edges[b], edges[b + 1],
              cnt[b], st[b], el[b] * 8e-9);
    double ac[5] = {0}, ae[5] = {0}, as[5] = {0};
    for (const AItem& it : aitems) {
      int b = 0;
      while (it.nrows > edges[b + 1]) ++b;
      const int rs = std::min(kStageVec, kStageDbl / it.Rp);
      ac[b] += 1;
      ae[b] += (double)it.nrows * it.Rp;
      as[b] += (it.nrows + rs - 1) / rs;
    }
    for (int b = 0; b < 5; ++b)
      fprintf(stderr, "[h2d] A items rows (%d, %d]: %.0f items, %.0f stages, %.3f GB\n", edges[b], edges[b + 1],
              ac[b], as[b], ae[b] * 8e-9);
  }
  std::vector<size_t> ord(bitems.size());
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](size_t a, size_t b) { return bcost[a] > bcost[b]; });
  // whole leaves of <= kSmallBRows rows: warp-per-item kernel (tail of the list; the
  // multi-RHS kernels still take the whole list)
  auto b_small = [&](size_t k) { return bitems[k].rows <= kSmallBRows && bitems[k].rows == bitems[k].mL; };
  const bool b_split = small_items && std::count_if(ord.begin(), ord.end(), b_small) >= small_min;
  h.n_bbig = std::stable_partition(ord.begin(), ord.end(), [&](size_t k) { return !(b_split && b_small(k)); }) -
             ord.begin();
  std::vector<BItem> bsorted;
  std::vector<BLevel> blev;
  bsorted.reserve(bitems.size());
  blev.reserve(bitems.size() * (size_t)std::max(1, h.kappa));
  for (size_t k : ord) {
    bsorted.push_back(bitems[k]);
    const int64_t lf = bleaf[k];
    for (int l = 1; l <= h.kappa; ++l) {
      const Level& L = h.levels[(size_t)l];
      const int64_t X = h.leaf_code(lf) >> (2 * (h.kappa - l));
      blev.push_back(BLevel{L.uoff[(size_t)(lf - h.leaf_begin)], L.ucolbase[(size_t)X],
                            L.ucolbase[(size_t)X + 1] - L.ucolbase[(size_t)X]});
    }
  }
  // near-field P2P: leaves the persistent fast kernel handles (whole near field served, all
  // three tiles <= kSymTile points, distance kernel) and the rest (generic kernel); adaptive
  // handles: every leaf on the column-range list kernel (R24)
  if (h.adaptive) {
    h.n_p2p_warp = h.n_p2p_fast = h.n_p2p_gen = 0;
    h.n_p2p_warp_rpl[0] = h.n_p2p_warp_rpl[1] = h.n_p2p_warp_rpl[2] = 0;
    // items (leaf, 64-row pass), most columns first (dynamic schedule ends with short items)
    std::vector<std::pair<int64_t, int64_t>> li;
    for (int64_t lf = h.leaf_begin; lf < h.leaf_end; ++lf) {
      const int64_t m = h.leaf_e(lf) - h.leaf_s(lf);
      if (m > 64 * 255) throw Error{H2D_EINVAL, "adaptive leaf larger than 16320 points"};
      int64_t cols = 0;
      for (int64_t e = h.ad_nf_off[(size_t)lf]; e < h.ad_nf_off[(size_t)lf + 1]; ++e) cols += h.ad_nf_rng[(size_t)(2 * e + 1)];
      for (int64_t p = 0; 64 * p < m; ++p) li.push_back({std::min<int64_t>(64, m - 64 * p) * cols, (lf << 8) | p});
    }
    std::stable_sort(li.begin(), li.end(), [](const auto& a, const auto& b) { return a.first > b.first; });
    std::vector<int64_t> items(li.size());
    for (size_t k = 0; k < li.size(); ++k) items[k] = li[k].second;
    h.n_p2p_list = (int64_t)items.size();
    h.release(h.d_p2p_list);
    h.d_p2p_list = h.alloc<int64_t>(items.size());
    if (!items.empty())
      H2D_CUDA(cudaMemcpyAsync(h.d_p2p_list, items.data(), items.size() * 8, cudaMemcpyHostToDevice, s));
  } else {
    auto compact = [](uint32_t v) {
      v &= 0x55555555u;
      v = (v | (v >> 1)) & 0x33333333u;
      v = (v | (v >> 2)) & 0x0F0F0F0Fu;
      v = (v | (v >> 4)) & 0x00FF00FFu;
      v = (v | (v >> 8)) & 0x0000FFFFu;
      return v;
    };
    auto spread = [](uint32_t v) {
      v &= 0xFFFFu;
      v = (v | (v << 8)) & 0x00FF00FFu;
      v = (v | (v << 4)) & 0x0F0F0F0Fu;
      v = (v | (v << 2)) & 0x33333333u;
      v = (v | (v << 1)) & 0x55555555u;
      return v;
    };
    const bool dist = h.kp.id == H2D_KERNEL_LOG || h.kp.id == H2D_KERNEL_IMQ || h.kp.id == H2D_KERNEL_ONE_OVER_R ||
                      h.kp.id == H2D_KERNEL_RBF_PHI1 || h.kp.id == H2D_KERNEL_RBF_PHI2;
    const uint32_t side = 1u << h.kappa;
    auto size_of = [&](int64_t lf) { return h.leaf_start[(size_t)lf + 1] - h.leaf_start[(size_t)lf]; };
    auto served = [&](int64_t lf) { return lf >= h.leaf_begin && lf < h.leaf_end; };
    std::vector<int32_t> fast, gen, wlist;
    // leaves up to warp_max points go to the warp-per-leaf kernels (RPL = ceil(m / 32)); the
    // CTA kernels keep larger leaves (H2D_P2P_WARP_MAX: diagnostics override, <= 96)
    const int warp_max = getenv("H2D_P2P_WARP_MAX") ? std::min(96, atoi(getenv("H2D_P2P_WARP_MAX"))) : kWarpLeaf;
    for (int64_t lf = h.leaf_begin; lf < h.leaf_end; ++lf) {
      const uint32_t cx = compact((uint32_t)lf), cy = compact((uint32_t)lf >> 1);
      bool served_all = true, small_nbrs = true;
      auto nb = [&](bool exists, uint32_t nx, uint32_t ny, bool check_size) {
        if (!exists) return;
        const int64_t Y = (int64_t)(spread(nx) | (spread(ny) << 1));
        served_all = served_all && served(Y);
        small_nbrs = small_nbrs && (!check_size || size_of(Y) <= kSymTile);
      };
      nb(cx + 1 < side, cx + 1, cy, true);
      nb(cy + 1 < side, cx, cy + 1, true);
      nb(cx > 0, cx - 1, cy, false);
      nb(cy > 0, cx, cy - 1, false);
      // warp path: <= 32-point leaves (any neighbour size); CTA fast path: three tiles
      // <= kSymTile points; both need a distance kernel and the whole near field served
      if (dist && served_all && size_of(lf) <= warp_max) wlist.push_back((int32_t)lf);
      else if (dist && served_all && small_nbrs && size_of(lf) <= kSymTile) fast.push_back((int32_t)lf);
      else gen.push_back((int32_t)lf);
    }
    if (getenv("H2D_P2P_NOWARP")) {   // diagnostics: small leaves on the CTA paths
      for (int32_t lf : wlist) {
        const uint32_t cx = compact((uint32_t)lf), cy = compact((uint32_t)lf >> 1);
        bool small = true;
        auto chk = [&](bool e, uint32_t nx, uint32_t ny) {
          if (e) small = small && size_of((int64_t)(spread(nx) | (spread(ny) << 1))) <= kSymTile;
        };
        chk(cx + 1 < side, cx + 1, cy);
        chk(cy + 1 < side, cx, cy + 1);
        (small ? fast : gen).push_back(lf);
      }
      wlist.clear();
    }
    std::stable_sort(wlist.begin(), wlist.end(), [&](int32_t a, int32_t b) {
      return (size_of(a) + 31) / 32 < (size_of(b) + 31) / 32;
    });
    for (int r = 0; r < 3; ++r)
      h.n_p2p_warp_rpl[r] = std::count_if(wlist.begin(), wlist.end(), [&](int32_t lf) {
        return std::max<int64_t>(1, (size_of(lf) + 31) / 32) == r + 1;
      });
    h.n_p2p_warp = (int64_t)wlist.size();
    h.release(h.d_p2p_warp);
    h.d_p2p_warp = h.alloc<int32_t>(wlist.size());
    if (!wlist.empty())
      H2D_CUDA(cudaMemcpyAsync(h.d_p2p_warp, wlist.data(), wlist.size() * 4, cudaMemcpyHostToDevice, s));
    h.n_p2p_fast = (int64_t)fast.size();
    h.n_p2p_gen = (int64_t)gen.size();
    h.release(h.d_p2p_fast);
    h.release(h.d_p2p_gen);
    h.d_p2p_fast = h.alloc<int32_t>(fast.size());
    h.d_p2p_gen = h.alloc<int32_t>(gen.size());
    if (!fast.empty())
      H2D_CUDA(cudaMemcpyAsync(h.d_p2p_fast, fast.data(), fast.size() * 4, cudaMemcpyHostToDevice, s));
    if (!gen.empty())
      H2D_CUDA(cudaMemcpyAsync(h.d_p2p_gen, gen.data(), gen.size() * 4, cudaMemcpyHostToDevice, s));
  }
  h.pairapply = h.pair_wanted && !h.pair_failed;
  if (h.pairapply) {
    // pair apply schedule (pairs.cuh): the big pairs of the coarse levels as row chunks per
    // phase (merged by byte position with a lag, every chunk after all chunks of the pair's
    // previous phase), then the medium pairs (one CTA each), then groups of 8 small pairs
    // (one warp each), each class largest first
    std::vector<PPair> prs;
    std::vector<std::pair<int64_t, int32_t>> big, whole, small;
    int64_t pvals = 0;
    int lv_lo = 1, lv_hi = h.kappa;   // diagnostics: H2D_PAIR_LEVELS=lo,hi (WRONG results; timing only)
    if (getenv("H2D_PAIR_LEVELS")) sscanf(getenv("H2D_PAIR_LEVELS"), "%d,%d", &lv_lo, &lv_hi);
    const int64_t small_max = getenv("H2D_PAIR_SMALL_MAX") ? atoll(getenv("H2D_PAIR_SMALL_MAX")) : kPSmallBytes;
    const int64_t whole_max = getenv("H2D_PAIR_WHOLE_MAX") ? atoll(getenv("H2D_PAIR_WHOLE_MAX")) : kPWholeBytes;
    for (int l = std::max(1, lv_lo); l <= std::min(h.kappa, lv_hi); ++l) {
      const Level& L = h.levels[(size_t)l];
      for (const auto& d : L.pairs) {
        const int32_t id = (int32_t)prs.size();
        prs.push_back(PPair{d.v_off, d.u_off, d.yv, d.yu, d.nv, d.nu, d.R, l});
        const int64_t bytes = (int64_t)(d.nv + d.nu) * d.R * 8;
        pvals += (int64_t)(d.nv + d.nu) * d.R;
        (bytes <= small_max ? small : bytes <= whole_max ? whole : big).push_back({bytes, id});
      }
    }
    h.pair_values = pvals;
    auto by_size = [](const auto& a, const auto& b) { return a.first > b.first; };
    std::stable_sort(big.begin(), big.end(), by_size);
    std::stable_sort(whole.begin(), whole.end(), by_size);
    std::stable_sort(small.begin(), small.end(), by_size);
    // groups reference consecutive descriptors: reorder the small pairs' descriptors
    std::vector<PPair> ordered;
    ordered.reserve(prs.size());
    std::vector<int32_t> newid(prs.size());
    for (auto* cls : {&big, &whole, &small})
      for (auto& b : *cls) {
        newid[(size_t)b.second] = (int32_t)ordered.size();
        ordered.push_back(prs[(size_t)b.second]);
        b.second = newid[(size_t)b.second];
      }
    std::vector<PWork> work;
    const int64_t nbig = (int64_t)big.size();
    std::vector<std::vector<PWork>> ph[3];
    for (int b = 0; b < 3; ++b) ph[b].resize((size_t)nbig);
    int64_t toff = 0, poff = 0;
    for (int64_t k = 0; k < nbig; ++k) {
      const PPair& p = ordered[(size_t)big[(size_t)k].second];
      for (int q = 1; q <= 3; ++q) {
        const int n = q == 2 ? p.nu : p.nv;
        const int nch = (n + kPChunkRows - 1) / kPChunkRows;
        for (int c = 0; c < nch; ++c) {
          PWork w{};
          w.kind = kPPhase1 + q - 1;
          w.first = big[(size_t)k].second;
          w.r0 = c * kPChunkRows;
          w.r1 = std::min(n, (c + 1) * kPChunkRows);
          w.big = (int32_t)k;
          w.chunk = c;
          w.nchunks = nch;
          w.toff = toff;
          w.poff = q < 3 ? poff : 0;
          ph[q - 1][(size_t)k].push_back(w);
        }
        if (q < 3) poff += (int64_t)nch * p.r;
      }
      toff += p.r;
    }
    const double lag = getenv("H2D_PAIR_LAG") ? atof(getenv("H2D_PAIR_LAG"))
                                              : 1.5 * (2.0 * h.num_sms) * kPChunkRows * 20 * 8.0;
    std::vector<std::pair<double, PWork>> keyed;
    std::vector<double> prev_end((size_t)nbig, -1.0);
    for (int q = 0; q < 3; ++q) {
      double pos = 0.0;
      std::vector<double> end((size_t)nbig, 0.0);
      for (int64_t k = 0; k < nbig; ++k) {
        const PPair& p = ordered[(size_t)big[(size_t)k].second];
        for (const PWork& w : ph[q][(size_t)k]) {
          const double key = std::max(pos + q * lag, prev_end[(size_t)k] + 1.0);
          keyed.push_back({key, w});
          end[(size_t)k] = std::max(end[(size_t)k], key);
          pos += (double)(w.r1 - w.r0) * p.r * 8.0;
        }
      }
      prev_end = end;
    }
    std::stable_sort(keyed.begin(), keyed.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    for (auto& kv : keyed) work.push_back(kv.second);
    for (auto& b : whole) {
      PWork w{};
      w.kind = kPWhole;
      w.first = b.second;
      work.push_back(w);
    }
    for (size_t i = 0; i < small.size(); i += kPWarps) {
      PWork w{};
      w.kind = kPGroup;
      w.first = small[i].second;
      w.count = (int32_t)std::min<size_t>(kPWarps, small.size() - i);
      work.push_back(w);
    }
    h.n_pitems = (int64_t)work.size();
    for (void* q : {h.d_pitems, h.d_ppairs, (void*)h.d_tP1, (void*)h.d_tP2, (void*)h.d_ptpart, (void*)h.d_pcount,
                    (void*)h.d_pflags})
      h.release(q);
    h.d_pitems = h.alloc<PWork>(work.size());
    h.d_ppairs = h.alloc<PPair>(ordered.size());
    if (!work.empty())
      H2D_CUDA(cudaMemcpyAsync(h.d_pitems, work.data(), work.size() * sizeof(PWork), cudaMemcpyHostToDevice, s));
    if (!ordered.empty())
      H2D_CUDA(cudaMemcpyAsync(h.d_ppairs, ordered.data(), ordered.size() * sizeof(PPair), cudaMemcpyHostToDevice, s));
    h.d_tP1 = h.alloc<double>(std::max<int64_t>(2, toff + 2));
    h.d_tP2 = h.alloc<double>(std::max<int64_t>(2, toff + 2));
    h.d_ptpart = h.alloc<double>(std::max<int64_t>(1, poff));
    h.d_pcount = h.alloc<int32_t>(std::max<int64_t>(2, 2 * nbig));
    h.d_pflags = h.alloc<int32_t>(std::max<int64_t>(2, 2 * nbig));
    H2D_CUDA(cudaMemsetAsync(h.d_pcount, 0, std::max<int64_t>(2, 2 * nbig) * 4, s));
    H2D_CUDA(cudaMemsetAsync(h.d_pflags, 0, std::max<int64_t>(2, 2 * nbig) * 4, s));
    h.pair_epoch = 0;
    if (!h.d_yacc) h.d_yacc = h.alloc<double>(h.n);
    // CTAs per SM (diagnostics: H2D_PAIR_CTAS): 3 measured faster overall than 2 (which leave
    // the registers for a co-resident near field but run the pairs 1.5x slower)
    h.pair_ctas_per_sm = getenv("H2D_PAIR_CTAS") ? std::max(1, atoi(getenv("H2D_PAIR_CTAS"))) : 3;
  }
  // the log kernel's near field: subnormal-safe table log only if some near pair needs it
  h.p2p_kid = h.kp.id;
  if (h.kp.id == H2D_KERNEL_LOG && h.leaf_end > h.leaf_begin) {
    int* d_flag = nullptr;
    H2D_CUDA(cudaMallocAsync(&d_flag, sizeof(int), s));
    H2D_CUDA(cudaMemsetAsync(d_flag, 0, sizeof(int), s));
    const int64_t nl = h.adaptive ? (int64_t)h.lf_code.size() : ((int64_t)1 << (2 * h.kappa));
    const int grid = (int)std::min<int64_t>(nl, 148 * 16);
    subnormal_check_kernel<<<grid, 128, 0, s>>>(h.kappa, nl, h.adaptive ? h.d_lf_start : h.d_leaf_start,
                                                h.adaptive ? h.d_ad_nf_off : nullptr,
                                                h.adaptive ? h.d_ad_nf_rng : nullptr, h.d_px, h.d_py, d_flag);
    H2D_LAUNCH_CHECK();
    int flag = 0;
    H2D_CUDA(cudaMemcpyAsync(&flag, d_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    H2D_CUDA(cudaStreamSynchronize(s));
    H2D_CUDA(cudaFreeAsync(d_flag, s));
    if (flag & 1) h.p2p_kid = kLogSafe;
    else if (!(flag & 2) && !getenv("H2D_P2P_SELECT")) h.p2p_kid = kLogNoSel;   // (diagnostics: keep the select)
  }
  h.tpart_len = tpart_len;
  h.d_tpart = h.alloc<double>(tpart_len);
  h.n_aitems = (int64_t)aitems.size();
  h.n_ritems = (int64_t)ritems.size();
  h.n_bitems = (int64_t)bsorted.size();
  h.d_aitems = h.alloc<AItem>(aitems.size());
  h.d_ritems = h.alloc<RItem>(ritems.size());
  h.d_rcount = h.alloc<int32_t>(ritems.size());
  h.d_bitems = h.alloc<BItem>(bsorted.size());
  h.d_blev = h.alloc<BLevel>(blev.size());
  if (!blev.empty())
    H2D_CUDA(cudaMemcpyAsync(h.d_blev, blev.data(), blev.size() * sizeof(BLevel), cudaMemcpyHostToDevice, s));
  H2D_CUDA(cudaMemsetAsync(h.d_rcount, 0, std::max<size_t>(1, ritems.size()) * sizeof(int32_t), s));
  if (!aitems.empty())
    H2D_CUDA(cudaMemcpyAsync(h.d_aitems, aitems.data(), aitems.size() * sizeof(AItem),
                             cudaMemcpyHostToDevice, s));
  if (!ritems.empty())
    H2D_CUDA(cudaMemcpyAsync(h.d_ritems, ritems.data(), ritems.size() * sizeof(RItem),
                             cudaMemcpyHostToDevice, s));
  if (!bsorted.empty())
    H2D_CUDA(cudaMemcpyAsync(h.d_bitems, bsorted.data(), bsorted.size() * sizeof(BItem),
                             cudaMemcpyHostToDevice, s));
  if (!h.d_ynear) h.d_ynear = h.alloc<double>(3 * h.n);   // three P2P slots (p2p_sym_kernel)
  if (h.adaptive)   // the list kernel writes slot 0 only; the combine reads all three
    H2D_CUDA(cudaMemsetAsync(h.d_ynear + h.n, 0, 2 * h.n * sizeof(double), s));
  if (!h.d_yfar) h.d_yfar = h.alloc<double>(std::max<int64_t>(1, h.row_end - h.row_begin));
  if (!h.d_counters) h.d_counters = h.alloc<int32_t>(12);   // 0 A, 1 B, 2 P2P fast, 3 B', 4-6 P2P warp, 7 A remote, 8 pairs
  if (!h.hi_stream) {
    int sm = 0, lo_prio = 0, hi_prio = 0;
    H2D_CUDA(cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, h.device));
    H2D_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
    H2D_CUDA(cudaStreamCreateWithPriority(&h.hi_stream, cudaStreamNonBlocking, hi_prio));
    H2D_CUDA(cudaStreamCreateWithPriority(&h.aux_stream, cudaStreamNonBlocking, lo_prio));
    H2D_CUDA(cudaEventCreateWithFlags(&h.ev_fork, cudaEventDisableTiming));
    H2D_CUDA(cudaEventCreateWithFlags(&h.ev_join, cudaEventDisableTiming));
    H2D_CUDA(cudaEventCreateWithFlags(&h.ev_far, cudaEventDisableTiming));
    H2D_CUDA(cudaEventCreateWithFlags(&h.ev_p2p_fork, cudaEventDisableTiming));
    for (int k = 0; k < 3; ++k) {
      H2D_CUDA(cudaStreamCreateWithPriority(&h.p2p_side[k], cudaStreamNonBlocking, lo_prio));
      H2D_CUDA(cudaEventCreateWithFlags(&h.ev_p2p_side[k], cudaEventDisableTiming));
    }
    // pipeline shape: 2 CTAs/SM with a 5-stage ring, or 1 CTA/SM with a 9-stage ring
    // (leaves room for two P2P CTAs per SM); H2D_PIPE_CTAS_PER_SM overrides the default.
    const char* env = getenv("H2D_PIPE_CTAS_PER_SM");
    const int per_sm = env && atoi(env) == 2 ? 2 : env && atoi(env) == 1 ? 1 : kDefaultCtasPerSm;
    h.pipe_ns = per_sm == 2 ? kNSShallow : kNSDeep;
    h.persist_ctas = per_sm * sm;
    set_pipe_attrs<kNSShallow>();
    set_pipe_attrs<kNSDeep>();
    {
      const int dsm = (int)sizeof(PipeSmem<kNSDual, kSDDual>);
      H2D_CUDA(cudaFuncSetAttribute(stageA_dual_kernel<kNSDual, kSDDual>, cudaFuncAttributeMaxDynamicSharedMemorySize, dsm));
      H2D_CUDA(cudaFuncSetAttribute(stageA_dual_kernel<kNSDual, kSDDual>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                    cudaSharedmemCarveoutMaxShared));
    }
    for (const void* f : {(const void*)p2p_sym_kernel<H2D_KERNEL_LOG>, (const void*)p2p_sym_kernel<H2D_KERNEL_IMQ>,
                          (const void*)p2p_sym_kernel<H2D_KERNEL_ONE_OVER_R>,
                          (const void*)p2p_sym_kernel<H2D_KERNEL_TEST_LOWRANK>,
                          (const void*)p2p_sym_kernel<H2D_KERNEL_RBF_PHI1>,
                          (const void*)p2p_sym_kernel<H2D_KERNEL_RBF_PHI2>,
                          (const void*)p2p_fast_kernel<H2D_KERNEL_LOG>, (const void*)p2p_fast_kernel<H2D_KERNEL_IMQ>,
                          (const void*)p2p_fast_kernel<H2D_KERNEL_ONE_OVER_R>,
                          (const void*)p2p_fast_kernel<H2D_KERNEL_RBF_PHI1>,
                          (const void*)p2p_fast_kernel<H2D_KERNEL_RBF_PHI2>})
      H2D_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout,
                                    cudaSharedmemCarveoutMaxShared));
    h.num_sms = sm;
  }
  if (h.p2p_kid == kLogNoSel && h.n_p2p_warp > 0) pick_log_table(h, s);
  h.list_repl = false;
  if (h.n_p2p_list > 0 && h.p2p_kid != kLogSafe && (h.kp.id == H2D_KERNEL_LOG || h.kp.id == H2D_KERNEL_RBF_PHI1))
    pick_list_table(h, s);
  H2D_CUDA(cudaMemsetAsync(h.d_counters, 0, 4 * sizeof(int32_t), s));
  H2D_CUDA(cudaStreamSynchronize(s));
}

void permute_in(Handle& h, const double* d_x, double* d_xtree) {
  int blocks = (int)std::min<int64_t>((h.n + 255) / 256, 148 * 16);
  permute_in_kernel<<<blocks, 256, 0, h.stream>>>(d_x, h.d_perm, h.n, d_xtree);
  H2D_LAUNCH_CHECK();
}

static void record(Handle& h, int slot, cudaStream_t s) {
  if (!h.timing) return;
  const int64_t idx = h.ev_base + slot;
  while ((int64_t)h.ev_pool.size() <= idx) {
    cudaEvent_t e;
    H2D_CUDA(cudaEventCreate(&e));
    h.ev_pool.push_back(e);
  }
  H2D_CUDA(cudaEventRecord(h.ev_pool[(size_t)idx], s));
}

void begin_matvec_timing(Handle& h) {
  if (!h.timing) return;
  h.ev_base = h.ev_used;
  h.ev_used += kEventsPerMatvec;
  record(h, 0, h.stream);
}

void mark_after_input(Handle& h) { record(h, 1, h.stream); }

template <int NS, int SD, int SV>
static void launch_stageB_geom(Handle& h, cudaStream_t hi) {
  static uint64_t seen = 0;
  const size_t smem = sizeof(PipeSmem<NS, SD, SV>);
  once_per_device(seen, [&] {
    H2D_CUDA(cudaFuncSetAttribute(stageB_tma_kernel<NS, SD, SV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    H2D_CUDA(cudaFuncSetAttribute(stageB_tma_kernel<NS, SD, SV>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  cudaSharedmemCarveoutMaxShared));
  });
  // persistent grid, but never more CTAs than items (small operators: ring set-up per CTA)
  stageB_tma_kernel<NS, SD, SV><<<(int)std::min<int64_t>(h.persist_ctas, h.n_bbig), kPipeThreads, smem, hi>>>(
      h.d_bitems, h.d_blev, (int)h.n_bbig, h.d_counters + 1, h.kappa, h.lp, h.d_yfar);
  H2D_LAUNCH_CHECK();
}

// part: stage A only — 0 all small items, 1 the local ones, 2 the rest (H2D_ORDER_LOCAL)
static void launch_small(Handle& h, bool stage_a, const double* d_xtree, double* t, cudaStream_t hi,
                         int part = 0) {
  int64_t first = stage_a ? h.n_abig : h.n_bbig;
  int64_t n = stage_a ? h.n_aitems - h.n_abig : h.n_bitems - h.n_bbig;
  if (stage_a && part == 1) n = h.n_asmall_loc;
  if (stage_a && part == 2) { first += h.n_asmall_loc; n -= h.n_asmall_loc; }
  if (n <= 0) return;
  // 16 CTAs x 8 warps per SM requested: the warps are latency-bound on their own loads
  const int grid = (int)std::min<int64_t>((int64_t)h.num_sms * 16, (n + 7) / 8);
  if (stage_a)
    stageA_small_kernel<<<grid, 256, 0, hi>>>(h.d_aitems + first, (int)n, h.lp, d_xtree, h.d_vdst, t);
  else
    stageB_small_kernel<<<grid, 256, 0, hi>>>(h.d_bitems + h.n_bbig, h.d_blev + h.n_bbig * h.kappa, (int)n,
                                              h.kappa, h.lp, h.d_yfar);
  H2D_LAUNCH_CHECK();
}

static void launch_stageB(Handle& h, cudaStream_t hi) {
  launch_small(h, false, nullptr, nullptr, hi);
  if (h.n_bbig <= 0) return;
  // (a 2 x 44 KB ring measured 1 % slower on C3; 5 x 16 KB stays)
  if (h.pipe_ns == kNSDeep) launch_stageB_geom<kNSDeep, kStageDbl, kStageVec>(h, hi);
  else launch_stageB_geom<kNSShallow, kStageDbl, kStageVec>(h, hi);
}

// Stage A then stage B on the high-priority stream.  gather (H2D_ORDER_LOCAL): only the
// served rows of x_tree are valid at the start; the items whose column box is local run
// first (ring items on counter 0, their own small-item launch), then the host-staged
// exchange (if any) runs on this thread while they stream, then this stream waits for the
// gathered slots, unpads them and runs the remaining items (counter 7) and stage B.
template <int NS>
static void launch_stages(Handle& h, const double* d_xtree, cudaStream_t hi, bool gather, cudaEvent_t* xready,
                          bool mark_a) {
  const size_t smem = sizeof(PipeSmem<NS>);
  auto ring = [&](int64_t first, int64_t cnt, int32_t* counter) {
    if (cnt <= 0) return;
    stageA_tma_kernel<NS><<<(int)std::min<int64_t>(h.persist_ctas, cnt), kPipeThreads, smem, hi>>>(
        h.d_aitems + first, (int)cnt, counter, h.lp, d_xtree, h.d_vdst, h.d_t, h.d_tpart, h.d_ritems, h.d_rcount);
    H2D_LAUNCH_CHECK();
  };
  if (!gather) {
    if (!h.small_a_after) launch_small(h, true, d_xtree, h.d_t, hi);
    ring(0, h.n_abig, h.d_counters);
    if (h.small_a_after) launch_small(h, true, d_xtree, h.d_t, hi);
  } else {
    launch_small(h, true, d_xtree, h.d_t, hi, 1);
    ring(0, h.n_abig_loc, h.d_counters);
    comm_gather_exchange(h);
    *xready = comm_gather_finish(h, h.d_xtree, hi);   // (gather: d_xtree == h.d_xtree)
    launch_small(h, true, d_xtree, h.d_t, hi, 2);
    ring(h.n_abig_loc, h.n_abig - h.n_abig_loc, h.d_counters + 7);
  }
  if (mark_a) {   // the near field waits for stage A (place_pick)
    if (!h.ev_b1) H2D_CUDA(cudaEventCreateWithFlags(&h.ev_b1, cudaEventDisableTiming));
    H2D_CUDA(cudaEventRecord(h.ev_b1, hi));
  }
  record(h, 2, hi);
  launch_stageB(h, hi);
}

// Near-field placement of a directed single-pass matvec: the P2P runs beside stage A (launched
// with it, the default) or beside stage B (waits for stage A's launches).  Which one hides it
// better depends on the GPU's power state more than on the input (profiles/r02ai_place.md): in
// the bench (after C3 has run, sw_power_cap) C4 is 67.8 matvecs/s beside A and 64.0 beside B;
// in a probe run straight after the build it is 61.8 beside A and 67.5 beside B; C3 is within
// noise either way.  Results are identical (same kernels, same per-row order).
// set_diag("p2p_place", 1) forces stage B; -1 times it: matvec calls 1-2 beside A, 3-4 beside
// B (call 0 is a warm-up), then keeps the faster once those events have completed (the bench's
// C4 shows that early calls can mislead it: measured, not the default).
static bool place_pick(Handle& h, int& slot) {
  slot = -1;
  if (h.p2p_place >= 0) return h.p2p_place == 1;
  const int c = h.place_calls;
  if (c < 5) ++h.place_calls;
  if (c >= 1 && c <= 4) {
    slot = c - 1;
    for (cudaEvent_t& e : h.place_ev[slot])
      if (!e) H2D_CUDA(cudaEventCreate(&e));
    return slot >= 2;
  }
  if (c < 5) return false;
  float t[4];
  for (int k = 0; k < 4; ++k) {
    const cudaError_t q = cudaEventQuery(h.place_ev[k][1]);
    if (q == cudaErrorNotReady) {
      (void)cudaGetLastError();   // not sticky; decide on a later call
      return false;
    }
    H2D_CUDA(q);
    H2D_CUDA(cudaEventElapsedTime(&t[k], h.place_ev[k][0], h.place_ev[k][1]));
  }
  h.p2p_place = t[2] + t[3] < t[0] + t[1] ? 1 : 0;
  if (getenv("H2D_VERBOSE")) fprintf(stderr, "[h2d] near field beside stage %c (A %.3f + %.3f ms, B %.3f + %.3f ms)\n",
                         h.p2p_place ? 'B' : 'A', t[0], t[1], t[2], t[3]);
  return h.p2p_place == 1;
}

// Matvec on TREE-order x (S7-S9).  Stages A and B (HBM-bound) run on the high-priority
// stream, the near-field P2P (FP64-bound) concurrently on the low-priority stream; the
// combine epilogue on the caller's stream joins them.
void matvec_tree(Handle& h, const double* d_xtree, double* d_y, int order_out, int64_t y_row0, bool gather) {
  cudaStream_t s = h.stream, hi = h.hi_stream, a = h.aux_stream;
  const int64_t nleaves = h.leaf_end - h.leaf_begin;
  // H2D_P2P_SERIAL=1 (diagnostics only): the P2P runs alone, before stage A
  const bool p2p_serial = h.diag_p2p_serial && !gather;
  if (gather && (h.symapply || h.pairapply)) {   // (single-rank symmetric handle: gather first, no overlap)
    comm_gather_exchange(h);
    comm_gather_finish(h, h.d_xtree, s);
    gather = false;
  }
  int place_slot = -1;
  const bool beside_b = !h.symapply && !h.pairapply && !gather && !p2p_serial && place_pick(h, place_slot);
  if (place_slot >= 0) H2D_CUDA(cudaEventRecord(h.place_ev[place_slot][0], s));
  cudaEvent_t xready = nullptr;
  H2D_CUDA(cudaEventRecord(h.ev_fork, s));
  H2D_CUDA(cudaStreamWaitEvent(hi, h.ev_fork, 0));
  H2D_CUDA(cudaStreamWaitEvent(a, h.ev_fork, 0));
  // H2D_P2P_ONESTREAM=1 (diagnostics only): every P2P class on aux_stream, one after another
  const bool p2p_one = h.diag_p2p_onestream;
  auto p2p = [&]() {
    record(h, 6, a);
    // an under-filled class (fewer CTAs than SMs: the big leaves of a clustered input) runs on
    // a side stream and no longer serialises the rest; full-grid classes stay one after another
    // on aux_stream (two of them at once measured 1 % slower on the C3 symmetric apply)
    bool forked[3] = {false, false, false};
    auto side = [&](int k) -> cudaStream_t {
      if (p2p_one) return a;
      if (!forked[k]) {
        if (!forked[0] && !forked[1] && !forked[2]) H2D_CUDA(cudaEventRecord(h.ev_p2p_fork, a));
        H2D_CUDA(cudaStreamWaitEvent(h.p2p_side[k], h.ev_p2p_fork, 0));
        forked[k] = true;
      }
      return h.p2p_side[k];
    };
    if (h.n_p2p_list > 0) {   // adaptive near field (R24)
      auto* kfn = h.p2p_kid == kLogSafe ? p2p_list_kernel<kLogSafe>
                : h.kp.id == H2D_KERNEL_LOG ? (h.list_repl ? p2p_list_kernel<kLogRepl> : p2p_list_kernel<H2D_KERNEL_LOG>)
                : h.kp.id == H2D_KERNEL_IMQ ? p2p_list_kernel<H2D_KERNEL_IMQ>
                : h.kp.id == H2D_KERNEL_ONE_OVER_R ? p2p_list_kernel<H2D_KERNEL_ONE_OVER_R>
                : h.kp.id == H2D_KERNEL_RBF_PHI1 ? (h.list_repl ? p2p_list_kernel<kPhi1Repl>
                                                                : p2p_list_kernel<H2D_KERNEL_RBF_PHI1>)
                : h.kp.id == H2D_KERNEL_RBF_PHI2 ? p2p_list_kernel<H2D_KERNEL_RBF_PHI2>
                                                   : p2p_list_kernel<H2D_KERNEL_TEST_LOWRANK>;
      H2D_CUDA(cudaMemsetAsync(h.d_counters + 4, 0, sizeof(int32_t), a));
      // beside the streams: one CTA per SM (66 registers x 256 threads), so that the two ring
      // CTAs of stage A / B' still fit on every SM (at 3 per SM, placed while the small-item
      // kernel drained, the list kernel held whole SMs: adaptive 1000^2 A' + B' 2.3 -> 3.0 ms)
      const int per_sm = p2p_serial ? 3 : h.diag_p2p_list_ctas;
      const int grid = (int)std::min<int64_t>((int64_t)h.num_sms * per_sm, (h.n_p2p_list + 7) / 8);
      kfn<<<grid, 256, 0, a>>>(h.d_p2p_list, (int)h.n_p2p_list, h.d_counters + 4, h.d_lf_start, h.d_ad_nf_off,
                               h.d_ad_nf_rng, h.d_px, h.d_py, d_xtree, h.kp, h.d_ynear);
      H2D_LAUNCH_CHECK();
    }
    if (h.n_p2p_gen > 0) {
      cudaStream_t sg = h.n_p2p_gen < h.num_sms ? side(0) : a;
      auto* kfn = h.p2p_kid == kLogSafe ? p2p_sym_kernel<kLogSafe>
                : h.kp.id == H2D_KERNEL_LOG ? p2p_sym_kernel<H2D_KERNEL_LOG>
                : h.kp.id == H2D_KERNEL_IMQ ? p2p_sym_kernel<H2D_KERNEL_IMQ>
                : h.kp.id == H2D_KERNEL_ONE_OVER_R ? p2p_sym_kernel<H2D_KERNEL_ONE_OVER_R>
                : h.kp.id == H2D_KERNEL_RBF_PHI1 ? p2p_sym_kernel<H2D_KERNEL_RBF_PHI1>
                : h.kp.id == H2D_KERNEL_RBF_PHI2 ? p2p_sym_kernel<H2D_KERNEL_RBF_PHI2>
                                                   : p2p_sym_kernel<H2D_KERNEL_TEST_LOWRANK>;
      kfn<<<(int)h.n_p2p_gen, 256, 0, sg>>>(h.kappa, h.leaf_begin, h.leaf_end, h.d_p2p_gen,
                                           h.d_leaf_start, h.d_px, h.d_py, d_xtree, h.kp, h.d_ynear,
                                           h.d_ynear + h.n, h.d_ynear + 2 * h.n);
      H2D_LAUNCH_CHECK();
    }
    if (h.n_p2p_fast > 0) {
      auto* kfn = h.p2p_kid == kLogSafe ? p2p_fast_kernel<kLogSafe>
                : h.kp.id == H2D_KERNEL_LOG ? p2p_fast_kernel<H2D_KERNEL_LOG>
                : h.kp.id == H2D_KERNEL_IMQ ? p2p_fast_kernel<H2D_KERNEL_IMQ>
                : h.kp.id == H2D_KERNEL_ONE_OVER_R ? p2p_fast_kernel<H2D_KERNEL_ONE_OVER_R>
                : h.kp.id == H2D_KERNEL_RBF_PHI1 ? p2p_fast_kernel<H2D_KERNEL_RBF_PHI1>
                                                 : p2p_fast_kernel<H2D_KERNEL_RBF_PHI2>;
      H2D_CUDA(cudaMemsetAsync(h.d_counters + 2, 0, sizeof(int32_t), a));
      const int grid = (int)std::min<int64_t>(h.num_sms, h.n_p2p_fast);
      kfn<<<grid, 256, 0, a>>>(h.kappa, h.d_p2p_fast, (int)h.n_p2p_fast, h.d_counters + 2,
                               h.d_leaf_start, h.d_px, h.d_py, d_xtree, h.kp, h.d_ynear,
                               h.d_ynear + h.n, h.d_ynear + 2 * h.n);
      H2D_LAUNCH_CHECK();
    }
    if (h.n_p2p_warp > 0) {
      int64_t off = 0;
      for (int r = 0; r < 3; ++r) {
        const int64_t cnt = h.n_p2p_warp_rpl[r];
        if (cnt <= 0) continue;
        auto pick = [&](auto rpl) -> decltype(&p2p_warp_kernel<H2D_KERNEL_LOG, 1>) {
          constexpr int R = decltype(rpl)::value;
          return h.p2p_kid == kLogSafe ? p2p_warp_kernel<kLogSafe, R>
               : h.p2p_kid == kLogNoSel ? p2p_warp_kernel<kLogNoSel, R>
               : h.p2p_kid == kLogNoSelRepl ? p2p_warp_kernel<kLogNoSelRepl, R>
               : h.kp.id == H2D_KERNEL_LOG ? p2p_warp_kernel<H2D_KERNEL_LOG, R>
               : h.kp.id == H2D_KERNEL_IMQ ? p2p_warp_kernel<H2D_KERNEL_IMQ, R>
               : h.kp.id == H2D_KERNEL_ONE_OVER_R ? p2p_warp_kernel<H2D_KERNEL_ONE_OVER_R, R>
               : h.kp.id == H2D_KERNEL_RBF_PHI1 ? p2p_warp_kernel<H2D_KERNEL_RBF_PHI1, R>
                                                : p2p_warp_kernel<H2D_KERNEL_RBF_PHI2, R>;
        };
        auto* kfn = r == 0 ? pick(std::integral_constant<int, 1>{})
                  : r == 1 ? pick(std::integral_constant<int, 2>{}) : pick(std::integral_constant<int, 3>{});
        // beside the streams one CTA per SM fits (registers); run alone (p2p_serial) the near
        // field has the GPU and 4 CTAs per SM hide its dependent DFMA chains
        const int grid = (int)std::min<int64_t>((p2p_serial ? 4 : 1) * (int64_t)h.num_sms, (cnt + 7) / 8);
        cudaStream_t sw = r > 0 && grid < h.num_sms ? side(3 - r) : a;
        H2D_CUDA(cudaMemsetAsync(h.d_counters + 4 + r, 0, sizeof(int32_t), sw));
        kfn<<<grid, 256, 0, sw>>>(h.kappa, h.d_p2p_warp + off, (int)cnt, h.d_counters + 4 + r, h.d_leaf_start,
                                 h.d_px, h.d_py, d_xtree, h.kp, h.d_ynear, h.d_ynear + h.n, h.d_ynear + 2 * h.n);
        H2D_LAUNCH_CHECK();
        off += cnt;
      }
    }
    for (int k = 0; k < 3; ++k)
      if (forked[k]) {
        H2D_CUDA(cudaEventRecord(h.ev_p2p_side[k], h.p2p_side[k]));
        H2D_CUDA(cudaStreamWaitEvent(a, h.ev_p2p_side[k], 0));
      }
    record(h, 7, a);
    H2D_CUDA(cudaEventRecord(h.ev_join, a));
  };
  if (p2p_serial) {
    p2p();
    H2D_CUDA(cudaStreamWaitEvent(hi, h.ev_join, 0));
  }
  if (h.pairapply) {
    // pair-local symmetric apply (pairs.cuh): every factor read once; dy -> yacc
    PairPtrs pp{};
    for (int l = 1; l <= h.kappa; ++l) pp.P[l] = h.levels[(size_t)l].Pr;
    H2D_CUDA(cudaMemsetAsync(h.d_yacc, 0, h.n * sizeof(double), hi));
    H2D_CUDA(cudaMemsetAsync(h.d_counters + 8, 0, sizeof(int32_t), hi));
    ++h.pair_epoch;
    if (h.n_pitems > 0) {
      pair_apply_kernel<<<(int)std::min<int64_t>(h.pair_ctas_per_sm * (int64_t)h.num_sms, h.n_pitems), 32 * kPWarps,
                          0, hi>>>(
          (const PWork*)h.d_pitems, (int)h.n_pitems, (const PPair*)h.d_ppairs, h.d_counters + 8, pp, d_xtree,
          h.d_yacc, h.d_tP1, h.d_tP2, h.d_ptpart, h.d_pcount, h.d_pflags, h.pair_epoch);
      H2D_LAUNCH_CHECK();
    }
    record(h, 2, hi);
  } else if (h.symapply) {
    // symmetric apply (R23): A' t1 = V^T x; B' t2 = U^T x and y1 = U t1; C' yfar = V t2
    const size_t smem = sizeof(PipeSmem<kNSShallow>);
    H2D_CUDA(cudaMemsetAsync(h.d_counters, 0, 4 * sizeof(int32_t), hi));
    if (!h.small_a_after) launch_small(h, true, d_xtree, h.d_t1, hi);
    if (h.n_abig > 0) {
      stageA_tma_kernel<kNSShallow><<<(int)std::min<int64_t>(h.persist_ctas, h.n_abig), kPipeThreads, smem, hi>>>(
          h.d_aitems, (int)h.n_abig, h.d_counters, h.lp, d_xtree, h.d_vdst, h.d_t1, h.d_tpart, h.d_ritems,
          h.d_rcount);
      H2D_LAUNCH_CHECK();
    }
    if (h.small_a_after) launch_small(h, true, d_xtree, h.d_t1, hi);
    if (h.n_b1big > 0) {
      stageA_dual_kernel<kNSDual, kSDDual><<<(int)std::min<int64_t>(h.persist_ctas, h.n_b1big), kPipeThreads,
                                             sizeof(PipeSmem<kNSDual, kSDDual>), hi>>>(
          h.d_b1items, (int)h.n_b1big, h.d_counters + 3, h.lp, d_xtree, h.d_udst, h.d_t, h.d_b1tpart,
          h.d_b1ritems, h.d_b1rcount, h.d_t1, h.d_y1,
          h.diag_dual_norow ? (int64_t)-1 : h.n);   // diagnostics: skip the row dots
      H2D_LAUNCH_CHECK();
    }
    if (h.n_b1items > h.n_b1big) {
      const int64_t nb = h.n_b1items - h.n_b1big;
      const int grid = (int)std::min<int64_t>((int64_t)h.num_sms * 16, (nb + 7) / 8);
      stageB1_small_kernel<<<grid, 256, 0, hi>>>(h.d_b1items + h.n_b1big, (int)nb, h.lp, d_xtree, h.d_udst, h.d_t,
                                                  h.d_t1, h.d_y1, h.n);
      H2D_LAUNCH_CHECK();
    }
    if (h.p2p_after_b1) {   // diagnostics: the near field only beside C'
      if (!h.ev_b1) H2D_CUDA(cudaEventCreateWithFlags(&h.ev_b1, cudaEventDisableTiming));
      H2D_CUDA(cudaEventRecord(h.ev_b1, hi));
    }
    record(h, 2, hi);
    launch_stageB(h, hi);
  } else {
    H2D_CUDA(cudaMemsetAsync(h.d_counters, 0, 2 * sizeof(int32_t), hi));
    if (gather) H2D_CUDA(cudaMemsetAsync(h.d_counters + 7, 0, sizeof(int32_t), hi));
    if (h.pipe_ns == kNSShallow) launch_stages<kNSShallow>(h, d_xtree, hi, gather, &xready, beside_b);
    else launch_stages<kNSDeep>(h, d_xtree, hi, gather, &xready, beside_b);
  }
  record(h, 3, hi);
  H2D_CUDA(cudaEventRecord(h.ev_far, hi));
  if (xready) H2D_CUDA(cudaStreamWaitEvent(a, xready, 0));   // the near field reads remote x
  if (h.symapply && h.p2p_after_b1 && !p2p_serial) H2D_CUDA(cudaStreamWaitEvent(a, h.ev_b1, 0));
  if (beside_b) H2D_CUDA(cudaStreamWaitEvent(a, h.ev_b1, 0));
  if (!p2p_serial) p2p();   // after stage A's launch: its CTAs are placed first
  H2D_CUDA(cudaStreamWaitEvent(s, h.ev_far, 0));
  H2D_CUDA(cudaStreamWaitEvent(s, h.ev_join, 0));
  record(h, 4, s);
  const int64_t rows = h.row_end - h.row_begin;
  if (rows > 0) {
    const int blocks = (int)std::min<int64_t>((rows + 255) / 256, 148 * 8);
    if (h.pairapply)
      combine_kernel<<<blocks, 256, 0, s>>>(h.row_begin, rows, h.d_yacc + h.row_begin, h.d_ynear, h.n, d_xtree,
                                            h.kp.scale, h.kp.shift, d_y, h.d_perm, order_out, y_row0);
    else if (h.symapply)
      combine_sym_kernel<<<blocks, 256, 0, s>>>(h.row_begin, rows, h.kappa, h.d_yfar, h.d_y1, h.d_ynear, h.n, d_xtree, h.kp.scale,
                                                h.kp.shift, d_y, h.d_perm, order_out, y_row0);
    else
      combine_kernel<<<blocks, 256, 0, s>>>(h.row_begin, rows, h.d_yfar, h.d_ynear, h.n, d_xtree,
                                            h.kp.scale, h.kp.shift, d_y, h.d_perm, order_out, y_row0);
    H2D_LAUNCH_CHECK();
  }
  record(h, 5, s);
  if (place_slot >= 0) H2D_CUDA(cudaEventRecord(h.place_ev[place_slot][1], s));
}

}  // namespace h2d
