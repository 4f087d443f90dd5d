// Factor packing (G7) and the matvec hot path (S7-S10).
//
// HBM layout:
//   U panel of row box X at level l : column-major m_X x R_X, the concatenation
//                                     [U_b1 | U_b2 | ...] of the blocks (X, Y), Y in I_X
//                                     ascending.  A leaf L inside X owns the contiguous
//                                     row segment [a, a + |L|) of every column.
//   V panel of column box Y         : row-major n_Y x RV_Y, the columns of the blocks
//                                     (X, Y), X in I_Y ascending.  Row i of the panel is the
//                                     RV_Y values that multiply x_i.
//   t                               : one value per (block, rank index) in U-panel column
//                                     order, so a row box's t is contiguous; stage A writes
//                                     it through vdst (V-panel column -> t position).
// Matvec (Alg. 2; stage order is free, R18):
//   p2p      ynear = shift x + scale K_near x  (second stream, overlaps stage A)
//   stage A  t = V^T x          one CTA per (column box, row chunk)
//   reduce   t = sum of chunk partials (boxes split over several CTAs only)
//   stage B  per leaf L: y_L = ynear_L + sum_l U_{X_l}[rows of L, :] t_{X_l}
//                               one CTA per leaf, one y write per row, no atomics.
#include <algorithm>

#include "h2d_internal.cuh"

namespace h2d {
namespace {

constexpr int kAThreads = 256;
constexpr int kBThreads = 256;
constexpr int64_t kATarget = 65536;  // stage-A elements per CTA
constexpr int kAMaxRows = 16384;     // rows per stage-A chunk
constexpr int kBUnroll = 8;

struct CopyItem {
  const double* src;
  double* dst;
  int64_t count;
};
__global__ void copy_items_kernel(const CopyItem* __restrict__ items) {
  const CopyItem it = items[blockIdx.x];
  for (int64_t i = threadIdx.x; i < it.count; i += blockDim.x) it.dst[i] = it.src[i];
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

// ---------------------------------------------------------------- stage A: t = V^T x
// The chunk is a contiguous row-major block nrows x R of the V panel.  Lane l owns the
// panel columns q0 + l + 32c (c < CPL) and warp w the rows w, w+8, ...: each row is one
// coalesced 32*CPL-double read at constant offsets, x_i is a warp-uniform broadcast load,
// 8 loads in flight per thread, partial sums reduced over the 8 warps in shared memory.
template <int CPL>
__device__ __forceinline__ void stageA_cols(const double* __restrict__ V, int R, int nrows, int q0,
                                            int W, const double* __restrict__ xx,
                                            double (&acc)[8]) {
  constexpr int RU = CPL >= 5 ? 1 : CPL >= 3 ? 2 : CPL == 2 ? 4 : 8;   // rows per step
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  bool valid[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) valid[c] = lane + 32 * c < W;
  const int64_t rstep = (int64_t)8 * R;
  // rows of this warp: w + 8k.  x for 32 of them is fetched by one coalesced load and
  // broadcast by shuffles.
  for (int k0 = 0; w + 8 * k0 < nrows; k0 += 32) {
    const int ib = w + 8 * k0;
    const int nk = min(32, (nrows - ib + 7) >> 3);
    const double xl = lane < nk ? __ldg(xx + ib + 8 * lane) : 0.0;
    const double* __restrict__ p = V + (int64_t)ib * R + q0 + lane;
    int k = 0;
    for (; k + RU <= nk; k += RU, p += RU * rstep) {
      double v[RU][CPL];
#pragma unroll
      for (int u = 0; u < RU; ++u)
#pragma unroll
        for (int c = 0; c < CPL; ++c) v[u][c] = valid[c] ? __ldcs(p + u * rstep + 32 * c) : 0.0;
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        const double xv = __shfl_sync(0xffffffffu, xl, k + u);
#pragma unroll
        for (int c = 0; c < CPL; ++c) acc[c] = fma(v[u][c], xv, acc[c]);
      }
    }
    for (; k < nk; ++k, p += rstep) {
      const double xv = __shfl_sync(0xffffffffu, xl, k);
#pragma unroll
      for (int c = 0; c < CPL; ++c) acc[c] = fma(valid[c] ? __ldcs(p + 32 * c) : 0.0, xv, acc[c]);
    }
  }
}

__global__ void __launch_bounds__(kAThreads, 4)
stageA_kernel(const AItem* __restrict__ items, LevelPtrs lp, const double* __restrict__ x,
              const int32_t* __restrict__ vdst, double* __restrict__ t,
              double* __restrict__ tpart, const RItem* __restrict__ ritems,
              int32_t* __restrict__ rcount) {
  __shared__ double red[8][256];
  __shared__ int s_last;
  const AItem it = items[blockIdx.x];
  const double* __restrict__ V = lp.V[it.level] + it.v_off;
  const double* __restrict__ xx = x + it.x_off;
  const int R = it.R, nrows = it.nrows, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int q0 = 0; q0 < R; q0 += 256) {
    const int W = min(R - q0, 256);
    double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    switch ((W + 31) >> 5) {
      case 1: stageA_cols<1>(V, R, nrows, q0, W, xx, acc); break;
      case 2: stageA_cols<2>(V, R, nrows, q0, W, xx, acc); break;
      case 3: stageA_cols<3>(V, R, nrows, q0, W, xx, acc); break;
      case 4: stageA_cols<4>(V, R, nrows, q0, W, xx, acc); break;
      case 5: stageA_cols<5>(V, R, nrows, q0, W, xx, acc); break;
      case 6: stageA_cols<6>(V, R, nrows, q0, W, xx, acc); break;
      case 7: stageA_cols<7>(V, R, nrows, q0, W, xx, acc); break;
      default: stageA_cols<8>(V, R, nrows, q0, W, xx, acc); break;
    }
    if (q0 > 0) __syncthreads();
#pragma unroll
    for (int c = 0; c < 8; ++c) red[w][lane + 32 * c] = acc[c];
    __syncthreads();
    if (tid < W) {
      double s = 0.0;
#pragma unroll
      for (int ww = 0; ww < 8; ++ww) s += red[ww][tid];
      if (it.out >= 0) t[vdst[it.out + q0 + tid]] = s;
      else tpart[(-(int64_t)it.out - 1) + q0 + tid] = s;
    }
  }
  if (it.ritem < 0) return;
  // Multi-chunk box: the last chunk CTA to finish sums the partials in chunk order
  // (deterministic) and resets the counter for the next matvec.
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const RItem ri = ritems[it.ritem];
    s_last = atomicAdd(rcount + it.ritem, 1) == ri.nchunks - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const RItem ri = ritems[it.ritem];
  for (int q = tid; q < ri.R; q += kAThreads) {
    const double* __restrict__ pp = tpart + ri.p_off + q;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int c = 0;
    for (; c + 3 < ri.nchunks; c += 4) {
      a0 += __ldcg(pp + (int64_t)c * ri.R);
      a1 += __ldcg(pp + (int64_t)(c + 1) * ri.R);
      a2 += __ldcg(pp + (int64_t)(c + 2) * ri.R);
      a3 += __ldcg(pp + (int64_t)(c + 3) * ri.R);
    }
    for (; c < ri.nchunks; ++c) a0 += __ldcg(pp + (int64_t)c * ri.R);
    t[vdst[ri.vpos + q]] = (a0 + a1) + (a2 + a3);
  }
  if (tid == 0) rcount[it.ritem] = 0;
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

// log(r2) for r2 > 0 (normal): r2 = 2^e m, m in [1, 2); c_k = 1 + (k + 1/2)/128 is the
// centre of m's 1/128 bin (k = top 7 mantissa bits), tab[k] = (1/c_k, log c_k);
// log r2 = e ln2 + log c_k + log1p(f), f = m/c_k - 1 in (-2^-8, 2^-8), log1p by its
// degree-8 Taylor polynomial.  11 FP64 operations instead of libdevice's 29; absolute
// error < 1e-15 (checked against libm over [1e-14, 8] when written).
__device__ __forceinline__ double log_r2_fast(double r2, const double2* __restrict__ tab) {
  const long long bits = __double_as_longlong(r2);
  const int e = (int)(bits >> 52) - 1023;
  const int k = (int)((bits >> 45) & 127);
  const double mnt = __longlong_as_double((bits & 0x000FFFFFFFFFFFFFLL) | 0x3FF0000000000000LL);
  const double2 tb = tab[k];
  const double f = fma(mnt, tb.x, -1.0);
  double p = fma(f, -0.125, 1.0 / 7.0);
  p = fma(f, p, -1.0 / 6.0);
  p = fma(f, p, 0.2);
  p = fma(f, p, -0.25);
  p = fma(f, p, 1.0 / 3.0);
  p = fma(f, p, -0.5);
  p = fma(f, p, 1.0);
  const double ed = (double)e;
  return fma(ed, 0.6931471805599453, fma(p, f, fma(ed, 2.3190468138462996e-17, tb.y)));
}

template <int KID>
__device__ __forceinline__ double p2p_eval(const KernelParams& kp, const double2* tab, double px,
                                           double py, double qx, double qy) {
  if (KID == H2D_KERNEL_LOG) {
    const double dx = px - qx, dy = py - qy;
    const double r2 = fma(dx, dx, dy * dy);
    return r2 > 0.0 ? 0.5 * log_r2_fast(r2, tab) : 0.0;
  }
  return kernel_eval_t<KID>(kp, px, py, qx, qy);
}

// One leaf-pair block on a 16 x 16 thread grid: thread (ti, tj) owns rows ti + 16a
// (a < A = ceil(m/16)) and columns tj + 16b (b < B = ceil(n/16)) of a super-tile of up to
// 96 x 96 points (a leaf of the configs fits one super-tile; larger blocks loop).  Row
// points live in registers one row at a time, column points are read from shared memory,
// column sums stay in registers (cacc[b]), row sums are reduced over tj by shuffles.
constexpr int kSymTile = 96, kSymMaxB = kSymTile / 16;
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
      double cacc[kSymMaxB];
#pragma unroll
      for (int bb = 0; bb < kSymMaxB; ++bb) cacc[bb] = 0.0;
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
              const double k = p2p_eval<KID>(kp, tab, rpx, rpy, s_b[j], s_b[kSymTile + j]);
              racc = fma(k, s_b[2 * kSymTile + j], racc);
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

__device__ __forceinline__ uint32_t p2p_spread(uint32_t v) {
  v &= 0xFFFFu;
  v = (v | (v << 8)) & 0x00FF00FFu;
  v = (v | (v << 4)) & 0x0F0F0F0Fu;
  v = (v | (v << 2)) & 0x33333333u;
  v = (v | (v << 1)) & 0x55555555u;
  return v;
}
__device__ __forceinline__ uint32_t p2p_compact(uint32_t v) {
  v &= 0x55555555u;
  v = (v | (v >> 1)) & 0x33333333u;
  v = (v | (v >> 2)) & 0x0F0F0F0Fu;
  v = (v | (v >> 4)) & 0x00FF00FFu;
  v = (v | (v >> 8)) & 0x0000FFFFu;
  return v;
}

template <int KID>
__global__ void __launch_bounds__(256, 3)
p2p_sym_kernel(int kappa, int64_t leaf_begin, int64_t leaf_end,
               const int32_t* __restrict__ leaf_start, const double* __restrict__ px,
               const double* __restrict__ py, const double* __restrict__ x, KernelParams kp,
               double* __restrict__ s0, double* __restrict__ sL, double* __restrict__ sD) {
  __shared__ double s_a[3 * kSymTile], s_b[3 * kSymTile], srow[kSymTile];
  __shared__ double scol[16][kSymTile + 1];
  __shared__ double2 s_logtab[128];
  const int64_t X = leaf_begin + blockIdx.x;
  const int tid = threadIdx.x;
  if (KID == H2D_KERNEL_LOG && tid < 128) {
    const double c = 1.0 + (tid + 0.5) / 128.0;
    s_logtab[tid] = make_double2(1.0 / c, log(c));
  }
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
  // phase 1: blocks in a fixed order (one code instance: keeps the I-cache footprint small)
  for (int task = 0; task < 5; ++task) {
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

// ---------------------------------------------------------------- stage B: y = ynear + U t
// One CTA (8 warps) per leaf L.  Lane i owns rows i, i+32, ... (RPL rows) of the leaf;
// warp w owns columns q = w, w+8, ... of every ancestor U panel.  For a column, the
// warp's loads are 256 B contiguous row segments at constant offsets (no per-load
// address math); t for 32 of the warp's columns is fetched with one coalesced load and
// broadcast by shuffles.  8 loads in flight per thread, one barrier (final row sum).
template <int RPL, int CU>
__device__ __forceinline__ void stageB_rows(int kappa, int rows_here, int64_t rowoff,
                                            const int* s_R, const int* s_cb,
                                            const int64_t* s_base, const int64_t* s_mX,
                                            const LevelPtrs& lp, double (&acc)[4]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  bool valid[RPL];
#pragma unroll
  for (int r = 0; r < RPL; ++r) valid[r] = lane + 32 * r < rows_here;
  for (int l = 1; l <= kappa; ++l) {
    const int R = s_R[l];
    const int64_t mX = s_mX[l];
    const double* __restrict__ base = lp.U[l] + s_base[l] + rowoff + lane;
    const double* __restrict__ tl = lp.tu[l] + s_cb[l];
    const int64_t stepc = 8 * mX;                    // this warp's next column
    for (int q0 = w; q0 < R; q0 += 8 * 32) {
      const int qq = q0 + 8 * lane;
      const double tq = qq < R ? __ldg(tl + qq) : 0.0;
      const int ncol = min(32, (R - q0 + 7) >> 3);
      const double* __restrict__ p = base + (int64_t)q0 * mX;
      int k = 0;
      for (; k + CU <= ncol; k += CU, p += CU * stepc) {
        double u[CU][RPL];
#pragma unroll
        for (int c = 0; c < CU; ++c)
#pragma unroll
          for (int r = 0; r < RPL; ++r) u[c][r] = valid[r] ? __ldcs(p + c * stepc + 32 * r) : 0.0;
#pragma unroll
        for (int c = 0; c < CU; ++c) {
          const double tv = __shfl_sync(0xffffffffu, tq, k + c);
#pragma unroll
          for (int r = 0; r < RPL; ++r) acc[r] = fma(u[c][r], tv, acc[r]);
        }
      }
      for (; k < ncol; ++k, p += stepc) {
        const double tv = __shfl_sync(0xffffffffu, tq, k);
#pragma unroll
        for (int r = 0; r < RPL; ++r) acc[r] = fma(valid[r] ? __ldcs(p + 32 * r) : 0.0, tv, acc[r]);
      }
    }
  }
}

__global__ void __launch_bounds__(kBThreads, 4)
stageB_kernel(int kappa, int64_t leaf_begin, const int32_t* __restrict__ leaf_start, LevelPtrs lp,
              const double* __restrict__ ynear, int64_t n, const double* __restrict__ x,
              double scale, double shift, double* __restrict__ y,
              const int32_t* __restrict__ perm, int order_out, int64_t y_row0) {
  __shared__ double red[8][128];
  __shared__ int s_R[H2D_MAX_LEVELS + 1], s_cb[H2D_MAX_LEVELS + 1];
  __shared__ int64_t s_base[H2D_MAX_LEVELS + 1], s_mX[H2D_MAX_LEVELS + 1];
  const int64_t L = leaf_begin + blockIdx.x;
  const int64_t s0 = leaf_start[L];
  const int mL = leaf_start[L + 1] - (int)s0;
  if (mL <= 0) return;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid >= 1 && tid <= kappa) {           // per-level metadata, fetched in parallel once
    const int l = tid, sh = 2 * (kappa - l);
    const int64_t X = L >> sh;
    const int32_t cb = lp.ucolbase[l][X];
    const int64_t bx0 = leaf_start[X << sh];
    s_R[l] = lp.ucolbase[l][X + 1] - cb;
    s_cb[l] = cb;
    s_mX[l] = leaf_start[(X + 1) << sh] - bx0;
    s_base[l] = lp.upan_off[l][X] + (s0 - bx0);
  }
  __syncthreads();
  for (int rp = 0; rp < mL; rp += 128) {
    const int rows = min(mL - rp, 128);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    if (rows <= 32) stageB_rows<1, 8>(kappa, rows, rp, s_R, s_cb, s_base, s_mX, lp, acc);
    else if (rows <= 64) stageB_rows<2, 4>(kappa, rows, rp, s_R, s_cb, s_base, s_mX, lp, acc);
    else if (rows <= 96) stageB_rows<3, 2>(kappa, rows, rp, s_R, s_cb, s_base, s_mX, lp, acc);
    else stageB_rows<4, 2>(kappa, rows, rp, s_R, s_cb, s_base, s_mX, lp, acc);
    if (rp > 0) __syncthreads();
#pragma unroll
    for (int r = 0; r < 4; ++r) red[w][lane + 32 * r] = acc[r];
    __syncthreads();
    if (tid < rows) {
      double s = 0.0;
#pragma unroll
      for (int ww = 0; ww < 8; ++ww) s += red[ww][tid];
      const int64_t r = s0 + rp + tid;
      // near field (three symmetric-P2P slots) + shift x
      s += fma(scale, (ynear[r] + ynear[n + r]) + ynear[2 * n + r], shift * x[r]);
      if (order_out == H2D_ORDER_ORIGINAL) y[perm[r]] = s;
      else y[r - y_row0] = s;
    }
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
// the U / V panels and fill the level's panel metadata.
void pack_level(Handle& h, Level& L, const std::vector<const double*>& srcU,
                const std::vector<const double*>& srcV) {
  cudaStream_t s = h.stream;
  const int l = L.l;
  const int64_t nbox = L.nbox;
  auto rank_of = [&](int64_t e) { return std::max<int32_t>(0, L.rank[(size_t)e]); };
  L.ucol.assign((size_t)L.nblocks, 0);
  L.vcol.assign((size_t)L.nblocks, 0);
  L.upan_off.assign((size_t)nbox, 0);
  L.vpan_off.assign((size_t)nbox, 0);
  L.ucolbase.assign((size_t)nbox + 1, 0);
  L.vR.assign((size_t)nbox, 0);
  int64_t uo = 0, vo = 0;
  int32_t cb = 0;
  for (int64_t X = 0; X < nbox; ++X) {
    const int64_t m = h.box_end(l, X) - h.box_begin(l, X);
    int32_t R = 0;
    for (int32_t e = L.off[(size_t)X]; e < L.off[(size_t)X + 1]; ++e) {
      L.ucol[(size_t)e] = R;
      R += rank_of(e);
    }
    L.ucolbase[(size_t)X] = cb;
    cb += R;
    L.upan_off[(size_t)X] = uo;
    uo += m * R;
    // V panel of column box X: blocks (Z, X) for Z in I_X ascending
    int32_t RV = 0;
    for (int32_t e2 = L.off[(size_t)X]; e2 < L.off[(size_t)X + 1]; ++e2) {
      const int32_t b = L.trans[(size_t)e2];
      L.vcol[(size_t)b] = RV;
      RV += rank_of(b);
    }
    L.vR[(size_t)X] = RV;
    L.vpan_off[(size_t)X] = vo;
    vo += m * RV;
  }
  L.ucolbase[(size_t)nbox] = cb;
  L.u_values = uo;
  L.v_values = vo;
  L.U = h.alloc<double>(uo);
  L.V = h.alloc<double>(vo);
  std::vector<CopyItem> citems;
  std::vector<VPackItem> vitems;
  for (int64_t X = 0; X < nbox; ++X) {
    const int64_t mX = h.box_end(l, X) - h.box_begin(l, X);
    for (int32_t e = L.off[(size_t)X]; e < L.off[(size_t)X + 1]; ++e) {
      const int r = rank_of(e);
      if (r == 0) continue;
      const int64_t Y = L.col[(size_t)e];
      const int64_t nY = h.box_end(l, Y) - h.box_begin(l, Y);
      if (mX * r > 0)
        citems.push_back(CopyItem{srcU[(size_t)e], L.U + L.upan_off[(size_t)X] + (int64_t)L.ucol[(size_t)e] * mX,
                                  mX * r});
      if (nY * r > 0)
        vitems.push_back(VPackItem{srcV[(size_t)e], L.V + L.vpan_off[(size_t)Y] + L.vcol[(size_t)e],
                                   (int32_t)nY, r, L.vR[(size_t)Y], 0});
    }
  }
  const size_t CH = 1 << 20;
  for (size_t c0 = 0; c0 < citems.size(); c0 += CH) {
    std::vector<CopyItem> part(citems.begin() + c0, citems.begin() + std::min(citems.size(), c0 + CH));
    CopyItem* d = upload_tmp(part, s);
    copy_items_kernel<<<(int)part.size(), 256, 0, s>>>(d);
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

// Build the stage-A / reduce schedule, the t layout (U-panel order) and the per-level
// device tables.
void finalize_schedule(Handle& h) {
  cudaStream_t s = h.stream;
  int64_t t_len = 0, tpart_len = 0;
  std::vector<AItem> aitems;
  std::vector<RItem> ritems;
  // t layout: level by level, U-panel column order (ucolbase) -> tu_base per level
  for (int l = 1; l <= h.kappa; ++l) {
    Level& L = h.levels[(size_t)l];
    L.tu_base = t_len;
    t_len += L.ucolbase[(size_t)L.nbox];
  }
  if (t_len > INT32_MAX) throw Error{H2D_EINVAL, "t vector exceeds 2^31 entries"};
  // vdst: V-panel columns in column-box order (per level, box, column) -> t index
  std::vector<int32_t> vdst((size_t)std::max<int64_t>(1, t_len));
  int64_t vpos = 0;
  for (int l = 1; l <= h.kappa; ++l) {
    Level& L = h.levels[(size_t)l];
    L.t_off.assign((size_t)L.nbox, 0);
    for (int64_t Y = 0; Y < L.nbox; ++Y) {
      L.t_off[(size_t)Y] = vpos;       // first vdst entry of the V panel of Y
      for (int32_t e2 = L.off[(size_t)Y]; e2 < L.off[(size_t)Y + 1]; ++e2) {
        const int32_t b = L.trans[(size_t)e2];           // block (X, Y)
        const int r = std::max<int32_t>(0, L.rank[(size_t)b]);
        if (r == 0) continue;
        const int64_t X = L.col[(size_t)e2];
        for (int q = 0; q < r; ++q)
          vdst[(size_t)(vpos + L.vcol[(size_t)b] + q)] =
              (int32_t)(L.tu_base + L.ucolbase[(size_t)X] + L.ucol[(size_t)b] + q);
      }
      vpos += L.vR[(size_t)Y];
    }
  }
  if (vpos != t_len) throw Error{H2D_ECUDA, "t layout mismatch"};
  h.t_len = t_len;
  h.d_t = h.alloc<double>(t_len);
  h.d_vdst = h.alloc<int32_t>(vdst.size());
  H2D_CUDA(cudaMemcpyAsync(h.d_vdst, vdst.data(), vdst.size() * 4, cudaMemcpyHostToDevice, s));
  for (int l = 1; l <= h.kappa; ++l) {
    Level& L = h.levels[(size_t)l];
    L.d_ucolbase = h.alloc<int32_t>(L.ucolbase.size());
    L.d_upan_off = h.alloc<int64_t>(L.upan_off.size());
    H2D_CUDA(cudaMemcpyAsync(L.d_ucolbase, L.ucolbase.data(), L.ucolbase.size() * 4,
                             cudaMemcpyHostToDevice, s));
    H2D_CUDA(cudaMemcpyAsync(L.d_upan_off, L.upan_off.data(), L.upan_off.size() * 8,
                             cudaMemcpyHostToDevice, s));
    H2D_CUDA(cudaStreamSynchronize(s));
    h.lp.U[l] = L.U;
    h.lp.V[l] = L.V;
    h.lp.ucolbase[l] = L.d_ucolbase;
    h.lp.upan_off[l] = L.d_upan_off;
    h.lp.tu[l] = h.d_t + L.tu_base;
    // stage-A items: chunks of <= kATarget elements and <= kAMaxRows rows
    for (int64_t Y = 0; Y < L.nbox; ++Y) {
      const int R = L.vR[(size_t)Y];
      const int64_t y0 = h.box_begin(l, Y);
      const int64_t nY = h.box_end(l, Y) - y0;
      if (R == 0 || nY == 0) continue;
      int64_t nch = std::max<int64_t>((nY * R + kATarget - 1) / kATarget, (nY + kAMaxRows - 1) / kAMaxRows);
      nch = std::min<int64_t>(nY, std::max<int64_t>(1, nch));
      const int64_t rows = (nY + nch - 1) / nch;
      nch = (nY + rows - 1) / rows;
      const int32_t vp = (int32_t)L.t_off[(size_t)Y];
      if (nch == 1) {
        aitems.push_back(AItem{L.vpan_off[(size_t)Y], y0, (int32_t)nY, R, vp, l, -1, 0});
      } else {
        if (tpart_len + nch * R > INT32_MAX) throw Error{H2D_EINVAL, "partial buffer too large"};
        ritems.push_back(RItem{vp, (int32_t)tpart_len, R, (int32_t)nch});
        for (int64_t c = 0; c < nch; ++c) {
          const int64_t r0 = c * rows, nr = std::min(rows, nY - r0);
          aitems.push_back(AItem{L.vpan_off[(size_t)Y] + r0 * R, y0 + r0, (int32_t)nr, R,
                                 (int32_t)(-(tpart_len + c * R) - 1), l,
                                 (int32_t)(ritems.size() - 1), 0});
        }
        tpart_len += nch * R;
      }
    }
  }
  h.tpart_len = tpart_len;
  h.d_tpart = h.alloc<double>(tpart_len);
  h.n_aitems = (int64_t)aitems.size();
  h.n_ritems = (int64_t)ritems.size();
  h.d_aitems = h.alloc<AItem>(aitems.size());
  h.d_ritems = h.alloc<RItem>(ritems.size());
  h.d_rcount = h.alloc<int32_t>(ritems.size());
  H2D_CUDA(cudaMemsetAsync(h.d_rcount, 0, std::max<size_t>(1, ritems.size()) * sizeof(int32_t), s));
  if (!aitems.empty())
    H2D_CUDA(cudaMemcpyAsync(h.d_aitems, aitems.data(), aitems.size() * sizeof(AItem),
                             cudaMemcpyHostToDevice, s));
  if (!ritems.empty())
    H2D_CUDA(cudaMemcpyAsync(h.d_ritems, ritems.data(), ritems.size() * sizeof(RItem),
                             cudaMemcpyHostToDevice, s));
  if (!h.d_ynear) h.d_ynear = h.alloc<double>(3 * h.n);   // three P2P slots (p2p_sym_kernel)
  H2D_CUDA(cudaFuncSetAttribute(stageA_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                cudaSharedmemCarveoutMaxShared));
  if (!h.aux_stream) {
    H2D_CUDA(cudaStreamCreateWithFlags(&h.aux_stream, cudaStreamNonBlocking));
    H2D_CUDA(cudaEventCreateWithFlags(&h.ev_fork, cudaEventDisableTiming));
    H2D_CUDA(cudaEventCreateWithFlags(&h.ev_join, cudaEventDisableTiming));
  }
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

// Matvec on TREE-order x (S7-S9).  The near-field P2P (compute-bound) runs on the aux
// stream concurrently with stage A (HBM-bound); stage B joins both.
void matvec_tree(Handle& h, const double* d_xtree, double* d_y, int order_out, int64_t y_row0) {
  cudaStream_t s = h.stream, a = h.aux_stream;
  const int64_t nleaves = h.leaf_end - h.leaf_begin;
  H2D_CUDA(cudaEventRecord(h.ev_fork, s));
  H2D_CUDA(cudaStreamWaitEvent(a, h.ev_fork, 0));
  record(h, 6, a);
  if (nleaves > 0) {
    auto* kfn = h.kp.id == H2D_KERNEL_LOG ? p2p_sym_kernel<H2D_KERNEL_LOG>
              : h.kp.id == H2D_KERNEL_IMQ ? p2p_sym_kernel<H2D_KERNEL_IMQ>
              : h.kp.id == H2D_KERNEL_ONE_OVER_R ? p2p_sym_kernel<H2D_KERNEL_ONE_OVER_R>
                                                 : p2p_sym_kernel<H2D_KERNEL_TEST_LOWRANK>;
    kfn<<<(int)nleaves, 256, 0, a>>>(h.kappa, h.leaf_begin, h.leaf_end, h.d_leaf_start, h.d_px,
                                     h.d_py, d_xtree, h.kp, h.d_ynear, h.d_ynear + h.n,
                                     h.d_ynear + 2 * h.n);
    H2D_LAUNCH_CHECK();
  }
  record(h, 7, a);
  H2D_CUDA(cudaEventRecord(h.ev_join, a));
  if (h.n_aitems > 0) {
    stageA_kernel<<<(int)h.n_aitems, kAThreads, 0, s>>>(h.d_aitems, h.lp, d_xtree, h.d_vdst, h.d_t,
                                                        h.d_tpart, h.d_ritems, h.d_rcount);
    H2D_LAUNCH_CHECK();
  }
  record(h, 2, s);
  record(h, 3, s);
  H2D_CUDA(cudaStreamWaitEvent(s, h.ev_join, 0));
  record(h, 4, s);
  if (nleaves > 0) {
    stageB_kernel<<<(int)nleaves, kBThreads, 0, s>>>(h.kappa, h.leaf_begin, h.d_leaf_start, h.lp,
                                                      h.d_ynear, h.n, d_xtree, h.kp.scale,
                                                      h.kp.shift, d_y, h.d_perm, order_out, y_row0);
    H2D_LAUNCH_CHECK();
  }
  record(h, 5, s);
}

}  // namespace h2d
