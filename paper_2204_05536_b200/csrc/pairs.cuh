// Pair-local symmetric apply (NEXT N1 payoff, R23 / §6 "pair apply").
//
// A symmetric build stores one factor pair per unordered box pair {X, Y}, X < Y (Morton):
// K(X, Y) ~ U V^T and K(Y, X) ~ V U^T (the paper's symmetric setting).  Alg. 2 l.15
// then needs, per pair, t1 = V^T x_Y, t2 = U^T x_X, y_X += U t1 and y_Y += V t2:
// each factor is used twice, and each product of one factor needs the other factor's
// reduction first.  The three-pass apply (A' / B' / C') reads 3 of the 4 factor streams;
// this kernel reads each factor once from HBM by keeping the pair local:
//   phase 1  V rows          -> column sums t1 = V^T x_Y
//   phase 2  U rows          -> column sums t2 = U^T x_X and row dots dy_X = U t1
//   phase 3  V rows again    -> row dots dy_Y = V t2 (an L2 hit: V was just read)
// The factors stay in the ACA's column-major layout, V then U per pair.  Lane = row: a warp
// reads a 32-row tile of a column as one coalesced 256-byte load, so the narrow per-pair
// panels (rank ~10-40) use every lane; column sums are reduced by warp shuffles, row dots
// need none.  dy rows go to the TREE-order accumulator yacc (L2-resident) by fp64 REDs on
// 32 consecutive rows.  Work items: groups of up to 8 small pairs (one warp each), medium
// pairs (the 8 warps of a CTA split the tiles), and row chunks of the big pairs of the coarse
// levels (any CTA; the last chunk of a phase reduces the partials in chunk order and
// publishes t1 / t2 with a flag = matvec epoch; a later phase's chunk waits for it).
// Not bitwise reproducible: the order of the y accumulations varies between runs.
#pragma once
#include "pipe.cuh"

namespace h2d {
namespace {

constexpr int kPWarps = 8;                  // warps per CTA
constexpr int kPMaxR = 128;                 // widest pair (rank), column blocks of <= 16
constexpr int kPSmallBytes = 48 * 1024;     // pairs up to this: one warp
constexpr int kPWholeBytes = 640 * 1024;    // pairs up to this: one CTA, all phases
constexpr int kPChunkRows = 2048;           // big pairs: row chunks (per phase)

enum { kPGroup = 0, kPWhole = 1, kPPhase1 = 2, kPPhase2 = 3, kPPhase3 = 4 };
#ifndef H2D_PAIR_NORED
#define H2D_PAIR_NORED 0
#endif
constexpr bool kPNoRed = H2D_PAIR_NORED;   // build-time diagnostics switch (timing of the REDs)

struct PPair {              // one stored pair
  int64_t v_off, u_off;     // V (nv x r) and U (nu x r), column-major, in the level's pair array
  int32_t yv, yu;           // TREE rows of Y (V rows) and X (U rows)
  int32_t nv, nu, r, level;
};
struct PWork {              // one work item (a CTA takes it)
  int32_t kind;
  int32_t first, count;     // kPGroup: pairs [first, first + count); else the pair `first`
  int32_t r0, r1;           // chunk: rows [r0, r1) of the phase's factor
  int32_t big, chunk, nchunks;
  int64_t toff, poff;       // big pair: t1 / t2 offset; partial slots of the phase
};
struct PairPtrs {
  const double* P[H2D_MAX_LEVELS + 1];
};

__device__ __forceinline__ int ld_acquire(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int32_t* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One warp over the rows {tile * 32 + lane : tile = t0, t0 + ts, ...} < rows of columns
// [c0, c0 + nc) (nc <= NC) of a column-major factor F (leading dimension ld):
//   COLS  acc[q] += F[i, c0 + q] x[i]           (column sums, per lane)
//   ROWS  dy[i]  += sum_q F[i, c0 + q] t[c0 + q] (row dots, one fp64 RED per row)
template <int NC, bool COLS, bool ROWS>
__device__ __forceinline__ void pair_tiles(const double* __restrict__ F, int64_t ld, int rows, int c0, int nc,
                                           int t0, int ts, const double* __restrict__ x, const double* tv,
                                           double* __restrict__ dy, double (&acc)[NC]) {
  const int lane = threadIdx.x & 31;
  for (int t = t0; 32 * t < rows; t += ts) {
    const int i = 32 * t + lane;
    const bool ok = i < rows;
    double v[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) v[q] = (ok && q < nc) ? __ldcs(F + (int64_t)(c0 + q) * ld + i) : 0.0;
    if (COLS) {
      const double xi = ok ? __ldg(x + i) : 0.0;
#pragma unroll
      for (int q = 0; q < NC; ++q) acc[q] = fma(v[q], xi, acc[q]);
    }
    if (ROWS) {
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int q = 0; q < NC; q += 2) {   // (t from shared memory: a broadcast load per column)
        if (q < nc) d0 = fma(v[q], tv[c0 + q], d0);
        if (q + 1 < NC && q + 1 < nc) d1 = fma(v[q + 1], tv[c0 + q + 1], d1);
      }
      if (ok) {
        if (kPNoRed) dy[i] = d0 + d1;   // diagnostics only (WRONG results)
        else atomicAdd(dy + i, d0 + d1);
      }
    }
  }
}

template <int NC>
__device__ __forceinline__ void zero_acc(double (&acc)[NC]) {
#pragma unroll
  for (int q = 0; q < NC; ++q) acc[q] = 0.0;
}

// Warp-level column sums of columns [c0, c0 + nc) into ts[c0 + q] (shared, per warp).
template <int NC>
__device__ __forceinline__ void warp_colsum_store(double (&acc)[NC], int c0, int nc, double* ts) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    const double s = warp_sum(acc[q]);
    if (lane == 0 && q < nc) ts[c0 + q] = s;
  }
  __syncwarp();
}

// ---------------------------------------------------------------- one warp, one pair
template <int NC>
__device__ void pair_warp(const PPair& p, const double* __restrict__ base, const double* __restrict__ x,
                          double* __restrict__ yacc, double* ts1, double* ts2) {
  const double* V = base + p.v_off;
  const double* U = base + p.u_off;
  double acc[NC];
  for (int c0 = 0; c0 < p.r; c0 += NC) {   // phase 1: t1 = V^T x_Y
    const int nc = min(NC, p.r - c0);
    zero_acc(acc);
    pair_tiles<NC, true, false>(V, p.nv, p.nv, c0, nc, 0, 1, x + p.yv, nullptr, nullptr, acc);
    warp_colsum_store(acc, c0, nc, ts1);
  }
  for (int c0 = 0; c0 < p.r; c0 += NC) {   // phase 2: t2 = U^T x_X, y_X += U t1
    const int nc = min(NC, p.r - c0);
    zero_acc(acc);
    pair_tiles<NC, true, true>(U, p.nu, p.nu, c0, nc, 0, 1, x + p.yu, ts1, yacc + p.yu, acc);
    warp_colsum_store(acc, c0, nc, ts2);
  }
  for (int c0 = 0; c0 < p.r; c0 += NC) {   // phase 3: y_Y += V t2
    const int nc = min(NC, p.r - c0);
    pair_tiles<NC, false, true>(V, p.nv, p.nv, c0, nc, 0, 1, nullptr, ts2, yacc + p.yv, acc);
  }
}

// ---------------------------------------------------------------- the CTA, one pair / chunk
// CTA column sums: warp partials -> red[w][q] -> sum over the warps -> out[q] (shared or
// global), then a barrier.
template <int NC>
__device__ __forceinline__ void cta_colsum(double (&acc)[NC], int c0, int nc, double* red, double* out) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    const double s = warp_sum(acc[q]);
    if (lane == 0) red[w * kPMaxR + c0 + q] = s;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < nc; q += blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int ww = 0; ww < kPWarps; ++ww) s += red[ww * kPMaxR + c0 + q];
    out[c0 + q] = s;
  }
  __syncthreads();
}

__device__ __forceinline__ void wait_flag(const int32_t* f, int epoch) {
  if (threadIdx.x == 0)
    while (ld_acquire(f) < epoch) __nanosleep(100);
  __syncthreads();
  __threadfence();   // (invalidates this SM's L1 before the t loads)
}

template <int NC>
__device__ void pair_cta(const PWork& w, const PPair& p, const double* __restrict__ base,
                         const double* __restrict__ x, double* __restrict__ yacc, double* __restrict__ tP1,
                         double* __restrict__ tP2, double* __restrict__ tpart, int32_t* __restrict__ pcount,
                         int32_t* __restrict__ flags, int epoch, double* st1, double* st2, double* red,
                         int* sflag) {
  const int wid = threadIdx.x >> 5;
  const double* V = base + p.v_off;
  const double* U = base + p.u_off;
  double acc[NC];
  if (w.kind == kPWhole) {
    for (int c0 = 0; c0 < p.r; c0 += NC) {
      const int nc = min(NC, p.r - c0);
      zero_acc(acc);
      pair_tiles<NC, true, false>(V, p.nv, p.nv, c0, nc, wid, kPWarps, x + p.yv, nullptr, nullptr, acc);
      cta_colsum(acc, c0, nc, red, st1);
    }
    for (int c0 = 0; c0 < p.r; c0 += NC) {
      const int nc = min(NC, p.r - c0);
      zero_acc(acc);
      pair_tiles<NC, true, true>(U, p.nu, p.nu, c0, nc, wid, kPWarps, x + p.yu, st1, yacc + p.yu, acc);
      cta_colsum(acc, c0, nc, red, st2);
    }
    for (int c0 = 0; c0 < p.r; c0 += NC) {
      const int nc = min(NC, p.r - c0);
      pair_tiles<NC, false, true>(V, p.nv, p.nv, c0, nc, wid, kPWarps, nullptr, st2, yacc + p.yv, acc);
    }
    return;
  }
  // a row chunk [r0, r1) of one phase of a big pair
  const int ph = w.kind - kPPhase1 + 1;
  const double* F = ph == 2 ? U : V;
  const int64_t ld = ph == 2 ? p.nu : p.nv;
  const int y0 = ph == 2 ? p.yu : p.yv;
  const int rows = w.r1 - w.r0;
  const double* Fc = F + w.r0;            // column q of the chunk: Fc + q ld
  if (ph >= 2) {                          // the other factor's reduction must be published
    wait_flag(flags + 2 * w.big + (ph - 2), epoch);
    const double* tg = (ph == 2 ? tP1 : tP2) + w.toff;
    for (int q = threadIdx.x; q < p.r; q += blockDim.x) st1[q] = tg[q];
    __syncthreads();
  }
  for (int c0 = 0; c0 < p.r; c0 += NC) {
    const int nc = min(NC, p.r - c0);
    zero_acc(acc);
    if (ph == 1)
      pair_tiles<NC, true, false>(Fc, ld, rows, c0, nc, wid, kPWarps, x + y0 + w.r0, nullptr, nullptr, acc);
    else if (ph == 2)
      pair_tiles<NC, true, true>(Fc, ld, rows, c0, nc, wid, kPWarps, x + y0 + w.r0, st1, yacc + y0 + w.r0, acc);
    else
      pair_tiles<NC, false, true>(Fc, ld, rows, c0, nc, wid, kPWarps, nullptr, st1, yacc + y0 + w.r0, acc);
    if (ph < 3) cta_colsum(acc, c0, nc, red, tpart + w.poff + (int64_t)w.chunk * p.r);
  }
  if (ph == 3) return;
  // the last chunk of the phase sums the partials in chunk order and publishes t1 / t2
  if (threadIdx.x == 0) {
    __threadfence();
    const int last = atomicAdd(pcount + 2 * w.big + (ph - 1), 1) == w.nchunks - 1;
    if (last) __threadfence();
    *sflag = last;
  }
  __syncthreads();
  if (*sflag) {
    double* tout = (ph == 1 ? tP1 : tP2) + w.toff;
    for (int q = threadIdx.x; q < p.r; q += blockDim.x) {
      const double* __restrict__ pq = tpart + w.poff + q;
      double a0 = 0.0, a1 = 0.0;
      int c = 0;
      for (; c + 1 < w.nchunks; c += 2) {
        a0 += __ldcg(pq + (int64_t)c * p.r);
        a1 += __ldcg(pq + (int64_t)(c + 1) * p.r);
      }
      if (c < w.nchunks) a0 += __ldcg(pq + (int64_t)c * p.r);
      tout[q] = a0 + a1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      pcount[2 * w.big + (ph - 1)] = 0;
      __threadfence();
      st_release(flags + 2 * w.big + (ph - 1), epoch);
    }
  }
}

__global__ void __launch_bounds__(32 * kPWarps, 3)
pair_apply_kernel(const PWork* __restrict__ work, int n_work, const PPair* __restrict__ pairs, int32_t* counter,
                  PairPtrs pp, const double* __restrict__ x, double* __restrict__ yacc, double* __restrict__ tP1,
                  double* __restrict__ tP2, double* __restrict__ tpart, int32_t* __restrict__ pcount,
                  int32_t* __restrict__ flags, int epoch) {
  __shared__ double st[kPWarps][2][kPMaxR];     // per-warp t1 / t2 (groups); st[0] for CTA items
  __shared__ double red[kPWarps * kPMaxR];
  __shared__ int sidx, sflag;
  const int wid = threadIdx.x >> 5;
  for (;;) {
    if (threadIdx.x == 0) sidx = atomicAdd(counter, 1);
    __syncthreads();
    const int idx = sidx;
    __syncthreads();
    if (idx >= n_work) break;
    const PWork w = work[idx];
    if (w.kind == kPGroup) {
      if (wid < w.count) {
        const PPair p = pairs[w.first + wid];
        const double* base = pp.P[p.level];
        if (p.r <= 8) pair_warp<8>(p, base, x, yacc, st[wid][0], st[wid][1]);
        else pair_warp<16>(p, base, x, yacc, st[wid][0], st[wid][1]);
      }
      continue;   // (the next item's barrier waits for every warp)
    }
    const PPair p = pairs[w.first];
    const double* base = pp.P[p.level];
    if (p.r <= 8)
      pair_cta<8>(w, p, base, x, yacc, tP1, tP2, tpart, pcount, flags, epoch, st[0][0], st[0][1], red, &sflag);
    else
      pair_cta<16>(w, p, base, x, yacc, tP1, tP2, tpart, pcount, flags, epoch, st[0][0], st[0][1], red, &sflag);
  }
}

}  // namespace
}  // namespace h2d
