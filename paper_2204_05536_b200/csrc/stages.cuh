// The factor-streaming stages of the single-vector matvec (apply.cu):
//   stage A  t = V^T x  over row-major V box panels (persistent, bulk-TMA ring)
//   stage B' the symmetric apply's fused pass: t2 = U^T x and y1 = U t1 over the first-side
//            U box panels (stage A's ring with the row dots added, DUAL)
//   stage B  yfar = U t over column-major U leaf panels (persistent, bulk-TMA ring; several
//            levels of a leaf per stage)
//   small-item kernels: warp per box / leaf for items too small for the ring
#pragma once
#include "pipe.cuh"


namespace h2d {
namespace {

// ---------------------------------------------------------------- stage A: t = V^T x
// Item = rows [0, nrows) of a row-major V panel chunk (stride Rp).  A stage holds
// rows_s = min(256, 2048 / Rp) whole rows (one bulk copy) and their x values.  Consumers:
// R <= 256 -> thread (g, q) = (tid / R, tid % R) owns panel column q and rows g, g + G, ...
// (G = 256 / R groups, reduced in smem at the end of the item); R > 256 -> thread owns
// columns tid + 256 c (c < CPL) over all rows.  Stage header: a = R, b = Rp, c = out,
// d = ritem.
// Symmetric stage B' (DUAL): the same stream over the first-side U box panels also computes
// the per-row dots y1 = U t1 with the row box's t1 values double-buffered in smem.
// The t1 values of the row box ride in every stage of its rows, right after them in the ring
// slot (rows_s shrinks by R / Rp rows), so no separate buffer or release handshake is needed.
constexpr int kT1Smem = 1024;   // widest first-side panel the slot layout supports
struct DualCtx {
  const double* t1;           // global t1
  double* y1;                 // global [kappa][n]
  int64_t n;
};

template <int NS, bool DUAL = false, int SD = kStageDbl>
__device__ void stageA_producer(PipeSmem<NS, SD>& S, const AItem* __restrict__ items, int n_items,
                                int32_t* counter, const LevelPtrs& lp, const double* __restrict__ x,
                                const DualCtx& dc = DualCtx{}) {
  const int lane = threadIdx.x & 31;
  const uint64_t pol = l2_evict_first_policy();
  int stage = 0;
  uint32_t phase = 0;
  // one-item lookahead: the next item's index (atomic) and descriptor (load) are in flight
  // while the current item streams, so item boundaries cost no memory latency
  int idx = 0, nidx = 0;
  if (lane == 0) idx = atomicAdd(counter, 1);
  idx = __shfl_sync(0xffffffffu, idx, 0);
  if (lane == 0) nidx = atomicAdd(counter, 1);
  AItem nit{};
  if (idx < n_items) nit = items[idx];
  for (;;) {
    const bool done = idx >= n_items;
    const AItem it = nit;
    const int cur = idx;
    idx = __shfl_sync(0xffffffffu, nidx, 0);       // issued one item ago
    if (!done && lane == 0) nidx = atomicAdd(counter, 1);
    if (!done && idx < n_items) nit = items[idx];
    const int t1w = DUAL ? (it.R + 1) & ~1 : 0;   // t1 values (+ zero pad) after the rows
    const int rows_s = done ? 1 : min(kStageVec, (SD - t1w) / it.Rp);
    const double* V = done ? nullptr : (DUAL ? lp.Ub[it.level] : lp.V[it.level]) + it.v_off;
    int r0 = 0;
    do {
      const int rows = done ? 0 : min(rows_s, it.nrows - r0);
      mbar_wait(&S.empty[stage], phase ^ 1);
      if (lane == 0) {
        StageHdr& h = S.hdr[stage];
        h.item = done ? -1 : cur;
        h.cnt = rows;
        h.flags = (r0 == 0 ? kFirst : 0) | (r0 + rows >= it.nrows ? kLast : 0);
        h.a = it.R;
        h.b = it.Rp;
        h.c = it.out;
        h.d = it.ritem;
        h.pad = it.level;
        h.e = (int32_t)it.x_off;
        // odd R: zero the t1 pad slot (released to the consumers by the arrive below)
        if (DUAL && !done && (it.R & 1)) S.ring[stage][rows * it.Rp + it.R] = 0.0;
        const uint32_t bytes = (uint32_t)rows * (uint32_t)it.Rp * 8u;
        mbar_arrive_expect_tx(&S.full[stage], bytes);
        if (bytes) bulk_g2s(S.ring[stage], V + (int64_t)r0 * it.Rp, bytes, &S.full[stage], pol);
      }
      for (int j = lane; j < rows; j += 32) cp_async8(&S.vec[stage][j], x + it.x_off + r0 + j);
      if (DUAL && !done) {
        double* t1s = S.ring[stage] + rows * it.Rp;
        for (int c = lane; c < it.R; c += 32) cp_async8(t1s + c, dc.t1 + it.t1_off + c);
      }
      cp_async_arrive_noinc(&S.full[stage]);
      if (++stage == NS) { stage = 0; phase ^= 1; }
      r0 += rows;
    } while (!done && r0 < it.nrows);
    if (done) break;
  }
}

// Sum the G group partials of the consumer threads (thread g W + i holds pair i of group g
// in red[2 (g W + i) .. + 1]) into group 0: serially for G <= 8, else by a fixed pairwise
// tree (ceil(log2 G) barrier steps instead of a G-long dependent chain per output: narrow
// panels / short rows have G up to 224).  Deterministic; ends with a barrier, so group 0's
// values are visible to all consumers.
__device__ __forceinline__ void group_tree_sum(double* red, int G, int W, int g) {
  const int tid = threadIdx.x;
  named_bar_sync(1, kCons);
  if (G <= 8) {   // few groups (the common wide-panel case): one serial pass, one barrier
    if (g == 0) {
      double u0 = red[2 * tid], u1 = red[2 * tid + 1];
      for (int gg = 1; gg < G; ++gg) {
        u0 += red[2 * (tid + gg * W)];
        u1 += red[2 * (tid + gg * W) + 1];
      }
      red[2 * tid] = u0;
      red[2 * tid + 1] = u1;
    }
    named_bar_sync(1, kCons);
    return;
  }
  for (int span = G; span > 1;) {
    const int half = (span + 1) >> 1;
    if (g < span - half) {
      red[2 * tid] += red[2 * (tid + half * W)];
      red[2 * tid + 1] += red[2 * (tid + half * W) + 1];
    }
    named_bar_sync(1, kCons);
    span = half;
  }
}

// Consumers work on column pairs (one 16-byte smem load = 2 panel elements; Rp is even
// and the padding column is zero, so a pair never straddles a row).  P = Rp / 2 pairs per
// row.  P <= kCons: thread (g, p) = (tid / P, tid % P) owns pair p, rows g, g + G, ...
// (G = kCons / P groups, reduced in smem at the end of the item).  P > kCons: thread owns
// pairs tid + kCons c (c < CP) over all rows.
constexpr int kMaxCP = (kStageDbl / 2 + kCons - 1) / kCons;

template <int CP, int NA>
__device__ __forceinline__ void stageA_consume(const double* __restrict__ sv, const double* __restrict__ sx,
                                               int rows, int Rp, int P, int p, int g, int G,
                                               double (&acc)[NA]) {
  if (CP == 1) {
    if (g >= G) return;
    const double* __restrict__ v = sv + (size_t)g * Rp + 2 * p;
    const int step = G * Rp;
    int j = g;
    for (; j + G < rows; j += 2 * G, v += 2 * step) {
      const double2 a = *reinterpret_cast<const double2*>(v);
      const double2 b = *reinterpret_cast<const double2*>(v + step);
      const double xa = sx[j], xb = sx[j + G];
      acc[0] = fma(a.x, xa, acc[0]);
      acc[1] = fma(a.y, xa, acc[1]);
      acc[2] = fma(b.x, xb, acc[2]);
      acc[3] = fma(b.y, xb, acc[3]);
    }
    if (j < rows) {
      const double2 a = *reinterpret_cast<const double2*>(v);
      const double xa = sx[j];
      acc[0] = fma(a.x, xa, acc[0]);
      acc[1] = fma(a.y, xa, acc[1]);
    }
  } else {
    bool valid[CP];
#pragma unroll
    for (int c = 0; c < CP; ++c) valid[c] = p + kCons * c < P;
    const double* __restrict__ v = sv + 2 * p;
    for (int j = 0; j < rows; ++j, v += Rp) {
      const double xv = sx[j];
#pragma unroll
      for (int c = 0; c < CP; ++c)
        if (valid[c]) {
          const double2 a = *reinterpret_cast<const double2*>(v + 2 * kCons * c);
          acc[2 * c] = fma(a.x, xv, acc[2 * c]);
          acc[2 * c + 1] = fma(a.y, xv, acc[2 * c + 1]);
        }
    }
  }
}

// Symmetric stage B' fused consumer: a warp per row, 4 rows per warp pass (rows w, w + 7,
// w + 14, w + 21 of every 28-row block, so a stage's rows spread evenly over the 7 warps),
// lane owns pairs lane + 32 c (c < C, P <= 32 C).  Each U pair is
// loaded once and feeds both products: the column sums t2 += u x_j (registers, reduced over
// the 7 warps at the end of the item) and the row dot y1_j = u . t1 (t1 pairs in registers
// for the stage; the 4 row dots of a pass are reduced together by a transposed butterfly,
// 6 double shuffles for 4 rows).  The stage's t1 values follow its rows in the ring slot;
// the pad slot R is zero for odd R.
constexpr int kDualMaxC = 4;
template <int C>
__device__ __forceinline__ void dual_consume(const double* __restrict__ sv, const double* __restrict__ sx,
                                             int rows, int Rp, int P, double (&acc)[16],
                                             double* __restrict__ y1row) {
  constexpr int kW = kCons / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const double2* __restrict__ t2 = reinterpret_cast<const double2*>(sv + rows * Rp);
  double2 tt[C];
#pragma unroll
  for (int c = 0; c < C; ++c) tt[c] = lane + 32 * c < P ? t2[lane + 32 * c] : make_double2(0.0, 0.0);
  for (int jb = w; jb < rows; jb += 4 * kW) {
    double r[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      r[k] = 0.0;
      const int j = jb + kW * k;
      if (j < rows) {     // warp-uniform
        const double xj = sx[j];
        const double2* __restrict__ u2 = reinterpret_cast<const double2*>(sv + j * Rp);
#pragma unroll
        for (int c = 0; c < C; ++c)
          if (lane + 32 * c < P) {
            const double2 a = u2[lane + 32 * c];
            acc[2 * c] = fma(a.x, xj, acc[2 * c]);
            acc[2 * c + 1] = fma(a.y, xj, acc[2 * c + 1]);
            r[k] = fma(a.x, tt[c].x, fma(a.y, tt[c].y, r[k]));
          }
      }
    }
    // transposed butterfly: after xor 16 a lane holds rows {2 h16, 2 h16 + 1}, after xor 8
    // row 2 h16 + h8; xor 4 / 2 / 1 finish the sums (lanes 0, 8, 16, 24 hold rows 0..3)
    const bool h16 = lane & 16, h8 = lane & 8;
    double a0 = h16 ? r[2] : r[0], a1 = h16 ? r[3] : r[1];
    const double b0 = h16 ? r[0] : r[2], b1 = h16 ? r[1] : r[3];
    a0 += __shfl_xor_sync(0xffffffffu, b0, 16);
    a1 += __shfl_xor_sync(0xffffffffu, b1, 16);
    double v = h8 ? a1 : a0;
    v += __shfl_xor_sync(0xffffffffu, h8 ? a0 : a1, 8);
    v += __shfl_xor_sync(0xffffffffu, v, 4);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    const int j = jb + kW * (lane >> 3);
    if ((lane & 7) == 0 && j < rows) y1row[j] = v;
  }
}

// End of a fused item: column sums over the 7 warps through smem, one 32-pair block at a
// time, handed to put(q, value).
template <int C, typename Put>
__device__ __forceinline__ void dual_finish(double* red, int P, double (&acc)[16], Put&& put) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    if (32 * c >= P) break;
    red[w * 64 + 2 * lane] = acc[2 * c];
    red[w * 64 + 2 * lane + 1] = acc[2 * c + 1];
    named_bar_sync(1, kCons);
    if (tid < 64) {
      double s = 0.0;
#pragma unroll
      for (int ww = 0; ww < kCons / 32; ++ww) s += red[ww * 64 + tid];
      put(64 * c + tid, s);
    }
    named_bar_sync(1, kCons);
  }
}

// fused mapping for P pairs: C = ceil(P / 32) <= kDualMaxC, -1 = too wide (two-pass path)
__device__ __forceinline__ int dual_cfg(int P) { return P <= 32 * kDualMaxC ? (P + 31) >> 5 : -1; }

template <int NS, bool DUAL = false, int SD = kStageDbl>
__device__ void stageA_consumers(PipeSmem<NS, SD>& S, const int32_t* __restrict__ vdst, double* __restrict__ t,
                                 double* __restrict__ tpart, const RItem* __restrict__ ritems,
                                 int32_t* __restrict__ rcount, const DualCtx& dc = DualCtx{}) {
  int rowoff = 0;
  const int tid = threadIdx.x, lane = tid & 31;
  int stage = 0;
  uint32_t phase = 0;
  int R = 1, Rp = 2, P = 1, CP = 1, G = 1, g = 0, p = 0;
  double* y1base = nullptr;   // DUAL: y1 row of the item's first row
  int dcfg = -1;   // DUAL: fused (LPR, C) mapping of the item, -1 = column pass + row pass
  constexpr int kAcc = DUAL ? 16 : 2 * kMaxCP;
  double acc[kAcc];
#pragma unroll
  for (int c = 0; c < kAcc; ++c) acc[c] = 0.0;
  for (;;) {
    mbar_wait(&S.full[stage], phase);
    const StageHdr h = S.hdr[stage];
    if (h.item < 0) break;
    if (h.flags & kFirst) {
      R = h.a;
      Rp = h.b;
      P = Rp >> 1;
      CP = (P + kCons - 1) / kCons;
      if (CP == 1) { G = kCons / P; g = tid / P; p = tid - g * P; }
      else { G = 1; g = 0; p = tid; }
      if (DUAL) {
        dcfg = dc.n > 0 ? dual_cfg(P) : -1;
        y1base = dc.y1 + (int64_t)(h.pad - 1) * dc.n + h.e;
      }
#pragma unroll
      for (int c = 0; c < kAcc; ++c) acc[c] = 0.0;
      rowoff = 0;
    }
    const double* sv = S.ring[stage];
    const double* sx = S.vec[stage];
    if constexpr (DUAL) if (dcfg >= 0) {
      double* y1row = y1base + rowoff;
      switch (dcfg) {
        case 1: dual_consume<1>(sv, sx, h.cnt, Rp, P, acc, y1row); break;
        case 2: dual_consume<2>(sv, sx, h.cnt, Rp, P, acc, y1row); break;
        case 3: dual_consume<3>(sv, sx, h.cnt, Rp, P, acc, y1row); break;
        default: dual_consume<4>(sv, sx, h.cnt, Rp, P, acc, y1row); break;
      }
      rowoff += h.cnt;
      goto consumed;
    }
    switch (CP) {
      case 1: stageA_consume<1>(sv, sx, h.cnt, Rp, P, p, g, G, acc); break;
      case 2: stageA_consume<2>(sv, sx, h.cnt, Rp, P, p, g, G, acc); break;
      case 3: stageA_consume<3>(sv, sx, h.cnt, Rp, P, p, g, G, acc); break;
      case 4: stageA_consume<4>(sv, sx, h.cnt, Rp, P, p, g, G, acc); break;
      default: stageA_consume<kMaxCP>(sv, sx, h.cnt, Rp, P, p, g, G, acc); break;
    }
  consumed:
    if (DUAL && dc.n > 0 && dcfg < 0) {
      // wide panels: row dots y1[level][row] = U[row, :] t1 over this stage's rows: 8 lanes per row (a warp
      // covers 4 rows per pass), each lane a strided set of column pairs (16-byte loads), a
      // 3-level shuffle reduction inside the 8-lane group; the first-side panels are narrow
      // (~100 columns), so a full-warp reduction per row would cost more than the dot.
      // t1 follows the rows in the slot; its pad slot R is zeroed by the producer (odd R: the
      // pair (R-1, R) hits the zero pad column).
      const double2* __restrict__ t2s = reinterpret_cast<const double2*>(sv + h.cnt * Rp);
      constexpr int kW = kCons / 32;
      const int w = tid >> 5, sub = lane >> 3, sl = lane & 7, P2 = (R + 1) >> 1;
      for (int jb = 4 * w; jb < h.cnt; jb += 4 * kW) {
        const int j = jb + sub;
        double v0 = 0.0, v1 = 0.0;
        if (j < h.cnt) {
          const double2* __restrict__ u2 = reinterpret_cast<const double2*>(sv + (size_t)j * Rp);
          int cp = sl;
          for (; cp + 8 < P2; cp += 16) {
            const double2 ua = u2[cp], ta = t2s[cp], ub = u2[cp + 8], tb = t2s[cp + 8];
            v0 = fma(ua.x, ta.x, fma(ua.y, ta.y, v0));
            v1 = fma(ub.x, tb.x, fma(ub.y, tb.y, v1));
          }
          if (cp < P2) {
            const double2 ua = u2[cp], ta = t2s[cp];
            v0 = fma(ua.x, ta.x, fma(ua.y, ta.y, v0));
          }
        }
        double v = v0 + v1;
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        if (sl == 0 && j < h.cnt) dc.y1[(int64_t)(h.pad - 1) * dc.n + h.e + rowoff + j] = v;
      }
      rowoff += h.cnt;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.empty[stage]);
    if (++stage == NS) { stage = 0; phase ^= 1; }
    if (!(h.flags & kLast)) continue;
    // ---- end of item: column sums -> t (or this chunk's partials)
    auto put = [&](int qq, double v) {
      if (qq >= R) return;
      if (h.c >= 0) t[vdst[h.c + qq]] = v;
      else tpart[(int64_t)(-h.c - 1) + qq] = v;
    };
    bool fin = false;
    if constexpr (DUAL) if (dcfg >= 0) {
      fin = true;
      switch (dcfg) {
        case 1: dual_finish<1>(S.red, P, acc, put); break;
        case 2: dual_finish<2>(S.red, P, acc, put); break;
        case 3: dual_finish<3>(S.red, P, acc, put); break;
        default: dual_finish<4>(S.red, P, acc, put); break;
      }
    }
    if (fin) {
    } else if (CP == 1) {
      const double s0 = acc[0] + acc[2], s1 = acc[1] + acc[3];
      if (G > 1) {
        S.red[2 * tid] = g < G ? s0 : 0.0;
        S.red[2 * tid + 1] = g < G ? s1 : 0.0;
        group_tree_sum(S.red, G, P, g);
        if (tid < P) {
          put(2 * tid, S.red[2 * tid]);
          put(2 * tid + 1, S.red[2 * tid + 1]);
        }
        named_bar_sync(1, kCons);
      } else if (tid < P) {
        put(2 * tid, s0);
        put(2 * tid + 1, s1);
      }
    } else {
#pragma unroll
      for (int c = 0; c < kMaxCP; ++c)
        if (c < CP && tid + kCons * c < P) {
          put(2 * (tid + kCons * c), acc[2 * c]);
          put(2 * (tid + kCons * c) + 1, acc[2 * c + 1]);
        }
    }
    if (h.d >= 0) {
      // Multi-chunk box: the last chunk to finish sums the partials in chunk order
      // (deterministic) and resets the counter for the next matvec.
      // (the barrier orders every consumer's partial writes before thread 0's gpu-scope
      // fence + atomic; the last arriver's fence orders the other chunks' partials before
      // its consumers' L2 reads)
      named_bar_sync(1, kCons);
      if (tid == 0) {
        __threadfence();
        const int last = atomicAdd(rcount + h.d, 1) == ritems[h.d].nchunks - 1;
        if (last) __threadfence();
        S.flag = last;
      }
      named_bar_sync(1, kCons);
      if (S.flag) {
        const RItem ri = ritems[h.d];
        for (int qq = tid; qq < ri.R; qq += kCons) {
          const double* __restrict__ pp = tpart + ri.p_off + qq;
          double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
          int c = 0;
          for (; c + 3 < ri.nchunks; c += 4) {
            a0 += __ldcg(pp + (int64_t)c * ri.R);
            a1 += __ldcg(pp + (int64_t)(c + 1) * ri.R);
            a2 += __ldcg(pp + (int64_t)(c + 2) * ri.R);
            a3 += __ldcg(pp + (int64_t)(c + 3) * ri.R);
          }
          for (; c < ri.nchunks; ++c) a0 += __ldcg(pp + (int64_t)c * ri.R);
          t[vdst[ri.vpos + qq]] = (a0 + a1) + (a2 + a3);
        }
        if (tid == 0) rcount[h.d] = 0;
      }
    }
  }
}

template <int NS>
__global__ void __launch_bounds__(kPipeThreads, 3)
stageA_tma_kernel(const AItem* __restrict__ items, int n_items, int32_t* counter, LevelPtrs lp,
                  const double* __restrict__ x, const int32_t* __restrict__ vdst, double* __restrict__ t,
                  double* __restrict__ tpart, const RItem* __restrict__ ritems,
                  int32_t* __restrict__ rcount) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  PipeSmem<NS>& S = *reinterpret_cast<PipeSmem<NS>*>(smem_raw);
  pipe_init(S);
  if (threadIdx.x >= kCons) stageA_producer(S, items, n_items, counter, lp, x);
  else stageA_consumers(S, vdst, t, tpart, ritems, rcount);
}

// Symmetric stage B' (R23): t2 = U^T x (stage A over the first-side U box panels,
// written through udst into the second-side t layout) and y1 = U t1 in the same pass.
template <int NS, int SD>
__global__ void __launch_bounds__(kPipeThreads, 3)
stageA_dual_kernel(const AItem* __restrict__ items, int n_items, int32_t* counter, LevelPtrs lp,
                   const double* __restrict__ x, const int32_t* __restrict__ udst, double* __restrict__ t2,
                   double* __restrict__ tpart, const RItem* __restrict__ ritems, int32_t* __restrict__ rcount,
                   const double* __restrict__ t1, double* __restrict__ y1, int64_t n) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  PipeSmem<NS, SD>& S = *reinterpret_cast<PipeSmem<NS, SD>*>(smem_raw);
  pipe_init(S);
  const DualCtx dc{t1, y1, n};
  if (threadIdx.x >= kCons) stageA_producer<NS, true, SD>(S, items, n_items, counter, lp, x, dc);
  else stageA_consumers<NS, true, SD>(S, udst, t2, tpart, ritems, rcount, dc);
}

// ---------------------------------------------------------------- small items
// Items too small for the bulk-copy ring (its per-stage and per-item overhead exceeds their
// bytes; clustered inputs such as the paper's Chebyshev grids put most boxes / leaves here)
// run one warp per item on direct, coalesced 16-byte loads instead.
constexpr int kSmallARows = 32, kSmallBRows = 8;

// Stage A, boxes of <= kSmallARows rows in one chunk: lane owns column pairs pb + lane and
// pb + 32 + lane of a 64-pair block, rows in order; t through vdst (no reduction: the warp
// owns the whole box).
// 8 CTAs per SM (32 registers, 88 bytes spilled): more rows in flight; 4 CTAs per SM at 64
// registers measured 6 % slower on the Chebyshev phi_1 system
constexpr int kSmallAMinBlocks = 8;
__global__ void __launch_bounds__(256, kSmallAMinBlocks)
stageA_small_kernel(const AItem* __restrict__ items, int n_items, LevelPtrs lp, const double* __restrict__ x,
                    const int32_t* __restrict__ vdst, double* __restrict__ t) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < n_items; k += nw) {
    const AItem it = items[k];
    const double* __restrict__ V = lp.V[it.level] + it.v_off;
    const double* __restrict__ xr = x + it.x_off;
    const int P = it.Rp >> 1;
    for (int pb = 0; pb < P; pb += 64) {
      const int p0 = pb + lane, p1 = pb + 32 + lane;
      double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
      for (int j = 0; j < it.nrows; ++j) {
        const double xj = __ldg(xr + j);
        const double2* __restrict__ row = reinterpret_cast<const double2*>(V + (int64_t)j * it.Rp);
        if (p0 < P) {
          const double2 v = __ldcs(row + p0);
          a0 = fma(v.x, xj, a0);
          a1 = fma(v.y, xj, a1);
        }
        if (p1 < P) {
          const double2 v = __ldcs(row + p1);
          b0 = fma(v.x, xj, b0);
          b1 = fma(v.y, xj, b1);
        }
      }
      if (2 * p0 < it.R) t[vdst[it.out + 2 * p0]] = a0;
      if (2 * p0 + 1 < it.R) t[vdst[it.out + 2 * p0 + 1]] = a1;
      if (2 * p1 < it.R) t[vdst[it.out + 2 * p1]] = b0;
      if (2 * p1 + 1 < it.R) t[vdst[it.out + 2 * p1 + 1]] = b1;
    }
  }
}
// Symmetric stage B' (DUAL), boxes of <= kSmallARows rows in one chunk: warp per box, lane owns
// column pair pb + lane of a 32-pair block, rows in groups of 8.  Each U pair feeds the
// column sums t2 (registers; no reduction: the warp owns the box) and the row dots
// y1 = U t1 (the 8 row partials of a group summed over the warp by one transposed butterfly,
// accumulated over the 32-pair blocks in lane 4 t: rows t, t + 8, t + 16, t + 24).  The
// U panel's pad column is zero (memset at pack time) and the t1 pad is read as 0.
__global__ void __launch_bounds__(256, 4)
stageB1_small_kernel(const AItem* __restrict__ items, int n_items, LevelPtrs lp, const double* __restrict__ x,
                     const int32_t* __restrict__ udst, double* __restrict__ t2, const double* __restrict__ t1,
                     double* __restrict__ y1, int64_t n) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < n_items; k += nw) {
    const AItem it = items[k];
    const double2* __restrict__ U2 = reinterpret_cast<const double2*>(lp.Ub[it.level] + it.v_off);
    const double* __restrict__ xr = x + it.x_off;
    const double* __restrict__ tb = t1 + it.t1_off;
    const int P = it.Rp >> 1, rows = it.nrows;
    double yr[4] = {0.0, 0.0, 0.0, 0.0};
    for (int pb = 0; pb < P; pb += 32) {
      const int p = pb + lane;
      const bool vp = p < P;
      const double2 tt = make_double2(vp ? __ldg(tb + 2 * p) : 0.0, vp && 2 * p + 1 < it.R ? __ldg(tb + 2 * p + 1) : 0.0);
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int q = 0; q < kSmallARows / 8; ++q) {
        if (8 * q >= rows) break;   // warp-uniform
        double c[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const int j = 8 * q + t;
          const bool ok = vp && j < rows;
          const double2 u = ok ? __ldcs(U2 + (int64_t)j * P + p) : make_double2(0.0, 0.0);
          const double xj = j < rows ? __ldg(xr + j) : 0.0;
          a0 = fma(u.x, xj, a0);
          a1 = fma(u.y, xj, a1);
          c[t] = fma(u.x, tt.x, u.y * tt.y);
        }
        yr[q] += warp_transpose_sum8(c, lane);
      }
      if (vp) {
        t2[udst[it.out + 2 * p]] = a0;
        if (2 * p + 1 < it.R) t2[udst[it.out + 2 * p + 1]] = a1;
      }
    }
    if ((lane & 3) == 0) {
      double* __restrict__ yrow = y1 + (int64_t)(it.level - 1) * n + it.x_off;
#pragma unroll
      for (int q = 0; q < kSmallARows / 8; ++q) {
        const int j = 8 * q + (lane >> 2);
        if (j < rows) yrow[j] = yr[q];
      }
    }
  }
}

// Stage B, whole leaves of <= kSmallBRows rows: warp per leaf; each level's (leaf, level)
// panel (column-major, mLp <= 8 rows) streams as flat 16-byte elements, 4 per lane in
// flight; 8 row accumulators, reduced over the warp by one transposed butterfly.  (The
// previous column-per-lane loop kept one to four loads per lane in flight and issued a
// dependent descriptor load per level: Chebyshev 500^2 phi_1 matvec 1.262 -> 1.178 ms.)
constexpr int kSmallBSteps = 4;   // flat elements in flight per lane (2: 64 regs but slower; 6, 8: slower)
__global__ void __launch_bounds__(256)
stageB_small_kernel(const BItem* __restrict__ items, const BLevel* __restrict__ blev, int n_items, int kappa,
                    LevelPtrs lp, double* __restrict__ yfar) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < n_items; k += nw) {
    const BItem it = items[k];
    const int mLp = (it.mL + 1) & ~1;
    double acc[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) acc[r] = 0.0;
    // every level's descriptor in one load (lane l - 1 holds level l): the U loads of a level
    // no longer wait behind a dependent descriptor load
    BLevel mine{0, 0, 0};
    if (lane < kappa) mine = blev[(int64_t)k * kappa + lane];
    double pa0 = 0.0, pa1 = 0.0;
    for (int l = 1; l <= kappa; ++l) {
      const int R = __shfl_sync(0xffffffffu, mine.R, l - 1);
      if (R <= 0 || mLp == 0) continue;
      const double* __restrict__ U = lp.U[l] + __shfl_sync(0xffffffffu, mine.uoff, l - 1);
      const double* __restrict__ tb = lp.tu[l] + __shfl_sync(0xffffffffu, mine.tcol, l - 1);
      // the panel as one flat stream of P * R 16-byte elements (P = mLp / 2 row pairs per
      // column): lane takes elements f = lane + 32 s, kSmallBSteps per pass, so every warp
      // load is 512 contiguous bytes whatever mLp is; element f is row pair f % P of column
      // f / P, tracked incrementally (a step of 32 elements: +32 / P columns, +32 % P pairs)
      const int P = mLp >> 1;
      const int Lf = P * R;
      const double2* __restrict__ U2 = reinterpret_cast<const double2*>(U);
      int col = lane / P, rp = lane - (lane / P) * P;
      const int dq = 32 / P, dr = 32 - (32 / P) * P;
      if (dr == 0) {
        // P = 1, 2, 4: the lane's row pair (lane % P) never changes: two accumulators
        for (int f0 = 0; f0 < Lf; f0 += 32 * kSmallBSteps) {
          double2 u[kSmallBSteps];
          double tc[kSmallBSteps];
#pragma unroll
          for (int q = 0; q < kSmallBSteps; ++q) {
            const int f = f0 + 32 * q + lane;
            u[q] = f < Lf ? __ldcs(U2 + f) : make_double2(0.0, 0.0);
            tc[q] = f < Lf ? __ldg(tb + col + q * dq) : 0.0;
          }
          col += kSmallBSteps * dq;
#pragma unroll
          for (int q = 0; q < kSmallBSteps; ++q) {
            pa0 = fma(u[q].x, tc[q], pa0);
            pa1 = fma(u[q].y, tc[q], pa1);
          }
        }
        continue;
      }
      for (int f0 = 0; f0 < Lf; f0 += 32 * kSmallBSteps) {
        double2 u[kSmallBSteps];
        double tc[kSmallBSteps];
        int pr[kSmallBSteps];
#pragma unroll
        for (int q = 0; q < kSmallBSteps; ++q) {
          const int f = f0 + 32 * q + lane;
          pr[q] = rp;
          u[q] = f < Lf ? __ldcs(U2 + f) : make_double2(0.0, 0.0);
          tc[q] = f < Lf ? __ldg(tb + col) : 0.0;
          rp += dr;
          col += dq;
          if (rp >= P) { rp -= P; ++col; }
        }
#pragma unroll
        for (int q = 0; q < kSmallBSteps; ++q)
#pragma unroll
          for (int r2 = 0; r2 < 4; ++r2) {   // selected multiplier: no dynamic register index
            const double w = pr[q] == r2 ? tc[q] : 0.0;
            acc[2 * r2] = fma(u[q].x, w, acc[2 * r2]);
            acc[2 * r2 + 1] = fma(u[q].y, w, acc[2 * r2 + 1]);
          }
      }
    }
    {   // fold the fixed-pair accumulators in (row pair lane % P; P = mLp / 2 <= 4)
      const int P = mLp >> 1;
      const int rp0 = P > 0 ? lane % P : 0;
#pragma unroll
      for (int r2 = 0; r2 < 4; ++r2)
        if (rp0 == r2) {
          acc[2 * r2] += pa0;
          acc[2 * r2 + 1] += pa1;
        }
    }
    const double v = warp_transpose_sum8(acc, lane);
    const int r = lane >> 2;
    if ((lane & 3) == 0 && r < it.rows) yfar[it.yrow + r] = v;
  }
}
// ---------------------------------------------------------------- stage B: yfar = U t
// Item = rows [r0, r0 + rows) (rows <= 256) of served leaf L.  For every ancestor level l
// the leaf's U columns form one contiguous column-major range (stride mLp); a stage holds
// cols_s = min(256, 2048 / rowsp) columns (one bulk copy for whole leaves, one per column
// for row blocks of a leaf > 256 rows) plus their t values (cp.async gather).  Thread
// (g, i) = (tid / rows, tid % rows) owns row i and columns g, g + G, ... (G = 256 / rows),
// reduced in smem at the end of the item: one yfar write per row, no atomics.
// Stage header: a = rows, b = rowsp (row stride inside the stage), c = output row.
template <int NS, int SD = kStageDbl, int SV = kStageVec>
__device__ void stageB_producer(PipeSmem<NS, SD, SV>& S, const BItem* __restrict__ items,
                                const BLevel* __restrict__ blev, int n_items, int32_t* counter,
                                int kappa, const LevelPtrs& lp) {
  const int lane = threadIdx.x & 31;
  const uint64_t pol = l2_evict_first_policy();
  int stage = 0;
  uint32_t phase = 0;
  // one-item lookahead (index + descriptor + per-level metadata in flight, see stage A)
  int idx = 0, nidx = 0;
  if (lane == 0) idx = atomicAdd(counter, 1);
  idx = __shfl_sync(0xffffffffu, idx, 0);
  if (lane == 0) nidx = atomicAdd(counter, 1);
  BItem nit{};
  BLevel nlv{0, 0, 0};
  if (idx < n_items) {
    nit = items[idx];
    if (lane < kappa) nlv = blev[(int64_t)idx * kappa + lane];
  }
  for (;;) {
    const bool done = idx >= n_items;
    const BItem it = nit;
    const BLevel lv = nlv;
    const int cur = idx;
    idx = __shfl_sync(0xffffffffu, nidx, 0);
    if (!done && lane == 0) nidx = atomicAdd(counter, 1);
    if (!done && idx < n_items) {
      nit = items[idx];
      if (lane < kappa) nlv = blev[(int64_t)idx * kappa + lane];
    }
    const int mL = it.mL;
    const int mLp = (mL + 1) & ~1, rowsp = (it.rows + 1) & ~1;
    const bool whole = !done && it.rows == mL;
    // per-level metadata, lane l - 1 <-> level l
    const int R = done || lane >= kappa ? 0 : lv.R;
    const int cb = lv.tcol;
    const int64_t ub = lv.uoff;
    const unsigned nz = __ballot_sync(0xffffffffu, R > 0);
    const int lastl = nz ? 32 - __clz(nz) : 0;
    const int yrow = it.yrow;
    if (done || nz == 0) {
      // terminator, or an item without low-rank columns (kappa = 0 / zero ranks): one
      // empty stage so the consumers still write the item's rows
      mbar_wait(&S.empty[stage], phase ^ 1);
      if (lane == 0) {
        StageHdr& h = S.hdr[stage];
        h.item = done ? -1 : cur;
        h.cnt = 0;
        h.flags = kFirst | kLast;
        h.a = it.rows;
        h.b = rowsp;
        h.c = yrow;
        mbar_arrive_expect_tx(&S.full[stage], 0);
      }
      cp_async_arrive_noinc(&S.full[stage]);
      if (++stage == NS) { stage = 0; phase ^= 1; }
      if (done) break;
      continue;
    }
    // a stage packs consecutive column ranges of successive levels: the (leaf, level)
    // panels share the row stride, so their concatenation is one column-major block and the
    // consumers never see level boundaries (small leaves: one stage per leaf, not per level)
    const int cols_s = min(SV, SD / rowsp);
    bool first = true;
    int fill = 0;
    for (int li = 0; li < lastl; ++li) {
      const int Rl = __shfl_sync(0xffffffffu, R, li);
      const int cbl = __shfl_sync(0xffffffffu, cb, li);
      const int64_t ubl = __shfl_sync(0xffffffffu, ub, li);
      if (Rl == 0) continue;
      const double* Ub = lp.U[li + 1] + ubl;
      const double* tb = lp.tu[li + 1] + cbl;
      for (int c0 = 0; c0 < Rl;) {
        if (fill == 0) mbar_wait(&S.empty[stage], phase ^ 1);
        const int cols = min(cols_s - fill, Rl - c0);
        const bool last = li == lastl - 1 && c0 + cols >= Rl;
        double* dst = S.ring[stage] + fill * rowsp;
        if (lane == 0) {
          mbar_expect_tx(&S.full[stage], (uint32_t)cols * (uint32_t)rowsp * 8u);
          if (whole) bulk_g2s(dst, Ub + (int64_t)c0 * mLp, (uint32_t)cols * (uint32_t)mLp * 8u, &S.full[stage], pol);
        }
        __syncwarp();
        if (!whole)
          for (int c = lane; c < cols; c += 32)
            bulk_g2s(dst + c * rowsp, Ub + (int64_t)(c0 + c) * mLp + it.r0, (uint32_t)rowsp * 8u, &S.full[stage],
                     pol);
        for (int c = lane; c < cols; c += 32) cp_async8(&S.vec[stage][fill + c], tb + c0 + c);
        fill += cols;
        c0 += cols;
        if (fill == cols_s || last) {
          if (lane == 0) {
            StageHdr& h = S.hdr[stage];
            h.item = cur;
            h.cnt = fill;
            h.flags = (first ? kFirst : 0) | (last ? kLast : 0);
            h.a = it.rows;
            h.b = rowsp;
            h.c = yrow;
            mbar_arrive(&S.full[stage]);
          }
          cp_async_arrive_noinc(&S.full[stage]);
          if (++stage == NS) { stage = 0; phase ^= 1; }
          first = false;
          fill = 0;
        }
      }
    }
  }
}

// Consumers work on row pairs (one 16-byte smem load = rows 2i, 2i+1 of a column; rowsp is
// even and the padding row is zero): thread (g, i) = (tid / RP, tid % RP), RP = rowsp / 2,
// owns row pair i and columns g, g + G, ... (G = kCons / RP), reduced in smem per item.
template <int NS, int SD = kStageDbl, int SV = kStageVec>
__device__ void stageB_consumers(PipeSmem<NS, SD, SV>& S, double* __restrict__ yfar) {
  const int tid = threadIdx.x, lane = tid & 31;
  int stage = 0;
  uint32_t phase = 0;
  int rows = 1, rowsp = 2, G = 1, g = 0, i = 0, RP = 1;
  double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
  for (;;) {
    mbar_wait(&S.full[stage], phase);
    const StageHdr h = S.hdr[stage];
    if (h.item < 0) break;
    if (h.flags & kFirst) {
      rows = h.a;
      rowsp = h.b;
      RP = rowsp >> 1;
      G = kCons / RP;
      g = tid / RP;
      i = tid - g * RP;
      a0 = a1 = b0 = b1 = 0.0;
    }
    if (g < G) {
      const double* __restrict__ u = S.ring[stage] + (size_t)g * rowsp + 2 * i;
      const double* __restrict__ tv = S.vec[stage];
      const int cols = h.cnt, step = G * rowsp;
      int c = g;
      for (; c + G < cols; c += 2 * G, u += 2 * step) {
        const double2 ua = *reinterpret_cast<const double2*>(u);
        const double2 ub = *reinterpret_cast<const double2*>(u + step);
        const double ta = tv[c], tb = tv[c + G];
        a0 = fma(ua.x, ta, a0);
        a1 = fma(ua.y, ta, a1);
        b0 = fma(ub.x, tb, b0);
        b1 = fma(ub.y, tb, b1);
      }
      if (c < cols) {
        const double2 ua = *reinterpret_cast<const double2*>(u);
        const double ta = tv[c];
        a0 = fma(ua.x, ta, a0);
        a1 = fma(ua.y, ta, a1);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.empty[stage]);
    if (++stage == NS) { stage = 0; phase ^= 1; }
    if (!(h.flags & kLast)) continue;
    S.red[2 * tid] = g < G ? a0 + b0 : 0.0;
    S.red[2 * tid + 1] = g < G ? a1 + b1 : 0.0;
    group_tree_sum(S.red, G, RP, g);
    if (tid < rows) yfar[h.c + tid] = S.red[tid];   // group 0: red[2 i + e] = row 2 i + e
    named_bar_sync(1, kCons);
  }
}

template <int NS, int SD = kStageDbl, int SV = kStageVec>
__global__ void __launch_bounds__(kPipeThreads, 3)
stageB_tma_kernel(const BItem* __restrict__ items, const BLevel* __restrict__ blev, int n_items,
                  int32_t* counter, int kappa, LevelPtrs lp, double* __restrict__ yfar) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  PipeSmem<NS, SD, SV>& S = *reinterpret_cast<PipeSmem<NS, SD, SV>*>(smem_raw);
  pipe_init(S);
  if (threadIdx.x >= kCons) stageB_producer(S, items, blev, n_items, counter, kappa, lp);
  else stageB_consumers(S, yfar);
}

}  // namespace
}  // namespace h2d
