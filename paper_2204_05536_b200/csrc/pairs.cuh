// Pair-local symmetric apply (NEXT N1 payoff, R23 / §6 "pair apply").
//
// A symmetric build stores one factor pair per unordered box pair {X, Y}, X < Y (Morton):
// K(X, Y) ~ U V^T and K(Y, X) ~ V U^T (the paper's symmetric setting).  Alg. 2 l.15
// then needs, per pair, t1 = V^T x_Y, t2 = U^T x_X, y_X += U t1 and y_Y += V t2:
// each factor is used twice, and each product of one factor needs the other factor's
// reduction first.  The three-pass apply (A' / B' / C') reads 3 of the 4 factor streams;
// this kernel reads each factor ONCE from HBM by keeping the pair local:
//   phase 1  stream V rows       -> column sums t1 = V^T x_Y
//   phase 2  stream U rows       -> column sums t2 = U^T x_X and row dots dy_X = U t1
//   phase 3  stream V rows again -> row dots dy_Y = V t2 (an L2 hit: V was just read)
// dy rows go to the TREE-order accumulator yacc (8 MB at C3: L2-resident) by fp64 REDs.  Pairs up to kPWholeBytes run all
// three phases in one CTA (t1 / t2 in shared memory); bigger pairs (the coarse levels) are cut
// into row chunks that any CTA takes: the last chunk of a phase reduces the partials (in
// chunk order, deterministic) and publishes t1 / t2 with a flag (epoch = matvec count); the
// producer of a later phase's chunk waits for that flag before it loads the t values.  The
// queue interleaves the big pairs (phase 1 of pair k beside phase 2 of pair k-1 and phase 3
// of pair k-2) so a V chunk is re-read while it is still in L2.
// Not bitwise reproducible: the order of the y accumulations varies between runs.
#pragma once
#include "pipe.cuh"

namespace h2d {
namespace {

constexpr int kPNS = 3;              // ring depth
constexpr int kPSD = 3072;           // factor doubles per stage (24 KB; 2 CTAs + the P2P per SM)
constexpr int kPSV = 256;            // rows per stage (x values, dy staging)
constexpr int kPMaxRp = 128;         // widest pair panel (Rp = rank rounded up to even)
constexpr int kPWholeBytes = 400 * 1024;   // pairs up to this size: one CTA, all phases
constexpr int kPChunkDbl = 8192;     // big pairs: row chunks of <= 64 KB

enum { kPWhole = 0, kPPhase1 = 1, kPPhase2 = 2, kPPhase3 = 3, kPOneStage = 4 };

struct PItem {
  int64_t v_off, u_off;   // pair array offsets of V (nv x Rp) and U (nu x Rp), row-major
  int32_t yv, yu;         // TREE rows of Y (V rows) and X (U rows)
  int32_t nv, nu;         // rows of V and U
  int32_t R, Rp;
  int32_t kind;           // kPWhole or the phase of a chunk
  int32_t r0, nrows;      // chunk: rows [r0, r0 + nrows) of the phase's factor
  int32_t big;            // chunk: big-pair index (flags, counters)
  int32_t part;           // chunk of phase 1 / 2: first partial slot of this chunk
  int32_t nchunks;        // chunk of phase 1 / 2: chunks of that phase
  int32_t chunk;          // chunk index inside its phase
  int64_t toff;           // big pair: offset of its t1 / t2 in tP1 / tP2
  int64_t poff;           // big pair: first partial slot of its phase (chunk c at poff + c R)
  int32_t level;          // pair array of the level (PairPtrs)
  int32_t pad;
};
struct PairPtrs {
  const double* P[H2D_MAX_LEVELS + 1];
};

struct PairSmem {
  double ring[kPNS][kPSD];
  double vec[kPNS][kPSV];          // x values of the stage rows
  double tslot[kPNS][kPMaxRp];     // chunks of phases 2 / 3: t1 / t2 of the pair
  double tS[2][kPMaxRp];           // whole pairs: t1, t2
  double red[7 * 64];
  StageHdr hdr[kPNS];
  uint64_t full[kPNS];
  uint64_t empty[kPNS];
  int flag;
};

__device__ __forceinline__ int ld_acquire(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int32_t* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// ---------------------------------------------------------------- producer
__device__ void pair_producer(PairSmem& S, const PItem* __restrict__ items, int n_items, int32_t* counter,
                              const PairPtrs& pp, const double* __restrict__ x,
                              const double* __restrict__ tP1, const double* __restrict__ tP2,
                              const int32_t* __restrict__ flags, int epoch) {
  const int lane = threadIdx.x & 31;
  const uint64_t pol_first = l2_evict_first_policy();
  int stage = 0;
  uint32_t phase = 0;
  // the next item is reserved only after the current one's flag wait (a producer that waits
  // holds no other item, so chains of waits stay two deep); its descriptor load overlaps the
  // current item's stages
  int idx = 0;
  if (lane == 0) idx = atomicAdd(counter, 1);
  idx = __shfl_sync(0xffffffffu, idx, 0);
  PItem nit{};
  if (idx < n_items) nit = items[idx];
  // one stage: rows [r0, r0 + rows) of a row-major panel at src, the x values of those rows
  // (xs != nullptr) and the t values of the phase (tsrc != nullptr, R of them)
  auto emit = [&](int item, int ph, int rows, int flags_, int Rp, int R, int y0, const double* src, bool keep,
                  const double* xs, const double* tsrc) {
    mbar_wait(&S.empty[stage], phase ^ 1);
    if (tsrc && lane == 0 && (R & 1)) S.tslot[stage][R] = 0.0;   // pad partner (released below)
    if (lane == 0) {
      StageHdr& h = S.hdr[stage];
      h.item = item;
      h.cnt = rows;
      h.flags = flags_;
      h.a = ph;
      h.b = Rp;
      h.c = R;
      h.e = y0;
      const uint32_t bytes = (uint32_t)rows * (uint32_t)Rp * 8u;
      mbar_arrive_expect_tx(&S.full[stage], bytes);
      if (bytes) {
        if (keep) bulk_g2s_keep(S.ring[stage], src, bytes, &S.full[stage]);
        else bulk_g2s(S.ring[stage], src, bytes, &S.full[stage], pol_first);
      }
    }
    if (xs)
      for (int j = lane; j < rows; j += 32) cp_async8(&S.vec[stage][j], xs + j);
    if (tsrc)
      for (int q = lane; q < R; q += 32) cp_async8(&S.tslot[stage][q], tsrc + q);
    cp_async_arrive_noinc(&S.full[stage]);
    if (++stage == kPNS) { stage = 0; phase ^= 1; }
  };
  for (;;) {
    if (idx >= n_items) {
      emit(-1, 0, 0, 0, 2, 0, 0, nullptr, false, nullptr, nullptr);
      break;
    }
    const PItem it = nit;
    const int cur = idx;
    const double* tsrc = nullptr;
    if (it.kind >= 2) {   // phase 2 / 3 chunk: the other factor's reduction must be published
      const int32_t* f = flags + 2 * it.big + (it.kind - 2);
      if (lane == 0)
        while (ld_acquire(f) < epoch) __nanosleep(100);
      __syncwarp();
      __threadfence();   // (invalidates this SM's L1 before the t loads)
      tsrc = (it.kind == 2 ? tP1 : tP2) + it.toff;
    }
    int nx = 0;
    if (lane == 0) nx = atomicAdd(counter, 1);
    idx = __shfl_sync(0xffffffffu, nx, 0);
    if (idx < n_items) nit = items[idx];
    const int rows_s = min(kPSV, kPSD / it.Rp);
    if (it.kind == kPWhole && (it.nv + it.nu) * it.Rp <= kPSD && it.nv + it.nu <= kPSV) {
      // the whole pair in one stage (V then U are adjacent in the pair array): phases 1-3
      // all read this stage, nothing is re-read
      mbar_wait(&S.empty[stage], phase ^ 1);
      if (lane == 0) {
        StageHdr& h = S.hdr[stage];
        h.item = cur;
        h.cnt = it.nv;
        h.flags = kFirst | kLast;
        h.a = kPOneStage;
        h.b = it.Rp;
        h.c = it.R;
        h.d = it.nu;
        h.e = it.yv;
        h.f = it.yu;
        const uint32_t bytes = (uint32_t)(it.nv + it.nu) * (uint32_t)it.Rp * 8u;
        mbar_arrive_expect_tx(&S.full[stage], bytes);
        bulk_g2s(S.ring[stage], pp.P[it.level] + it.v_off, bytes, &S.full[stage], pol_first);
      }
      for (int j = lane; j < it.nv; j += 32) cp_async8(&S.vec[stage][j], x + it.yv + j);
      for (int j = lane; j < it.nu; j += 32) cp_async8(&S.vec[stage][it.nv + j], x + it.yu + j);
      cp_async_arrive_noinc(&S.full[stage]);
      if (++stage == kPNS) { stage = 0; phase ^= 1; }
      continue;
    }
    if (it.kind == kPWhole) {
      for (int ph = 1; ph <= 3; ++ph) {
        const int n = ph == 2 ? it.nu : it.nv;
        const double* src = pp.P[it.level] + (ph == 2 ? it.u_off : it.v_off);
        const int y0 = ph == 2 ? it.yu : it.yv;
        for (int r0 = 0; r0 < n; r0 += rows_s) {
          const int rows = min(rows_s, n - r0);
          const int fl = (r0 == 0 ? kFirst : 0) | (r0 + rows >= n ? kLast : 0);
          emit(cur, ph, rows, fl, it.Rp, it.R, y0 + r0, src + (int64_t)r0 * it.Rp, ph == 1,
               ph == 3 ? nullptr : x + y0 + r0, nullptr);
        }
      }
      continue;
    }
    // a chunk of one phase of a big pair
    const int ph = it.kind;
    const double* src = pp.P[it.level] + (ph == 2 ? it.u_off : it.v_off) + (int64_t)it.r0 * it.Rp;
    const int y0 = (ph == 2 ? it.yu : it.yv) + it.r0;
    for (int r0 = 0; r0 < it.nrows; r0 += rows_s) {
      const int rows = min(rows_s, it.nrows - r0);
      const int fl = (r0 == 0 ? kFirst : 0) | (r0 + rows >= it.nrows ? kLast : 0);
      emit(cur, ph, rows, fl, it.Rp, it.R, y0 + r0, src + (int64_t)r0 * it.Rp, ph == 1,
           ph == 3 ? nullptr : x + y0 + r0, tsrc);
    }
  }
}

// ---------------------------------------------------------------- consumers
// Warp per row group (rows w, w + 7, w + 14, w + 21 of every 28-row block), lane owns column
// pairs lane + 32 c (c < C); COLS: column sums acc += v x_j; ROWS: row dots dy_j = v . t,
// four rows reduced together by a transposed butterfly (as the symmetric B' kernel); each
// row's dot is added to the TREE-order accumulator (dy = yacc + first row) by an fp64 RED.
template <int C, bool COLS, bool ROWS>
__device__ __forceinline__ void pair_consume(const double* __restrict__ sv, const double* __restrict__ sx, int rows,
                                             int Rp, int P, double (&acc)[4], const double* __restrict__ tv,
                                             double* __restrict__ dy) {
  constexpr int kW = kCons / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double2 tt[C];
  if (ROWS) {
    const double2* __restrict__ t2 = reinterpret_cast<const double2*>(tv);
#pragma unroll
    for (int c = 0; c < C; ++c) tt[c] = lane + 32 * c < P ? t2[lane + 32 * c] : make_double2(0.0, 0.0);
  }
  for (int jb = w; jb < rows; jb += 4 * kW) {
    double r[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      r[k] = 0.0;
      const int j = jb + kW * k;
      if (j < rows) {
        const double xj = COLS ? sx[j] : 0.0;
        const double2* __restrict__ u2 = reinterpret_cast<const double2*>(sv + j * Rp);
#pragma unroll
        for (int c = 0; c < C; ++c)
          if (lane + 32 * c < P) {
            const double2 a = u2[lane + 32 * c];
            if (COLS) {
              acc[2 * c] = fma(a.x, xj, acc[2 * c]);
              acc[2 * c + 1] = fma(a.y, xj, acc[2 * c + 1]);
            }
            if (ROWS) r[k] = fma(a.x, tt[c].x, fma(a.y, tt[c].y, r[k]));
          }
      }
    }
    if (ROWS) {
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
      if ((lane & 7) == 0 && j < rows) atomicAdd(dy + j, v);   // RED.ADD.F64 into yacc
    }
  }
}

// Column sums over the 7 warps, handed to put(q, value) for q < 2 P (one 64-value block of
// column pairs at a time, as dual_finish).
template <int C, typename Put>
__device__ __forceinline__ void pair_colsum_finish(double* red, int P, double (&acc)[4], Put&& put) {
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

__device__ void pair_consumers(PairSmem& S, const PItem* __restrict__ items, double* __restrict__ yacc,
                               double* __restrict__ tP1, double* __restrict__ tP2, double* __restrict__ tpart,
                               int32_t* __restrict__ pcount, int32_t* __restrict__ flags, int epoch) {
  const int tid = threadIdx.x;
  int stage = 0;
  uint32_t phase = 0;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (;;) {
    mbar_wait(&S.full[stage], phase);
    const StageHdr h = S.hdr[stage];
    if (h.item < 0) break;
    const int ph = h.a, Rp = h.b, R = h.c, P = Rp >> 1, rows = h.cnt;
    const bool two = P > 32;
    if (ph == kPOneStage) {
      // whole pair in this stage: rows [0, nv) = V (x_Y in vec[0, nv)), rows [nv, nv + nu) = U
      const int nv = rows, nu = h.d;
      const double* sv = S.ring[stage];
      const double* sx = S.vec[stage];
      auto zero = [&] { acc[0] = acc[1] = acc[2] = acc[3] = 0.0; };
      auto put_t = [&](double* ts) { return [ts, R, Rp](int q, double v) { if (q < Rp) ts[q] = q < R ? v : 0.0; }; };
      // phase 1: t1 = V^T x_Y
      zero();
      if (two) pair_consume<2, true, false>(sv, sx, nv, Rp, P, acc, nullptr, nullptr);
      else pair_consume<1, true, false>(sv, sx, nv, Rp, P, acc, nullptr, nullptr);
      if (two) pair_colsum_finish<2>(S.red, P, acc, put_t(S.tS[0]));
      else pair_colsum_finish<1>(S.red, P, acc, put_t(S.tS[0]));
      // phase 2: t2 = U^T x_X, dy_X = U t1
      zero();
      if (two) pair_consume<2, true, true>(sv + nv * Rp, sx + nv, nu, Rp, P, acc, S.tS[0], yacc + h.f);
      else pair_consume<1, true, true>(sv + nv * Rp, sx + nv, nu, Rp, P, acc, S.tS[0], yacc + h.f);
      if (two) pair_colsum_finish<2>(S.red, P, acc, put_t(S.tS[1]));
      else pair_colsum_finish<1>(S.red, P, acc, put_t(S.tS[1]));
      // phase 3: dy_Y = V t2
      if (two) pair_consume<2, false, true>(sv, sx, nv, Rp, P, acc, S.tS[1], yacc + h.e);
      else pair_consume<1, false, true>(sv, sx, nv, Rp, P, acc, S.tS[1], yacc + h.e);
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&S.empty[stage]);
      if (++stage == kPNS) { stage = 0; phase ^= 1; }
      continue;
    }
    if (h.flags & kFirst) acc[0] = acc[1] = acc[2] = acc[3] = 0.0;
    const double* sv = S.ring[stage];
    const double* sx = S.vec[stage];
    const bool whole = items[h.item].kind == kPWhole;
    const double* tv = ph == 1 ? nullptr : whole ? S.tS[ph - 2] : S.tslot[stage];
    double* dy = yacc + h.e;
    if (ph == 1) {
      if (two) pair_consume<2, true, false>(sv, sx, rows, Rp, P, acc, tv, dy);
      else pair_consume<1, true, false>(sv, sx, rows, Rp, P, acc, tv, dy);
    } else if (ph == 2) {
      if (two) pair_consume<2, true, true>(sv, sx, rows, Rp, P, acc, tv, dy);
      else pair_consume<1, true, true>(sv, sx, rows, Rp, P, acc, tv, dy);
    } else {
      if (two) pair_consume<2, false, true>(sv, sx, rows, Rp, P, acc, tv, dy);
      else pair_consume<1, false, true>(sv, sx, rows, Rp, P, acc, tv, dy);
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&S.empty[stage]);
    if (++stage == kPNS) { stage = 0; phase ^= 1; }
    if (!(h.flags & kLast) || ph == 3) continue;
    // ---- end of a column-sum phase (1 or 2): t1 / t2
    const PItem it = items[h.item];
    if (it.kind == kPWhole) {
      double* ts = S.tS[ph - 1];
      auto put = [&](int q, double v) { if (q < Rp) ts[q] = q < R ? v : 0.0; };
      if (two) pair_colsum_finish<2>(S.red, P, acc, put);
      else pair_colsum_finish<1>(S.red, P, acc, put);
      continue;   // (the finish ends with a consumer barrier: tS is visible)
    }
    double* part = tpart + it.poff + (int64_t)it.chunk * R;
    auto put = [&](int q, double v) { if (q < R) part[q] = v; };
    if (two) pair_colsum_finish<2>(S.red, P, acc, put);
    else pair_colsum_finish<1>(S.red, P, acc, put);
    // the last chunk of the phase sums the partials in chunk order and publishes the t values
    if (tid == 0) {
      __threadfence();
      const int32_t* cntp = pcount + 2 * it.big + (ph - 1);
      const int last = atomicAdd(const_cast<int32_t*>(cntp), 1) == it.nchunks - 1;
      if (last) __threadfence();
      S.flag = last;
    }
    named_bar_sync(1, kCons);
    if (S.flag) {
      double* tout = (ph == 1 ? tP1 : tP2) + it.toff;
      for (int q = tid; q < R; q += kCons) {
        const double* __restrict__ pp = tpart + it.poff + q;
        double a0 = 0.0, a1 = 0.0;
        int c = 0;
        for (; c + 1 < it.nchunks; c += 2) {
          a0 += __ldcg(pp + (int64_t)c * R);
          a1 += __ldcg(pp + (int64_t)(c + 1) * R);
        }
        if (c < it.nchunks) a0 += __ldcg(pp + (int64_t)c * R);
        tout[q] = a0 + a1;
      }
      named_bar_sync(1, kCons);
      if (tid == 0) {
        pcount[2 * it.big + (ph - 1)] = 0;
        __threadfence();
        st_release(flags + 2 * it.big + (ph - 1), epoch);
      }
    }
  }
}

__global__ void __launch_bounds__(kPipeThreads, 2)
pair_apply_kernel(const PItem* __restrict__ items, int n_items, int32_t* counter, PairPtrs pp,
                  const double* __restrict__ x, double* __restrict__ yacc, double* __restrict__ tP1,
                  double* __restrict__ tP2, double* __restrict__ tpart, int32_t* __restrict__ pcount,
                  int32_t* __restrict__ flags, int epoch) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  PairSmem& S = *reinterpret_cast<PairSmem*>(smem_raw);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kPNS; ++s) {
      mbar_init(&S.full[s], 1 + 32);
      mbar_init(&S.empty[s], kCons / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x >= kCons) pair_producer(S, items, n_items, counter, pp, x, tP1, tP2, flags, epoch);
  else pair_consumers(S, items, yacc, tP1, tP2, tpart, pcount, flags, epoch);
}

}  // namespace
}  // namespace h2d
