// Pair-local symmetric apply (NEXT N1 payoff, R23 / §10 "pair apply").
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
// Layout: each factor (n rows x r columns) is stored tile-major — 32-row tiles (the last one
// padded to an even row count), each tile column-major — so any (tile, block of <= 16
// columns) is one contiguous range: a "sub-tile".  Every warp runs its own pipeline: it
// reserves work items from a queue, issues the sub-tiles of its items into a ring of kPSlots
// shared-memory slots by bulk copies (TMA engine; the x values of the rows by 8-byte
// cp.async on the same mbarrier) up to kPSlots ahead, across item boundaries, and consumes
// them in order with lane = row: column sums by warp shuffles at the end of each column block,
// row dots added to the TREE-order accumulator yacc by fp64 REDs.  Items: a whole small /
// medium pair (all three phases in one warp), or a chunk of tiles of one phase of a big pair
// (any warp; the last chunk of a phase reduces the partials in chunk order and publishes t1 /
// t2 behind a flag = matvec epoch; a later phase's chunk waits for it when it starts consuming).
// The queue puts every chunk after all chunks of its pair's previous phase, and a warp only
// waits on items earlier in the queue than the one it consumes, so the earliest unfinished
// item always progresses.  Not bitwise reproducible (the order of the y accumulations varies).
#pragma once
#include "pipe.cuh"

namespace h2d {
namespace {

constexpr int kPWarps = 8;                  // warps per CTA (each its own pipeline)
constexpr int kPSlots = 5;                  // ring slots per warp
constexpr int kPCB = 16;                    // columns per sub-tile
constexpr int kPMaxR = 128;                 // widest pair (rank)
constexpr int kPWholeBytes = 96 * 1024;     // pairs up to this: one warp, all phases
constexpr int kPChunkTiles = 16;            // big pairs: chunks of 16 tiles (512 rows) per phase

enum { kPWhole = 0, kPPhase1 = 1, kPPhase2 = 2, kPPhase3 = 3 };

struct PPair {              // one stored pair
  int64_t v_off, u_off;     // V (nv x r) and U (nu x r), tile-major, in the level's pair array
  int32_t yv, yu;           // TREE rows of Y (V rows) and X (U rows)
  int32_t nv, nu, r, level;
};
struct PWork {              // one work item (a warp takes it)
  int32_t kind;             // kPWhole, or the phase of a chunk
  int32_t pair;
  int32_t t0, t1;           // chunk: tiles [t0, t1) of the phase's factor
  int32_t big, chunk, nchunks, pad;
  int64_t toff, poff;       // big pair: t1 / t2 offset; partial slots of the phase
};
struct PairPtrs {
  const double* P[H2D_MAX_LEVELS + 1];
};

// one issued sub-tile (shared, per slot)
struct PSub {
  int32_t item;             // work item index; -1 = none (end of the queue)
  int32_t ph;               // phase 1..3
  int32_t c0, nc;           // column block
  int32_t rows;             // rows of the tile (unpadded)
  int32_t y0;               // TREE row of the tile's first row
  int32_t flags;            // kSubFirstBlk / kSubLastBlk / kSubLastPh / kSubFirstItem
  int32_t prow;             // padded rows (leading dimension in the slot)
  int32_t t;                // tile index in the factor
};
constexpr int kSubFirstBlk = 1, kSubLastBlk = 2, kSubLastPh = 4, kSubFirstItem = 8;

struct PairWarpSmem {
  double data[kPSlots][32 * kPCB];
  double xs[kPSlots][32];
  PSub sub[kPSlots];
  uint64_t full[kPSlots];
  double t[2][kPMaxR];      // whole pairs: t1, t2; chunks: t of the phase in t[0]
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

// The issue side of a warp's pipeline: walks the sub-tiles of its reserved items in order.
struct PIssue {
  int item = -1;            // current item (-1: reserve the next one)
  PWork w;
  PPair p;
  int ph = 1, cb = 0, t = 0, tend = 0;
  bool done = false;
  bool first = true;
};

__device__ void pair_issue_next(PIssue& is, const PWork* __restrict__ work, int n_work, const PPair* __restrict__ pairs,
                                int32_t* counter, PSub& s) {
  const int lane = threadIdx.x & 31;
  if (is.done) { s.item = -1; return; }
  if (is.item < 0) {
    int idx = 0;
    if (lane == 0) idx = atomicAdd(counter, 1);
    idx = __shfl_sync(0xffffffffu, idx, 0);
    if (idx >= n_work) { is.done = true; s.item = -1; return; }
    is.item = idx;
    is.w = work[idx];
    is.p = pairs[is.w.pair];
    is.ph = is.w.kind == kPWhole ? 1 : is.w.kind;
    is.cb = 0;
    const int n = is.ph == 2 ? is.p.nu : is.p.nv;
    is.t = is.w.kind == kPWhole ? 0 : is.w.t0;
    is.tend = is.w.kind == kPWhole ? (n + 31) / 32 : is.w.t1;
    is.first = true;
  }
  const PPair& p = is.p;
  const int n = is.ph == 2 ? p.nu : p.nv;
  const int nblk = (p.r + kPCB - 1) / kPCB;
  s.item = is.item;
  s.ph = is.ph;
  s.c0 = is.cb * kPCB;
  s.nc = min(kPCB, p.r - s.c0);
  s.rows = min(32, n - 32 * is.t);
  s.prow = (s.rows + 1) & ~1;
  s.y0 = (is.ph == 2 ? p.yu : p.yv) + 32 * is.t;
  s.t = is.t;
  const int t0 = is.w.kind == kPWhole ? 0 : is.w.t0;
  s.flags = (is.t == t0 ? kSubFirstBlk : 0) | (is.t + 1 == is.tend ? kSubLastBlk : 0) |
            (is.first ? kSubFirstItem : 0);
  const bool last_blk_of_phase = is.t + 1 == is.tend && is.cb + 1 == nblk;
  if (last_blk_of_phase) s.flags |= kSubLastPh;
  is.first = false;
  // advance: tiles inner, column blocks outer, phases (whole pairs) outermost
  if (++is.t == is.tend) {
    is.t = t0;
    if (++is.cb == nblk) {
      is.cb = 0;
      if (is.w.kind == kPWhole && is.ph < 3) {
        ++is.ph;
        const int n2 = is.ph == 2 ? p.nu : p.nv;
        is.t = 0;
        is.tend = (n2 + 31) / 32;
      } else {
        is.item = -1;
      }
    }
  }
}

__global__ void __launch_bounds__(32 * kPWarps, 1)
pair_apply_kernel(const PWork* __restrict__ work, int n_work, const PPair* __restrict__ pairs, int32_t* counter,
                  PairPtrs pp, const double* __restrict__ x, double* __restrict__ yacc, double* __restrict__ tP1,
                  double* __restrict__ tP2, double* __restrict__ tpart, int32_t* __restrict__ pcount,
                  int32_t* __restrict__ flags, int epoch) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  PairWarpSmem& S = reinterpret_cast<PairWarpSmem*>(smem_raw)[wid];
  if (lane == 0) {
    for (int k = 0; k < kPSlots; ++k) mbar_init(&S.full[k], 1 + 32);
    mbar_fence_init();
  }
  __syncwarp();
  const uint64_t pol_first = l2_evict_first_policy();
  PIssue is;
  uint32_t phase_bits = 0;   // parity of each slot's next completion
  int issue_k = 0, cons_k = 0, inflight = 0;
  // issue one sub-tile into slot issue_k (returns false at the end of the queue)
  auto issue = [&]() -> bool {
    PSub s;
    pair_issue_next(is, work, n_work, pairs, counter, s);
    if (s.item < 0) return false;
    const int k = issue_k;
    __syncwarp();
    if (lane == 0) S.sub[k] = s;
    const PPair& p = is.p;   // (the pair of s: replaced only when the next item is reserved)
    const double* base = pp.P[p.level] + (s.ph == 2 ? p.u_off : p.v_off);
    // tile t starts after t full tiles (32 x r each); column block c0 inside it
    const double* src = base + (int64_t)32 * s.t * p.r + (int64_t)s.c0 * s.prow;
    if (lane == 0) {
      const uint32_t bytes = (uint32_t)s.prow * (uint32_t)s.nc * 8u;
      mbar_arrive_expect_tx(&S.full[k], bytes);
      if (s.ph == 1) bulk_g2s_keep(S.data[k], src, bytes, &S.full[k]);
      else bulk_g2s(S.data[k], src, bytes, &S.full[k], pol_first);
    }
    if (s.ph != 3 && lane < s.rows) cp_async8(&S.xs[k][lane], x + s.y0 + lane);
    cp_async_arrive_noinc(&S.full[k]);
    issue_k = issue_k + 1 == kPSlots ? 0 : issue_k + 1;
    ++inflight;
    return true;
  };
  bool more = true;
  while (more && inflight < kPSlots - 1) more = issue();
  double acc[kPCB];
  while (inflight > 0) {
    const int k = cons_k;
    mbar_wait(&S.full[k], (phase_bits >> k) & 1u);
    phase_bits ^= 1u << k;
    const PSub s = S.sub[k];
    const PWork w = work[s.item];
    const PPair p = pairs[w.pair];
    const bool whole = w.kind == kPWhole;
    double* tv = S.t[0];      // t of the phase's row dots (whole: t1 in t[0], t2 in t[1])
    if (whole && s.ph == 3) tv = S.t[1];
    if (!whole && s.ph >= 2 && (s.flags & kSubFirstItem)) {
      // a phase 2 / 3 chunk: wait for the other factor's published reduction
      const int32_t* f = flags + 2 * w.big + (s.ph - 2);
      if (lane == 0)
        while (ld_acquire(f) < epoch) __nanosleep(100);
      __syncwarp();
      __threadfence();
      const double* tg = (s.ph == 2 ? tP1 : tP2) + w.toff;
      for (int q = lane; q < p.r; q += 32) S.t[0][q] = __ldcg(tg + q);
      __syncwarp();
    }
    if (s.flags & kSubFirstBlk) {
#pragma unroll
      for (int q = 0; q < kPCB; ++q) acc[q] = 0.0;
    }
    const double* d = S.data[k];
    const bool ok = lane < s.rows;
    const double xv = (s.ph != 3 && ok) ? S.xs[k][lane] : 0.0;
    double dot0 = 0.0, dot1 = 0.0;
#pragma unroll
    for (int q = 0; q < kPCB; ++q) {
      if (q < s.nc) {
        const double v = ok ? d[q * s.prow + lane] : 0.0;
        if (s.ph != 3) acc[q] = fma(v, xv, acc[q]);
        if (s.ph != 1) {
          if (q & 1) dot1 = fma(v, tv[s.c0 + q], dot1);
          else dot0 = fma(v, tv[s.c0 + q], dot0);
        }
      }
    }
    __syncwarp();   // the slot's data and header are read: it may be refilled
    cons_k = cons_k + 1 == kPSlots ? 0 : cons_k + 1;
    --inflight;
    if (more) more = issue();
    if (s.ph != 1 && ok) atomicAdd(yacc + s.y0 + lane, dot0 + dot1);
    if (s.ph != 3 && (s.flags & kSubLastBlk)) {
      // end of a column block: column sums of this warp
      double* out = whole ? S.t[s.ph - 1] : tpart + w.poff + (int64_t)w.chunk * p.r;
#pragma unroll
      for (int q = 0; q < kPCB; ++q) {
        const double v = warp_sum(acc[q]);
        if (lane == 0 && q < s.nc) out[s.c0 + q] = v;
      }
      __syncwarp();
      if (!whole && (s.flags & kSubLastPh)) {
        // the last chunk of the phase reduces the partials in chunk order and publishes t
        int last = 0;
        if (lane == 0) {
          __threadfence();
          last = atomicAdd(pcount + 2 * w.big + (s.ph - 1), 1) == w.nchunks - 1;
          if (last) __threadfence();
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {
          double* tout = (s.ph == 1 ? tP1 : tP2) + w.toff;
          for (int q = lane; q < p.r; q += 32) {
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
          __syncwarp();
          if (lane == 0) {
            pcount[2 * w.big + (s.ph - 1)] = 0;
            __threadfence();
            st_release(flags + 2 * w.big + (s.ph - 1), epoch);
          }
        }
      }
    }
  }
}

}  // namespace
}  // namespace h2d
