// Pair-local symmetric apply (NEXT N1 payoff, R23 / §10 "pair apply").
//
// A symmetric build stores one factor pair per unordered box pair {X, Y}, X < Y (Morton):
// K(X, Y) ~ U V^T and K(Y, X) ~ V U^T (the paper's symmetric setting).  Alg. 2 l.15
// then needs, per pair, t1 = V^T x_Y, t2 = U^T x_X, y_X += U t1 and y_Y += V t2:
// each factor is used twice, and each product of one factor needs the other factor's
// reduction first.  The three-pass apply (A' / B' / C') reads 3 of the 4 factor streams;
// this kernel reads each factor once from HBM:
//   phase 1  V rows          -> column sums t1 = V^T x_Y
//   phase 2  U rows          -> column sums t2 = U^T x_X and row dots dy_X = U t1
//   phase 3  V rows again    -> row dots dy_Y = V t2
// Persistent kernel, one CTA per SM: a producer warp streams work units into a ring of
// 32 KB shared-memory slots (cp.async.bulk: the unit's factor block plus the x segments of
// its rows, completion on the slot's mbarrier); consumer warps take the slots in order and
// compute from shared memory only (lane = row of a column-major block: conflict-free), so
// a unit costs no global round trip (the y / t updates are fire-and-forget REDs).  The
// producer takes units from the global queue in batches (one atomic and one coalesced
// descriptor load per batch, the next batch's atomic in flight meanwhile).
// Units:
//   whole  a pair whose V and U fit one slot together: all three phases in one warp, phase 3
//          re-reads V from shared memory (no second HBM or L2 read);
//   chunk  one row chunk of one phase of a larger pair (the coarse levels): phases 1 / 2
//          add their column sums to t1 / t2 in global memory (fp64 REDs); the last chunk of
//          a phase publishes a flag (= matvec epoch); a phase-2 / 3 chunk waits for it.
//          The phase-3 V chunk is re-read (the schedule places it close behind phase 1, so
//          it mostly hits L2; phase-1 copies carry no evict-first hint for that reason).
// Deadlock freedom: the global queue puts every chunk after all chunks of its pair's
// previous phase, the producer takes a unit only once a slot is free (it never waits on
// anything else), and consumers take units in queue order; the earliest unfinished unit
// therefore has its inputs complete and is being processed.
// dy rows go to the TREE-order accumulator yacc (L2-resident) by fp64 REDs; not bitwise
// reproducible (the order of the y accumulations varies between runs).
#pragma once
#include "pipe.cuh"

namespace h2d {
namespace {

constexpr int kPSlotDbl = 4096;             // ring slot: 32 KB (factor block + x segments)
constexpr int kPSlots = 5;                  // slots per CTA (160 KB: a near-field CTA co-resides)
constexpr int kPCons = 5;                   // consumer warps (<= kPSlots: the end markers)
constexpr int kPBatch = 16;                 // units per queue grab
constexpr int kPThreads = 32 * (kPCons + 1);
constexpr int kPMaxR = 128;                 // widest pair (rank)

enum { kPWhole = 0, kPPhase1 = 1, kPPhase2 = 2, kPPhase3 = 3, kPEnd = 4 };
#ifndef H2D_PAIR_NORED
#define H2D_PAIR_NORED 0
#endif
constexpr bool kPNoRed = H2D_PAIR_NORED;   // build-time diagnostics switch (timing of the REDs)

// One ring unit: `bytes` of factors from the level's pair array at `off`, then the x
// segments of its rows (whole: V rows, U rows; phase 1 / 2 chunk: its rows; phase 3: none),
// each copied from the even row at or below its first row (16-byte aligned).
struct PUnit {
  int64_t off;
  int32_t bytes, kind, level, r;
  int32_t ya, rows_a, lda;  // first block (whole: V; chunk: the chunk): TREE row, rows, ld
  int32_t yb, rows_b, ldb;  // whole: U
  int32_t big, nchunks;     // chunk: counter / flag index of the pair, chunks of the phase
  int32_t toff, pad;        // chunk: t1 / t2 offset of the pair
};
static_assert(sizeof(PUnit) == 64, "PUnit layout");

struct PairPtrs {
  const double* P[H2D_MAX_LEVELS + 1];
};

struct PairSmem {
  double slot[kPSlots][kPSlotDbl];
  double ts[kPCons][2][kPMaxR];      // per consumer warp: t1 / t2 of its unit
  PUnit meta[kPSlots];
  PUnit batch[kPBatch];
  uint64_t full[kPSlots], empty[kPSlots];
  int next;
};

__host__ __device__ __forceinline__ int pair_xseg(int y, int rows) {   // doubles copied
  return ((y & 1) + rows + 1) & ~1;
}

__device__ __forceinline__ int ld_acquire(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int32_t* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void pair_red(double* p, double v) {
  if (kPNoRed) *p = v;   // diagnostics only (WRONG results)
  else atomicAdd(p, v);
}

// Column sums of a column-major block F (ld, rows, columns [0, r)) against x[0, rows), in
// blocks of 8 columns (transposed butterfly, pipe.cuh).  The sum of column c ends up in
// lane 4 (c & 7) for its block; emit(c, value) is called by that lane.
template <class Emit>
__device__ __forceinline__ void pair_colsums(const double* F, int ld, int rows, int r, const double* x, Emit emit) {
  const int lane = threadIdx.x & 31;
  for (int c0 = 0; c0 < r; c0 += 8) {
    double acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.0;
    const double* Fc = F + (int64_t)c0 * ld;
    const int nc = min(8, r - c0);
#pragma unroll 2
    for (int i = lane; i < rows; i += 32) {
      const double xi = x[i];
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q < nc) acc[q] = fma(Fc[q * ld + i], xi, acc[q]);
    }
    const double s = warp_transpose_sum8(acc, lane);
    const int c = c0 + (lane >> 2);
    if ((lane & 3) == 0 && c < r) emit(c, s);
  }
}

// Row dots dy[i] = sum_q F[i, q] t[q] (t in shared memory), one RED per row.
__device__ __forceinline__ void pair_rowdots(const double* F, int ld, int rows, int r, const double* t,
                                             double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < rows; i += 32) {
    double d0 = 0.0, d1 = 0.0;
    int q = 0;
    for (; q + 1 < r; q += 2) {
      d0 = fma(F[q * ld + i], t[q], d0);
      d1 = fma(F[(q + 1) * ld + i], t[q + 1], d1);
    }
    if (q < r) d0 = fma(F[q * ld + i], t[q], d0);
    pair_red(y + i, d0 + d1);
  }
}

// Phase 2 of a narrow pair (r <= 8) in one pass: column sums against x and row dots with t.
template <class Emit>
__device__ __forceinline__ void pair_colsum_rowdot8(const double* F, int ld, int rows, int r,
                                                    const double* x, const double* t,
                                                    double* __restrict__ y, Emit emit) {
  const int lane = threadIdx.x & 31;
  double acc[8], tq[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    acc[q] = 0.0;
    tq[q] = q < r ? t[q] : 0.0;
  }
#pragma unroll 2
  for (int i = lane; i < rows; i += 32) {
    const double xi = x[i];
    double d0 = 0.0, d1 = 0.0;
#pragma unroll
    for (int q = 0; q < 8; q += 2) {
      if (q < r) {
        const double f = F[q * ld + i];
        acc[q] = fma(f, xi, acc[q]);
        d0 = fma(f, tq[q], d0);
      }
      if (q + 1 < r) {
        const double f = F[(q + 1) * ld + i];
        acc[q + 1] = fma(f, xi, acc[q + 1]);
        d1 = fma(f, tq[q + 1], d1);
      }
    }
    pair_red(y + i, d0 + d1);
  }
  const double s = warp_transpose_sum8(acc, lane);
  const int c = lane >> 2;
  if ((lane & 3) == 0 && c < r) emit(c, s);
}

__device__ __forceinline__ void pair_wait_flag(const int32_t* f, int epoch) {
  if ((threadIdx.x & 31) == 0)
    while (ld_acquire(f) < epoch) __nanosleep(64);
  __syncwarp();
  __threadfence();
}

// A chunk of phase 1 / 2 has added its column sums: count it; the last chunk publishes.
__device__ __forceinline__ void pair_chunk_done(int32_t* cnt, int32_t* flag, int nchunks, int epoch) {
  __threadfence();
  __syncwarp();
  if ((threadIdx.x & 31) == 0 && atomicAdd(cnt, 1) == nchunks - 1) {
    *cnt = 0;   // (the next matvec's chunks start after this kernel)
    __threadfence();
    st_release(flag, epoch);
  }
}

__global__ void __launch_bounds__(kPThreads, 1)
pair_apply_kernel(const PUnit* __restrict__ units, int n_units, int32_t* counter, PairPtrs pp,
                  const double* __restrict__ x, double* __restrict__ yacc, double* __restrict__ tP1,
                  double* __restrict__ tP2, int32_t* __restrict__ pcount, int32_t* __restrict__ flags, int epoch) {
  extern __shared__ __align__(128) unsigned char pair_smem_raw[];
  PairSmem& S = *reinterpret_cast<PairSmem*>(pair_smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kPSlots; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.empty[s], 1);
    }
    S.next = 0;
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == 0) {   // producer
    const uint64_t pol = l2_evict_first_policy();
    int k = 0, ends = 0;
    int base = 0;
    if (lane == 0) base = atomicAdd(counter, kPBatch);
    base = __shfl_sync(0xffffffffu, base, 0);
    PUnit cur;
    if (base + lane < n_units && lane < kPBatch) cur = units[base + lane];
    for (;;) {
      const int cnt = max(0, min(kPBatch, n_units - base));
      if (lane < cnt) S.batch[lane] = cur;
      int nbase = 0;
      if (lane == 0 && cnt > 0) nbase = atomicAdd(counter, kPBatch);   // (used after this batch)
      __syncwarp();
      if (lane == 0) {
        for (int j = 0; j < cnt; ++j, ++k) {
          const int s = k % kPSlots;
          if (k >= kPSlots) mbar_wait(&S.empty[s], ((k / kPSlots) - 1) & 1);
          const PUnit u = S.batch[j];
          S.meta[s] = u;
          const int xa = u.kind == kPPhase3 ? 0 : pair_xseg(u.ya, u.rows_a);
          const int xb = u.kind == kPWhole ? pair_xseg(u.yb, u.rows_b) : 0;
          mbar_arrive_expect_tx(&S.full[s], (uint32_t)(u.bytes + 8 * (xa + xb)));
          double* dst = S.slot[s];
          if (u.kind == kPPhase1) bulk_g2s_keep(dst, pp.P[u.level] + u.off, (uint32_t)u.bytes, &S.full[s]);
          else bulk_g2s(dst, pp.P[u.level] + u.off, (uint32_t)u.bytes, &S.full[s], pol);
          dst += u.bytes / 8;
          if (xa) bulk_g2s_keep(dst, x + (u.ya & ~1), 8u * xa, &S.full[s]);
          if (xb) bulk_g2s_keep(dst + xa, x + (u.yb & ~1), 8u * xb, &S.full[s]);
        }
        if (cnt == 0) {   // queue exhausted: one end marker per consumer warp
          for (; ends < kPCons; ++ends, ++k) {
            const int s = k % kPSlots;
            if (k >= kPSlots) mbar_wait(&S.empty[s], ((k / kPSlots) - 1) & 1);
            S.meta[s].kind = kPEnd;
            mbar_arrive(&S.full[s]);
          }
        }
      }
      if (cnt == 0) break;
      __syncwarp();
      base = __shfl_sync(0xffffffffu, nbase, 0);
      if (base + lane < n_units && lane < kPBatch) cur = units[base + lane];
    }
    return;
  }
  const int cw = warp - 1;
  double* ts1 = S.ts[cw][0];
  double* ts2 = S.ts[cw][1];
  for (;;) {
    int k = 0;
    if (lane == 0) k = atomicAdd(&S.next, 1);
    k = __shfl_sync(0xffffffffu, k, 0);
    const int s = k % kPSlots;
    mbar_wait(&S.full[s], (k / kPSlots) & 1);
    const PUnit u = S.meta[s];
    if (u.kind == kPEnd) break;
    const double* F = S.slot[s];
    const int r = u.r;
    const double* xa = F + u.bytes / 8 + (u.ya & 1);                      // x of the first block's rows
    const double* xb = F + u.bytes / 8 + pair_xseg(u.ya, u.rows_a) + (u.yb & 1);   // whole: x of U's rows
    auto release = [&]() {
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.empty[s]);
    };
    if (u.kind == kPWhole) {
      const double* V = F;
      const double* U = F + (int64_t)u.lda * r;
      pair_colsums(V, u.lda, u.rows_a, r, xa, [&](int c, double v) { ts1[c] = v; });
      __syncwarp();
      if (r <= 8) {
        pair_colsum_rowdot8(U, u.ldb, u.rows_b, r, xb, ts1, yacc + u.yb, [&](int c, double v) { ts2[c] = v; });
      } else {
        pair_colsums(U, u.ldb, u.rows_b, r, xb, [&](int c, double v) { ts2[c] = v; });
        pair_rowdots(U, u.ldb, u.rows_b, r, ts1, yacc + u.yb);
      }
      __syncwarp();
      pair_rowdots(V, u.lda, u.rows_a, r, ts2, yacc + u.ya);
      release();
      continue;
    }
    if (u.kind == kPPhase1) {
      pair_colsums(F, u.lda, u.rows_a, r, xa, [&](int c, double v) { pair_red(tP1 + u.toff + c, v); });
      release();
      pair_chunk_done(pcount + 2 * u.big, flags + 2 * u.big, u.nchunks, epoch);
      continue;
    }
    // phases 2 / 3 need the other factor's column sums
    pair_wait_flag(flags + 2 * u.big + (u.kind - 2), epoch);
    const double* tg = (u.kind == kPPhase2 ? tP1 : tP2) + u.toff;
    for (int q = lane; q < r; q += 32) ts1[q] = __ldcg(tg + q);
    __syncwarp();
    if (u.kind == kPPhase2) {
      auto emit = [&](int c, double v) { pair_red(tP2 + u.toff + c, v); };
      if (r <= 8) {
        pair_colsum_rowdot8(F, u.lda, u.rows_a, r, xa, ts1, yacc + u.ya, emit);
      } else {
        pair_colsums(F, u.lda, u.rows_a, r, xa, emit);
        pair_rowdots(F, u.lda, u.rows_a, r, ts1, yacc + u.ya);
      }
      release();
      pair_chunk_done(pcount + 2 * u.big + 1, flags + 2 * u.big + 1, u.nchunks, epoch);
    } else {
      pair_rowdots(F, u.lda, u.rows_a, r, ts1, yacc + u.ya);
      release();
    }
  }
}

}  // namespace
}  // namespace h2d
