// Multi-RHS HODLR2D matvec (NEXT N2): Y = A X for a batch of vectors, every factor panel
// streamed once per chunk of NR <= 8 vectors (the paper applies its matvec to "ten
// different input vectors psi").  Same operator, same three stages as apply.cu; the
// low-rank stages do NR FMAs per factor element loaded and the near field NR FMAs per
// kernel evaluation, so the HBM-bound matvec becomes NR times more arithmetic-intense.
//
// Layouts (TREE order): x_m[s * NR + j] and t_m[q * NR + j], yfar_m[r * NR + j] interleave
// the vectors so a stage's vector data is one contiguous run; x_cols[j * N + s] and
// ynear_m[j * N + s] keep one vector per column for the near field.
//
// Stage A items are tiled to <= 2 * kCons columns so a consumer thread owns one column
// pair x NR accumulators; the near field is evaluated per leaf in both directions
// (row sums only: one writer per output row, no column reduction; twice the kernel
// evaluations of the symmetric single-vector kernel, amortised over NR vectors).
#include <algorithm>
#include <cstdlib>
#include <numeric>
#include <type_traits>

#include "pipe.cuh"

namespace h2d {
namespace {

constexpr int kTileW = 2 * kCons;    // stage-A column tile (<= kCons pairs)
constexpr int kMaxNR = 16;           // vectors per chunk (16: two 8-vector DMMA groups)
constexpr int kTileW16 = kCons;      // stage-A column tile for 16 vectors (<= 4 m-tiles per warp)
constexpr int kSymNR = 8;            // symmetric handles: 8-vector chunks
constexpr int kBRowsMax = 224;       // stage-B item rows (apply.cu kBRows)
constexpr int kNSMulti = 2, kSDMulti = 5632, kSVMulti = 704;   // ring: stages, doubles, vector values
constexpr int kSDMulti16 = 4096, kSVMulti16 = 1024;              // 16 vectors: 64 rows x 64 columns

// 16-vector records (x_m, t_m: 128 bytes each) are stored swizzled: vector v of the record
// at address A sits in slot v ^ 8 * ((A >> 7) & 1), i.e. the two 8-vector halves swap in
// every other record.  The DMMA B fragments read vector gq (and 8 + gq) of 4 consecutive
// records (lanes tq): unswizzled all 32 lanes hit 8 bank pairs (4-way conflicts, ncu r02x:
// 68 % of stage B's shared wavefronts were replays); swizzled each bank pair serves 2 lanes.
// Every writer and reader derives the swap from the record's own address (global) or from
// the parity of the stage's first record passed in the stage header (shared memory copies).
template <int NR>
__device__ __forceinline__ int rec_swz(const double* rec) {
  return NR == 16 ? (int)((reinterpret_cast<uintptr_t>(rec) >> 7) & 1) << 3 : 0;
}

// ---------------------------------------------------------------- stage A (multi)
// Stage header: a = W (tile width), b = Wp (row stride of the stage, W rounded up to even),
// c = out, d = ritem.
template <int NS, int NR, int SD, int SV>
__device__ void mA_producer(PipeSmem<NS, SD, SV>& S, const AItem* __restrict__ items, int n_items, int32_t* counter,
                            const LevelPtrs& lp, const double* __restrict__ xm) {
  const int lane = threadIdx.x & 31;
  const uint64_t pol = l2_evict_first_policy();
  int stage = 0;
  uint32_t phase = 0;
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
    idx = __shfl_sync(0xffffffffu, nidx, 0);
    if (!done && lane == 0) nidx = atomicAdd(counter, 1);
    if (!done && idx < n_items) nit = items[idx];
    const int Wp = (it.R + 1) & ~1;
    const bool contiguous = Wp == it.Rp;
    const int rows_s = done ? 1 : min(SV / NR, SD / max(Wp, 2));
    const double* V = done ? nullptr : lp.V[it.level] + it.v_off;
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
        h.b = Wp;
        h.c = it.out;
        h.d = it.ritem;
        h.f = done ? 0 : rec_swz<NR>(xm + (it.x_off + r0) * NR);
        const uint32_t bytes = (uint32_t)rows * (uint32_t)Wp * 8u, xbytes = (uint32_t)rows * NR * 8u;
        mbar_arrive_expect_tx(&S.full[stage], bytes + xbytes);
        if (bytes && contiguous) bulk_g2s(S.ring[stage], V + (int64_t)r0 * it.Rp, bytes, &S.full[stage], pol);
        // the rows' x records are contiguous (x_m[s][NR]): one bulk copy, not rows x NR
        // 8-byte cp.async from one producer warp (the producer was the stage's bottleneck)
        if (xbytes) bulk_g2s_keep(S.vec[stage], xm + (it.x_off + r0) * NR, xbytes, &S.full[stage]);
      }
      if (!contiguous)
        for (int r = lane; r < rows; r += 32)
          bulk_g2s(S.ring[stage] + r * Wp, V + (int64_t)(r0 + r) * it.Rp, (uint32_t)Wp * 8u, &S.full[stage], pol);
      cp_async_arrive_noinc(&S.full[stage]);
      if (++stage == NS) { stage = 0; phase ^= 1; }
      r0 += rows;
    } while (!done && r0 < it.nrows);
    if (done) break;
  }
}

template <int NS, int NR, int SD, int SV>
__device__ void mA_consumers(PipeSmem<NS, SD, SV>& S, const int32_t* __restrict__ vdst, double* __restrict__ tm,
                             double* __restrict__ tpartm, const RItem* __restrict__ ritems,
                             int32_t* __restrict__ rcount) {
  const int tid = threadIdx.x, lane = tid & 31;
  int stage = 0;
  uint32_t phase = 0;
  int W = 1, Wp = 2, P = 1, G = 1, g = 0, p = 0;
  double acc[2 * NR];
#pragma unroll
  for (int c = 0; c < 2 * NR; ++c) acc[c] = 0.0;
  for (;;) {
    mbar_wait(&S.full[stage], phase);
    const StageHdr h = S.hdr[stage];
    if (h.item < 0) break;
    if (h.flags & kFirst) {
      W = h.a;
      Wp = h.b;
      P = Wp >> 1;
      G = kCons / P;
      g = tid / P;
      p = tid - g * P;
#pragma unroll
      for (int c = 0; c < 2 * NR; ++c) acc[c] = 0.0;
    }
    if (g < G) {
      const double* __restrict__ v = S.ring[stage] + (size_t)g * Wp + 2 * p;
      const double* __restrict__ sx = S.vec[stage] + (size_t)g * NR;
      const int step = G * Wp;
      for (int j = g; j < h.cnt; j += G, v += step, sx += G * NR) {
        const double2 a = *reinterpret_cast<const double2*>(v);
#pragma unroll
        for (int k = 0; k < NR; k += 2) {
          const double2 xv = *reinterpret_cast<const double2*>(sx + k);
          acc[k] = fma(a.x, xv.x, acc[k]);
          acc[NR + k] = fma(a.y, xv.x, acc[NR + k]);
          if (k + 1 < NR) {
            acc[k + 1] = fma(a.x, xv.y, acc[k + 1]);
            acc[NR + k + 1] = fma(a.y, xv.y, acc[NR + k + 1]);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.empty[stage]);
    if (++stage == NS) { stage = 0; phase ^= 1; }
    if (!(h.flags & kLast)) continue;
    // ---- end of item: per vector, sum the G groups of each column pair
    auto put = [&](int q, int k, double v) {
      if (q >= W) return;
      if (h.c >= 0) tm[(int64_t)vdst[h.c + q] * NR + k] = v;
      else tpartm[((int64_t)(-h.c - 1) + q) * NR + k] = v;
    };
#pragma unroll
    for (int k = 0; k < NR; ++k) {
      if (G > 1) {
        S.red[2 * tid] = g < G ? acc[k] : 0.0;
        S.red[2 * tid + 1] = g < G ? acc[NR + k] : 0.0;
        named_bar_sync(1, kCons);
        if (tid < P) {
          double u0 = 0.0, u1 = 0.0;
          for (int gg = 0; gg < G; ++gg) {
            u0 += S.red[2 * (tid + gg * P)];
            u1 += S.red[2 * (tid + gg * P) + 1];
          }
          put(2 * tid, k, u0);
          put(2 * tid + 1, k, u1);
        }
        named_bar_sync(1, kCons);
      } else if (tid < P) {
        put(2 * tid, k, acc[k]);
        put(2 * tid + 1, k, acc[NR + k]);
      }
    }
    if (h.d >= 0) {
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
        for (int e = tid; e < ri.R * NR; e += kCons) {
          const int q = e / NR, k = e - q * NR;
          const double* __restrict__ pp = tpartm + ((int64_t)ri.p_off + q) * NR + k;
          const int64_t cs = (int64_t)ri.R * NR;
          double a0 = 0.0, a1 = 0.0;
          int c = 0;
          for (; c + 1 < ri.nchunks; c += 2) {
            a0 += __ldcg(pp + c * cs);
            a1 += __ldcg(pp + (c + 1) * cs);
          }
          if (c < ri.nchunks) a0 += __ldcg(pp + c * cs);
          double* rec = tm + (int64_t)vdst[ri.vpos + q] * NR;
          rec[k ^ rec_swz<NR>(rec)] = a0 + a1;
        }
        if (tid == 0) rcount[h.d] = 0;
      }
    }
  }
}

// ---------------------------------------------------------------- FP64 tensor cores (NR = 8)
// With 8 vectors both low-rank stages are small dense fp64 contractions, T = V^T X and
// Y = U T with N = 8 = the vector count, so they run on the FP64 tensor cores (DMMA,
// mma.sync m8n8k4 f64 — tcgen05 has no f64 kind): 256 FMAs per warp instruction instead of
// 32, which takes the consumers off the issue limit.  Fragments (PTX m8n8k4 .f64): lane t
// holds A[t/4][t%4], B[t%4][t/4] and D[t/4][2(t%4) + {0,1}].
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

constexpr int kConsWarps = kCons / 32;
constexpr int kMaxMTA = (kTileW / 8 + kConsWarps - 1) / kConsWarps;   // m-tiles per warp, stage A
constexpr int kMaxMTB = (kBRowsMax / 8 + kConsWarps - 1) / kConsWarps; // m-tiles per warp, stage B

// Column sums of one stage for the CNT m-tiles warp w owns (w + 7 i, i < CNT): M = panel
// columns, N = 8 vectors, K = rows (4 per DMMA).  Dispatched on the exact count so narrow
// panels (1-2 m-tiles per warp) do not issue the predicates of all kMaxMTA slots; whole
// k-steps run without bounds checks.
template <int CNT>
__device__ __forceinline__ void colsum_mtiles(double (&d)[kMaxMTA][2], const double* __restrict__ sv,
                                              const double* __restrict__ sx, int rows, int Wp, int w, int gq, int tq) {
  int cidx[CNT];
#pragma unroll
  for (int i = 0; i < CNT; ++i) cidx[i] = (w + kConsWarps * i) * 8 + gq;
  int k0 = 0;
  if constexpr (CNT <= 2) {   // few m-tiles: a second accumulator per m-tile (more DMMA chains in flight)
    double e[CNT][2];
#pragma unroll
    for (int i = 0; i < CNT; ++i) e[i][0] = e[i][1] = 0.0;
    for (; k0 + 8 <= rows; k0 += 8) {
      const int r = k0 + tq;
      const double b = sx[r * 8 + gq], b2 = sx[(r + 4) * 8 + gq];
#pragma unroll
      for (int i = 0; i < CNT; ++i) {
        dmma884(d[i][0], d[i][1], cidx[i] < Wp ? sv[r * Wp + cidx[i]] : 0.0, b);
        dmma884(e[i][0], e[i][1], cidx[i] < Wp ? sv[(r + 4) * Wp + cidx[i]] : 0.0, b2);
      }
    }
#pragma unroll
    for (int i = 0; i < CNT; ++i) {
      d[i][0] += e[i][0];
      d[i][1] += e[i][1];
    }
  }
  for (; k0 + 4 <= rows; k0 += 4) {
    const int r = k0 + tq;
    const double b = sx[r * 8 + gq];
#pragma unroll
    for (int i = 0; i < CNT; ++i) dmma884(d[i][0], d[i][1], cidx[i] < Wp ? sv[r * Wp + cidx[i]] : 0.0, b);
  }
  if (k0 < rows) {
    const int r = k0 + tq;
    const bool rv = r < rows;
    const double b = rv ? sx[r * 8 + gq] : 0.0;
#pragma unroll
    for (int i = 0; i < CNT; ++i) dmma884(d[i][0], d[i][1], (rv && cidx[i] < Wp) ? sv[r * Wp + cidx[i]] : 0.0, b);
  }
}

__device__ __forceinline__ void colsum_dispatch(double (&d)[kMaxMTA][2], const double* __restrict__ sv,
                                                const double* __restrict__ sx, int rows, int Wp, int MT, int w, int gq,
                                                int tq) {
  const int cnt = MT > w ? (MT - w + kConsWarps - 1) / kConsWarps : 0;
  switch (cnt) {
    case 0: break;
    case 1: colsum_mtiles<1>(d, sv, sx, rows, Wp, w, gq, tq); break;
    case 2: colsum_mtiles<2>(d, sv, sx, rows, Wp, w, gq, tq); break;
    case 3: colsum_mtiles<3>(d, sv, sx, rows, Wp, w, gq, tq); break;
    case 4: colsum_mtiles<4>(d, sv, sx, rows, Wp, w, gq, tq); break;
    case 5: colsum_mtiles<5>(d, sv, sx, rows, Wp, w, gq, tq); break;
    case 6: colsum_mtiles<6>(d, sv, sx, rows, Wp, w, gq, tq); break;
    case 7: colsum_mtiles<7>(d, sv, sx, rows, Wp, w, gq, tq); break;
    default: colsum_mtiles<kMaxMTA>(d, sv, sx, rows, Wp, w, gq, tq); break;
  }
}

// Stage A: M = tile columns (m-tile i of the item owned by warp i % 7, all rows), N = the 8
// vectors, K = rows, 4 per DMMA.  No cross-warp reduction: every T entry has one owner.
template <int NS, int SD, int SV>
__device__ void mA_consumers_dmma(PipeSmem<NS, SD, SV>& S, const int32_t* __restrict__ vdst, double* __restrict__ tm,
                                  double* __restrict__ tpartm, const RItem* __restrict__ ritems,
                                  int32_t* __restrict__ rcount) {
  constexpr int NR = 8;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  int stage = 0;
  uint32_t phase = 0;
  int W = 1, Wp = 2, MT = 1;
  double d[kMaxMTA][2];
#pragma unroll
  for (int i = 0; i < kMaxMTA; ++i) d[i][0] = d[i][1] = 0.0;
  for (;;) {
    mbar_wait(&S.full[stage], phase);
    const StageHdr h = S.hdr[stage];
    if (h.item < 0) break;
    if (h.flags & kFirst) {
      W = h.a;
      Wp = h.b;
      MT = (W + 7) >> 3;
#pragma unroll
      for (int i = 0; i < kMaxMTA; ++i) d[i][0] = d[i][1] = 0.0;
    }
    const double* __restrict__ sv = S.ring[stage];
    const double* __restrict__ sx = S.vec[stage];
    colsum_dispatch(d, sv, sx, h.cnt, Wp, MT, w, gq, tq);
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.empty[stage]);
    if (++stage == NS) { stage = 0; phase ^= 1; }
    if (!(h.flags & kLast)) continue;
#pragma unroll
    for (int i = 0; i < kMaxMTA; ++i) {
      const int mt = w + kConsWarps * i;
      const int q = mt * 8 + gq;
      if (mt < MT && q < W) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int k = 2 * tq + e;
          if (h.c >= 0) tm[(int64_t)vdst[h.c + q] * NR + k] = d[i][e];
          else tpartm[((int64_t)(-h.c - 1) + q) * NR + k] = d[i][e];
        }
      }
    }
    if (h.d >= 0) {
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
        for (int e = tid; e < ri.R * NR; e += kCons) {
          const int q = e / NR, k = e - q * NR;
          const double* __restrict__ pp = tpartm + ((int64_t)ri.p_off + q) * NR + k;
          const int64_t cs = (int64_t)ri.R * NR;
          double a0 = 0.0, a1 = 0.0;
          int c = 0;
          for (; c + 1 < ri.nchunks; c += 2) {
            a0 += __ldcg(pp + c * cs);
            a1 += __ldcg(pp + (c + 1) * cs);
          }
          if (c < ri.nchunks) a0 += __ldcg(pp + c * cs);
          double* rec = tm + (int64_t)vdst[ri.vpos + q] * NR;
          rec[k ^ rec_swz<NR>(rec)] = a0 + a1;
        }
        if (tid == 0) rcount[h.d] = 0;
      }
    }
  }
}

// Stage B: M = leaf rows, N = the 8 vectors, K = U columns.  Leaves of <= 64 rows (<= 8
// m-tiles, the configs' case) split K over the 7 warps (every warp all m-tiles, K steps
// 4w, 4w + 28, ...) and reduce the 7 partials per m-tile in smem at the end of the item;
// taller row blocks give m-tile i to warp i % 7.
constexpr int kMaxMTK = 12;
// Stage-B DMMA k-split for CNT m-tiles (the leaf's rows / 8): warp w takes k-steps 4 w,
// 4 w + 28, ... over all m-tiles; only the last m-tile can run past the leaf's rows.
template <int CNT, int KD>
__device__ __forceinline__ void bsplit_mtiles(double (&d)[KD][2], const double* __restrict__ su,
                                              const double* __restrict__ tv, int cols, int rowsp, int w, int gq,
                                              int tq) {
  const bool last_ok = (CNT - 1) * 8 + gq < rowsp;
  for (int k0 = 4 * w; k0 < cols; k0 += 4 * kConsWarps) {
    const int c = k0 + tq;
    const bool cv = c < cols;
    const double b = cv ? tv[c * 8 + gq] : 0.0;
    const double* __restrict__ col = su + c * rowsp + gq;
#pragma unroll
    for (int i = 0; i < CNT - 1; ++i) dmma884(d[i][0], d[i][1], cv ? col[i * 8] : 0.0, b);
    dmma884(d[CNT - 1][0], d[CNT - 1][1], (cv && last_ok) ? col[(CNT - 1) * 8] : 0.0, b);
  }
}

template <int NS, int SD, int SV>
__device__ void mB_consumers_dmma(PipeSmem<NS, SD, SV>& S, double* __restrict__ yfarm) {
  constexpr int NR = 8;
  constexpr int kD = kMaxMTK > kMaxMTB ? kMaxMTK : kMaxMTB;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  int stage = 0;
  uint32_t phase = 0;
  int rows = 1, rowsp = 2, MT = 1;
  bool ksplit = true;
  double d[kD][2];
#pragma unroll
  for (int i = 0; i < kD; ++i) d[i][0] = d[i][1] = 0.0;
  for (;;) {
    mbar_wait(&S.full[stage], phase);
    const StageHdr h = S.hdr[stage];
    if (h.item < 0) break;
    if (h.flags & kFirst) {
      rows = h.a;
      rowsp = h.b;
      MT = (rows + 7) >> 3;
      ksplit = MT <= kMaxMTK;
#pragma unroll
      for (int i = 0; i < kD; ++i) d[i][0] = d[i][1] = 0.0;
    }
    const double* __restrict__ su = S.ring[stage];
    const double* __restrict__ tv = S.vec[stage];
    const int cols = h.cnt;
    if (ksplit) {
      switch (MT) {   // exact m-tile count: no per-slot predicates
        case 1: bsplit_mtiles<1>(d, su, tv, cols, rowsp, w, gq, tq); break;
        case 2: bsplit_mtiles<2>(d, su, tv, cols, rowsp, w, gq, tq); break;
        case 3: bsplit_mtiles<3>(d, su, tv, cols, rowsp, w, gq, tq); break;
        case 4: bsplit_mtiles<4>(d, su, tv, cols, rowsp, w, gq, tq); break;
        case 5: bsplit_mtiles<5>(d, su, tv, cols, rowsp, w, gq, tq); break;
        case 6: bsplit_mtiles<6>(d, su, tv, cols, rowsp, w, gq, tq); break;
        case 7: bsplit_mtiles<7>(d, su, tv, cols, rowsp, w, gq, tq); break;
        case 8: bsplit_mtiles<8>(d, su, tv, cols, rowsp, w, gq, tq); break;
        case 9: bsplit_mtiles<9>(d, su, tv, cols, rowsp, w, gq, tq); break;
        case 10: bsplit_mtiles<10>(d, su, tv, cols, rowsp, w, gq, tq); break;
        case 11: bsplit_mtiles<11>(d, su, tv, cols, rowsp, w, gq, tq); break;
        default: bsplit_mtiles<kMaxMTK>(d, su, tv, cols, rowsp, w, gq, tq); break;
      }
    } else {
      for (int k0 = 0; k0 < cols; k0 += 4) {
        const int c = k0 + tq;
        const bool cv = c < cols;
        const double b = cv ? tv[c * NR + gq] : 0.0;
#pragma unroll
        for (int i = 0; i < kMaxMTB; ++i) {
          const int mt = w + kConsWarps * i;
          if (mt < MT) {
            const int r = mt * 8 + gq;
            const double a = (cv && r < rowsp) ? su[c * rowsp + r] : 0.0;
            dmma884(d[i][0], d[i][1], a, b);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.empty[stage]);
    if (++stage == NS) { stage = 0; phase ^= 1; }
    if (!(h.flags & kLast)) continue;
    if (ksplit) {
#pragma unroll
      for (int i = 0; i < kMaxMTK; ++i) {
        if (i < MT) {
          S.red[w * 64 + gq * 8 + 2 * tq] = d[i][0];
          S.red[w * 64 + gq * 8 + 2 * tq + 1] = d[i][1];
          named_bar_sync(1, kCons);
          if (tid < 64) {
            const int r = i * 8 + (tid >> 3);
            double u = 0.0;
#pragma unroll
            for (int ww = 0; ww < kConsWarps; ++ww) u += S.red[ww * 64 + tid];
            if (r < rows) yfarm[(int64_t)(h.c + r) * NR + (tid & 7)] = u;
          }
          named_bar_sync(1, kCons);
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < kMaxMTB; ++i) {
        const int mt = w + kConsWarps * i;
        const int r = mt * 8 + gq;
        if (mt < MT && r < rows) {
          double2* dst = reinterpret_cast<double2*>(yfarm + (int64_t)(h.c + r) * NR + 2 * tq);
          *dst = make_double2(d[i][0], d[i][1]);
        }
      }
    }
  }
}

// ---------------------------------------------------------------- 16 vectors per chunk
// Two 8-vector groups share every A fragment (factor values loaded once from smem, one DMMA
// per group).  Registers (80 at 3 CTAs/SM) bound the m-tiles a warp accumulates: stage-A
// tiles of <= kTileW16 columns (<= 4 m-tiles per warp), stage-B k-split up to 6 m-tiles.
constexpr int kMaxMTA16 = (kTileW16 / 8 + kConsWarps - 1) / kConsWarps;
constexpr int kMaxMTK16 = 6;   // (8: 80-register cap spills, 4.39 vs 3.32 ms)

template <int CNT>
__device__ __forceinline__ void colsum16_mtiles(double (&d)[kMaxMTA16][2][2], const double* __restrict__ sv,
                                                const double* __restrict__ sx, int rows, int Wp, int w, int gq,
                                                int tq, int swz0) {
  int cidx[CNT];
#pragma unroll
  for (int i = 0; i < CNT; ++i) cidx[i] = (w + kConsWarps * i) * 8 + gq;
  // record r's swap is swz0 ^ 8 (r & 1); r = k0 + tq with k0 a multiple of 4
  const int o0 = gq ^ swz0 ^ ((tq & 1) << 3);
  int k0 = 0;
  for (; k0 + 4 <= rows; k0 += 4) {
    const int r = k0 + tq;
    const double b0 = sx[r * 16 + o0], b1 = sx[r * 16 + (o0 ^ 8)];
#pragma unroll
    for (int i = 0; i < CNT; ++i) {
      const double a = cidx[i] < Wp ? sv[r * Wp + cidx[i]] : 0.0;
      dmma884(d[i][0][0], d[i][0][1], a, b0);
      dmma884(d[i][1][0], d[i][1][1], a, b1);
    }
  }
  if (k0 < rows) {
    const int r = k0 + tq;
    const bool rv = r < rows;
    const double b0 = rv ? sx[r * 16 + o0] : 0.0, b1 = rv ? sx[r * 16 + (o0 ^ 8)] : 0.0;
#pragma unroll
    for (int i = 0; i < CNT; ++i) {
      const double a = (rv && cidx[i] < Wp) ? sv[r * Wp + cidx[i]] : 0.0;
      dmma884(d[i][0][0], d[i][0][1], a, b0);
      dmma884(d[i][1][0], d[i][1][1], a, b1);
    }
  }
}

template <int NS, int SD, int SV>
__device__ void mA16_consumers(PipeSmem<NS, SD, SV>& S, const int32_t* __restrict__ vdst, double* __restrict__ tm,
                               double* __restrict__ tpartm, const RItem* __restrict__ ritems,
                               int32_t* __restrict__ rcount) {
  constexpr int NR = 16;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  int stage = 0;
  uint32_t phase = 0;
  int W = 1, Wp = 2, MT = 1;
  double d[kMaxMTA16][2][2];
#pragma unroll
  for (int i = 0; i < kMaxMTA16; ++i) d[i][0][0] = d[i][0][1] = d[i][1][0] = d[i][1][1] = 0.0;
  for (;;) {
    mbar_wait(&S.full[stage], phase);
    const StageHdr h = S.hdr[stage];
    if (h.item < 0) break;
    if (h.flags & kFirst) {
      W = h.a;
      Wp = h.b;
      MT = (W + 7) >> 3;
#pragma unroll
      for (int i = 0; i < kMaxMTA16; ++i) d[i][0][0] = d[i][0][1] = d[i][1][0] = d[i][1][1] = 0.0;
    }
    const double* __restrict__ sv = S.ring[stage];
    const double* __restrict__ sx = S.vec[stage];
    const int cnt = MT > w ? (MT - w + kConsWarps - 1) / kConsWarps : 0;
    switch (cnt) {
      case 0: break;
      case 1: colsum16_mtiles<1>(d, sv, sx, h.cnt, Wp, w, gq, tq, h.f); break;
      case 2: colsum16_mtiles<2>(d, sv, sx, h.cnt, Wp, w, gq, tq, h.f); break;
      case 3: colsum16_mtiles<3>(d, sv, sx, h.cnt, Wp, w, gq, tq, h.f); break;
      default: colsum16_mtiles<kMaxMTA16>(d, sv, sx, h.cnt, Wp, w, gq, tq, h.f); break;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.empty[stage]);
    if (++stage == NS) { stage = 0; phase ^= 1; }
    if (!(h.flags & kLast)) continue;
#pragma unroll
    for (int i = 0; i < kMaxMTA16; ++i) {
      const int mt = w + kConsWarps * i;
      const int q = mt * 8 + gq;
      if (mt < MT && q < W) {
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int k = 8 * g + 2 * tq + e;
            if (h.c >= 0) {
              double* rec = tm + (int64_t)vdst[h.c + q] * NR;
              rec[k ^ rec_swz<NR>(rec)] = d[i][g][e];
            } else {
              tpartm[((int64_t)(-h.c - 1) + q) * NR + k] = d[i][g][e];
            }
          }
      }
    }
    if (h.d >= 0) {
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
        for (int e = tid; e < ri.R * NR; e += kCons) {
          const int q = e / NR, k = e - q * NR;
          const double* __restrict__ pp = tpartm + ((int64_t)ri.p_off + q) * NR + k;
          const int64_t cs = (int64_t)ri.R * NR;
          double a0 = 0.0, a1 = 0.0;
          int c = 0;
          for (; c + 1 < ri.nchunks; c += 2) {
            a0 += __ldcg(pp + c * cs);
            a1 += __ldcg(pp + (c + 1) * cs);
          }
          if (c < ri.nchunks) a0 += __ldcg(pp + c * cs);
          double* rec = tm + (int64_t)vdst[ri.vpos + q] * NR;
          rec[k ^ rec_swz<NR>(rec)] = a0 + a1;
        }
        if (tid == 0) rcount[h.d] = 0;
      }
    }
  }
}

constexpr int kAcc16 = 4 * 6;   // flat accumulators of the 16-vector stage B (both mappings)
template <int CNT>
__device__ __forceinline__ void bsplit16_mtiles(double (&d)[kAcc16], const double* __restrict__ su,
                                                const double* __restrict__ tv, int cols, int rowsp, int w, int gq,
                                                int tq, int swz0) {
  const bool last_ok = (CNT - 1) * 8 + gq < rowsp;
  const int o0 = gq ^ swz0 ^ ((tq & 1) << 3);   // record c = k0 + tq, k0 a multiple of 4
  for (int k0 = 4 * w; k0 < cols; k0 += 4 * kConsWarps) {
    const int c = k0 + tq;
    const bool cv = c < cols;
    const double b0 = cv ? tv[c * 16 + o0] : 0.0, b1 = cv ? tv[c * 16 + (o0 ^ 8)] : 0.0;
    const double* __restrict__ col = su + c * rowsp + gq;
#pragma unroll
    for (int i = 0; i < CNT; ++i) {
      const double a = (cv && (i < CNT - 1 || last_ok)) ? col[i * 8] : 0.0;
      dmma884(d[4 * i], d[4 * i + 1], a, b0);
      dmma884(d[4 * i + 2], d[4 * i + 3], a, b1);
    }
  }
}

// Taller leaves (> 6 m-tiles): m-tile i of warp w is w + 7 i (both vector groups, one A
// load for two DMMAs), each warp over all k-steps of the stage, exact per-warp count.
template <int CNT>
__device__ __forceinline__ void bmt16(double (&d)[kAcc16], const double* __restrict__ su,
                                      const double* __restrict__ tv, int cols, int rowsp, int w, int gq, int tq,
                                      int swz0) {
  const int o0 = gq ^ swz0 ^ ((tq & 1) << 3);
  int roff[CNT];
  bool rok[CNT];
#pragma unroll
  for (int j = 0; j < CNT; ++j) {
    roff[j] = (w + kConsWarps * j) * 8 + gq;
    rok[j] = roff[j] < rowsp;
  }
  for (int k0 = 0; k0 < cols; k0 += 4) {
    const int c = k0 + tq;
    const bool cv = c < cols;
    const double b0 = cv ? tv[c * 16 + o0] : 0.0, b1 = cv ? tv[c * 16 + (o0 ^ 8)] : 0.0;
    const double* __restrict__ col = su + c * rowsp;
#pragma unroll
    for (int j = 0; j < CNT; ++j) {
      const double a = (cv && rok[j]) ? col[roff[j]] : 0.0;
      dmma884(d[4 * j], d[4 * j + 1], a, b0);
      dmma884(d[4 * j + 2], d[4 * j + 3], a, b1);
    }
  }
}

template <int NS, int SD, int SV>
__device__ void mB16_consumers(PipeSmem<NS, SD, SV>& S, double* __restrict__ yfarm) {
  constexpr int NR = 16;
  static_assert(4 * kMaxMTK16 <= kAcc16 && 4 * kMaxMTB <= kAcc16, "accumulator size");
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  int stage = 0;
  uint32_t phase = 0;
  int rows = 1, rowsp = 2, MT = 1;
  bool ksplit = true;
  double d[kAcc16];   // m-tile i, vector group g: d[4 i + 2 g + (0, 1)]
#pragma unroll
  for (int i = 0; i < kAcc16; ++i) d[i] = 0.0;
  for (;;) {
    mbar_wait(&S.full[stage], phase);
    const StageHdr h = S.hdr[stage];
    if (h.item < 0) break;
    if (h.flags & kFirst) {
      rows = h.a;
      rowsp = h.b;
      MT = (rows + 7) >> 3;
      ksplit = MT <= kMaxMTK16;
#pragma unroll
      for (int i = 0; i < kAcc16; ++i) d[i] = 0.0;
    }
    const double* __restrict__ su = S.ring[stage];
    const double* __restrict__ tv = S.vec[stage];
    const int cols = h.cnt;
    if (ksplit) {
      switch (MT) {
        case 1: bsplit16_mtiles<1>(d, su, tv, cols, rowsp, w, gq, tq, h.f); break;
        case 2: bsplit16_mtiles<2>(d, su, tv, cols, rowsp, w, gq, tq, h.f); break;
        case 3: bsplit16_mtiles<3>(d, su, tv, cols, rowsp, w, gq, tq, h.f); break;
        case 4: bsplit16_mtiles<4>(d, su, tv, cols, rowsp, w, gq, tq, h.f); break;
        case 5: bsplit16_mtiles<5>(d, su, tv, cols, rowsp, w, gq, tq, h.f); break;
        default: bsplit16_mtiles<kMaxMTK16>(d, su, tv, cols, rowsp, w, gq, tq, h.f); break;
      }
    } else {
      const int cnt = MT > w ? (MT - w + kConsWarps - 1) / kConsWarps : 0;
      switch (cnt) {
        case 0: break;
        case 1: bmt16<1>(d, su, tv, cols, rowsp, w, gq, tq, h.f); break;
        case 2: bmt16<2>(d, su, tv, cols, rowsp, w, gq, tq, h.f); break;
        case 3: bmt16<3>(d, su, tv, cols, rowsp, w, gq, tq, h.f); break;
        default: bmt16<kMaxMTB>(d, su, tv, cols, rowsp, w, gq, tq, h.f); break;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.empty[stage]);
    if (++stage == NS) { stage = 0; phase ^= 1; }
    if (!(h.flags & kLast)) continue;
    if (ksplit) {
#pragma unroll
      for (int i = 0; i < kMaxMTK16; ++i) {
        if (i < MT) {
#pragma unroll
          for (int g = 0; g < 2; ++g) {
            S.red[w * 64 + gq * 8 + 2 * tq] = d[4 * i + 2 * g];
            S.red[w * 64 + gq * 8 + 2 * tq + 1] = d[4 * i + 2 * g + 1];
            named_bar_sync(1, kCons);
            if (tid < 64) {
              const int r = i * 8 + (tid >> 3);
              double u = 0.0;
#pragma unroll
              for (int ww = 0; ww < kConsWarps; ++ww) u += S.red[ww * 64 + tid];
              if (r < rows) yfarm[(int64_t)(h.c + r) * NR + 8 * g + (tid & 7)] = u;
            }
            named_bar_sync(1, kCons);
          }
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < kMaxMTB; ++j) {
        const int mt = w + kConsWarps * j;
        const int r = mt * 8 + gq;
        if (mt < MT && r < rows) {
#pragma unroll
          for (int g = 0; g < 2; ++g) {
            double2* dst = reinterpret_cast<double2*>(yfarm + (int64_t)(h.c + r) * NR + 8 * g + 2 * tq);
            *dst = make_double2(d[4 * j + 2 * g], d[4 * j + 2 * g + 1]);
          }
        }
      }
    }
  }
}

template <int NR>
constexpr int kMultiMinBlocks = 3;

template <int NS, int NR, int SD, int SV>
__global__ void __launch_bounds__(kPipeThreads, kMultiMinBlocks<NR>)
stageA_multi_kernel(const AItem* __restrict__ items, int n_items, int32_t* counter, LevelPtrs lp,
                    const double* __restrict__ xm, const int32_t* __restrict__ vdst, double* __restrict__ tm,
                    double* __restrict__ tpartm, const RItem* __restrict__ ritems, int32_t* __restrict__ rcount) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  PipeSmem<NS, SD, SV>& S = *reinterpret_cast<PipeSmem<NS, SD, SV>*>(smem_raw);
  pipe_init(S);
  if (threadIdx.x >= kCons) mA_producer<NS, NR, SD, SV>(S, items, n_items, counter, lp, xm);
  else if constexpr (NR == 8) mA_consumers_dmma<NS, SD, SV>(S, vdst, tm, tpartm, ritems, rcount);
  else if constexpr (NR == 16) mA16_consumers<NS, SD, SV>(S, vdst, tm, tpartm, ritems, rcount);
  else mA_consumers<NS, NR, SD, SV>(S, vdst, tm, tpartm, ritems, rcount);
}

// ---------------------------------------------------------------- symmetric stage B' (multi)
// Eight vectors through the first-side U box panels of the symmetric apply (R23): the
// column sums T2 = U^T X (written through udst into the second-side t layout) and the row
// products Y1 = U T1 (per level, [kappa][n][8]) from one read of U.  Items are whole panels
// (R <= kTileW) in row chunks; a stage holds rows x Wp of U and, after them, the item's
// Wp x 8 T1 tile (one more bulk copy: T1 is contiguous per row box, 64-byte aligned).
// Stage header: a = R, b = Wp, c = out, d = ritem, pad = level, e = first TREE row.
template <int NS, int SD, int SV>
__device__ void mD_producer(PipeSmem<NS, SD, SV>& S, const AItem* __restrict__ items, int n_items, int32_t* counter,
                            const LevelPtrs& lp, const double* __restrict__ xm, const double* __restrict__ t1m) {
  constexpr int NR = 8;
  const int lane = threadIdx.x & 31;
  const uint64_t pol = l2_evict_first_policy();
  int stage = 0;
  uint32_t phase = 0;
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
    idx = __shfl_sync(0xffffffffu, nidx, 0);
    if (!done && lane == 0) nidx = atomicAdd(counter, 1);
    if (!done && idx < n_items) nit = items[idx];
    const int Wp = it.Rp;
    const int rows_s = done ? 1 : min(SV / NR, (SD - Wp * NR) / max(Wp, 2));
    const double* U = done ? nullptr : lp.Ub[it.level] + it.v_off;
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
        h.b = Wp;
        h.c = it.out;
        h.d = it.ritem;
        h.pad = it.level;
        h.e = (int32_t)(it.x_off + r0);
        const uint32_t ub = (uint32_t)rows * (uint32_t)Wp * 8u, tb = done ? 0u : (uint32_t)Wp * NR * 8u;
        const uint32_t xb = (uint32_t)rows * NR * 8u;
        mbar_arrive_expect_tx(&S.full[stage], ub + tb + xb);
        if (ub) bulk_g2s(S.ring[stage], U + (int64_t)r0 * Wp, ub, &S.full[stage], pol);
        if (tb) bulk_g2s(S.ring[stage] + rows * Wp, t1m + it.t1_off * NR, tb, &S.full[stage], pol);
        if (xb) bulk_g2s_keep(S.vec[stage], xm + (it.x_off + r0) * NR, xb, &S.full[stage]);   // x records
      }
      cp_async_arrive_noinc(&S.full[stage]);
      if (++stage == NS) { stage = 0; phase ^= 1; }
      r0 += rows;
    } while (!done && r0 < it.nrows);
    if (done) break;
  }
}

// Consumers: column sums as mA_consumers_dmma (M = panel columns, K = rows); row products
// M = the stage's rows (row m-tile i of warp w: w + 7 i), N = 8 vectors, K = columns, two
// accumulator chains per m-tile.
template <int NS, int SD, int SV>
__device__ void mD_consumers(PipeSmem<NS, SD, SV>& S, const int32_t* __restrict__ udst, double* __restrict__ t2m,
                             double* __restrict__ tpartm, const RItem* __restrict__ ritems,
                             int32_t* __restrict__ rcount, double* __restrict__ y1m, int64_t n) {
  constexpr int NR = 8;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  int stage = 0;
  uint32_t phase = 0;
  int W = 1, Wp = 2, MT = 1;
  double d[kMaxMTA][2];
#pragma unroll
  for (int i = 0; i < kMaxMTA; ++i) d[i][0] = d[i][1] = 0.0;
  for (;;) {
    mbar_wait(&S.full[stage], phase);
    const StageHdr h = S.hdr[stage];
    if (h.item < 0) break;
    if (h.flags & kFirst) {
      W = h.a;
      Wp = h.b;
      MT = (W + 7) >> 3;
#pragma unroll
      for (int i = 0; i < kMaxMTA; ++i) d[i][0] = d[i][1] = 0.0;
    }
    const double* __restrict__ sv = S.ring[stage];
    const double* __restrict__ sx = S.vec[stage];
    const int rows = h.cnt;
    const double* __restrict__ t1s = sv + rows * Wp;
    colsum_dispatch(d, sv, sx, rows, Wp, MT, w, gq, tq);   // column sums
    const int RT = (rows + 7) >> 3;   // row products
    for (int rt = w; rt < RT; rt += kConsWarps) {
      const int r = rt * 8 + gq;
      const bool rv = r < rows;
      const double* __restrict__ urow = sv + (rv ? r : 0) * Wp;   // rows past the stage read row 0, masked
      double e0 = 0.0, e1 = 0.0, f0 = 0.0, f1 = 0.0, g0 = 0.0, g1 = 0.0, q0 = 0.0, q1 = 0.0;
      int k0 = 0;
      for (; k0 + 16 <= Wp; k0 += 16) {   // four accumulator chains
        const int c = k0 + tq;
        dmma884(e0, e1, rv ? urow[c] : 0.0, t1s[c * NR + gq]);
        dmma884(f0, f1, rv ? urow[c + 4] : 0.0, t1s[(c + 4) * NR + gq]);
        dmma884(g0, g1, rv ? urow[c + 8] : 0.0, t1s[(c + 8) * NR + gq]);
        dmma884(q0, q1, rv ? urow[c + 12] : 0.0, t1s[(c + 12) * NR + gq]);
      }
      e0 += g0;
      e1 += g1;
      f0 += q0;
      f1 += q1;
      for (; k0 + 8 <= Wp; k0 += 8) {
        const int c = k0 + tq;
        dmma884(e0, e1, rv ? urow[c] : 0.0, t1s[c * NR + gq]);
        dmma884(f0, f1, rv ? urow[c + 4] : 0.0, t1s[(c + 4) * NR + gq]);
      }
      for (; k0 < Wp; k0 += 4) {
        const int c = k0 + tq;
        dmma884(e0, e1, (rv && c < Wp) ? urow[c] : 0.0, c < Wp ? t1s[c * NR + gq] : 0.0);
      }
      if (rv) {
        double2* dst = reinterpret_cast<double2*>(y1m + ((int64_t)(h.pad - 1) * n + h.e + r) * NR + 2 * tq);
        *dst = make_double2(e0 + f0, e1 + f1);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.empty[stage]);
    if (++stage == NS) { stage = 0; phase ^= 1; }
    if (!(h.flags & kLast)) continue;
#pragma unroll
    for (int i = 0; i < kMaxMTA; ++i) {
      const int mt = w + kConsWarps * i;
      const int q = mt * 8 + gq;
      if (mt < MT && q < W) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int k = 2 * tq + e;
          if (h.c >= 0) t2m[(int64_t)udst[h.c + q] * NR + k] = d[i][e];
          else tpartm[((int64_t)(-h.c - 1) + q) * NR + k] = d[i][e];
        }
      }
    }
    if (h.d >= 0) {
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
        for (int e = tid; e < ri.R * NR; e += kCons) {
          const int q = e / NR, k = e - q * NR;
          const double* __restrict__ pp = tpartm + ((int64_t)ri.p_off + q) * NR + k;
          const int64_t cs = (int64_t)ri.R * NR;
          double a0 = 0.0, a1 = 0.0;
          int c = 0;
          for (; c + 1 < ri.nchunks; c += 2) {
            a0 += __ldcg(pp + c * cs);
            a1 += __ldcg(pp + (c + 1) * cs);
          }
          if (c < ri.nchunks) a0 += __ldcg(pp + c * cs);
          t2m[(int64_t)udst[ri.vpos + q] * NR + k] = a0 + a1;
        }
        if (tid == 0) rcount[h.d] = 0;
      }
    }
  }
}

template <int NS, int SD, int SV>
__global__ void __launch_bounds__(kPipeThreads, 3)
stageA_dual_multi_kernel(const AItem* __restrict__ items, int n_items, int32_t* counter, LevelPtrs lp,
                         const double* __restrict__ xm, const int32_t* __restrict__ udst, double* __restrict__ t2m,
                         double* __restrict__ tpartm, const RItem* __restrict__ ritems, int32_t* __restrict__ rcount,
                         const double* __restrict__ t1m, double* __restrict__ y1m, int64_t n) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  PipeSmem<NS, SD, SV>& S = *reinterpret_cast<PipeSmem<NS, SD, SV>*>(smem_raw);
  pipe_init(S);
  if (threadIdx.x >= kCons) mD_producer<NS, SD, SV>(S, items, n_items, counter, lp, xm, t1m);
  else mD_consumers<NS, SD, SV>(S, udst, t2m, tpartm, ritems, rcount, y1m, n);
}

// ---------------------------------------------------------------- stage B (multi)
template <int NS, int NR, int SD, int SV>
__device__ void mB_producer(PipeSmem<NS, SD, SV>& S, const BItem* __restrict__ items, const BLevel* __restrict__ blev,
                            int n_items, int32_t* counter, int kappa, const LevelPtrs& lp,
                            const double* const* __restrict__ tml) {
  const int lane = threadIdx.x & 31;
  const uint64_t pol = l2_evict_first_policy();
  int stage = 0;
  uint32_t phase = 0;
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
    const int R = done || lane >= kappa ? 0 : lv.R;
    const unsigned nz = __ballot_sync(0xffffffffu, R > 0);
    const int lastl = nz ? 32 - __clz(nz) : 0;
    if (done || nz == 0) {
      mbar_wait(&S.empty[stage], phase ^ 1);
      if (lane == 0) {
        StageHdr& h = S.hdr[stage];
        h.item = done ? -1 : cur;
        h.cnt = 0;
        h.flags = kFirst | kLast;
        h.a = it.rows;
        h.b = rowsp;
        h.c = it.yrow;
        mbar_arrive_expect_tx(&S.full[stage], 0);
      }
      cp_async_arrive_noinc(&S.full[stage]);
      if (++stage == NS) { stage = 0; phase ^= 1; }
      if (done) break;
      continue;
    }
    const int cols_s = min(SV / NR, SD / rowsp);
    bool first = true;
    for (int li = 0; li < lastl; ++li) {
      const int Rl = __shfl_sync(0xffffffffu, R, li);
      const int cbl = __shfl_sync(0xffffffffu, lv.tcol, li);
      const int64_t ubl = __shfl_sync(0xffffffffu, lv.uoff, li);
      if (Rl == 0) continue;
      const double* Ub = lp.U[li + 1] + ubl;
      const double* tb = tml[li + 1] + (int64_t)cbl * NR;
      for (int c0 = 0; c0 < Rl; c0 += cols_s) {
        const int cols = min(cols_s, Rl - c0);
        const bool last = li == lastl - 1 && c0 + cols >= Rl;
        mbar_wait(&S.empty[stage], phase ^ 1);
        if (lane == 0) {
          StageHdr& h = S.hdr[stage];
          h.item = cur;
          h.cnt = cols;
          h.flags = (first ? kFirst : 0) | (last ? kLast : 0);
          h.a = it.rows;
          h.b = rowsp;
          h.c = it.yrow;
          h.f = rec_swz<NR>(tb + (int64_t)c0 * NR);
          const uint32_t tbytes = (uint32_t)cols * NR * 8u;
          mbar_arrive_expect_tx(&S.full[stage], (uint32_t)cols * (uint32_t)rowsp * 8u + tbytes);
          if (whole)
            bulk_g2s(S.ring[stage], Ub + (int64_t)c0 * mLp, (uint32_t)cols * (uint32_t)mLp * 8u, &S.full[stage], pol);
          // the columns' t records are contiguous (t[index][NR]): one bulk copy
          bulk_g2s_keep(S.vec[stage], tb + (int64_t)c0 * NR, tbytes, &S.full[stage]);
        }
        if (!whole)
          for (int c = lane; c < cols; c += 32)
            bulk_g2s(S.ring[stage] + c * rowsp, Ub + (int64_t)(c0 + c) * mLp + it.r0, (uint32_t)rowsp * 8u,
                     &S.full[stage], pol);
        cp_async_arrive_noinc(&S.full[stage]);
        if (++stage == NS) { stage = 0; phase ^= 1; }
        first = false;
      }
    }
  }
}

template <int NS, int NR, int SD, int SV>
__device__ void mB_consumers(PipeSmem<NS, SD, SV>& S, double* __restrict__ yfarm) {
  const int tid = threadIdx.x, lane = tid & 31;
  int stage = 0;
  uint32_t phase = 0;
  int rows = 1, rowsp = 2, G = 1, g = 0, i = 0, RP = 1;
  double acc[2 * NR];
#pragma unroll
  for (int c = 0; c < 2 * NR; ++c) acc[c] = 0.0;
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
#pragma unroll
      for (int c = 0; c < 2 * NR; ++c) acc[c] = 0.0;
    }
    if (g < G) {
      const double* __restrict__ u = S.ring[stage] + (size_t)g * rowsp + 2 * i;
      const double* __restrict__ tv = S.vec[stage] + (size_t)g * NR;
      const int step = G * rowsp;
      for (int c = g; c < h.cnt; c += G, u += step, tv += G * NR) {
        const double2 a = *reinterpret_cast<const double2*>(u);
#pragma unroll
        for (int k = 0; k < NR; k += 2) {
          const double2 t2 = *reinterpret_cast<const double2*>(tv + k);
          acc[k] = fma(a.x, t2.x, acc[k]);
          acc[NR + k] = fma(a.y, t2.x, acc[NR + k]);
          if (k + 1 < NR) {
            acc[k + 1] = fma(a.x, t2.y, acc[k + 1]);
            acc[NR + k + 1] = fma(a.y, t2.y, acc[NR + k + 1]);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.empty[stage]);
    if (++stage == NS) { stage = 0; phase ^= 1; }
    if (!(h.flags & kLast)) continue;
#pragma unroll
    for (int k = 0; k < NR; ++k) {
      S.red[2 * tid] = g < G ? acc[k] : 0.0;
      S.red[2 * tid + 1] = g < G ? acc[NR + k] : 0.0;
      named_bar_sync(1, kCons);
      if (tid < rows) {
        const int ip = tid >> 1, e = tid & 1;
        double u = 0.0;
        for (int gg = 0; gg < G; ++gg) u += S.red[2 * (ip + gg * RP) + e];
        yfarm[(int64_t)(h.c + tid) * NR + k] = u;
      }
      named_bar_sync(1, kCons);
    }
  }
}

struct TmPtrs {
  const double* p[H2D_MAX_LEVELS + 1];
};

template <int NS, int NR, int SD, int SV>
__global__ void __launch_bounds__(kPipeThreads, kMultiMinBlocks<NR>)
stageB_multi_kernel(const BItem* __restrict__ items, const BLevel* __restrict__ blev, int n_items,
                    int32_t* counter, int kappa, LevelPtrs lp, TmPtrs tml, double* __restrict__ yfarm) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  PipeSmem<NS, SD, SV>& S = *reinterpret_cast<PipeSmem<NS, SD, SV>*>(smem_raw);
  pipe_init(S);
  if (threadIdx.x >= kCons) mB_producer<NS, NR, SD, SV>(S, items, blev, n_items, counter, kappa, lp, tml.p);
  else if constexpr (NR == 8) mB_consumers_dmma<NS, SD, SV>(S, yfarm);
  else if constexpr (NR == 16) mB16_consumers<NS, SD, SV>(S, yfarm);
  else mB_consumers<NS, NR, SD, SV>(S, yfarm);
}

// ---------------------------------------------------------------- near field (multi)
// One CTA per served leaf X; rows of X in blocks of <= 128, thread (g, i) = (tid / RB,
// tid % RB) owns row i and the tile columns g, g + G, ...; every column tile (<= 96
// points of {X} u E_X) is staged in smem with its NR x values; K(r) is evaluated once
// per (row, column) and applied to the NR vectors, whose values sit in the tile as one
// record per column (NR / 2 16-byte loads per evaluation; vector-major, NR 8-byte loads:
// 16 vectors at C3 1.71 -> 1.50 ms standalone).  ynear_m[row * NR + k] = sum_Y K x_Y.
// (A DMMA version, every A-fragment entry evaluated by its lane, measured slower:
// tools/scratch/p2p_multi_dmma.cuh.txt.)
constexpr int kMTile = 96, kMRows = 128;

template <int KID>
__device__ __forceinline__ double keval_m(const KernelParams& kp, const double2* tab, double px, double py,
                                          double qx, double qy) {
  if constexpr (kDistKernel<KID>) {
    const double dx = px - qx, dy = py - qy;
    return kfast<KID>(fma(dx, dx, dy * dy), tab, kp);
  }
  return kernel_eval_t<KID>(kp, px, py, qx, qy);
}

template <int KID, int NR>
__global__ void __launch_bounds__(256, 3)
p2p_multi_kernel(int kappa, int64_t leaf_begin, const int32_t* __restrict__ leaf_start,
                 const double* __restrict__ px, const double* __restrict__ py,
                 const double* __restrict__ xm, int64_t n, KernelParams kp, double* __restrict__ ynearm) {
  __shared__ double tpx[kMTile], tpy[kMTile];
  __shared__ __align__(16) double tx[kMTile][NR];   // the tile's x records, unswizzled
  __shared__ double red[256];
  __shared__ double2 tab[kHlogBins];
  const int tid = threadIdx.x;
  if (kNeedsLogTable<KID>) hlog_table<KID>(tab);
  const int64_t X = leaf_begin + blockIdx.x;
  const uint32_t cx = p2p_compact((uint32_t)X), cy = p2p_compact((uint32_t)X >> 1);
  const uint32_t side = 1u << kappa;
  int64_t nb[5];
  int nn = 0;
  nb[nn++] = X;
  if (cx + 1 < side) nb[nn++] = (int64_t)(p2p_spread(cx + 1) | (p2p_spread(cy) << 1));
  if (cy + 1 < side) nb[nn++] = (int64_t)(p2p_spread(cx) | (p2p_spread(cy + 1) << 1));
  if (cx > 0) nb[nn++] = (int64_t)(p2p_spread(cx - 1) | (p2p_spread(cy) << 1));
  if (cy > 0) nb[nn++] = (int64_t)(p2p_spread(cx) | (p2p_spread(cy - 1) << 1));
  const int64_t xs = leaf_start[X];
  const int m = leaf_start[X + 1] - (int)xs;
  for (int rb = 0; rb < m; rb += kMRows) {
    const int RB = min(kMRows, m - rb), G = 256 / RB;
    const int g = tid / RB, i = tid - g * RB;
    const bool act = g < G;
    const double rpx = act ? px[xs + rb + i] : 0.0, rpy = act ? py[xs + rb + i] : 0.0;
    double racc[NR];
#pragma unroll
    for (int k = 0; k < NR; ++k) racc[k] = 0.0;
    for (int a = 0; a < nn; ++a) {
      const int64_t ys = leaf_start[nb[a]];
      const int ny = leaf_start[nb[a] + 1] - (int)ys;
      for (int cb = 0; cb < ny; cb += kMTile) {
        const int nt = min(kMTile, ny - cb);
        __syncthreads();
        for (int e = tid; e < nt; e += 256) {
          tpx[e] = px[ys + cb + e];
          tpy[e] = py[ys + cb + e];
        }
        for (int q = tid; q < nt * NR; q += 256) {   // x records of the tile, coalesced
          const int e = q / NR;
          tx[e][(q - e * NR) ^ rec_swz<NR>(xm + (ys + cb + e) * NR)] = xm[(ys + cb) * NR + q];
        }
        __syncthreads();
        if (act) {
          int j = g;
          // a column's NR x values are one record: NR / 2 16-byte loads; two columns per step
          // below 16 vectors, one at 16 (two would spill at the 80-register cap)
          constexpr int CPS = NR >= 16 ? 1 : 2;
          for (; j + (CPS - 1) * G < nt; j += CPS * G) {
            double kv[CPS];
#pragma unroll
            for (int c = 0; c < CPS; ++c) kv[c] = keval_m<KID>(kp, tab, rpx, rpy, tpx[j + c * G], tpy[j + c * G]);
#pragma unroll
            for (int c = 0; c < CPS; ++c) {
              const double2* rc = reinterpret_cast<const double2*>(tx[j + c * G]);
#pragma unroll
              for (int k = 0; k < NR; k += 2) {
                const double2 v = rc[k >> 1];
                racc[k] = fma(kv[c], v.x, racc[k]);
                racc[k + 1] = fma(kv[c], v.y, racc[k + 1]);
              }
            }
          }
          if (CPS == 2 && j < nt) {
            const double k0v = keval_m<KID>(kp, tab, rpx, rpy, tpx[j], tpy[j]);
            const double2* r0 = reinterpret_cast<const double2*>(tx[j]);
#pragma unroll
            for (int k = 0; k < NR; k += 2) {
              const double2 v = r0[k >> 1];
              racc[k] = fma(k0v, v.x, racc[k]);
              racc[k + 1] = fma(k0v, v.y, racc[k + 1]);
            }
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < NR; ++k) {
      __syncthreads();
      red[tid] = act ? racc[k] : 0.0;
      __syncthreads();
      if (tid < RB) {
        double u = 0.0;
        for (int gg = 0; gg < G; ++gg) u += red[gg * RB + tid];
        ynearm[(xs + rb + tid) * NR + k] = u;
      }
    }
  }
}

// ---------------------------------------------------------------- stored near field (16 vectors)
// Alg. 1 l.5 computes the dense self and edge-sharer blocks of every leaf once, at
// build time; the single-vector path instead evaluates them on the fly (the evaluations hide
// under the factor streams, and storing them would add 2.7 GB of HBM reads per matvec at C3).
// With 16 vectors per call the evaluations no longer hide (~0.95 ms exposed beside the DMMA
// stage kernels, profiles/r02ae_multi16.md) while reading the stored blocks costs ~0.4 ms of
// HBM, so 16-vector chunks use the paper's stored blocks, built on the first such call when
// they fit in half the free device memory (C3: 2.9 GB; C3 16 vectors 5.40 -> 4.97 ms per call,
// the kernel alone 0.86 ms: latency-bound; 80 registers with four k-steps of both tiles' A
// loads in flight beat more warps at 64 / 48 registers and B prefetch at 122,
// profiles/r02ae_multi16.md).  Per served leaf X: the columns of
// {X} u E_X (order X, +x, +y, -x, -y, each segment padded to a multiple of 4 with zero
// columns), rows padded to mp = 8 ceil(m / 8) with zeros, column-major mp x ncolp.  The
// product Y_X = D_X X_near runs on DMMA: lane t loads its A-fragment entry D[8 i + t/4][4 k +
// t%4] straight from HBM (four 64-byte runs per warp load) and the B fragments from the x
// records (L1 / L2: a leaf's columns are shared by its m-tiles and neighbours).
__device__ __forceinline__ int nf_segments(int kappa, int64_t X, const int32_t* __restrict__ leaf_start,
                                           int64_t (&ys)[5], int (&ny)[5]) {
  const uint32_t cx = p2p_compact((uint32_t)X), cy = p2p_compact((uint32_t)X >> 1);
  const uint32_t side = 1u << kappa;
  int64_t nb[5];
  int nn = 0;
  nb[nn++] = X;
  if (cx + 1 < side) nb[nn++] = (int64_t)(p2p_spread(cx + 1) | (p2p_spread(cy) << 1));
  if (cy + 1 < side) nb[nn++] = (int64_t)(p2p_spread(cx) | (p2p_spread(cy + 1) << 1));
  if (cx > 0) nb[nn++] = (int64_t)(p2p_spread(cx - 1) | (p2p_spread(cy) << 1));
  if (cy > 0) nb[nn++] = (int64_t)(p2p_spread(cx) | (p2p_spread(cy - 1) << 1));
#pragma unroll
  for (int a = 0; a < 5; ++a) {
    ys[a] = a < nn ? leaf_start[nb[a]] : 0;
    ny[a] = a < nn ? leaf_start[nb[a] + 1] - (int)ys[a] : 0;
  }
  return nn;
}

template <int KID>
__global__ void __launch_bounds__(256) nf_fill_kernel(int kappa, int64_t leaf_begin, const int32_t* __restrict__ leaf_start,
                                                      const double* __restrict__ px, const double* __restrict__ py,
                                                      KernelParams kp, const int64_t* __restrict__ nf_off,
                                                      double* __restrict__ nf) {
  __shared__ double2 tab[kHlogBins];
  if (kNeedsLogTable<KID>) hlog_table<KID>(tab);
  __syncthreads();
  const int64_t X = leaf_begin + blockIdx.x;
  int64_t ys[5];
  int ny[5];
  nf_segments(kappa, X, leaf_start, ys, ny);
  const int64_t xs = ys[0];
  const int m = ny[0], mp = (m + 7) & ~7;
  double* __restrict__ D = nf + nf_off[blockIdx.x];
  int64_t cb = 0;
#pragma unroll 1
  for (int a = 0; a < 5; ++a) {
    const int nyp = (ny[a] + 3) & ~3;
    for (int64_t q = threadIdx.x; q < (int64_t)nyp * mp; q += blockDim.x) {
      const int c = (int)(q / mp), r = (int)(q - (int64_t)c * mp);
      double v = 0.0;
      if (c < ny[a] && r < m) v = keval_m<KID>(kp, tab, px[xs + r], py[xs + r], px[ys[a] + c], py[ys[a] + c]);
      D[(cb + c) * mp + r] = v;
    }
    cb += nyp;
  }
}

constexpr int kNfWarps = 4;

#ifndef H2D_NF_MINB
#define H2D_NF_MINB 6
#endif
__global__ void __launch_bounds__(32 * kNfWarps, H2D_NF_MINB)
p2p_stored_kernel(int kappa, int64_t leaf_begin, const int32_t* __restrict__ leaf_start,
                  const double* __restrict__ xm, const int64_t* __restrict__ nf_off,
                  const double* __restrict__ nf, double* __restrict__ ynearm) {
  constexpr int NR = 16;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, tr = lane >> 2, tc = lane & 3;
  const int64_t X = leaf_begin + blockIdx.x;
  int64_t ys[5];
  int ny[5];
  nf_segments(kappa, X, leaf_start, ys, ny);
  const int64_t xs = ys[0];
  const int m = ny[0], mp = (m + 7) & ~7, MT = mp >> 3;
  const double* __restrict__ D = nf + nf_off[blockIdx.x];
  // padded column starts of the segments: every k-step (4 columns) lies in one segment
  int cp1 = (ny[0] + 3) & ~3;
  const int cp2 = cp1 + ((ny[1] + 3) & ~3), cp3 = cp2 + ((ny[2] + 3) & ~3), cp4 = cp3 + ((ny[3] + 3) & ~3);
  const int nkt = (cp4 + ((ny[4] + 3) & ~3)) >> 2;
  // a warp takes m-tile pairs (2 p, 2 p + 1), p = w, w + 4, ...: the pair shares every B
  // fragment; the k-steps of all segments run as one loop, four per iteration, with the
  // next iteration's A loads (HBM) issued before this iteration's DMMAs
  for (int p = w; 2 * p < MT; p += kNfWarps) {
    const int mt0 = 2 * p;
    const bool two = mt0 + 1 < MT;
    double d[2][2][2] = {};   // [tile][vector group][pair]
    const double* __restrict__ D0 = D + 8 * mt0 + tr;
    const double* __restrict__ D1 = D0 + (two ? 8 : 0);   // (the first tile again when there is no second)
    auto bfrag = [&](int kk, double& b0, double& b1) {
      const int c = 4 * kk + tc;
      const int sa = (c >= cp1) + (c >= cp2) + (c >= cp3) + (c >= cp4);
      // selects, not ys[sa] / ny[sa]: a dynamic index would put the arrays in local memory
      const int base = sa == 0 ? 0 : sa == 1 ? cp1 : sa == 2 ? cp2 : sa == 3 ? cp3 : cp4;
      const int n = sa == 0 ? ny[0] : sa == 1 ? ny[1] : sa == 2 ? ny[2] : sa == 3 ? ny[3] : ny[4];
      const int64_t y0 = sa == 0 ? ys[0] : sa == 1 ? ys[1] : sa == 2 ? ys[2] : sa == 3 ? ys[3] : ys[4];
      const int loc = c - base;
      const double* rec = xm + (y0 + min(loc, n - 1)) * NR;
      const int sw = rec_swz<NR>(rec);
      b0 = loc < n ? rec[tr ^ sw] : 0.0;
      b1 = loc < n ? rec[(8 + tr) ^ sw] : 0.0;
    };
    double a0[4], a1[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t o = (int64_t)(4 * min(u, nkt - 1) + tc) * mp;
      a0[u] = __ldcs(D0 + o);
      a1[u] = __ldcs(D1 + o);
    }
    for (int k = 0; k < nkt; k += 4) {
      double b0[4], b1[4], n0[4], n1[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) bfrag(min(k + u, nkt - 1), b0[u], b1[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u) {   // next iteration's A (clamped to the leaf's last k-step)
        const int64_t o = (int64_t)(4 * min(k + 4 + u, nkt - 1) + tc) * mp;
        n0[u] = __ldcs(D0 + o);
        n1[u] = __ldcs(D1 + o);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (k + u < nkt) {
          dmma884(d[0][0][0], d[0][0][1], a0[u], b0[u]);
          dmma884(d[0][1][0], d[0][1][1], a0[u], b1[u]);
          dmma884(d[1][0][0], d[1][0][1], a1[u], b0[u]);
          dmma884(d[1][1][0], d[1][1][1], a1[u], b1[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a0[u] = n0[u];
        a1[u] = n1[u];
      }
    }
    // D fragment: lane t holds rows 8 mt + t/4, vectors 8 g + 2 (t%4) + {0, 1}
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int r = 8 * (mt0 + q) + tr;
      if ((q == 0 || two) && r < m) {
#pragma unroll
        for (int g = 0; g < 2; ++g)
          *reinterpret_cast<double2*>(ynearm + (xs + r) * NR + 8 * g + 2 * tc) = make_double2(d[q][g][0], d[q][g][1]);
      }
    }
  }
}

__global__ void invert_perm_kernel(const int32_t* __restrict__ perm, int64_t n, int32_t* __restrict__ iperm) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x)
    iperm[perm[s]] = (int32_t)s;
}

// x_m[s * NR + k] (one record of the NR values per TREE row s) from NR vectors of length
// xlen in the caller's order (ORIGINAL: s = iperm[o]; TREE: s = o), and back in combine.
// Both go through a shared-memory tile of 256 rows x NR values (row stride NR + 1): the
// vector-major side moves in coalesced 256-element runs, the record side in whole records
// (consecutive lanes on consecutive values of a record), so a warp access touches no more
// lines than it fills (thread-per-record versions: 32 partial lines per instruction,
// 0.155 / 0.227 ms for 16 vectors at C3).
constexpr int kPermTile = 256;

template <int NR>
__global__ void __launch_bounds__(256) permute_multi_kernel(const double* __restrict__ X, int64_t xlen,
                                                            const int32_t* __restrict__ iperm, int64_t n,
                                                            double* __restrict__ xm) {
  __shared__ double sm[kPermTile][NR + 1];
  const int tid = threadIdx.x;
  for (int64_t o0 = (int64_t)blockIdx.x * kPermTile; o0 < n; o0 += (int64_t)gridDim.x * kPermTile) {
    const int cnt = (int)min((int64_t)kPermTile, n - o0);
    __syncthreads();
    if (tid < cnt) {
#pragma unroll
      for (int k = 0; k < NR; ++k) sm[tid][k] = X[(int64_t)k * xlen + o0 + tid];
    }
    __syncthreads();
    for (int q = tid; q < cnt * NR; q += 256) {
      const int e = q / NR, k = q - e * NR;
      const int64_t sr = iperm ? (int64_t)iperm[o0 + e] : o0 + e;
      double* rec = xm + sr * NR;
      rec[k ^ rec_swz<NR>(rec)] = sm[e][k];
    }
  }
}

// Y[k * ylen + o] = yfar_m[r] + scale ynear_m[r] + shift x_m[r] (records of NR values per
// TREE row r).  ORIGINAL: output index o = q, r = iperm[q]; TREE: r = row_begin + q,
// o = r - y_row0.
template <int NR>
__global__ void __launch_bounds__(256) combine_multi_kernel(int64_t row_begin, int64_t rows,
                                                            const double* __restrict__ yfarm,
                                                            const double* __restrict__ ynearm, int64_t n,
                                                            const double* __restrict__ xm, double scale, double shift,
                                                            double* __restrict__ Y, int64_t ylen,
                                                            const int32_t* __restrict__ iperm, int order_out,
                                                            int64_t y_row0) {
  __shared__ double sm[kPermTile][NR + 1];
  const int tid = threadIdx.x;
  const bool orig = order_out == H2D_ORDER_ORIGINAL;
  for (int64_t q0 = (int64_t)blockIdx.x * kPermTile; q0 < rows; q0 += (int64_t)gridDim.x * kPermTile) {
    const int cnt = (int)min((int64_t)kPermTile, rows - q0);
    __syncthreads();
    for (int q = tid; q < cnt * NR; q += 256) {
      const int e = q / NR, k = q - e * NR;
      const int64_t r = orig ? (int64_t)iperm[q0 + e] : row_begin + q0 + e;
      const double* xr = xm + r * NR;
      sm[e][k] = yfarm[(r - row_begin) * NR + k] + fma(scale, ynearm[r * NR + k], shift * xr[k ^ rec_swz<NR>(xr)]);
    }
    __syncthreads();
    if (tid < cnt) {
      const int64_t o = orig ? q0 + tid : row_begin + q0 + tid - y_row0;
#pragma unroll
      for (int k = 0; k < NR; ++k) Y[(int64_t)k * ylen + o] = sm[tid][k];
    }
  }
}

// symmetric apply: + the kappa per-level row products Y1 of B' (8 vectors; records of 8)
__global__ void combine_multi_sym_kernel(int64_t rows, int kappa, const double* __restrict__ yfarm,
                                         const double* __restrict__ y1m, const double* __restrict__ ynearm, int64_t n,
                                         const double* __restrict__ xm, double scale, double shift,
                                         double* __restrict__ Y, int64_t ylen, const int32_t* __restrict__ iperm,
                                         int order_out, int64_t y_row0) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < rows; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = order_out == H2D_ORDER_ORIGINAL ? (int64_t)iperm[q] : q;
    const int64_t o = order_out == H2D_ORDER_ORIGINAL ? q : r - y_row0;
    double v[8];
    const double2* __restrict__ yf = reinterpret_cast<const double2*>(yfarm + r * 8);
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) {
      const double2 a = yf[k2];
      v[2 * k2] = a.x;
      v[2 * k2 + 1] = a.y;
    }
    for (int l = 0; l < kappa; ++l) {
      const double2* __restrict__ y1 = reinterpret_cast<const double2*>(y1m + ((int64_t)l * n + r) * 8);
#pragma unroll
      for (int k2 = 0; k2 < 4; ++k2) {
        const double2 a = __ldcs(y1 + k2);
        v[2 * k2] += a.x;
        v[2 * k2 + 1] += a.y;
      }
    }
    const double2* __restrict__ yn = reinterpret_cast<const double2*>(ynearm + r * 8);
    const double2* __restrict__ xr = reinterpret_cast<const double2*>(xm + r * 8);
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) {
      const double2 e = yn[k2], xv = xr[k2];
      Y[(int64_t)(2 * k2) * ylen + o] = v[2 * k2] + fma(scale, e.x, shift * xv.x);
      Y[(int64_t)(2 * k2 + 1) * ylen + o] = v[2 * k2 + 1] + fma(scale, e.y, shift * xv.y);
    }
  }
}

}  // namespace

// Tiled stage-A schedule for the multi-RHS kernels (columns in tiles of <= kTileW).
static void build_multi_schedule(Handle& h) {
  int64_t elems = 0;
  for (int l = 1; l <= h.kappa; ++l) {
    const Level& L = h.levels[(size_t)l];
    for (int64_t Y = 0; Y < L.nbox; ++Y)
      elems += (h.box_end(l, Y) - h.box_begin(l, Y)) * ((L.vR[(size_t)Y] + 1) & ~1);
  }
  const int64_t target = std::min<int64_t>(262144, std::max<int64_t>(16384, elems / (4 * (int64_t)h.persist_ctas)));
  cudaStream_t s = h.stream;
  // tiles of <= tile_w columns of every V box panel, row chunks of <= target elements (the
  // 8- and 16-vector chunks use different tile widths: register budget of the consumers)
  auto build_items = [&](int tile_w, AItem*& d_items, int64_t& n_items, RItem*& d_ritems, int32_t*& d_rcount,
                         double*& d_tpart) {
    std::vector<AItem> items;
    std::vector<RItem> ritems;
    int64_t p_len = 0;
    for (int l = 1; l <= h.kappa; ++l) {
      const Level& L = h.levels[(size_t)l];
      for (int64_t Y = 0; Y < L.nbox; ++Y) {
        const int R = L.vR[(size_t)Y], Rp = (R + 1) & ~1;
        const int64_t y0 = h.box_begin(l, Y), nY = h.box_end(l, Y) - y0;
        if (R == 0 || nY == 0) continue;
        const int32_t vp = (int32_t)L.t_off[(size_t)Y];
        for (int q0 = 0; q0 < R; q0 += tile_w) {
          const int Wt = std::min(tile_w, R - q0), Wp = (Wt + 1) & ~1;
          int64_t nch = std::max<int64_t>(1, (nY * Wp + target - 1) / target);
          nch = std::min<int64_t>(nY, nch);
          const int64_t rows = (nY + nch - 1) / nch;
          nch = (nY + rows - 1) / rows;
          const int64_t base = L.vpan_off[(size_t)Y] + q0;
          if (nch == 1) {
            items.push_back(AItem{base, y0, (int32_t)nY, Wt, vp + q0, l, -1, Rp});
          } else {
            if (p_len + nch * Wt > INT32_MAX / kMaxNR) throw Error{H2D_EINVAL, "multi partial buffer too large"};
            ritems.push_back(RItem{vp + q0, (int32_t)p_len, Wt, (int32_t)nch});
            for (int64_t c = 0; c < nch; ++c) {
              const int64_t r0 = c * rows, nr = std::min(rows, nY - r0);
              items.push_back(AItem{base + r0 * Rp, y0 + r0, (int32_t)nr, Wt, (int32_t)(-(p_len + c * Wt) - 1), l,
                                    (int32_t)(ritems.size() - 1), Rp});
            }
            p_len += nch * Wt;
          }
        }
      }
    }
    std::stable_sort(items.begin(), items.end(), [](const AItem& a, const AItem& b) {
      return (int64_t)a.nrows * a.R > (int64_t)b.nrows * b.R;
    });
    n_items = (int64_t)items.size();
    d_items = h.alloc<AItem>(items.size());
    d_ritems = h.alloc<RItem>(ritems.size());
    d_rcount = h.alloc<int32_t>(ritems.size());
    d_tpart = h.alloc<double>((size_t)std::max<int64_t>(1, p_len) * kMaxNR);
    H2D_CUDA(cudaMemsetAsync(d_rcount, 0, std::max<size_t>(1, ritems.size()) * 4, s));
    if (!items.empty())
      H2D_CUDA(cudaMemcpyAsync(d_items, items.data(), items.size() * sizeof(AItem), cudaMemcpyHostToDevice, s));
    if (!ritems.empty())
      H2D_CUDA(cudaMemcpyAsync(d_ritems, ritems.data(), ritems.size() * sizeof(RItem), cudaMemcpyHostToDevice, s));
  };
  build_items(kTileW, h.m_aitems, h.m_n_aitems, h.m_ritems, h.m_rcount, h.m_tpart);
  if (!h.symapply)
    build_items(kTileW16, h.m16_aitems, h.m16_n_aitems, h.m16_ritems, h.m16_rcount, h.m16_tpart);
  if (h.symapply) {
    // symmetric B' for 8 vectors: whole first-side U box panels (R <= kTileW, else the
    // symmetric handle keeps one vector at a time) in row chunks of <= target elements
    std::vector<AItem> bitems;
    std::vector<RItem> britems;
    int64_t bp_len = 0, upos = 0;
    bool ok = true;
    for (int l = 1; l <= h.kappa && ok; ++l) {
      const Level& L = h.levels[(size_t)l];
      for (int64_t X = 0; X < L.nbox; ++X) {
        const int R = L.ubR[(size_t)X], Rp = (R + 1) & ~1;
        if (R > kTileW) { ok = false; break; }
        const int64_t x0 = h.box_begin(l, X), nX = h.box_end(l, X) - x0;
        if (R > 0 && nX > 0) {
          const int64_t t1o = L.t1_base + L.t1base[(size_t)X];
          int64_t nch = std::max<int64_t>(1, (nX * Rp + target - 1) / target);
          nch = std::min<int64_t>(nX, nch);
          const int64_t rows = (nX + nch - 1) / nch;
          nch = (nX + rows - 1) / rows;
          if (nch == 1) {
            bitems.push_back(AItem{L.ub_off[(size_t)X], x0, (int32_t)nX, R, (int32_t)upos, l, -1, Rp, t1o});
          } else {
            if (bp_len + nch * R > INT32_MAX / kSymNR) throw Error{H2D_EINVAL, "multi partial buffer too large"};
            britems.push_back(RItem{(int32_t)upos, (int32_t)bp_len, R, (int32_t)nch});
            for (int64_t c = 0; c < nch; ++c) {
              const int64_t r0 = c * rows, nr = std::min(rows, nX - r0);
              bitems.push_back(AItem{L.ub_off[(size_t)X] + r0 * Rp, x0 + r0, (int32_t)nr, R,
                                     (int32_t)(-(bp_len + c * R) - 1), l, (int32_t)(britems.size() - 1), Rp, t1o});
            }
            bp_len += nch * R;
          }
        }
        upos += R;
      }
    }
    h.m_sym_ok = ok && h.row_begin == 0 && h.row_end == h.n;   // (multi-rank: one vector at a time)
    if (ok) {
      std::stable_sort(bitems.begin(), bitems.end(), [](const AItem& a, const AItem& b) {
        return (int64_t)a.nrows * a.R > (int64_t)b.nrows * b.R;
      });
      h.m_n_b1items = (int64_t)bitems.size();
      h.m_b1items = h.alloc<AItem>(bitems.size());
      h.m_b1ritems = h.alloc<RItem>(britems.size());
      h.m_b1rcount = h.alloc<int32_t>(britems.size());
      h.m_b1tpart = h.alloc<double>((size_t)std::max<int64_t>(1, bp_len) * kSymNR);
      h.m_t1 = h.alloc<double>((size_t)std::max<int64_t>(1, h.t1_len) * kSymNR + 16);   // + tile over-read
      h.m_y1 = h.alloc<double>((size_t)h.kappa * h.n * kSymNR);
      // rows without a first-side panel at a level are never written: zero once
      H2D_CUDA(cudaMemsetAsync(h.m_y1, 0, (size_t)h.kappa * h.n * kSymNR * sizeof(double), s));
      H2D_CUDA(cudaMemsetAsync(h.m_t1, 0, ((size_t)std::max<int64_t>(1, h.t1_len) * kSymNR + 16) * sizeof(double), s));
      H2D_CUDA(cudaMemsetAsync(h.m_b1rcount, 0, std::max<size_t>(1, britems.size()) * 4, s));
      if (!bitems.empty())
        H2D_CUDA(cudaMemcpyAsync(h.m_b1items, bitems.data(), bitems.size() * sizeof(AItem), cudaMemcpyHostToDevice, s));
      if (!britems.empty())
        H2D_CUDA(cudaMemcpyAsync(h.m_b1ritems, britems.data(), britems.size() * sizeof(RItem), cudaMemcpyHostToDevice,
                                 s));
    }
  }
  const int64_t served = h.row_end - h.row_begin;
  h.m_xm = h.alloc<double>((size_t)h.n * kMaxNR);
  h.m_iperm = h.alloc<int32_t>((size_t)h.n);   // original index -> TREE row (record permutes)
  invert_perm_kernel<<<(int)std::min<int64_t>((h.n + 255) / 256, 148 * 16), 256, 0, s>>>(h.d_perm, h.n, h.m_iperm);
  H2D_LAUNCH_CHECK();
  h.m_t = h.alloc<double>((size_t)std::max<int64_t>(1, h.t_len) * kMaxNR);
  h.m_yfar = h.alloc<double>((size_t)std::max<int64_t>(1, served) * kMaxNR);
  h.m_ynear = h.alloc<double>((size_t)h.n * kMaxNR);
  H2D_CUDA(cudaStreamSynchronize(s));
  h.multi_ready = true;
}

template <int NR, int NS, int SD, int SV>
static void set_multi_attrs() {
  static uint64_t seen = 0;   // per instantiation and device (attributes live in the device's context)
  once_per_device(seen, [] {
    const int smem = (int)sizeof(PipeSmem<NS, SD, SV>);
    H2D_CUDA(cudaFuncSetAttribute(stageA_multi_kernel<NS, NR, SD, SV>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    H2D_CUDA(cudaFuncSetAttribute(stageB_multi_kernel<NS, NR, SD, SV>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    H2D_CUDA(cudaFuncSetAttribute(stageA_multi_kernel<NS, NR, SD, SV>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  cudaSharedmemCarveoutMaxShared));
    H2D_CUDA(cudaFuncSetAttribute(stageB_multi_kernel<NS, NR, SD, SV>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  cudaSharedmemCarveoutMaxShared));
  });
}

template <int KID, int NR>
static void launch_p2p_multi(Handle& h, cudaStream_t a) {
  const int64_t nleaves = h.leaf_end - h.leaf_begin;
  if (nleaves <= 0) return;
  p2p_multi_kernel<KID, NR><<<(int)nleaves, 256, 0, a>>>(h.kappa, h.leaf_begin, h.d_leaf_start, h.d_px, h.d_py,
                                                         h.m_xm, h.n, h.kp, h.m_ynear);
  H2D_LAUNCH_CHECK();
}

// The stored near field of the served leaves (16-vector chunks): sizes from the host copy
// of leaf_start, one fill launch; skipped (on-the-fly kernel) when it would take more than
// half the free device memory.
static void build_stored_near(Handle& h) {
  const int64_t nl = h.leaf_end - h.leaf_begin;
  std::vector<int64_t> off((size_t)nl + 1, 0);
  const uint32_t side = 1u << h.kappa;
  auto spread = [](uint32_t v) {
    uint64_t x = v & 0xffffu;
    x = (x | (x << 8)) & 0x00ff00ffu;
    x = (x | (x << 4)) & 0x0f0f0f0fu;
    x = (x | (x << 2)) & 0x33333333u;
    x = (x | (x << 1)) & 0x55555555u;
    return x;
  };
  auto cnt = [&](uint64_t Y) { return (int64_t)h.leaf_start[(size_t)Y + 1] - h.leaf_start[(size_t)Y]; };
  for (int64_t i = 0; i < nl; ++i) {
    const uint64_t X = (uint64_t)(h.leaf_begin + i);
    uint32_t cx = 0, cy = 0;
    for (int b = 0; b < h.kappa; ++b) {
      cx |= (uint32_t)((X >> (2 * b)) & 1) << b;
      cy |= (uint32_t)((X >> (2 * b + 1)) & 1) << b;
    }
    int64_t ncolp = (cnt(X) + 3) & ~3LL;
    if (cx + 1 < side) ncolp += (cnt(spread(cx + 1) | (spread(cy) << 1)) + 3) & ~3LL;
    if (cy + 1 < side) ncolp += (cnt(spread(cx) | (spread(cy + 1) << 1)) + 3) & ~3LL;
    if (cx > 0) ncolp += (cnt(spread(cx - 1) | (spread(cy) << 1)) + 3) & ~3LL;
    if (cy > 0) ncolp += (cnt(spread(cx) | (spread(cy - 1) << 1)) + 3) & ~3LL;
    off[(size_t)i + 1] = off[(size_t)i] + ((cnt(X) + 7) & ~7LL) * ncolp;
  }
  size_t fr = 0, tot = 0;
  H2D_CUDA(cudaMemGetInfo(&fr, &tot));
  const int64_t values = off[(size_t)nl];
  if (nl <= 0 || (size_t)values * 8 > fr / 2) {
    h.nf_state = -1;
    return;
  }
  h.d_snf = h.alloc<double>((size_t)values);
  h.d_snf_off = h.alloc<int64_t>((size_t)nl + 1);
  h.nf_values = values;
  cudaStream_t s = h.stream;
  H2D_CUDA(cudaMemcpyAsync(h.d_snf_off, off.data(), off.size() * sizeof(int64_t), cudaMemcpyHostToDevice, s));
  auto fill = [&](auto kid) {
    constexpr int KID = decltype(kid)::value;
    nf_fill_kernel<KID><<<(int)nl, 256, 0, s>>>(h.kappa, h.leaf_begin, h.d_leaf_start, h.d_px, h.d_py, h.kp,
                                                h.d_snf_off, h.d_snf);
  };
  switch (h.kp.id) {
    case H2D_KERNEL_LOG:
      if (h.p2p_kid == kLogSafe) fill(std::integral_constant<int, kLogSafe>{});
      else fill(std::integral_constant<int, H2D_KERNEL_LOG>{});
      break;
    case H2D_KERNEL_IMQ: fill(std::integral_constant<int, H2D_KERNEL_IMQ>{}); break;
    case H2D_KERNEL_ONE_OVER_R: fill(std::integral_constant<int, H2D_KERNEL_ONE_OVER_R>{}); break;
    case H2D_KERNEL_RBF_PHI1: fill(std::integral_constant<int, H2D_KERNEL_RBF_PHI1>{}); break;
    case H2D_KERNEL_RBF_PHI2: fill(std::integral_constant<int, H2D_KERNEL_RBF_PHI2>{}); break;
    default: fill(std::integral_constant<int, H2D_KERNEL_TEST_LOWRANK>{}); break;
  }
  H2D_LAUNCH_CHECK();
  H2D_CUDA(cudaStreamSynchronize(s));
  h.nf_state = 1;
}

template <int NR, int NS, int SD, int SV>
static void multi_chunk(Handle& h, const double* dX, int64_t xlen, double* dY, int64_t ylen, int order) {
  set_multi_attrs<NR, NS, SD, SV>();
  if (NR == 16 && h.nf_enabled && h.nf_state == 0) build_stored_near(h);
  cudaStream_t s = h.stream, hi = h.hi_stream, a = h.aux_stream;
  const int grid = (int)std::min<int64_t>((h.n + 255) / 256, 148 * 16);
  permute_multi_kernel<NR><<<grid, 256, 0, s>>>(dX, xlen, order == H2D_ORDER_ORIGINAL ? h.m_iperm : nullptr, h.n,
                                            h.m_xm);
  H2D_LAUNCH_CHECK();
  H2D_CUDA(cudaEventRecord(h.ev_fork, s));
  H2D_CUDA(cudaStreamWaitEvent(hi, h.ev_fork, 0));
  H2D_CUDA(cudaStreamWaitEvent(a, h.ev_fork, 0));
  H2D_CUDA(cudaMemsetAsync(h.d_counters, 0, 2 * sizeof(int32_t), hi));
  const size_t smem = sizeof(PipeSmem<NS, SD, SV>);
  const bool w16 = NR == 16;   // 16 vectors: the narrower-tile schedule
  const int64_t n_ai = w16 ? h.m16_n_aitems : h.m_n_aitems;
  if (n_ai > 0) {
    stageA_multi_kernel<NS, NR, SD, SV><<<h.persist_ctas, kPipeThreads, smem, hi>>>(
        w16 ? h.m16_aitems : h.m_aitems, (int)n_ai, h.d_counters, h.lp, h.m_xm, h.d_vdst, h.m_t,
        w16 ? h.m16_tpart : h.m_tpart, w16 ? h.m16_ritems : h.m_ritems, w16 ? h.m16_rcount : h.m_rcount);
    H2D_LAUNCH_CHECK();
  }
  if (h.n_bitems > 0) {
    TmPtrs tml{};
    for (int l = 1; l <= h.kappa; ++l) tml.p[l] = h.m_t + h.levels[(size_t)l].tu_base * NR;
    stageB_multi_kernel<NS, NR, SD, SV><<<h.persist_ctas, kPipeThreads, smem, hi>>>(
        h.d_bitems, h.d_blev, (int)h.n_bitems, h.d_counters + 1, h.kappa, h.lp, tml, h.m_yfar);
    H2D_LAUNCH_CHECK();
  }
  H2D_CUDA(cudaEventRecord(h.ev_far, hi));
  if (NR == 16 && h.nf_state == 1 && h.nf_enabled) {
    p2p_stored_kernel<<<(int)(h.leaf_end - h.leaf_begin), 32 * kNfWarps, 0, a>>>(
        h.kappa, h.leaf_begin, h.d_leaf_start, h.m_xm, h.d_snf_off, h.d_snf, h.m_ynear);
    H2D_LAUNCH_CHECK();
  } else {
    switch (h.kp.id) {
      case H2D_KERNEL_LOG:
        if (h.p2p_kid == kLogSafe) launch_p2p_multi<kLogSafe, NR>(h, a);
        else if (h.multi_repl) launch_p2p_multi<kLogRepl, NR>(h, a);
        else launch_p2p_multi<H2D_KERNEL_LOG, NR>(h, a);
        break;
      case H2D_KERNEL_IMQ: launch_p2p_multi<H2D_KERNEL_IMQ, NR>(h, a); break;
      case H2D_KERNEL_ONE_OVER_R: launch_p2p_multi<H2D_KERNEL_ONE_OVER_R, NR>(h, a); break;
      case H2D_KERNEL_RBF_PHI1: launch_p2p_multi<H2D_KERNEL_RBF_PHI1, NR>(h, a); break;
      case H2D_KERNEL_RBF_PHI2: launch_p2p_multi<H2D_KERNEL_RBF_PHI2, NR>(h, a); break;
      default: launch_p2p_multi<H2D_KERNEL_TEST_LOWRANK, NR>(h, a); break;
    }
  }
  H2D_CUDA(cudaEventRecord(h.ev_join, a));
  H2D_CUDA(cudaStreamWaitEvent(s, h.ev_far, 0));
  H2D_CUDA(cudaStreamWaitEvent(s, h.ev_join, 0));
  const int64_t rows = h.row_end - h.row_begin;
  if (rows > 0) {
    const int blocks = (int)std::min<int64_t>((rows + 255) / 256, 148 * 8);
    combine_multi_kernel<NR><<<blocks, 256, 0, s>>>(h.row_begin, rows, h.m_yfar, h.m_ynear, h.n, h.m_xm,
                                                h.kp.scale, h.kp.shift, dY, ylen, h.m_iperm,
                                                order == H2D_ORDER_ORIGINAL ? H2D_ORDER_ORIGINAL : H2D_ORDER_TREE,
                                                h.row_begin);
    H2D_LAUNCH_CHECK();
  }
}

// Symmetric apply, 8 vectors: A' (stage A multi over the first-side V box panels -> T1),
// B' (T2 = U^T X and Y1 = U T1 over the first-side U box panels), C' (stage B multi over
// the second-side leaf panels with T2), P2P, combine with the kappa Y1 rows.
static void multi_chunk_sym(Handle& h, const double* dX, int64_t xlen, double* dY, int64_t ylen, int order) {
  constexpr int NR = 8;
  set_multi_attrs<NR, kNSMulti, kSDMulti, kSVMulti>();
  static uint64_t dual_seen = 0;
  const size_t smem = sizeof(PipeSmem<kNSMulti, kSDMulti, kSVMulti>);
  once_per_device(dual_seen, [&] {
    H2D_CUDA(cudaFuncSetAttribute(stageA_dual_multi_kernel<kNSMulti, kSDMulti, kSVMulti>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    H2D_CUDA(cudaFuncSetAttribute(stageA_dual_multi_kernel<kNSMulti, kSDMulti, kSVMulti>,
                                  cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared));
  });
  cudaStream_t s = h.stream, hi = h.hi_stream, a = h.aux_stream;
  const int grid = (int)std::min<int64_t>((h.n + 255) / 256, 148 * 16);
  permute_multi_kernel<NR><<<grid, 256, 0, s>>>(dX, xlen, order == H2D_ORDER_ORIGINAL ? h.m_iperm : nullptr, h.n,
                                            h.m_xm);
  H2D_LAUNCH_CHECK();
  H2D_CUDA(cudaEventRecord(h.ev_fork, s));
  H2D_CUDA(cudaStreamWaitEvent(hi, h.ev_fork, 0));
  H2D_CUDA(cudaStreamWaitEvent(a, h.ev_fork, 0));
  H2D_CUDA(cudaMemsetAsync(h.d_counters, 0, 4 * sizeof(int32_t), hi));
  if (h.m_n_aitems > 0) {
    stageA_multi_kernel<kNSMulti, NR, kSDMulti, kSVMulti><<<h.persist_ctas, kPipeThreads, smem, hi>>>(
        h.m_aitems, (int)h.m_n_aitems, h.d_counters, h.lp, h.m_xm, h.d_vdst, h.m_t1, h.m_tpart, h.m_ritems,
        h.m_rcount);
    H2D_LAUNCH_CHECK();
  }
  if (h.m_n_b1items > 0) {
    stageA_dual_multi_kernel<kNSMulti, kSDMulti, kSVMulti><<<h.persist_ctas, kPipeThreads, smem, hi>>>(
        h.m_b1items, (int)h.m_n_b1items, h.d_counters + 3, h.lp, h.m_xm, h.d_udst, h.m_t, h.m_b1tpart,
        h.m_b1ritems, h.m_b1rcount, h.m_t1, h.m_y1, h.n);
    H2D_LAUNCH_CHECK();
  }
  if (h.n_bitems > 0) {
    TmPtrs tml{};
    for (int l = 1; l <= h.kappa; ++l) tml.p[l] = h.m_t + h.levels[(size_t)l].tu_base * NR;
    stageB_multi_kernel<kNSMulti, NR, kSDMulti, kSVMulti><<<h.persist_ctas, kPipeThreads, smem, hi>>>(
        h.d_bitems, h.d_blev, (int)h.n_bitems, h.d_counters + 1, h.kappa, h.lp, tml, h.m_yfar);
    H2D_LAUNCH_CHECK();
  }
  H2D_CUDA(cudaEventRecord(h.ev_far, hi));
  switch (h.kp.id) {
    case H2D_KERNEL_LOG:
      if (h.p2p_kid == kLogSafe) launch_p2p_multi<kLogSafe, NR>(h, a);
      else if (h.multi_repl) launch_p2p_multi<kLogRepl, NR>(h, a);
      else launch_p2p_multi<H2D_KERNEL_LOG, NR>(h, a);
      break;
    case H2D_KERNEL_IMQ: launch_p2p_multi<H2D_KERNEL_IMQ, NR>(h, a); break;
    case H2D_KERNEL_ONE_OVER_R: launch_p2p_multi<H2D_KERNEL_ONE_OVER_R, NR>(h, a); break;
    case H2D_KERNEL_RBF_PHI1: launch_p2p_multi<H2D_KERNEL_RBF_PHI1, NR>(h, a); break;
    case H2D_KERNEL_RBF_PHI2: launch_p2p_multi<H2D_KERNEL_RBF_PHI2, NR>(h, a); break;
    default: launch_p2p_multi<H2D_KERNEL_TEST_LOWRANK, NR>(h, a); break;
  }
  H2D_CUDA(cudaEventRecord(h.ev_join, a));
  H2D_CUDA(cudaStreamWaitEvent(s, h.ev_far, 0));
  H2D_CUDA(cudaStreamWaitEvent(s, h.ev_join, 0));
  const int64_t rows = h.row_end - h.row_begin;   // symmetric apply: single-rank handles
  if (rows > 0) {
    const int blocks = (int)std::min<int64_t>((rows + 255) / 256, 148 * 8);
    combine_multi_sym_kernel<<<blocks, 256, 0, s>>>(rows, h.kappa, h.m_yfar, h.m_y1, h.m_ynear, h.n, h.m_xm,
                                                    h.kp.scale, h.kp.shift, dY, ylen, h.m_iperm,
                                                    order == H2D_ORDER_ORIGINAL ? H2D_ORDER_ORIGINAL : H2D_ORDER_TREE,
                                                    h.row_begin);
    H2D_LAUNCH_CHECK();
  }
}

// Y = A X for nrhs vectors (device pointers; vector k at X + k * xlen, Y + k * ylen).
void matvec_multi(Handle& h, const double* dX, double* dY, int nrhs, int order) {
  if (order != H2D_ORDER_ORIGINAL && order != H2D_ORDER_TREE)
    throw Error{H2D_EINVAL, "multi-RHS matvec supports ORIGINAL and TREE orders"};
  const bool part = h.row_begin != 0 || h.row_end != h.n;
  if (order == H2D_ORDER_ORIGINAL && part)
    throw Error{H2D_EINVAL, "ORIGINAL order needs a single-rank (full-range) handle"};
  if (h.symapply) {
    // the symmetric apply keeps no directed panels: chunks of 8 through A' / B' / C' multi
    // (when every first-side panel fits one tile), the rest one vector at a time
    if (!h.multi_ready) build_multi_schedule(h);
    const int64_t ylen1 = order == H2D_ORDER_ORIGINAL ? h.n : h.row_end - h.row_begin;
    int k0 = 0;
    if (h.m_sym_ok)
      for (; k0 + 8 <= nrhs; k0 += 8) multi_chunk_sym(h, dX + (int64_t)k0 * h.n, h.n, dY + (int64_t)k0 * ylen1, ylen1, order);
    for (int k = k0; k < nrhs; ++k) {
      const double* X = dX + (int64_t)k * h.n;
      double* Y = dY + (int64_t)k * ylen1;
      if (order == H2D_ORDER_ORIGINAL) {
        permute_in(h, X, h.d_xtree);
        matvec_tree(h, h.d_xtree, Y, H2D_ORDER_ORIGINAL, h.row_begin);
      } else {
        matvec_tree(h, X, Y, H2D_ORDER_TREE, h.row_begin);
      }
    }
    return;
  }
  if (!h.multi_ready) build_multi_schedule(h);
  const int64_t xlen = h.n;
  const int64_t ylen = order == H2D_ORDER_ORIGINAL ? h.n : h.row_end - h.row_begin;
  // ring geometry: 2 x 44 KB slots (+ 8 x 88 vector values each) -- the DMMA consumers are
  // issue- / chain-bound per stage, so fewer, larger stages amortise the per-stage overhead:
  // C3 8 vectors 4.43 -> 3.88 ms per call, 4 vectors +9 % (5 x 16 KB measured alongside)
  auto chunk = [&](auto nr, const double* X, double* Y) {
    constexpr int R = decltype(nr)::value;
    if constexpr (R == 16) multi_chunk<16, kNSMulti, kSDMulti16, kSVMulti16>(h, X, xlen, Y, ylen, order);
    else multi_chunk<R, kNSMulti, kSDMulti, kSVMulti>(h, X, xlen, Y, ylen, order);
  };
  int k0 = 0;
  while (k0 < nrhs) {
    const int left = nrhs - k0;
    const double* X = dX + (int64_t)k0 * xlen;
    double* Y = dY + (int64_t)k0 * ylen;
    if (left >= 16) { chunk(std::integral_constant<int, 16>{}, X, Y); k0 += 16; }
    else if (left >= 8) { chunk(std::integral_constant<int, 8>{}, X, Y); k0 += 8; }
    else if (left >= 4) { chunk(std::integral_constant<int, 4>{}, X, Y); k0 += 4; }
    else if (left >= 2) { chunk(std::integral_constant<int, 2>{}, X, Y); k0 += 2; }
    else {
      // one vector: the single-vector path (symmetric P2P)
      if (order == H2D_ORDER_ORIGINAL) {
        permute_in(h, X, h.d_xtree);
        matvec_tree(h, h.d_xtree, Y, H2D_ORDER_ORIGINAL, h.row_begin);
      } else {
        matvec_tree(h, X, Y, H2D_ORDER_TREE, h.row_begin);
      }
      k0 += 1;
    }
  }
}

}  // namespace h2d
