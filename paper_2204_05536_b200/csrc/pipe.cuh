// Device building blocks shared by the matvec kernels (apply.cu: one vector; multi.cu: a
// batch of vectors): the bulk-TMA pipeline layout of the streaming stages, the near-field
// kernel evaluation (0.5 log r^2 by table + polynomial, distance kernels K(r) from r^2) and
// the Morton bit helpers.  Product code only (shares nothing with oracle/).
#pragma once
#include "h2d_internal.cuh"
#include "tma.cuh"

namespace h2d {
namespace {

// ---------------------------------------------------------------- pipeline layout
// One producer warp (bulk TMA of the factor stream + 8-byte cp.async of the x / t values
// a stage needs) and 7 consumer warps per CTA, NS-deep ring of 16 KB stages.  With
// 2 CTAs per SM (grid = 2 x SMs, ~93 KB smem, <= 80 registers) a third CTA of the P2P
// kernel still fits on every SM, so the FP64-bound near field runs under the HBM stream.
constexpr int kNSShallow = 5, kNSDeep = 9;   // ring depth at 2 / 1 CTAs per SM
constexpr int kDefaultCtasPerSm = 2;
constexpr int kStageDbl = 2048;      // factor doubles per stage (16 KB)
constexpr int kStageVec = 256;       // x (stage A) / t (stage B) values per stage
constexpr int kCons = 224;           // consumer threads (7 warps: 8-warp CTAs spread evenly
                                     // over the 4 SM sub-partitions' register files)
constexpr int kPipeThreads = kCons + 32;

constexpr int kFirst = 1, kLast = 2;

struct StageHdr {
  int32_t item;    // work item index; < 0: no more work (terminator)
  int32_t cnt;     // rows (stage A) / columns (stage B) held by this stage
  int32_t flags;   // kFirst / kLast stage of the item
  int32_t a, b, c, d, pad;   // item fields for the consumers (see the producers)
  int32_t e, f;
};

template <int NS, int SD = kStageDbl, int SV = kStageVec>
struct PipeSmem {
  double ring[NS][SD];
  double vec[NS][SV];
  double red[2 * kCons];
  StageHdr hdr[NS];
  uint64_t full[NS];    // 1 producer arrival (+ tx bytes) + 32 cp.async arrivals
  uint64_t empty[NS];   // 8 consumer-warp arrivals
  int flag;
};

template <int NS, int SD, int SV>
__device__ __forceinline__ void pipe_init(PipeSmem<NS, SD, SV>& S) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&S.full[s], 1 + 32);
      mbar_init(&S.empty[s], kCons / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();
}

// Sum 8 per-lane values c[0..7] over the 32 lanes of a warp (a transposed butterfly: 9
// double shuffles instead of 8 x 5).  Lane 4 t + (0..3) ends up holding the sum of c[t];
// read it from lane 4 t.  Fixed order, deterministic.
__device__ __forceinline__ double warp_transpose_sum8(const double (&c)[8], int lane) {
  const bool b16 = lane & 16, b8 = lane & 8, b4 = lane & 4;
  double a[4];
#pragma unroll
  for (int k = 0; k < 4; ++k)
    a[k] = (b16 ? c[k + 4] : c[k]) + __shfl_xor_sync(0xffffffffu, b16 ? c[k] : c[k + 4], 16);
  double b[2];
#pragma unroll
  for (int k = 0; k < 2; ++k)
    b[k] = (b8 ? a[k + 2] : a[k]) + __shfl_xor_sync(0xffffffffu, b8 ? a[k] : a[k + 2], 8);
  double v = (b4 ? b[1] : b[0]) + __shfl_xor_sync(0xffffffffu, b4 ? b[0] : b[1], 4);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  return v;
}

constexpr int kSymTile = 96, kSymMaxB = kSymTile / 16;

// 0.5 log(r2) for r2 > 0: r2 = 2^e m, m in [1, 2); c_k = 1 + (k + 1/2)/512 is the
// centre of m's 1/512 bin (k = top 9 mantissa bits), tab[k] = (1/c_k, 0.5 log c_k);
// 0.5 log r2 = e ln2/2 + 0.5 log c_k + 0.5 log1p(f), f = m/c_k - 1, |f| <= 2^-10, with
// 0.5 log1p(f) = f p(f), p the degree-3 Taylor polynomial (truncation f^5/10 <= 9e-17).
// 7 DFMA in a chain of 6 (the 128-bin, degree-5 version: 9 / 8): the near field is bound by
// these dependent chains.  The coefficients are constant-bank operands.
// (Measured, not kept: an 8-byte table of -0.5 log r_k with r_k = rcp.approx(c_k) from the
// MUFU halves the shared-memory wavefronts of the random lookups but costs 5 instructions
// more per evaluation, and the near field turns issue-bound: 0.40 -> 0.42 ms on C3;
// tools/scratch/hlog_rcp_table.cuh.txt.)
// REPL (kLogNoSelRepl handles): 64 bins, each stored 8 times side by side (the same 8 KB);
// lane l reads copy l % 8, so the 8 lanes of a 128-bit shared-memory phase always hit 8
// distinct bank quads (no replays) at two more DFMAs (degree 5: |f| <= 2^-7, truncation
// f^7 / 14 <= 1.3e-16).  The 512-bin table's random lookups replay on bank conflicts, and
// on a regular grid (few distinct r^2 mantissas) far more than on random points: C4's near
// field 2.59 -> 1.34 ms alone, C3's 0.46 -> 0.49 (profiles/r02ai_logtable.md).
constexpr int kHlogBins = 512;       // table entries (bins, or 64 bins x 8 copies)
__constant__ double c_hlog[8] = {0.34657359027997264,   // ln2 / 2 (high part)
                                 1.1595234069231498e-17, // ln2 / 2 (low part)
                                 0.5, -0.25, 1.0 / 6.0, -0.125, 0.1, -1.0 / 12.0};

// SAFE: subnormal r2 (points closer than ~1.5e-154) are normalised in the integer pipe: the
// mantissa is shifted until its leading one is the implicit bit (sh = 0 for normal r2) and
// the exponent becomes 1 - sh - 1023.  r2 = 0 gives a finite value the callers replace by
// K(0) = 0 (R8).
// SAFE = false (the default near field): r2 must be normal or 0; the build checks the
// near field once and switches the handle to SAFE kernels (kLogSafe) if any pair of distinct
// points has a subnormal r2, so the common case pays no normalisation.
template <bool SAFE = false, bool REPL = false>
__device__ __forceinline__ double hlog_r2(double r2, const double2* __restrict__ tab) {
  static_assert(!(SAFE && REPL), "the subnormal-safe log uses the 512-bin table");
  if (!SAFE) {
    // the same arithmetic on the high word only (r2 >= 0, normal or 0): the table byte offset
    // 16 k = (hi >> 7) & 0x1ff0, the mantissa's high word (hi & 0xfffff) | 0x3ff00000, and
    // the biased exponent E = hi >> 20 dropped straight into the low word of 2^52 (three
    // integer instructions fewer per evaluation than the 64-bit shifts and the signed e)
    static_assert(kHlogBins == 512, "offset mask assumes 512 bins");
    const uint32_t hi = (uint32_t)__double2hiint(r2);
    // REPL: bin = top 6 mantissa bits, byte offset 128 bin + 16 (lane % 8) (the lane part is
    // loop-invariant and hoisted)
    const double2 tb = REPL ? *reinterpret_cast<const double2*>(reinterpret_cast<const char*>(tab + (threadIdx.x & 7)) +
                                                                ((hi >> 7) & 0x1f80u))
                            : *reinterpret_cast<const double2*>(reinterpret_cast<const char*>(tab) + ((hi >> 7) & 0x1ff0u));
    const double mnt = __hiloint2double((int)((hi & 0x000fffffu) | 0x3ff00000u), __double2loint(r2));
    const double f = fma(mnt, tb.x, -1.0);
    double p;
    if (REPL) {
      p = fma(f, c_hlog[7], c_hlog[6]);
      p = fma(f, p, c_hlog[5]);
      p = fma(f, p, c_hlog[4]);
    } else {
      p = fma(f, c_hlog[5], c_hlog[4]);
    }
    p = fma(f, p, c_hlog[3]);
    p = fma(f, p, c_hlog[2]);
    const double ed = __hiloint2double(0x43300000, (int)(hi >> 20)) - 4503599627371519.0;
    // ln2 / 2 without its lo part: |e| x 1.2e-17 absolute (e = -14 at C3's near-field
    // distances: 1.6e-16 on |0.5 log r2| ~ 5, below one ulp of the sums it enters), one DFMA
    // less per evaluation; the SAFE path keeps the hi + lo pair
    return fma(ed, c_hlog[0], fma(p, f, tb.y));
  }
  long long bits = __double_as_longlong(r2);
  const int E = (int)(bits >> 52);
  const int sh = max(0, __clzll(bits) - 11);
  bits <<= sh;
  const int e = (E == 0 ? 1 - sh : E) - 1023;
  const double mnt = __longlong_as_double((bits & 0x000FFFFFFFFFFFFFLL) | 0x3FF0000000000000LL);
  const int k = (int)(bits >> 43) & (kHlogBins - 1);
  const double2 tb = tab[k];
  const double f = fma(mnt, tb.x, -1.0);
  double p = fma(f, c_hlog[5], c_hlog[4]);
  p = fma(f, p, c_hlog[3]);
  p = fma(f, p, c_hlog[2]);
  const double ed = (double)e;
  return fma(ed, c_hlog[0], fma(p, f, fma(ed, c_hlog[1], tb.y)));
}

template <int KID>
__device__ __forceinline__ void hlog_table(double2* tab) {
  constexpr bool repl = KID == kLogNoSelRepl || KID == kLogRepl || KID == kPhi1Repl;
  for (int k = threadIdx.x; k < kHlogBins; k += blockDim.x) {
    const int b = repl ? k >> 3 : k;   // (replicated: entry k is copy k % 8 of bin k / 8)
    const double c = 1.0 + (b + 0.5) / (repl ? 64 : kHlogBins);
    tab[k] = make_double2(1.0 / c, 0.5 * log(c));
  }
}

// K(r) from r^2 with K(0) := K0 by a select (no branch; phi_1 / phi_2 branch only for
// the rare pairs closer than a); distance kernels only.
template <int KID>
__device__ __forceinline__ double kfast(double r2, const double2* __restrict__ tab, const KernelParams& kp) {
  if (KID == kLogNoSel || KID == kLogNoSelRepl) {   // no r2 = 0 select: the caller corrects the diagonal (warp kernel)
    return hlog_r2<false, KID == kLogNoSelRepl>(r2, tab);
  } else if (KID == H2D_KERNEL_LOG || KID == kLogSafe || KID == kLogRepl) {
    const double v = hlog_r2<KID == kLogSafe, KID == kLogRepl>(r2, tab);
    return r2 > 0.0 ? v : 0.0;
  } else if (KID == H2D_KERNEL_IMQ) {
    return rsqrt(fma(r2, kp.inv_c2, 1.0));
  } else if (KID == H2D_KERNEL_ONE_OVER_R) {
    const double v = rsqrt(r2);
    return r2 > 0.0 ? v : 0.0;
  } else if (KID == H2D_KERNEL_RBF_PHI1 || KID == kPhi1Repl) {
    double v = hlog_r2<false, KID == kPhi1Repl>(r2, tab) * kp.inv_log_a;   // log r / log a
    if (r2 < kp.a2) {
      const double r = sqrt(r2);
      v = r2 > 0.0 ? fma(r, log(r), -1.0) * kp.inv_phi1_den : 0.0;
    }
    return v;
  } else {   // H2D_KERNEL_RBF_PHI2
    const double v = kp.a * rsqrt(r2);
    return r2 >= kp.a2 ? v : sqrt(r2) / kp.a;
  }
}

template <int KID>
constexpr bool kDistKernel = KID == H2D_KERNEL_LOG || KID == kLogSafe || KID == kLogNoSel || KID == kLogNoSelRepl || KID == kLogRepl || KID == kPhi1Repl || KID == H2D_KERNEL_IMQ || KID == H2D_KERNEL_ONE_OVER_R ||
                             KID == H2D_KERNEL_RBF_PHI1 || KID == H2D_KERNEL_RBF_PHI2;
template <int KID>
constexpr bool kNeedsLogTable = KID == H2D_KERNEL_LOG || KID == kLogSafe || KID == kLogNoSel || KID == kLogNoSelRepl || KID == kLogRepl || KID == kPhi1Repl || KID == H2D_KERNEL_RBF_PHI1;

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

}  // namespace
}  // namespace h2d
