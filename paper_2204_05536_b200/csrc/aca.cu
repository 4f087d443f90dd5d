// Batched Adaptive Cross Approximation (S6) of every directed admissible block.
//
// The ACA variant is the reading R7 of DESIGN.md (the paper only cites ACA, P:42 / P:882):
// partial pivoting, first row pivot = local row 0; each step
//   (1) residual row R(i*,:) = A(i*,Y) - sum_q U[i*,q] V[:,q]
//   (2) j* = argmax |R(i*,:)| (ties -> smallest j)
//   (3) zero pivot -> mark i* used, next = smallest unused row; stop after 3 in a row
//   (4) v = R(i*,:)/R(i*,j*),  u = A(X,j*) - sum_q V[j*,q] U[:,q]
//   (5) ||S_k||_F^2 += 2 sum_q (u.U_q)(V_q.v) + ||u||^2 ||v||^2
//   (7) stop when ||u|| ||v|| <= tol ||S_k||_F held on `consecutive` steps (then drop the
//       `trim` streak terms) or k = min(m, n, max_rank)
//   (8) next row = argmax over unused rows of |u| (ties -> smallest)
//
// Two execution shapes, same arithmetic (only the summation order of reductions differs):
//  * small blocks (deep levels, thousands of blocks): one CTA per block, factors written
//    straight into a scratch slot (m x cap, n x cap, column-major);
//  * big blocks (top levels, few huge blocks): level-synchronous multi-CTA steps — every
//    phase of a step is one launch over (block, 4096-element chunk) items across all SMs.
#include <algorithm>
#include <chrono>
#include <climits>

#include "h2d_internal.cuh"

namespace h2d {
namespace {

constexpr int kSmallThreads = 256;
constexpr int kBigThreads = 256;
constexpr int kChunk = 4096;

struct AcaBlock {
  int64_t r0, c0;      // TREE offsets of the row / column boxes
  int32_t m, n, cap;   // sizes; cap = scratch columns
  int32_t pad;
  int64_t u_off, v_off, used_off;  // scratch offsets (doubles, doubles, bytes)
  int64_t p_off;       // big path: partial-buffer offset
  int32_t nchm, nchn;  // big path: chunk counts over m and n
};
struct AcaState {      // big path per-block state
  double S2, piv, nu2, nv2;
  int32_t k, istar, jstar, hits, zs, done, rank, trunc, skip, pad;
};
struct AcaParamsDev {
  double tol;
  int max_rank, consecutive, trim;
};
struct BigItem {
  int32_t blk, kind, start, len, chunk, pad;  // kind 0: rows (m), 1: columns (n)
};

__device__ __forceinline__ void argmax_merge(double& v, int& i, double v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
}

// Block-wide argmax (ties -> smallest index). red_v / red_i: >= 32 entries of smem.
__device__ void block_argmax(double& v, int& i, double* red_v, int* red_i) {
  for (int o = 16; o > 0; o >>= 1) {
    double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    int i2 = __shfl_xor_sync(0xffffffffu, i, o);
    argmax_merge(v, i, v2, i2);
  }
  int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) { red_v[w] = v; red_i[w] = i; }
  __syncthreads();
  if (w == 0) {
    v = lane < nw ? red_v[lane] : -1.0;
    i = lane < nw ? red_i[lane] : INT_MAX;
    for (int o = 16; o > 0; o >>= 1) {
      double v2 = __shfl_xor_sync(0xffffffffu, v, o);
      int i2 = __shfl_xor_sync(0xffffffffu, i, o);
      argmax_merge(v, i, v2, i2);
    }
    if (lane == 0) { red_v[0] = v; red_i[0] = i; }
  }
  __syncthreads();
  v = red_v[0];
  i = red_i[0];
  __syncthreads();
}

// Block-wide sum in a fixed order (deterministic).
__device__ double block_sum(double s, double* red) {
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = s;
  __syncthreads();
  if (w == 0) {
    s = lane < nw ? red[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[0] = s;
  }
  __syncthreads();
  s = red[0];
  __syncthreads();
  return s;
}

__device__ int block_min_int(int v, int* red) {
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = lane < nw ? red[lane] : INT_MAX;
    for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  v = red[0];
  __syncthreads();
  return v;
}

// ---------------------------------------------------------------- small path: CTA per block
// dynamic smem: coef[cap] + prod[cap]
__global__ void __launch_bounds__(kSmallThreads)
aca_small_kernel(const AcaBlock* __restrict__ blocks, const int32_t* __restrict__ ids,
                 int32_t* out_rank, uint8_t* out_trunc, double* scr, uint8_t* used_scr,
                 const double* __restrict__ px, const double* __restrict__ py, KernelParams kp,
                 AcaParamsDev ap) {
  extern __shared__ double smem[];
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  __shared__ int s_state[4];
  const int bid = ids[blockIdx.x];
  const AcaBlock b = blocks[bid];
  const int m = b.m, n = b.n, tid = threadIdx.x, T = blockDim.x;
  if (m == 0 || n == 0) {
    if (tid == 0) { out_rank[bid] = 0; out_trunc[bid] = 0; }
    return;
  }
  double* coef = smem;
  double* prod = smem + b.cap;
  double* U = scr + b.u_off;
  double* V = scr + b.v_off;
  uint8_t* used = used_scr + b.used_off;
  const double* PXr = px + b.r0;
  const double* PYr = py + b.r0;
  const double* PXc = px + b.c0;
  const double* PYc = py + b.c0;
  for (int i = tid; i < m; i += T) used[i] = 0;
  const int kmax = min(min(m, n), ap.max_rank);
  int k = 0, istar = 0, zs = 0, hits = 0;
  bool tol_stop = false;
  double S2 = 0.0;
  __syncthreads();
  while (true) {
    // (1) residual row -> V[:, k]
    for (int q = tid; q < k; q += T) coef[q] = U[istar + (size_t)q * m];
    __syncthreads();
    const double pxi = PXr[istar], pyi = PYr[istar];
    double best = -1.0;
    int bj = INT_MAX;
    double* Vk = V + (size_t)k * n;
    for (int j = tid; j < n; j += T) {
      double a = kp.scale * kernel_eval(kp, pxi, pyi, PXc[j], PYc[j]);
      for (int q = 0; q < k; ++q) a = fma(-coef[q], V[j + (size_t)q * n], a);
      Vk[j] = a;
      argmax_merge(best, bj, fabs(a), j);
    }
    block_argmax(best, bj, red_v, red_i);
    if (tid == 0) used[istar] = 1;
    if (best == 0.0) {
      // (3) zero pivot
      ++zs;
      __syncthreads();
      int cand = INT_MAX;
      for (int i = tid; i < m; i += T)
        if (!used[i]) { cand = i; break; }
      cand = block_min_int(cand, red_i);
      if (zs >= 3 || cand == INT_MAX) break;
      istar = cand;
      continue;
    }
    zs = 0;
    const int jstar = bj;
    // (4) v = row / pivot; u = A(X, j*) - sum_q V[j*, q] U[:, q]
    for (int q = tid; q < k; q += T) coef[q] = V[jstar + (size_t)q * n];
    __syncthreads();
    const double piv = Vk[jstar];
    __syncthreads();  // everyone has read the pivot before normalisation overwrites it
    double nv2 = 0.0;
    for (int j = tid; j < n; j += T) {
      double v = Vk[j] / piv;
      Vk[j] = v;
      nv2 = fma(v, v, nv2);
    }
    const double pxj = PXc[jstar], pyj = PYc[jstar];
    double* Uk = U + (size_t)k * m;
    double nu2 = 0.0, ub = -1.0;
    int ui = INT_MAX;
    for (int i = tid; i < m; i += T) {
      double a = kp.scale * kernel_eval(kp, PXr[i], PYr[i], pxj, pyj);
      for (int q = 0; q < k; ++q) a = fma(-coef[q], U[i + (size_t)q * m], a);
      Uk[i] = a;
      nu2 = fma(a, a, nu2);
      if (!used[i]) argmax_merge(ub, ui, fabs(a), i);
    }
    nu2 = block_sum(nu2, red_v);
    nv2 = block_sum(nv2, red_v);
    block_argmax(ub, ui, red_v, red_i);
    // (5) cross terms: warp per previous column
    const int w = tid >> 5, lane = tid & 31, nw = T >> 5;
    for (int q = w; q < k; q += nw) {
      double du = 0.0, dv = 0.0;
      const double* Uq = U + (size_t)q * m;
      const double* Vq = V + (size_t)q * n;
      for (int i = lane; i < m; i += 32) du = fma(Uq[i], Uk[i], du);
      for (int j = lane; j < n; j += 32) dv = fma(Vq[j], Vk[j], dv);
      for (int o = 16; o > 0; o >>= 1) {
        du += __shfl_xor_sync(0xffffffffu, du, o);
        dv += __shfl_xor_sync(0xffffffffu, dv, o);
      }
      if (lane == 0) prod[q] = du * dv;
    }
    __syncthreads();
    double cross = 0.0;
    for (int q = 0; q < k; ++q) cross += prod[q];   // fixed order, every thread identical
    S2 += 2.0 * cross + nu2 * nv2;
    ++k;
    // (7) stopping
    if (sqrt(nu2) * sqrt(nv2) <= ap.tol * sqrt(S2)) ++hits; else hits = 0;
    if (hits >= ap.consecutive) { tol_stop = true; break; }
    if (k == kmax) {
      if (tid == 0) s_state[0] = (k == ap.max_rank && k < min(m, n)) ? 1 : 0;
      break;
    }
    // (8) next row
    if (ui == INT_MAX) break;  // rows exhausted
    istar = ui;
    __syncthreads();
  }
  if (tid == 0) {
    int rank = tol_stop ? k - min(ap.trim, k) : k;
    out_rank[bid] = rank;
    out_trunc[bid] = (!tol_stop && k == ap.max_rank && k < min(m, n)) ? 1 : 0;
  }
}

// ---------------------------------------------------------------- big path (multi-CTA steps)
__global__ void big_init_kernel(const AcaBlock* __restrict__ blocks, AcaState* st, int nblk,
                                uint8_t* used_scr) {
  int b = blockIdx.x;
  if (b >= nblk) return;
  const AcaBlock B = blocks[b];
  for (int i = threadIdx.x; i < B.m; i += blockDim.x) used_scr[B.used_off + i] = 0;
  if (threadIdx.x == 0) {
    AcaState s{};
    s.done = (B.m == 0 || B.n == 0) ? 1 : 0;
    st[b] = s;
  }
}

// Phase R: residual row chunk -> V[:, k] (unnormalised) + chunk argmax.
__global__ void __launch_bounds__(kBigThreads)
big_row_kernel(const AcaBlock* __restrict__ blocks, const AcaState* __restrict__ st,
               const BigItem* __restrict__ items, double* scr, double* part_v, int32_t* part_i,
               const double* __restrict__ px, const double* __restrict__ py, KernelParams kp,
               int max_rank) {
  extern __shared__ double coef[];
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  const BigItem it = items[blockIdx.x];
  const AcaState s = st[it.blk];
  if (s.done) return;
  const AcaBlock B = blocks[it.blk];
  const double* U = scr + B.u_off;
  double* V = scr + B.v_off;
  const int k = s.k, m = B.m, n = B.n;
  for (int q = threadIdx.x; q < k; q += blockDim.x) coef[q] = U[s.istar + (size_t)q * m];
  __syncthreads();
  const double pxi = px[B.r0 + s.istar], pyi = py[B.r0 + s.istar];
  double best = -1.0;
  int bj = INT_MAX;
  double* Vk = V + (size_t)k * n;
  for (int j = it.start + threadIdx.x; j < it.start + it.len; j += blockDim.x) {
    double a = kp.scale * kernel_eval(kp, pxi, pyi, px[B.c0 + j], py[B.c0 + j]);
    for (int q = 0; q < k; ++q) a = fma(-coef[q], V[j + (size_t)q * n], a);
    Vk[j] = a;
    argmax_merge(best, bj, fabs(a), j);
  }
  block_argmax(best, bj, red_v, red_i);
  if (threadIdx.x == 0) {
    part_v[B.p_off + it.chunk] = best;
    part_i[B.p_off + it.chunk] = bj;
  }
}

// Phase P: per block, reduce the row argmax; handle zero pivots.
__global__ void big_pivot_kernel(const AcaBlock* __restrict__ blocks, AcaState* st, int nblk,
                                 const double* part_v, const int32_t* part_i, const double* scr,
                                 uint8_t* used_scr) {
  __shared__ int red_i[32];
  int b = blockIdx.x;
  if (b >= nblk) return;
  AcaState s = st[b];
  if (s.done) return;
  const AcaBlock B = blocks[b];
  double best = -1.0;
  int bj = INT_MAX;
  for (int c = 0; c < B.nchn; ++c) argmax_merge(best, bj, part_v[B.p_off + c], part_i[B.p_off + c]);
  uint8_t* used = used_scr + B.used_off;
  if (threadIdx.x == 0) used[s.istar] = 1;
  __syncthreads();
  if (best == 0.0) {
    s.zs += 1;
    int cand = INT_MAX;
    for (int i = threadIdx.x; i < B.m; i += blockDim.x)
      if (!used[i]) { cand = i; break; }
    cand = block_min_int(cand, red_i);
    if (threadIdx.x == 0) {
      if (s.zs >= 3 || cand == INT_MAX) { s.done = 1; s.rank = s.k; }
      else s.istar = cand;
      s.skip = 1;
      st[b] = s;
    }
    return;
  }
  if (threadIdx.x == 0) {
    s.zs = 0;
    s.skip = 0;
    s.jstar = bj;
    s.piv = scr[B.v_off + (size_t)s.k * B.n + bj];
    st[b] = s;
  }
}

// Phase C: column residual (row chunks) and normalisation of v (column chunks).
__global__ void __launch_bounds__(kBigThreads)
big_col_kernel(const AcaBlock* __restrict__ blocks, const AcaState* __restrict__ st,
               const BigItem* __restrict__ items, double* scr, const uint8_t* __restrict__ used_scr,
               double* part_v, int32_t* part_i, double* part_s, const double* __restrict__ px,
               const double* __restrict__ py, KernelParams kp) {
  extern __shared__ double coef[];
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  const BigItem it = items[blockIdx.x];
  const AcaState s = st[it.blk];
  if (s.done || s.skip) return;
  const AcaBlock B = blocks[it.blk];
  double* U = scr + B.u_off;
  double* V = scr + B.v_off;
  const int k = s.k, m = B.m, n = B.n;
  if (it.kind == 1) {   // normalise v over a column chunk, partial ||v||^2
    double* Vk = V + (size_t)k * n;
    double nv2 = 0.0;
    for (int j = it.start + threadIdx.x; j < it.start + it.len; j += blockDim.x) {
      double v = Vk[j] / s.piv;
      Vk[j] = v;
      nv2 = fma(v, v, nv2);
    }
    nv2 = block_sum(nv2, red_v);
    if (threadIdx.x == 0) part_s[B.p_off + B.nchn + B.nchm + it.chunk] = nv2;
    return;
  }
  for (int q = threadIdx.x; q < k; q += blockDim.x) coef[q] = V[s.jstar + (size_t)q * n];
  __syncthreads();
  const double pxj = px[B.c0 + s.jstar], pyj = py[B.c0 + s.jstar];
  const uint8_t* used = used_scr + B.used_off;
  double* Uk = U + (size_t)k * m;
  double nu2 = 0.0, ub = -1.0;
  int ui = INT_MAX;
  for (int i = it.start + threadIdx.x; i < it.start + it.len; i += blockDim.x) {
    double a = kp.scale * kernel_eval(kp, px[B.r0 + i], py[B.r0 + i], pxj, pyj);
    for (int q = 0; q < k; ++q) a = fma(-coef[q], U[i + (size_t)q * m], a);
    Uk[i] = a;
    nu2 = fma(a, a, nu2);
    if (!used[i]) argmax_merge(ub, ui, fabs(a), i);
  }
  nu2 = block_sum(nu2, red_v);
  block_argmax(ub, ui, red_v, red_i);
  if (threadIdx.x == 0) {
    part_s[B.p_off + B.nchn + it.chunk] = nu2;
    part_v[B.p_off + B.nchn + it.chunk] = ub;
    part_i[B.p_off + B.nchn + it.chunk] = ui;
  }
}

// Phase D: partial dot products U_q . u (row chunks) or V_q . v (column chunks), q < k.
// part_d layout per block: [(nchm + nchn) x cap], chunk-major.
__global__ void __launch_bounds__(kBigThreads)
big_dots_kernel(const AcaBlock* __restrict__ blocks, const AcaState* __restrict__ st,
                const BigItem* __restrict__ items, const double* __restrict__ scr, double* part_d,
                const int64_t* __restrict__ d_off) {
  const BigItem it = items[blockIdx.x];
  const AcaState s = st[it.blk];
  if (s.done || s.skip) return;
  const AcaBlock B = blocks[it.blk];
  const int k = s.k;
  const double* F = it.kind == 0 ? scr + B.u_off : scr + B.v_off;
  const int64_t ld = it.kind == 0 ? B.m : B.n;
  const double* Fk = F + (size_t)k * ld;
  const int row = it.kind == 0 ? it.chunk : B.nchm + it.chunk;
  double* out = part_d + d_off[it.blk] + (int64_t)row * B.cap;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int q = w; q < k; q += nw) {
    const double* Fq = F + (size_t)q * ld;
    double d = 0.0;
    for (int i = it.start + lane; i < it.start + it.len; i += 32) d = fma(Fq[i], Fk[i], d);
    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    if (lane == 0) out[q] = d;
  }
}

// Phase S: per block, finish the step (norm estimate, stopping rule, next pivot row).
__global__ void big_update_kernel(const AcaBlock* __restrict__ blocks, AcaState* st, int nblk,
                                  const double* part_v, const int32_t* part_i, const double* part_s,
                                  const double* part_d, const int64_t* __restrict__ d_off,
                                  AcaParamsDev ap, int* active) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nblk) return;
  AcaState s = st[b];
  if (s.done) return;
  if (s.skip) { atomicAdd(active, 1); return; }
  const AcaBlock B = blocks[b];
  double nu2 = 0.0, nv2 = 0.0, ub = -1.0;
  int ui = INT_MAX;
  for (int c = 0; c < B.nchm; ++c) {
    nu2 += part_s[B.p_off + B.nchn + c];
    argmax_merge(ub, ui, part_v[B.p_off + B.nchn + c], part_i[B.p_off + B.nchn + c]);
  }
  for (int c = 0; c < B.nchn; ++c) nv2 += part_s[B.p_off + B.nchn + B.nchm + c];
  double cross = 0.0;
  const double* D = part_d + d_off[b];
  for (int q = 0; q < s.k; ++q) {
    double du = 0.0, dv = 0.0;
    for (int c = 0; c < B.nchm; ++c) du += D[(int64_t)c * B.cap + q];
    for (int c = 0; c < B.nchn; ++c) dv += D[(int64_t)(B.nchm + c) * B.cap + q];
    cross += du * dv;
  }
  s.S2 += 2.0 * cross + nu2 * nv2;
  s.k += 1;
  const int kmax = min(min(B.m, B.n), ap.max_rank);
  if (sqrt(nu2) * sqrt(nv2) <= ap.tol * sqrt(s.S2)) s.hits += 1; else s.hits = 0;
  if (s.hits >= ap.consecutive) {
    s.done = 1;
    s.rank = s.k - min(ap.trim, s.k);
  } else if (s.k == kmax) {
    s.done = 1;
    s.rank = s.k;
    s.trunc = (s.k == ap.max_rank && s.k < min(B.m, B.n)) ? 1 : 0;
  } else if (ui == INT_MAX) {
    s.done = 1;
    s.rank = s.k;
  } else {
    s.istar = ui;
  }
  st[b] = s;
  if (!s.done) atomicAdd(active, 1);
}

__global__ void big_finish_kernel(const AcaState* __restrict__ st, const int32_t* __restrict__ ids,
                                  int nblk, int32_t* out_rank, uint8_t* out_trunc) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nblk) return;
  out_rank[ids[b]] = st[b].rank;
  out_trunc[ids[b]] = (uint8_t)st[b].trunc;
}

// Batched contiguous copies (compaction of ACA scratch into exact-size stores).
struct CopyItem {
  const double* src;
  double* dst;
  int64_t count;
};
__global__ void batched_copy_kernel(const CopyItem* __restrict__ items) {
  const CopyItem it = items[blockIdx.x];
  for (int64_t i = threadIdx.x; i < it.count; i += blockDim.x) it.dst[i] = it.src[i];
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

template <class T>
T* dev_upload(const std::vector<T>& v, cudaStream_t s) {
  T* p = nullptr;
  H2D_CUDA(cudaMallocAsync(&p, std::max<size_t>(1, v.size()) * sizeof(T), s));
  if (!v.empty())
    H2D_CUDA(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  return p;
}

// Run the multi-CTA ACA on a set of big blocks already laid out in scratch.
void run_big(Handle& h, std::vector<AcaBlock>& blk, const std::vector<int32_t>& ids,
             double* d_scr, uint8_t* d_used, int32_t* d_rank, uint8_t* d_trunc,
             const AcaParamsDev& ap) {
  cudaStream_t s = h.stream;
  const int nb = (int)blk.size();
  if (nb == 0) return;
  std::vector<BigItem> row_items, all_items;
  std::vector<int64_t> doff(nb);
  int64_t p_tot = 0, d_tot = 0;
  int maxcap = 1;
  for (int b = 0; b < nb; ++b) {
    AcaBlock& B = blk[b];
    B.nchm = (B.m + kChunk - 1) / kChunk;
    B.nchn = (B.n + kChunk - 1) / kChunk;
    B.p_off = p_tot;
    p_tot += 2 * (int64_t)(B.nchm + B.nchn);
    doff[b] = d_tot;
    d_tot += (int64_t)(B.nchm + B.nchn) * B.cap;
    maxcap = std::max(maxcap, B.cap);
    for (int c = 0; c < B.nchn; ++c) {
      BigItem it{b, 1, c * kChunk, std::min(kChunk, B.n - c * kChunk), c, 0};
      row_items.push_back(it);
      all_items.push_back(it);
    }
    for (int c = 0; c < B.nchm; ++c)
      all_items.push_back(BigItem{b, 0, c * kChunk, std::min(kChunk, B.m - c * kChunk), c, 0});
  }
  AcaBlock* d_blk = dev_upload(blk, s);
  int32_t* d_ids = dev_upload(ids, s);
  BigItem* d_row = dev_upload(row_items, s);
  BigItem* d_all = dev_upload(all_items, s);
  int64_t* d_doff = dev_upload(doff, s);
  AcaState* d_st = nullptr;
  double *d_pv = nullptr, *d_ps = nullptr, *d_pd = nullptr;
  int32_t* d_pi = nullptr;
  int* d_active = nullptr;
  H2D_CUDA(cudaMallocAsync(&d_st, nb * sizeof(AcaState), s));
  H2D_CUDA(cudaMallocAsync(&d_pv, std::max<int64_t>(1, p_tot) * sizeof(double), s));
  H2D_CUDA(cudaMallocAsync(&d_ps, std::max<int64_t>(1, p_tot) * sizeof(double), s));
  H2D_CUDA(cudaMallocAsync(&d_pi, std::max<int64_t>(1, p_tot) * sizeof(int32_t), s));
  H2D_CUDA(cudaMallocAsync(&d_pd, std::max<int64_t>(1, d_tot) * sizeof(double), s));
  H2D_CUDA(cudaMallocAsync(&d_active, sizeof(int), s));
  big_init_kernel<<<nb, 256, 0, s>>>(d_blk, d_st, nb, d_used);
  H2D_LAUNCH_CHECK();
  const size_t smem = (size_t)maxcap * sizeof(double);
  int maxk = 0;
  for (auto& B : blk) maxk = std::max(maxk, std::min(std::min(B.m, B.n), ap.max_rank));
  // Each block needs at most maxk productive steps plus zero-pivot retries; poll the
  // active count every few steps.
  int step = 0;
  while (true) {
    for (int rep = 0; rep < 4; ++rep, ++step) {
      H2D_CUDA(cudaMemsetAsync(d_active, 0, sizeof(int), s));
      if (row_items.empty() || all_items.empty()) throw Error{H2D_ECUDA, "ACA big path: empty block"};
      big_row_kernel<<<(int)row_items.size(), kBigThreads, smem, s>>>(
          d_blk, d_st, d_row, d_scr, d_pv, d_pi, h.d_px, h.d_py, h.kp, ap.max_rank);
      big_pivot_kernel<<<nb, 256, 0, s>>>(d_blk, d_st, nb, d_pv, d_pi, d_scr, d_used);
      big_col_kernel<<<(int)all_items.size(), kBigThreads, smem, s>>>(
          d_blk, d_st, d_all, d_scr, d_used, d_pv, d_pi, d_ps, h.d_px, h.d_py, h.kp);
      big_dots_kernel<<<(int)all_items.size(), kBigThreads, 0, s>>>(d_blk, d_st, d_all, d_scr,
                                                                    d_pd, d_doff);
      big_update_kernel<<<(nb + 127) / 128, 128, 0, s>>>(d_blk, d_st, nb, d_pv, d_pi, d_ps, d_pd,
                                                         d_doff, ap, d_active);
      H2D_LAUNCH_CHECK();
    }
    int active = 0;
    H2D_CUDA(cudaMemcpyAsync(&active, d_active, sizeof(int), cudaMemcpyDeviceToHost, s));
    H2D_CUDA(cudaStreamSynchronize(s));
    if (active == 0) break;
    if (step > 4 * (maxk + 16) + 64)
      throw Error{H2D_ECUDA, "ACA (big path) did not terminate"};
  }
  big_finish_kernel<<<(nb + 127) / 128, 128, 0, s>>>(d_st, d_ids, nb, d_rank, d_trunc);
  H2D_LAUNCH_CHECK();
  for (void* p : {(void*)d_blk, (void*)d_ids, (void*)d_row, (void*)d_all, (void*)d_doff,
                  (void*)d_st, (void*)d_pv, (void*)d_ps, (void*)d_pi, (void*)d_pd, (void*)d_active})
    H2D_CUDA(cudaFreeAsync(p, s));
}

}  // namespace

void run_aca(Handle& h) {
  cudaStream_t s = h.stream;
  const AcaParamsDev ap{h.tol, h.opts.max_rank, h.opts.aca_consecutive, h.opts.aca_trim};
  for (int l = h.kappa; l >= 1; --l) {
    Level& L = h.levels[(size_t)l];
    const int64_t nbk = L.nblocks;
    L.rank.assign((size_t)nbk, -1);
    L.truncated.assign((size_t)nbk, 0);
    // blocks served by this rank (row box intersects the served rows)
    // symmetric (R23): one ACA per unordered pair, on K(X, Y) with X < Y; the block (Y, X)
    // takes the swapped factors after the level's ACA
    const bool sym = h.opts.symmetric != 0;
    std::vector<int64_t> todo;
    for (int64_t X = 0; X < L.nbox; ++X) {
      const bool mz = h.box_end(l, X) == h.box_begin(l, X);
      for (int32_t e = L.off[(size_t)X]; e < L.off[(size_t)X + 1]; ++e) {
        const int64_t Y = L.col[(size_t)e];
        const bool need = sym ? X < Y && (h.row_box_active(l, X) || h.row_box_active(l, Y))
                              : h.row_box_active(l, X);
        if (!need) continue;
        if (mz || h.box_end(l, Y) == h.box_begin(l, Y)) L.rank[(size_t)e] = 0;   // empty side (R5)
        else todo.push_back(e);
      }
    }
    std::vector<const double*> srcU((size_t)nbk, nullptr), srcV((size_t)nbk, nullptr);
    auto mirror = [&]() {   // symmetric: block (X, Y), X > Y, from block (Y, X)
      if (!sym) return;
      for (int64_t X = 0; X < L.nbox; ++X) {
        if (!h.row_box_active(l, X)) continue;
        for (int32_t e = L.off[(size_t)X]; e < L.off[(size_t)X + 1]; ++e) {
          if (L.col[(size_t)e] > X) continue;
          const int32_t t = L.trans[(size_t)e];
          L.rank[(size_t)e] = L.rank[(size_t)t];
          L.truncated[(size_t)e] = L.truncated[(size_t)t];
          srcU[(size_t)e] = srcV[(size_t)t];
          srcV[(size_t)e] = srcU[(size_t)t];
        }
      }
    };
    if (todo.empty()) {
      mirror();
      pack_level(h, L, srcU, srcV);
      continue;
    }
    double t0 = now_s();
    size_t free_b = 0, tot_b = 0;
    H2D_CUDA(cudaMemGetInfo(&free_b, &tot_b));
    size_t budget = h.opts.aca_scratch_bytes ? h.opts.aca_scratch_bytes : (size_t)(0.4 * free_b);
    budget = std::max<size_t>(budget, 64ull << 20);
    int32_t* d_rank = nullptr;
    uint8_t* d_trunc = nullptr;
    H2D_CUDA(cudaMallocAsync(&d_rank, nbk * sizeof(int32_t), s));
    H2D_CUDA(cudaMallocAsync(&d_trunc, nbk, s));
    H2D_CUDA(cudaMemsetAsync(d_rank, 0xff, nbk * sizeof(int32_t), s));
    H2D_CUDA(cudaMemsetAsync(d_trunc, 0, nbk, s));
    std::vector<double*> stores;      // compacted per-batch stores (when >1 batch)
    size_t pos = 0;
    bool single_batch = true;
    std::vector<double*> scratches;
    while (pos < todo.size()) {
      // form a batch within the scratch budget
      std::vector<AcaBlock> small_blk, big_blk;
      std::vector<int32_t> small_ids, big_ids;
      std::vector<AcaBlock> all_blk;
      std::vector<int64_t> all_e;
      int64_t dbl = 0, byt = 0;
      size_t start = pos;
      while (pos < todo.size()) {
        int64_t e = todo[pos];
        int64_t X = -1;
        // row box of block e: binary search in off
        X = (int64_t)(std::upper_bound(L.off.begin(), L.off.end(), (int32_t)e) - L.off.begin()) - 1;
        while (L.off[(size_t)X + 1] <= e) ++X;
        int64_t Y = L.col[(size_t)e];
        AcaBlock B{};
        B.r0 = h.box_begin(l, X);
        B.m = (int32_t)(h.box_end(l, X) - B.r0);
        B.c0 = h.box_begin(l, Y);
        B.n = (int32_t)(h.box_end(l, Y) - B.c0);
        B.cap = std::max(1, std::min(std::min(B.m, B.n), h.opts.max_rank));
        int64_t need_d = (int64_t)B.cap * (B.m + B.n);
        int64_t need_b = need_d * 8 + B.m;
        if (pos > start && (size_t)((dbl + need_d) * 8 + byt + B.m) > budget) break;
        B.u_off = dbl;
        B.v_off = dbl + (int64_t)B.cap * B.m;
        B.used_off = byt;
        dbl += need_d;
        byt += B.m;
        (void)need_b;
        all_blk.push_back(B);
        all_e.push_back(e);
        ++pos;
      }
      if (pos < todo.size() || start > 0) single_batch = false;
      double* d_scr = nullptr;
      uint8_t* d_used = nullptr;
      H2D_CUDA(cudaMalloc(&d_scr, std::max<int64_t>(1, dbl) * sizeof(double)));
      H2D_CUDA(cudaMalloc(&d_used, std::max<int64_t>(1, byt)));
      // classify: multi-CTA path for few, huge blocks
      for (size_t i = 0; i < all_blk.size(); ++i) {
        const AcaBlock& B = all_blk[i];
        bool big = (int64_t)B.m + B.n > 8192 || (L.nblocks < 296 && (int64_t)B.m + B.n > 2048);
        if (big) { big_blk.push_back(B); big_ids.push_back((int32_t)all_e[i]); }
        else { small_blk.push_back(B); small_ids.push_back((int32_t)all_e[i]); }
      }
      if (!small_blk.empty()) {
        // index small blocks through ids: upload blocks indexed by CSR id
        std::vector<AcaBlock> by_id(small_blk);
        AcaBlock* d_blk = nullptr;
        int32_t* d_ids = nullptr;
        // kernel reads blocks[ids[blockIdx]] -> build a dense array + identity-free indexing
        std::vector<int32_t> local((size_t)small_blk.size());
        for (size_t i = 0; i < local.size(); ++i) local[i] = (int32_t)i;
        d_blk = dev_upload(by_id, s);
        d_ids = dev_upload(local, s);
        int32_t* d_r = nullptr;
        uint8_t* d_t = nullptr;
        H2D_CUDA(cudaMallocAsync(&d_r, small_blk.size() * sizeof(int32_t), s));
        H2D_CUDA(cudaMallocAsync(&d_t, small_blk.size(), s));
        int maxcap = 1;
        for (auto& B : small_blk) maxcap = std::max(maxcap, B.cap);
        size_t smem = 2 * (size_t)maxcap * sizeof(double);
        if (smem > 48 * 1024)
          H2D_CUDA(cudaFuncSetAttribute(aca_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
        aca_small_kernel<<<(int)small_blk.size(), kSmallThreads, smem, s>>>(
            d_blk, d_ids, d_r, d_t, d_scr, d_used, h.d_px, h.d_py, h.kp, ap);
        H2D_LAUNCH_CHECK();
        std::vector<int32_t> r(small_blk.size());
        std::vector<uint8_t> t(small_blk.size());
        H2D_CUDA(cudaMemcpyAsync(r.data(), d_r, r.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        H2D_CUDA(cudaMemcpyAsync(t.data(), d_t, t.size(), cudaMemcpyDeviceToHost, s));
        H2D_CUDA(cudaStreamSynchronize(s));
        for (size_t i = 0; i < r.size(); ++i) {
          L.rank[(size_t)small_ids[i]] = r[i];
          L.truncated[(size_t)small_ids[i]] = t[i];
        }
        for (void* p : {(void*)d_blk, (void*)d_ids, (void*)d_r, (void*)d_t}) H2D_CUDA(cudaFreeAsync(p, s));
      }
      if (!big_blk.empty()) {
        run_big(h, big_blk, big_ids, d_scr, d_used, d_rank, d_trunc, ap);
        std::vector<int32_t> r((size_t)nbk);
        std::vector<uint8_t> t((size_t)nbk);
        H2D_CUDA(cudaMemcpyAsync(r.data(), d_rank, nbk * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        H2D_CUDA(cudaMemcpyAsync(t.data(), d_trunc, nbk, cudaMemcpyDeviceToHost, s));
        H2D_CUDA(cudaStreamSynchronize(s));
        for (int32_t e : big_ids) {
          L.rank[(size_t)e] = r[(size_t)e];
          L.truncated[(size_t)e] = t[(size_t)e];
        }
      }
      H2D_CUDA(cudaStreamSynchronize(s));
      H2D_CUDA(cudaFree(d_used));
      if (single_batch) {
        for (size_t i = 0; i < all_blk.size(); ++i) {
          srcU[(size_t)all_e[i]] = d_scr + all_blk[i].u_off;
          srcV[(size_t)all_e[i]] = d_scr + all_blk[i].v_off;
        }
        scratches.push_back(d_scr);
      } else {
        // compact into an exact-size store
        int64_t tot = 0;
        for (size_t i = 0; i < all_blk.size(); ++i) {
          int r = L.rank[(size_t)all_e[i]];
          tot += (int64_t)r * (all_blk[i].m + all_blk[i].n);
        }
        double* store = nullptr;
        H2D_CUDA(cudaMalloc(&store, std::max<int64_t>(1, tot) * sizeof(double)));
        std::vector<CopyItem> items;
        int64_t o = 0;
        for (size_t i = 0; i < all_blk.size(); ++i) {
          const AcaBlock& B = all_blk[i];
          int r = L.rank[(size_t)all_e[i]];
          srcU[(size_t)all_e[i]] = store + o;
          if ((int64_t)r * B.m) items.push_back(CopyItem{d_scr + B.u_off, store + o, (int64_t)r * B.m});
          o += (int64_t)r * B.m;
          srcV[(size_t)all_e[i]] = store + o;
          if ((int64_t)r * B.n) items.push_back(CopyItem{d_scr + B.v_off, store + o, (int64_t)r * B.n});
          o += (int64_t)r * B.n;
        }
        for (size_t c0 = 0; c0 < items.size(); c0 += 1 << 20) {
          std::vector<CopyItem> part(items.begin() + c0,
                                     items.begin() + std::min(items.size(), c0 + (1 << 20)));
          CopyItem* d_items = dev_upload(part, s);
          batched_copy_kernel<<<(int)part.size(), 256, 0, s>>>(d_items);
          H2D_LAUNCH_CHECK();
          H2D_CUDA(cudaFreeAsync(d_items, s));
        }
        H2D_CUDA(cudaStreamSynchronize(s));
        H2D_CUDA(cudaFree(d_scr));
        stores.push_back(store);
      }
    }
    H2D_CUDA(cudaStreamSynchronize(s));
    h.aca_seconds += now_s() - t0;
    for (int64_t e : todo) h.truncated += L.truncated[(size_t)e];
    mirror();
    double t1 = now_s();
    pack_level(h, L, srcU, srcV);
    H2D_CUDA(cudaStreamSynchronize(s));
    h.pack_seconds += now_s() - t1;
    for (double* p : scratches) H2D_CUDA(cudaFree(p));
    for (double* p : stores) H2D_CUDA(cudaFree(p));
    H2D_CUDA(cudaFreeAsync(d_rank, s));
    H2D_CUDA(cudaFreeAsync(d_trunc, s));
  }
}

}  // namespace h2d
