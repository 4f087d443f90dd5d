// Quadtree (S1-S3) and interaction / near-field lists (S4-S5) as integer GPU kernels.
//
//  S1 quantise + Morton code  : ix = min(2^k - 1, floor(((x - lo) / side) * 2^k)) with
//                               correctly rounded __dsub_rn / __ddiv_rn / __dmul_rn (no FMA
//                               contraction) so the result is bit-exact with the oracle
//                               (R3); Z-order with the x bit at even positions (R4).
//  S2 stable radix sort       : CUB DeviceRadixSort (LSD, stable) of (code, index) pairs.
//  S3 box ranges              : leaf_start[b] = lower_bound(codes, b); box (l, b) spans
//                               leaves [b << 2(k-l), (b+1) << 2(k-l)).
//  S4 interaction lists       : closed form of Eq. eq:ilist:
//                               I_C = { D : |parent(C) - parent(D)|_1 <= 1, |C - D|_1 >= 2 }
//                               (clan = siblings + children of the parent's edge sharers,
//                               Def. 4.4; minus self and edge sharers, Defs 4.1-4.3),
//                               partners in ascending Morton order (R5).
//  S5 near field              : {X} u E_X at the leaves (Alg. 1 l.5).
#include <algorithm>

#include <cub/cub.cuh>

#include "h2d_internal.cuh"

namespace h2d {
namespace {

__host__ __device__ __forceinline__ uint32_t spread_bits(uint32_t v) {
  v &= 0xFFFFu;
  v = (v | (v << 8)) & 0x00FF00FFu;
  v = (v | (v << 4)) & 0x0F0F0F0Fu;
  v = (v | (v << 2)) & 0x33333333u;
  v = (v | (v << 1)) & 0x55555555u;
  return v;
}
__host__ __device__ __forceinline__ uint32_t compact_bits(uint32_t v) {
  v &= 0x55555555u;
  v = (v | (v >> 1)) & 0x33333333u;
  v = (v | (v >> 2)) & 0x0F0F0F0Fu;
  v = (v | (v >> 4)) & 0x00FF00FFu;
  v = (v | (v >> 8)) & 0x0000FFFFu;
  return v;
}
__device__ __forceinline__ uint32_t morton(uint32_t ix, uint32_t iy) {
  return spread_bits(ix) | (spread_bits(iy) << 1);
}

// Per-CTA bounding box + first non-finite index.
__global__ void bbox_kernel(const double* __restrict__ pts, int64_t n, double4* partial,
                            unsigned long long* bad) {
  double mnx = INFINITY, mny = INFINITY, mxx = -INFINITY, mxy = -INFINITY;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double x = pts[2 * i], y = pts[2 * i + 1];
    if (!isfinite(x) || !isfinite(y)) {
      atomicMin(bad, (unsigned long long)i);
      continue;
    }
    mnx = fmin(mnx, x); mny = fmin(mny, y);
    mxx = fmax(mxx, x); mxy = fmax(mxy, y);
  }
  __shared__ double s[4][32];
  for (int o = 16; o > 0; o >>= 1) {
    mnx = fmin(mnx, __shfl_xor_sync(0xffffffffu, mnx, o));
    mny = fmin(mny, __shfl_xor_sync(0xffffffffu, mny, o));
    mxx = fmax(mxx, __shfl_xor_sync(0xffffffffu, mxx, o));
    mxy = fmax(mxy, __shfl_xor_sync(0xffffffffu, mxy, o));
  }
  int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { s[0][w] = mnx; s[1][w] = mny; s[2][w] = mxx; s[3][w] = mxy; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
      mnx = fmin(mnx, s[0][k]); mny = fmin(mny, s[1][k]);
      mxx = fmax(mxx, s[2][k]); mxy = fmax(mxy, s[3][k]);
    }
    partial[blockIdx.x] = make_double4(mnx, mny, mxx, mxy);
  }
}

// S1: quantise + Morton code (bit-exact: no contraction, correctly rounded ops).
__global__ void quantize_kernel(const double* __restrict__ pts, int64_t n, double lo_x,
                                double lo_y, double side, int kappa, uint32_t* codes,
                                int32_t* idx, unsigned long long* outside) {
  const double scale = (double)(1u << kappa);
  const int maxc = (1 << kappa) - 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double qx = __ddiv_rn(__dsub_rn(pts[2 * i], lo_x), side);
    double qy = __ddiv_rn(__dsub_rn(pts[2 * i + 1], lo_y), side);
    if (!(qx >= 0.0 && qx <= 1.0 && qy >= 0.0 && qy <= 1.0)) {
      atomicMin(outside, (unsigned long long)i);
      qx = fmin(fmax(qx, 0.0), 1.0);
      qy = fmin(fmax(qy, 0.0), 1.0);
    }
    int ix = min((int)floor(__dmul_rn(qx, scale)), maxc);
    int iy = min((int)floor(__dmul_rn(qy, scale)), maxc);
    codes[i] = morton((uint32_t)ix, (uint32_t)iy);
    idx[i] = (int32_t)i;
  }
}

// S2 epilogue: SoA points in TREE order.
__global__ void gather_points_kernel(const double* __restrict__ pts, const int32_t* __restrict__ perm,
                                     int64_t n, double* px, double* py) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n;
       s += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = perm[s];
    px[s] = pts[2 * i];
    py[s] = pts[2 * i + 1];
  }
}

// S3: leaf_start[b] = first TREE position whose code >= b, b in [0, 4^kappa].
__global__ void leaf_start_kernel(const uint32_t* __restrict__ codes, int64_t n, int64_t nleaf,
                                  int32_t* leaf_start) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b <= nleaf;
       b += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if ((int64_t)codes[mid] < b) lo = mid + 1; else hi = mid;
    }
    leaf_start[b] = (int32_t)lo;
  }
}

// S4: closed-form interaction list of box b at level l (sorted ascending).
__device__ int box_list(int l, uint32_t b, uint32_t* out) {
  int cx = (int)compact_bits(b), cy = (int)compact_bits(b >> 1);
  int px = cx >> 1, py = cy >> 1, pside = 1 << (l - 1);
  int cnt = 0;
  const int dxs[5] = {0, -1, 1, 0, 0}, dys[5] = {0, 0, 0, -1, 1};
  for (int k = 0; k < 5; ++k) {               // parent and its edge sharers
    int qx = px + dxs[k], qy = py + dys[k];
    if (qx < 0 || qy < 0 || qx >= pside || qy >= pside) continue;
    for (int c = 0; c < 4; ++c) {             // their children
      int dx = 2 * qx + (c & 1), dy = 2 * qy + (c >> 1);
      if (abs(dx - cx) + abs(dy - cy) >= 2) {
        uint32_t code = morton((uint32_t)dx, (uint32_t)dy);
        int j = cnt++;
        while (j > 0 && out[j - 1] > code) { out[j] = out[j - 1]; --j; }   // insertion sort
        out[j] = code;
      }
    }
  }
  return cnt;
}

// S5: near field of leaf b: self + edge sharers (sorted ascending).
__device__ int near_list(int l, uint32_t b, uint32_t* out) {
  int cx = (int)compact_bits(b), cy = (int)compact_bits(b >> 1), side = 1 << l;
  const int dxs[5] = {0, -1, 1, 0, 0}, dys[5] = {0, 0, 0, -1, 1};
  int cnt = 0;
  for (int k = 0; k < 5; ++k) {
    int qx = cx + dxs[k], qy = cy + dys[k];
    if (qx < 0 || qy < 0 || qx >= side || qy >= side) continue;
    uint32_t code = morton((uint32_t)qx, (uint32_t)qy);
    int j = cnt++;
    while (j > 0 && out[j - 1] > code) { out[j] = out[j - 1]; --j; }
    out[j] = code;
  }
  return cnt;
}

__global__ void list_count_kernel(int l, int near, int64_t nbox, int32_t* count) {
  uint32_t tmp[20];
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nbox;
       b += (int64_t)gridDim.x * blockDim.x)
    count[b] = near ? near_list(l, (uint32_t)b, tmp) : box_list(l, (uint32_t)b, tmp);
}

__global__ void list_fill_kernel(int l, int near, int64_t nbox, const int32_t* __restrict__ off,
                                 int32_t* col) {
  uint32_t tmp[20];
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nbox;
       b += (int64_t)gridDim.x * blockDim.x) {
    int c = near ? near_list(l, (uint32_t)b, tmp) : box_list(l, (uint32_t)b, tmp);
    int32_t o = off[b];
    for (int k = 0; k < c; ++k) col[o + k] = (int32_t)tmp[k];
  }
}

int grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 32));
}

// CSR of one level (near = 0) or of the leaf near field (near = 1).
void make_csr(Handle& h, int l, int near, int32_t*& d_off, int32_t*& d_col,
              std::vector<int32_t>& off, std::vector<int32_t>& col) {
  int64_t nbox = (int64_t)1 << (2 * l);
  d_off = h.alloc<int32_t>(nbox + 1);
  int32_t* d_cnt = nullptr;
  H2D_CUDA(cudaMallocAsync(&d_cnt, (nbox + 1) * sizeof(int32_t), h.stream));
  H2D_CUDA(cudaMemsetAsync(d_cnt, 0, (nbox + 1) * sizeof(int32_t), h.stream));
  list_count_kernel<<<grid_for(nbox, 256), 256, 0, h.stream>>>(l, near, nbox, d_cnt);
  H2D_LAUNCH_CHECK();
  size_t tmp_bytes = 0;
  H2D_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, d_cnt, d_off, (int)(nbox + 1), h.stream));
  void* d_tmp = nullptr;
  H2D_CUDA(cudaMallocAsync(&d_tmp, tmp_bytes, h.stream));
  H2D_CUDA(cub::DeviceScan::ExclusiveSum(d_tmp, tmp_bytes, d_cnt, d_off, (int)(nbox + 1), h.stream));
  off.resize((size_t)nbox + 1);
  H2D_CUDA(cudaMemcpyAsync(off.data(), d_off, (nbox + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost,
                           h.stream));
  H2D_CUDA(cudaStreamSynchronize(h.stream));
  int64_t tot = off[(size_t)nbox];
  d_col = h.alloc<int32_t>(tot);
  list_fill_kernel<<<grid_for(nbox, 256), 256, 0, h.stream>>>(l, near, nbox, d_off, d_col);
  H2D_LAUNCH_CHECK();
  col.resize((size_t)tot);
  if (tot)
    H2D_CUDA(cudaMemcpyAsync(col.data(), d_col, tot * sizeof(int32_t), cudaMemcpyDeviceToHost,
                             h.stream));
  H2D_CUDA(cudaFreeAsync(d_cnt, h.stream));
  H2D_CUDA(cudaFreeAsync(d_tmp, h.stream));
  H2D_CUDA(cudaStreamSynchronize(h.stream));
}

}  // namespace

void build_tree(Handle& h, const double* d_points) {
  const int64_t n = h.n;
  cudaStream_t s = h.stream;
  // R2: root box (explicit or bounding square); reject non-finite input.
  {
    int blocks = grid_for(n, 256);
    double4* d_part = nullptr;
    unsigned long long* d_bad = nullptr;
    H2D_CUDA(cudaMallocAsync(&d_part, blocks * sizeof(double4), s));
    H2D_CUDA(cudaMallocAsync(&d_bad, sizeof(unsigned long long), s));
    H2D_CUDA(cudaMemsetAsync(d_bad, 0xff, sizeof(unsigned long long), s));
    bbox_kernel<<<blocks, 256, 0, s>>>(d_points, n, d_part, d_bad);
    H2D_LAUNCH_CHECK();
    std::vector<double4> part(blocks);
    unsigned long long bad = 0;
    H2D_CUDA(cudaMemcpyAsync(part.data(), d_part, blocks * sizeof(double4), cudaMemcpyDeviceToHost, s));
    H2D_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost, s));
    H2D_CUDA(cudaStreamSynchronize(s));
    H2D_CUDA(cudaFreeAsync(d_part, s));
    H2D_CUDA(cudaFreeAsync(d_bad, s));
    if (bad != ~0ull) throw Error{H2D_EINVAL, "non-finite point at index " + std::to_string(bad)};
    if (h.opts.box_side > 0) {
      h.lo[0] = h.opts.box_lo[0];
      h.lo[1] = h.opts.box_lo[1];
      h.side = h.opts.box_side;
    } else {
      double mnx = INFINITY, mny = INFINITY, mxx = -INFINITY, mxy = -INFINITY;
      for (auto& p : part) {
        mnx = std::min(mnx, p.x); mny = std::min(mny, p.y);
        mxx = std::max(mxx, p.z); mxy = std::max(mxy, p.w);
      }
      h.lo[0] = mnx;
      h.lo[1] = mny;
      h.side = std::max(mxx - mnx, mxy - mny);
      if (h.side == 0.0) h.side = 1.0;
    }
  }
  const int kappa = h.kappa;
  const int64_t nleaf = (int64_t)1 << (2 * kappa);
  uint32_t *d_codes = nullptr, *d_codes_sorted = nullptr;
  int32_t* d_idx = nullptr;
  unsigned long long* d_out = nullptr;
  H2D_CUDA(cudaMallocAsync(&d_codes, n * sizeof(uint32_t), s));
  H2D_CUDA(cudaMallocAsync(&d_codes_sorted, n * sizeof(uint32_t), s));
  H2D_CUDA(cudaMallocAsync(&d_idx, n * sizeof(int32_t), s));
  H2D_CUDA(cudaMallocAsync(&d_out, sizeof(unsigned long long), s));
  H2D_CUDA(cudaMemsetAsync(d_out, 0xff, sizeof(unsigned long long), s));
  quantize_kernel<<<grid_for(n, 256), 256, 0, s>>>(d_points, n, h.lo[0], h.lo[1], h.side, kappa,
                                                   d_codes, d_idx, d_out);
  H2D_LAUNCH_CHECK();
  unsigned long long outside = 0;
  H2D_CUDA(cudaMemcpyAsync(&outside, d_out, sizeof(outside), cudaMemcpyDeviceToHost, s));
  H2D_CUDA(cudaStreamSynchronize(s));
  if (outside != ~0ull)
    throw Error{H2D_EOUTOFBOX, "point " + std::to_string(outside) + " outside the root box"};
  // S2: stable LSD radix sort by code
  h.d_perm = h.alloc<int32_t>(n);
  size_t tmp_bytes = 0;
  int end_bit = std::max(1, 2 * kappa);
  H2D_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, d_codes, d_codes_sorted, d_idx,
                                           h.d_perm, (int)n, 0, end_bit, s));
  void* d_tmp = nullptr;
  H2D_CUDA(cudaMallocAsync(&d_tmp, tmp_bytes, s));
  H2D_CUDA(cub::DeviceRadixSort::SortPairs(d_tmp, tmp_bytes, d_codes, d_codes_sorted, d_idx,
                                           h.d_perm, (int)n, 0, end_bit, s));
  h.d_px = h.alloc<double>(n);
  h.d_py = h.alloc<double>(n);
  gather_points_kernel<<<grid_for(n, 256), 256, 0, s>>>(d_points, h.d_perm, n, h.d_px, h.d_py);
  H2D_LAUNCH_CHECK();
  // S3
  h.d_leaf_start = h.alloc<int32_t>(nleaf + 1);
  leaf_start_kernel<<<grid_for(nleaf + 1, 256), 256, 0, s>>>(d_codes_sorted, n, nleaf, h.d_leaf_start);
  H2D_LAUNCH_CHECK();
  h.leaf_start.resize((size_t)nleaf + 1);
  H2D_CUDA(cudaMemcpyAsync(h.leaf_start.data(), h.d_leaf_start, (nleaf + 1) * sizeof(int32_t),
                           cudaMemcpyDeviceToHost, s));
  H2D_CUDA(cudaFreeAsync(d_tmp, s));
  H2D_CUDA(cudaFreeAsync(d_codes, s));
  H2D_CUDA(cudaFreeAsync(d_codes_sorted, s));
  H2D_CUDA(cudaFreeAsync(d_idx, s));
  H2D_CUDA(cudaFreeAsync(d_out, s));
  H2D_CUDA(cudaStreamSynchronize(s));
}

// Adaptive quadtree (R24): subdivided flags top-down from the box counts of the deepest
// Morton order (the tree above is built at R22's depth, the deepest adaptive level), then the
// leaves (existing, unsubdivided boxes) in Morton order of their first level-kappa
// descendant.  Host work on 4^l flags per level.
void build_adaptive(Handle& h) {
  const int kappa = h.kappa;
  const int nmax = h.leaf_size;
  h.ad_sub.assign((size_t)kappa + 1, {});
  for (int l = 0; l <= kappa; ++l) {
    const int64_t nb = (int64_t)1 << (2 * l);
    h.ad_sub[(size_t)l].assign((size_t)nb, 0);
    if (l == kappa) break;
    for (int64_t b = 0; b < nb; ++b)
      if (h.box_exists(l, b) && h.box_end(l, b) - h.box_begin(l, b) > nmax) h.ad_sub[(size_t)l][(size_t)b] = 1;
  }
  h.lf_code.clear();
  h.lf_level.clear();
  h.lf_start.clear();
  // depth-first in Morton order = ascending first descendant
  std::vector<std::pair<int, int64_t>> stack{{0, 0}};
  while (!stack.empty()) {
    const auto [l, b] = stack.back();
    stack.pop_back();
    if (l < kappa && h.ad_sub[(size_t)l][(size_t)b]) {
      for (int c = 3; c >= 0; --c) stack.push_back({l + 1, (b << 2) | c});
      continue;
    }
    h.lf_code.push_back(b << (2 * (kappa - l)));
    h.lf_level.push_back(l);
    h.lf_start.push_back((int32_t)h.box_begin(l, b));
  }
  h.lf_start.push_back((int32_t)h.n);
}

// The adaptive near field (R24): dense blocks (X, Y), Y in {X} u E_X, of existing boxes at any
// level with X or Y a leaf; every leaf collects the column ranges of the blocks whose row box
// contains it (its own and its subdivided ancestors' mixed blocks), so each row has one
// writer and each (i, j) of a dense block is evaluated once for row i.
void build_adaptive_near(Handle& h) {
  const int kappa = h.kappa;
  const int64_t nlf = (int64_t)h.lf_code.size();
  h.ad_nf_off.assign((size_t)nlf + 1, 0);
  h.ad_nf_rng.clear();
  auto leaf = [&](int l, int64_t b) { return l == kappa || !h.ad_sub[(size_t)l][(size_t)b]; };
  for (int64_t lf = 0; lf < nlf; ++lf) {
    h.ad_nf_off[(size_t)lf] = (int64_t)h.ad_nf_rng.size() / 2;
    const int ll = h.lf_level[(size_t)lf];
    const int64_t code = h.lf_code[(size_t)lf];
    for (int l = 0; l <= ll; ++l) {
      const int64_t X = code >> (2 * (kappa - l));
      const uint32_t cx = compact_bits((uint32_t)X), cy = compact_bits((uint32_t)(X >> 1));
      const int64_t side = (int64_t)1 << l;
      // {X} u E_X in ascending Morton order
      int64_t cand[5];
      int nc = 0;
      const int dxs[5] = {0, -1, 1, 0, 0}, dys[5] = {0, 0, 0, -1, 1};
      for (int k = 0; k < 5; ++k) {
        const int64_t qx = (int64_t)cx + dxs[k], qy = (int64_t)cy + dys[k];
        if (qx < 0 || qy < 0 || qx >= side || qy >= side) continue;
        cand[nc++] = (int64_t)(spread_bits((uint32_t)qx) | (spread_bits((uint32_t)qy) << 1));
      }
      std::sort(cand, cand + nc);
      for (int k = 0; k < nc; ++k) {
        const int64_t Y = cand[k];
        if (!h.box_exists(l, Y) || (!leaf(l, X) && !leaf(l, Y))) continue;
        const int64_t c0 = h.box_begin(l, Y), cnt = h.box_end(l, Y) - c0;
        if (cnt == 0) continue;
        h.ad_nf_rng.push_back(c0);
        h.ad_nf_rng.push_back(cnt);
      }
    }
  }
  h.ad_nf_off[(size_t)nlf] = (int64_t)h.ad_nf_rng.size() / 2;
  h.d_ad_nf_off = h.alloc<int64_t>(h.ad_nf_off.size());
  h.d_ad_nf_rng = h.alloc<int64_t>(std::max<size_t>(1, h.ad_nf_rng.size()));
  h.d_lf_start = h.alloc<int32_t>(h.lf_start.size());
  H2D_CUDA(cudaMemcpy(h.d_ad_nf_off, h.ad_nf_off.data(), h.ad_nf_off.size() * 8, cudaMemcpyHostToDevice));
  if (!h.ad_nf_rng.empty())
    H2D_CUDA(cudaMemcpy(h.d_ad_nf_rng, h.ad_nf_rng.data(), h.ad_nf_rng.size() * 8, cudaMemcpyHostToDevice));
  H2D_CUDA(cudaMemcpy(h.d_lf_start, h.lf_start.data(), h.lf_start.size() * 4, cudaMemcpyHostToDevice));
}

void build_lists(Handle& h) {
  h.levels.assign((size_t)h.kappa + 1, Level());
  for (int l = 1; l <= h.kappa; ++l) {
    Level& L = h.levels[(size_t)l];
    L.l = l;
    L.nbox = (int64_t)1 << (2 * l);
    make_csr(h, l, 0, L.d_off, L.d_col, L.off, L.col);
    if (h.adaptive) {   // R24: Eq. eq:ilist restricted to existing boxes
      std::vector<int32_t> off((size_t)L.nbox + 1, 0), col;
      col.reserve(L.col.size());
      for (int64_t X = 0; X < L.nbox; ++X) {
        off[(size_t)X] = (int32_t)col.size();
        if (!h.box_exists(l, X)) continue;
        for (int32_t e = L.off[(size_t)X]; e < L.off[(size_t)X + 1]; ++e)
          if (h.box_exists(l, L.col[(size_t)e])) col.push_back(L.col[(size_t)e]);
      }
      off[(size_t)L.nbox] = (int32_t)col.size();
      L.off.swap(off);
      L.col.swap(col);
      h.release(L.d_col);
      L.d_col = h.alloc<int32_t>(std::max<size_t>(1, L.col.size()));
      H2D_CUDA(cudaMemcpy(L.d_off, L.off.data(), L.off.size() * 4, cudaMemcpyHostToDevice));
      if (!L.col.empty()) H2D_CUDA(cudaMemcpy(L.d_col, L.col.data(), L.col.size() * 4, cudaMemcpyHostToDevice));
    }
    L.nblocks = L.off[(size_t)L.nbox];
    // transpose map: block (X, Y) -> block (Y, X) (the relation is symmetric)
    L.trans.assign((size_t)L.nblocks, -1);
    for (int64_t X = 0; X < L.nbox; ++X)
      for (int32_t e = L.off[(size_t)X]; e < L.off[(size_t)X + 1]; ++e) {
        int32_t Y = L.col[(size_t)e];
        const int32_t* b = L.col.data() + L.off[(size_t)Y];
        const int32_t* en = L.col.data() + L.off[(size_t)Y + 1];
        const int32_t* it = std::lower_bound(b, en, (int32_t)X);
        if (it == en || *it != (int32_t)X) throw Error{H2D_ECUDA, "interaction lists not symmetric"};
        L.trans[(size_t)e] = (int32_t)(it - L.col.data());
      }
  }
  make_csr(h, h.kappa, 1, h.d_nf_off, h.d_nf_col, h.nf_off, h.nf_col);
}

}  // namespace h2d
