// Restarted GMRES(m) on the HODLR2D operator: the iterative solver the paper accelerates
// with the fast matvec (§5: ACA tolerance 1e-12, "stopping criteria for GMRES is
// residual less than 1e-10 with restart ..."; RBF interpolation P:1020-1048; reading R20 in
// relative residual, x0 = 0, restart length a parameter).
//
// Every vector lives on the device in TREE order; one matvec (matvec_tree) per Arnoldi
// step; classical Gram-Schmidt with one reorthogonalisation (CGS2) as batched dot products
// (fixed-order reductions: the solve is bitwise reproducible) and a batched update; the
// (m+1) x m Hessenberg matrix, its Givens rotations and the back substitution live on the
// host (one small device->host copy per step).
#include <cmath>
#include <vector>

#include "h2d_internal.cuh"

namespace h2d {
namespace {

constexpr int kDotThreads = 256;
constexpr int64_t kDotChunk = 8192;   // rows per CTA of the partial dot products

// partial[k * nchunk + c] = sum_{i in chunk c} V_k[i] w[i], V_k = V + k * ldv.
__global__ void __launch_bounds__(kDotThreads)
mdot_partial_kernel(const double* __restrict__ V, int64_t ldv, const double* __restrict__ w, int64_t n,
                    int nchunk, double* __restrict__ partial) {
  __shared__ double red[kDotThreads];
  const int c = blockIdx.x, k = blockIdx.y, tid = threadIdx.x;
  const int64_t i0 = (int64_t)c * kDotChunk, i1 = min(n, i0 + kDotChunk);
  const double* __restrict__ v = V + (int64_t)k * ldv;
  double s0 = 0.0, s1 = 0.0;
  int64_t i = i0 + tid;
  for (; i + kDotThreads < i1; i += 2 * kDotThreads) {
    s0 = fma(v[i], w[i], s0);
    s1 = fma(v[i + kDotThreads], w[i + kDotThreads], s1);
  }
  if (i < i1) s0 = fma(v[i], w[i], s0);
  red[tid] = s0 + s1;
  __syncthreads();
  for (int o = kDotThreads / 2; o > 0; o >>= 1) {
    if (tid < o) red[tid] += red[tid + o];
    __syncthreads();
  }
  if (tid == 0) partial[(int64_t)k * nchunk + c] = red[0];
}

// out[k] = sum_c partial[k * nchunk + c] (one warp per k, fixed order).
__global__ void mdot_final_kernel(const double* __restrict__ partial, int nchunk, double* __restrict__ out) {
  const int k = blockIdx.x, lane = threadIdx.x;
  double s = 0.0;
  for (int c = lane; c < nchunk; c += 32) s += partial[(int64_t)k * nchunk + c];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[k] = s;
}

// w += alpha * sum_k V_k coef[k]
__global__ void vupdate_kernel(const double* __restrict__ V, int64_t ldv, int nvec,
                               const double* __restrict__ coef, double alpha, double* __restrict__ w,
                               int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < nvec; ++k) s = fma(V[(int64_t)k * ldv + i], coef[k], s);
    w[i] = fma(alpha, s, w[i]);
  }
}

// v = w / sqrt(*nrm2)
__global__ void normalize_kernel(const double* __restrict__ w, const double* __restrict__ nrm2,
                                 double* __restrict__ v, int64_t n) {
  const double inv = 1.0 / sqrt(*nrm2);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = w[i] * inv;
}

// r = b - y
__global__ void residual_kernel(const double* __restrict__ b, const double* __restrict__ y,
                                double* __restrict__ r, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    r[i] = b[i] - y[i];
}

// x[perm[s]] = xt[s] (TREE -> ORIGINAL order)
__global__ void permute_out_kernel(const double* __restrict__ xt, const int32_t* __restrict__ perm, int64_t n,
                                   double* __restrict__ x) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x)
    x[perm[s]] = xt[s];
}

struct GmresWork {
  Handle& h;
  cudaStream_t s;
  int64_t n;
  int nchunk, grid;
  double* partial;
  double* dres;   // device results of the dot products

  // out (device, nvec values) = V_k . w for k < nvec
  void mdot(const double* V, int64_t ldv, int nvec, const double* w, double* out) {
    mdot_partial_kernel<<<dim3(nchunk, nvec), kDotThreads, 0, s>>>(V, ldv, w, n, nchunk, partial);
    H2D_LAUNCH_CHECK();
    mdot_final_kernel<<<nvec, 32, 0, s>>>(partial, nchunk, out);
    H2D_LAUNCH_CHECK();
  }
  double norm2_host(const double* w) {
    mdot(w, 0, 1, w, dres);
    double v = 0.0;
    H2D_CUDA(cudaMemcpyAsync(&v, dres, sizeof(double), cudaMemcpyDeviceToHost, s));
    H2D_CUDA(cudaStreamSynchronize(s));
    return v;
  }
  void matvec(const double* xt, double* yt) { matvec_tree(h, xt, yt, H2D_ORDER_TREE, h.row_begin); }
};

}  // namespace

void gmres_solve(Handle& h, const double* d_b, double* d_x, double tol, int restart, int max_iter,
                 int* iters_out, double* relres_out) {
  if (h.row_begin != 0 || h.row_end != h.n) throw Error{H2D_EINVAL, "GMRES needs a single-rank handle"};
  if (!(tol > 0.0) || restart < 1 || max_iter < 1) throw Error{H2D_EINVAL, "bad GMRES parameters"};
  cudaStream_t s = h.stream;
  const int64_t n = h.n;
  const int m = restart;
  const int nchunk = (int)((n + kDotChunk - 1) / kDotChunk);
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  double *V = nullptr, *w = nullptr, *xt = nullptr, *bt = nullptr, *partial = nullptr, *dv = nullptr;
  H2D_CUDA(cudaMallocAsync(&V, (size_t)(m + 1) * n * sizeof(double), s));
  H2D_CUDA(cudaMallocAsync(&w, n * sizeof(double), s));
  H2D_CUDA(cudaMallocAsync(&xt, n * sizeof(double), s));
  H2D_CUDA(cudaMallocAsync(&bt, n * sizeof(double), s));
  H2D_CUDA(cudaMallocAsync(&partial, (size_t)(m + 2) * nchunk * sizeof(double), s));
  H2D_CUDA(cudaMallocAsync(&dv, (size_t)(3 * m + 8) * sizeof(double), s));
  struct Free {
    cudaStream_t s;
    std::vector<void*> p;
    ~Free() { for (void* q : p) cudaFreeAsync(q, s); }
  } guard{s, {V, w, xt, bt, partial, dv}};
  GmresWork G{h, s, n, nchunk, grid, partial, dv};
  double* h1 = dv;              // [m + 1]
  double* h2 = dv + (m + 1);    // [m + 1]
  double* hn = dv + 2 * (m + 1);
  double* ydev = dv + 2 * (m + 1) + 1;  // [m]
  permute_in(h, d_b, bt);
  H2D_CUDA(cudaMemsetAsync(xt, 0, n * sizeof(double), s));
  const double bnorm = std::sqrt(G.norm2_host(bt));
  int its = 0;
  double relres = 0.0;
  if (bnorm == 0.0) {
    H2D_CUDA(cudaMemsetAsync(d_x, 0, n * sizeof(double), s));
    if (iters_out) *iters_out = 0;
    if (relres_out) *relres_out = 0.0;
    return;
  }
  std::vector<double> H((size_t)(m + 1) * m), cs(m), sn(m), g(m + 1), y(m), hv(2 * (m + 1) + 1);
  auto Hij = [&](int i, int j) -> double& { return H[(size_t)j * (m + 1) + i]; };
  bool first = true;
  for (;;) {
    // r = b - A x (x0 = 0: r = b without a matvec)
    double* v0 = V;
    if (first) {
      H2D_CUDA(cudaMemcpyAsync(v0, bt, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    } else {
      G.matvec(xt, w);
      residual_kernel<<<grid, 256, 0, s>>>(bt, w, v0, n);
      H2D_LAUNCH_CHECK();
    }
    const double beta2 = G.norm2_host(v0);
    const double beta = std::sqrt(beta2);
    relres = beta / bnorm;
    if ((!first && relres < tol) || its >= max_iter || beta == 0.0) break;
    first = false;
    H2D_CUDA(cudaMemcpyAsync(hn, &beta2, sizeof(double), cudaMemcpyHostToDevice, s));
    normalize_kernel<<<grid, 256, 0, s>>>(v0, hn, v0, n);
    H2D_LAUNCH_CHECK();
    std::fill(H.begin(), H.end(), 0.0);
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    int k = 0;
    for (int j = 0; j < m; ++j) {
      const double* vj = V + (int64_t)j * n;
      double* vn = V + (int64_t)(j + 1) * n;
      G.matvec(vj, w);
      // CGS2: h1 = V^T w, w -= V h1, h2 = V^T w, w -= V h2
      G.mdot(V, n, j + 1, w, h1);
      vupdate_kernel<<<grid, 256, 0, s>>>(V, n, j + 1, h1, -1.0, w, n);
      H2D_LAUNCH_CHECK();
      G.mdot(V, n, j + 1, w, h2);
      vupdate_kernel<<<grid, 256, 0, s>>>(V, n, j + 1, h2, -1.0, w, n);
      H2D_LAUNCH_CHECK();
      G.mdot(w, 0, 1, w, hn);
      normalize_kernel<<<grid, 256, 0, s>>>(w, hn, vn, n);
      H2D_LAUNCH_CHECK();
      H2D_CUDA(cudaMemcpyAsync(hv.data(), dv, hv.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
      H2D_CUDA(cudaStreamSynchronize(s));
      for (int i = 0; i <= j; ++i) Hij(i, j) = hv[(size_t)i] + hv[(size_t)(m + 1 + i)];
      Hij(j + 1, j) = std::sqrt(hv[(size_t)(2 * (m + 1))]);
      for (int i = 0; i < j; ++i) {   // previous rotations
        const double t = cs[(size_t)i] * Hij(i, j) + sn[(size_t)i] * Hij(i + 1, j);
        Hij(i + 1, j) = -sn[(size_t)i] * Hij(i, j) + cs[(size_t)i] * Hij(i + 1, j);
        Hij(i, j) = t;
      }
      const double d = std::hypot(Hij(j, j), Hij(j + 1, j));
      cs[(size_t)j] = d > 0.0 ? Hij(j, j) / d : 1.0;
      sn[(size_t)j] = d > 0.0 ? Hij(j + 1, j) / d : 0.0;
      Hij(j, j) = d;
      Hij(j + 1, j) = 0.0;
      g[(size_t)j + 1] = -sn[(size_t)j] * g[(size_t)j];
      g[(size_t)j] = cs[(size_t)j] * g[(size_t)j];
      k = j + 1;
      ++its;
      if (std::fabs(g[(size_t)j + 1]) / bnorm < tol || its >= max_iter || d == 0.0) break;
    }
    // a zero diagonal (d == 0 without convergence: the Krylov space stopped growing and H is
    // singular there) would divide by zero: keep the columns before it (their least-squares
    // solution is still exact) and stop after this update
    bool singular = false;
    for (int i = 0; i < k; ++i)
      if (Hij(i, i) == 0.0) { k = i; singular = true; break; }
    for (int i = k - 1; i >= 0; --i) {   // back substitution
      double t = g[(size_t)i];
      for (int l = i + 1; l < k; ++l) t -= Hij(i, l) * y[(size_t)l];
      y[(size_t)i] = t / Hij(i, i);
    }
    if (k > 0) {
      H2D_CUDA(cudaMemcpyAsync(ydev, y.data(), k * sizeof(double), cudaMemcpyHostToDevice, s));
      vupdate_kernel<<<grid, 256, 0, s>>>(V, n, k, ydev, 1.0, xt, n);
      H2D_LAUNCH_CHECK();
    }
    if (singular) {   // true residual of the returned x, then stop (H2D_WNOCONV unless below tol)
      G.matvec(xt, w);
      residual_kernel<<<grid, 256, 0, s>>>(bt, w, v0, n);
      H2D_LAUNCH_CHECK();
      relres = std::sqrt(G.norm2_host(v0)) / bnorm;
      break;
    }
  }
  permute_out_kernel<<<grid, 256, 0, s>>>(xt, h.d_perm, n, d_x);
  H2D_LAUNCH_CHECK();
  H2D_CUDA(cudaStreamSynchronize(s));
  if (iters_out) *iters_out = its;
  if (relres_out) *relres_out = relres;
}

}  // namespace h2d
