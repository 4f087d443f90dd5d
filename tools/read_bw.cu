// Pure-read HBM bandwidth microbenchmark (the practical ceiling of a read-only factor
// stream, beside the driver's copy bandwidth in MEASURED_PEAKS.json, which moves read +
// write bytes): 16-byte loads (ld.global.cs), grid-stride, 148 x k CTAs x 256 threads over
// an 8 GB buffer (>> L2), best of 10 with CUDA events; also a 16 KB-per-request bulk-TMA
// variant is NOT included (the product kernels are measured directly by bench.py / ncu).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/read_bw tools/read_bw.cu
#include <cuda_runtime.h>

#include <cstdio>

__global__ void read_kernel(const double2* __restrict__ a, size_t n, double* out) {
  double s0 = 0.0, s1 = 0.0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    const double2 v0 = __ldcs(a + i), v1 = __ldcs(a + i + stride), v2 = __ldcs(a + i + 2 * stride),
                  v3 = __ldcs(a + i + 3 * stride);
    s0 += (v0.x + v1.x) + (v2.x + v3.x);
    s1 += (v0.y + v1.y) + (v2.y + v3.y);
  }
  for (; i < n; i += stride) {
    const double2 v = __ldcs(a + i);
    s0 += v.x;
    s1 += v.y;
  }
  if (s0 + s1 == 12345.678) *out = s0;   // keeps the loads
}

int main() {
  const size_t bytes = 8ull << 30, n = bytes / sizeof(double2);
  double2* a;
  double* out;
  cudaMalloc(&a, bytes);
  cudaMalloc(&out, 8);
  cudaMemset(a, 0, bytes);
  int sm = 0;
  cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("{\"bytes\": %zu, \"results\": [", bytes);
  const int ks[] = {2, 4, 8, 16};
  for (int q = 0; q < 4; ++q) {
    const int blocks = sm * ks[q];
    read_kernel<<<blocks, 256>>>(a, n, out);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) {
      cudaEventRecord(e0);
      read_kernel<<<blocks, 256>>>(a, n, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("%s{\"ctas_per_sm\": %d, \"ms\": %.4f, \"read_gbs\": %.1f}", q ? ", " : "", ks[q], best,
           bytes / (best * 1e-3) / 1e9);
  }
  printf("], \"error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
