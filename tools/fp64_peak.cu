// FP64 throughput microbenchmark for the roofline denominators the driver does not measure
// (MEASURED_PEAKS.json has HBM and bf16 only; SURVEY §8(d) asks for a measured FP64 peak):
//   dfma : CUDA-core DFMA, 8 independent chains per thread, 148 x 8 CTAs x 256 threads;
//   dmma : FP64 tensor core, mma.sync.m8n8k4.f64 (256 FMA per warp instruction), 8
//          independent accumulators per warp.
// Each kernel runs ~1 s of back-to-back work (sustained, under the power cap) timed with
// CUDA events; prints one JSON line.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cuda_runtime.h>

#include <cstdio>

__global__ void dfma_kernel(double* out, long iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
         x7 = x0 + 7;
  for (long i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void dmma_kernel(double* out, long iters, double a, double b) {
  double d[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = threadIdx.x + i;
  const double av = a + threadIdx.x * 1e-9, bv = b;
  for (long it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(d[i][0]), "+d"(d[i][1])
                   : "d"(av), "d"(bv));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sm = 0;
  cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sm * 8, threads = 256;
  double* out;
  cudaMalloc(&out, (size_t)blocks * threads * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](bool mma, long iters) {
    if (mma) dmma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    else dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
  };
  double res[2];
  for (int k = 0; k < 2; ++k) {
    const bool mma = k == 1;
    run(mma, 1000);   // warm-up
    cudaDeviceSynchronize();
    long iters = 1000;
    float ms = 0;
    for (;;) {   // grow to ~1 s
      cudaEventRecord(e0);
      run(mma, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms > 800 || iters > (1L << 40)) break;
      iters = (long)(iters * 1000.0 / (ms + 1e-3)) + 1;
    }
    // flops: dfma 2 * 8 chains * 16 unroll per thread-iteration; dmma 2 * 256 * 8 per warp-iteration
    const double flops = mma ? 2.0 * 256 * 8 * iters * (double)blocks * threads / 32
                             : 2.0 * 8 * 16 * iters * (double)blocks * threads;
    res[k] = flops / (ms * 1e-3) / 1e12;
  }
  cudaError_t err = cudaGetLastError();
  printf("{\"fp64_dfma_tflops\": %.3f, \"fp64_dmma_tflops\": %.3f, \"sms\": %d, \"error\": \"%s\", "
         "\"how\": \"tools/fp64_peak.cu: ~1 s sustained each, 148 x 8 CTAs x 256 threads; dfma 8 "
         "independent chains/thread, dmma m8n8k4 8 independent accumulators/warp; 1 FMA = 2 flops\"}\n",
         res[0], res[1], sm, cudaGetErrorString(err));
  return 0;
}
