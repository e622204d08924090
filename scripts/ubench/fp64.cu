// Microbenchmark: FP64 DFMA latency / throughput and rsqrt latency on this GPU (clock64 cycles).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, double a, double b, int n, long long* cyc) {
  double x = threadIdx.x * 1e-9 + 1.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_rsq(double* out, int n, long long* cyc) {
  double x = threadIdx.x * 1e-9 + 1.3;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = rsqrt(x) + 0.5; }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void thr(double* out, double a, double b, int n, long long* cyc) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1 << 24); cudaMallocManaged(&cyc, 1024 * 8);
  const int n = 4096;
  lat<<<1, 32>>>(out, 0.999, 1e-3, n, cyc); cudaDeviceSynchronize();
  lat<<<1, 32>>>(out, 0.999, 1e-3, n, cyc); cudaDeviceSynchronize();
  printf("DFMA dependent latency: %.2f cycles\n", (double)cyc[0] / (4.0 * n));
  lat_rsq<<<1, 32>>>(out, n, cyc); cudaDeviceSynchronize();
  lat_rsq<<<1, 32>>>(out, n, cyc); cudaDeviceSynchronize();
  printf("rsqrt + add dependent latency: %.2f cycles\n", (double)cyc[0] / n);
  for (int warps = 1; warps <= 32; warps *= 2) {
    thr<<<1, 32 * warps>>>(out, 0.999, 1e-3, n, cyc); cudaDeviceSynchronize();
    thr<<<1, 32 * warps>>>(out, 0.999, 1e-3, n, cyc); cudaDeviceSynchronize();
    printf("warps %2d x 8 chains: %.3f warp-DFMA per cycle per SM\n", warps, 8.0 * n * warps / (double)cyc[0]);
  }
  // device-wide DFMA throughput (wall time, CUDA events): 4 CTAs x 512 threads per SM, 8 chains each
  int dev = 0, nsm = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const int nbig = 1 << 16, grid = 4 * nsm;
  long long* cyc2; cudaMalloc(&cyc2, grid * 8);
  double* out2; cudaMalloc(&out2, (size_t)grid * 512 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  thr<<<grid, 512>>>(out2, 0.999, 1e-3, nbig, cyc2);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    thr<<<grid, 512>>>(out2, 0.999, 1e-3, nbig, cyc2);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flop = 2.0 * 8.0 * nbig * (double)grid * 512;
  printf("{\"fp64_tflops\": %.3f, \"sms\": %d, \"max_clock_mhz\": %d, \"ms\": %.3f, \"how\": \"%d CTAs x 512 threads x 8 "
         "independent DFMA chains x %d iterations, best of 5, CUDA events\"}\n",
         flop / (best * 1e-3) / 1e12, nsm, clk / 1000, best, grid, nbig);
  return 0;
}
