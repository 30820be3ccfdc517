// Measurement tool (not product code): the B200's fp64 FMA-pipe throughput,
// measured live so the Hydro2D roofline has a measured denominator
// (MEASURED_PEAKS.json carries HBM and bf16 only).  Every thread runs 8
// independent DFMA chains; 2 flops per DFMA.
#include <cuda_runtime.h>

namespace {
constexpr int CHAINS = 8;
__global__ void __launch_bounds__(256) dfma_chains(double* out, int iters, double a, double b) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;  // keep the chains live
}
}  // namespace

// Returns 0 and the best-of-`reps` fp64 FMA throughput in TFLOP/s.
extern "C" int lf_probe_fp64_tflops(int reps, double* tflops) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out = nullptr;
  if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return 1;
  const int blocks = sms * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_chains<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);  // warm-up
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    dfma_chains<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (cudaGetLastError() != cudaSuccess) return 1;
  *tflops = 2.0 * CHAINS * (double)iters * blocks * threads / (best * 1e-3) / 1e12;
  return 0;
}
