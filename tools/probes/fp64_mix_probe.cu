// Measurement tool (not product code): fp64-pipe throughput of instruction
// forms other than the DFMA-with-uniform-operands chain of tools/fp64_probe.cu:
// three register sources, DMUL, DADD, a DFMA/DMUL/DADD mix like the Riemann
// solver's, and 12 vs 8 warps per SM.  Prints fp64 warp-instructions per clock
// per SM (the DFMA peak is 2.0).
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 12;  // live values per thread
template <int MODE>
__global__ void __launch_bounds__(128) k(double* out, int iters, double a, double b) {
  double x[N];
#pragma unroll
  for (int c = 0; c < N; ++c) x[c] = threadIdx.x * 1e-9 + c + a;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < N; ++c) {
      if (MODE == 0) x[c] = fma(x[c], a, b);                           // 1 register + 2 uniform sources
      if (MODE == 1) x[c] = fma(x[(c + 1) % N], x[(c + 5) % N], x[c]);  // 3 register sources
      if (MODE == 2) x[c] = x[(c + 1) % N] * x[c];                      // DMUL, 2 registers
      if (MODE == 3) x[c] = x[(c + 1) % N] + x[c];                      // DADD, 2 registers
      if (MODE == 4) {                                                  // mix: 2 DFMA (3 regs) + DMUL + DADD
        if (c % 4 < 2) x[c] = fma(x[(c + 1) % N], x[(c + 5) % N], x[c]);
        else if (c % 4 == 2) x[c] = x[(c + 1) % N] * x[c];
        else x[c] = x[(c + 7) % N] + x[c];
      }
      if (MODE == 5) x[c] = fma(x[(c + 1) % N], a, x[c]);               // 2 registers + 1 uniform
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < N; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

template <int MODE>
void run(const char* name, int warps_per_sm, double* out, int sms, double mhz) {
  const int iters = 2048, threads = 128, blocks = sms * (warps_per_sm / 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<MODE><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k<MODE><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double winst = (double)N * iters * blocks * (threads / 32);
  const double clk = best * 1e-3 * mhz * 1e6;
  printf("%-34s %2d warps/SM: %.3f fp64 warp-inst/clk/SM (%.1f %% of 2.0)\n", name, warps_per_sm, winst / clk / sms,
         50.0 * winst / clk / sms);
}

int main() {
  int sms = 0, khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  const double mhz = khz / 1e3;
  printf("SMs %d, clock %.0f MHz (max; rates assume it)\n", sms, mhz);
  double* out;
  cudaMalloc(&out, 8);
  for (int w : {8, 12, 32}) {
    run<0>("DFMA reg,uniform,uniform", w, out, sms, mhz);
    run<5>("DFMA reg,uniform,reg", w, out, sms, mhz);
    run<1>("DFMA reg,reg,reg", w, out, sms, mhz);
    run<2>("DMUL reg,reg", w, out, sms, mhz);
    run<3>("DADD reg,reg", w, out, sms, mhz);
    run<4>("mix 2 DFMA + DMUL + DADD (regs)", w, out, sms, mhz);
  }
  return cudaDeviceSynchronize() != cudaSuccess;
}
