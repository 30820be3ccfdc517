// Latency probe (measurement tool, not product code): cycles per dependent
// fp64 op / fast-path sqrt / division / MUFU seed on one warp, and the
// throughput of independent DFMA chains per SM at several chain counts.
#include <cstdio>
#include "../../paper_1710_08774_b200/csrc/exec/fastmath.cuh"
using namespace lfx;

__global__ void lat(double* out, long long* cyc, double x0, int n) {
  double x = x0, y = x0 * 0.5;
  unsigned bad = 0;
  long long t0, t1;
  // 1. dependent DFMA
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __fma_rn(x, 0.999999, 1e-7);
  t1 = clock64();
  cyc[0] = t1 - t0;
  // 2. dependent DADD
  t0 = clock64();
  for (int i = 0; i < n; ++i) y = __dadd_rn(y, 1e-9);
  t1 = clock64();
  cyc[1] = t1 - t0;
  // 3. dependent fast sqrt
  double s = x + 2.0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) s = lf_sqrt_fast(s + 1.5, &bad);
  t1 = clock64();
  cyc[2] = t1 - t0;
  // 4. dependent fast division
  double d = y + 3.0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) d = lf_div_fast(d, 0.9999999, &bad) + 0.5;
  t1 = clock64();
  cyc[3] = t1 - t0;
  // 5. dependent MUFU.RSQ64H seed
  double m = 2.0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double r;
    asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(m));
    m = r + 1.0;
  }
  t1 = clock64();
  cyc[4] = t1 - t0;
  out[threadIdx.x] = x + y + s + d + m + bad;
}

template <int C>
__global__ void thr(double* out, int n) {
  double a[C];
#pragma unroll
  for (int c = 0; c < C; ++c) a[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int c = 0; c < C; ++c) a[c] = __fma_rn(a[c], 0.9999999, 1e-7);
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int C>
void run_thr(double* d, int warps_per_sm) {
  int sms = 148, n = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  thr<C><<<sms, 32 * warps_per_sm>>>(d, n);
  cudaEventRecord(e0);
  thr<C><<<sms, 32 * warps_per_sm>>>(d, n);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double tf = 2.0 * sms * 32.0 * warps_per_sm * C * (double)n / (ms * 1e-3) / 1e12;
  printf("DFMA chains/thread %d, warps/SM %2d (chains per SMSP %3d): %.2f TFLOP/s\n", C, warps_per_sm,
         C * warps_per_sm / 4, tf);
}

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 1 << 24);
  cudaMallocManaged(&c, 64);
  const int n = 1024;
  lat<<<1, 32>>>(d, c, 1.0, n);
  cudaDeviceSynchronize();
  lat<<<1, 32>>>(d, c, 1.0, n);
  cudaDeviceSynchronize();
  const char* names[] = {"DFMA", "DADD", "sqrt fast path (+DADD)", "div fast path (+DADD)", "MUFU.RSQ64H (+DADD)"};
  for (int k = 0; k < 5; ++k) printf("latency %-24s %.1f cycles\n", names[k], (double)c[k] / n);
  for (int w : {4, 8, 12, 16, 24, 32}) {
    run_thr<1>(d, w);
    run_thr<2>(d, w);
    run_thr<4>(d, w);
  }
  return 0;
}
