// Tuning probe (not product code): attainable HBM bandwidth of the access
// patterns the row-marching executors use, next to a plain linear copy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/stream_probe tools/stream_probe.cu
//   tools/stream_probe [N]      (N x N fp64 grid with a 2-cell ghost ring, pitch N + 4)
// Patterns: linear copy of the whole buffer; strip marching (one warp per CTA,
// 32*CPL columns per strip, contiguous row ranges per CTA) with the output
// shifted by the 2-cell ghost offset or aligned, plain or evict-first stores.
#include <cstdio>
#include <cstdlib>
#include <cstdint>

#include <cuda_runtime.h>

__global__ void copy_linear(const double2* __restrict__ in, double2* __restrict__ out, long long n2) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x)
    out[i] = __ldg(in + i);
}

template <int CPL, bool EF>
__global__ void __launch_bounds__(32) copy_strips(const double* __restrict__ in, double* __restrict__ out, int n,
                                                  long long pitch, int strips, int out_shift) {
  const int lane = threadIdx.x;
  const long long total = (long long)strips * n;
  long long a = total * blockIdx.x / gridDim.x, b = total * (blockIdx.x + 1) / gridDim.x;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  while (a < b) {
    const int s = (int)(a / n);
    const long long end = b < (long long)(s + 1) * n ? b : (long long)(s + 1) * n;
    const int jb = (int)(a - (long long)s * n), je = (int)(end - (long long)s * n);
    for (int j = jb; j < je; ++j) {
      const double* src = in + (long long)(j + 2) * pitch + 2 + (long long)s * 32 * CPL + CPL * lane;
      double* dst = out + (long long)(j + 2) * pitch + out_shift + (long long)s * 32 * CPL + CPL * lane;
#pragma unroll
      for (int h = 0; h < CPL / 2; ++h) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(src) + h);
        if (EF)
          asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(dst + 2 * h), "d"(v.x), "d"(v.y),
                       "l"(pol)
                       : "memory");
        else
          *reinterpret_cast<double2*>(dst + 2 * h) = v;
      }
    }
    a = end;
  }
}

// NW warps per CTA marching NW adjacent sub-strips of 32*CPL columns in lockstep
template <int CPL, int NW>
__global__ void __launch_bounds__(32 * NW) copy_strips_nw(const double* __restrict__ in, double* __restrict__ out,
                                                          int n, long long pitch, int strips, int out_shift) {
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
  const long long total = (long long)strips * n;
  long long a = total * blockIdx.x / gridDim.x, b = total * (blockIdx.x + 1) / gridDim.x;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  while (a < b) {
    const int s = (int)(a / n);
    const long long end = b < (long long)(s + 1) * n ? b : (long long)(s + 1) * n;
    const int jb = (int)(a - (long long)s * n), je = (int)(end - (long long)s * n);
    for (int j = jb; j < je; ++j) {
      const long long col = (long long)s * 32 * CPL * NW + wq * 32 * CPL + CPL * lane;
      const double* src = in + (long long)(j + 2) * pitch + 2 + col;
      double* dst = out + (long long)(j + 2) * pitch + out_shift + col;
#pragma unroll
      for (int h = 0; h < CPL / 2; ++h) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(src) + h);
        asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(dst + 2 * h), "d"(v.x), "d"(v.y),
                     "l"(pol)
                     : "memory");
      }
    }
    a = end;
  }
}

template <class F>
float time_ms(F f, int reps = 10) {
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(s);
  for (int r = 0; r < reps; ++r) f();
  cudaEventRecord(e);
  cudaEventSynchronize(e);
  float ms = 0;
  cudaEventElapsedTime(&ms, s, e);
  return ms / reps;
}

template <int CPL, bool EF>
void strips(const double* in, double* out, int n, long long pitch, int occ, int shift, int sms) {
  const int nstrips = n / (32 * CPL);
  int ctas = sms * occ;
  if (ctas >= nstrips) ctas = ctas / nstrips * nstrips;
  const float ms = time_ms([&] { copy_strips<CPL, EF><<<ctas, 32>>>(in, out, n, pitch, nstrips, shift); });
  const double bytes = 2.0 * 8.0 * n * (double)n;
  printf("strips cpl=%d ef=%d occ=%2d shift=%d: %8.1f GB/s (%.3f ms)\n", CPL, EF, occ, shift, bytes / ms * 1e-6, ms);
}

template <int CPL, int NW>
void strips_nw(const double* in, double* out, int n, long long pitch, int occ, int sms) {
  const int nstrips = n / (32 * CPL * NW);
  int ctas = sms * occ;
  if (ctas >= nstrips) ctas = ctas / nstrips * nstrips;
  const float ms = time_ms([&] { copy_strips_nw<CPL, NW><<<ctas, 32 * NW>>>(in, out, n, pitch, nstrips, 2); });
  const double bytes = 2.0 * 8.0 * n * (double)n;
  printf("strips cpl=%d nw=%d occ=%2d (CTAs/SM): %8.1f GB/s (%.3f ms)\n", CPL, NW, occ, bytes / ms * 1e-6, ms);
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 16384;
  const long long pitch = n + 4;
  const long long elems = pitch * (n + 4);
  double *in, *out;
  cudaMalloc(&in, elems * 8);
  cudaMalloc(&out, elems * 8);
  cudaMemset(in, 0, elems * 8);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long n2 = elems / 2;
  const float ms = time_ms([&] {
    copy_linear<<<sms * 8, 256>>>(reinterpret_cast<const double2*>(in), reinterpret_cast<double2*>(out), n2);
  });
  printf("linear copy: %8.1f GB/s (%.3f ms, %lld B)\n", 2.0 * elems * 8 / ms * 1e-6, ms, elems * 8);
  for (int occ : {4, 6, 8, 12}) {
    strips_nw<2, 2>(in, out, n, pitch, occ, sms);
    strips_nw<2, 4>(in, out, n, pitch, occ / 2 > 0 ? occ / 2 : 1, sms);
    strips_nw<4, 2>(in, out, n, pitch, occ, sms);
  }
  for (int occ : {8, 12, 16, 24}) {
    strips<2, true>(in, out, n, pitch, occ, 2, sms);
    strips<2, true>(in, out, n, pitch, occ, 0, sms);
    strips<2, false>(in, out, n, pitch, occ, 2, sms);
    strips<4, true>(in, out, n, pitch, occ, 2, sms);
    strips<8, true>(in, out, n, pitch, occ, 2, sms);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
