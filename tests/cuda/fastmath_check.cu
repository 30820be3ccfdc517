// Test harness for csrc/exec/fastmath.cuh: the branch-free fast paths next to
// the native IEEE operations on the same operands (tests/test_gpu_fastmath.py).
#include <cuda_runtime.h>

#include "../../paper_1710_08774_b200/csrc/exec/fastmath.cuh"

__global__ void check(const double* a, const double* b, long long n, double* qf, double* qn, double* sf, double* sn,
                      double* rf, double* rn, unsigned* flags) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    unsigned bd = 0, bs = 0, br = 0;
    qf[i] = lfx::lf_div_fast(a[i], b[i], &bd);
    qn[i] = a[i] / b[i];
    sf[i] = lfx::lf_sqrt_fast(a[i], &bs);
    sn[i] = sqrt(a[i]);
    rf[i] = lfx::lf_rcp_fast(b[i], &br);
    rn[i] = 1.0 / b[i];
    flags[i] = bd | (bs << 1) | (br << 2);
  }
}

extern "C" int fastmath_check(const double* a, const double* b, long long n, double* qf, double* qn, double* sf,
                              double* sn, double* rf, double* rn, unsigned* flags) {
  check<<<592, 256>>>(a, b, n, qf, qn, sf, sn, rf, rn, flags);
  return (int)cudaDeviceSynchronize();
}

// lf_div3f / lf_div3f2 (userkernels/stencil_kernels.h) against x / 3.0f for
// every float bit pattern: counts the mismatches (NaN == NaN)
#include "../../paper_1710_08774_b200/userkernels/stencil_kernels.h"

__global__ void div3_all(unsigned long long* bad) {
  unsigned long long nb = 0;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x * 2;
  for (unsigned long long i = 2ull * (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x); i < (1ull << 32); i += stride) {
    const float x0 = __uint_as_float((unsigned)i), x1 = __uint_as_float((unsigned)(i + 1));
    const float ref0 = __fdiv_rn(x0, 3.0f), ref1 = __fdiv_rn(x1, 3.0f);
    const float s0 = lf_div3f(x0), s1 = lf_div3f(x1);
    const float2 p = lf_div3f2(make_float2(x0, x1));
    auto same = [](float a, float b) { return __float_as_uint(a) == __float_as_uint(b) || (a != a && b != b); };
    nb += !same(s0, ref0) + !same(s1, ref1) + !same(p.x, ref0) + !same(p.y, ref1);
  }
  atomicAdd(bad, nb);
}

extern "C" long long div3_exhaustive() {
  unsigned long long* d = nullptr;
  cudaMalloc(&d, sizeof *d);
  cudaMemset(d, 0, sizeof *d);
  div3_all<<<148 * 8, 256>>>(d);
  unsigned long long h = ~0ull;
  if (cudaMemcpy(&h, d, sizeof h, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  cudaFree(d);
  return (long long)h;
}
