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
