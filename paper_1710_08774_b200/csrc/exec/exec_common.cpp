// Host helpers shared by the executors: TMA descriptor encoding through the
// runtime's driver entry point, CUDA error mapping.
#include <algorithm>
#include <vector>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "exec.hpp"

namespace lfx {

int cuda_status(cudaError_t e, const char* what, std::string& err) {
  if (e == cudaSuccess) return LF_OK;
  err = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return LF_ERR_CUDA;
}

int resident_slots(LaunchCache& cache, const void* kernel, int threads, int smem, int occ_cap, const char* what,
                   int* slots, std::string& err) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_status(e, "cudaGetDevice", err);
  if (dev < 0 || dev >= kMaxDevices) {
    err = "device ordinal out of range";
    return LF_ERR_CUDA;
  }
  std::call_once(cache.once[dev], [&] {
    cudaError_t x = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int sms = 148, per_sm = 1;
    if (x == cudaSuccess) x = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (x == cudaSuccess) x = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
    per_sm = std::max(1, occ_cap > 0 ? std::min(per_sm, occ_cap) : per_sm);
    cache.slots[dev] = sms * per_sm;
    cache.err[dev] = x;
  });
  if (cache.err[dev] != cudaSuccess) return cuda_status(cache.err[dev], what, err);
  *slots = cache.slots[dev];
  return LF_OK;
}

static bool band_guard_on() {
  const char* e = option("LF_BAND_GUARD");
  return e && std::atoi(e) != 0;
}

int band_memory(ExecMem& mem, size_t need, cudaStream_t stream, void** ptr, std::string& err) {
  const bool guard = band_guard_on();
  cudaError_t e = mem.ensure(need + (guard ? 2 * kBandGuard : 0));
  if (e != cudaSuccess) return cuda_status(e, "cudaMalloc(in-place bands)", err);
  char* base = static_cast<char*>(mem.ptr);
  if (guard) {  // canary bytes 0xA5 either side of the executor's range
    e = cudaMemsetAsync(base, 0xA5, kBandGuard, stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(base + kBandGuard + need, 0xA5, kBandGuard, stream);
    if (e != cudaSuccess) return cuda_status(e, "cudaMemsetAsync(band guard)", err);
    base += kBandGuard;
    // LF_BAND_GUARD=2 (fault injection, tests): hand the executor a range that
    // ends 64 bytes inside the rear guard, so a store to its last bytes is caught
    if (std::atoi(option("LF_BAND_GUARD")) == 2) base += 64;
  }
  *ptr = base;
  return LF_OK;
}

int band_guard_check(const ExecMem& mem, size_t need, cudaStream_t stream, std::string& err) {
  if (!band_guard_on()) return LF_OK;
  std::vector<unsigned char> h(2 * kBandGuard);
  const char* base = static_cast<const char*>(mem.ptr);
  cudaError_t e = cudaStreamSynchronize(stream);
  if (e == cudaSuccess) e = cudaMemcpy(h.data(), base, kBandGuard, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(h.data() + kBandGuard, base + kBandGuard + need, kBandGuard, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_status(e, "band guard read-back", err);
  for (size_t i = 0; i < h.size(); ++i)
    if (h[i] != 0xA5) {
      err = "in-place band store outside its buffer (guard byte " + std::to_string(i % kBandGuard) +
            (i < kBandGuard ? " before" : " after") + " the bands)";
      return LF_ERR_INTERNAL;
    }
  return LF_OK;
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool make_tensor_map(CUtensorMap* map, const void* base, CUtensorMapDataType dtype, int elem_bytes, int rank,
                     const uint64_t* dims, const uint32_t* box, std::string& err) {
  auto fn = encode_fn();
  if (!fn) {
    err = "cuTensorMapEncodeTiled unavailable from the CUDA driver";
    return false;
  }
  cuuint64_t gdim[5];
  cuuint64_t gstride[4];
  cuuint32_t bdim[5], estride[5];
  uint64_t acc = static_cast<uint64_t>(elem_bytes);
  for (int d = 0; d < rank; ++d) {
    gdim[d] = dims[d];
    bdim[d] = box[d];
    estride[d] = 1;
    if (d > 0) gstride[d - 1] = acc;
    acc *= dims[d];
  }
  // L2 sector promotion of TMA fetches; LF_TMA_PROMOTION=0/64/128/256 overrides
  // the default for tuning runs
  const CUtensorMapL2promotion promo = [] {
    const char* e = lfx::option("LF_TMA_PROMOTION");
    const int v = e ? std::atoi(e) : 256;
    return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                  : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                            : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }();
  CUresult r = fn(map, dtype, rank, const_cast<void*>(base), gdim, gstride, bdim, estride,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    err = "cuTensorMapEncodeTiled failed with CUresult " + std::to_string(static_cast<int>(r));
    return false;
  }
  return true;
}

}  // namespace lfx
