// hostutil.cu -- host helpers shared by the kernel launchers: the TMA tensor-map encoder,
// the per-device opt-in to > 48 KB of dynamic shared memory, the SM count of the current
// device, and (testing build only) the device-side lens range counters.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>
#include <set>
#include <utility>

#include "internal.h"

namespace hydra {

static PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool tensor_maps_available() { return encoder() != nullptr; }

bool encode_bf16_map(void *map, int rank, const void *base, const uint64_t *dims, const uint64_t *strides_bytes,
                     const uint32_t *box) {
  auto fn = encoder();
  if (!fn || rank < 1 || rank > 5) return false;
  cuuint64_t d[5], s[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    e[i] = 1;
    if (i + 1 < rank) s[i] = strides_bytes[i];
  }
  return fn(reinterpret_cast<CUtensorMap *>(map), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, (cuuint32_t)rank,
            const_cast<void *>(base), d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// The opt-in is a per-device function attribute: cached per (kernel, device), so a process
// that drives several GPUs sets it once on each.
cudaError_t ensure_smem_attr(const void *func, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void *, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({func, dev})) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.insert({func, dev});
  return e;
}

int device_sm_count() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

#ifdef HYDRA_TESTING
// Debug check of the documented precondition 0 <= lens[b] <= S_cap (hydra.h): counted on
// the device, read back by hydra_debug_lens_violations.  The release kernels clamp instead.
__device__ unsigned long long g_lens_violations;

__global__ void lens_check_kernel(const int32_t *lens, int64_t B, int64_t S_cap) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < B; b += (int64_t)gridDim.x * blockDim.x)
    if (lens[b] < 0 || lens[b] > S_cap) atomicAdd(&g_lens_violations, 1ull);
}

hydra_status launch_lens_check(const int32_t *lens, int64_t B, int64_t S_cap, cudaStream_t s) {
  if (B <= 0 || !lens) return HYDRA_OK;
  const int blocks = (int)std::min<int64_t>((B + 255) / 256, 1024);
  lens_check_kernel<<<blocks, 256, 0, s>>>(lens, B, S_cap);
  return cudaGetLastError() == cudaSuccess ? HYDRA_OK : HYDRA_ECUDA;
}

int64_t read_lens_violations(bool reset) {
  unsigned long long v = 0;
  if (cudaDeviceSynchronize() != cudaSuccess) return -2;
  if (cudaMemcpyFromSymbol(&v, g_lens_violations, sizeof v) != cudaSuccess) return -2;
  if (reset) {
    const unsigned long long z = 0;
    cudaMemcpyToSymbol(g_lens_violations, &z, sizeof z);
  }
  return (int64_t)v;
}
#else
hydra_status launch_lens_check(const int32_t *, int64_t, int64_t, cudaStream_t) { return HYDRA_OK; }
int64_t read_lens_violations(bool) { return -1; }
#endif

}  // namespace hydra
