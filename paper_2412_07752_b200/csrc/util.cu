// util.cu -- small device utilities used by the ABI layer.
#include <cuda_bf16.h>

#include "kernels.h"

namespace frnn {
namespace {

template <class T>
__global__ void finite_kernel(const T* p, size_t n, int* flag) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float v;
    if constexpr (sizeof(T) == 2)
      v = __bfloat162float(p[i]);
    else
      v = p[i];
    if (!isfinite(v)) {
      *flag = 1;
      return;
    }
  }
}

}  // namespace

// engine.hpp:131-135 check_finite, on the device.
cudaError_t check_finite(const void* ptr, size_t n, bool bf16, int* flag, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  int grid = (int)std::min<size_t>((n + 255) / 256, (size_t)sm_count() * 8);
  if (bf16)
    finite_kernel<<<grid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(ptr), n, flag);
  else
    finite_kernel<<<grid, 256, 0, s>>>(static_cast<const float*>(ptr), n, flag);
  note_launch();
  return cudaGetLastError();
}

int sm_count() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 1;
}

}  // namespace frnn
