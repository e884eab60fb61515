// SM-resident 2-D time-tiling kernels (st_resident.cuh): R = 1, 2, 4.
#include "st_resident.cuh"

namespace st {

static void* resident_fn(int R, int fast) {
  switch (R) {
    case 1: return fast ? (void*)&resident2d_kernel<1, true> : (void*)&resident2d_kernel<1, false>;
    case 2: return fast ? (void*)&resident2d_kernel<2, true> : (void*)&resident2d_kernel<2, false>;
    case 4: return fast ? (void*)&resident2d_kernel<4, true> : (void*)&resident2d_kernel<4, false>;
  }
  return nullptr;
}

bool resident2d_supported(int R) { return resident_fn(R, 0) != nullptr; }

int launch_resident2d(int R, int fast, const KParams& p, int grid, int smem, void* stream) {
  void* fn = resident_fn(R, fast);
  if (!fn) return (int)cudaErrorInvalidDeviceFunction;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return (int)e;
  void* args[] = {(void*)&p};
  return (int)cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kResThreads), args, (size_t)smem,
                                          (cudaStream_t)stream);
}

}  // namespace st
