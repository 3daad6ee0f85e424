// attn_sm100.cu — placeholder dispatch for bf16 d=128 until the tcgen05 kernels land.
#include "tt_internal.cuh"

namespace tt {

bool sm100_available() {
  static int cached = -1;
  if (cached < 0) {
    int dev = 0, major = 0, minor = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    cached = (major == 10 && minor == 0) ? 1 : 0;
  }
  return cached == 1;
}

}  // namespace tt
