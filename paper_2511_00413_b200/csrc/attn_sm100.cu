// attn_sm100.cu — device capability check for the sm_100a tensor-core attention path (bf16, d = 128).
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
