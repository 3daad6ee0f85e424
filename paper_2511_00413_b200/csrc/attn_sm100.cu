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

tt_status sm100_attn_bwd(const tt_packed& pk, const void* q, const void* k, const void* v, const float* lse,
                         const float* Dvec, const void* dout, int restore, int hq, int hkv, int d, float scale,
                         float* dq_acc, void* dq, void* dk, void* dv, cudaStream_t st) {
  (void)dq_acc;
  return simt_attn_bwd(pk, q, k, v, lse, Dvec, dout, restore, TT_BF16, hq, hkv, d, scale, dq, dk, dv, st);
}

}  // namespace tt
