// attn_sm100.cu — device capability check for the sm_100a tensor-core attention path (bf16, d = 128)
// and the CTA-order choice the forward and backward share.
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

bool head_major_order(const tt_packed& pk, int hkv) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  if (pk.sched_sum_nq <= 0 || hkv <= 0) return false;
  return (double)sms * pk.sched_max_nq < 0.3 * (double)hkv * (double)pk.sched_sum_nq;
}

}  // namespace tt
