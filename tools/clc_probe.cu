// clc_probe.cu — which CTA does clusterlaunchcontrol.try_cancel hand out?  Development probe for the
// persistent attention kernels (DESIGN.md §5.2 / §5.3).  One CTA per SM (large dynamic shared memory);
// each CTA "works" on an item for a number of cycles proportional to a per-item weight, claims the next
// item with try_cancel a fixed time before its current item ends (or at its start: mode 1), and records
// (item, sm, start clock).  The host prints the order in which items started and the makespan against
// the greedy list schedule.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/clc_probe tools/clc_probe.cu && /tmp/clc_probe
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const int* weight, int* rec_item, int* rec_sm, long long* rec_t0, long long* rec_t1, int mode,
                      int unit) {
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(16) uint4 resp;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  sm[0] = 0;
  int smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  int x = blockIdx.x;
  uint32_t ph = 0;
  bool more = true;
  while (true) {
    const long long t0 = clock64();
    long long t_end = t0 + (long long)weight[x] * unit;
    const long long t_claim = mode == 1 ? t0 : t_end - 6 * unit;
    bool claimed = false;
    while (clock64() < t_end) {
      if (more && !claimed && clock64() >= t_claim) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16;" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("clusterlaunchcontrol.try_cancel.async.shared::cta.mbarrier::complete_tx::bytes.b128 [%0], [%1];" ::"r"(
                         smem_u32(&resp)),
                     "r"(smem_u32(&bar))
                     : "memory");
        claimed = true;
      }
    }
    rec_item[x] = x;
    rec_sm[x] = smid;
    rec_t0[x] = t0;
    rec_t1[x] = clock64();
    if (!more) break;
    if (!claimed) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16;" ::"r"(smem_u32(&bar)) : "memory");
      asm volatile("clusterlaunchcontrol.try_cancel.async.shared::cta.mbarrier::complete_tx::bytes.b128 [%0], [%1];" ::"r"(
                       smem_u32(&resp)),
                   "r"(smem_u32(&bar))
                   : "memory");
    }
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(smem_u32(&bar)),
        "r"(ph)
        : "memory");
    ph ^= 1;
    uint32_t nx = 0, ok = 0;
    asm volatile(
        "{\n.reg .pred p;\n.reg .b128 r;\nld.shared.b128 r, [%2];\n"
        "clusterlaunchcontrol.query_cancel.is_canceled.pred.b128 p, r;\nselp.u32 %1, 1, 0, p;\n"
        "@p clusterlaunchcontrol.query_cancel.get_first_ctaid::x.b32.b128 %0, r;\n}\n"
        : "+r"(nx), "=r"(ok)
        : "r"(smem_u32(&resp))
        : "memory");
    if (!ok) break;
    x = (int)nx;
  }
}

int main() {
  const int n = 2048, unit = 2000;
  std::vector<int> w(n);
  for (int i = 0; i < n; ++i) w[i] = 40 - (i * 39) / n;  // heavy first: 40 .. 1 units
  int *dw, *di, *ds;
  long long *d0, *d1;
  cudaMalloc(&dw, n * 4); cudaMalloc(&di, n * 4); cudaMalloc(&ds, n * 4);
  cudaMalloc(&d0, n * 8); cudaMalloc(&d1, n * 8);
  cudaMemcpy(dw, w.data(), n * 4, cudaMemcpyHostToDevice);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(di, 0xff, n * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    probe<<<n, 32, smem>>>(dw, di, ds, d0, d1, mode, unit);
    cudaEventRecord(b);
    cudaError_t e = cudaDeviceSynchronize();
    float ms = 0; cudaEventElapsedTime(&ms, a, b);
    std::vector<int> it(n), s(n);
    std::vector<long long> t0(n), t1(n);
    cudaMemcpy(it.data(), di, n * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(s.data(), ds, n * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(t0.data(), d0, n * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(t1.data(), d1, n * 8, cudaMemcpyDeviceToHost);
    // order in which items started (per-SM clocks are not synchronised across SMs; use per-SM sequence)
    std::vector<std::vector<std::pair<long long, int>>> per(200);
    for (int i = 0; i < n; ++i) if (it[i] >= 0) per[s[i]].push_back({t0[i], i});
    long long tot = 0, mx = 0; int nsm = 0;
    for (auto& v : per) {
      if (v.empty()) continue;
      ++nsm;
      std::sort(v.begin(), v.end());
      long long l = 0; for (auto& q : v) l += w[q.second];
      tot += l; mx = std::max(mx, l);
    }
    printf("mode %d (%s): %s, %.3f ms, SMs %d, work units per SM mean %.1f max %lld\n", mode,
           mode ? "claim at item start" : "claim 6 units before item end", cudaGetErrorString(e), ms, nsm,
           (double)tot / nsm, mx);
    int shown = 0;
    for (auto& v : per) {
      if (v.empty() || shown >= 6) continue;
      ++shown;
      printf("  sm items:");
      for (auto& q : v) printf(" %d", q.second);
      printf("\n");
    }
  }
  return 0;
}
