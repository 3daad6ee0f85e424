// Internal helpers shared by the libtt.so translation units (never by the oracle).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <string>

#include <cuda.h>

#include "../../include/tt.h"

namespace tt {

// Development A/B switches (ablations, variant sweeps, CTA orders, cycle counters) exist only in a
// build compiled with -DTT_DEV (python -m paper_2511_00413_b200.build --dev).  In the shipped
// library dev_getenv() is always null and dev_dbg() a constant 0, so no environment variable can
// change what a kernel computes or skip work (tests/test_abi.py checks the release build ignores
// them).
#ifdef TT_DEV
inline const char* dev_getenv(const char* name) { return getenv(name); }
__host__ __device__ constexpr int dev_dbg(int d) { return d; }
constexpr bool kDevBuild = true;
#else
inline const char* dev_getenv(const char*) { return nullptr; }
__host__ __device__ constexpr int dev_dbg(int) { return 0; }
constexpr bool kDevBuild = false;
#endif

void set_error(const char* fmt, ...);
void clear_error();
void count_launch(int n = 1);

// Check the launch that was just issued on this thread's runtime.
tt_status check_launch(const char* what);

inline cudaStream_t as_cuda(tt_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

template <typename T>
__host__ __device__ inline T ceil_div(T a, T b) { return (a + b - 1) / b; }

constexpr int kBlock = TT_BLOCK;           // 128: tile edge of all tile metadata
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

// fwd tile-list entry encoding
constexpr int kClsShift = 28;
constexpr int32_t kKbMask = (1 << kClsShift) - 1;
constexpr int kClsPartial = 1;
constexpr int kClsFull = 2;

__host__ __device__ inline int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ inline int64_t tri_off(int64_t qb) { return qb * (qb + 1) / 2; }

// ---- kernel launchers implemented in the .cu files ----
tt_status launch_pack_fill(const tt_packed& pk, const int32_t* order, const int32_t* order_start, int32_t n_order,
                           const int32_t* kb_lo, const int32_t* blk_first,
                           int32_t* pos, int32_t* w, int32_t* E, int32_t* node, int32_t* kminE, int32_t* kmaxE,
                           int32_t* fwd_cnt, int32_t* fwd_list, cudaStream_t st);

tt_status simt_attn_fwd(const tt_packed& pk, const void* q, const void* k, const void* v, tt_dtype dt, int hq,
                        int hkv, int d, float scale, void* o, float* lse, cudaStream_t st);
tt_status simt_attn_bwd(const tt_packed& pk, const void* q, const void* k, const void* v, const float* lse,
                        const float* Dvec, const void* dout, int restore, tt_dtype dt, int hq, int hkv, int d,
                        float scale, void* dq, void* dk, void* dv, cudaStream_t st);
tt_status launch_bwd_pre_tc(const void* o, const void* dout, const float* lse, const int32_t* w, const float* wr, int restore, int fold,
                            int64_t N, int64_t Np, int hq, float* Dp, float* L2p, float* wf, float* dq_acc,
                            cudaStream_t st);
tt_status launch_bwd_pre(const void* o, const void* dout, tt_dtype dt, int64_t N, int hq, int d, float* Dvec,
                         float* dq_acc, cudaStream_t st);

bool sm100_available();
tt_status make_tmap_thd(CUtensorMap* m, const void* ptr, int64_t rows, int heads, int d, int box_rows,
                        CUtensorMapDataType dt, int elem_bytes, CUtensorMapSwizzle sw, int box_inner);
tt_status make_tmap_3d(CUtensorMap* m, const void* ptr, CUtensorMapDataType dt, int elem_bytes, const int64_t dims3[3],
                       const int64_t strides2[2], const int box3[3]);
// fp32 dQ accumulator of the tensor-core backward: [N][hq][d] (0) or [hq][N][d] (TT_DQ_HND=1: every 32-row
// TMA reduce box one contiguous 16 KB run)
#ifndef TT_DQ_HND
#define TT_DQ_HND 0
#endif
tt_status sm100_attn_fwd(const tt_packed& pk, const void* q, const void* k, const void* v, int hq, int hkv,
                         int d, float scale, void* o, float* lse, cudaStream_t st);
// ws: the tensor-core backward workspace (tt_attn_bwd_workspace bytes); see sm100_bwd_ws_bytes
size_t sm100_bwd_ws_bytes(int64_t N, int hq, int hkv, int d);
tt_status sm100_attn_bwd(const tt_packed& pk, const void* q, const void* k, const void* v, const void* o,
                         const float* lse, const void* dout, int restore, int hq, int hkv, int d, float scale,
                         void* ws, void* dq, void* dk, void* dv, double* sqnorm, cudaStream_t st);

tt_status launch_loss(const tt_packed& pk, const __nv_bfloat16* logits, int64_t ld, int vocab, const int32_t* tok,
                      const uint8_t* node_mask, int boundary_mode, float gamma, __nv_bfloat16* dlogits,
                      float* tok_loss, double* sums, int32_t* d_err, float* ws_loss, float* ws_omega,
                      cudaStream_t st);
tt_status launch_sqnorm(const void* const* xs, const int64_t* ns, int count, tt_dtype dt, double* out,
                        double* partials, cudaStream_t st);

tt_status launch_loss_sums(int64_t N, const float* ws_loss, const float* ws_omega, double* sums, cudaStream_t st);
size_t lmhead_ws_bytes(int64_t N, int D, int V, int Vc, int max_t);

// tcgen05 GEMM of gemm_sm100.cu (CTA pairs): D[M, N] = A . B, epilogue selected by `epi`
namespace gemm {
enum { kEpiStoreBF16 = 0, kEpiAccF32 = 1, kEpiLsePartial = 2, kEpiDlogits = 3 };
struct GemmEpilogue {
  void* out = nullptr;       // bf16 (kEpiStoreBF16, kEpiDlogits) / fp32 (kEpiAccF32) [M, ldo]
  int64_t ldo = 0;
  int beta = 0;              // kEpiAccF32: accumulate
  int col_offset = 0, vocab = 0;
  void* part = nullptr;      // float2 [2 ceil(N / 256)][M]
  int max_t = 1;
  const int* tgt_cnt = nullptr;
  const int* tgt_y = nullptr;
  const float* tgt_w = nullptr;
  float* tgt_x = nullptr;
  const float* lse2 = nullptr;
  const float* g_omega = nullptr;
  float gamma = 1.f;
};
tt_status gemm_run(int epi, int M, int N, int K, const void* A, int64_t lda, int a_mn, const void* B, int64_t ldb,
                   int b_mn, const GemmEpilogue& ep, cudaStream_t st);
}  // namespace gemm
tt_status launch_lmhead_loss(const tt_packed& pk, const __nv_bfloat16* H, const __nv_bfloat16* W, int D, int V, int Vc,
                             const int32_t* tok, const uint8_t* node_mask, int boundary_mode, float gamma,
                             __nv_bfloat16* dH, __nv_bfloat16* dW, float* tok_loss, double* sums, int32_t* d_err,
                             void* ws, cudaStream_t st);
tt_status launch_rope(const tt_packed& pk, void* x, tt_dtype dt, int H, int d, double base, int inverse,
                      cudaStream_t st);
tt_status launch_restore_grad(const tt_packed& pk, void* g, tt_dtype dt, int64_t row_elems, cudaStream_t st);

constexpr int kSqnormBlocks = 296;

// CTA orders of the attention kernels (chunk = consecutive query-block pairs / key blocks whose CTAs are
// ordered kv-head-major; 1 = heads fastest).  Measured under the power cap (profiles/r2d_cta_chunk.txt):
// head-major (one chunk) is 1-2% faster on the deep / 64K trees (the Q / dO / dQ or K / V rows of one
// head group stay L2-resident: the backward runs 80 MHz higher at the same power) and 5-8% slower on the
// 8K and wide trees (their heaviest CTAs would start late).  Head-major when the heaviest backward CTA
// is under 30% of one SM's share of the work: sms * max_nq / (hkv * sum_nq) < 0.3.
bool head_major_order(const tt_packed& pk, int hkv);
inline int fwd_cta_chunk(const tt_packed& pk, int npairs, int hkv) { return head_major_order(pk, hkv) ? npairs : 1; }
inline int bwd_cta_chunk(const tt_packed& pk, int hkv) { return head_major_order(pk, hkv) ? pk.n_blk : 1; }
// backward kernel choice (tt_attn_bwd_kernel): the persistent kernel for short work items, the flat one for
// long items (mean 64-row query tiles per (key block, kv head) item >= 80; profiles/r2q_bwd_ab.txt, r2ad_bwd_threshold.txt)
constexpr double kBwdFlatMinTilesPerItem = 80.0;
inline bool bwd_use_flat(const tt_packed& pk, int hq, int hkv) {
  const double tiles_per_item = (double)pk.sched_sum_nq * (hq / hkv) / (pk.n_blk > 0 ? pk.n_blk : 1);
  return tiles_per_item >= kBwdFlatMinTilesPerItem;
}

}  // namespace tt
