/* =====================================================================================
 * tt.h — C ABI of libtt.so: the B200 (sm_100a) hot path of Tree Training (arXiv 2511.00413).
 *
 * Citations: "P:n" = PAPER.md line n (the paper's LaTeX source), "S:n" = SPEC.md line n,
 * "R<k>" = reading k in DESIGN.md §3 (where the paper is silent or ambiguous).
 *
 * The library implements the data-parallel hot path named by BASELINE.json:north_star:
 *   tt_pack          Tree Packing of ONE tree/forest into a DFS-serialised token sequence plus the
 *                    three per-token artifacts of Fig. 6impl: restored position ids
 *                    (P:536-539), gradient-scale ("tree-scale") and the shared-prefix
 *                    mask, the latter as one subtree-end E_j per key (j <= i < E_j)
 *                    plus 128x128 tile metadata (empty / partial / full classes).
 *   tt_attn_fwd      shared-prefix-masked attention forward (Eq. 1), O and LSE.
 *   tt_attn_bwd      its backward with Gradient Restoration: the upstream gradient of every row i
 *                    is scaled by the tree-scale w_i (Fig. 4gradient; Eqs. 20-21
 *                    P:483-497), giving dQ/dK/dV equal to the sum over per-branch gradients
 *                    (Eqs. 14-16).
 *   tt_restore_loss  next-token cross entropy with the tree-scale folded into every prediction
 *                    (the "gradient scaling step before the backward propagation"; R6-R8),
 *                    its gradient w.r.t. the logits, and deterministic fp64 sums.
 *   tt_grad_sqnorm   deterministic fp64 sum of squares (per-tree gradient-norm scalars; also fused
 *                    into tt_attn_bwd through its optional `sqnorm` output).
 * Beyond the hot path:
 *   tt_plan_traversals / tt_traversal_forest   capacity-constrained Tree Packing (NEXT-f1)
 *   tt_rope / tt_restore_grad                  restored-position RoPE and the Gradient Scaler (NEXT-f2)
 *   tt_lmhead_loss                             LM head + restoration loss without [N, V] logits (NEXT-f3)
 *   tt_gemm                                    its tcgen05 GEMM (CTA pairs, fused epilogues)
 *   tt_pack_weights                            real-valued per-trajectory weights (NEXT-f4)
 *
 * Conventions (all entry points):
 *   - Status: every call returns tt_status; TT_OK == 0.  On error nothing is launched and a
 *     thread-local message is available from tt_last_error().
 *   - Memory: the CALLER owns every buffer.  The library never allocates device memory, never
 *     frees, never synchronises a stream, and keeps no global state except the thread-local
 *     error string, a cached per-device attribute query, and lazily created per-thread,
 *     per-device handles: one side stream + two events
 *     (tt_restore_loss; never created while `stream` is capturing) and a ring of 4 pinned host
 *     staging buffers + events (tt_pack / tt_pack_weights; released at thread exit).
 *   - Host vs device: pointers documented as HOST are read synchronously during the call;
 *     all others are DEVICE pointers and are accessed asynchronously on `stream`.
 *   - Layout "thd": Q/O/dO/dQ are [N, Hq, d], K/V/dK/dV are [N, Hkv, d], contiguous, row major,
 *     16-byte aligned.  LSE and D are [Hq, N] fp32.  GQA: the kv head of q head h is h / (Hq/Hkv)
 *     (R10).
 *   - Supported (d, dtype): (128, TT_BF16) on the tcgen05/TMEM/TMA kernels; (64, TT_BF16),
 *     (64, TT_FP32) and (128, TT_FP32) on the SIMT "test mode" kernels (R13).  Anything else
 *     returns TT_ERR_UNSUPPORTED.  There is no CPU fallback.
 * ===================================================================================== */
#ifndef TT_H_
#define TT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* tt_stream_t; /* == cudaStream_t */

typedef enum {
  TT_OK = 0,
  TT_ERR_INVALID_ARGUMENT = 1, /* null pointer, negative size, bad enum value              */
  TT_ERR_NOT_A_FOREST = 2,     /* parent out of range, self-parent, cycle                   */
  TT_ERR_EMPTY = 3,            /* the forest holds zero tokens                       */
  TT_ERR_TOO_LARGE = 4,        /* N, counts or pair totals overflow their types             */
  TT_ERR_UNSUPPORTED = 5,      /* head_dim / dtype / Hq % Hkv not supported                 */
  TT_ERR_ALIGNMENT = 6,        /* tensor not 16-byte aligned                                */
  TT_ERR_WORKSPACE = 7,        /* workspace too small                                       */
  TT_ERR_CUDA = 8              /* a CUDA runtime / driver call failed                       */
} tt_status;

typedef enum { TT_BF16 = 0, TT_FP32 = 1 } tt_dtype;

/* Tile edge used by all tile metadata and by the tensor-core kernels. */
#define TT_BLOCK 128

const char* tt_status_string(tt_status s);
/* Thread-local detail of the last error raised on this thread ("" if none). */
const char* tt_last_error(void);
/* ABI version (major * 100 + minor). */
int32_t tt_version(void);
/* Build flags of the loaded library: bit 0 (TT_BUILD_DEV) set only in a development build
 * (-DTT_DEV, `python -m paper_2511_00413_b200.build --dev`), whose kernels read A/B switches from
 * environment variables (ablations that skip work).  The shipped build returns 0 and ignores every
 * such variable; bench.py refuses to time a development build. */
#define TT_BUILD_DEV 1
int32_t tt_build_flags(void);

/* --------------------------------------------------------------------------------------
 * Tree Packing ("merge trajectories into a tree"; Eq. 13 P:395-400 "X_ours =
 * pack_ours[P;S_1;...;S_n]"; Fig. 6impl).
 *
 * Input (HOST, read during the call):
 *   parent[n]  int32, -1 for a root, else the parent node id (0 <= parent < n).
 *   len[n]     int32 >= 0, the node's segment token count l(y). Zero is allowed.
 *   term[n]    int32 >= 0 or NULL: trajectories that END at the node (duplicates and
 *              trajectories ending at an internal node).  NULL means 1 on childless
 *              nodes and 0 elsewhere.
 * Serialisation (R3): DFS pre-order, roots by ascending id, children by ascending id.
 * Per packed token i (node u = node(i)):
 *   pos[i]  = tokens on u's root path strictly before i (restored position id, R4)
 *   w[i]    = sum of term over subtree(u) = trajectories through i (tree-scale, R5)
 *   E[i]    = packed end (exclusive) of subtree(u); token i may attend j iff j <= i < E_j (R2)
 *   node[i] = u
 * Per 128-token block kb: kblk_minE / kblk_maxE = min / max of E over its keys.
 * Forward tile lists: for q-block qb, the k-blocks kb <= qb with a non-empty tile, ascending,
 *   at fwd_list[qb*(qb+1)/2 + t], t < fwd_cnt[qb]; each entry is kb | (cls << 28) with
 *   cls 1 = partial (mask needed), 2 = full (every pair allowed).  Tile classes are exact:
 *   for kb < qb, empty iff maxE_kb <= 128*qb, full iff minE_kb >= min(N, 128*qb+128);
 *   the diagonal tile is partial unless it holds a single token.
 * Backward: the q-blocks that see k-block kb are exactly [kb, ceil(kblk_maxE[kb] / 128)).
 * Loss targets (App. D of SURVEY, R7): for the LAST token of every node u, the packed indices
 *   of the first token of every continuation (children of u in order; a zero-length child
 *   contributes its own continuations recursively) at succ_tok[succ_ptr[u] .. succ_ptr[u+1]).
 * -------------------------------------------------------------------------------------- */
typedef struct {
  int32_t n_nodes;
  int32_t n_roots;
  int32_t n_traj;          /* trajectories = sum of term                                  */
  int32_t n_blk;           /* ceil(N / 128)                                               */
  int32_t n_succ;          /* entries of succ_tok                                         */
  int32_t reserved;
  int64_t n_tokens;        /* N = sum of len                                              */
  int64_t n_linear_tokens; /* sum_l L_l = sum_i w_i  (per-branch linear token count)      */
  int64_t n_pairs;         /* A     = sum_i (pos_i + 1)   (allowed (i, j) pairs)          */
  int64_t n_linear_pairs;  /* A_lin = sum_i w_i (pos_i + 1) = sum_l L_l (L_l + 1) / 2     */
  size_t ws_bytes;         /* device workspace tt_pack needs                              */
} tt_pack_info;

typedef struct {
  /* device pointers into the caller's pack workspace (valid while it lives) */
  const int32_t* pos;          /* [N]      */
  const int32_t* w;            /* [N]      */
  const int32_t* E;            /* [N]      */
  const int32_t* node;         /* [N]      */
  const int32_t* node_start;   /* [n]      */
  const int32_t* node_len;     /* [n]      */
  const int32_t* node_sub_end; /* [n]      */
  const int32_t* node_depth;   /* [n]      tokens on the root path before the node          */
  const int32_t* node_leaves;  /* [n]      */
  const int32_t* succ_ptr;     /* [n + 1]  */
  const int32_t* succ_tok;     /* [n_succ] */
  const int32_t* kblk_minE;    /* [n_blk]  */
  const int32_t* kblk_maxE;    /* [n_blk]  */
  const int32_t* fwd_cnt;      /* [n_blk]  */
  const int32_t* fwd_list;     /* [n_blk * (n_blk + 1) / 2] */
  const float* wr;             /* [n_blk * 128] real-valued tree-scale W (NEXT-f4), NULL after tt_pack;
                                  set by tt_pack_weights.  When non-NULL it replaces w as the
                                  restoration weight of tt_attn_bwd and tt_restore_loss.          */
  int64_t n_tokens;
  int32_t n_nodes;
  int32_t n_blk;
  int32_t n_succ;
  int32_t max_succ;            /* longest continuation list (tt_restore_loss supports <= 1024) */
  /* host-computed schedule statistics of the backward's key-stationary walk (64-row query tiles per
     128-key block: nq_kb = ceil(kblk_maxE[kb] / 64) - 2 kb): their sum and maximum.  The attention
     kernels order their CTAs kv-head-major when the heaviest CTA is a small share of one SM's work
     (better L2 locality under the power cap), heads-fastest otherwise (no late heavy tail). */
  int64_t sched_sum_nq;
  int32_t sched_max_nq;
  int32_t wr_negative;         /* 1 when tt_pack_weights produced some W < 0 (else the backward folds
                                  the tree-scale into the log-sum-exp: P w = exp2(. + log2 w))      */
} tt_packed;

/* Validate the forest and size the pack (HOST only, synchronous, no CUDA calls). */
tt_status tt_pack_plan(const int32_t* parent, const int32_t* len, const int32_t* term, int32_t n_nodes,
                       tt_pack_info* info);

/* Pack: host validation + O(n) node DFS, one async H2D copy of the node tables, then device
 * kernels that fill the per-token arrays and the tile metadata into d_ws (ws_bytes >=
 * info.ws_bytes).  `out` receives device pointers into d_ws.  `info` may be NULL.
 * The node tables are staged through a per-thread ring of 4 pinned host buffers (the copy never
 * synchronises the stream; a slot is reused once its previous copy has completed, so the host may
 * wait for a pack issued 4 calls earlier).  Not capturable: a capturing `stream` returns
 * TT_ERR_INVALID_ARGUMENT (pack outside the capture and capture the fwd / loss / bwd calls). */
tt_status tt_pack(const int32_t* parent, const int32_t* len, const int32_t* term, int32_t n_nodes,
                  void* d_ws, size_t ws_bytes, tt_packed* out, tt_pack_info* info, tt_stream_t stream);

/* --------------------------------------------------------------------------------------
 * Real-valued leaf weights ("leaf_weights: per leaf in batch,
 * real" and "tree_scale of a token in node u = sum of weights of leaves in u's subtree that are
 * present in THIS traversal", "non-uniform leaf weights ... scaler = weight sums"; linear
 * extension of Eq. 12, reading R20).
 *   The training objective becomes sum_l alpha_l * Loss_l over trajectories l (alpha: e.g. RL
 *   advantages, any sign).  By linearity every identity of the integer case holds with the
 *   leaf count w_i replaced by W_i = sum of alpha_l over the trajectories through token i.
 * traj_weight: HOST [n_traj] fp32, trajectory l in canonical order (DFS pre-order of trajectory
 *   end nodes, roots / children ascending id, the term(u) trajectories of a node consecutive) —
 *   the same order tt_plan_traversals numbers trajectories in; for one traversal of a plan, pass
 *   the weights of its trajectories in that order over the forest tt_traversal_forest returns.
 * parent/len/term/n_nodes: exactly the forest pk was packed from (checked: n_nodes, N).
 * wr: DEVICE [n_blk * 128] fp32, 16-byte aligned, caller-owned; W per token (fp64 subtree sums
 *   rounded once to fp32), 0 in the padding.  On success pk->wr = wr.  Host work O(n + N), one
 *   async H2D copy on `stream` through the same pinned staging ring as tt_pack (not capturable).
 * -------------------------------------------------------------------------------------- */
tt_status tt_pack_weights(const int32_t* parent, const int32_t* len, const int32_t* term, int32_t n_nodes,
                          const float* traj_weight, tt_packed* pk, float* wr, tt_stream_t stream);

/* --------------------------------------------------------------------------------------
 * Tree-masked attention forward (Eq. 1 P:119-126 with softmax scale, R1; mask R2):
 *   O_i   = sum_{j : j <= i < E_j} softmax_j(scale * q_i . k_j) v_j
 *   LSE_i = ln sum_{j : j <= i < E_j} exp(scale * q_i . k_j)      (natural log, R9)
 * q [N,hq,d], k/v [N,hkv,d] (dtype dt), o [N,hq,d] (dtype dt), lse [hq,N] fp32.
 * Empty tiles are skipped, full tiles run unmasked, partial tiles are masked in registers.
 * bf16 / d = 128 runs persistent CTAs (cluster launch control takes over not-yet-launched CTAs' work
 * items); results do not depend on which CTA runs an item (bitwise reproducible).
 * -------------------------------------------------------------------------------------- */
tt_status tt_attn_fwd(const tt_packed* pk, const void* q, const void* k, const void* v, tt_dtype dt,
                      int32_t hq, int32_t hkv, int32_t d, float softmax_scale, void* o, float* lse,
                      tt_stream_t stream);

/* Bytes of device workspace tt_attn_bwd needs (fp32 dQ accumulator + D). */
tt_status tt_attn_bwd_workspace(const tt_packed* pk, int32_t hq, int32_t hkv, int32_t d, tt_dtype dt,
                                size_t* bytes);

/* Which backward kernel tt_attn_bwd launches for this packed forest and head layout (host only, no CUDA
 * call): *kernel = 0 for tree_attn_bwd_sm100, the persistent kernel (cluster-launch-control work stealing
 * over (128-key block, kv head) items; chosen when the mean number of 64-row query tiles per item,
 * sched_sum_nq * (hq / hkv) / n_blk, is below 80: small trees), 1 for tree_attn_bwd_flat_sm100 (one CTA
 * per item; long items), 2 for the SIMT kernel (fp32 or d != 128).  Same result either way. */
tt_status tt_attn_bwd_kernel(const tt_packed* pk, int32_t hq, int32_t hkv, int32_t d, tt_dtype dt,
                             int32_t* kernel);

/* --------------------------------------------------------------------------------------
 * Tree-masked attention backward with Gradient Restoration (Eqs. 2, 14-16, 20-21; R6):
 *   omega_i = (pk->wr ? pk->wr[i] : w_i) if restore else 1;  P_ij = exp(scale q_i.k_j - LSE_i);  D_i = dO_i . O_i
 *   dV_j = sum_i omega_i P_ij dO_i
 *   dS_ij = omega_i P_ij (dO_i . v_j - D_i)
 *   dQ_i = scale sum_j dS_ij k_j,   dK_j = scale sum_i dS_ij q_i     (sums over j <= i < E_j)
 *   GQA: dK/dV of a kv head sum over its q heads.
 * With restore = 1, `dout` is the per-token upstream gradient G of ONE branch (identical for
 * every branch through the token) and the outputs equal the sum over branches of ordinary
 * causal-attention gradients.  With restore = 0, `dout` must already be restored (w (.) G).
 * o / lse are the outputs of tt_attn_fwd.  dq [N,hq,d], dk/dv [N,hkv,d] in dtype dt.
 * sqnorm (nullable, DEVICE double[3]): the per-tree gradient-norm scalars of SURVEY §8(a) row a6,
 *   ||dQ||^2, ||dK||^2, ||dV||^2 of the STORED outputs, fused into the backward (per-CTA / per-block
 *   partials written by the kernels that produce dK/dV and dQ, summed in a fixed order in fp64:
 *   bitwise reproducible, no extra pass over the gradients).
 * -------------------------------------------------------------------------------------- */
tt_status tt_attn_bwd(const tt_packed* pk, const void* q, const void* k, const void* v, const void* o,
                      const float* lse, const void* dout, int32_t restore, tt_dtype dt, int32_t hq,
                      int32_t hkv, int32_t d, float softmax_scale, void* dq, void* dk, void* dv, double* sqnorm,
                      void* d_ws, size_t ws_bytes, tt_stream_t stream);

/* --------------------------------------------------------------------------------------
 * Gradient-Restoration loss (R6, R7, R8, R17).  For every packed row t
 * with targets T(t) (next token inside the node, else the continuation list succ_tok; a target
 * counts iff node_loss_mask[node(target)] != 0 when the mask is given, and — boundary_mode 1 —
 * only when the trajectories through t continue to a single next token, i.e. at most one entry of
 * the continuation list has w > 0 — subtrees carrying no trajectory are no branch), each target k with weight omega_k = w[k] (pk->wr[k]
 * when real-valued leaf weights are set, NEXT-f4):
 *   loss_t   = sum_k omega_k (lse(x_t) - x_t[tok[k]])
 *   dlogits_t = grad_scale * (Omega_t softmax(x_t) - sum_k omega_k e_{tok[k]}),  Omega_t = sum omega_k
 * logits [N, ld] bf16 (row stride ld >= vocab elements, 16-byte aligned rows); dlogits has the
 * same layout and MAY ALIAS logits (each row is read before it is written).  tok [N] int32.
 * tok_loss [N] fp32 (nullable) receives loss_t.  sums [2] fp64 (device) receives
 * (sum_t loss_t, sum_t Omega_t), reduced in a fixed order (bitwise reproducible).
 * d_err (device int32, nullable) is set to 1 if a target token id is outside [0, vocab); that
 * row's loss is NaN.  ws: >= tt_restore_loss_workspace() bytes.
 * Execution: when vocab % 16 == 0, rows are 32-byte aligned and N >= 8 rows per SM, the call forks
 * a library-owned side stream from `stream` (event record + wait) for the tail rows, which run on
 * the SMs the 4-CTA clusters leave idle, and joins it back into `stream` before the final sum:
 * the call stays stream-ordered on `stream` and may be captured into a CUDA graph.
 * Row results do not depend on which kernel computed a row beyond fp32 rounding order.
 * -------------------------------------------------------------------------------------- */
size_t tt_restore_loss_workspace(const tt_packed* pk);
tt_status tt_restore_loss(const tt_packed* pk, const void* logits, int64_t ld, int32_t vocab, const int32_t* tok,
                          const uint8_t* node_loss_mask, int32_t boundary_mode, float grad_scale, void* dlogits,
                          float* tok_loss, double* sums, int32_t* d_err, void* d_ws, size_t ws_bytes,
                          tt_stream_t stream);

/* Deterministic sum of squares of n elements of x (dtype dt) into *out (device, fp64): the squares
 * of each 16-byte vector are summed in fp32 (exact squares for bf16; <= 2^-21 relative for the
 * 8-term sum), vectors are accumulated in fp64 over a fixed partition and reduced in a fixed order,
 * so the result is bitwise reproducible.  x must be 16-byte aligned.
 * ws >= tt_grad_sqnorm_workspace(n) bytes. */
size_t tt_grad_sqnorm_workspace(int64_t n);
tt_status tt_grad_sqnorm(const void* x, int64_t n, tt_dtype dt, double* out, void* d_ws, size_t ws_bytes,
                         tt_stream_t stream);
/* The per-tree gradient-norm scalars of §8(a) a6 in one launch: out[k] = sum of squares of tensor k
 * (e.g. dQ, dK, dV).  Same numerics as tt_grad_sqnorm; ws >= tt_grad_sqnorm_workspace(0). */
tt_status tt_grad_sqnorm3(const void* x0, int64_t n0, const void* x1, int64_t n1, const void* x2, int64_t n2,
                          tt_dtype dt, double* out, void* d_ws, size_t ws_bytes, tt_stream_t stream);

/* --------------------------------------------------------------------------------------
 * Capacity-constrained Tree Packing.  HOST only, synchronous.
 *
 * Splits the trajectories of a tree/forest (same parent/len/term input as tt_pack) into traversals
 * (training steps) whose induced sub-forest holds at most `capacity` tokens (Eq. 3
 * generalised to multi-path traversals), with the heuristic of P:303-306 (reading R19 in DESIGN.md:
 * DFS with children in descending order of their deepest trajectory end, a new traversal whenever
 * the next trajectory's uncovered tokens would exceed the capacity).
 * Trajectories are numbered in canonical order: DFS pre-order (roots / children ascending id) of
 * their end nodes, term(u) consecutive copies.  traversal_of_traj [n_traj] (nullable for sizing)
 * receives each trajectory's traversal id.  TT_ERR_TOO_LARGE if one trajectory exceeds capacity.
 * tt_traversal_forest writes the sub-forest induced by one traversal (node ids keep their relative
 * order; out_term counts the traversal's trajectories ending at each node, so tt_pack on it yields
 * the in-traversal tree-scale) into caller arrays of n_nodes entries; out_node maps new ids
 * to original ids.
 * -------------------------------------------------------------------------------------- */
typedef struct {
  int32_t n_traj;
  int32_t n_traversals;
  int64_t capacity;
  int64_t linear_tokens;  /* sum over trajectories of their path length (per-branch packing)   */
  int64_t tree_tokens;    /* tokens on at least one trajectory (whole tree in one step)        */
  int64_t planned_tokens; /* sum over traversals of their induced sub-forest tokens            */
} tt_plan_info;

tt_status tt_plan_traversals(const int32_t* parent, const int32_t* len, const int32_t* term, int32_t n_nodes,
                             int64_t capacity, int32_t* traversal_of_traj, tt_plan_info* info);
tt_status tt_traversal_forest(const int32_t* parent, const int32_t* len, const int32_t* term, int32_t n_nodes,
                              const int32_t* traversal_of_traj, int32_t traversal, int32_t* out_parent,
                              int32_t* out_len, int32_t* out_term, int32_t* out_node, int32_t* n_out);

/* --------------------------------------------------------------------------------------
 * LM head + Gradient-Restoration cross entropy without materialising [N, V] logits
 * (P:549 and readings R6-R8, R17, R20 exactly as tt_restore_loss, on logits
 * X = H W^T computed and kept in fp32):
 *   loss_t = sum_k omega_k (lse(x_t) - x_t[y_k]),   G_t = gamma (Omega_t softmax(x_t) - sum_k omega_k e_{y_k})
 *   dH = G W  [N, hidden],   dW = G^T H  [vocab, hidden]
 * Every contraction is the library's own tcgen05 GEMM (tt_gemm below) with the cross-entropy steps
 * fused into its epilogues: sweep 1 is ONE GEMM over the whole vocabulary whose epilogue keeps only
 * per-row (max, sum-exp) partials of each 128-column slice and the target logits (the [N, vocab]
 * logits are never written); sweep 2 recomputes X per chunk of vocab_chunk columns with an epilogue
 * that writes G in bf16 (largest temporary [N, vocab_chunk] bf16 + the fp32 dH accumulator), then
 * dH (+)= G_c W_c and dW_c = G_c^T H.
 * h: DEVICE [N, hidden] bf16; w: DEVICE [vocab, hidden] bf16 (row-major, the LM-head weight);
 * tok / node_loss_mask / boundary_mode / grad_scale / tok_loss / sums / d_err: as tt_restore_loss.
 * dh: DEVICE [N, hidden] bf16 (written); dw: DEVICE [vocab, hidden] bf16 (written).
 * d_ws: DEVICE workspace of tt_lmhead_loss_workspace bytes (16-byte aligned), caller-owned.
 * hidden % 8 == 0.  Errors: as tt_restore_loss; TT_ERR_CUDA if a launch fails.
 * -------------------------------------------------------------------------------------- */
tt_status tt_lmhead_loss_workspace(const tt_packed* pk, int32_t hidden, int32_t vocab, int32_t vocab_chunk,
                                   size_t* bytes);
tt_status tt_lmhead_loss(const tt_packed* pk, const void* h, const void* w, int32_t hidden, int32_t vocab,
                         int32_t vocab_chunk, const int32_t* tok, const uint8_t* node_loss_mask, int32_t boundary_mode,
                         float grad_scale, void* dh, void* dw, float* tok_loss, double* sums, int32_t* d_err,
                         void* d_ws, size_t ws_bytes, tt_stream_t stream);

/* --------------------------------------------------------------------------------------
 * GEMM building block of tt_lmhead_loss, exposed for direct testing:
 *   D[M, N] (=|+=) A[M, K] . B[K, N]     bf16 operands, fp32 accumulation (tcgen05, CTA pairs)
 * a: DEVICE bf16, stored row-major [M, K] (a_mn = 0) or [K, M] (a_mn = 1), row stride lda elements;
 * b: DEVICE bf16, stored row-major [N, K] (b_mn = 0) or [K, N] (b_mn = 1), row stride ldb elements;
 * d: DEVICE [M, ldd] row-major, bf16 (d_dt = TT_BF16, written) or fp32 (TT_FP32; accumulate = 1
 *    adds into it).  Strides and base pointers 16-byte aligned.  M, N, K > 0.
 * -------------------------------------------------------------------------------------- */
tt_status tt_gemm(int32_t M, int32_t N, int32_t K, const void* a, int64_t lda, int32_t a_mn, const void* b,
                  int64_t ldb, int32_t b_mn, void* d, int64_t ldd, tt_dtype d_dt, int32_t accumulate,
                  tt_stream_t stream);

/* --------------------------------------------------------------------------------------
 * Position-embedding correction (Eq. 23):
 * RoPE must rotate every token by its RESTORED position pos_i (pk->pos, R4) so that dY/dX is the
 * same in tree and per-branch packing.  Convention (reading R21): rotate-half over the whole head
 * dim d, theta_j = base^(-2j/d) for j < d/2, a = pos_i * theta_j,
 *   y_j = x_j cos a - x_{j+d/2} sin a,   y_{j+d/2} = x_j sin a + x_{j+d/2} cos a.
 * inverse != 0 rotates by -a (the backward: dX = R(-a) dY).  Angles are reduced mod 2 pi in fp64.
 * x: DEVICE [N, n_heads, d] (dtype dt, contiguous, 16-byte aligned), rotated IN PLACE.
 * d in {64, 128}; base > 0 (Qwen3: 1e6).  HBM-bound: reads and writes x once.
 * -------------------------------------------------------------------------------------- */
tt_status tt_rope(const tt_packed* pk, void* x, tt_dtype dt, int32_t n_heads, int32_t d, double base,
                  int32_t inverse, tt_stream_t stream);

/* --------------------------------------------------------------------------------------
 * Gradient Scaler for an arbitrary upstream gradient ("a gradient scaling step before the
 * backward propagation"; Fig. 4gradient): g[i, :] *= W_i IN PLACE, W_i = pk->wr[i] when
 * tt_pack_weights set real weights (R20), else the leaf count pk->w[i] (R5).  After it, every later
 * backward op runs uncorrected (transitivity, Eqs. 17-21), e.g. tt_attn_bwd(restore=0).
 * g: DEVICE [N, row_elems] (dtype dt, contiguous, 16-byte aligned, row bytes a multiple of 16).
 * -------------------------------------------------------------------------------------- */
tt_status tt_restore_grad(const tt_packed* pk, void* g, tt_dtype dt, int64_t row_elems, tt_stream_t stream);

/* Kernel-level launch counters (for bench.py's gpu_launches claim): number of kernels this
 * thread has launched through the library since the last reset. */
int64_t tt_launch_count(void);
void tt_launch_count_reset(void);

#ifdef __cplusplus
}
#endif
#endif /* TT_H_ */
