/*
 * loza.h — C ABI of libloza.so, the B200 (sm_100a) hot path of LoZA
 * (LongCat ZigZag Attention, arXiv 2512.23966): streaming sparse attention (SSA)
 * over the absorbed latent MLA key/value cache, its full-attention comparator,
 * and the LoZA calibration blend.
 *
 * Notation (Eq. 1-4):
 *   B batch, n_q query tokens, n_kv key tokens, H query heads, one shared latent
 *   KV head (MLA), d_qk = 512 latent + 64 RoPE = 576, d_v = 512
 *   (V = the first d_v columns of the latent KV row; pass v == k).
 *   Pattern (s, l, b) = (#sink blocks, #local blocks, block size), PAPER.md:57;
 *   paper default (1, 7, 128) = 1,024-token window.
 *   Query at absolute position p attends key j  <=>  j <= p and
 *   ( floor(j/b) < s  or  floor(p/b) - floor(j/b) < l ).
 *   The query's own (partial) block is one of the l local blocks (DESIGN R2).
 *
 * Conventions shared by every entry point:
 *   - All pointers named *_dev / q / k / v / o / lse / ws are DEVICE pointers;
 *     the caller owns every buffer; the library never allocates device memory
 *     (workspace sizes are queried with loza_workspace_size).
 *   - Every call is asynchronous on `stream` (a cudaStream_t passed as void*,
 *     NULL = legacy default stream) and never synchronises the host. seq_lens,
 *     alpha and d_alpha live on the device, so decode and blend steps are
 *     CUDA-graph capturable.
 *   - Strides are in ELEMENTS. Offsets are int64 (a 1M-token Q has 3.9e10 elems).
 *   - Errors: host-side validation happens before any launch and returns a
 *     status; nothing is launched on error. LOZA_ERR_CUDA / LOZA_ERR_NCCL carry
 *     text in loza_last_error() (thread-local). No exceptions cross the ABI.
 *     There is NO fallback path: an unsupported combination returns
 *     LOZA_ERR_UNSUPPORTED.
 *   - Dispatch: in_dtype LOZA_F32 -> SIMT fp32 kernels (any d_qk <= 576,
 *     d_v <= 512, any b >= 1); in_dtype LOZA_BF16 with (d_qk, d_v) = (576, 512)
 *     and b % 128 == 0 -> tcgen05/TMEM/TMA kernels. Anything else: UNSUPPORTED.
 */
#ifndef LOZA_H_
#define LOZA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* loza_stream_t;     /* cudaStream_t */
typedef void* loza_nccl_comm_t;  /* ncclComm_t (NCCL 2.28, the libnccl.so.2 torch loads) */

typedef enum {
  LOZA_OK = 0,
  LOZA_ERR_INVALID = 1,      /* bad pattern / scale / flags / alpha */
  LOZA_ERR_SHAPE = 2,        /* inconsistent dims or strides, misalignment, n_kv < q_start + n_q */
  LOZA_ERR_UNSUPPORTED = 3,  /* valid but not implemented on this path (no fallback) */
  LOZA_ERR_CUDA = 4,
  LOZA_ERR_NCCL = 5
} loza_status_t;

typedef enum { LOZA_F32 = 0, LOZA_BF16 = 1 } loza_dtype_t;

/* Sparse pattern of Eq. 4: s >= 0, l >= 1, b >= 1. */
typedef struct {
  int32_t sink_blocks;   /* s */
  int32_t local_blocks;  /* l (includes the query's own block) */
  int32_t block_size;    /* b */
} loza_pattern_t;

/* One attention problem. Q row (batch, i, head) sits at absolute position
 * q_start + i and attends keys [0, n_kv) of its batch under the mask. */
typedef struct {
  int32_t batch, n_q, heads, d_qk, d_v;
  int64_t n_kv;          /* keys available per batch (prefill: >= q_start + n_q) */
  int64_t q_start;       /* absolute position of query row 0 (multiple of b for SSA) */
  loza_dtype_t in_dtype;   /* q, k, v */
  loza_dtype_t out_dtype;  /* o (bf16 RN-even or fp32) */
  float softmax_scale;   /* logits = softmax_scale * q.k (Eq. 1 "details omitted": DESIGN R1) */
  int32_t causal;        /* 1 = causal (required by SSA), 0 = bidirectional (full_attn_ref only) */
  const void* q; int64_t q_stride_b, q_stride_tok, q_stride_head;  /* [B, n_q, H, d_qk] */
  const void* k; int64_t k_stride_b, k_stride_tok;                 /* [B, n_kv, d_qk] latent, 1 KV head */
  const void* v; int64_t v_stride_b, v_stride_tok;                 /* [B, n_kv, d_v]; MLA: v == k */
  void* o;       int64_t o_stride_b, o_stride_tok, o_stride_head;  /* [B, n_q, H, d_v] */
  float* lse;    /* optional [B, H, n_q] fp32, natural log: m + ln(sum) ; NULL = skip */
} loza_attn_args_t;

/* SSA prefill, Eq. 4: O* = softmax(scale Q K*^T) V* with K*, V*
 * the sink + local blocks of each query block. Causal only (causal = 0 returns
 * LOZA_ERR_UNSUPPORTED, DESIGN R9). bf16 path: q/o rows must be head-contiguous
 * (q_stride_head == d_qk, q_stride_tok == H*d_qk, same for o), H*b % 128 == 0. */
loza_status_t ssa_prefill(const loza_attn_args_t* args, loza_pattern_t pattern, loza_stream_t stream);

/* SSA decode (one new token per sequence), Eq. 4 with the query at position
 * p = seq_lens[b] - 1 (seq_len INCLUDES the current token, DESIGN R8): reads only
 * the sink block(s) and the last l blocks of the cache, so its cost is
 * independent of the context length. args->n_q must be 1; args->n_kv = cache
 * capacity T_cap; seq_lens_dev [B] int32 on the device, 1 <= seq_len <= T_cap. q [B,1,H,d_qk] ->
 * o [B,1,H,d_v]. batch == 0 returns LOZA_OK without touching anything (seq_lens_dev may then be NULL).
 * ws: loza_workspace_size(LOZA_WS_DECODE, ...) bytes, initialised ONCE with loza_workspace_init (or any zero
 * fill) before its first use; every call leaves it reusable. Bytes [0, 4) are an int32 status word: the
 * kernels set it to LOZA_ERR_SHAPE when a seq_len was outside [1, T_cap] (they clamp it and continue); the
 * caller reads and resets it. The rest holds the flattened kernel's per-sequence counters (left at zero by
 * every call) and split partials.
 * bf16 path kernels: while 2*batch <= SM count, a CTA pair per sequence -- the pair-cooperative kernel
 * (attn_tc_decode_coop.cu) for any H <= 64 (H < 64: decode sharded by heads; every GPU still reads the whole
 * latent window, the missing heads are zero-padded); otherwise (H == 64 only) a flattened split-KV kernel.
 * The key-split pair kernel (attn_tc_decode_ks.cu) is reachable through loza_debug_force_kernel. */
loza_status_t ssa_decode(const loza_attn_args_t* args, const int32_t* seq_lens_dev,
                         loza_pattern_t pattern, void* ws, size_t ws_bytes, loza_stream_t stream);

/* Full-attention comparator, Eq. 1 with a causal (or, for
 * causal = 0, bidirectional) mask. seq_lens_dev == NULL: prefill over
 * [q_start, q_start + n_q); otherwise decode as in ssa_decode over the whole
 * context [0, seq_len). ws sized by loza_workspace_size(LOZA_WS_FULL_DECODE, ...). */
loza_status_t full_attn_ref(const loza_attn_args_t* args, const int32_t* seq_lens_dev, void* ws,
                            size_t ws_bytes, loza_stream_t stream);

/* LoZA calibration blend, Eq. 3:
 *   o_hat = alpha * o_full + (1 - alpha) * o_sparse, evaluated as
 *   fma(alpha, o_full, (1-alpha) * o_sparse) in fp32 so alpha in {0, 1} is exact,
 * and, if d_o_hat and d_alpha_dev are non-NULL, the scalar gradient
 *   d_alpha = sum_e d_o_hat[e] * (o_full[e] - o_sparse[e])
 * (per-thread fp32, per-CTA fp64, final fixed-order fp64 sum: deterministic).
 * All arrays contiguous, numel elements of `dtype`; alpha_dev one device fp32.
 * o_hat may be NULL (gradient only). If alpha is NaN or outside [0, 1] the kernel
 * writes LOZA_ERR_INVALID to status_dev (if non-NULL) and NaN to d_alpha
 * (out-of-range alpha is a contract error); otherwise it writes
 * LOZA_OK to status_dev. ws: loza_workspace_size(LOZA_WS_BLEND, ...) bytes,
 * required when d_alpha_dev != NULL. numel must be a multiple of 8 and
 * pointers 16-byte aligned (LOZA_ERR_SHAPE). */
loza_status_t loza_blend(const void* o_full, const void* o_sparse, const float* alpha_dev, void* o_hat,
                         const void* d_o_hat, double* d_alpha_dev, int64_t numel, loza_dtype_t dtype,
                         int32_t* status_dev, void* ws, size_t ws_bytes, loza_stream_t stream);

/* Fused calibration forward (Eq. 3, with O' = the SSA prefill of
 * `args`, Eq. 4): the SSA result O' is blended in the prefill epilogue and never written to HBM,
 *   args->o <- o_hat = fma(alpha, o_full, (1 - alpha) * O')   with O' in fp32 before rounding,
 * so alpha = 0 gives exactly ssa_prefill's bf16 output and alpha = 1 gives o_full; and, if d_o_hat
 * and d_alpha_dev are non-NULL,
 *   d_alpha = sum_e d_o_hat[e] * (o_full[e] - O'[e])
 * (per thread fp32 per 128 outputs, then fp64; per-CTA fp64 partials; final fixed-order fp64 sum:
 * deterministic). o_full and d_o_hat use o's layout and strides ([B, n_q, H, d_v], rows contiguous).
 * bf16 in and out, the absorbed MLA shape only (else LOZA_ERR_UNSUPPORTED); same validation as
 * ssa_prefill; o_full / d_o_hat 16-byte aligned (LOZA_ERR_SHAPE). alpha out of [0, 1] or NaN: the
 * output is computed with that alpha, LOZA_ERR_INVALID goes to status_dev (if non-NULL) and NaN to
 * d_alpha. ws: loza_workspace_size(LOZA_WS_BLEND, ...) bytes, required when d_alpha_dev != NULL. */
loza_status_t ssa_prefill_blend(const loza_attn_args_t* args, loza_pattern_t pattern, const void* o_full,
                                const float* alpha_dev, const void* d_o_hat, double* d_alpha_dev,
                                int32_t* status_dev, void* ws, size_t ws_bytes, loza_stream_t stream);

/* Attention backward: the gradients of Eq. 4 (sparse = 1, `pattern`) or Eq. 1 (sparse = 0,
 * args->causal) for a loss with dL/dO = d_o. args describes the FORWARD call (q, k, v, o, softmax_scale,
 * q_start, layouts as in ssa_prefill) and args->lse (the forward's LSE [B, H, n_q], natural log) is required;
 * d_o has o's dtype and layout. Outputs (fp32, contiguous):
 *   d_q [B, n_q, H, d_qk] = scale * sum_j dS_rj k_j,    dS_rj = P_rj (d_o_r . v_j - d_o_r . o_r)
 *   d_k [B, n_kv, d_qk]   = scale * sum_r dS_rj q_r,    P_rj  = exp(scale q_r . k_j - lse_r)
 *   d_v [B, n_kv, d_v]    = sum_r P_rj d_o_r
 * summed over every query row (all heads) that attends the key (n_q == 0: d_k = d_v = 0, and d_o, lse, d_q
 * may be NULL). For the absorbed MLA cache (v = the first
 * d_v columns of k) the cache gradient is d_k + [d_v, 0]. Deterministic (no atomics), fp32 accumulation;
 * d_qk <= 576, d_v <= 512 (else LOZA_ERR_UNSUPPORTED). bf16 with d_qk 576, d_v 512 and v aliasing k runs
 * on the tensor cores (tcgen05 when q / d_o rows are packed token x head; P and dS enter the second
 * products as bf16), everything else on FFMA.
 * ws: loza_workspace_size(LOZA_WS_BACKWARD, args, pattern, 1) bytes: D [B, n_q*H] fp32, for SSA the sink-tile
 * partials, the local-tile row-split partials (short sequences, sized from the current device's SM count:
 * query the size on the device that runs the call) and the dS rows [B, n_q*H, (s+l)*b] bf16 (1 GiB at B1, 8K
 * tokens, H64, (1,7,128)). */
loza_status_t attention_backward(const loza_attn_args_t* args, int32_t sparse, loza_pattern_t pattern,
                                 const void* d_o, float* d_q, float* d_k, float* d_v, void* ws, size_t ws_bytes,
                                 loza_stream_t stream);

/* SSA prefill in the non-absorbed (MHA) form of MLA (Eq. 4, applied to the
 * per-head keys/values an MLA layer produces when its latent window is up-projected). Each head
 * h has its own K, V: q [B, n_q, H, 192] (128 nope + 64 RoPE dims), k [B, n_kv, H, 192], v [B, n_kv, H, 128],
 * o [B, n_q, H, 128]; args->k_stride_b / k_stride_tok / v_* are the batch / token strides and
 * k_stride_head / v_stride_head the head strides, all in elements (any layout whose innermost dimension is
 * contiguous and whose strides are multiples of 16 bytes). Same selection as ssa_prefill (sparse = 1, b %
 * 128 == 0) or, with sparse = 0, the full-attention comparator of Eq. 1 (causal, or bidirectional with
 * q_start == 0). bf16 inputs; o bf16 (RN-even) or fp32; optional lse [B, H, n_q]. Returns
 * LOZA_ERR_UNSUPPORTED for other head dims, LOZA_ERR_SHAPE for misaligned pointers/strides. */
loza_status_t ssa_prefill_mha(const loza_attn_args_t* args, int64_t k_stride_head, int64_t v_stride_head,
                              int32_t sparse, loza_pattern_t pattern, loza_stream_t stream);

/* Bounded SSA KV cache. Per sequence R = (s+l)*b rows:
 * the s sink blocks at rows [0, s*b) and a ring of l blocks, block kb >= s at rows
 * s*b + ((kb - s) mod l)*b. Appending in position order evicts a local block exactly when it can no longer
 * be attended (block-boundary eviction), so after positions [0, t) were appended the cache holds every key
 * allowed for the query at t and nothing else; (s+l)*b*d*elem bytes per sequence whatever the context
 * (B64 at 1M: 75 MB instead of 77 GB).
 *
 * ssa_ring_append: copy m new rows per sequence (rows [B, m, d], strides in elements) at absolute positions
 * pos0_dev[b] .. pos0_dev[b] + m - 1 (pos0 = the sequence's length before the append, on the device) into
 * `cache` [B, (s+l)*b, d]. Rows evicted within the same append are skipped (a whole prompt is appended with
 * m = n, pos0 = 0). d*elem must be a multiple of 16 and base pointers / strides 16-byte aligned
 * (LOZA_ERR_SHAPE). */
loza_status_t ssa_ring_append(const void* rows, int64_t rows_stride_b, int64_t rows_stride_tok, int32_t m,
                              const int32_t* pos0_dev, loza_pattern_t pattern, void* cache, int64_t cache_stride_b,
                              int64_t cache_stride_tok, int32_t batch, int32_t d, loza_dtype_t dtype,
                              loza_stream_t stream);

/* ssa_decode over the bounded ring cache: args->k / args->v point into the ring cache, args->n_kv must be
 * (s+l)*b; seq_lens_dev are absolute lengths (any value >= 1: the ring holds the window of position
 * seq_len - 1 once positions [0, seq_len) were appended). Bitwise identical to ssa_decode over a contiguous
 * cache with the same rows. bf16, H <= 64, b % 128 == 0 and 2*batch <= SM count (the CTA-pair kernels);
 * else LOZA_ERR_UNSUPPORTED. No workspace (no status word: out-of-range seq_lens are clamped silently). */
loza_status_t ssa_decode_ring(const loza_attn_args_t* args, const int32_t* seq_lens_dev, loza_pattern_t pattern,
                              loza_stream_t stream);

/* Sequence-parallel SSA prefill (north star; SURVEY.md §8 a10 / e; "uniform compute across
 * all ranks"). Rank r of `world` owns the contiguous, block-aligned shard of one
 * sequence at positions [q_start, q_start + n_local) with n_local = args->n_q,
 * q_start = r * n_local (equal shards), and k/v holding exactly the shard's own
 * rows (args->n_kv == n_local; k row 0 = position q_start; rows contiguous).
 * The exchange is the plan loza_seqpar_plan returns, in two NCCL groups:
 *   1. on `stream`: rank 0 broadcasts its first s*b KV rows (the sink blocks);
 *   2. on a library-owned communication stream forked from `stream`: rank r sends
 *      its last (l-1)*b KV rows to rank r+1 and receives the halo from rank r-1.
 * The shard's query blocks [l-1, n_local/b) need only [sink | shard] and run on
 * `stream` while the halo is in flight; the first l-1 blocks (the only ones that
 * reach into the halo) run after it, over the segmented KV [sink | halo | shard].
 * The output stays sharded (o/lse hold the shard's rows); no gather, no LSE merge.
 * Splitting the launch does not change any result: every 128-row unit is computed
 * the same way in either launch (tests: bitwise equal to the one-GPU ssa_prefill).
 * Requires n_local % b == 0 and n_local >= max(s, l-1) * b (LOZA_ERR_SHAPE).
 * `comm` (an ncclComm_t of `world` ranks) may be NULL when world == 1.
 * ws: loza_workspace_size(LOZA_WS_SEQPAR, args, pattern, world) bytes.
 * The communication stream and its two events are created once per (host thread,
 * device) and reused (the only state the library keeps). */
loza_status_t ssa_seqpar_prefill(const loza_attn_args_t* args, loza_pattern_t pattern, loza_nccl_comm_t comm,
                                 int32_t rank, int32_t world, void* ws, size_t ws_bytes, loza_stream_t stream);

/* One transfer of the sequence-parallel exchange (host description, no device work). */
enum { LOZA_XFER_BCAST = 0, LOZA_XFER_SEND = 1, LOZA_XFER_RECV = 2 };
typedef struct {
  int32_t op;         /* LOZA_XFER_*; BCAST is group 1 (sink), SEND / RECV group 2 (halo) */
  int32_t peer;       /* BCAST: root rank (0); SEND: destination rank; RECV: source rank */
  int32_t batch;      /* sequence index b in [0, B) */
  int32_t tensor;     /* 0 = k rows, 1 = v rows (only when v does not alias k) */
  int64_t src_row;    /* first row moved, as a row index of the SENDER's shard (BCAST: the root's) */
  int64_t rows;       /* rows moved */
  int64_t row_elems;  /* elements per row (d_qk for k, d_v for v) */
  int64_t ws_offset;  /* byte offset of the destination in ws; -1 = none (the BCAST root keeps its rows) */
} loza_xfer_t;

/* The exchange plan of rank `rank` (host only; callable without a GPU): writes up to max_out entries to
 * out and returns their number (>= 0; the full count even when max_out is smaller), or -(status) if the
 * arguments are invalid for ssa_seqpar_prefill (see loza_last_error()). Entries are listed in issue order. */
int32_t loza_seqpar_plan(const loza_attn_args_t* args, loza_pattern_t pattern, int32_t rank, int32_t world,
                         loza_xfer_t* out, int32_t max_out);

/* The segmented KV view rank `rank` attends over after the exchange (host only): for segment i < the returned
 * count (1..3), seg_out[6*i + 0..5] = (pos_begin, pos_end, byte offset in ws of its k rows for batch 0, same
 * for its v rows, k batch stride in bytes, v batch stride in bytes); offsets are -1 for the shard's own k / v
 * (then the strides are the args' ones). Returns -(status) on invalid arguments. Key at absolute position j
 * of batch b lives in the segment with pos_begin <= j < pos_end, at row j - pos_begin. */
int32_t loza_seqpar_segments(const loza_attn_args_t* args, loza_pattern_t pattern, int32_t rank, int32_t world,
                             int64_t* seg_out);

/* Test hook ("virtual ranks"): ssa_seqpar_prefill with every RECV / BCAST of the
 * plan done by a device-to-device copy from the other shards' k/v on this GPU
 * (rank0_k/v: rank 0's shard base; prev_k/v: rank r-1's shard base; ignored for
 * rank 0); same streams, same split launch. */
loza_status_t loza_seqpar_prefill_local(const loza_attn_args_t* args, loza_pattern_t pattern, int32_t rank,
                                        int32_t world, const void* rank0_k, const void* rank0_v,
                                        const void* prev_k, const void* prev_v, void* ws, size_t ws_bytes,
                                        loza_stream_t stream);

/* Test hook ("NCCL loopback"): like loza_seqpar_prefill_local, but the plan's transfers go through NCCL on
 * a ONE-rank communicator `comm` (e.g. torch's ProcessGroupNCCL at world size 1): each BCAST becomes
 * ncclBroadcast(rank 0's rows -> ws, root 0), each RECV an ncclSend(rank r-1's rows, peer 0) +
 * ncclRecv(ws, peer 0) pair in the same group (SEND entries are the next virtual rank's RECVs). Exercises
 * the NCCL calls, counts, datatypes and offsets of ssa_seqpar_prefill on one GPU without cross-process
 * waits. */
loza_status_t loza_seqpar_prefill_loopback(const loza_attn_args_t* args, loza_pattern_t pattern,
                                           loza_nccl_comm_t comm, int32_t rank, int32_t world,
                                           const void* rank0_k, const void* rank0_v, const void* prev_k,
                                           const void* prev_v, void* ws, size_t ws_bytes, loza_stream_t stream);

/* Test hook for the integer prologue: for the query blocks of
 * queries [q_start, q_start + n_q) (q_start % b == 0), local block qb:
 *   idx_dev[qb*(s+l) + t] = t-th selected key block (absolute, ascending), -1 padded;
 *   count_dev[qb] = |sel| = number of selected key blocks.
 * sel(QB) = {kb <= QB : kb < s or QB - kb < l} (closed form of the mask). */
loza_status_t ssa_select_blocks(int64_t n_q, int64_t q_start, loza_pattern_t pattern, int32_t causal,
                                int32_t* idx_dev, int32_t* count_dev, loza_stream_t stream);

enum { LOZA_WS_DECODE = 0, LOZA_WS_FULL_DECODE = 1, LOZA_WS_BLEND = 2, LOZA_WS_SEQPAR = 3, LOZA_WS_BACKWARD = 4 };
/* Workspace bytes for `which`; args may be NULL for LOZA_WS_BLEND. */
size_t loza_workspace_size(int32_t which, const loza_attn_args_t* args, loza_pattern_t pattern, int32_t world);
/* Zero-fill a workspace of `which` (its loza_workspace_size bytes) on `stream`: the required one-time
 * initialisation of the decode workspaces (status word, split counters); harmless for the others. */
loza_status_t loza_workspace_init(int32_t which, const loza_attn_args_t* args, loza_pattern_t pattern, int32_t world,
                                  void* ws, size_t ws_bytes, loza_stream_t stream);

const char* loza_status_string(loza_status_t status);
const char* loza_last_error(void);           /* thread-local text of the last error, "" if none */
uint64_t loza_kernel_launches(void);         /* number of library kernel launches so far (process) */
int32_t loza_num_sms(void);                  /* SM count of the current device (0 if unknown) */
/* Test hook: override the automatic kernel choice of a family, process-wide (the library never reads the
 * environment). "decode": 0 auto, 1 pair-cooperative (H <= 64), 2 key-split pair; "backward": 0 auto, 1 FFMA
 * kernels, 2 warp-MMA key and row kernels, 3 tcgen05 key kernel + warp-MMA row kernel for dQ, 4 the 32-key
 * tcgen05 key kernel (dK and dV in one pass) instead of the 64-key dV / dK kernel pair, 5 the 64-key dV / dK
 * kernels instead of the 128-key CTA-pair kernels (SSA with b = 128). A forced
 * kernel that cannot take a problem falls back to the automatic choice. Returns 0, or -1 for an unknown
 * family / variant. */
int32_t loza_debug_force_kernel(const char* family, int32_t variant);

#ifdef __cplusplus
}
#endif
#endif /* LOZA_H_ */
