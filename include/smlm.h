/*
 * smlm.h -- C ABI of the B200-native Segmented Multi-LoRA Multiplication (SMLM) library.
 *
 * What the library computes (§3.3 "Unified computation flow management
 * and SMLM kernel"): for one linear layer ("we adapt the Punica kernel to process LoRA weights
 * one linear layer at a time"), a single call computes, for every row of a packed mixed
 * batch, the base projection plus the LoRA term of the adapter assigned to the row's segment,
 * for all four request kinds ("fine-tuning (training), evaluation, prefilling, and decoding",
 * P:384), with a static per-adapter scale and an optional dynamic per-request scale.
 * The backward covers fine-tune rows only ("a shared backward pass") and masks
 * gradients per adapter (MixedLoRAModelForTrainer).  The adapter pool mirrors the
 * paper's Virtualized Module contract: adapters are loaded and unloaded at runtime without
 * re-splicing and the base weight is shared, never copied.
 *
 * Math (row t in segment g, adapter a = seg_slot[g], s = slot_scale[a] * seg_scale[g]):
 *     V[t]  = A_a x_t                         (rank-r intermediate)
 *     y_t   = W x_t + s B_a V[t]              (a == -1: y_t = W x_t)
 *   fine-tune rows only:
 *     U[t]  = B_a^T dy_t
 *     dx_t  = W^T dy_t + s A_a^T U[t]
 *     dA_a  = s sum_t U[t] x_t^T     dB_a = s sum_t dy_t V[t]^T
 *
 * Layout: row-major everywhere (nn.Linear / PEFT convention).
 *     X [S,in]   W [out,in]   A_a [r,in]   B_a [out,r]   Y [S,out]   V_save [S,r]
 *     dY [S,out] dX [S,in]    dA_a [r,in] (fp32)         dB_a [out,r] (fp32)
 * Element type of every tensor is the pool dtype (SMLM_BF16, or SMLM_FP32 test mode) except
 * dA/dB, which are always fp32.  All tensor pointers are DEVICE pointers unless marked "host".
 *
 * Ownership: the caller owns every tensor (X, W, Y, A, B, V_save, dY, dX, dA, dB, workspace).
 * smlm_adapter_register BORROWS A and B (zero copy): they must stay alive and unchanged in
 * shape until smlm_adapter_unregister has been ordered on the stream; their VALUES may be
 * updated in place (e.g. by an optimizer) between calls.  The pool owns only its slot table.
 *
 * Errors: every entry point validates on the host before anything is enqueued; on error no
 * output is touched and a status below is returned; smlm_last_error() gives a thread-local
 * message.  Asynchronous CUDA faults surface as SMLM_E_CUDA from a later call.
 * There is no CPU fallback: a device that is not sm_100 gives SMLM_E_UNSUPPORTED.
 *
 * Threading: all work is stream-ordered on the given stream with no host synchronisation
 * (plans ride in kernel parameters or a pinned ring buffer).  A pool must be used by one host
 * thread at a time.  Its calls may be issued on several streams (e.g. the next micro-batch's
 * forward overlapping this one's backward): the self-resetting cross-CTA counters of the split-K
 * passes and of the decode kernel are kept per launching stream, so only calls on the SAME
 * stream share them, and those are ordered.  A CUDA graph keeps the counters of its capture
 * stream: do not replay it concurrently with direct calls issued on that capture stream.
 * The decode kernel spin-waits across CTAs: its grid is capped to one co-resident wave
 * (cudaOccupancyMaxActiveClusters; a pure decode batch that does not fit takes the mixed-batch
 * path), and decode calls that may run concurrently on several streams need the pool option
 * SMLM_OPT_DEC_COOPERATIVE (cooperative launch).
 */
#ifndef SMLM_H_
#define SMLM_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SMLM_API __attribute__((visibility("default")))
#else
#define SMLM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct smlm_pool_s *smlm_pool; /* one pool per (layer, projection) */

enum smlm_status {
    SMLM_OK = 0,
    SMLM_E_INVALID = 1,     /* malformed offsets, mode outside 0..3, bad scale, null pointer */
    SMLM_E_SHAPE = 2,       /* shape or dtype mismatch */
    SMLM_E_SLOT = 3,        /* slot not registered / out of range */
    SMLM_E_CAPACITY = 4,    /* pool full */
    SMLM_E_CUDA = 5,        /* a CUDA runtime/driver error (sticky device errors included) */
    SMLM_E_UNSUPPORTED = 6, /* not an sm_100 device, or a shape/rank the dtype path lacks */
    SMLM_E_WORKSPACE = 7    /* workspace smaller than smlm_workspace_size() */
};

/* Request kinds, PAPER.md P:384 ("fine-tuning (training), evaluation, prefilling, and decoding") */
enum smlm_mode { SMLM_FINETUNE = 0, SMLM_EVAL = 1, SMLM_PREFILL = 2, SMLM_DECODE = 3 };

/* SMLM_BF16: bf16 tensors, fp32 accumulation on tcgen05 tensor cores (production path).
 * SMLM_FP32: fp32 tensors, fp32 SIMT kernels with chunked accumulation (1e-5 parity mode). */
enum smlm_dtype { SMLM_BF16 = 0, SMLM_FP32 = 1 };

/* Options for smlm_pool_set_option */
enum smlm_option {
    SMLM_OPT_L_LONG = 0,  /* segments with >= L_long rows take the long (per-segment tile) path; default 64 */
    SMLM_OPT_CTA_PAIR = 1, /* 1 (default): forward long tiles on CTA pairs (tcgen05 cta_group::2); 0: one CTA */
    SMLM_OPT_DECODE_KERNEL = 2, /* 1 (default): pure short/decode batches of <= 512 rows take the
                                 * single-launch decode kernel; 0: the mixed-batch path (same math) */
    SMLM_OPT_DEC_KSPLIT = 3,    /* decode kernel W split-K factor in [1, 8]; 0 (default) = automatic.
                                 * Changes only the fp32 summation order (results within tolerance) */
    SMLM_OPT_DEC_COOPERATIVE = 4 /* 1: launch the decode kernel cooperatively (whole grid co-scheduled);
                                  * needed when decode calls of several pools/streams can run at once
                                  * (two partially resident spin-waiting grids could wait on each
                                  * other).  0 (default): grid capped to one co-resident wave */
};

/*
 * Create a pool for one (layer, projection) of shape (in_features -> out_features) with LoRA
 * rank `rank` and room for `capacity` adapters, on CUDA device `device`.
 * bf16: rank in {8,16,32,64}; in/out multiples of 64.  fp32: 1 <= rank <= 64; in/out >= 1.
 * Errors: SMLM_E_INVALID (capacity < 1, null out), SMLM_E_UNSUPPORTED (device not sm_100,
 * rank/shape not supported by the dtype path), SMLM_E_CUDA.
 */
SMLM_API int smlm_pool_create(int device, int in_features, int out_features, int rank, int capacity,
                     int dtype, smlm_pool *out);
SMLM_API int smlm_pool_destroy(smlm_pool pool);
SMLM_API int smlm_pool_set_option(smlm_pool pool, int option, int value);

/*
 * Register (load) an adapter: A [rank,in], B [out,rank] (device, pool dtype, row-major,
 * 16-byte aligned, borrowed).  `scale` is the static slot scale alpha/r (> 0, finite; pass 1 if
 * the caller baked the scale into B).  The device slot table update is ordered on
 * `stream` (a cudaStream_t; NULL = legacy default stream).  Writes the slot index to *slot_out.
 * Errors: SMLM_E_INVALID, SMLM_E_CAPACITY (no free slot), SMLM_E_CUDA.
 */
SMLM_API int smlm_adapter_register(smlm_pool pool, const void *A, const void *B, float scale, void *stream,
                          int *slot_out);
/*
 * Same, for an adapter of its own rank r_a <= the pool rank (heterogeneous ranks in one layer,
 * SURVEY.md §8 f2): A [r_a,in], B [out,r_a].  The result is exactly that of the
 * adapter zero-padded to the pool rank (the kernels read rank indices >= r_a as zero), and its
 * gradient buffers are dA [r_a,in], dB [out,r_a].  bf16 pools: r_a a multiple of 8 in
 * [8, pool rank] (TMA row pitch); fp32 pools: r_a = pool rank.
 * Errors: as smlm_adapter_register, plus SMLM_E_SHAPE for a rank outside that range.
 */
SMLM_API int smlm_adapter_register_rank(smlm_pool pool, const void *A, const void *B, int rank, float scale,
                                        void *stream, int *slot_out);
/* Bind fp32 gradient buffers dA [rank,in], dB [out,rank] (device; rank = the adapter's) to a slot;
 * NULL = frozen (masked).  Takes effect for calls issued after it.  Errors: SMLM_E_SLOT. */
SMLM_API int smlm_adapter_set_grad(smlm_pool pool, int slot, float *dA, float *dB);
/* Unload an adapter; the slot may be reused by a later register.  Errors: SMLM_E_SLOT. */
SMLM_API int smlm_adapter_unregister(smlm_pool pool, int slot, void *stream);

/*
 * A segmented mixed batch (Alg. 1 Require P:326-329: rows packed over all requests).
 * All arrays are HOST memory, read during the call only.
 *   seg_offsets [G+1]: 0 = off[0] <= off[1] <= ... <= off[G] = S; empty segments allowed
 *   seg_slot    [G]  : -1 = base only, else a registered slot
 *   seg_mode    [G]  : SMLM_FINETUNE .. SMLM_DECODE
 *   seg_scale   [G]  : dynamic per-request scale (finite, > 0) or NULL (= 1); multiplies the
 *                      slot scale ("applied on a per-request basis during the forward pass")
 *   dropout_p, dropout_seed: LoRA dropout of the FINETUNE rows (App. D
 *                      Table 5 lora_dropout 0.05; PEFT y = W x + s B A dropout(x), training mode =
 *                      fine-tune rows only; R13).  p in [0, 1), 0 = off (zero-initialise
 *                      the struct); quantised to thr = round(p * 65536).  Element (t, k) of X is kept
 *                      iff u >= thr, u the 16-bit half (k odd: high) of
 *                      lowbias32(lowbias32((t * ceil(in/2) + k/2) ^ seed_lo) ^ seed_hi), and kept
 *                      elements are scaled by 65536 / (65536 - thr).  The forward and the backward of
 *                      one step must pass the same seed (the mask is recomputed, never stored).
 *                      smlm_forward_multi / smlm_backward_multi use seed + i * 0x9E3779B97F4A7C15 for
 *                      projection i (independent masks, as PEFT's per-module dropout).  bf16 pools
 *                      need SMLM_OPT_CTA_PAIR = 1 and W != NULL for fine-tune rows with dropout
 *                      (else SMLM_E_UNSUPPORTED).
 */
typedef struct {
    int S;
    int G;
    const int32_t *seg_offsets;
    const int32_t *seg_slot;
    const int8_t *seg_mode;
    const float *seg_scale;
    float dropout_p;
    uint64_t dropout_seed;
} smlm_batch;

/* Bytes of device workspace a forward (backward = 0) or backward (backward = 1) call needs. */
SMLM_API size_t smlm_workspace_size(smlm_pool pool, const smlm_batch *batch, int backward);

/*
 * Forward: Y = W X + s B_a (A_a X) per segment.
 *   X [S,in]; W [out,in] or NULL (then Y holds the base output on entry and only the LoRA term
 *   is added in place); Y [S,out]; V_save [S,rank] or NULL: receives the unscaled V = A_a x_t of
 *   every FINETUNE row that has an adapter (other rows untouched).
 *   ws: device workspace of ws_bytes >= smlm_workspace_size(pool, batch, 0).
 * Errors: SMLM_E_INVALID / SMLM_E_SLOT / SMLM_E_WORKSPACE / SMLM_E_CUDA; S == 0 or G == 0 is a
 * no-op returning SMLM_OK.
 */
SMLM_API int smlm_forward(smlm_pool pool, const smlm_batch *batch, const void *X, const void *W, void *Y,
                 void *V_save, void *ws, size_t ws_bytes, void *stream);

/*
 * Multi-projection forward (Alg. 1 P:331 computes q, k, v of a layer from
 * the same hidden states): for i in [0, n_proj), exactly the result of
 *     smlm_forward(pools[i], batch, X, W[i], Y[i], V_save ? V_save[i] : NULL, ...)
 * up to the fp32 summation order (within the bf16 tolerance), but a pure short/decode batch
 * (<= 512 rows, no segment >= L_long) runs as ONE launch that streams every W[i] once and reads X
 * once, and a mixed bf16 batch computes s*V of its long tiles for every projection in ONE
 * pre-shrink pass over X (n_proj * r_pad <= 128; bit-identical to the per-pool calls) before each
 * projection's short-row shrink, and (n_proj <= 3) all projections' GEMMs run as ONE persistent
 * CTA-pair launch over the n-tiles of every projection.  Otherwise (e.g. different slot scales
 * across pools) the per-pool calls run in sequence.
 *   n_proj in [1, 4]; pools share device, in_features, rank and dtype; every slot of the batch
 *   must be registered in every pool (else SMLM_E_SLOT);
 *   W[i] != NULL; Y[i] [S, out_i]; V_save NULL or an array of n_proj pointers (each may be NULL).
 *   ws: ws_bytes >= smlm_workspace_size_multi(n_proj, pools, batch).
 * The decode kernel uses pools[0]'s counters: calls that share pools[0] must be stream-ordered.
 */
SMLM_API size_t smlm_workspace_size_multi(int n_proj, const smlm_pool *pools, const smlm_batch *batch);
SMLM_API int smlm_forward_multi(int n_proj, const smlm_pool *pools, const smlm_batch *batch, const void *X,
                                const void *const *W, void *const *Y, void *const *V_save, void *ws,
                                size_t ws_bytes, void *stream);

/*
 * Backward over FINETUNE rows.
 *   X [S,in], W [out,in] (required when dX != NULL), dY [S,out];
 *   V_save [S,rank] from the forward, or NULL (V is then recomputed from X);
 *   dX [S,in] or NULL: FINETUNE rows written, other rows untouched;
 *   dA/dB of every slot that has grad buffers AND fine-tune rows in this batch are overwritten
 *   (accumulate = 0) or incremented (accumulate = 1) with the sum over all of that slot's
 *   fine-tune rows, reduced in the fixed canonical order (bitwise deterministic).  Slots with
 *   grad buffers but no fine-tune rows are untouched; slots without grad buffers get none.
 */
SMLM_API int smlm_backward(smlm_pool pool, const smlm_batch *batch, const void *X, const void *W,
                  const void *dY, const void *V_save, void *dX, int accumulate, void *ws,
                  size_t ws_bytes, void *stream);

/*
 * Multi-projection backward (SURVEY §8(f1) for the backward; "a shared backward
 * pass"; Alg. 1: q, k, v -- or gate, up -- read the same X): for i in [0, n_proj), exactly
 *     smlm_backward(pools[i], batch, X, W[i], dY[i], V_save ? V_save[i] : NULL, dX[i], accumulate, ...)
 * (bit-identical), but the dX GEMMs of all projections run as ONE persistent CTA-pair launch over
 * the n-tiles of every projection (no per-projection wave tail); each projection's U pass and
 * dA/dB contraction are its own launches.
 *   n_proj in [1, 3]; pools share device, in_features, rank, dtype and options; W[i], dY[i] [S,out_i]
 *   and dX[i] [S,in] non-NULL; V_save NULL or an array of n_proj pointers (each may be NULL).
 *   ws: ws_bytes >= smlm_workspace_size_backward_multi(n_proj, pools, batch).
 * Errors as smlm_backward; SMLM_E_INVALID for n_proj outside [1, 3], SMLM_E_SHAPE for pools that
 * differ in in_features / rank / dtype / options.
 */
SMLM_API size_t smlm_workspace_size_backward_multi(int n_proj, const smlm_pool *pools, const smlm_batch *batch);
SMLM_API int smlm_backward_multi(int n_proj, const smlm_pool *pools, const smlm_batch *batch, const void *X,
                                 const void *const *W, const void *const *dY, const void *const *V_save,
                                 void *const *dX, int accumulate, void *ws, size_t ws_bytes, void *stream);

/*
 * The canonical work plan (segment scheduler output), as int32
 * records of 6 words, written to HOST memory `items` (capacity max_items records);
 * *n_items receives the record count (also when the buffer is too small: SMLM_E_WORKSPACE).
 * smlm_plan is a pure host function (no device needed): slot_registered [capacity] host flags.
 */
SMLM_API int smlm_plan(const smlm_batch *batch, int capacity, const uint8_t *slot_registered, int l_long,
              int backward, int32_t *items, int max_items, int *n_items);
SMLM_API int smlm_plan_export(smlm_pool pool, const smlm_batch *batch, int backward, int32_t *items,
                     int max_items, int *n_items);

/*
 * AdamW step over the fine-tune adapters' parameters (Table 5, P:1067:
 * HF Trainer, learning_rate 2e-5; optimizer defaults = DESIGN.md R12; masking P:422 = the caller
 * puts only the trained adapters' parameters in the buffer).  One call = one optimizer step of ONE
 * fine-tune job (each job is its own trainer: its own clip norm over its own parameters and its
 * own step count; optim.AdamW calls this once per job on the job's contiguous sub-range of a
 * shared flat store).  All buffers are DEVICE memory of n elements with the same flat layout
 * (e.g. the job's adapters' A then B, concatenated):
 *   param [n] fp32 master weights, exp_avg [n], exp_avg_sq [n] fp32 optimizer state -- updated;
 *   grad [n] fp32 -- the (all-reduced) gradient sum; read, and zeroed if zero_grad != 0;
 *   param_bf16 [n] bf16 or NULL -- receives bf16(param) after the update (the tensors the pools
 *   borrow can be views of it, so the next forward sees the new weights).
 * With t = step (>= 1) and g = grad * grad_scale:
 *   if max_grad_norm > 0: g *= min(1, max_grad_norm / (||g||_2 + 1e-6))  (norm over the buffer)
 *   param *= 1 - lr * weight_decay;  m = beta1 m + (1 - beta1) g;  v = beta2 v + (1 - beta2) g^2
 *   param -= lr / (1 - beta1^t) * m / (sqrt(v) / sqrt(1 - beta2^t) + eps)
 * fp32 arithmetic; the clip norm is reduced in a fixed order (bitwise reproducible).  Clipping
 * needs ws of smlm_adamw_workspace_size() bytes (ws may be NULL otherwise).  Stream-ordered, no
 * host synchronisation; 1 launch (2 with clipping).
 * Errors: SMLM_E_INVALID (null/misaligned buffer: fp32 16-byte, bf16 8-byte; step < 1;
 * hyper-parameter out of range), SMLM_E_WORKSPACE, SMLM_E_UNSUPPORTED (current device not
 * sm_100), SMLM_E_CUDA.
 */
SMLM_API size_t smlm_adamw_workspace_size(void);
SMLM_API int smlm_adamw_step(float *param, float *exp_avg, float *exp_avg_sq, float *grad, void *param_bf16,
                             size_t n, int step, float lr, float beta1, float beta2, float eps,
                             float weight_decay, float grad_scale, float max_grad_norm, int zero_grad,
                             void *ws, size_t ws_bytes, void *stream);

/*
 * Fused cross-rank reduction of the fine-tune gradients + optimizer (BASELINE.json
 * north_star "the fine-tuning LoRA gradients are all-reduced ... over NVLink"; PAPER.md P:422 masking
 * = only the trained adapters' gradients are reduced).  Data-parallel ranks replicate the adapters;
 * rank r of N keeps a STAGING buffer of N gradient slots [N][n] fp32 (slot q = rank q's gradient,
 * same flat layout), binds its pools' dA/dB to views of ITS slot r, and maps the peers' staging
 * buffers over NVLink with the IPC calls below.  Then:
 *   smlm_pool_set_grad_fanout(pool, N - 1, deltas): the dA/dB contraction kernel stores every
 *     gradient value it writes at p AND at p + deltas[q] -- slot r of peer q's buffer (delta =
 *     peer base - own base, bytes, a multiple of 4) -- so the transfer overlaps the contraction
 *     tile by tile (plain stores: each rank is the only writer of its slot everywhere);
 *   smlm_fanout_signal(N, ready, stream): after the step's backward (stream order), a system-scope
 *     release increment of every rank's ready counter (an int in each rank's device memory,
 *     zero-initialised, peer-mapped; ready[q] = rank q's counter as mapped here);
 *   smlm_adamw_step_reduce(...): the AdamW step of smlm_adamw_step on g = sum_{q < n_slots} of
 *     grad_slots[q * slot_stride + i] IN RANK ORDER (deterministic, the same on every rank, so the
 *     replicas stay bit-identical), after waiting until *ready >= ready_target (= N x steps so far);
 *     zero_grad clears only slot own_slot.
 * Use two staging buffers alternating by step parity (a fast peer may write step t + 1 while this
 * rank still reads step t); the wait itself keeps ranks within one step of each other.
 * Errors: SMLM_E_INVALID (NULL, counts outside [1, 8], misaligned deltas / strides), SMLM_E_CUDA
 * (IPC failures), SMLM_E_UNSUPPORTED (fan-out on an fp32 pool with gradients).
 */
#define SMLM_IPC_HANDLE_BYTES 64
/* handle of the allocation that contains dev_ptr, and dev_ptr's byte offset in it; open returns the
 * allocation BASE in this process (add the offset); close unmaps it */
SMLM_API int smlm_ipc_get_handle(const void *dev_ptr, void *handle_out /* SMLM_IPC_HANDLE_BYTES, host */,
                                 uint64_t *offset_out);
SMLM_API int smlm_ipc_open_handle(const void *handle /* host */, void **base_out);
SMLM_API int smlm_ipc_close_handle(void *dev_ptr);
SMLM_API int smlm_pool_set_grad_fanout(smlm_pool pool, int n_peers, const int64_t *byte_deltas);
SMLM_API int smlm_fanout_signal(int n_ranks, int *const *ready_counters, void *stream);
/* the stream waits (device-side) until *ready >= target: every rank's slots of the step are in
 * this rank's staging buffer (the all-reduce post-condition; the sum itself is folded into the
 * consumer, e.g. smlm_adamw_step_reduce) */
SMLM_API int smlm_fanout_wait(const int *ready, int target, void *stream);
SMLM_API int smlm_adamw_step_reduce(float *param, float *exp_avg, float *exp_avg_sq, float *grad_slots, int n_slots,
                                   size_t slot_stride, int own_slot, void *param_bf16, size_t n, int step, float lr,
                                   float beta1, float beta2, float eps, float weight_decay, float grad_scale,
                                   float max_grad_norm, int zero_grad, const int *ready, int ready_target, void *ws,
                                   size_t ws_bytes, void *stream);

/*
 * The Alg. 1 attention branch (reading R14): for a
 * packed batch of segments, causal scaled-dot-product attention of every row over the keys of its
 * own request, grouped-query heads (query head h reads KV head h / (n_heads / n_kv_heads)):
 *   FINETUNE / EVAL / PREFILL segment (a fresh sequence): row i attends to the segment's rows 0..i;
 *     a PREFILL segment with seg_cache[g] >= 0 also writes its K/V rows to cache positions [0, L)
 *     ("Initialize KVCache for prefills");
 *   DECODE segment: row i is appended at cache position seg_past[g] + i ("Append KVCache for
 *     decodes") and attends to cache positions [0, seg_past[g] + i].
 *   Q [S, n_heads, 128], K / V [S, n_kv_heads, 128], O [S, n_heads, 128] bf16 (the projections'
 *   outputs: position encoding, e.g. RoPE, is applied by the caller); K_cache / V_cache
 *   [cache_slots, cache_capacity, n_kv_heads, 128] bf16; scale = softmax scale (1/sqrt(128)).
 *   head_dim must be 128; n_heads / n_kv_heads in {1, 2, 4, 8}.
 *   Host arrays: seg_offsets [G+1], seg_mode [G], seg_cache [G] (or NULL: no cache use),
 *   seg_past [G] (or NULL: 0).  ws: >= smlm_attention_workspace_size(batch, n_heads, n_kv_heads)
 *   bytes (device): the plan and the split-KV partials of the decode rows.
 * Forward only (fine-tune rows' attention gradients are outside the SMLM path).
 * Errors: SMLM_E_INVALID, SMLM_E_SHAPE, SMLM_E_UNSUPPORTED, SMLM_E_WORKSPACE, SMLM_E_CUDA.
 */
typedef struct {
    int S;
    int G;
    const int32_t *seg_offsets;
    const int8_t *seg_mode;
    const int32_t *seg_cache;
    const int32_t *seg_past;
} smlm_attn_batch;
SMLM_API size_t smlm_attention_workspace_size(const smlm_attn_batch *batch, int n_heads, int n_kv_heads);
SMLM_API int smlm_attention(const smlm_attn_batch *batch, int n_heads, int n_kv_heads, int head_dim, const void *Q,
                            const void *K, const void *V, void *O, void *K_cache, void *V_cache, int cache_slots,
                            int cache_capacity, float scale, void *ws, size_t ws_bytes, void *stream);

SMLM_API const char *smlm_status_string(int status);
SMLM_API const char *smlm_last_error(void);

/* ---- instrumentation (used by bench.py; not needed for correctness) ---- */
/* Number of kernels this library has launched in this process. */
SMLM_API uint64_t smlm_launch_count(void);
/* smlm_profile_enable(mask): for every kernel class k with bit k set in `mask`, the library records
 * CUDA events around its launches on the launching stream (0 disables; 1 = forward GEMM only;
 * 0xF = all).  smlm_profile_read synchronises those events and returns the summed milliseconds and
 * launch count for class `kind` (0 = forward GEMM, 1 = backward dX GEMM, 2 = short-row shrink,
 * 3 = dA/dB, 4 = AdamW step) since the last read, then resets that class.  Events between launches serialise
 * programmatic dependent launch, so enable only what is measured. */
SMLM_API int smlm_profile_enable(int on);
SMLM_API int smlm_profile_read(int kind, double *total_ms, int *count);

#ifdef __cplusplus
}
#endif
#endif /* SMLM_H_ */
