/*
 * droidspeak.h — C ABI of the B200-native DroidSpeak cross-model prefill path.
 *
 * Plain C: device/host pointers, sizes and cudaStream_t passed as void*.  No
 * torch types.  Every entry point validates all arguments before its first
 * kernel launch (an error never leaves a half-written cache), returns a
 * ds_status, and records a message retrievable with ds_last_error()
 * (thread-local).  Nothing allocates device memory: callers pass workspace.
 *
 * Each entry point names the reference interface it replaces
 * (/root/reference/pkg/src/crosskv/...).  INTEGRATION.md shows the ctypes
 * binding a crosskv maintainer would add.
 */
#ifndef DROIDSPEAK_H
#define DROIDSPEAK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DS_ABI_VERSION 2

#if defined(__GNUC__)
#define DS_API __attribute__((visibility("default")))
#else
#define DS_API
#endif
#define DS_PAGE_SIZE 64 /* tokens per KV page */

/* Status codes -> Python exceptions (errors.py:6-27):
 * DS_ERR_INVALID -> ValueError, DS_ERR_CACHE_MISS -> CacheMissError(layer, kind),
 * DS_ERR_DEGENERATE -> DegenerateInputError, DS_ERR_CUDA -> RuntimeError. */
enum ds_status { DS_OK = 0, DS_ERR_INVALID = 1, DS_ERR_CACHE_MISS = 2, DS_ERR_DEGENERATE = 3, DS_ERR_CUDA = 4 };
enum ds_miss_kind { DS_MISS_NONE = 0, DS_MISS_KV = 1, DS_MISS_E = 2 };

/* ModelConfig (model.py:70-124) minus the seed.  mlp_kind: DS_MLP_UNGATED is the
 * reference block (silu(x W1) W2, model.py:532-533); DS_MLP_SWIGLU is the
 * Llama-3 MLP (silu(x Wg) * (x Wu)) W2 with W1 = [2*d_ff][d] holding gate and
 * up rows interleaved in blocks of 16 (rows 32b..32b+15 gate, 32b+16..32b+31 up). */
enum ds_mlp_kind { DS_MLP_UNGATED = 0, DS_MLP_SWIGLU = 1 };
typedef struct ds_dims {
  int32_t n_layers, d_model, n_heads, n_kv_heads, head_dim, d_ff, vocab_size, max_seq;
  int32_t mlp_kind;
} ds_dims;

/* One layer's weights on device.  Matrices are the reference's [in,out]
 * tensors (model.py:256-270) transposed once to K-major [out][in] bf16. */
typedef struct ds_layer_weights {
  const void* wqkv;    /* bf16 [(H+2*KVH)*D][d] = concat(wq, wk, wv)^T */
  const void* wo;      /* bf16 [d][H*D]          = wo^T */
  const void* w1;      /* bf16 [d_ff][d] = w1^T (ungated) or [2*d_ff][d] interleaved gate/up (SwiGLU) */
  const void* w2;      /* bf16 [d][d_ff]         = w2^T */
  const float* g_attn; /* f32 [d] */
  const float* g_mlp;  /* f32 [d] */
} ds_layer_weights;

/* ModelWeights (model.py:234-243) on device. */
typedef struct ds_model {
  ds_dims dims;
  const void* embed;              /* bf16 [V][d] */
  const void* unembed;            /* bf16 [V][d] = unembed^T */
  const float* g_final;           /* f32 [d] */
  const float* rope_cos;          /* f32 [max_seq][D/2] (angles in f64, model.py:475-479) */
  const float* rope_sin;          /* f32 [max_seq][D/2] */
  const ds_layer_weights* layers; /* HOST array [n_layers] */
} ds_model;

/* A K/V cache over layers.  Element offset of (layer, head, pos, j):
 *   layer*layer_stride + head*head_stride + table[pos/64]*page_stride + (pos%64)*head_dim + j
 * Dense export [L][KVH][n][D] (LayerKV, model.py:342-370):
 *   layer_stride = KVH*n*D, head_stride = n*D, page_stride = 64*D, block_table = NULL.
 * Consumer paged cache [L][pages][KVH][64][D]:
 *   layer_stride = pages*KVH*64*D, head_stride = 64*D, page_stride = KVH*64*D. */
typedef struct ds_kv_cache {
  void* k;                    /* bf16 */
  void* v;                    /* bf16 */
  int64_t layer_stride, head_stride, page_stride;
  const int32_t* block_table; /* device int32 [ceil(positions/64)] or NULL (identity) */
  int32_t n_layers;           /* layers addressable */
  int32_t positions;          /* positions present per layer */
  /* Optional HOST arrays [n_layers] of per-layer K / V bases (replacing
   * k/v + layer*layer_stride); a NULL entry means the layer is absent (a
   * cache miss).  Used for per-layer store payloads (store.py:351-395) that
   * the ingest kernel reads in place — including peer-GPU memory. */
  void* const* layer_k;
  void* const* layer_v;
} ds_kv_cache;

/* ECache (model.py:373-391): residual-stream input of `layer`, f32 [positions][width]
 * (exact, as the reference keeps it: the recompute resumes the producer's residual
 * stream bit for bit). */
typedef struct ds_e_cache {
  int32_t layer;
  int32_t positions;
  int32_t width;
  const void* hidden;
} ds_e_cache;

DS_API int ds_abi_version(void);
DS_API const char* ds_last_error(void);
/* Kernels this library has launched in this process (benchmark evidence). */
DS_API unsigned long long ds_launch_count(void);

/* Stage timeline (profiling aid, this host thread only).  Between
 * ds_trace_begin() and ds_trace_end(), ds_partial_prefill / ds_full_prefill
 * record a timing event at every stage boundary on the stream the stage ran
 * on: tag 0 = step start, DS_TRACE_INGEST, DS_TRACE_QKV + l (layer l's window
 * K/V in the cache), DS_TRACE_LAYER + l (window layer l done), DS_TRACE_ANCHOR + l
 * (anchor row through layer l), DS_TRACE_LOGITS.  ds_trace_end synchronises the
 * events and writes up to `cap` (ms since the step start, tag) pairs; it returns
 * the number of events (or -1).  Not capturable into a CUDA graph. */
enum { DS_TRACE_INGEST = 1, DS_TRACE_QKV = 1000, DS_TRACE_LAYER = 2000, DS_TRACE_ANCHOR = 3000, DS_TRACE_LOGITS = 4000 };
DS_API int ds_trace_begin(void);
DS_API int ds_trace_end(float* ms_out, int32_t* tag_out, int32_t cap);
/* SM id of each CTA of the last persistent anchor launch that used this
 * workspace (one CTA per SM is the design; profiling aid).  Returns the count, or -1. */
DS_API int ds_anchor_placement(const ds_dims* dims, int32_t n_tokens, const void* workspace, int32_t* sm_out,
                               int32_t cap);
/* Global-timer ns of the last persistent anchor launch on this workspace: after
 * its seed, then after each of the 5 phases (qkv, attention, o-proj, w1, w2) of
 * every layer.  Returns the count (1 + 5 * n_layers), or -1. */
DS_API int ds_anchor_timeline(const ds_dims* dims, int32_t n_tokens, const void* workspace, uint64_t* ns_out,
                              int32_t cap);

/* Anchor-shape override for measurements and tests (process-wide):
 * 0 = by workload (the persistent co-resident kernel when k * P >= 800 * L),
 * 1 = always the persistent kernel when it fits, 2 = always the per-launch
 * kernels.  Both shapes run the same arithmetic (bit-identical results).
 * The DS_ANCHOR_SHAPE environment variable sets the initial value.  Returns
 * the previous value, or -1 for an unknown shape. */
DS_API int ds_set_anchor_shape(int32_t shape);
/* Fused calls that ran the per-launch anchor because another call's fused step
 * (persistent anchor) was still in flight on the same GPU on other streams
 * (one persistent anchor per GPU at a time).  Process-wide count. */
DS_API unsigned long long ds_fused_fallbacks(void);

/* Bytes of device workspace ds_partial_prefill / ds_full_prefill need for n tokens. */
DS_API size_t ds_workspace_size(const ds_dims* dims, int32_t n_tokens);

/* KV ingest — the reuse copy of _mixed_prefill (model.py:590-603):
 * for l in reused[0..n_reused) (HOST array, ascending): dst[l, :, 0:window] = src[l, :, 0:window],
 * bit-exact bf16, TMA bulk-copied 64-position page blocks.  Misses (src lacks
 * layer l or window positions) are reported in ascending layer order. */
DS_API int ds_kv_ingest(const ds_kv_cache* src, const ds_kv_cache* dst, const int32_t* reused, int32_t n_reused,
                 int32_t window, int32_t n_kv_heads, int32_t head_dim, void* stream, int32_t* miss_layer);

/* Consumer partial prefill — partial_prefill (model.py:660-679) / the paper's
 * partial_prefill(recompute_config, context).
 *   tokens_host   int64 [n] (validated here: check_tokens, model.py:425-437)
 *   tokens_dev    optional device copy (NULL: copied into the workspace on compute_stream)
 *   groups        HOST int32 [n_groups][2], RecomputeConfig normal form (model.py:166-178)
 *   sender_kv     producer export (may be NULL iff groups cover every layer)
 *   sender_e      E caches; one per transition layer (group start > 0)
 *   out_kv        consumer cache receiving K/V for positions 0..n-1 of every layer
 *   logits_out    device f32 [V];  token_out  device int32 [1] (argmax, lowest id on ties)
 *   copy_stream   optional second stream: the anchor pass (with the reused layers' KV
 *                 ingest fused into it) runs beside the recompute (sched.py:212-263)
 * On DS_ERR_CACHE_MISS, *miss_layer / *miss_kind name the first miss in the
 * reference's order (KV misses ascending, then E per group, model.py:590-617). */
DS_API int ds_partial_prefill(const ds_model* m, const int64_t* tokens_host, const int64_t* tokens_dev, int32_t n_tokens,
                       const int32_t* groups, int32_t n_groups, const ds_kv_cache* sender_kv,
                       const ds_e_cache* sender_e, int32_t n_e, const ds_kv_cache* out_kv, float* logits_out,
                       int32_t* token_out, void* workspace, size_t workspace_bytes, void* compute_stream,
                       void* copy_stream, int32_t* miss_layer, int32_t* miss_kind);

/* Producer export — full_prefill (model.py:641-649): K/V of all n positions into
 * out_kv, E (f32 [n-1][d]) for each layer listed in e_layers (store_prefill's
 * serving-mode filter keeps only transition layers, store.py:202-203), logits.
 * Same structure as the reference (_mixed_prefill: the window through every
 * layer, then the anchor row), so it equals ds_partial_prefill with every layer
 * recomputed bit for bit.  copy_stream: optional, the anchor beside the window. */
DS_API int ds_full_prefill(const ds_model* m, const int64_t* tokens_host, const int64_t* tokens_dev, int32_t n_tokens,
                    const ds_kv_cache* out_kv, const int32_t* e_layers, int32_t n_e, void* const* e_out,
                    float* logits_out, int32_t* token_out, void* workspace, size_t workspace_bytes,
                    void* stream, void* copy_stream);

/* ---- stage entry points (the layer-pipelined scheduler drives these on its own
 * streams: ingest on the link stream, recompute gated on E, anchor last;
 * sched.py:212-263) ---- */

/* Selective recompute of ONE group [a, b] over the window positions 0..n-2
 * (model.py:607-625): h = embed[tokens[0..n-1)] (a == 0, tokens_dev required)
 * or the sender's E at layer a (seed: f32 [seed_positions >= n-1][d], may live
 * in a peer GPU's HBM); layers a..b run over the window and write K/V of
 * positions 0..n-2 into out_kv.  The E read is the first kernel of the group, so
 * a peer-resident seed is pulled over NVLink by the compute itself. */
DS_API int ds_recompute_group(const ds_model* m, const int64_t* tokens_dev, int32_t n_tokens, int32_t a, int32_t b,
                              const void* seed, int32_t seed_positions, const ds_kv_cache* out_kv, void* workspace,
                              size_t workspace_bytes, void* stream);

/* Anchor pass (model.py:627-637): position n-1 through every layer with the
 * receiver's weights, attending over kv[l, :, 0..n-2] plus itself (its K/V are
 * written at n-1), then logits = RMSNorm(h)*g_final @ unembed and the greedy
 * token (lowest id on ties, model.py:779). */
DS_API int ds_anchor(const ds_model* m, const int64_t* tokens_dev, int32_t n_tokens, const ds_kv_cache* kv,
                     float* logits_out, int32_t* token_out, void* workspace, size_t workspace_bytes, void* stream);

/* Token-selective baseline (token_selective_prefill, model.py:682-743; the
 * CacheBlend comparison point): every layer starts from the
 * sender's K/V; the ceil(ratio * (n-1)) window positions whose receiver layer-0
 * K/V deviate most from the sender's (L2 over heads x head_dim, ties to the
 * lowest position) are recomputed through the whole stack, then the anchor.
 * *n_selected receives the count.  ratio is a double and the count is
 * ceil(ratio * (n-1)) in double precision, as the reference's math.ceil (a
 * float32 ratio would select one position more whenever ratio * (n-1) is an
 * integer in double, e.g. 0.1 * 10).  Misses: layer count first, then positions
 * (CacheMissError(layer, "kv")). */
DS_API int ds_token_selective_prefill(const ds_model* m, const int64_t* tokens_host, const int64_t* tokens_dev,
                                      int32_t n_tokens, const ds_kv_cache* sender_kv, double ratio,
                                      const ds_kv_cache* out_kv, float* logits_out, int32_t* token_out,
                                      int32_t* n_selected, void* workspace, size_t workspace_bytes, void* stream,
                                      int32_t* miss_layer);

/* Greedy decode (decode_greedy, model.py:751-788): tokens_out[0] = *first_token
 * (argmax of the prefill logits); each further step runs the previous token at
 * the next position through every layer over kv (appending its K/V at
 * positions, positions+1, ... -- the cache needs that capacity) and takes the
 * argmax (lowest id on ties).  Device int32 in/out. */
DS_API int ds_decode_greedy(const ds_model* m, const ds_kv_cache* kv, int32_t positions, const int32_t* first_token,
                            int32_t steps, int32_t* tokens_out, void* workspace, size_t workspace_bytes,
                            void* stream);

/* ---- batched requests (config 4: a consumer's batch of requests; batched decode) ----
 * The anchor rows of a batch share ONE stream of the weights per layer (a
 * GEMV over up to DS_MAX_BATCH rows) and one attention launch; each row's
 * arithmetic is the single-request pass's, so a batch gives its requests'
 * one-by-one results bit for bit.  Workspace: ds_workspace_size_batch(dims,
 * longest request (or positions + steps), batch). */
#define DS_MAX_BATCH 8
DS_API size_t ds_workspace_size_batch(const ds_dims* dims, int32_t max_tokens, int32_t batch);

/* `batch` partial prefills (model.py:660-679) with one RecomputeConfig, each
 * request its own tokens (varlen), producer export and output cache:
 *   tokens_host / tokens_dev  [batch] pointers (tokens_dev may be NULL or hold NULLs)
 *   sender_kv  [batch] (a request without an export: k = v = NULL), sender_e [batch]
 *   pointers to n_e[b] E caches; out_kv [batch]; logits_out device f32 [batch][V];
 *   token_out device int32 [batch].
 * Validation per request in the reference's order, requests in order; on error
 * *bad_request names the request (and *miss_layer / *miss_kind the miss).
 * copy_stream (optional): every request's reused-layer KV ingest beside the
 * compute stream's recompute of the batch; then one batched anchor pass. */
DS_API int ds_partial_prefill_batch(const ds_model* m, int32_t batch, const int64_t* const* tokens_host,
                                    const int64_t* const* tokens_dev, const int32_t* n_tokens, const int32_t* groups,
                                    int32_t n_groups, const ds_kv_cache* sender_kv, const ds_e_cache* const* sender_e,
                                    const int32_t* n_e, const ds_kv_cache* out_kv, float* logits_out,
                                    int32_t* token_out, void* workspace, size_t workspace_bytes,
                                    void* compute_stream, void* copy_stream, int32_t* bad_request,
                                    int32_t* miss_layer, int32_t* miss_kind);

/* Batched anchor pass (ds_anchor for `batch` rows): row b = token
 * anchor_tokens_dev[b] at position positions[b] (host) over kv[b]; logits
 * [batch][V], token_out [batch]. */
DS_API int ds_anchor_batch(const ds_model* m, int32_t batch, const int64_t* anchor_tokens_dev, const int32_t* positions,
                           const ds_kv_cache* kv, float* logits_out, int32_t* token_out, void* workspace,
                           size_t workspace_bytes, void* stream);

/* Batched greedy decode (ds_decode_greedy for `batch` sequences, each its own
 * cache and length): tokens_out device int32 [batch][steps]; first_token
 * device int32 [batch]; positions host int32 [batch]. */
DS_API int ds_decode_greedy_batch(const ds_model* m, int32_t batch, const ds_kv_cache* kv, const int32_t* positions,
                                  const int32_t* first_token, int32_t steps, int32_t* tokens_out, void* workspace,
                                  size_t workspace_bytes, void* stream);

/* ---- producer -> consumer over NVLink (P2P pull through CUDA IPC) ----
 * The producer exports a device buffer once; a consumer process maps it and
 * hands the mapped pointer to ds_kv_ingest (ds_kv_cache.k/v or layer_k/v) and
 * to ds_recompute_group (seed): the consumer's kernels then read the
 * producer's HBM in place over NVLink.  handle = 64 opaque bytes. */
#define DS_IPC_HANDLE_BYTES 64
DS_API int ds_ipc_export(const void* device_ptr, void* handle_out, uint64_t* offset_out);
/* Maps an exported buffer into this process: *base_out = mapping base (pass to
 * ds_ipc_close), *ptr_out = base + offset. */
DS_API int ds_ipc_open(const void* handle, uint64_t offset, void** base_out, void** ptr_out);
DS_API int ds_ipc_close(void* base);

/* ---- single-kernel entry points (used by the parity tests and the scheduler) ---- */

/* C = epilogue(A[M][K] . B[N][K]^T); mode 0 bf16 store, 1 f32 out = resid + acc,
 * 2 bf16 silu, 4 f32 store.  tcgen05/TMEM kernel. */
DS_API int ds_gemm(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc, const float* resid,
            int64_t ld_resid, int32_t M, int32_t N, int32_t K, int32_t mode, void* stream);

/* RMSNorm (model.py:466-468): out_bf16[r] = bf16(x[r] / sqrt(mean(x[r]^2) + 1e-6) * gain).
 * x is f32 (x_is_bf16 = 0) or bf16; optional row gather (int64 ids); optional f32 and
 * bf16 copies of the (gathered) input rows. */
DS_API int ds_rmsnorm(const void* x, int32_t x_is_bf16, const int64_t* gather, int32_t M, int32_t d, const float* gain,
               void* out_bf16, float* copy_f32, void* copy_bf16, void* stream);

/* Causal GQA flash-attention prefill over a cache layer (model.py:506-519):
 * q bf16 [n_q][H*D] (row r at absolute position q_pos0 + r, keys 0..q_pos0+r),
 * o bf16 [n_q][H*D]. */
DS_API int ds_attention_prefill(const void* q, int64_t ldq, const ds_kv_cache* kv, int32_t layer, int32_t n_q,
                         int32_t q_pos0, int32_t n_heads, int32_t n_kv_heads, int32_t head_dim, void* o,
                         int64_t ldo, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* DROIDSPEAK_H */
