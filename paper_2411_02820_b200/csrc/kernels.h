// Internal kernel-launch interface shared by the .cu translation units.
// (The public C ABI is include/droidspeak.h; this header is not installed.)
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/droidspeak.h"
#include "common.cuh"

namespace ds {

enum EpiMode { EPI_STORE_BF16 = 0, EPI_RESID_F32 = 1, EPI_SILU_BF16 = 2, EPI_QKV_ROPE = 3, EPI_STORE_F32 = 4,
               EPI_SWIGLU_BF16 = 5 };

struct GemmEpi {
  int mode;
  int M, N;
  void* out;            // bf16 / f32 [M][ld_out]
  long long ld_out;
  const float* resid;   // EPI_RESID_F32 (may alias out)
  long long ld_resid;
  // EPI_QKV_ROPE
  int n_offset;         // column of the fused [q|k|v] projection that tile column 0 maps to
  int n_heads, n_kv_heads, head_dim;
  bf16* q_out;
  long long ld_q;
  KvAddr kv;
  int pos0;             // absolute position of row 0
  const int32_t* pos_rows;  // or, if set, the absolute position of each row (token-selective recompute)
  int group;            // raster: m-blocks per group (set by gemm_launch)
  int l2_hint;          // pair GEMM: 1 = B (weights) loaded L2 evict_last, A evict_first (long-K shapes)
  const float* rope_cos;  // [max_seq][head_dim/2]
  const float* rope_sin;
  unsigned int* done;   // optional: +1 per (tile, epilogue warp) once its stores are visible
  // RMSNorm folded into the GEMMs (model.py:466-468): RMSNorm(h)*g @ W = ((h*g) @ W) * inv_rms(h).
  // Producer side (EPI_RESID_F32): also store norm_out = bf16(h_new * norm_gain) and, per output
  // column tile nb, ssq_out[nb * ld_ssq + row] = sum of h_new^2 over the tile's columns.
  bf16* norm_out;
  const float* norm_gain;
  float* ssq_out;
  // Consumer side (QKV / SiLU / SwiGLU): scale each row's accumulator by
  // 1 / sqrt(sum_p ssq_in[p * ld_ssq + row] / norm_dim + 1e-6), partials summed in order.
  const float* ssq_in;
  int ssq_parts;
  int norm_dim;
  long long ld_ssq;
};

// Base of layer `layer`'s K (v = false) or V block in a cache descriptor:
// the per-layer pointer table when present, else base + layer * layer_stride.
inline bf16* kv_layer_base(const ds_kv_cache& c, int layer, bool v) {
  void* const* tab = v ? c.layer_v : c.layer_k;
  if (tab) return static_cast<bf16*>(tab[layer]);
  return static_cast<bf16*>(v ? c.v : c.k) + (long long)layer * c.layer_stride;
}
inline bool kv_layer_present(const ds_kv_cache& c, int layer) {
  return layer >= 0 && layer < c.n_layers && kv_layer_base(c, layer, false) && kv_layer_base(c, layer, true);
}

// Kernels of the two streams only share an SM when their shared-memory
// carveouts agree: the tcgen05 GEMM / attention need the maximum, so every
// kernel asks for it (otherwise an anchor GEMV waits for an SM to drain).
template <typename F>
inline bool prefer_max_smem(F* kern) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared) ==
         cudaSuccess;
}

// Function attributes are per device: a once-flag per (kernel, device).
struct PerDevice {
  int v[64] = {};
  int& operator()() {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess || d < 0) d = 0;
    return v[d & 63];
  }
};
// Raise a kernel's dynamic shared-memory limit to `bytes` (and ask for the
// maximum carveout) on the current device, once per size increase.
template <typename F>
inline cudaError_t ensure_smem_attr(F* kern, int bytes, PerDevice& seen) {
  int& s = seen();
  if (bytes <= s) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return e;
  prefer_max_smem(kern);
  s = bytes;
  return cudaSuccess;
}

template <typename F>
inline void prefer_max_smem_once(F* kern, PerDevice& seen) {
  int& s = seen();
  if (s & 1) return;
  prefer_max_smem(kern);
  s |= 1;
}

// Launch with programmatic stream serialization (PDL): the kernel may begin
// while the previous kernel in the stream drains; it must call pdl_wait()
// before touching anything the predecessor writes or reads.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                              Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

// Status of the launch just made; the CUDA error is kept for ds_last_error()
// (cudaGetLastError clears it, so the C ABI layer reads it from here).
extern thread_local cudaError_t g_cuda_err;
inline int launch_status(cudaError_t e = cudaGetLastError()) {
  if (e == cudaSuccess) return DS_OK;
  g_cuda_err = e;
  return DS_ERR_CUDA;
}

// Every kernel launch of this library bumps this counter (ds_launch_count()).
extern unsigned long long g_launches;
inline void count_launch(int n = 1) { __atomic_fetch_add(&g_launches, (unsigned long long)n, __ATOMIC_RELAXED); }

int make_tmap_bf16(CUtensorMap* map, const void* ptr, long long rows, long long cols, long long ld, int box_rows,
                   int box_cols);
int num_sms();
int gemm_launch(const void* A, long long lda, const void* B, long long ldb, int K, const GemmEpi& epi,
                cudaStream_t stream, int force_bn = 0, int max_ctas = 0);
unsigned int gemm_done_target(int M, int N);
int gemm_col_tile(int M, int N);  // output columns per epilogue tile (the ssq partial granularity)

// False when p is device memory of another GPU (a peer export mapped through
// CUDA IPC / peer access): kernels then read it with plain loads only.
bool ptr_on_this_device(const void* p);
int kv_ingest_launch(const ds_kv_cache& src, const ds_kv_cache& dst, const int32_t* layers_host, int n_layers,
                     int n_kv_heads, int head_dim, int window, cudaStream_t stream, bool background = false);

int rmsnorm_launch(const void* x, bool x_bf16, const int64_t* gather, int M, int d, const float* gain, bf16* out,
                   float* copy_f32, bf16* copy_bf16, int copy_rows, cudaStream_t stream);
int norm_seed_launch(const void* x, bool x_bf16, const int64_t* gather, int M, int d, int T, const float* gain,
                     bf16* out, float* copy_f32, float* ssq, long long ld, cudaStream_t stream);

// Causal GQA prefill attention over one cache layer.  layer_rows = rows of the
// layer region viewed as a [rows][head_dim] matrix (TMA bound).  Cache memory
// beyond the written positions must hold finite values (allocations are zeroed).
int attention_prefill_launch(const bf16* q, long long ldq, const bf16* k_layer, const bf16* v_layer,
                             long long head_stride, long long page_stride, long long layer_rows, const int32_t* table,
                             int n_q, int q_pos0, int n_heads, int n_kv_heads, int head_dim, bf16* o, long long ldo,
                             cudaStream_t stream, const int32_t* q_pos = nullptr);

// Token-selective (CacheBlend-style) baseline helpers, see select.cu.
int kv_deviation_launch(const bf16* k0, const bf16* v0, long long head_stride0, const ds_kv_cache& sender, int window,
                        int n_kv_heads, int head_dim, float* dev, cudaStream_t stream);
int select_topk_launch(const float* dev, int window, int n_sel, const int64_t* tokens, int32_t* sel_pos,
                       int64_t* sel_tok, cudaStream_t stream);

// Single-row GEMV (anchor pass); see anchor.cu.
struct GemvArgs {
  const bf16* W;
  long long ldw;
  int N, K;
  const float* x_f32;   // normalised when gain != nullptr
  const float* gain;
  const bf16* x_bf16;   // used when x_f32 == nullptr
  int mode;             // EPI_QKV_ROPE / EPI_RESID_F32 / EPI_SILU_BF16 / EPI_SWIGLU_BF16 / EPI_STORE_F32
  float* out_f32;
  const float* resid;
  bf16* out_bf16;
  int n_heads, n_kv_heads, head_dim, pos;
  bf16* q_out;
  KvAddr kv;
  const float* rope_cos;
  const float* rope_sin;
  unsigned long long* argmax;  // EPI_STORE_F32: packed (orderable value, ~index) max
  // TMA kernel: [ticket, done] words, zero at launch (the last CTA re-zeroes
  // them): tiles are claimed in order by whichever CTA is ready, instead of
  // blockIdx-strided, so CTAs that start late (an SM still merging the
  // attention before it) take fewer tiles.  nullptr: strided.
  unsigned int* tile_ctr;
};

int gemv_launch(const GemvArgs& a, cudaStream_t stream, bool staged = true);
constexpr int kGemvCtrWords = 16;  // workspace words for GemvArgs::tile_ctr pairs (5 launch roles used)
int argmax_finalize_launch(const unsigned long long* packed, int32_t* token, int64_t* token64, cudaStream_t stream);

// Batched GEMV: nb rows (requests) against one weight stream.  Row b's view is
// GemvArgs `a` with x / out / resid / out_bf16 advanced by b * stride, q_out by
// b * q_stride, argmax by b, and the QKV epilogue's position and cache from
// pos[b] / kv[b].  Every row's result is the single-row GEMV's bit for bit.
constexpr int kMaxBatch = 8;
struct GemvBatch {
  int nb;
  long long x_stride;    // elements between rows of x_f32 / x_bf16
  long long out_stride;  // elements between rows of out_f32 / resid / out_bf16
  long long q_stride;    // elements between rows of q_out
  int pos[kMaxBatch];
  KvAddr kv[kMaxBatch];
};
int gemv_batch_launch(const GemvArgs& a, const GemvBatch& bt, cudaStream_t stream);
// token[b * token_stride] = token64[b] = argmax of row b's packed maxima
int argmax_finalize_batch_launch(const unsigned long long* packed, int nb, int32_t* token, int token_stride,
                                 int64_t* token64, cudaStream_t stream);
int token_copy_launch(const int32_t* src, int32_t* dst32, int64_t* dst64, cudaStream_t stream);

// Split-KV attention of one query row (the anchor / a decode step) over a
// cache layer; see anchor.cu.  Keys < n_lo are read from `lo`, the rest from
// `hi`; copy_lo also stores every lo row into hi (fused KV ingest).
struct AttnArgs {
  const bf16* q;  // [H*D], RoPE applied
  KvAddr lo, hi;
  int copy_lo;
  int lo_remote;             // lo is a peer GPU's memory: no bulk L2 prefetch of its rows
  int n_lo, n_keys, n_heads, n_kv_heads;
  int splits, split_keys;    // set by the launcher
  float* part_o;             // [H][splits][D]
  float* part_ml;            // [H][splits][2]
  unsigned int* counters;    // [KVH], zero between launches (the merging CTA resets)
  bf16* out;                 // [H*D]
  float scale_log2;
};
int attn_split_keys(int n_keys, int n_kv_heads, int R);
int attn_max_splits(int n_keys, int n_kv_heads, int R);  // workspace bound for any n <= n_keys
int decode_attention_launch(AttnArgs a, int head_dim, cudaStream_t stream);
// nb independent rows (each its own cache, keys and scratch) in one launch;
// each row gets the splits decode_attention_launch would give it alone, so the
// results are the single-row launches' bit for bit.
int decode_attention_batch_launch(const AttnArgs* rows, int nb, int head_dim, cudaStream_t stream);

// The whole anchor pass as one persistent kernel (one CTA per SM), see anchor.cu.
constexpr int kAnchorClaimSlots = 256;  // > any SM id
struct AnchorLayer {
  const bf16* wqkv;
  const bf16* wo;
  const bf16* w1;
  const bf16* w2;
  const float* g_attn;
  const float* g_mlp;
  KvAddr src;         // keys 0..pos-1 (a reused layer: the producer's export, read in place)
  KvAddr dst;         // the consumer cache layer (the anchor's own key goes here)
  unsigned int wait;  // > 0: GemmEpi::done arrivals to wait for before the attention
  int copy;           // store the src rows into dst while reading them (fused ingest)
  int src_remote;     // src lives on a peer GPU (plain loads only)
};
struct AnchorArgs {
  AnchorLayer layer[kMaxLayers];
  int n_layers, d_model, n_heads, n_kv_heads, head_dim, d_ff, mlp_kind, pos;
  const int64_t* token;  // device: the anchor row's token id
  const bf16* embed;
  const float* rope_cos;
  const float* rope_sin;
  float* h;              // [d] residual stream of the anchor row
  bf16* q;               // [H*D]
  bf16* o;               // [H*D]
  bf16* u;               // [d_ff]
  float* part_o;
  float* part_ml;
  unsigned int* head_count;  // [KVH] zero
  unsigned int* done;        // [n_layers] zero at launch; re-armed by the kernel
  unsigned int* bar;         // [2] grid barrier (count zero), then [gridDim] SM id of each CTA
  unsigned long long* stamps;  // [1 + 5 * n_layers] global ns after the seed and each phase (rank 0)
  unsigned int* claim;       // [kAnchorClaimSlots] CTAs seen per SM id, zero
  unsigned int* n_active;    // [1] working CTAs, zero
  int per_sm;                // working CTAs per SM (set by the launcher)
  int splits, split_keys;    // set by the launcher
  float scale_log2;
};
int anchor_persistent_smem(const ds_dims& d, int n_keys);
bool anchor_persistent_fits(const ds_dims& d, int n_keys);
// DS_ERR_INVALID when the shape does not fit the co-resident budget (callers fall back).
// co_resident: sized to share each SM with a GEMM / FA CTA of another stream
// (launch it once those hold the SMs); else it claims enough shared memory that
// no two of its CTAs share an SM.
int anchor_persistent_launch(AnchorArgs a, cudaStream_t stream, bool co_resident);

}  // namespace ds
