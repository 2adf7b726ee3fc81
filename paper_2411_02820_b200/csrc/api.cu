// C ABI (include/droidspeak.h) and the native orchestration of the
// cross-model prefill: validation in the reference's order, workspace
// carving, the per-layer kernel sequence, and the two-stream pipeline
// (ingest on the copy stream overlapping recompute on the compute stream,
// anchor gated on both — the pipelined plan of sched.py:212-263).
#include <stdarg.h>
#include <stdlib.h>
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.h"

using namespace ds;

namespace ds {
unsigned long long g_launches = 0;
thread_local cudaError_t g_cuda_err = cudaSuccess;
}

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_fail(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = ds::g_cuda_err;
  ds::g_cuda_err = cudaSuccess;
  return fail(DS_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define DS_TRY(expr, what)                      \
  do {                                          \
    int _rc = (expr);                           \
    if (_rc != DS_OK) {                         \
      if (_rc == DS_ERR_CUDA) return cuda_fail(what); \
      return fail(_rc, "%s: invalid launch arguments", what); \
    }                                           \
  } while (0)

// Stage timeline (ds_trace_begin / ds_trace_end): a pool of timing events
// recorded at stage boundaries while tracing is on.
struct Trace {
  bool on = false;
  int n = 0;
  std::vector<cudaEvent_t> ev;
  std::vector<int32_t> tag;
};
thread_local Trace g_trace;

void trace(cudaStream_t s, int tag) {
  Trace& t = g_trace;
  if (!t.on) return;
  if (t.n == (int)t.ev.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    t.ev.push_back(e);
    t.tag.push_back(0);
  }
  t.tag[t.n] = tag;
  cudaEventRecord(t.ev[t.n++], s);
}

constexpr int kMaxAnchorCtas = 1024;
// persistent anchor control block (zeroed per step): done[kMaxLayers] | bar[2] |
// smid[kMaxAnchorCtas] | claim[kAnchorClaimSlots] | n_active[1]
constexpr int kAnchorCtlWords = kMaxLayers + 2 + kMaxAnchorCtas + kAnchorClaimSlots + 1;

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

struct Workspace {
  int64_t* tokens;
  float* h;   // [n][d] residual stream
  bf16* a;    // [n][d] normalised GEMM operand
  bf16* q;    // [n][H*D]
  bf16* o;    // [n][H*D]
  bf16* u;    // [n][d_ff]
  float* h_a;  // [d] anchor residual
  bf16* a_a;   // [d] scratch
  bf16* q_a;   // [H*D]
  bf16* o_a;   // [H*D]
  bf16* u_a;   // [d_ff]
  float* part_o;
  float* part_ml;
  unsigned long long* argmax;
  int64_t* tok64;     // greedy token feeding the next decode step's embedding gather
  float* logits_dec;  // [V] decode-step logits
  float* dev;         // [n] token-selective baseline: per-position KV deviation
  int32_t* sel_pos;   // [n] selected positions (ascending)
  int64_t* sel_tok;   // [n] their token ids
  bf16* k0;           // [KVH][n][D] receiver's exact layer-0 K of the window
  bf16* v0;
  unsigned int* dec_count;  // [n_kv_heads] split-merge counters (zero between launches)
  unsigned int* gemv_ctr;   // [kGemvCtrWords] per-launch GEMV tile tickets (zero between launches; after dec_count)
  float* ssq;               // [ceil(d/128)][n] per-column-tile sums of squares (RMSNorm folded into the GEMMs)
  long long rows;           // positions the workspace was carved for
  unsigned int* an_ctl;     // persistent anchor control block: done[kMaxLayers], bar[2], smid[kMaxAnchorCtas]
  unsigned long long* an_stamps;  // persistent anchor phase times (ds_anchor_timeline)
  size_t bytes;
};

Workspace carve(const ds_dims& m, int n, void* base) {
  Workspace w{};
  uint8_t* p = static_cast<uint8_t*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) -> uint8_t* {
    uint8_t* r = p ? p + off : nullptr;
    off += align_up(bytes);
    return r;
  };
  const size_t hd = (size_t)m.n_heads * m.head_dim;
  const int splits = attn_max_splits(n, m.n_kv_heads, m.n_heads / (m.n_kv_heads > 0 ? m.n_kv_heads : 1));
  w.tokens = reinterpret_cast<int64_t*>(take(8ull * n));
  w.h = reinterpret_cast<float*>(take(4ull * n * m.d_model));
  w.a = reinterpret_cast<bf16*>(take(2ull * n * m.d_model));
  w.q = reinterpret_cast<bf16*>(take(2ull * n * hd));
  w.o = reinterpret_cast<bf16*>(take(2ull * n * hd));
  w.u = reinterpret_cast<bf16*>(take(2ull * n * m.d_ff));
  w.h_a = reinterpret_cast<float*>(take(4ull * m.d_model));
  w.a_a = reinterpret_cast<bf16*>(take(2ull * m.d_model));
  w.q_a = reinterpret_cast<bf16*>(take(2ull * hd));
  w.o_a = reinterpret_cast<bf16*>(take(2ull * hd));
  w.u_a = reinterpret_cast<bf16*>(take(2ull * m.d_ff));
  w.part_o = reinterpret_cast<float*>(take(4ull * splits * hd));
  w.part_ml = reinterpret_cast<float*>(take(8ull * splits * m.n_heads));
  w.argmax = reinterpret_cast<unsigned long long*>(take(8));
  w.tok64 = reinterpret_cast<int64_t*>(take(8));
  w.logits_dec = reinterpret_cast<float*>(take(4ull * m.vocab_size));
  w.dev = reinterpret_cast<float*>(take(4ull * n));
  w.sel_pos = reinterpret_cast<int32_t*>(take(4ull * n));
  w.sel_tok = reinterpret_cast<int64_t*>(take(8ull * n));
  w.k0 = reinterpret_cast<bf16*>(take(2ull * m.n_kv_heads * n * m.head_dim));
  w.v0 = reinterpret_cast<bf16*>(take(2ull * m.n_kv_heads * n * m.head_dim));
  w.dec_count = reinterpret_cast<unsigned int*>(take(4ull * (m.n_kv_heads + kGemvCtrWords)));
  w.gemv_ctr = w.dec_count ? w.dec_count + m.n_kv_heads : nullptr;
  w.ssq = reinterpret_cast<float*>(take(4ull * ((m.d_model + 127) / 128) * n));
  w.an_ctl = reinterpret_cast<unsigned int*>(take(4ull * kAnchorCtlWords));
  w.an_stamps = reinterpret_cast<unsigned long long*>(take(8ull * (1 + 5 * kMaxLayers)));
  w.bytes = off;
  w.rows = n;
  return w;
}

int check_dims(const ds_dims& d) {
  if (d.n_layers < 1 || d.n_layers > kMaxLayers) return fail(DS_ERR_INVALID, "n_layers %d outside [1,%d]", d.n_layers, kMaxLayers);
  if (d.head_dim != 64 && d.head_dim != 128) return fail(DS_ERR_INVALID, "head_dim %d unsupported (64|128)", d.head_dim);
  if (d.n_kv_heads < 1 || d.n_heads % d.n_kv_heads) return fail(DS_ERR_INVALID, "n_kv_heads must divide n_heads");
  if (d.n_heads / d.n_kv_heads > 8) return fail(DS_ERR_INVALID, "GQA ratio > 8 unsupported");
  if (d.d_model != d.n_heads * d.head_dim) return fail(DS_ERR_INVALID, "d_model != n_heads*head_dim");
  if (d.d_model % 64 || d.d_ff % 64) return fail(DS_ERR_INVALID, "d_model and d_ff must be multiples of 64");
  if (d.vocab_size < 2 || d.vocab_size % 2) return fail(DS_ERR_INVALID, "vocab_size must be even");
  if (d.max_seq < 2) return fail(DS_ERR_INVALID, "max_seq must be >= 2");
  if (d.mlp_kind != DS_MLP_UNGATED && d.mlp_kind != DS_MLP_SWIGLU) return fail(DS_ERR_INVALID, "unknown mlp_kind %d", d.mlp_kind);
  return DS_OK;
}

// check_tokens (model.py:425-437)
int check_tokens(const ds_dims& d, const int64_t* tokens, int n) {
  if (!tokens) return fail(DS_ERR_INVALID, "tokens_host is NULL");
  if (n < 2) return fail(DS_ERR_DEGENERATE, "need at least 2 tokens, got %d", n);
  if (n > d.max_seq) return fail(DS_ERR_INVALID, "sequence length %d exceeds max_seq %d", n, d.max_seq);
  for (int i = 0; i < n; ++i)
    if (tokens[i] < 0 || tokens[i] >= d.vocab_size) return fail(DS_ERR_INVALID, "token id out of vocabulary range");
  return DS_OK;
}

KvAddr layer_addr(const ds_kv_cache& c, int layer, int head_dim) {
  KvAddr a;
  a.k = kv_layer_base(c, layer, false);
  a.v = kv_layer_base(c, layer, true);
  a.head_stride = c.head_stride;
  a.page_stride = c.page_stride;
  a.table = c.block_table;
  a.head_dim = head_dim;
  return a;
}

// Rows of one cache layer viewed as a [rows][head_dim] matrix (the TMA bound).
long long layer_rows(const ds_kv_cache& c, int n_kv_heads, int head_dim) {
  if (c.layer_stride > 0) return c.layer_stride / head_dim;
  const long long pages = (c.positions + kPage - 1) / kPage;
  return ((n_kv_heads - 1) * c.head_stride + pages * c.page_stride) / head_dim;
}

struct Ctx {
  const ds_model* m;
  const ds_dims& d;
  Workspace w;
  const ds_kv_cache* kv;
  cudaStream_t s;
  cudaEvent_t* layer_ready = nullptr;  // recorded once layer l's window K/V are in the cache
  unsigned int* qkv_done = nullptr;    // per layer: QKV GEMM epilogue arrivals (persistent anchor waits)
  float* const* e_export = nullptr;    // [L] producer export: E (the window's f32 residual input) per layer
  cudaEvent_t after_seed = nullptr;    // recorded after the first group's seed kernel
};

// QKV (+RoPE, K/V into the cache) -> [attention -> o-proj+resid -> W1+SiLU -> W2+resid]
// over `rows` window rows at positions 0..rows-1 (model.py:536-544).  `kv_only`: the window output of
// this layer is dead (last layer of a group, model.py:625), so only the K/V columns are projected.
// RMSNorm is folded into the GEMMs: the residual epilogues (o-proj, W2) store bf16(h * g) and
// per-column-tile sums of squares, and the consuming GEMM (W1, next QKV) scales its rows by 1/rms.
// fuse_in: the QKV operand comes from the previous layer's W2 epilogue (else from an RMSNorm
// kernel, already normalised); g_next: the next layer's attention gain (W2 prepares its operand).
// DS_FUSE_NORM=0: the stand-alone RMSNorm kernels instead (A/B measurements).
bool fuse_norm() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DS_FUSE_NORM");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

int window_layer(Ctx& c, int l, int rows, bool kv_only, const int32_t* row_pos = nullptr, bool fuse_in = false,
                 const float* g_next = nullptr) {
  const ds_dims& d = c.d;
  const ds_layer_weights& W = c.m->layers[l];
  const int hd = d.n_heads * d.head_dim, kvd = d.n_kv_heads * d.head_dim;
  const int parts = (d.d_model + gemm_col_tile(rows, d.d_model) - 1) / gemm_col_tile(rows, d.d_model);
  auto norm_in = [&](GemmEpi& g) {
    g.ssq_in = c.w.ssq;
    g.ssq_parts = parts;
    g.norm_dim = d.d_model;
    g.ld_ssq = c.w.rows;
  };
  auto norm_out = [&](GemmEpi& g, const float* gain) {
    g.norm_out = c.w.a;
    g.norm_gain = gain;
    g.ssq_out = c.w.ssq;
    g.ld_ssq = c.w.rows;
  };
  GemmEpi e{};
  e.mode = EPI_QKV_ROPE;
  e.M = rows;
  e.N = kv_only ? 2 * kvd : hd + 2 * kvd;
  e.n_offset = kv_only ? hd : 0;
  e.n_heads = d.n_heads;
  e.n_kv_heads = d.n_kv_heads;
  e.head_dim = d.head_dim;
  e.q_out = c.w.q;
  e.ld_q = hd;
  e.kv = layer_addr(*c.kv, l, d.head_dim);
  e.pos0 = 0;
  e.pos_rows = row_pos;  // token-selective rows sit at scattered positions
  e.rope_cos = c.m->rope_cos;
  e.rope_sin = c.m->rope_sin;
  if (fuse_in) norm_in(e);
  if (c.qkv_done) e.done = c.qkv_done + l;
  const bf16* wqkv = static_cast<const bf16*>(W.wqkv) + (kv_only ? (long long)hd * d.d_model : 0);
  DS_TRY(gemm_launch(c.w.a, d.d_model, wqkv, d.d_model, d.d_model, e, c.s), "qkv gemm");
  trace(c.s, DS_TRACE_QKV + l);
  if (c.layer_ready && cudaEventRecord(c.layer_ready[l], c.s) != cudaSuccess) return cuda_fail("event record");
  if (kv_only) return DS_OK;
  const KvAddr ka = layer_addr(*c.kv, l, d.head_dim);
  DS_TRY(attention_prefill_launch(c.w.q, hd, ka.k, ka.v, ka.head_stride, ka.page_stride,
                                  layer_rows(*c.kv, d.n_kv_heads, d.head_dim), ka.table, rows, 0,
                                  d.n_heads, d.n_kv_heads, d.head_dim, c.w.o, hd, c.s, row_pos),
         "attention");
  GemmEpi r{};
  r.mode = EPI_RESID_F32;
  r.M = rows;
  r.N = d.d_model;
  r.out = c.w.h;
  r.ld_out = d.d_model;
  r.resid = c.w.h;
  r.ld_resid = d.d_model;
  if (fuse_norm()) norm_out(r, W.g_mlp);
  DS_TRY(gemm_launch(c.w.o, hd, W.wo, hd, hd, r, c.s), "o-proj gemm");
  if (!fuse_norm())
    DS_TRY(rmsnorm_launch(c.w.h, false, nullptr, rows, d.d_model, W.g_mlp, c.w.a, nullptr, nullptr, 0, c.s),
           "rmsnorm");
  GemmEpi f{};
  const bool swiglu = d.mlp_kind == DS_MLP_SWIGLU;
  f.mode = swiglu ? EPI_SWIGLU_BF16 : EPI_SILU_BF16;
  f.M = rows;
  f.N = swiglu ? 2 * d.d_ff : d.d_ff;
  f.out = c.w.u;
  f.ld_out = d.d_ff;
  if (fuse_norm()) norm_in(f);
  DS_TRY(gemm_launch(c.w.a, d.d_model, W.w1, d.d_model, d.d_model, f, c.s), "w1 gemm");
  GemmEpi r2{};
  r2.mode = EPI_RESID_F32;
  r2.M = rows;
  r2.N = d.d_model;
  r2.out = c.w.h;
  r2.ld_out = d.d_model;
  r2.resid = c.w.h;
  r2.ld_resid = d.d_model;
  if (g_next && fuse_norm()) norm_out(r2, g_next);
  DS_TRY(gemm_launch(c.w.u, d.d_ff, W.w2, d.d_ff, d.d_ff, r2, c.s), "w2 gemm");
  trace(c.s, DS_TRACE_LAYER + l);
  return DS_OK;
}

// The single anchor row at position `pos` through layer l (_layer_single, model.py:547-562).
// A producer export on another GPU (DS_FORCE_REMOTE=1 treats every sender as
// remote: single-GPU validation of that path).
bool sender_is_remote(const void* p) {
  static int force = -1;
  if (force < 0) {
    const char* e = getenv("DS_FORCE_REMOTE");
    force = (e && e[0] == '1') ? 1 : 0;
  }
  return force || !ptr_on_this_device(p);
}

// sender (optional): keys 0..pos-1 are read from the producer's export and
// copied into the consumer cache as they are read (the fused KV ingest).
// wait (optional): an event the attention waits for (the layer's window K/V on
// another stream); the QKV GEMV before it does not depend on it.
// DS_ABLATE_ANCHOR=<mask>: timing ablation of the per-launch anchor kernels
// (1 qkv, 2 attention, 4 o-proj, 8 w1, 16 w2 skipped).  The results are wrong
// under it; tools/anchor_alone.py under it prices each kernel inside the chain.
static int ablate_anchor() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DS_ABLATE_ANCHOR");
    v = e ? atoi(e) : 0;
  }
  return v;
}

int anchor_layer(Ctx& c, int l, int pos, float* h_a, const ds_kv_cache* sender = nullptr,
                 cudaEvent_t wait = nullptr) {
  const ds_dims& d = c.d;
  const int skip = ablate_anchor();
  const ds_layer_weights& W = c.m->layers[l];
  const int hd = d.n_heads * d.head_dim, kvd = d.n_kv_heads * d.head_dim;
  GemvArgs g{};
  g.W = static_cast<const bf16*>(W.wqkv);
  g.ldw = d.d_model;
  g.N = hd + 2 * kvd;
  g.K = d.d_model;
  g.x_f32 = h_a;
  g.gain = W.g_attn;
  g.mode = EPI_QKV_ROPE;
  g.n_heads = d.n_heads;
  g.n_kv_heads = d.n_kv_heads;
  g.head_dim = d.head_dim;
  g.pos = pos;
  g.q_out = c.w.q_a;
  g.kv = layer_addr(*c.kv, l, d.head_dim);
  g.rope_cos = c.m->rope_cos;
  g.rope_sin = c.m->rope_sin;
  g.tile_ctr = c.w.gemv_ctr + 0;  // one [ticket, done] pair per GEMV of the layer: consecutive launches never share
  if (!(skip & 1)) DS_TRY(gemv_launch(g, c.s), "anchor qkv");
  if (wait && cudaStreamWaitEvent(c.s, wait, 0) != cudaSuccess) return cuda_fail("wait");
  const KvAddr ka = g.kv;
  AttnArgs at{};
  at.q = c.w.q_a;
  at.lo = sender ? layer_addr(*sender, l, d.head_dim) : ka;
  at.hi = ka;
  at.copy_lo = sender ? 1 : 0;
  at.lo_remote = sender && sender_is_remote(at.lo.k) ? 1 : 0;
  at.n_lo = pos;
  at.n_keys = pos + 1;
  at.n_heads = d.n_heads;
  at.n_kv_heads = d.n_kv_heads;
  at.part_o = c.w.part_o;
  at.part_ml = c.w.part_ml;
  at.counters = c.w.dec_count;
  at.out = c.w.o_a;
  if (!(skip & 2)) DS_TRY(decode_attention_launch(at, d.head_dim, c.s), "anchor attention");
  GemvArgs o{};
  o.W = static_cast<const bf16*>(W.wo);
  o.ldw = hd;
  o.N = d.d_model;
  o.K = hd;
  o.x_bf16 = c.w.o_a;
  o.mode = EPI_RESID_F32;
  o.out_f32 = h_a;
  o.resid = h_a;
  o.tile_ctr = c.w.gemv_ctr + 2;
  if (!(skip & 4)) DS_TRY(gemv_launch(o, c.s), "anchor o-proj");
  GemvArgs f{};
  f.W = static_cast<const bf16*>(W.w1);
  f.ldw = d.d_model;
  f.N = d.mlp_kind == DS_MLP_SWIGLU ? 2 * d.d_ff : d.d_ff;
  f.K = d.d_model;
  f.x_f32 = h_a;
  f.gain = W.g_mlp;
  f.mode = d.mlp_kind == DS_MLP_SWIGLU ? EPI_SWIGLU_BF16 : EPI_SILU_BF16;
  f.out_bf16 = c.w.u_a;
  f.tile_ctr = c.w.gemv_ctr + 4;
  if (!(skip & 8)) DS_TRY(gemv_launch(f, c.s), "anchor w1");
  GemvArgs s2{};
  s2.W = static_cast<const bf16*>(W.w2);
  s2.ldw = d.d_ff;
  s2.N = d.d_model;
  s2.K = d.d_ff;
  s2.x_bf16 = c.w.u_a;
  s2.mode = EPI_RESID_F32;
  s2.out_f32 = h_a;
  s2.resid = h_a;
  s2.tile_ctr = c.w.gemv_ctr + 6;
  if (!(skip & 16)) DS_TRY(gemv_launch(s2, c.s), "anchor w2");
  return DS_OK;
}

// _final_logits + greedy first token (model.py:565-566, 779).
int lm_head(Ctx& c, const float* h_a, float* logits, int32_t* token, int64_t* token64 = nullptr) {
  const ds_dims& d = c.d;
  if (cudaMemsetAsync(c.w.argmax, 0, 8, c.s) != cudaSuccess) return cuda_fail("memset");
  GemvArgs g{};
  g.W = static_cast<const bf16*>(c.m->unembed);
  g.ldw = d.d_model;
  g.N = d.vocab_size;
  g.K = d.d_model;
  g.x_f32 = h_a;
  g.gain = c.m->g_final;
  g.mode = EPI_STORE_F32;
  g.out_f32 = logits;
  g.argmax = c.w.argmax;
  g.tile_ctr = c.w.gemv_ctr + 8;
  static const bool lm_tma = !(getenv("DS_LMHEAD_TMA") && getenv("DS_LMHEAD_TMA")[0] == '0');  // A/B switch
  DS_TRY(gemv_launch(g, c.s, /*staged=*/lm_tma), "lm head");
  if (token || token64) DS_TRY(argmax_finalize_launch(c.w.argmax, token, token64, c.s), "argmax");
  return DS_OK;
}

// One recompute group [a,b] over the window rows 0..P-1 (model.py:607-625):
// seed h from the token embeddings (a == 0) or the sender's E at layer a.
int recompute_group(Ctx& c, const int64_t* tok, int P, int a, int b, const void* seed) {
  const ds_dims& d = c.d;
  const ds_layer_weights& Wa = c.m->layers[a];
  // E at layer l = the window's f32 residual-stream input of layer l (model.py:620-621),
  // exported exactly (a = 0: the token embeddings, model.py:609)
  auto export_e = [&](int l) -> int {
    if (!c.e_export || !c.e_export[l]) return DS_OK;
    if (cudaMemcpyAsync(c.e_export[l], c.w.h, 4ull * P * d.d_model, cudaMemcpyDeviceToDevice, c.s) != cudaSuccess)
      return cuda_fail("e export");
    return DS_OK;
  };
  const bool fuse = fuse_norm();
  if (fuse)
    DS_TRY(norm_seed_launch(a == 0 ? c.m->embed : seed, a == 0, a == 0 ? tok : nullptr, P, d.d_model,
                            gemm_col_tile(P, d.d_model), Wa.g_attn, c.w.a, c.w.h, c.w.ssq, c.w.rows, c.s),
           "seed");
  else if (a == 0)
    DS_TRY(rmsnorm_launch(c.m->embed, true, tok, P, d.d_model, Wa.g_attn, c.w.a, c.w.h, nullptr, P, c.s), "seed");
  else
    DS_TRY(rmsnorm_launch(seed, false, nullptr, P, d.d_model, Wa.g_attn, c.w.a, c.w.h, nullptr, P, c.s), "seed");
  if (int rc = export_e(a)) return rc;
  if (c.after_seed) {
    if (cudaEventRecord(c.after_seed, c.s) != cudaSuccess) return cuda_fail("event record");
    c.after_seed = nullptr;
  }
  for (int l = a; l <= b; ++l) {
    if (l > a) {
      if (!fuse)
        DS_TRY(rmsnorm_launch(c.w.h, false, nullptr, P, d.d_model, c.m->layers[l].g_attn, c.w.a, nullptr, nullptr, 0,
                              c.s),
               "rmsnorm");
      if (int rc = export_e(l)) return rc;
    }
    int rc = window_layer(c, l, P, l == b, nullptr, /*fuse_in=*/fuse, l < b ? c.m->layers[l + 1].g_attn : nullptr);
    if (rc) return rc;
  }
  return DS_OK;
}

// The anchor position P through every layer, then logits + greedy token
// (model.py:627-637).
int reset_counters(Ctx& c) {
  if (cudaMemsetAsync(c.w.dec_count, 0, 4ull * (c.d.n_kv_heads + kGemvCtrWords), c.s) != cudaSuccess)
    return cuda_fail("memset");
  return DS_OK;
}

// How the anchor pass reads each layer.  Default (no plan): every layer from
// the consumer cache, no waits.
struct AnchorPlan {
  const ds_kv_cache* sender = nullptr;  // reused layers are read from here (and copied into the cache)
  const char* reused = nullptr;         // [L] 1 = reused layer
  unsigned int wait[kMaxLayers] = {};   // persistent path: QKV GEMM arrivals to wait for per layer
  const cudaEvent_t* wait_for = nullptr;  // per-launch path: per-layer events to wait for
  bool ctl_zeroed = false;              // the caller zeroed the control block in stream order
  bool co_resident = false;             // runs beside the recompute (small footprint); else one CTA per SM forced
  int persistent_layers = -1;           // co-resident: layers the persistent kernel runs (the rest per-launch)
  const cudaEvent_t* layer_event = nullptr;  // per-launch tail: per-layer QKV events of the compute stream
};

// The whole anchor pass as one persistent kernel (anchor.cu).
int anchor_persistent(Ctx& c, const int64_t* token_id, int P, const AnchorPlan* plan) {
  const ds_dims& d = c.d;
  static thread_local AnchorArgs A;  // ~20 KB of kernel parameters
  memset(&A, 0, sizeof(A));
  for (int l = 0; l < d.n_layers; ++l) {
    const ds_layer_weights& W = c.m->layers[l];
    AnchorLayer& al = A.layer[l];
    al.wqkv = static_cast<const bf16*>(W.wqkv);
    al.wo = static_cast<const bf16*>(W.wo);
    al.w1 = static_cast<const bf16*>(W.w1);
    al.w2 = static_cast<const bf16*>(W.w2);
    al.g_attn = W.g_attn;
    al.g_mlp = W.g_mlp;
    al.dst = layer_addr(*c.kv, l, d.head_dim);
    const bool from_sender = plan && plan->sender && plan->reused && plan->reused[l];
    al.src = from_sender ? layer_addr(*plan->sender, l, d.head_dim) : al.dst;
    al.copy = from_sender ? 1 : 0;
    al.src_remote = from_sender && sender_is_remote(al.src.k) ? 1 : 0;
    al.wait = plan ? plan->wait[l] : 0u;
  }
  A.n_layers = (plan && plan->persistent_layers >= 0) ? plan->persistent_layers : d.n_layers;
  A.d_model = d.d_model;
  A.n_heads = d.n_heads;
  A.n_kv_heads = d.n_kv_heads;
  A.head_dim = d.head_dim;
  A.d_ff = d.d_ff;
  A.mlp_kind = d.mlp_kind;
  A.pos = P;
  A.token = token_id;
  A.embed = static_cast<const bf16*>(c.m->embed);
  A.rope_cos = c.m->rope_cos;
  A.rope_sin = c.m->rope_sin;
  A.h = c.w.h_a;
  A.q = c.w.q_a;
  A.o = c.w.o_a;
  A.u = c.w.u_a;
  A.part_o = c.w.part_o;
  A.part_ml = c.w.part_ml;
  A.head_count = c.w.dec_count;
  A.done = c.w.an_ctl;
  A.bar = c.w.an_ctl + kMaxLayers;
  A.stamps = c.w.an_stamps;
  A.claim = c.w.an_ctl + kMaxLayers + 2 + kMaxAnchorCtas;
  A.n_active = A.claim + kAnchorClaimSlots;
  return anchor_persistent_launch(A, c.s, plan && plan->co_resident);
}

int zero_anchor_ctl(Ctx& c, cudaStream_t s) {
  if (cudaMemsetAsync(c.w.an_ctl, 0, 4ull * kAnchorCtlWords, s) != cudaSuccess ||
      cudaMemsetAsync(c.w.dec_count, 0, 4ull * (c.d.n_kv_heads + kGemvCtrWords), s) != cudaSuccess)
    return cuda_fail("memset");
  return DS_OK;
}

// token_id: device pointer to the row's token id; P: its position.  The
// persistent kernel runs the whole pass when the shape fits its co-resident
// budget; otherwise one launch per kernel (same device functions, same
// results), waiting on plan->wait_for events.
int anchor_pass(Ctx& c, const int64_t* token_id, int P, float* logits, int32_t* token,
                const AnchorPlan* plan = nullptr, int64_t* token64 = nullptr) {
  const ds_dims& d = c.d;
  // The persistent kernel runs the pass beside the recompute (one CTA per SM).
  // Alone, the per-launch kernels are faster (PDL-chained, TMA-staged GEMVs:
  // 4.05 ms vs 4.94 ms for the persistent kernel at four CTAs per SM, whose 592
  // grid barriers and uneven tile counts cost more than the kernel boundaries);
  // DS_ANCHOR_ALONE=persistent selects it for measurements.  Same device
  // functions everywhere, same results.
  static int alone_persistent = -1;
  if (alone_persistent < 0) {
    const char* e = getenv("DS_ANCHOR_ALONE");
    alone_persistent = (e && e[0] == 'p') ? 1 : 0;
  }
  const bool co = plan && plan->co_resident;
  const bool alone = !(plan && plan->wait_for) && !co && alone_persistent;
  if ((co || alone) && anchor_persistent_fits(d, P + 1)) {
    if (!(plan && plan->ctl_zeroed))
      if (int rc = zero_anchor_ctl(c, c.s)) return rc;
    DS_TRY(anchor_persistent(c, token_id, P, plan), "anchor");
    const int done_layers = (plan && plan->persistent_layers >= 0) ? plan->persistent_layers : d.n_layers;
    trace(c.s, DS_TRACE_ANCHOR + done_layers - 1);
    // the tail layers on the per-launch kernels (whole SMs once the recompute is done)
    for (int l = done_layers; l < d.n_layers; ++l) {
      const bool from_sender = plan && plan->sender && plan->reused && plan->reused[l];
      const cudaEvent_t ev = (plan && plan->layer_event && !from_sender) ? plan->layer_event[l] : nullptr;
      int rc = anchor_layer(c, l, P, c.w.h_a, from_sender ? plan->sender : nullptr, ev);
      if (rc) return rc;
      trace(c.s, DS_TRACE_ANCHOR + l);
    }
  } else {
    if (int rc = reset_counters(c)) return rc;
    DS_TRY(rmsnorm_launch(c.m->embed, true, token_id, 1, d.d_model, c.m->layers[0].g_attn, c.w.a_a, c.w.h_a, nullptr,
                          1, c.s),
           "anchor seed");
    for (int l = 0; l < d.n_layers; ++l) {
      if (plan && plan->wait_for && plan->wait_for[l] && cudaStreamWaitEvent(c.s, plan->wait_for[l], 0) != cudaSuccess)
        return cuda_fail("wait");
      const bool from_sender = plan && plan->sender && plan->reused && plan->reused[l];
      int rc = anchor_layer(c, l, P, c.w.h_a, from_sender ? plan->sender : nullptr);
      if (rc) return rc;
      trace(c.s, DS_TRACE_ANCHOR + l);
    }
  }
  int rc = lm_head(c, c.w.h_a, logits, token, token64);
  trace(c.s, DS_TRACE_LOGITS);
  return rc;
}

// ---------------------------------------------------------------- batched anchor rows
//
// Config 4's batch of requests on one consumer, and batched greedy decode:
// nb anchor rows (each its own cache, position and token) through every
// layer against ONE stream of the weights per layer (gemv_batch_launch), the
// attention of every row in one launch (decode_attention_batch_launch), and
// one lm-head pass.  Row b's arithmetic is the single-row per-launch pass's
// bit for bit (same kernels' per-row order), so a batch equals its requests
// run one by one.
struct BatchWs {
  int64_t* tokens;  // [nb][n_max] staged request ids
  int64_t* ids;     // [nb] anchor token ids (the seed gather)
  float* h;         // [nb][d] residual stream of each row
  bf16* a;          // [nb][d] seed scratch
  bf16* q;          // [nb][H*D]
  bf16* o;          // [nb][H*D]
  bf16* u;          // [nb][d_ff]
  float* part_o;    // [nb][splits][H*D]
  float* part_ml;   // [nb][splits][H][2]
  unsigned int* count;         // [nb][KVH] split-merge counters
  unsigned long long* argmax;  // [nb]
  int64_t* tok64;   // [nb] greedy tokens feeding the next decode step
  float* logits;    // [nb][V] decode-step logits
  long long splits;  // per-row split capacity
  size_t bytes;
};

BatchWs carve_batch(const ds_dims& m, int n_max, int nb, void* base) {
  BatchWs w{};
  uint8_t* p = static_cast<uint8_t*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) -> uint8_t* {
    uint8_t* r = p ? p + off : nullptr;
    off += align_up(bytes);
    return r;
  };
  const size_t hd = (size_t)m.n_heads * m.head_dim;
  w.splits = attn_max_splits(n_max, m.n_kv_heads, m.n_heads / (m.n_kv_heads > 0 ? m.n_kv_heads : 1));
  w.tokens = reinterpret_cast<int64_t*>(take(8ull * nb * n_max));
  w.ids = reinterpret_cast<int64_t*>(take(8ull * nb));
  w.h = reinterpret_cast<float*>(take(4ull * nb * m.d_model));
  w.a = reinterpret_cast<bf16*>(take(2ull * nb * m.d_model));
  w.q = reinterpret_cast<bf16*>(take(2ull * nb * hd));
  w.o = reinterpret_cast<bf16*>(take(2ull * nb * hd));
  w.u = reinterpret_cast<bf16*>(take(2ull * nb * m.d_ff));
  w.part_o = reinterpret_cast<float*>(take(4ull * nb * w.splits * hd));
  w.part_ml = reinterpret_cast<float*>(take(8ull * nb * w.splits * m.n_heads));
  w.count = reinterpret_cast<unsigned int*>(take(4ull * nb * m.n_kv_heads));
  w.argmax = reinterpret_cast<unsigned long long*>(take(8ull * nb));
  w.tok64 = reinterpret_cast<int64_t*>(take(8ull * nb));
  w.logits = reinterpret_cast<float*>(take(4ull * nb * m.vocab_size));
  w.bytes = off;
  return w;
}

// The batch section follows the single-request workspace of n_max rows.
size_t batch_ws_bytes(const ds_dims& d, int n_max, int nb) {
  return carve(d, n_max, nullptr).bytes + carve_batch(d, n_max, nb, nullptr).bytes;
}

int anchor_layer_batch(const ds_model* m, BatchWs& bw, const ds_kv_cache* kv, const int* pos, int nb, int l,
                       cudaStream_t s) {
  const ds_dims& d = m->dims;
  const ds_layer_weights& W = m->layers[l];
  const int hd = d.n_heads * d.head_dim, kvd = d.n_kv_heads * d.head_dim;
  GemvBatch bt{};
  bt.nb = nb;
  for (int b = 0; b < nb; ++b) {
    bt.pos[b] = pos[b];
    bt.kv[b] = layer_addr(kv[b], l, d.head_dim);
  }
  GemvArgs g{};
  g.W = static_cast<const bf16*>(W.wqkv);
  g.ldw = d.d_model;
  g.N = hd + 2 * kvd;
  g.K = d.d_model;
  g.x_f32 = bw.h;
  g.gain = W.g_attn;
  g.mode = EPI_QKV_ROPE;
  g.n_heads = d.n_heads;
  g.n_kv_heads = d.n_kv_heads;
  g.head_dim = d.head_dim;
  g.q_out = bw.q;
  g.rope_cos = m->rope_cos;
  g.rope_sin = m->rope_sin;
  bt.x_stride = d.d_model;
  bt.q_stride = hd;
  DS_TRY(gemv_batch_launch(g, bt, s), "batched anchor qkv");
  AttnArgs rows[kMaxBatch];
  for (int b = 0; b < nb; ++b) {
    AttnArgs& at = rows[b];
    at = AttnArgs{};
    at.q = bw.q + (long long)b * hd;
    at.lo = at.hi = bt.kv[b];
    at.n_lo = pos[b];
    at.n_keys = pos[b] + 1;
    at.n_heads = d.n_heads;
    at.n_kv_heads = d.n_kv_heads;
    at.part_o = bw.part_o + (long long)b * bw.splits * hd;
    at.part_ml = bw.part_ml + (long long)b * bw.splits * d.n_heads * 2;
    at.counters = bw.count + (long long)b * d.n_kv_heads;
    at.out = bw.o + (long long)b * hd;
  }
  DS_TRY(decode_attention_batch_launch(rows, nb, d.head_dim, s), "batched anchor attention");
  GemvArgs o{};
  o.W = static_cast<const bf16*>(W.wo);
  o.ldw = hd;
  o.N = d.d_model;
  o.K = hd;
  o.x_bf16 = bw.o;
  o.mode = EPI_RESID_F32;
  o.out_f32 = bw.h;
  o.resid = bw.h;
  bt.x_stride = hd;
  bt.out_stride = d.d_model;
  DS_TRY(gemv_batch_launch(o, bt, s), "batched anchor o-proj");
  GemvArgs f{};
  f.W = static_cast<const bf16*>(W.w1);
  f.ldw = d.d_model;
  f.N = d.mlp_kind == DS_MLP_SWIGLU ? 2 * d.d_ff : d.d_ff;
  f.K = d.d_model;
  f.x_f32 = bw.h;
  f.gain = W.g_mlp;
  f.mode = d.mlp_kind == DS_MLP_SWIGLU ? EPI_SWIGLU_BF16 : EPI_SILU_BF16;
  f.out_bf16 = bw.u;
  bt.x_stride = d.d_model;
  bt.out_stride = d.d_ff;
  DS_TRY(gemv_batch_launch(f, bt, s), "batched anchor w1");
  GemvArgs s2{};
  s2.W = static_cast<const bf16*>(W.w2);
  s2.ldw = d.d_ff;
  s2.N = d.d_model;
  s2.K = d.d_ff;
  s2.x_bf16 = bw.u;
  s2.mode = EPI_RESID_F32;
  s2.out_f32 = bw.h;
  s2.resid = bw.h;
  bt.x_stride = d.d_ff;
  bt.out_stride = d.d_model;
  DS_TRY(gemv_batch_launch(s2, bt, s), "batched anchor w2");
  return DS_OK;
}

// ids: device [nb] token of each row; pos: host [nb] position of each row.
// logits [nb][V]; token[b * token_stride] (optional) and tok64[b] (optional)
// receive the greedy tokens.
int anchor_pass_batch(const ds_model* m, BatchWs& bw, const ds_kv_cache* kv, const int* pos, int nb,
                      const int64_t* ids, float* logits, int32_t* token, int token_stride, int64_t* tok64,
                      cudaStream_t s) {
  const ds_dims& d = m->dims;
  if (cudaMemsetAsync(bw.count, 0, 4ull * nb * d.n_kv_heads, s) != cudaSuccess) return cuda_fail("memset");
  DS_TRY(rmsnorm_launch(m->embed, true, ids, nb, d.d_model, m->layers[0].g_attn, bw.a, bw.h, nullptr, nb, s),
         "batched anchor seed");
  for (int l = 0; l < d.n_layers; ++l) {
    if (int rc = anchor_layer_batch(m, bw, kv, pos, nb, l, s)) return rc;
    trace(s, DS_TRACE_ANCHOR + l);
  }
  if (cudaMemsetAsync(bw.argmax, 0, 8ull * nb, s) != cudaSuccess) return cuda_fail("memset");
  GemvArgs g{};
  g.W = static_cast<const bf16*>(m->unembed);
  g.ldw = d.d_model;
  g.N = d.vocab_size;
  g.K = d.d_model;
  g.x_f32 = bw.h;
  g.gain = m->g_final;
  g.mode = EPI_STORE_F32;
  g.out_f32 = logits;
  g.argmax = bw.argmax;
  GemvBatch bt{};
  bt.nb = nb;
  bt.x_stride = d.d_model;
  bt.out_stride = d.vocab_size;
  DS_TRY(gemv_batch_launch(g, bt, s), "batched lm head");
  if (token || tok64) DS_TRY(argmax_finalize_batch_launch(bw.argmax, nb, token, token_stride, tok64, s), "argmax");
  trace(s, DS_TRACE_LOGITS);
  return DS_OK;
}

const int64_t* stage_tokens(const int64_t* host, const int64_t* dev, int n, Workspace& w, cudaStream_t s) {
  if (dev) return dev;
  if (cudaMemcpyAsync(w.tokens, host, 8ull * n, cudaMemcpyHostToDevice, s) != cudaSuccess) return nullptr;
  return w.tokens;
}

int check_cache(const ds_kv_cache* c, const ds_dims& d, int n, const char* what) {
  if (!c || ((!c->k || !c->v) && !(c->layer_k && c->layer_v))) return fail(DS_ERR_INVALID, "%s cache is NULL", what);
  if (c->n_layers < d.n_layers || c->positions < n)
    return fail(DS_ERR_INVALID, "%s cache holds %d layers x %d positions, need %d x %d", what, c->n_layers,
                c->positions, d.n_layers, n);
  return DS_OK;
}

// Anchor-shape override (ds_set_anchor_shape; initial value from DS_ANCHOR_SHAPE).
std::atomic<int> g_anchor_shape{-1};
int anchor_shape() {
  int v = g_anchor_shape.load(std::memory_order_relaxed);
  if (v < 0) {
    const char* e = getenv("DS_ANCHOR_SHAPE");
    v = !e ? 0 : (e[0] == 'p' ? 1 : (e[0] == 'l' ? 2 : 0));
    int expect = -1;
    g_anchor_shape.compare_exchange_strong(expect, v);
    v = g_anchor_shape.load(std::memory_order_relaxed);
  }
  return v;
}

// One persistent (co-resident) anchor in flight per GPU.  The persistent
// kernel spins on its own recompute's GEMM counters, which is safe beside any
// other kernel of this library (each fits beside one anchor CTA per SM) but
// not beside a second persistent anchor: two of them could hold the slots
// each other's GEMMs need.  A fused call therefore takes the per-device slot;
// while another call's fused step (on other streams) has not finished on the
// GPU, a new call runs the per-launch anchor instead (event waits, no spins;
// same arithmetic, same bits).  Calls on the same stream pair are ordered
// behind the previous one and keep the fused shape.  Under stream capture the
// slot is neither checked nor armed: the replays' order is the caller's.
struct FusedSlot {
  std::mutex mu;
  cudaEvent_t done = nullptr;
  cudaStream_t cs = nullptr, xs = nullptr;
  bool armed = false;
};
constexpr int kMaxDevices = 64;
FusedSlot g_fused[kMaxDevices];
std::atomic<unsigned long long> g_fused_denied{0};

int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) dev = 0;
  return dev % kMaxDevices;
}

bool capturing(cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(s, &st) == cudaSuccess && st != cudaStreamCaptureStatusNone;
}

bool fused_slot_free(cudaStream_t cs, cudaStream_t xs) {
  if (capturing(cs)) return true;
  FusedSlot& f = g_fused[current_device()];
  std::lock_guard<std::mutex> lk(f.mu);
  if (!f.armed || (f.cs == cs && f.xs == xs)) return true;
  if (cudaEventQuery(f.done) == cudaErrorNotReady) {
    g_fused_denied.fetch_add(1, std::memory_order_relaxed);
    return false;
  }
  return true;
}

int fused_slot_arm(cudaStream_t cs, cudaStream_t xs) {
  if (capturing(cs)) return DS_OK;
  FusedSlot& f = g_fused[current_device()];
  std::lock_guard<std::mutex> lk(f.mu);
  if (!f.done && cudaEventCreateWithFlags(&f.done, cudaEventDisableTiming) != cudaSuccess) return cuda_fail("event");
  if (cudaEventRecord(f.done, cs) != cudaSuccess) return cuda_fail("event record");
  f.cs = cs;
  f.xs = xs;
  f.armed = true;
  return DS_OK;
}

// The prefill after validation, shared by ds_partial_prefill and
// ds_full_prefill (= every layer recomputed, no sender: the reference's
// full_prefill is _mixed_prefill over the same window + anchor structure,
// model.py:641-649, so recompute-all is the full prefill bit for bit).
// Persistent co-resident anchor when the recompute covers at least this many
// row-layers per model layer (k * P >= kFuseRowLayers * L); measured crossover.
constexpr long long kFuseRowLayers = 800;

int prefill_core(Ctx& c, const int64_t* tok, int n, const int32_t* groups, int n_groups,
                 const std::vector<const ds_e_cache*>& seed, const ds_kv_cache* sender_kv,
                 const std::vector<int32_t>& reused, const std::vector<char>& covered, float* logits_out,
                 int32_t* token_out, cudaStream_t xs) {
  const ds_model* m = c.m;
  const ds_dims& d = c.d;
  Workspace& w = c.w;
  const ds_kv_cache* out_kv = c.kv;
  const cudaStream_t cs = c.s;
  const int L = d.n_layers, P = n - 1;
  int rc;

  // The anchor reads the reused layers straight from the sender's export and
  // stores them into the consumer cache as it goes (the KV ingest fused into
  // the anchor's read of the same bytes), in both orders.  `fused`: the
  // persistent co-resident anchor runs beside the recompute (two streams).
  // It is the right shape when the recompute is long enough to hide it (its
  // 4 warps per SM stream the weights slower than the per-launch kernels,
  // which take whole SMs): measured crossover (config-5 sweep, 8B shapes) at
  // k * P ~ 800 * L recomputed row-layers.
  long long recomputed = 0;
  for (int l = 0; l < L; ++l) recomputed += covered[l];
  // DS_ANCHOR_SHAPE=persistent|launch / ds_set_anchor_shape override the rule (crossover measurements, tests)
  const int shape = anchor_shape();
  const bool fused = anchor_persistent_fits(d, n) &&
                     (shape == 1 || (shape == 0 && recomputed * P >= (long long)kFuseRowLayers * L)) &&
                     xs != cs && fused_slot_free(cs, xs);
  std::vector<char> reused_flag(L, 0);
  for (int l : reused) reused_flag[l] = 1;
  AnchorPlan plan;
  if (!reused.empty()) {
    plan.sender = sender_kv;
    plan.reused = reused_flag.data();
  }

  if (xs == cs) {
    // single stream: recompute, then the anchor (sched.py:256), per-launch kernels
    for (int i = 0; i < n_groups; ++i) {
      rc = recompute_group(c, tok, P, groups[2 * i], groups[2 * i + 1], seed[i] ? seed[i]->hidden : nullptr);
      if (rc) return rc;
    }
    return anchor_pass(c, tok + P, P, logits_out, token_out, &plan);
  }

  // Two streams.  Compute stream: the recompute groups.  Copy stream: the
  // anchor pass.  The anchor's layer l needs only layer l's window K/V
  // (model.py:559) and its own layer l-1 output, so for a recomputed layer it
  // waits for that layer's QKV GEMM and nothing else: the HBM-bound anchor
  // streams weights while the tensor-bound recompute runs.  Persistent path:
  // the wait is on the GEMM epilogue's arrival counter (one kernel, no events);
  // per-launch path (shapes beyond its budget): on an event after the QKV GEMM.
  // Same kernels, same results as the single-stream order.  Events are created
  // once per host thread (capturable into CUDA graphs).
  thread_local cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_seed = nullptr;
  thread_local cudaEvent_t ev_layer[kMaxLayers] = {};
  if (!ev_fork) {
    if (cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev_seed, cudaEventDisableTiming) != cudaSuccess)
      return cuda_fail("event");
    for (int l = 0; l < kMaxLayers; ++l)
      if (cudaEventCreateWithFlags(&ev_layer[l], cudaEventDisableTiming) != cudaSuccess) return cuda_fail("event");
  }
  cudaEvent_t wait_for[kMaxLayers] = {};
  if (fused) {
    // counters zeroed in stream order before either stream can touch them
    if (int rc2 = zero_anchor_ctl(c, cs)) return rc2;
    plan.ctl_zeroed = true;
    const int hd = d.n_heads * d.head_dim, kvd = d.n_kv_heads * d.head_dim;
    for (int i = 0; i < n_groups; ++i)
      for (int l = groups[2 * i]; l <= groups[2 * i + 1]; ++l)
        plan.wait[l] = gemm_done_target(P, l == groups[2 * i + 1] ? 2 * kvd : hd + 2 * kvd);
    c.qkv_done = w.an_ctl;
    // the last layer's anchor runs per-launch once the recompute is done
    if (covered[L - 1] && L > 1) {
      plan.persistent_layers = L - 1;
      plan.layer_event = ev_layer;
      c.layer_ready = ev_layer;
    }
    // The anchor launches once the first QKV GEMM's CTAs (PDL-launched while
    // the seed kernel drains) hold every SM: its CTAs then land one per SM,
    // beside them, instead of packing onto idle SMs.
    if (n_groups > 0) c.after_seed = ev_seed;
  } else {
    for (int l = 0; l < L; ++l) wait_for[l] = covered[l] ? ev_layer[l] : nullptr;
    plan.wait_for = wait_for;
    c.layer_ready = ev_layer;
  }
  cudaEventRecord(ev_fork, cs);
  cudaStreamWaitEvent(xs, ev_fork, 0);
  Ctx cx{m, d, w, out_kv, xs};
  // enqueue the recompute (which records ev_layer[l]) before the anchor's waits:
  // a cudaStreamWaitEvent binds to the latest record at enqueue time
  for (int i = 0; i < n_groups; ++i) {
    rc = recompute_group(c, tok, P, groups[2 * i], groups[2 * i + 1], seed[i] ? seed[i]->hidden : nullptr);
    if (rc) return rc;
  }
  if (fused && n_groups > 0) cudaStreamWaitEvent(xs, ev_seed, 0);
  plan.co_resident = fused && n_groups > 0;
  rc = anchor_pass(cx, tok + P, P, logits_out, token_out, &plan);
  if (rc) return rc;
  cudaEventRecord(ev_join, xs);
  cudaStreamWaitEvent(cs, ev_join, 0);
  if (fused) return fused_slot_arm(cs, xs);
  return DS_OK;
}

}  // namespace

extern "C" {

int ds_abi_version(void) { return DS_ABI_VERSION; }
unsigned long long ds_fused_fallbacks(void) { return g_fused_denied.load(std::memory_order_relaxed); }
int ds_set_anchor_shape(int32_t shape) {
  if (shape < 0 || shape > 2) return -1;
  const int prev = anchor_shape();
  g_anchor_shape.store(shape, std::memory_order_relaxed);
  return prev;
}
int ds_anchor_placement(const ds_dims* dims, int32_t n_tokens, const void* workspace, int32_t* sm_out, int32_t cap) {
  g_err.clear();
  if (!dims || !workspace || !sm_out || n_tokens < 1) return fail(DS_ERR_INVALID, "bad placement arguments"), -1;
  Workspace w = carve(*dims, n_tokens, const_cast<void*>(workspace));
  const int n = num_sms() < cap ? num_sms() : cap;
  if (cudaMemcpy(sm_out, w.an_ctl + kMaxLayers + 2, 4ull * n, cudaMemcpyDeviceToHost) != cudaSuccess)
    return cuda_fail("placement copy"), -1;
  return n;
}

int ds_anchor_timeline(const ds_dims* dims, int32_t n_tokens, const void* workspace, uint64_t* ns_out, int32_t cap) {
  g_err.clear();
  if (!dims || !workspace || !ns_out || n_tokens < 1) return fail(DS_ERR_INVALID, "bad timeline arguments"), -1;
  Workspace w = carve(*dims, n_tokens, const_cast<void*>(workspace));
  int n = 1 + 5 * dims->n_layers;
  if (n > cap) n = cap;
  if (cudaMemcpy(ns_out, w.an_stamps, 8ull * n, cudaMemcpyDeviceToHost) != cudaSuccess)
    return cuda_fail("timeline copy"), -1;
  return n;
}

int ds_trace_begin(void) {
  g_trace.on = true;
  g_trace.n = 0;
  return DS_OK;
}

int ds_trace_end(float* ms_out, int32_t* tag_out, int32_t cap) {
  Trace& t = g_trace;
  t.on = false;
  if (t.n == 0) return 0;
  for (int i = 0; i < t.n; ++i)
    if (cudaEventSynchronize(t.ev[i]) != cudaSuccess) return cuda_fail("trace sync"), -1;
  for (int i = 0; i < t.n && i < cap; ++i) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, t.ev[0], t.ev[i]) != cudaSuccess) return cuda_fail("trace elapsed"), -1;
    if (ms_out) ms_out[i] = ms;
    if (tag_out) tag_out[i] = t.tag[i];
  }
  return t.n;
}

unsigned long long ds_launch_count(void) { return __atomic_load_n(&ds::g_launches, __ATOMIC_RELAXED); }
const char* ds_last_error(void) { return g_err.c_str(); }

size_t ds_workspace_size(const ds_dims* dims, int32_t n_tokens) {
  if (!dims || n_tokens < 1) return 0;
  return carve(*dims, n_tokens, nullptr).bytes;
}

int ds_kv_ingest(const ds_kv_cache* src, const ds_kv_cache* dst, const int32_t* reused, int32_t n_reused,
                  int32_t window, int32_t n_kv_heads, int32_t head_dim, void* stream, int32_t* miss_layer) {
  g_err.clear();
  if (!dst || (!reused && n_reused) || n_reused < 0 || window < 1 || n_kv_heads < 1 ||
      (head_dim != 64 && head_dim != 128))
    return fail(DS_ERR_INVALID, "bad ingest arguments");
  if (n_reused > kMaxLayers) return fail(DS_ERR_INVALID, "too many layers");
  for (int i = 0; i < n_reused; ++i) {
    const int l = reused[i];
    if (i && reused[i - 1] >= l) return fail(DS_ERR_INVALID, "reused layers must ascend");
    if (!src || !kv_layer_present(*src, l) || src->positions < window) {
      if (miss_layer) *miss_layer = l;
      return fail(DS_ERR_CACHE_MISS, "missing kv cache for layer %d", l);
    }
    if (l < 0 || l >= dst->n_layers || dst->positions < window) return fail(DS_ERR_INVALID, "destination too small");
  }
  DS_TRY(kv_ingest_launch(*src, *dst, reused, n_reused, n_kv_heads, head_dim, window, (cudaStream_t)stream),
         "kv ingest");
  return DS_OK;
}

int ds_token_selective_prefill(const ds_model* m, const int64_t* tokens_host, const int64_t* tokens_dev,
                               int32_t n_tokens, const ds_kv_cache* sender_kv, double ratio, const ds_kv_cache* out_kv,
                               float* logits_out, int32_t* token_out, int32_t* n_selected, void* workspace,
                               size_t workspace_bytes, void* stream, int32_t* miss_layer) {
  g_err.clear();
  if (!m || !m->layers) return fail(DS_ERR_INVALID, "model is NULL");
  const ds_dims& d = m->dims;
  int rc;
  if ((rc = check_dims(d))) return rc;
  if (!(ratio > 0.0 && ratio <= 1.0)) return fail(DS_ERR_INVALID, "ratio must lie in (0, 1], got %g", ratio);
  if ((rc = check_tokens(d, tokens_host, n_tokens))) return rc;
  const int L = d.n_layers, n = n_tokens, P = n - 1;
  // sender checks in the reference's order (model.py:699-702)
  int have = 0;
  while (sender_kv && have < L && kv_layer_present(*sender_kv, have)) ++have;
  if (have < L) {
    if (miss_layer) *miss_layer = have;
    return fail(DS_ERR_CACHE_MISS, "sender cache missing layers");
  }
  if (sender_kv->positions < P) {
    if (miss_layer) *miss_layer = 0;
    return fail(DS_ERR_CACHE_MISS, "sender cache has %d positions, need %d", sender_kv->positions, P);
  }
  if ((rc = check_cache(out_kv, d, n, "output"))) return rc;
  if (!logits_out) return fail(DS_ERR_INVALID, "logits_out is NULL");
  Workspace w = carve(d, n, workspace);
  if (!workspace || workspace_bytes < w.bytes)
    return fail(DS_ERR_INVALID, "workspace of %zu bytes < required %zu", workspace_bytes, w.bytes);
  const int n_sel = (int)ceil(ratio * P);  // math.ceil(ratio * window) in double (model.py:715)
  if (n_selected) *n_selected = n_sel;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t* tok = stage_tokens(tokens_host, tokens_dev, n, w, s);
  if (!tok) return cuda_fail("token upload");
  Ctx c{m, d, w, out_kv, s};
  // 1. every layer starts from the sender's K/V over the window
  std::vector<int32_t> all(L);
  for (int l = 0; l < L; ++l) all[l] = l;
  DS_TRY(kv_ingest_launch(*sender_kv, *out_kv, all.data(), L, d.n_kv_heads, d.head_dim, P, s), "kv ingest");
  // 2. the receiver's exact layer-0 K/V of the window into scratch, deviation per position
  DS_TRY(rmsnorm_launch(m->embed, true, tok, P, d.d_model, m->layers[0].g_attn, w.a, nullptr, nullptr, 0, s),
         "embed");
  {
    const int hd = d.n_heads * d.head_dim, kvd = d.n_kv_heads * d.head_dim;
    GemmEpi e{};
    e.mode = EPI_QKV_ROPE;
    e.M = P;
    e.N = 2 * kvd;
    e.n_offset = hd;
    e.n_heads = d.n_heads;
    e.n_kv_heads = d.n_kv_heads;
    e.head_dim = d.head_dim;
    e.kv.k = w.k0;
    e.kv.v = w.v0;
    e.kv.head_stride = (long long)n * d.head_dim;
    e.kv.page_stride = (long long)kPage * d.head_dim;
    e.kv.table = nullptr;
    e.kv.head_dim = d.head_dim;
    e.rope_cos = m->rope_cos;
    e.rope_sin = m->rope_sin;
    DS_TRY(gemm_launch(w.a, d.d_model, static_cast<const bf16*>(m->layers[0].wqkv) + (long long)hd * d.d_model,
                       d.d_model, d.d_model, e, s),
           "layer-0 kv");
  }
  DS_TRY(kv_deviation_launch(w.k0, w.v0, (long long)n * d.head_dim, *sender_kv, P, d.n_kv_heads, d.head_dim, w.dev, s),
         "deviation");
  DS_TRY(select_topk_launch(w.dev, P, n_sel, tok, w.sel_pos, w.sel_tok, s), "select");
  // 3. the selected positions through every layer (model.py:726-734): their K/V
  //    replace the sender's in the cache, attention is causal by absolute position
  //    (the same per-layer sequence as a recompute group, so ratio 1 is recompute-all bit for bit)
  const bool fuse = fuse_norm();
  if (fuse)
    DS_TRY(norm_seed_launch(m->embed, true, w.sel_tok, n_sel, d.d_model, gemm_col_tile(n_sel, d.d_model),
                            m->layers[0].g_attn, w.a, w.h, w.ssq, w.rows, s),
           "seed");
  else
    DS_TRY(rmsnorm_launch(m->embed, true, w.sel_tok, n_sel, d.d_model, m->layers[0].g_attn, w.a, w.h, nullptr, n_sel,
                          s),
           "seed");
  for (int l = 0; l < L; ++l) {
    if (l > 0 && !fuse)
      DS_TRY(rmsnorm_launch(w.h, false, nullptr, n_sel, d.d_model, m->layers[l].g_attn, w.a, nullptr, nullptr, 0, s),
             "rmsnorm");
    rc = window_layer(c, l, n_sel, l == L - 1, w.sel_pos, fuse, l < L - 1 ? m->layers[l + 1].g_attn : nullptr);
    if (rc) return rc;
  }
  // 4. the anchor through every layer
  return anchor_pass(c, tok + P, P, logits_out, token_out);
}

int ds_decode_greedy(const ds_model* m, const ds_kv_cache* kv, int32_t positions, const int32_t* first_token,
                     int32_t steps, int32_t* tokens_out, void* workspace, size_t workspace_bytes, void* stream) {
  g_err.clear();
  if (!m || !m->layers) return fail(DS_ERR_INVALID, "model is NULL");
  const ds_dims& d = m->dims;
  int rc;
  if ((rc = check_dims(d))) return rc;
  if (steps < 1) return fail(DS_ERR_INVALID, "steps must be at least 1");
  if (positions < 1) return fail(DS_ERR_INVALID, "cache must hold at least one position");
  if ((long long)positions + steps > d.max_seq)
    return fail(DS_ERR_INVALID, "decoding %d steps from %d positions exceeds max_seq %d", steps, positions, d.max_seq);
  if (!first_token || !tokens_out) return fail(DS_ERR_INVALID, "first_token and tokens_out are required");
  if ((rc = check_cache(kv, d, positions + steps - 1, "cache"))) return rc;
  Workspace w = carve(d, positions + steps, workspace);
  if (!workspace || workspace_bytes < w.bytes)
    return fail(DS_ERR_INVALID, "workspace of %zu bytes < required %zu", workspace_bytes, w.bytes);
  Ctx c{m, d, w, kv, (cudaStream_t)stream};
  // step 0's token is argmax of the prefill logits; each further step runs that
  // token through every layer at the next position (model.py:771-787)
  DS_TRY(token_copy_launch(first_token, tokens_out, w.tok64, c.s), "token copy");
  for (int s = 1; s < steps; ++s) {
    rc = anchor_pass(c, w.tok64, positions + s - 1, w.logits_dec, tokens_out + s, nullptr, w.tok64);
    if (rc) return rc;
  }
  return DS_OK;
}

int ds_ipc_export(const void* device_ptr, void* handle_out, uint64_t* offset_out) {
  g_err.clear();
  if (!device_ptr || !handle_out || !offset_out) return fail(DS_ERR_INVALID, "bad ipc export arguments");
  // driver entry point resolved at run time: the library must load without libcuda (CPU build box)
  typedef CUresult (*RangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
  static RangeFn range = nullptr;
  if (!range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return fail(DS_ERR_CUDA, "cuMemGetAddressRange unavailable");
    range = reinterpret_cast<RangeFn>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, (CUdeviceptr)device_ptr) != CUDA_SUCCESS)
    return fail(DS_ERR_CUDA, "cuMemGetAddressRange failed for %p", device_ptr);
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)) != cudaSuccess) return cuda_fail("cudaIpcGetMemHandle");
  static_assert(sizeof(h) == DS_IPC_HANDLE_BYTES, "ipc handle size");
  memcpy(handle_out, &h, sizeof(h));
  *offset_out = (uint64_t)((CUdeviceptr)device_ptr - base);
  return DS_OK;
}

int ds_ipc_open(const void* handle, uint64_t offset, void** base_out, void** ptr_out) {
  g_err.clear();
  if (!handle || !base_out || !ptr_out) return fail(DS_ERR_INVALID, "bad ipc open arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* base = nullptr;
  if (cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
    return cuda_fail("cudaIpcOpenMemHandle");
  *base_out = base;
  *ptr_out = static_cast<uint8_t*>(base) + offset;
  return DS_OK;
}

int ds_ipc_close(void* base) {
  g_err.clear();
  if (!base) return DS_OK;
  if (cudaIpcCloseMemHandle(base) != cudaSuccess) return cuda_fail("cudaIpcCloseMemHandle");
  return DS_OK;
}

int ds_gemm(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc, const float* resid,
            int64_t ld_resid, int32_t M, int32_t N, int32_t K, int32_t mode, void* stream) {
  g_err.clear();
  if (!A || !B || !C || M < 1 || N < 16 || K < 8 || (N % 16) || (K % 8))
    return fail(DS_ERR_INVALID, "bad gemm shape M=%d N=%d K=%d", M, N, K);
  if (mode != EPI_STORE_BF16 && mode != EPI_RESID_F32 && mode != EPI_SILU_BF16 && mode != EPI_STORE_F32 &&
      !(mode == EPI_SWIGLU_BF16 && N % 32 == 0))
    return fail(DS_ERR_INVALID, "bad epilogue mode %d", mode);
  if (mode == EPI_RESID_F32 && !resid) return fail(DS_ERR_INVALID, "resid required");
  GemmEpi e{};
  e.mode = mode;
  e.M = M;
  e.N = N;
  e.out = C;
  e.ld_out = ldc;
  e.resid = resid;
  e.ld_resid = ld_resid;
  DS_TRY(gemm_launch(A, lda, B, ldb, K, e, (cudaStream_t)stream), "gemm");
  return DS_OK;
}

int ds_rmsnorm(const void* x, int32_t x_is_bf16, const int64_t* gather, int32_t M, int32_t d, const float* gain,
               void* out_bf16, float* copy_f32, void* copy_bf16, void* stream) {
  g_err.clear();
  if (!x || !gain || !out_bf16 || M < 1 || d < 8 || (d % 8)) return fail(DS_ERR_INVALID, "bad rmsnorm arguments");
  DS_TRY(rmsnorm_launch(x, x_is_bf16 != 0, gather, M, d, gain, static_cast<bf16*>(out_bf16), copy_f32,
                        static_cast<bf16*>(copy_bf16), M, (cudaStream_t)stream),
         "rmsnorm");
  return DS_OK;
}

int ds_attention_prefill(const void* q, int64_t ldq, const ds_kv_cache* kv, int32_t layer, int32_t n_q,
                         int32_t q_pos0, int32_t n_heads, int32_t n_kv_heads, int32_t head_dim, void* o,
                         int64_t ldo, void* stream) {
  g_err.clear();
  if (!q || !kv || !o || n_q < 1 || q_pos0 < 0 || n_kv_heads < 1 || n_heads % n_kv_heads ||
      (head_dim != 64 && head_dim != 128) || layer < 0 || layer >= kv->n_layers || q_pos0 + n_q > kv->positions)
    return fail(DS_ERR_INVALID, "bad attention arguments");
  const KvAddr a = layer_addr(*kv, layer, head_dim);
  DS_TRY(attention_prefill_launch(static_cast<const bf16*>(q), ldq, a.k, a.v, a.head_stride, a.page_stride,
                                  layer_rows(*kv, n_kv_heads, head_dim), a.table,
                                  n_q, q_pos0, n_heads, n_kv_heads, head_dim, static_cast<bf16*>(o), ldo,
                                  (cudaStream_t)stream),
         "attention");
  return DS_OK;
}

int ds_partial_prefill(const ds_model* m, const int64_t* tokens_host, const int64_t* tokens_dev, int32_t n_tokens,
                       const int32_t* groups, int32_t n_groups, const ds_kv_cache* sender_kv,
                       const ds_e_cache* sender_e, int32_t n_e, const ds_kv_cache* out_kv, float* logits_out,
                       int32_t* token_out, void* workspace, size_t workspace_bytes, void* compute_stream,
                       void* copy_stream, int32_t* miss_layer, int32_t* miss_kind) {
  g_err.clear();
  if (miss_kind) *miss_kind = DS_MISS_NONE;
  if (!m || !m->layers) return fail(DS_ERR_INVALID, "model is NULL");
  const ds_dims& d = m->dims;
  int rc;
  if ((rc = check_dims(d))) return rc;
  if ((rc = check_tokens(d, tokens_host, n_tokens))) return rc;
  const int L = d.n_layers, n = n_tokens, P = n - 1;
  // RecomputeConfig normal form + validate_for (model.py:166-178, 204-208)
  if (n_groups < 0 || (n_groups && !groups)) return fail(DS_ERR_INVALID, "bad groups");
  std::vector<char> covered(L, 0);
  for (int i = 0; i < n_groups; ++i) {
    const int a = groups[2 * i], b = groups[2 * i + 1];
    if (a < 0 || a > b) return fail(DS_ERR_INVALID, "range [%d,%d] invalid", a, b);
    if (i && a <= groups[2 * i - 1] + 1) return fail(DS_ERR_INVALID, "groups not in normal form");
    if (b > L - 1) return fail(DS_ERR_INVALID, "config exceeds layer range [0,%d]", L - 1);
    for (int l = a; l <= b; ++l) covered[l] = 1;
  }
  if ((rc = check_cache(out_kv, d, n, "output"))) return rc;
  if (!logits_out) return fail(DS_ERR_INVALID, "logits_out is NULL");
  // KV misses in ascending layer order (model.py:590-601)
  std::vector<int32_t> reused;
  for (int l = 0; l < L; ++l) {
    if (covered[l]) continue;
    if (!sender_kv || !kv_layer_present(*sender_kv, l) || sender_kv->positions < P) {
      if (miss_layer) *miss_layer = l;
      if (miss_kind) *miss_kind = DS_MISS_KV;
      return fail(DS_ERR_CACHE_MISS, "missing kv cache for layer %d", l);
    }
    reused.push_back(l);
  }
  // E misses per group (model.py:611-617)
  std::vector<const ds_e_cache*> seed(n_groups, nullptr);
  for (int i = 0; i < n_groups; ++i) {
    const int a = groups[2 * i];
    if (a == 0) continue;
    for (int j = 0; j < n_e; ++j)
      if (sender_e && sender_e[j].layer == a) seed[i] = &sender_e[j];
    const ds_e_cache* e = seed[i];
    if (!e || !e->hidden || e->positions < P || e->width != d.d_model) {
      if (miss_layer) *miss_layer = a;
      if (miss_kind) *miss_kind = DS_MISS_E;
      return fail(DS_ERR_CACHE_MISS, "missing e cache for layer %d", a);
    }
  }
  Workspace w = carve(d, n, workspace);
  if (!workspace || workspace_bytes < w.bytes)
    return fail(DS_ERR_INVALID, "workspace of %zu bytes < required %zu", workspace_bytes, w.bytes);

  cudaStream_t cs = (cudaStream_t)compute_stream;
  cudaStream_t xs = copy_stream ? (cudaStream_t)copy_stream : cs;
  const int64_t* tok = stage_tokens(tokens_host, tokens_dev, n, w, cs);
  if (!tok) return cuda_fail("token upload");
  Ctx c{m, d, w, out_kv, cs};
  trace(cs, 0);
  return prefill_core(c, tok, n, groups, n_groups, seed, sender_kv, reused, covered, logits_out, token_out, xs);
}

int ds_recompute_group(const ds_model* m, const int64_t* tokens_dev, int32_t n_tokens, int32_t a, int32_t b,
                       const void* seed, int32_t seed_positions, const ds_kv_cache* out_kv, void* workspace,
                       size_t workspace_bytes, void* stream) {
  g_err.clear();
  if (!m || !m->layers) return fail(DS_ERR_INVALID, "model is NULL");
  const ds_dims& d = m->dims;
  int rc;
  if ((rc = check_dims(d))) return rc;
  if (n_tokens < 2) return fail(DS_ERR_DEGENERATE, "need at least 2 tokens, got %d", n_tokens);
  if (n_tokens > d.max_seq) return fail(DS_ERR_INVALID, "sequence length %d exceeds max_seq %d", n_tokens, d.max_seq);
  if (a < 0 || a > b || b >= d.n_layers) return fail(DS_ERR_INVALID, "range [%d,%d] invalid for %d layers", a, b, d.n_layers);
  const int P = n_tokens - 1;
  if (a == 0 && !tokens_dev) return fail(DS_ERR_INVALID, "tokens_dev required for a group starting at layer 0");
  if (a > 0 && (!seed || seed_positions < P)) return fail(DS_ERR_CACHE_MISS, "missing e cache for layer %d", a);
  if ((rc = check_cache(out_kv, d, n_tokens, "output"))) return rc;
  Workspace w = carve(d, n_tokens, workspace);
  if (!workspace || workspace_bytes < w.bytes)
    return fail(DS_ERR_INVALID, "workspace of %zu bytes < required %zu", workspace_bytes, w.bytes);
  Ctx c{m, d, w, out_kv, (cudaStream_t)stream};
  return recompute_group(c, tokens_dev, P, a, b, a > 0 ? seed : nullptr);
}

int ds_anchor(const ds_model* m, const int64_t* tokens_dev, int32_t n_tokens, const ds_kv_cache* kv,
              float* logits_out, int32_t* token_out, void* workspace, size_t workspace_bytes, void* stream) {
  g_err.clear();
  if (!m || !m->layers) return fail(DS_ERR_INVALID, "model is NULL");
  const ds_dims& d = m->dims;
  int rc;
  if ((rc = check_dims(d))) return rc;
  if (n_tokens < 2) return fail(DS_ERR_DEGENERATE, "need at least 2 tokens, got %d", n_tokens);
  if (n_tokens > d.max_seq) return fail(DS_ERR_INVALID, "sequence length %d exceeds max_seq %d", n_tokens, d.max_seq);
  if (!tokens_dev || !logits_out) return fail(DS_ERR_INVALID, "tokens_dev and logits_out are required");
  if ((rc = check_cache(kv, d, n_tokens, "cache"))) return rc;
  Workspace w = carve(d, n_tokens, workspace);
  if (!workspace || workspace_bytes < w.bytes)
    return fail(DS_ERR_INVALID, "workspace of %zu bytes < required %zu", workspace_bytes, w.bytes);
  Ctx c{m, d, w, kv, (cudaStream_t)stream};
  return anchor_pass(c, tokens_dev + (n_tokens - 1), n_tokens - 1, logits_out, token_out);
}

int ds_full_prefill(const ds_model* m, const int64_t* tokens_host, const int64_t* tokens_dev, int32_t n_tokens,
                    const ds_kv_cache* out_kv, const int32_t* e_layers, int32_t n_e, void* const* e_out,
                    float* logits_out, int32_t* token_out, void* workspace, size_t workspace_bytes, void* stream,
                    void* copy_stream) {
  g_err.clear();
  if (!m || !m->layers) return fail(DS_ERR_INVALID, "model is NULL");
  const ds_dims& d = m->dims;
  int rc;
  if ((rc = check_dims(d))) return rc;
  if ((rc = check_tokens(d, tokens_host, n_tokens))) return rc;
  if ((rc = check_cache(out_kv, d, n_tokens, "output"))) return rc;
  if (!logits_out) return fail(DS_ERR_INVALID, "logits_out is NULL");
  const int L = d.n_layers, n = n_tokens;
  std::vector<float*> e_at(L, nullptr);
  for (int i = 0; i < n_e; ++i) {
    const int l = e_layers[i];
    if (l < 0 || l >= L || !e_out || !e_out[i]) return fail(DS_ERR_INVALID, "bad e export layer %d", l);
    e_at[l] = static_cast<float*>(e_out[i]);
  }
  Workspace w = carve(d, n, workspace);
  if (!workspace || workspace_bytes < w.bytes)
    return fail(DS_ERR_INVALID, "workspace of %zu bytes < required %zu", workspace_bytes, w.bytes);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t* tok = stage_tokens(tokens_host, tokens_dev, n, w, s);
  if (!tok) return cuda_fail("token upload");
  Ctx c{m, d, w, out_kv, s};
  c.e_export = e_at.data();
  trace(s, 0);
  const int32_t all[2] = {0, L - 1};
  std::vector<const ds_e_cache*> seed(1, nullptr);
  std::vector<int32_t> reused;
  std::vector<char> covered(L, 1);
  return prefill_core(c, tok, n, all, 1, seed, nullptr, reused, covered, logits_out, token_out,
                      copy_stream ? (cudaStream_t)copy_stream : s);
}

size_t ds_workspace_size_batch(const ds_dims* dims, int32_t max_tokens, int32_t batch) {
  if (!dims || max_tokens < 1 || batch < 1 || batch > kMaxBatch) return 0;
  return batch_ws_bytes(*dims, max_tokens, batch);
}

int ds_partial_prefill_batch(const ds_model* m, int32_t batch, const int64_t* const* tokens_host,
                             const int64_t* const* tokens_dev, const int32_t* n_tokens, const int32_t* groups,
                             int32_t n_groups, const ds_kv_cache* sender_kv, const ds_e_cache* const* sender_e,
                             const int32_t* n_e, const ds_kv_cache* out_kv, float* logits_out, int32_t* token_out,
                             void* workspace, size_t workspace_bytes, void* compute_stream, void* copy_stream,
                             int32_t* bad_request, int32_t* miss_layer, int32_t* miss_kind) {
  g_err.clear();
  if (miss_kind) *miss_kind = DS_MISS_NONE;
  if (bad_request) *bad_request = -1;
  if (!m || !m->layers) return fail(DS_ERR_INVALID, "model is NULL");
  const ds_dims& d = m->dims;
  int rc;
  if ((rc = check_dims(d))) return rc;
  if (batch < 1 || batch > kMaxBatch) return fail(DS_ERR_INVALID, "batch %d outside [1,%d]", batch, kMaxBatch);
  if (!tokens_host || !n_tokens || !out_kv || !logits_out) return fail(DS_ERR_INVALID, "batch arrays are NULL");
  const int L = d.n_layers, nb = batch;
  // each request in the reference's order (check_tokens, validate_for, KV
  // misses ascending, E per group); requests in order
  std::vector<char> covered(L, 0);
  std::vector<int32_t> reused;
  std::vector<std::vector<const ds_e_cache*>> seed(nb, std::vector<const ds_e_cache*>(n_groups > 0 ? n_groups : 0));
  int n_max = 0;
  for (int b = 0; b < nb; ++b) {
    auto bad = [&](int code) {
      if (bad_request) *bad_request = b;
      return code;
    };
    if ((rc = check_tokens(d, tokens_host[b], n_tokens[b]))) return bad(rc);
    const int n = n_tokens[b], P = n - 1;
    n_max = n > n_max ? n : n_max;
    if (b == 0) {
      if (n_groups < 0 || (n_groups && !groups)) return bad(fail(DS_ERR_INVALID, "bad groups"));
      for (int i = 0; i < n_groups; ++i) {
        const int a = groups[2 * i], e = groups[2 * i + 1];
        if (a < 0 || a > e) return bad(fail(DS_ERR_INVALID, "range [%d,%d] invalid", a, e));
        if (i && a <= groups[2 * i - 1] + 1) return bad(fail(DS_ERR_INVALID, "groups not in normal form"));
        if (e > L - 1) return bad(fail(DS_ERR_INVALID, "config exceeds layer range [0,%d]", L - 1));
        for (int l = a; l <= e; ++l) covered[l] = 1;
      }
      for (int l = 0; l < L; ++l)
        if (!covered[l]) reused.push_back(l);
    }
    if ((rc = check_cache(&out_kv[b], d, n, "output"))) return bad(rc);
    for (int l : reused) {
      const ds_kv_cache* skv = sender_kv ? &sender_kv[b] : nullptr;
      if (!skv || !kv_layer_present(*skv, l) || skv->positions < P) {
        if (miss_layer) *miss_layer = l;
        if (miss_kind) *miss_kind = DS_MISS_KV;
        return bad(fail(DS_ERR_CACHE_MISS, "request %d: missing kv cache for layer %d", b, l));
      }
    }
    for (int i = 0; i < n_groups; ++i) {
      const int a = groups[2 * i];
      if (a == 0) continue;
      const int ne = n_e ? n_e[b] : 0;
      for (int j = 0; j < ne; ++j)
        if (sender_e && sender_e[b] && sender_e[b][j].layer == a) seed[b][i] = &sender_e[b][j];
      const ds_e_cache* e = seed[b][i];
      if (!e || !e->hidden || e->positions < P || e->width != d.d_model) {
        if (miss_layer) *miss_layer = a;
        if (miss_kind) *miss_kind = DS_MISS_E;
        return bad(fail(DS_ERR_CACHE_MISS, "request %d: missing e cache for layer %d", b, a));
      }
    }
  }
  Workspace w = carve(d, n_max, workspace);
  BatchWs bw = carve_batch(d, n_max, nb, workspace ? static_cast<uint8_t*>(workspace) + w.bytes : nullptr);
  if (!workspace || workspace_bytes < w.bytes + bw.bytes)
    return fail(DS_ERR_INVALID, "workspace of %zu bytes < required %zu", workspace_bytes, w.bytes + bw.bytes);
  cudaStream_t cs = (cudaStream_t)compute_stream;
  cudaStream_t xs = copy_stream ? (cudaStream_t)copy_stream : cs;
  std::vector<const int64_t*> tok(nb);
  for (int b = 0; b < nb; ++b) {
    if (tokens_dev && tokens_dev[b]) {
      tok[b] = tokens_dev[b];
    } else {
      int64_t* dst = bw.tokens + (long long)b * n_max;
      if (cudaMemcpyAsync(dst, tokens_host[b], 8ull * n_tokens[b], cudaMemcpyHostToDevice, cs) != cudaSuccess)
        return cuda_fail("token upload");
      tok[b] = dst;
    }
  }
  trace(cs, 0);
  // copy stream: every request's reused layers into its cache (HBM-bound),
  // beside the compute stream's tensor-bound recompute of the batch
  thread_local cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  if (!ev_fork && (cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming) != cudaSuccess ||
                   cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming) != cudaSuccess))
    return cuda_fail("event");
  if (!reused.empty()) {
    if (xs != cs) {
      if (cudaEventRecord(ev_fork, cs) != cudaSuccess || cudaStreamWaitEvent(xs, ev_fork, 0) != cudaSuccess)
        return cuda_fail("fork");
    }
    for (int b = 0; b < nb; ++b)
      DS_TRY(kv_ingest_launch(sender_kv[b], out_kv[b], reused.data(), (int)reused.size(), d.n_kv_heads, d.head_dim,
                              n_tokens[b] - 1, xs),
             "kv ingest");
    trace(xs, DS_TRACE_INGEST);
  }
  for (int b = 0; b < nb; ++b) {
    Ctx c{m, d, w, &out_kv[b], cs};
    for (int i = 0; i < n_groups; ++i) {
      rc = recompute_group(c, tok[b], n_tokens[b] - 1, groups[2 * i], groups[2 * i + 1],
                           seed[b][i] ? seed[b][i]->hidden : nullptr);
      if (rc) return rc;
    }
  }
  std::vector<int> pos(nb);
  for (int b = 0; b < nb; ++b) {
    pos[b] = n_tokens[b] - 1;
    if (cudaMemcpyAsync(bw.ids + b, tok[b] + pos[b], 8, cudaMemcpyDeviceToDevice, cs) != cudaSuccess)
      return cuda_fail("anchor ids");
  }
  if (!reused.empty() && xs != cs) {
    if (cudaEventRecord(ev_join, xs) != cudaSuccess || cudaStreamWaitEvent(cs, ev_join, 0) != cudaSuccess)
      return cuda_fail("join");
  }
  return anchor_pass_batch(m, bw, out_kv, pos.data(), nb, bw.ids, logits_out, token_out, 1, nullptr, cs);
}

int ds_anchor_batch(const ds_model* m, int32_t batch, const int64_t* anchor_tokens_dev, const int32_t* positions,
                    const ds_kv_cache* kv, float* logits_out, int32_t* token_out, void* workspace,
                    size_t workspace_bytes, void* stream) {
  g_err.clear();
  if (!m || !m->layers) return fail(DS_ERR_INVALID, "model is NULL");
  const ds_dims& d = m->dims;
  int rc;
  if ((rc = check_dims(d))) return rc;
  if (batch < 1 || batch > kMaxBatch) return fail(DS_ERR_INVALID, "batch %d outside [1,%d]", batch, kMaxBatch);
  if (!anchor_tokens_dev || !positions || !kv || !logits_out)
    return fail(DS_ERR_INVALID, "anchor tokens, positions, caches and logits_out are required");
  int n_max = 0;
  std::vector<int> pos(batch);
  for (int b = 0; b < batch; ++b) {
    if (positions[b] < 1) return fail(DS_ERR_DEGENERATE, "row %d: need at least 2 tokens", b);
    if (positions[b] + 1 > d.max_seq) return fail(DS_ERR_INVALID, "row %d: position %d beyond max_seq", b, positions[b]);
    if ((rc = check_cache(&kv[b], d, positions[b] + 1, "cache"))) return rc;
    pos[b] = positions[b];
    n_max = positions[b] + 1 > n_max ? positions[b] + 1 : n_max;
  }
  Workspace w = carve(d, n_max, workspace);
  BatchWs bw = carve_batch(d, n_max, batch, workspace ? static_cast<uint8_t*>(workspace) + w.bytes : nullptr);
  if (!workspace || workspace_bytes < w.bytes + bw.bytes)
    return fail(DS_ERR_INVALID, "workspace of %zu bytes < required %zu", workspace_bytes, w.bytes + bw.bytes);
  return anchor_pass_batch(m, bw, kv, pos.data(), batch, anchor_tokens_dev, logits_out, token_out, 1, nullptr,
                           (cudaStream_t)stream);
}

int ds_decode_greedy_batch(const ds_model* m, int32_t batch, const ds_kv_cache* kv, const int32_t* positions,
                           const int32_t* first_token, int32_t steps, int32_t* tokens_out, void* workspace,
                           size_t workspace_bytes, void* stream) {
  g_err.clear();
  if (!m || !m->layers) return fail(DS_ERR_INVALID, "model is NULL");
  const ds_dims& d = m->dims;
  int rc;
  if ((rc = check_dims(d))) return rc;
  if (batch < 1 || batch > kMaxBatch) return fail(DS_ERR_INVALID, "batch %d outside [1,%d]", batch, kMaxBatch);
  if (steps < 1) return fail(DS_ERR_INVALID, "steps must be at least 1");
  if (!kv || !positions || !first_token || !tokens_out) return fail(DS_ERR_INVALID, "batch arrays are NULL");
  int n_max = 0;
  for (int b = 0; b < batch; ++b) {
    if (positions[b] < 1) return fail(DS_ERR_INVALID, "row %d: cache must hold at least one position", b);
    if ((long long)positions[b] + steps > d.max_seq)
      return fail(DS_ERR_INVALID, "row %d: decoding %d steps from %d positions exceeds max_seq %d", b, steps,
                  positions[b], d.max_seq);
    if ((rc = check_cache(&kv[b], d, positions[b] + steps - 1, "cache"))) return rc;
    n_max = positions[b] + steps > n_max ? positions[b] + steps : n_max;
  }
  Workspace w = carve(d, n_max, workspace);
  BatchWs bw = carve_batch(d, n_max, batch, workspace ? static_cast<uint8_t*>(workspace) + w.bytes : nullptr);
  if (!workspace || workspace_bytes < w.bytes + bw.bytes)
    return fail(DS_ERR_INVALID, "workspace of %zu bytes < required %zu", workspace_bytes, w.bytes + bw.bytes);
  cudaStream_t s = (cudaStream_t)stream;
  for (int b = 0; b < batch; ++b)
    DS_TRY(token_copy_launch(first_token + b, tokens_out + (long long)b * steps, bw.tok64 + b, s), "token copy");
  std::vector<int> pos(batch);
  for (int st = 1; st < steps; ++st) {
    for (int b = 0; b < batch; ++b) pos[b] = positions[b] + st - 1;
    rc = anchor_pass_batch(m, bw, kv, pos.data(), batch, bw.tok64, bw.logits, tokens_out + st, steps, bw.tok64, s);
    if (rc) return rc;
  }
  return DS_OK;
}

}  // extern "C"
