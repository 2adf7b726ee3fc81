// Token-selective (CacheBlend-style) baseline: per-position KV deviation and
// the top-k position selection of token_selective_prefill (model.py:682-743).
//
//   kv_deviation   dev[p] = ||K0[:, p, :] - Ks[0, :, p, :]||_2 + ||V0 - Vs||_2 over
//                  heads x head_dim, one warp per position (K0/V0: the receiver's
//                  exact layer-0 projection of the window, Ks/Vs: the sender's cache)
//   select_topk    the ceil(ratio * window) largest deviations, ties to the lowest
//                  position (argsort(-dev, stable)), emitted in ascending position
//                  order with their token ids.  One CTA: an 8-bit radix select on
//                  the (non-negative) float bits finds the k-th largest key, then a
//                  stable block-wide compaction takes every key above it and the
//                  lowest-indexed keys equal to it.
#include "common.cuh"
#include "kernels.h"

namespace ds {

constexpr int DEV_THREADS = 256;

__global__ void __launch_bounds__(DEV_THREADS) kv_deviation_kernel(const bf16* k0, const bf16* v0,
                                                                   long long head_stride0, KvAddr s, int window,
                                                                   int n_kv_heads, int head_dim, float* dev) {
  const int warp = (blockIdx.x * DEV_THREADS + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= window) return;
  const int p = warp;
  float dk = 0.f, dv = 0.f;
  for (int h = 0; h < n_kv_heads; ++h) {
    const bf16* a = k0 + (long long)h * head_stride0 + (long long)p * head_dim;
    const bf16* b = v0 + (long long)h * head_stride0 + (long long)p * head_dim;
    const long long so = s.off(h, p);
    for (int j = lane * 2; j < head_dim; j += 64) {
      const float2 ka = unpack_bf16x2(*reinterpret_cast<const uint32_t*>(a + j));
      const float2 kb = unpack_bf16x2(*reinterpret_cast<const uint32_t*>(s.k + so + j));
      const float2 va = unpack_bf16x2(*reinterpret_cast<const uint32_t*>(b + j));
      const float2 vb = unpack_bf16x2(*reinterpret_cast<const uint32_t*>(s.v + so + j));
      dk += (ka.x - kb.x) * (ka.x - kb.x) + (ka.y - kb.y) * (ka.y - kb.y);
      dv += (va.x - vb.x) * (va.x - vb.x) + (va.y - vb.y) * (va.y - vb.y);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    dk += __shfl_xor_sync(0xffffffffu, dk, o);
    dv += __shfl_xor_sync(0xffffffffu, dv, o);
  }
  if (lane == 0) dev[p] = sqrtf(dk) + sqrtf(dv);
}

int kv_deviation_launch(const bf16* k0, const bf16* v0, long long head_stride0, const ds_kv_cache& sender, int window,
                        int n_kv_heads, int head_dim, float* dev, cudaStream_t stream) {
  KvAddr s;
  s.k = kv_layer_base(sender, 0, false);
  s.v = kv_layer_base(sender, 0, true);
  s.head_stride = sender.head_stride;
  s.page_stride = sender.page_stride;
  s.table = sender.block_table;
  s.head_dim = head_dim;
  const int blocks = (window * 32 + DEV_THREADS - 1) / DEV_THREADS;
  count_launch();
  kv_deviation_kernel<<<blocks, DEV_THREADS, 0, stream>>>(k0, v0, head_stride0, s, window, n_kv_heads, head_dim, dev);
  return launch_status();
}

constexpr int SEL_THREADS = 1024;

// inclusive block scan of one int per thread (SEL_THREADS threads)
DS_DEV int block_scan(int v, int* warp_sums) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  if (lane == 31) warp_sums[warp] = v;
  __syncthreads();
  if (warp == 0) {
    int w = warp_sums[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += t;
    }
    warp_sums[lane] = w;
  }
  __syncthreads();
  const int r = v + (warp ? warp_sums[warp - 1] : 0);
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(SEL_THREADS) select_topk_kernel(const float* dev, int window, int n_sel,
                                                                  const int64_t* tokens, int32_t* sel_pos,
                                                                  int64_t* sel_tok) {
  __shared__ int hist[256];
  __shared__ int warp_sums[32];
  __shared__ uint32_t s_prefix, s_remaining;
  const int tid = threadIdx.x;
  const int chunk = (window + SEL_THREADS - 1) / SEL_THREADS;
  const int lo = tid * chunk, hi = min(window, lo + chunk);
  auto key = [&](int p) { return __float_as_uint(fmaxf(dev[p], 0.f)); };  // non-negative: bits order = value order
  if (tid == 0) {
    s_prefix = 0;
    s_remaining = (uint32_t)n_sel;
  }
  uint32_t mask = 0;
  for (int shift = 24; shift >= 0; shift -= 8) {
    if (tid < 256) hist[tid] = 0;
    __syncthreads();
    const uint32_t prefix = s_prefix;
    for (int p = lo; p < hi; ++p) {
      const uint32_t k = key(p);
      if ((k & mask) == prefix) atomicAdd(&hist[(k >> shift) & 0xFF], 1);
    }
    __syncthreads();
    if (tid == 0) {
      uint32_t rem = s_remaining;
      int d = 255;
      for (; d > 0; --d) {
        if ((uint32_t)hist[d] >= rem) break;
        rem -= (uint32_t)hist[d];
      }
      s_prefix = prefix | ((uint32_t)d << shift);
      s_remaining = rem;  // how many keys equal to the final threshold are still needed (after this digit)
    }
    mask |= 0xFFu << shift;
    __syncthreads();
  }
  const uint32_t thr = s_prefix;      // the n_sel-th largest key
  const int need_eq = (int)s_remaining;  // keys == thr to take, lowest positions first
  // stable compaction in position order
  int n_gt = 0, n_eq = 0;
  for (int p = lo; p < hi; ++p) {
    const uint32_t k = key(p);
    n_gt += k > thr;
    n_eq += k == thr;
  }
  const int eq_before = block_scan(n_eq, warp_sums) - n_eq;
  int take_eq = min(n_eq, max(0, need_eq - eq_before));
  const int mine = n_gt + take_eq;
  int out = block_scan(mine, warp_sums) - mine;
  for (int p = lo; p < hi; ++p) {
    const uint32_t k = key(p);
    bool sel = k > thr;
    if (k == thr && take_eq > 0) {
      sel = true;
      --take_eq;
    }
    if (sel) {
      sel_pos[out] = p;
      sel_tok[out] = tokens[p];
      ++out;
    }
  }
}

int select_topk_launch(const float* dev, int window, int n_sel, const int64_t* tokens, int32_t* sel_pos,
                       int64_t* sel_tok, cudaStream_t stream) {
  if (n_sel < 1 || n_sel > window) return DS_ERR_INVALID;
  count_launch();
  select_topk_kernel<<<1, SEL_THREADS, 0, stream>>>(dev, window, n_sel, tokens, sel_pos, sel_tok);
  return launch_status();
}

}  // namespace ds
