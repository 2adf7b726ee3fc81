// KV ingest: the reuse copy of _mixed_prefill (model.py:590-603) as a
// TMA-bulk-staged scatter into the consumer's paged cache.
//
// Work unit = one (reused layer, K|V, kv head, 64-position page): a
// contiguous run of rows*head_dim bf16 in both the producer's dense export
// [L][KVH][n][D] and the consumer's paged [L][pages][KVH][64][D] layouts
// (16 KB at D=128).  One elected thread per CTA streams its units through a
// STAGES-deep ring of shared-memory buffers:
//   cp.async.bulk global->shared (mbarrier complete_tx)  ->  cp.async.bulk shared->global
// so every byte moves as a 16-byte-aligned bulk transfer with no register
// staging.  HBM-bound: algorithmic bytes = 2 (read+write) x copied bytes.
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"

namespace ds {

constexpr int INGEST_STAGES_MAX = 4;

// Per-(reused layer) K/V bases travel by value (graph-capturable, 4 KB of
// kernel parameters); they may point into a peer GPU's HBM (P2P pull).
struct IngestArgs {
  const uint8_t* src_k[kMaxLayers];
  const uint8_t* src_v[kMaxLayers];
  uint8_t* dst_k[kMaxLayers];
  uint8_t* dst_v[kMaxLayers];
  long long src_head_stride, src_page_stride;  // bytes
  long long dst_head_stride, dst_page_stride;  // bytes
  const int32_t* src_table;
  const int32_t* dst_table;
  int n_layers, n_kv_heads, head_dim, window, n_pages;
};

DS_DEV void ingest_unit(const IngestArgs& a, int u, const uint8_t*& src, uint8_t*& dst, uint32_t& bytes) {
  // u = ((li * 2 + kv) * KVH + h) * n_pages + p
  int p = u % a.n_pages;
  int t = u / a.n_pages;
  int h = t % a.n_kv_heads;
  t /= a.n_kv_heads;
  int kv = t & 1;
  int li = t >> 1;
  int rows = min(kPage, a.window - p * kPage);
  bytes = (uint32_t)rows * a.head_dim * 2;
  int sp = a.src_table ? __ldg(a.src_table + p) : p;
  int dp = a.dst_table ? __ldg(a.dst_table + p) : p;
  src = (kv ? a.src_v[li] : a.src_k[li]) + h * a.src_head_stride + sp * a.src_page_stride;
  dst = (kv ? a.dst_v[li] : a.dst_k[li]) + h * a.dst_head_stride + dp * a.dst_page_stride;
}

__global__ void __launch_bounds__(32) kv_ingest_kernel(const __grid_constant__ IngestArgs a, int total_units, int stage_bytes,
                                                       int stages) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t bars[INGEST_STAGES_MAX];
  if (threadIdx.x != 0) return;
  const int n_my = (total_units - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  if (n_my <= 0) return;
  for (int s = 0; s < stages; ++s) mbar_init(&bars[s], 1);
  fence_mbar_init();

  auto issue_load = [&](int i) {
    const uint8_t* src;
    uint8_t* dst;
    uint32_t bytes;
    ingest_unit(a, (int)blockIdx.x + i * (int)gridDim.x, src, dst, bytes);
    const int s = i % stages;
    mbar_expect_tx(&bars[s], bytes);
    bulk_g2s(ring + s * stage_bytes, src, bytes, &bars[s]);
  };

  const int pro = n_my < stages ? n_my : stages;
  for (int i = 0; i < pro; ++i) issue_load(i);
  for (int i = 0; i < n_my; ++i) {
    const int s = i % stages;
    mbar_wait(&bars[s], (uint32_t)(i / stages) & 1u);
    const uint8_t* src;
    uint8_t* dst;
    uint32_t bytes;
    ingest_unit(a, (int)blockIdx.x + i * (int)gridDim.x, src, dst, bytes);
    bulk_s2g(dst, ring + s * stage_bytes, bytes);
    bulk_commit();
    const int refill = i - 1 + stages;
    if (i >= 1 && refill < n_my) {
      bulk_wait_read<1>();  // the store of unit i-1 has finished reading its stage
      issue_load(refill);
    }
  }
  bulk_wait<0>();
}

// Peer-source variant: when the producer's export lives on another GPU (mapped
// through CUDA IPC / peer access), every byte is pulled over NVLink with plain
// 16-byte vector loads (4 per thread in flight) and stored into the local
// paged cache -- the transfer and the scatter are one kernel.
constexpr int PEER_THREADS = 256;

__global__ void __launch_bounds__(PEER_THREADS) kv_ingest_peer_kernel(const __grid_constant__ IngestArgs a,
                                                                     long long total_units, int chunks_per_unit) {
  const long long n_chunks = total_units * chunks_per_unit;
  const long long stride = (long long)gridDim.x * PEER_THREADS;
  for (long long base = (long long)blockIdx.x * PEER_THREADS + threadIdx.x; base < n_chunks; base += 4 * stride) {
    uint4 v[4];
    uint4* dst[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long c = base + u * stride;
      dst[u] = nullptr;
      if (c < n_chunks) {
        const uint8_t* sp;
        uint8_t* dp;
        uint32_t bytes;
        ingest_unit(a, (int)(c / chunks_per_unit), sp, dp, bytes);
        const uint32_t off = (uint32_t)(c % chunks_per_unit) * 16;
        if (off < bytes) {
          v[u] = *reinterpret_cast<const uint4*>(sp + off);
          dst[u] = reinterpret_cast<uint4*>(dp + off);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (dst[u]) *dst[u] = v[u];
  }
}

bool ptr_on_this_device(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  return at.type != cudaMemoryTypeDevice || at.device == dev;
}

int kv_ingest_launch(const ds_kv_cache& src, const ds_kv_cache& dst, const int32_t* layers_host, int n_layers,
                     int n_kv_heads, int head_dim, int window, cudaStream_t stream, bool background) {
  if (n_layers <= 0 || window <= 0) return DS_OK;
  IngestArgs a;
  a.src_head_stride = src.head_stride * 2;
  a.src_page_stride = src.page_stride * 2;
  a.dst_head_stride = dst.head_stride * 2;
  a.dst_page_stride = dst.page_stride * 2;
  a.src_table = src.block_table;
  a.dst_table = dst.block_table;
  if (n_layers > kMaxLayers) return DS_ERR_INVALID;
  for (int i = 0; i < n_layers; ++i) {
    const int l = layers_host[i];
    a.src_k[i] = reinterpret_cast<const uint8_t*>(kv_layer_base(src, l, false));
    a.src_v[i] = reinterpret_cast<const uint8_t*>(kv_layer_base(src, l, true));
    a.dst_k[i] = reinterpret_cast<uint8_t*>(kv_layer_base(dst, l, false));
    a.dst_v[i] = reinterpret_cast<uint8_t*>(kv_layer_base(dst, l, true));
  }
  a.n_layers = n_layers;
  a.n_kv_heads = n_kv_heads;
  a.head_dim = head_dim;
  a.window = window;
  a.n_pages = (window + kPage - 1) / kPage;
  const int stage_bytes = kPage * head_dim * 2;
  // DS_INGEST_PEER_KERNEL=1 forces the peer-source kernel (single-GPU validation of that path)
  static const bool force_peer = getenv("DS_INGEST_PEER_KERNEL") && atoi(getenv("DS_INGEST_PEER_KERNEL"));
  if (force_peer || !ptr_on_this_device(a.src_k[0])) {
    const long long units = (long long)n_layers * 2 * n_kv_heads * a.n_pages;
    const int cpu = stage_bytes / 16;
    long long grid = (units * cpu + 4LL * PEER_THREADS - 1) / (4LL * PEER_THREADS);
    const long long cap = (long long)num_sms() * (background ? 1 : 8);
    if (grid > cap) grid = cap;
    count_launch();
    kv_ingest_peer_kernel<<<(int)grid, PEER_THREADS, 0, stream>>>(a, units, cpu);
    return launch_status();
  }
  // foreground: 4-stage rings, up to 8 CTAs per SM (HBM roofline when alone);
  // background: one 2-stage CTA per SM, small enough to share every SM with
  // a persistent tcgen05 GEMM of the concurrent recompute
  const int stages = background ? 2 : INGEST_STAGES_MAX;
  const int smem = stages * stage_bytes;
  static PerDevice attr;
  if (int rc_ = launch_status(ensure_smem_attr(kv_ingest_kernel, smem, attr))) return rc_;
  const long long total = (long long)n_layers * 2 * n_kv_heads * a.n_pages;
  if (total > 0x7fffffffLL) return DS_ERR_INVALID;
  int per_sm = background ? 1 : (200 * 1024) / (smem + 1024);
  if (per_sm < 1) per_sm = 1;
  if (per_sm > 8) per_sm = 8;
  long long grid = (long long)num_sms() * per_sm;
  if (grid > total) grid = total;
  count_launch();
  static PerDevice carve;
  prefer_max_smem_once(kv_ingest_kernel, carve);
  kv_ingest_kernel<<<(int)grid, 32, smem, stream>>>(a, (int)total, stage_bytes, stages);
  return launch_status();
}

}  // namespace ds
