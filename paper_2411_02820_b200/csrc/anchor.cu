// Anchor pass kernels: the single final position through every layer
// (_layer_single, model.py:547-562) and the first-token logits
// (_final_logits + argmax, model.py:565-566, 779).  All HBM-bound.
//
// The building blocks are device functions shared by two launch shapes, so
// both give bit-identical results:
//
//   gemv_tile      y = W[N][K] . x for one tile of 8 weight rows: 128 threads
//                  split K (16-byte coalesced row chunks, 16 loads in flight per
//                  thread), block-reduce, fused epilogue: RoPE + q / KV-cache
//                  write, residual add, SiLU / SwiGLU, logits + packed argmax
//                  (lowest id on ties).  An f32 input is RMSNorm'ed when staged
//                  (model.py:466-468).
//   attn_item      one (kv head, key split) item of the anchor row's attention
//                  over the cache (model.py:555-560) on the CUDA cores: scores
//                  of the R = H/KVH query heads into shared memory, split
//                  softmax, P.V; the last CTA of a kv head merges the splits.
//
// Launch shapes:
//   gemv_kernel / attn_decode_kernel   one launch per step (full prefill's last
//                  layer, the fallback path).
//   anchor_persistent_kernel           the whole anchor pass (32 layers x 5
//                  phases separated by grid barriers) in ONE launch of one
//                  128-thread CTA per SM.  Its footprint (88 registers x 128
//                  threads = 11 K registers, <= 33 KB shared memory) fits beside
//                  a tcgen05 GEMM CTA (24.6 K registers, 198.8 KB) and a flash
//                  attention CTA (53.8 K registers, 198.9 KB) of the other
//                  stream, so the anchor streams weights through the whole
//                  tensor-bound recompute without ever taking an SM away from
//                  it.  A recomputed layer's attention waits on the counter the
//                  recompute's QKV GEMM epilogue bumps (GemmEpi::done), not on
//                  a stream event.
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace ds {

constexpr int GEMV_THREADS = 128;
constexpr int GEMV_WARPS = GEMV_THREADS / 32;
constexpr int GEMV_ROWS = 8;    // weight rows per tile
constexpr int GEMV_UNROLL = 2;  // 16-byte chunks per row per thread in flight
constexpr int ATT_THREADS = GEMV_THREADS;
constexpr int ATT_TARGET_ITEMS = 296;  // two (kv head, split) items per SM of a B200

#if DS_ANCHOR_L2_HINT
// Weights are read once per pass: mark them first to go in L2, so the stream
// does not evict the recompute GEMMs' operand tiles.
DS_DEV uint64_t l2_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
DS_DEV uint4 ld_stream16(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(l2_evict_first()));
  return r;
}
DS_DEV void prefetch_weights_l2(const void* p, uint32_t bytes) {
#if DS_ANCHOR_L2_HINT > 1
  asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(p), "r"(bytes),
               "l"(l2_evict_first())
               : "memory");
#else
  prefetch_l2(p, bytes);
#endif
}
#else
DS_DEV uint4 ld_stream16(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
DS_DEV void prefetch_weights_l2(const void* p, uint32_t bytes) { prefetch_l2(p, bytes); }
#endif

// L2-coherent 16-byte load: data another CTA (or another stream's kernel)
// wrote while this kernel runs.
DS_DEV uint4 ld_cg16(const void* p) {
  uint4 r;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p)
               : "memory");
  return r;
}

DS_DEV unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

DS_DEV unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

DS_DEV float dot8(uint4 w, uint4 x) {
  float2 a = unpack_bf16x2(w.x), b = unpack_bf16x2(w.y), c = unpack_bf16x2(w.z), d = unpack_bf16x2(w.w);
  float2 p = unpack_bf16x2(x.x), q = unpack_bf16x2(x.y), r = unpack_bf16x2(x.z), s = unpack_bf16x2(x.w);
  float acc = a.x * p.x;
  acc = fmaf(a.y, p.y, acc);
  acc = fmaf(b.x, q.x, acc);
  acc = fmaf(b.y, q.y, acc);
  acc = fmaf(c.x, r.x, acc);
  acc = fmaf(c.y, r.y, acc);
  acc = fmaf(d.x, s.x, acc);
  acc = fmaf(d.y, s.y, acc);
  return acc;
}

DS_DEV unsigned long long pack_argmax(float v, int idx) {
  uint32_t u = __float_as_uint(v);
  uint32_t key = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return ((unsigned long long)key << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)idx);
}

// Sum each of a lane's V values over the LPK lanes of its key group (the lane
// bits below LPK), the same association tree as the xor butterfly (each node
// is partial(lane) + partial(lane ^ o) of the same two partials; + commutes),
// so bitwise equal to it -- with fewer shuffles: while a lane holds more than
// one value, a level keeps half of them and receives the partner's partials
// of that half instead of exchanging all of them (8 shuffles instead of 32 for
// 8 values over 16 lanes).  On return v[0 .. max(1, V / LPK)) hold the sums of
// values base.. (the returned index); lanes that end with the same index hold
// the same sum.
template <int V, int LPK>
DS_DEV int rs_sum(float (&v)[V], int lane) {
  int base = 0;
#pragma unroll
  for (int lvl = 0; (LPK >> (lvl + 1)) > 0; ++lvl) {
    const int o = LPK >> (lvl + 1);
    const int cnt = V >> lvl;  // values still held (compile time after unrolling)
    if (cnt >= 2) {
      const int h = cnt / 2;
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int i = 0; i < h; ++i) {
        const float keep = up ? v[i + h] : v[i];
        const float send = up ? v[i] : v[i + h];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
      if (up) base += h;
    } else {
      v[0] = v[0] + __shfl_xor_sync(0xffffffffu, v[0], o);
    }
  }
  return base;
}

// ---------------------------------------------------------------- GEMV

// Global row of slot r (0..7) of tile t.  QKV tiles hold 4 RoPE pairs
// (rows head*D + j0 + i and head*D + half + j0 + i, i < 4) so the rotation
// happens in the epilogue; other modes take 8 consecutive rows.
DS_DEV int gemv_row(const GemvArgs& a, int t, int r) {
  if (a.mode == EPI_SWIGLU_BF16) {
    // 4 gate rows and the 4 up rows that pair with them (blocks of 16, see ds_dims)
    const int blk = t >> 2, q = t & 3;
    return blk * 32 + (r < 4 ? q * 4 + r : 16 + q * 4 + r - 4);
  }
  if (a.mode != EPI_QKV_ROPE) return t * GEMV_ROWS + r;
  const int half = a.head_dim >> 1;
  const int per_head = half / 4;
  const int head = t / per_head, j0 = (t - head * per_head) * 4;
  return head * a.head_dim + (r < 4 ? j0 + r : half + j0 + r - 4);
}

// Threads 0..7: stream tile t's weight rows toward L2 (no wait).
DS_DEV void gemv_prefetch(const GemvArgs& a, int t) {
  if (threadIdx.x < GEMV_ROWS)
    prefetch_weights_l2(a.W + (long long)gemv_row(a, t, threadIdx.x) * a.ldw, (uint32_t)a.K * 2);
}

// Stage the input vector in shared memory as bf16 (RMSNorm fused when a.gain).
// `sync`: a barrier over the 128 staging threads (default: the whole CTA).
DS_DEV void cta_sync() { __syncthreads(); }
// tid: the thread's index among the 128 staging threads (a batched GEMV runs
// one staging group per 128-thread consumer warpgroup).
// The loads are issued in blocks of XB per thread before any is used (the
// loop one-load-per-iteration form waited one L2 round trip per 512 columns:
// ~15% of a batched GEMV's samples); for K <= XB * 512 the f32 row stays in
// registers between the sum of squares and the normalisation.  Accumulation
// order is unchanged (ascending k per thread).
// XB: loads in flight per thread (8 in the TMA-staged kernels; 2 in the
// register-capped persistent kernel, where more would spill).
template <int GEMV_XB = 8, typename SyncF>
DS_DEV void gemv_stage_x_t(const GemvArgs& a, bf16* xs, float* ssq, int tid, SyncF sync) {
  const int warp = tid >> 5, lane = tid & 31;
  const bool active = tid < GEMV_THREADS;
  constexpr int STEP = GEMV_THREADS * 4;
  if (a.x_f32) {
    float4 v[GEMV_XB];
    const bool one_block = a.K <= GEMV_XB * STEP;
    auto load_block = [&](int k0) {
#pragma unroll
      for (int u = 0; u < GEMV_XB; ++u) {
        const int k = k0 + u * STEP;
        v[u] = (active && k < a.K) ? __ldcg(reinterpret_cast<const float4*>(a.x_f32 + k)) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    float inv = 1.f;
    if (a.gain) {
      float ss = 0.f;
      for (int k0 = tid * 4; k0 < a.K; k0 += GEMV_XB * STEP) {
        load_block(k0);
#pragma unroll
        for (int u = 0; u < GEMV_XB; ++u)
          if (active && k0 + u * STEP < a.K)
            // explicit roundings: every kernel that inlines this gets the same bits
            ss = __fadd_rn(ss, __fmaf_rn(v[u].w, v[u].w,
                                         __fmaf_rn(v[u].z, v[u].z, __fmaf_rn(v[u].y, v[u].y, __fmul_rn(v[u].x, v[u].x)))));
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (lane == 0 && active) ssq[warp] = ss;
      sync();
      float t = 0.f;
#pragma unroll
      for (int w = 0; w < GEMV_WARPS; ++w) t += ssq[w];
      inv = 1.0f / sqrtf(t / (float)a.K + 1e-6f);
    }
    for (int k0 = tid * 4; k0 < a.K; k0 += GEMV_XB * STEP) {
      if (!(one_block && a.gain)) load_block(k0);
      float4 g[GEMV_XB];
#pragma unroll
      for (int u = 0; u < GEMV_XB; ++u) {
        const int k = k0 + u * STEP;
        g[u] = (a.gain && active && k < a.K) ? __ldg(reinterpret_cast<const float4*>(a.gain + k))
                                             : make_float4(1.f, 1.f, 1.f, 1.f);
      }
#pragma unroll
      for (int u = 0; u < GEMV_XB; ++u) {
        const int k = k0 + u * STEP;
        if (active && k < a.K) {
          uint2 p;
          p.x = pack_bf16x2(v[u].x * inv * g[u].x, v[u].y * inv * g[u].y);
          p.y = pack_bf16x2(v[u].z * inv * g[u].z, v[u].w * inv * g[u].w);
          *reinterpret_cast<uint2*>(xs + k) = p;
        }
      }
    }
  } else {
    constexpr int STEP8 = GEMV_THREADS * 8;
    for (int k0 = tid * 8; k0 < a.K; k0 += GEMV_XB * STEP8) {
      uint4 v[GEMV_XB];
#pragma unroll
      for (int u = 0; u < GEMV_XB; ++u) {
        const int k = k0 + u * STEP8;
        v[u] = (active && k < a.K) ? ld_cg16(a.x_bf16 + k) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int u = 0; u < GEMV_XB; ++u)
        if (active && k0 + u * STEP8 < a.K) *reinterpret_cast<uint4*>(xs + k0 + u * STEP8) = v[u];
    }
  }
  sync();
}
template <void (*Sync)() = cta_sync, int XB = 2>
DS_DEV void gemv_stage_x(const GemvArgs& a, bf16* xs, float* ssq) {
  gemv_stage_x_t<XB>(a, xs, ssq, (int)threadIdx.x, [] { Sync(); });
}

// The 128 accumulating threads' per-row pair sums -> row results (warp
// shuffles, then the 4 warps in order) -> the fused epilogue.  `sync`: a
// barrier over (at least) the 128 threads.
// The epilogue's own global inputs for tile t (RoPE cos/sin of the row pair,
// the residual of the row), loaded by threads 0..7 when the tile starts so
// their latency hides under the weight stream instead of following it.
struct EpiPre {
  float a, b;
};
DS_DEV EpiPre gemv_epi_pre(const GemvArgs& a, int t, int tid = threadIdx.x) {
  EpiPre e{0.f, 0.f};
  if (a.mode == EPI_QKV_ROPE) {
    if (tid < 4) {
      const int r0 = gemv_row(a, t, tid);
      const int half = a.head_dim >> 1, j = r0 % a.head_dim;
      e.a = __ldg(a.rope_cos + (long long)a.pos * half + j);
      e.b = __ldg(a.rope_sin + (long long)a.pos * half + j);
    }
  } else if (a.mode == EPI_RESID_F32) {
    if (tid < GEMV_ROWS) e.a = __ldcg(a.resid + t * GEMV_ROWS + tid);
  }
  return e;
}

template <typename Sync>
DS_DEV void gemv_finish(const GemvArgs& a, int t, const float2* s2, float (*red)[GEMV_ROWS], unsigned long long& best,
                        const EpiPre& pre, Sync sync, int tid = threadIdx.x) {
  const int warp = tid >> 5, lane = tid & 31;
  float s[GEMV_ROWS];
#pragma unroll
  for (int r = 0; r < GEMV_ROWS; ++r) s[r] = s2[r].x + s2[r].y;
  // the 8 rows' warp sums: the xor butterfly's tree by reduce-scatter (rs_sum), 9 shuffles instead of 40
  const int vb = rs_sum<GEMV_ROWS, 32>(s, lane);
  if ((lane & 3) == 0) red[warp][vb] = s[0];
  sync();
  if (tid < GEMV_ROWS) {
    float v = 0.f;
#pragma unroll
    for (int w = 0; w < GEMV_WARPS; ++w) v += red[w][tid];
    red[0][tid] = v;  // only thread tid touches column tid
  }
  sync();
  if (a.mode == EPI_QKV_ROPE) {
    if (tid < 4) {
      const int r0 = gemv_row(a, t, tid);
      const int head = r0 / a.head_dim, j = r0 - head * a.head_dim, half = a.head_dim >> 1;
      float lo = red[0][tid], hi = red[0][tid + 4];
      const bool is_q = head < a.n_heads, is_k = !is_q && head < a.n_heads + a.n_kv_heads;
      if (is_q || is_k) {
        const float cs = pre.a, sn = pre.b;
        const float x1 = lo, x2 = hi;
        // explicit roundings (no FMA contraction, whose choice may differ
        // between the kernels inlining this): one result for every launch shape
        lo = __fsub_rn(__fmul_rn(x1, cs), __fmul_rn(x2, sn));
        hi = __fadd_rn(__fmul_rn(x1, sn), __fmul_rn(x2, cs));
      }
      bf16* dst = is_q ? a.q_out + (long long)head * a.head_dim
                       : (is_k ? a.kv.k + a.kv.off(head - a.n_heads, a.pos)
                               : a.kv.v + a.kv.off(head - a.n_heads - a.n_kv_heads, a.pos));
      dst[j] = __float2bfloat16_rn(lo);
      dst[j + half] = __float2bfloat16_rn(hi);
    }
  } else if (a.mode == EPI_SWIGLU_BF16) {
    if (tid < 4) {
      const int o = (t >> 2) * 16 + (t & 3) * 4 + tid;
      a.out_bf16[o] = __float2bfloat16_rn(silu(red[0][tid]) * red[0][tid + 4]);
    }
  } else if (tid < GEMV_ROWS) {
    const int row = t * GEMV_ROWS + tid;
    const float v = red[0][tid];
    if (a.mode == EPI_RESID_F32) {
      a.out_f32[row] = pre.a + v;
    } else if (a.mode == EPI_SILU_BF16) {
      a.out_bf16[row] = __float2bfloat16_rn(silu(v));
    } else {
      a.out_f32[row] = v;
      const unsigned long long p = pack_argmax(v, row);
      best = p > best ? p : best;
    }
  }
  sync();  // red[] reused by the next tile
}

// One tile of 8 weight rows against the staged x, with its epilogue.  UNROLL
// (16-byte chunks per row per thread in flight) only batches the loads: every
// thread still accumulates its chunks in ascending order, so the persistent
// kernel (register-capped, UNROLL 2) and the stand-alone GEMV (UNROLL 4) give
// bit-identical results.
template <int UNROLL = GEMV_UNROLL>
DS_DEV void gemv_tile(const GemvArgs& a, int t, const bf16* xs, float (*red)[GEMV_ROWS], unsigned long long& best) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nchunk = a.K >> 3;
  const bf16* wr[GEMV_ROWS];
#pragma unroll
  for (int r = 0; r < GEMV_ROWS; ++r) wr[r] = a.W + (long long)gemv_row(a, t, r) * a.ldw;
  // even / odd element partial sums per row on packed fp32 pairs; the chunk of
  // x is unpacked once and serves all 8 rows
  const EpiPre pre = gemv_epi_pre(a, t);
  float2 s2[GEMV_ROWS];
#pragma unroll
  for (int r = 0; r < GEMV_ROWS; ++r) s2[r] = make_float2(0.f, 0.f);
  auto fma_chunk = [&](const uint4& w, const float2* xf, float2& acc) {
    acc = ffma2(bf16x2_to_float2(w.x), xf[0], acc);
    acc = ffma2(bf16x2_to_float2(w.y), xf[1], acc);
    acc = ffma2(bf16x2_to_float2(w.z), xf[2], acc);
    acc = ffma2(bf16x2_to_float2(w.w), xf[3], acc);
  };
  auto unpack_x = [&](int chunk, float2* xf) {
    const uint4 xv = *reinterpret_cast<const uint4*>(xs + chunk * 8);
    xf[0] = bf16x2_to_float2(xv.x);
    xf[1] = bf16x2_to_float2(xv.y);
    xf[2] = bf16x2_to_float2(xv.z);
    xf[3] = bf16x2_to_float2(xv.w);
  };
  int c = tid;
  for (; c + (UNROLL - 1) * GEMV_THREADS < nchunk; c += UNROLL * GEMV_THREADS) {
    uint4 w[UNROLL][GEMV_ROWS];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u)
#pragma unroll
      for (int r = 0; r < GEMV_ROWS; ++r) w[u][r] = ld_stream16(wr[r] + (c + u * GEMV_THREADS) * 8);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      float2 xf[4];
      unpack_x(c + u * GEMV_THREADS, xf);
#pragma unroll
      for (int r = 0; r < GEMV_ROWS; ++r) fma_chunk(w[u][r], xf, s2[r]);
    }
  }
  for (; c < nchunk; c += GEMV_THREADS) {
    float2 xf[4];
    unpack_x(c, xf);
#pragma unroll
    for (int r = 0; r < GEMV_ROWS; ++r) fma_chunk(ld_stream16(wr[r] + c * 8), xf, s2[r]);
  }
  gemv_finish(a, t, s2, red, best, pre, [] { __syncthreads(); });
}

// Every tile of one GEMV, strided over the grid; the next tile's weights are
// prefetched into L2 while the current one is reduced.
template <int UNROLL = GEMV_UNROLL>
DS_DEV unsigned long long gemv_all_tiles(const GemvArgs& a, const bf16* xs, float (*red)[GEMV_ROWS], int rank,
                                         int nranks) {
  const int tiles = a.N / GEMV_ROWS;
  unsigned long long best = 0ull;
  for (int t = rank; t < tiles; t += nranks) {
    if (t + nranks < tiles) gemv_prefetch(a, t + nranks);
    gemv_tile<UNROLL>(a, t, xs, red, best);
  }
  return best;
}

__global__ void __launch_bounds__(GEMV_THREADS) gemv_kernel(GemvArgs a) {
  extern __shared__ __align__(16) uint8_t smem_x[];
  bf16* xs = reinterpret_cast<bf16*>(smem_x);
  __shared__ float red[GEMV_WARPS][GEMV_ROWS];
  __shared__ float ssq[GEMV_WARPS];
  const int tid = threadIdx.x;
  // weights do not depend on the predecessor kernel: start streaming this
  // CTA's first tile into L2, let the successor launch, then wait (PDL)
  if ((int)blockIdx.x < a.N / GEMV_ROWS) gemv_prefetch(a, blockIdx.x);
  pdl_trigger();
  pdl_wait();
  gemv_stage_x(a, xs, ssq);
  unsigned long long best = gemv_all_tiles<2 * GEMV_UNROLL>(a, xs, red, blockIdx.x, gridDim.x);
  if (a.mode == EPI_STORE_F32 && a.argmax && tid < GEMV_ROWS) {
#pragma unroll
    for (int o = 4; o; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0x000000ffu, best, o);
      best = other > best ? other : best;
    }
    if (tid == 0 && best) atomicMax(a.argmax, best);
  }
}


// ---------------------------------------------------------------- TMA-staged stand-alone GEMV
//
// One CTA per SM: a producer warp streams each tile's 8 weight rows through a
// shared-memory ring in K-slices of KS columns (`cp.async.bulk`, one
// elected thread, complete_tx on the slot's mbarrier), so ~160 KB per SM are in
// flight without a register per byte; the 4 consumer warps read the slices
// from shared memory.  Thread t still accumulates its chunks c = t, t+128, ...
// in ascending order and the reduction is gemv_finish, so the results are the
// register-streaming gemv_tile's bit for bit.  Used alone (not beside the
// recompute), for K a multiple of 1024.
constexpr int TMA_THREADS = GEMV_THREADS + 32;   // + producer warp

DS_DEV void named_sync_consumers() { asm volatile("bar.sync 1, %0;" ::"n"(GEMV_THREADS) : "memory"); }

// KS: columns per ring slot (a multiple of 128 threads x 8); each row's slice
// is one bulk copy of KS*2 bytes.  Thread t's chunks stay t, t+128, ... in
// ascending order for every KS.
template <int KS>
__global__ void __launch_bounds__(TMA_THREADS, 1) gemv_tma_kernel(GemvArgs a, int slots) {
  constexpr int SLOT = GEMV_ROWS * KS * 2;
  constexpr int CPT = KS / (GEMV_THREADS * 8);  // chunks per thread per slot
  extern __shared__ __align__(128) uint8_t smem_dyn[];
  uint8_t* ring = smem_dyn;
  bf16* xs = reinterpret_cast<bf16*>(smem_dyn + (size_t)slots * SLOT);
  __shared__ __align__(8) uint64_t full[16], empty[16];
  __shared__ int tile_of[16];  // the tile whose first slice a slot holds (-1: no more tiles)
  __shared__ float red[GEMV_WARPS][GEMV_ROWS];
  __shared__ float ssq[GEMV_WARPS];
  const int tid = threadIdx.x;
  const int tiles = a.N / GEMV_ROWS, ks = a.K / KS;
  if (tid == GEMV_THREADS) {
    for (int i = 0; i < slots; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], GEMV_WARPS);
    }
    fence_mbar_init();
  }
  __syncthreads();
  pdl_trigger();
  if (tid >= GEMV_THREADS) {
    // producer: weights never depend on the predecessor -- start before the PDL wait
    if (tid == GEMV_THREADS) {
      int slot = 0;
      uint32_t phase = 0;
      // the next tile's ticket is claimed as soon as the current tile's first
      // slice is issued, so its round trip overlaps the slot waits
      int t = a.tile_ctr ? (int)atomicAdd(a.tile_ctr, 1u) : (int)blockIdx.x;
      for (;;) {
        mbar_wait(&empty[slot], phase ^ 1);
        if (t >= tiles) {
          tile_of[slot] = -1;
          mbar_arrive(&full[slot]);
          break;
        }
        tile_of[slot] = t;
        int nt = 0;
        for (int s = 0; s < ks; ++s) {
          if (s) mbar_wait(&empty[slot], phase ^ 1);
          mbar_expect_tx(&full[slot], SLOT);
#pragma unroll
          for (int r = 0; r < GEMV_ROWS; ++r)
            bulk_g2s(ring + slot * SLOT + r * KS * 2, a.W + (long long)gemv_row(a, t, r) * a.ldw + (long long)s * KS,
                     KS * 2, &full[slot]);
          if (s == 0) nt = a.tile_ctr ? (int)atomicAdd(a.tile_ctr, 1u) : t + (int)gridDim.x;
          if (++slot == slots) {
            slot = 0;
            phase ^= 1;
          }
        }
        t = nt;
      }
      // every ticket of this CTA is claimed: the grid's last CTA re-zeroes the counters
      if (a.tile_ctr) {
        __threadfence();
        if (atomicAdd(a.tile_ctr + 1, 1u) == gridDim.x - 1) {
          a.tile_ctr[0] = 0u;
          a.tile_ctr[1] = 0u;
        }
      }
    }
    return;
  }
  pdl_wait();
  gemv_stage_x<named_sync_consumers, 8>(a, xs, ssq);
  int slot = 0;
  uint32_t phase = 0;
  unsigned long long best = 0ull;
  for (;;) {
    mbar_wait(&full[slot], phase);  // the tile's first slice (or the end mark)
    const int t = *reinterpret_cast<volatile int*>(&tile_of[slot]);
    if (t < 0) break;
    const EpiPre pre = gemv_epi_pre(a, t);
    float2 s2[GEMV_ROWS];
#pragma unroll
    for (int r = 0; r < GEMV_ROWS; ++r) s2[r] = make_float2(0.f, 0.f);
    for (int s = 0; s < ks; ++s) {
      if (s) mbar_wait(&full[slot], phase);
#pragma unroll
      for (int cc = 0; cc < CPT; ++cc) {
        const int c = s * (KS / 8) + cc * GEMV_THREADS + tid;  // this thread's chunk
        const uint4 xv = *reinterpret_cast<const uint4*>(xs + c * 8);
        const float2 xf[4] = {bf16x2_to_float2(xv.x), bf16x2_to_float2(xv.y), bf16x2_to_float2(xv.z),
                              bf16x2_to_float2(xv.w)};
#pragma unroll
        for (int r = 0; r < GEMV_ROWS; ++r) {
          const uint4 w =
              *reinterpret_cast<const uint4*>(ring + slot * SLOT + r * KS * 2 + (cc * GEMV_THREADS + tid) * 16);
          s2[r] = ffma2(bf16x2_to_float2(w.x), xf[0], s2[r]);
          s2[r] = ffma2(bf16x2_to_float2(w.y), xf[1], s2[r]);
          s2[r] = ffma2(bf16x2_to_float2(w.z), xf[2], s2[r]);
          s2[r] = ffma2(bf16x2_to_float2(w.w), xf[3], s2[r]);
        }
      }
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&empty[slot]);
      if (++slot == slots) {
        slot = 0;
        phase ^= 1;
      }
    }
    gemv_finish(a, t, s2, red, best, pre, [] { named_sync_consumers(); });
  }
  if (a.mode == EPI_STORE_F32 && a.argmax && tid < GEMV_ROWS) {
#pragma unroll
    for (int o = 4; o; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0x000000ffu, best, o);
      best = other > best ? other : best;
    }
    if (tid == 0 && best) atomicMax(a.argmax, best);
  }
}

__global__ void argmax_finalize_kernel(const unsigned long long* packed, int32_t* token, int64_t* token64) {
  const int32_t t = (int32_t)(0xFFFFFFFFu - (uint32_t)(*packed & 0xFFFFFFFFull));
  if (token) *token = t;
  if (token64) *token64 = t;
}

// Decode bookkeeping: dst32 = dst64 = *src (the greedy token that seeds the next step).
__global__ void token_copy_kernel(const int32_t* src, int32_t* dst32, int64_t* dst64) {
  const int32_t t = *src;
  if (dst32) *dst32 = t;
  if (dst64) *dst64 = t;
}

int token_copy_launch(const int32_t* src, int32_t* dst32, int64_t* dst64, cudaStream_t stream) {
  count_launch();
  static PerDevice carve;
  prefer_max_smem_once(token_copy_kernel, carve);
  token_copy_kernel<<<1, 1, 0, stream>>>(src, dst32, dst64);
  return launch_status();
}

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

template <int KS>
static int gemv_tma_launch_t(const GemvArgs& a, cudaStream_t stream, int ctas_per_sm) {
  constexpr int SLOT = GEMV_ROWS * KS * 2;
  const int xbytes = (a.K * 2 + 127) & ~127;
  // 196 KB: one CTA fits beside a persistent anchor CTA (28 KB + reservations)
  // on an SM, so this kernel on another stream can always be placed while a
  // fused call's anchor holds every SM -- a 200 KB ring could not, and the GPU's
  // CTA dispatch then starved the fused call's GEMMs (deadlock, 10 s trap).
  // 1% slower alone than 200 KB (DS_GEMV_SMEM_KB: experiments).
  static const int budget = env_int("DS_GEMV_SMEM_KB", 196) * 1024;
  int slots = (budget / ctas_per_sm - xbytes) / SLOT;
  slots = slots > 16 ? 16 : slots;
  if (slots < 2) return DS_ERR_INVALID;
  const int smem = slots * SLOT + xbytes;
  auto kern = gemv_tma_kernel<KS>;
  static PerDevice attr;
  if (int rc_ = launch_status(ensure_smem_attr(kern, smem, attr))) return rc_;
  const int tiles = a.N / GEMV_ROWS, cap = num_sms() * ctas_per_sm;
  const int grid = tiles < cap ? tiles : cap;
  count_launch();
  return launch_status(launch_pdl(kern, dim3(grid), dim3(TMA_THREADS), smem, stream, a, slots));
}

// Slice width and CTAs per SM (DS_GEMV_KS, DS_GEMV_TMA_CTAS: experiments).
static int gemv_tma_launch(const GemvArgs& a_in, cudaStream_t stream) {
  static const bool claim = env_int("DS_GEMV_CLAIM", 1) != 0;  // 0: blockIdx-strided tiles (A/B)
  GemvArgs a = a_in;
  if (!claim) a.tile_ctr = nullptr;
  static const int ks_max = env_int("DS_GEMV_KS", 4096);
  static const int ctas = env_int("DS_GEMV_TMA_CTAS", 1) < 1 ? 1 : env_int("DS_GEMV_TMA_CTAS", 1);
  if (ks_max >= 4096 && a.K % 4096 == 0) return gemv_tma_launch_t<4096>(a, stream, ctas);
  if (ks_max >= 2048 && a.K % 2048 == 0) return gemv_tma_launch_t<2048>(a, stream, ctas);
  if (a.K % 1024 == 0) return gemv_tma_launch_t<1024>(a, stream, ctas);
  return DS_ERR_INVALID;
}

// DS_GEMV_TMA=0: the register-streaming kernel for every stand-alone GEMV (A/B).
static bool gemv_tma_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DS_GEMV_TMA");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// staged: the TMA-staged kernel may serve the call (K a multiple of 1024, at
// least one tile per SM).  With one bulk copy per 8 KB row slice it streams
// faster than the register kernel (stand-alone anchor 2.79 vs 4.30 ms); with
// 2 KB copies it did not (the bulk-copy count, not the bytes, was the limit).
int gemv_launch(const GemvArgs& a, cudaStream_t stream, bool staged) {
  if ((a.N % GEMV_ROWS) || (a.K & 7) || (a.mode == EPI_SWIGLU_BF16 && a.N % 32)) return DS_ERR_INVALID;
  if (a.mode == EPI_QKV_ROPE && (a.head_dim % 8 || a.N % a.head_dim)) return DS_ERR_INVALID;
  if (staged && gemv_tma_enabled() && a.K % 1024 == 0 && a.N / GEMV_ROWS >= 148)
    if (gemv_tma_launch(a, stream) == DS_OK) return DS_OK;
  const int tiles = a.N / GEMV_ROWS;
  const int smem = a.K * 2;
  static PerDevice attr;
  if (int rc_ = launch_status(ensure_smem_attr(gemv_kernel, smem > 48 * 1024 ? smem : 48 * 1024, attr))) return rc_;
  static int per_sm_cap = -1;
  if (per_sm_cap < 0) {
    const char* v = getenv("DS_GEMV_PER_SM");  // experiments
    per_sm_cap = v ? atoi(v) : 16;
    if (per_sm_cap < 1) per_sm_cap = 16;
  }
  int per_sm = (200 * 1024) / (smem + 1024);
  per_sm = per_sm < 1 ? 1 : (per_sm > per_sm_cap ? per_sm_cap : per_sm);
  const int cap = num_sms() * per_sm;
  const int grid = tiles < cap ? tiles : cap;
  count_launch();
  static PerDevice carve;
  prefer_max_smem_once(gemv_kernel, carve);
  return launch_status(launch_pdl(gemv_kernel, dim3(grid), dim3(GEMV_THREADS), smem, stream, a));
}

// ---------------------------------------------------------------- batched GEMV
//
// nb anchor rows (one per request of a consumer's batch, or one per sequence
// of a batched decode step) against ONE stream of the weights: the TMA ring
// of gemv_tma_kernel, read by WG consumer warpgroups of 128 threads, each
// holding up to NBW rows' accumulators.  Row b's x is staged (RMSNorm'ed) by
// its warpgroup exactly as the single-row kernel stages it; thread t of the
// warpgroup accumulates chunks t, t+128, ... in ascending order for each row,
// and gemv_finish reduces and runs the epilogue per row -- so every row's
// result is the single-row GEMV's bit for bit, with the weight bytes read once
// per launch instead of once per row.
DS_DEV void bar_named(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

DS_HOST_DEV_INLINE GemvArgs gemv_row_view(const GemvArgs& a, const GemvBatch& bt, int b) {
  GemvArgs v = a;
  if (v.x_f32) v.x_f32 += b * bt.x_stride;
  if (v.x_bf16) v.x_bf16 += b * bt.x_stride;
  if (v.out_f32) v.out_f32 += b * bt.out_stride;
  if (v.resid) v.resid += b * bt.out_stride;
  if (v.out_bf16) v.out_bf16 += b * bt.out_stride;
  if (v.q_out) v.q_out += b * bt.q_stride;
  if (v.argmax) v.argmax += b;
  v.tile_ctr = nullptr;  // rows launched one by one would share the counters
  v.pos = bt.pos[b];
  v.kv = bt.kv[b];
  return v;
}

// Two rows per warpgroup and one warpgroup per row pair: the per-thread
// instruction count per weight byte stays near the single-row kernel's (each
// bf16 pair is unpacked once and feeds 2 rows' FFMA2s), and the SM runs
// WG + 1 warps per sub-partition instead of one, so the FMA / issue work of
// several rows never throttles the weight stream (4 rows on one warpgroup: 3.5x
// slower than one row).  Registers: every CTA must fit beside one
// persistent-anchor warp (2.8 K registers) per SM sub-partition, which holds
// WG + 1 of this kernel's warps.
// Rows per epilogue thread group: QKV / SwiGLU pair two accumulators per output.
DS_DEV int gemv_epi_per(int mode) { return (mode == EPI_QKV_ROPE || mode == EPI_SWIGLU_BF16) ? 4 : GEMV_ROWS; }

// gemv_finish for the nbw rows of a warpgroup with two barriers in all (one
// gemv_finish per row takes three): the same shuffles, the same warp order of
// the cross-warp sum and the same epilogue arithmetic per row, so the same
// bits.  Epilogue thread tid < per * nbw handles row tid / per, slot tid % per
// (its `pre` loaded for that slot); argmax maxima stay with that thread.
template <int NBW, typename Sync>
DS_DEV void gemv_finish_rows(const GemvArgs& a, const GemvBatch& bt, int b0, int nbw, int t,
                             const float2 (*s2)[GEMV_ROWS], float (*red)[NBW * GEMV_ROWS], unsigned long long& best,
                             const EpiPre& pre, Sync sync, int tid) {
  const int warp = tid >> 5, lane = tid & 31;
  {
    // all rows' warp sums at once: the butterfly's tree by reduce-scatter (rs_sum)
    constexpr int NV = NBW * GEMV_ROWS;
    float sr[NV];
#pragma unroll
    for (int i = 0; i < NBW; ++i)
#pragma unroll
      for (int r = 0; r < GEMV_ROWS; ++r) sr[i * GEMV_ROWS + r] = i < nbw ? s2[i][r].x + s2[i][r].y : 0.f;
    const int vb = rs_sum<NV, 32>(sr, lane);
    constexpr int VC = NV / 32 > 0 ? NV / 32 : 1;
    constexpr int DUP = NV >= 32 ? 1 : 32 / NV;  // lanes holding the same sum
    if (lane % DUP == 0) {
#pragma unroll
      for (int q = 0; q < VC; ++q)
        if (vb + q < GEMV_ROWS * nbw) red[warp][vb + q] = sr[q];
    }
  }
  sync();
  if (tid < GEMV_ROWS * nbw) {
    float v = 0.f;
#pragma unroll
    for (int w = 0; w < GEMV_WARPS; ++w) v += red[w][tid];
    red[0][tid] = v;  // only thread tid touches column tid
  }
  sync();
  const int per = gemv_epi_per(a.mode);
  if (tid < per * nbw) {
    const int i = tid / per, r = tid - i * per;
    const GemvArgs v = gemv_row_view(a, bt, b0 + i);
    const float* rv = red[0] + i * GEMV_ROWS;
    if (a.mode == EPI_QKV_ROPE) {
      const int r0 = gemv_row(v, t, r);
      const int head = r0 / v.head_dim, j = r0 - head * v.head_dim, half = v.head_dim >> 1;
      float lo = rv[r], hi = rv[r + 4];
      const bool is_q = head < v.n_heads, is_k = !is_q && head < v.n_heads + v.n_kv_heads;
      if (is_q || is_k) {
        const float cs = pre.a, sn = pre.b;
        const float x1 = lo, x2 = hi;
        lo = __fsub_rn(__fmul_rn(x1, cs), __fmul_rn(x2, sn));
        hi = __fadd_rn(__fmul_rn(x1, sn), __fmul_rn(x2, cs));
      }
      bf16* dst = is_q ? v.q_out + (long long)head * v.head_dim
                       : (is_k ? v.kv.k + v.kv.off(head - v.n_heads, v.pos)
                               : v.kv.v + v.kv.off(head - v.n_heads - v.n_kv_heads, v.pos));
      dst[j] = __float2bfloat16_rn(lo);
      dst[j + half] = __float2bfloat16_rn(hi);
    } else if (a.mode == EPI_SWIGLU_BF16) {
      const int o = (t >> 2) * 16 + (t & 3) * 4 + r;
      v.out_bf16[o] = __float2bfloat16_rn(silu(rv[r]) * rv[r + 4]);
    } else {
      const int row = t * GEMV_ROWS + r;
      const float x = rv[r];
      if (a.mode == EPI_RESID_F32) {
        v.out_f32[row] = pre.a + x;
      } else if (a.mode == EPI_SILU_BF16) {
        v.out_bf16[row] = __float2bfloat16_rn(silu(x));
      } else {
        v.out_f32[row] = x;
        const unsigned long long pk = pack_argmax(x, row);
        best = pk > best ? pk : best;
      }
    }
  }
  sync();  // red[] reused by the next tile
}

template <int KS, int NBW, int WG, bool xstream>
__global__ void __maxnreg__(WG == 1 ? 168 : (WG == 2 ? 136 : (WG == 3 ? 104 : 80)))
    gemv_batch_kernel(const __grid_constant__ GemvArgs a, const __grid_constant__ GemvBatch bt, int slots) {
  constexpr int SLOT = GEMV_ROWS * KS * 2;
  constexpr int CPT = KS / (GEMV_THREADS * 8);
  constexpr int NC = WG * GEMV_THREADS;
  // xstream (bf16 x too large to stage whole, e.g. W2 at 8 rows): each ring slot
  // also carries the rows' x slice for its K range (the same bytes, per tile)
  const int SLOTX = xstream ? SLOT + bt.nb * KS * 2 : SLOT;
  extern __shared__ __align__(128) uint8_t smem_dyn[];
  uint8_t* ring = smem_dyn;
  bf16* xs = reinterpret_cast<bf16*>(smem_dyn + (size_t)slots * SLOTX);  // [nb][K] (not xstream)
  __shared__ __align__(8) uint64_t full[16], empty[16];
  __shared__ float red[WG][GEMV_WARPS][NBW * GEMV_ROWS];
  __shared__ float ssq[WG][GEMV_WARPS];
  const int tid = threadIdx.x;
  const int tiles = a.N / GEMV_ROWS, ks = a.K / KS;
  if (tid == NC) {
    for (int i = 0; i < slots; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], WG * GEMV_WARPS);
    }
    fence_mbar_init();
  }
  __syncthreads();
  pdl_trigger();
  if (tid >= NC) {
    if (tid == NC) {  // producer: the weights never depend on the predecessor (x does)
      int slot = 0;
      uint32_t phase = 0;
      bool waited = false;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x)
        for (int s = 0; s < ks; ++s) {
          mbar_wait(&empty[slot], phase ^ 1);
          mbar_expect_tx(&full[slot], SLOTX);
          uint8_t* dst = ring + (size_t)slot * SLOTX;
#pragma unroll
          for (int r = 0; r < GEMV_ROWS; ++r)
            bulk_g2s(dst + r * KS * 2, a.W + (long long)gemv_row(a, t, r) * a.ldw + (long long)s * KS, KS * 2,
                     &full[slot]);
          if (xstream) {
            if (!waited) {
              pdl_wait();
              waited = true;
            }
            for (int b = 0; b < bt.nb; ++b)
              bulk_g2s(dst + SLOT + b * KS * 2, a.x_bf16 + b * bt.x_stride + (long long)s * KS, KS * 2, &full[slot]);
          }
          if (++slot == slots) {
            slot = 0;
            phase ^= 1;
          }
        }
    }
    return;
  }
  const int wg = tid / GEMV_THREADS, t = tid - wg * GEMV_THREADS;
  const int b0 = wg * NBW;
  const int nbw = min(NBW, bt.nb - b0);
  auto sync = [wg] { bar_named(1 + wg, GEMV_THREADS); };
  pdl_wait();
  if (!xstream) {
    for (int i = 0; i < nbw; ++i) {
      const GemvArgs v = gemv_row_view(a, bt, b0 + i);
      gemv_stage_x_t(v, xs + (long long)(b0 + i) * a.K, ssq[wg], t, sync);
    }
  }
  int slot = 0;
  uint32_t phase = 0;
  unsigned long long best = 0ull;
  const int per = gemv_epi_per(a.mode);
  for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    // the epilogue inputs of the (row, slot) this thread finishes, loaded at tile start
    const EpiPre pre = t < per * nbw ? gemv_epi_pre(gemv_row_view(a, bt, b0 + t / per), tile, t % per)
                                     : EpiPre{0.f, 0.f};
    float2 s2[NBW][GEMV_ROWS];
#pragma unroll
    for (int i = 0; i < NBW; ++i)
#pragma unroll
      for (int r = 0; r < GEMV_ROWS; ++r) s2[i][r] = make_float2(0.f, 0.f);
    for (int s = 0; s < ks; ++s) {
      mbar_wait(&full[slot], phase);
#pragma unroll
      for (int cc = 0; cc < CPT; ++cc) {
        const int c = s * (KS / 8) + cc * GEMV_THREADS + t;  // this thread's chunk
        float2 xf[NBW][4];
#pragma unroll
        for (int i = 0; i < NBW; ++i) {
          const uint4* xp =
              xstream ? reinterpret_cast<const uint4*>(ring + (size_t)slot * SLOTX + SLOT + (b0 + i) * KS * 2 +
                                                       (cc * GEMV_THREADS + t) * 16)
                      : reinterpret_cast<const uint4*>(xs + (long long)(b0 + i) * a.K + c * 8);
          const uint4 xv = i < nbw ? *xp : make_uint4(0u, 0u, 0u, 0u);
          xf[i][0] = bf16x2_to_float2(xv.x);
          xf[i][1] = bf16x2_to_float2(xv.y);
          xf[i][2] = bf16x2_to_float2(xv.z);
          xf[i][3] = bf16x2_to_float2(xv.w);
        }
#pragma unroll
        for (int r = 0; r < GEMV_ROWS; ++r) {
          const uint4 w =
              *reinterpret_cast<const uint4*>(ring + (size_t)slot * SLOTX + r * KS * 2 + (cc * GEMV_THREADS + t) * 16);
          const float2 w0 = bf16x2_to_float2(w.x), w1 = bf16x2_to_float2(w.y);
          const float2 w2 = bf16x2_to_float2(w.z), w3 = bf16x2_to_float2(w.w);
#pragma unroll
          for (int i = 0; i < NBW; ++i) {
            if (i < nbw) {
              s2[i][r] = ffma2(w0, xf[i][0], s2[i][r]);
              s2[i][r] = ffma2(w1, xf[i][1], s2[i][r]);
              s2[i][r] = ffma2(w2, xf[i][2], s2[i][r]);
              s2[i][r] = ffma2(w3, xf[i][3], s2[i][r]);
            }
          }
        }
      }
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&empty[slot]);
      if (++slot == slots) {
        slot = 0;
        phase ^= 1;
      }
    }
    gemv_finish_rows<NBW>(a, bt, b0, nbw, tile, s2, red[wg], best, pre, sync, t);
  }
  if (a.mode == EPI_STORE_F32 && a.argmax && t < 32) {
    // row i's maxima sit with threads 8i..8i+7 (warp 0 of the warpgroup)
#pragma unroll
    for (int o = 4; o; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
      best = other > best ? other : best;
    }
    if ((t & 7) == 0 && t < GEMV_ROWS * nbw && best) atomicMax(a.argmax + b0 + t / GEMV_ROWS, best);
  }
}

template <int KS, int NBW, int WG>
static int gemv_batch_launch_t(const GemvArgs& a, const GemvBatch& bt, cudaStream_t stream, bool xstream = false) {
  constexpr int SLOT = GEMV_ROWS * KS * 2;
  const int slotx = xstream ? SLOT + bt.nb * KS * 2 : SLOT;
  const int xbytes = xstream ? 0 : (bt.nb * a.K * 2 + 127) & ~127;
  static const int budget = env_int("DS_GEMV_SMEM_KB", 196) * 1024;  // fits beside a persistent anchor CTA
  int slots = (budget - xbytes) / slotx;
  slots = slots > 16 ? 16 : slots;
  if (slots < 2) return DS_ERR_INVALID;
  const int smem = slots * slotx + xbytes;
  auto kern = xstream ? gemv_batch_kernel<KS, NBW, WG, true> : gemv_batch_kernel<KS, NBW, WG, false>;
  static PerDevice attr[2];
  if (int rc_ = launch_status(ensure_smem_attr(kern, smem, attr[xstream ? 1 : 0]))) return rc_;
  const int tiles = a.N / GEMV_ROWS, cap = num_sms();
  const int grid = tiles < cap ? tiles : cap;
  count_launch();
  return launch_status(launch_pdl(kern, dim3(grid), dim3(WG * GEMV_THREADS + 32), smem, stream, a, bt, slots));
}

#ifndef DS_GEMVB_NBW
#define DS_GEMVB_NBW 2  // rows per consumer warpgroup (experiments: 1, 2, 4)
#endif
template <int KS>
static int gemv_batch_launch_ks(const GemvArgs& a, const GemvBatch& bt, cudaStream_t stream, bool xstream = false) {
  if (DS_GEMVB_NBW == 1 && bt.nb <= 4) {
    switch (bt.nb) {
      case 1: return gemv_batch_launch_t<KS, 1, 1>(a, bt, stream, xstream);
      case 2: return gemv_batch_launch_t<KS, 1, 2>(a, bt, stream, xstream);
      case 3: return gemv_batch_launch_t<KS, 1, 3>(a, bt, stream, xstream);
      default: return gemv_batch_launch_t<KS, 1, 4>(a, bt, stream, xstream);
    }
  }
  if (DS_GEMVB_NBW == 4) {
    if (bt.nb <= 4) return gemv_batch_launch_t<KS, 4, 1>(a, bt, stream, xstream);
    return gemv_batch_launch_t<KS, 4, 2>(a, bt, stream, xstream);
  }
  switch ((bt.nb + 1) / 2) {
    case 1: return gemv_batch_launch_t<KS, 2, 1>(a, bt, stream, xstream);
    case 2: return gemv_batch_launch_t<KS, 2, 2>(a, bt, stream, xstream);
    case 3: return gemv_batch_launch_t<KS, 2, 3>(a, bt, stream, xstream);
    default: return gemv_batch_launch_t<KS, 2, 4>(a, bt, stream, xstream);
  }
}

// Rows per launch: as many as fit in shared memory beside a 2-slot ring (the
// 8B shape's K = 4096 GEMVs: 8).  A bf16 x that does not fit whole (W2 at
// d_ff = 14336 beyond 4 rows of 28 KB) is streamed through the ring with the
// weights instead (DS_GEMVB_XSTREAM=0: split into launches of `fit` rows, each
// re-reading the weights).  Shapes the TMA kernel does not take (K not a
// multiple of 1024, fewer tiles than SMs) run the single-row GEMV per row --
// the same bits either way.
int gemv_batch_launch(const GemvArgs& a, const GemvBatch& bt, cudaStream_t stream) {
  if (bt.nb < 1 || bt.nb > kMaxBatch) return DS_ERR_INVALID;
  if ((a.N % GEMV_ROWS) || (a.K & 7) || (a.mode == EPI_SWIGLU_BF16 && a.N % 32)) return DS_ERR_INVALID;
  if (a.mode == EPI_QKV_ROPE && (a.head_dim % 8 || a.N % a.head_dim)) return DS_ERR_INVALID;
  static const int ks_max = env_int("DS_GEMVB_KS", 4096);  // slice width (experiments)
  const int ks = (ks_max >= 4096 && a.K % 4096 == 0) ? 4096 : ((ks_max >= 2048 && a.K % 2048 == 0) ? 2048 : 1024);
  static const int budget = env_int("DS_GEMV_SMEM_KB", 196) * 1024;
  int fit = (budget - 2 * GEMV_ROWS * ks * 2) / (a.K * 2);
  fit = fit > kMaxBatch ? kMaxBatch : fit;
  const bool tma = gemv_tma_enabled() && a.K % 1024 == 0 && a.N / GEMV_ROWS >= 148 && fit >= 2 && bt.nb > 1;
  if (!tma) {
    for (int b = 0; b < bt.nb; ++b)
      if (int rc = gemv_launch(gemv_row_view(a, bt, b), stream)) return rc;
    return DS_OK;
  }
  static const bool xstream_ok = env_int("DS_GEMVB_XSTREAM", 1) != 0;
  // bf16 x: stream it with the weights when that keeps more weight slots in
  // flight than staging it whole (or when it does not fit at all)
  const int slot_b = GEMV_ROWS * ks * 2;
  const int staged_slots = bt.nb <= fit ? (budget - ((bt.nb * a.K * 2 + 127) & ~127)) / slot_b : 0;
  const int stream_slots = budget / (slot_b + bt.nb * ks * 2);
  if (xstream_ok && !a.x_f32 && a.x_bf16 && stream_slots >= 2 && stream_slots > staged_slots) {
    if (ks == 4096) return gemv_batch_launch_ks<4096>(a, bt, stream, true);
    if (ks == 2048) return gemv_batch_launch_ks<2048>(a, bt, stream, true);
    return gemv_batch_launch_ks<1024>(a, bt, stream, true);
  }
  for (int b0 = 0; b0 < bt.nb; b0 += fit) {
    GemvArgs sa = gemv_row_view(a, bt, b0);  // row b0 becomes row 0 of the launch
    GemvBatch sb = bt;
    sb.nb = bt.nb - b0 < fit ? bt.nb - b0 : fit;
    for (int i = 0; i < sb.nb; ++i) {
      sb.pos[i] = bt.pos[b0 + i];
      sb.kv[i] = bt.kv[b0 + i];
    }
    int rc = DS_ERR_INVALID;
    if (ks == 4096) rc = gemv_batch_launch_ks<4096>(sa, sb, stream);
    else if (ks == 2048) rc = gemv_batch_launch_ks<2048>(sa, sb, stream);
    else rc = gemv_batch_launch_ks<1024>(sa, sb, stream);
    if (rc) return rc;
  }
  return DS_OK;
}

__global__ void argmax_finalize_batch_kernel(const unsigned long long* packed, int nb, int32_t* token,
                                             int token_stride, int64_t* token64) {
  const int b = threadIdx.x;
  if (b >= nb) return;
  const int32_t t = (int32_t)(0xFFFFFFFFu - (uint32_t)(packed[b] & 0xFFFFFFFFull));
  if (token) token[(long long)b * token_stride] = t;
  if (token64) token64[b] = t;
}

int argmax_finalize_batch_launch(const unsigned long long* packed, int nb, int32_t* token, int token_stride,
                                 int64_t* token64, cudaStream_t stream) {
  count_launch();
  static PerDevice carve;
  prefer_max_smem_once(argmax_finalize_batch_kernel, carve);
  argmax_finalize_batch_kernel<<<1, 32, 0, stream>>>(packed, nb, token, token_stride, token64);
  return launch_status();
}

int argmax_finalize_launch(const unsigned long long* packed, int32_t* token, int64_t* token64, cudaStream_t stream) {
  count_launch();
  static PerDevice carve;
  prefer_max_smem_once(argmax_finalize_kernel, carve);
  argmax_finalize_kernel<<<1, 1, 0, stream>>>(packed, token, token64);
  return launch_status();
}

// ---------------------------------------------------------------- attention
//
// Item (g, s) = kv head g, keys [s*sk, min(n_keys, (s+1)*sk)).  Keys below
// n_lo come from `lo` (for a reused layer: the producer's export, read in
// place), the rest from `hi` (the consumer cache, where the anchor's own key
// was written by its QKV phase).  With `copy_lo`, every lo row the item loads
// is also stored into `hi` at the same position: the reused-layer KV ingest
// (model.py:590-603) fused into the anchor's read of the same bytes.
//
//   scores  lanes = 16-byte chunks of a key row (D/8 lanes per key), 4 rows in
//           flight per lane, butterfly-reduced over the row's lanes; log2
//           domain, into shared memory [R][sk]
//   softmax warp r: max / exp2 / sum of head r over the item's keys
//   P.V     warp w owns D/4 dims; its lanes are (dim chunk, key stream) and
//           reduce the streams with shuffles; partial (m, l, o) per split
//   merge   the last CTA of the kv head combines the splits (fixed order)

// Items per row (kv head x key split) the split size aims for; DS_ATT_ITEMS
// overrides it for measurements (every path reads the same value, so the
// persistent and per-launch kernels keep the same split of every row).
static int att_target_items() {
  static const int v = [] {
    const char* e = getenv("DS_ATT_ITEMS");
    const int x = e ? atoi(e) : ATT_TARGET_ITEMS;
    return x > 0 ? x : ATT_TARGET_ITEMS;
  }();
  return v;
}
int attn_split_keys(int n_keys, int n_kv_heads, int R) {
  const int splits = (att_target_items() + n_kv_heads - 1) / n_kv_heads;
  int sk = (n_keys + splits - 1) / splits;
  sk = (sk + 31) & ~31;
  if (sk < 32) sk = 32;
  const int cap = 4096 / R;  // an item's scores: R * sk floats <= 16 KB
  return sk > cap ? cap : sk;
}
int attn_max_splits(int n_keys, int n_kv_heads, int R) {
  return (att_target_items() + n_kv_heads - 1) / n_kv_heads + (n_keys + 4096 / R - 1) / (4096 / R) + 1;
}
static int attn_smem_bytes(int R, int sk, int splits) {
  const int scores = R * sk, merge = R * splits + R;
  return 4 * (scores > merge ? scores : merge);
}

DS_DEV const bf16* attn_row(const AttnArgs& a, bool v, int g, int key) {
  const KvAddr& kv = key < a.n_lo ? a.lo : a.hi;
  return (v ? kv.v : kv.k) + kv.off(g, key);
}

// Threads: bring the item's K and V rows into L2 (32-key pieces; never across
// a page or the lo/hi boundary).
DS_DEV void attn_prefetch(const AttnArgs& a, int item, int D) {
  const int g = item / a.splits, s = item - g * a.splits;
  const int k0 = s * a.split_keys;
  const int nk = min(a.split_keys, a.n_keys - k0);
  for (int p = threadIdx.x; p < ((nk + 31) >> 5) * 2; p += blockDim.x) {
    const int key = k0 + (p >> 1) * 32;
    int cnt = min(32, k0 + nk - key);
    if (key < a.n_lo && key + cnt > a.n_lo) cnt = a.n_lo - key;
    if (key < a.n_lo && a.lo_remote) continue;  // peer memory: plain loads only
    prefetch_l2(attn_row(a, p & 1, g, key), (uint32_t)cnt * D * 2);
  }
}

// Softmax of each head over the item's nk scores (log2 domain, in place):
// stat = (max, sum) per head.
// Four of a lane's elements per step (independent loads and exponentials in
// flight); the max is order-free and l still adds the lane's elements in
// ascending order, so the result is the one-element loop's bit for bit.
template <int R>
DS_DEV void attn_softmax(int nk, int sk, float* sc, float* stat) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = warp; r < R; r += ATT_THREADS / 32) {
    float* row = sc + r * sk;
    float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
    for (int i = lane; i < nk; i += 128) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i + 32 * u < nk) m4[u] = fmaxf(m4[u], row[i + 32 * u]);
    }
    float m = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float l = 0.f;
    for (int i = lane; i < nk; i += 128) {
      float e[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) e[u] = i + 32 * u < nk ? exp2f(row[i + 32 * u] - m) : 0.f;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (i + 32 * u < nk) {
          row[i + 32 * u] = e[u];
          l += e[u];
        }
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    if (lane == 0) {
      stat[2 * r] = m;
      stat[2 * r + 1] = l;
    }
  }
}

// P.V partials of one thread (lane = (dim chunk, key stream)): reduce the key
// streams with shuffles, store the item's unnormalised output.
// NR heads from r0 (of the kv head's R), dim chunk `chunk`.
template <int D, int R, int NR = R>
DS_DEV void attn_store_part(const AttnArgs& a, int g, int s, float (*acc)[8], int chunk, int r0 = 0) {
  constexpr int CPW = D / 32;
  const int lane = threadIdx.x & 31, st = lane / CPW;
#pragma unroll
  for (int o = CPW; o < 32; o <<= 1)
#pragma unroll
    for (int r = 0; r < NR; ++r)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[r][e] += __shfl_xor_sync(0xffffffffu, acc[r][e], o);
  if (st == 0) {
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      float4* po =
          reinterpret_cast<float4*>(a.part_o + ((long long)(g * R + r0 + r) * a.splits + s) * D + chunk * 8);
      __stcg(po, make_float4(acc[r][0], acc[r][1], acc[r][2], acc[r][3]));
      __stcg(po + 1, make_float4(acc[r][4], acc[r][5], acc[r][6], acc[r][7]));
    }
  }
}

// The item's (m, l); the last CTA of kv head g merges every split.
// `sync`: a barrier over the CTA's 128 compute threads.
template <int D, int R, typename Sync>
DS_DEV void attn_finish(const AttnArgs& a, int g, int s, float* sc, const float* stat, unsigned int* is_last,
                        Sync sync) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid < R) {
    float* ml = a.part_ml + ((long long)(g * R + tid) * a.splits + s) * 2;
    __stcg(ml, stat[2 * tid]);
    __stcg(ml + 1, stat[2 * tid + 1]);
  }
  // ---- the last CTA of this kv head merges every split (threadfence reduction)
  __threadfence();
  sync();
  if (tid == 0) *is_last = (atomicAdd(a.counters + g, 1u) == (unsigned)a.splits - 1);
  sync();
  if (*is_last) {
    __threadfence();
    float* wts = sc;  // [R][splits] then den[R]
    float* den = wts + R * a.splits;
    for (int r = warp; r < R; r += ATT_THREADS / 32) {
      const float* ml = a.part_ml + (long long)(g * R + r) * a.splits * 2;
      float M = -INFINITY;
      for (int s2 = lane; s2 < a.splits; s2 += 32) M = fmaxf(M, __ldcg(ml + 2 * s2));
#pragma unroll
      for (int off = 16; off; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
      float dn = 0.f;
      for (int s2 = lane; s2 < a.splits; s2 += 32) {
        const float w = exp2f(__ldcg(ml + 2 * s2) - M);
        wts[r * a.splits + s2] = w;
        dn = __fmaf_rn(w, __ldcg(ml + 2 * s2 + 1), dn);
      }
#pragma unroll
      for (int off = 16; off; off >>= 1) dn += __shfl_xor_sync(0xffffffffu, dn, off);
      if (lane == 0) den[r] = dn;
    }
    sync();
    // R*D outputs, R*D/128 per thread, each over every split: the loads of
    // 8 splits x all of a thread's outputs are in flight together
    constexpr int PER = (R * D + ATT_THREADS - 1) / ATT_THREADS;
    float num[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) num[q] = 0.f;
    for (int s0 = 0; s0 < a.splits; s0 += 8) {
      float v[PER][8];
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        const int idx = tid + q * ATT_THREADS;
        const int r = idx / D, dd = idx % D;
        const float* po = a.part_o + (long long)(g * R + r) * a.splits * D + dd;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          v[q][u] = (idx < R * D && s0 + u < a.splits) ? __ldcg(po + (long long)(s0 + u) * D) : 0.f;
      }
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        const int idx = tid + q * ATT_THREADS;
        const int r = idx < R * D ? idx / D : 0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (s0 + u < a.splits) num[q] = fmaf(wts[r * a.splits + s0 + u], v[q][u], num[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int idx = tid + q * ATT_THREADS;
      if (idx < R * D) {
        const int r = idx / D, dd = idx % D;
        a.out[(long long)(g * R + r) * D + dd] = __float2bfloat16_rn(num[q] / den[r]);
      }
    }
    if (tid == 0) a.counters[g] = 0u;
  }
  sync();  // shared memory reused by the next item
}

// DEEP: rows in flight per lane doubled (the stand-alone kernel, no register
// cap); batching only -- every score and every P.V accumulation keeps its order.
template <int D, int R, bool DEEP = false>
DS_DEV void attn_item(const AttnArgs& a, int item, float* sc, float* stat, unsigned int* is_last) {
  constexpr int LPK = D / 8;       // lanes per key row
  constexpr int KPW = 32 / LPK;    // key rows per warp load
  constexpr int U = (R >= 8 ? 2 : 4) * (DEEP ? 2 : 1);   // rows in flight per lane (scores)
  constexpr int CPW = LPK / 4;     // dim chunks per warp (P.V)
  constexpr int NS = 32 / CPW;     // key streams per warp (P.V)
  constexpr int U2 = (R >= 8 ? 1 : 4) * (DEEP ? 2 : 1);  // rows in flight per lane (P.V)
  const int g = item / a.splits, s = item - g * a.splits;
  const int k0 = s * a.split_keys;
  const int nk = min(a.split_keys, a.n_keys - k0);
  const int sk = a.split_keys;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---- scores
  {
    const int c = lane % LPK, kk = lane / LPK;
    uint4 qv[R];
#pragma unroll
    for (int r = 0; r < R; ++r) qv[r] = ld_cg16(a.q + (long long)(g * R + r) * D + c * 8);
    for (int base = warp * KPW * U; base < nk; base += 4 * KPW * U) {
      uint4 kv[U];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int key = base + j * KPW + kk;
        kv[j] = make_uint4(0u, 0u, 0u, 0u);
        if (key < nk) kv[j] = ld_cg16(attn_row(a, false, g, k0 + key) + c * 8);
      }
      if (a.copy_lo) {  // after every load of the step is in flight
#pragma unroll
        for (int j = 0; j < U; ++j) {
          const int pos = k0 + base + j * KPW + kk;
          if (base + j * KPW + kk < nk && pos < a.n_lo)
            *reinterpret_cast<uint4*>(a.hi.k + a.hi.off(g, pos) + c * 8) = kv[j];
        }
      }
      float p[U * R];  // value (j, r) at j * R + r
#pragma unroll
      for (int j = 0; j < U; ++j)
#pragma unroll
        for (int r = 0; r < R; ++r) p[j * R + r] = dot8(kv[j], qv[r]);
      const int vb = rs_sum<U * R, LPK>(p, lane);
      constexpr int VC = (U * R) / LPK > 0 ? (U * R) / LPK : 1;
#pragma unroll
      for (int i = 0; i < VC; ++i) {
        const int idx = vb + i, j = idx / R, r = idx - j * R;
        const int key = base + j * KPW + kk;
        if (key < nk) sc[r * sk + key] = p[i] * a.scale_log2;
      }
    }
  }
  __syncthreads();
  attn_softmax<R>(nk, sk, sc, stat);
  __syncthreads();
  // ---- P.V: warp w owns dim chunks [w*CPW, (w+1)*CPW)
  {
    const int cw = lane % CPW, st = lane / CPW;
    const int chunk = warp * CPW + cw;
    float acc[R][8];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[r][e] = 0.f;
    for (int i = st; i < nk; i += NS * U2) {
      uint4 vv[U2];
#pragma unroll
      for (int j = 0; j < U2; ++j) {
        const int key = i + j * NS;
        vv[j] = make_uint4(0u, 0u, 0u, 0u);
        if (key < nk) vv[j] = ld_cg16(attn_row(a, true, g, k0 + key) + chunk * 8);
      }
      if (a.copy_lo) {
#pragma unroll
        for (int j = 0; j < U2; ++j) {
          const int key = i + j * NS, pos = k0 + key;
          if (key < nk && pos < a.n_lo) *reinterpret_cast<uint4*>(a.hi.v + a.hi.off(g, pos) + chunk * 8) = vv[j];
        }
      }
#pragma unroll
      for (int j = 0; j < U2; ++j) {
        const int key = i + j * NS;
        if (key < nk) {
          const float2 v0 = unpack_bf16x2(vv[j].x), v1 = unpack_bf16x2(vv[j].y);
          const float2 v2 = unpack_bf16x2(vv[j].z), v3 = unpack_bf16x2(vv[j].w);
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const float pr = sc[r * sk + key];
            acc[r][0] = fmaf(pr, v0.x, acc[r][0]);
            acc[r][1] = fmaf(pr, v0.y, acc[r][1]);
            acc[r][2] = fmaf(pr, v1.x, acc[r][2]);
            acc[r][3] = fmaf(pr, v1.y, acc[r][3]);
            acc[r][4] = fmaf(pr, v2.x, acc[r][4]);
            acc[r][5] = fmaf(pr, v2.y, acc[r][5]);
            acc[r][6] = fmaf(pr, v3.x, acc[r][6]);
            acc[r][7] = fmaf(pr, v3.y, acc[r][7]);
          }
        }
      }
    }
    attn_store_part<D, R>(a, g, s, acc, chunk);
  }
  attn_finish<D, R>(a, g, s, sc, stat, is_last, [] { __syncthreads(); });
}

template <int D, int R>
__global__ void __launch_bounds__(ATT_THREADS) attn_decode_kernel(AttnArgs a) {
  extern __shared__ __align__(16) float sc[];
  __shared__ float stat[2 * R];
  __shared__ unsigned int is_last;
  // the cache rows (except the anchor's own key, written by the predecessor)
  // are in HBM already: stream them toward L2, then wait for the predecessor
  attn_prefetch(a, blockIdx.x, D);
  pdl_trigger();
  pdl_wait();
  attn_item<D, R, true>(a, blockIdx.x, sc, stat, &is_last);
}

// ---------------------------------------------------------------- TMA-staged stand-alone attention
//
// The per-launch kernel's memory side as a ring: a producer warp bulk-copies
// the item's K rows, then its V rows, in 32-key pieces (one copy per piece and
// source; never across a page or the lo/hi boundary) into ATT_SLOTS shared
// slots, so the whole item streams from the first cycle -- every row except
// those the predecessor writes (keys >= n_lo, the anchor's own) is issued
// before the PDL wait.  The 4 compute warps run attn_item's arithmetic on the
// staged rows: each key's score from the same LPK lanes and butterfly, each
// lane's P.V keys in the same ascending order, the same softmax and merge --
// so results are the register kernel's (and the persistent kernel's) bit for
// bit.  With copy_lo, one thread bulk-stores each staged lo piece into hi (the
// fused KV ingest) before the slot is released.
// Reading lo rows before the PDL wait requires them complete before the
// kernel's own predecessor started, which every caller guarantees: lo is the
// sender's export (an input of the call), or cache rows written before the
// anchor chain began (anchor_pass starts with a memset, a full stream
// barrier) or by a recompute the chain waited on with an event before the
// layer's QKV GEMV / this kernel launched.
constexpr int ATT_PIECE = 32;  // keys per ring piece (pages are 64-key aligned)
// P.V by key streams across warps (1, default) or attn_item's lane layout (0: A/B)
#ifndef DS_ATT_PV_STREAMS
#define DS_ATT_PV_STREAMS 1
#endif
constexpr int ATT_SLOTS_MAX = 16;
constexpr int ATT_TW = 8;                         // compute warps
constexpr int ATT_TTHREADS = ATT_TW * 32 + 32;  // + producer warp

DS_DEV void named_sync_compute() { asm volatile("bar.sync 2, %0;" ::"n"(ATT_TW * 32) : "memory"); }

#if DS_ATT_STAMPS
// Debug timeline (build with DS_NVCC_EXTRA=-DDS_ATT_STAMPS=1): a few CTAs of
// one launch print global-timer stamps of their phases.
__device__ unsigned int g_att_launch;
#define ATT_STAMP(i) \
  do {                \
    if (tid == 0) st_ns[i] = global_ns(); \
  } while (0)
#else
#define ATT_STAMP(i) \
  do {                \
  } while (0)
#endif

// attn_finish for the 8-warp stand-alone kernel: the same (m, l) store,
// arrival count and merge arithmetic (same max, same lane-strided sums, each
// output accumulated over the splits in ascending order).  The merging CTA
// stages the kv head's partial outputs in the (idle) ring with one bulk copy
// and its (m, l) with one load per thread, so the merge costs one round trip
// instead of one per group of splits.
template <int D, int R>
DS_DEV void attn_finish_wide(const AttnArgs& a, int g, int s, float* sc, const float* stat, unsigned int* is_last,
                             uint8_t* stage, int stage_bytes, uint64_t* bar, unsigned long long* st_ns) {
  constexpr int NT = ATT_TW * 32;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid < R) {
    float* ml = a.part_ml + ((long long)(g * R + tid) * a.splits + s) * 2;
    __stcg(ml, stat[2 * tid]);
    __stcg(ml + 1, stat[2 * tid + 1]);
  }
  // release: the CTA barrier orders every thread's part_o / (m, l) stores
  // before thread 0's gpu-scope fence and arrival; the last arrival's thread 0
  // fences again (acquire) before the barrier that releases the merge's
  // reads (the grid-barrier pattern: one thread waits on each fence)
  named_sync_compute();
  if (tid == 0) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    const bool last = atomicAdd(a.counters + g, 1u) == (unsigned)a.splits - 1;
    if (last) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    *is_last = last;
  }
  named_sync_compute();
  ATT_STAMP(7);
  if (!*is_last) return;
  const int n_ml = R * a.splits * 2;
  const uint32_t o_bytes = (uint32_t)R * a.splits * D * 4;
  const bool staged = (int)o_bytes + 4 * n_ml <= stage_bytes;
  float* po_s = reinterpret_cast<float*>(stage);
  float* ml_s = po_s + (size_t)R * a.splits * D;
  const float* po_g = a.part_o + (long long)g * R * a.splits * D;
  const float* ml_g = a.part_ml + (long long)g * R * a.splits * 2;
  if (staged) {
    if (tid == 0) {
      asm volatile("fence.proxy.async.global;" ::: "memory");  // the other CTAs' generic stores, acquired above
      mbar_expect_tx(bar, o_bytes);
      bulk_g2s(po_s, po_g, o_bytes, bar);
    }
    for (int i = tid; i < n_ml; i += NT) ml_s[i] = __ldcg(ml_g + i);
    named_sync_compute();
  }
  const float* ml_src = staged ? ml_s : ml_g;
  float* wts = sc;  // [R][splits] then den[R]
  float* den = wts + R * a.splits;
  if (warp < ATT_THREADS / 32) {  // warps 0..3, as attn_finish
    for (int r = warp; r < R; r += ATT_THREADS / 32) {
      const float* ml = ml_src + (long long)r * a.splits * 2;
      float M = -INFINITY;
      for (int s2 = lane; s2 < a.splits; s2 += 32) M = fmaxf(M, staged ? ml[2 * s2] : __ldcg(ml + 2 * s2));
#pragma unroll
      for (int off = 16; off; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
      float dn = 0.f;
      for (int s2 = lane; s2 < a.splits; s2 += 32) {
        const float w = exp2f((staged ? ml[2 * s2] : __ldcg(ml + 2 * s2)) - M);
        wts[r * a.splits + s2] = w;
        dn = __fmaf_rn(w, staged ? ml[2 * s2 + 1] : __ldcg(ml + 2 * s2 + 1), dn);
      }
#pragma unroll
      for (int off = 16; off; off >>= 1) dn += __shfl_xor_sync(0xffffffffu, dn, off);
      if (lane == 0) den[r] = dn;
    }
  }
  if (staged) mbar_wait(bar, 0);
  named_sync_compute();  // wts / den written, partial outputs landed
  ATT_STAMP(8);
  // each output over the splits in ascending order (attn_finish's chain); a
  // thread's PER outputs advance together (independent chains), the staged
  // form reads shared memory explicitly and keeps 8 splits' loads ahead
  constexpr int PER = (R * D + NT - 1) / NT;
  float num[PER];
  int rq[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    num[q] = 0.f;
    rq[q] = min((tid + q * NT) / D, R - 1);
  }
  const int sp = a.splits;
  if (staged) {
    uint32_t pa[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int idx = min(tid + q * NT, R * D - 1);
      pa[q] = smem_u32(po_s + (long long)rq[q] * sp * D + idx % D);
    }
    int s2 = 0;
    for (; s2 + 8 <= sp; s2 += 8) {
      float v[PER][8];
#pragma unroll
      for (int q = 0; q < PER; ++q)
#pragma unroll
        for (int u = 0; u < 8; ++u)
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v[q][u]) : "r"(pa[q] + (uint32_t)((s2 + u) * D * 4)));
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int q = 0; q < PER; ++q) num[q] = fmaf(wts[rq[q] * sp + s2 + u], v[q][u], num[q]);
    }
    for (; s2 < sp; ++s2)
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        float v;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(pa[q] + (uint32_t)(s2 * D * 4)));
        num[q] = fmaf(wts[rq[q] * sp + s2], v, num[q]);
      }
  } else {
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int idx = min(tid + q * NT, R * D - 1);
      const float* po = po_g + (long long)rq[q] * sp * D + idx % D;
      for (int s2 = 0; s2 < sp; ++s2) num[q] = fmaf(wts[rq[q] * sp + s2], __ldcg(po + (long long)s2 * D), num[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int idx = tid + q * NT;
    if (idx < R * D) a.out[(long long)(g * R) * D + idx] = __float2bfloat16_rn(num[q] / den[rq[q]]);
  }
  if (tid == 0) a.counters[g] = 0u;
}


// One (kv head, split) item of row `a` (the kernel body; `item` replaces item).
template <int D, int R>
DS_DEV void attn_tma_item(const AttnArgs& a, int item, int slots, int prefetch) {
#if DS_ATT_STAMPS
  unsigned long long st_ns[11] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long ck0 = 0, ck1 = 0;  // SM cycles over the P.V phase (clock rate check)
#else
  unsigned long long* st_ns = nullptr;
#endif
  constexpr int ROWB = D * 2, PIECE_B = ATT_PIECE * ROWB;
  // scores: each warp takes ATT_PIECE / ATT_TW keys of a piece, LPK lanes per key
  constexpr int LPK = D / 8, KPW = 32 / LPK, UK = (ATT_PIECE / ATT_TW) / KPW;
  static_assert(UK >= 1, "piece too small for the warp count");
  // P.V: warps (w & 3) own dim chunks like attn_item's 4 warps; warps >= 4
  // take the upper half of the heads (R >= 2), so every accumulator sums the
  // same keys in the same order
  constexpr int CPW = LPK / 4, NS = 32 / CPW;
  [[maybe_unused]] constexpr int UV = ATT_PIECE / NS;
  [[maybe_unused]] constexpr int HR = R >= 2 ? R / 2 : 1;
  constexpr int RP = R >= 2 ? R / 2 : 1;  // head pairs (scores, packed)
  extern __shared__ __align__(128) uint8_t smem_dyn[];
  uint8_t* ring = smem_dyn;
  float* sc = reinterpret_cast<float*>(smem_dyn + slots * PIECE_B);
  __shared__ __align__(8) uint64_t full[ATT_SLOTS_MAX], empty[ATT_SLOTS_MAX], merge_bar;
  __shared__ float stat[2 * R];
  __shared__ unsigned int is_last;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = item / a.splits, s = item - g * a.splits;
  const int k0 = s * a.split_keys;
  const int nk = min(a.split_keys, a.n_keys - k0);
  const int sk = a.split_keys;
  const int np = (nk + ATT_PIECE - 1) / ATT_PIECE;
  if (tid == ATT_TW * 32) {
    for (int i = 0; i < slots; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], ATT_TW);
    }
    mbar_init(&merge_bar, 1);
    fence_mbar_init();
  }
  // optionally pull the whole item toward L2 first (the ring then reads L2)
  if (prefetch & 1) attn_prefetch(a, item, D);
  // timing experiments (results are wrong): data movement only, or no scores / no P.V math / no softmax (bit 4)
  const bool no_scores = prefetch & 6, no_pv = prefetch & 10, no_softmax = prefetch & 16;
  __syncthreads();
  pdl_trigger();
  if (warp == ATT_TW) {
    if (lane == 0) {
      bool waited = false;
      int slot = 0;
      uint32_t phase = 0;
      for (int p = 0; p < 2 * np; ++p) {
        const bool v = p >= np;
        const int a0 = k0 + (v ? p - np : p) * ATT_PIECE;
        const int a1 = a0 + min(ATT_PIECE, k0 + nk - a0);
        mbar_wait(&empty[slot], phase ^ 1);
        mbar_expect_tx(&full[slot], (uint32_t)(a1 - a0) * ROWB);
        uint8_t* dst = ring + slot * PIECE_B;
        const int lo_end = min(a1, a.n_lo), hi0 = max(a0, a.n_lo);
        if (lo_end > a0) bulk_g2s(dst, attn_row(a, v, g, a0), (uint32_t)(lo_end - a0) * ROWB, &full[slot]);
        if (a1 > hi0) {  // rows the predecessor writes
          if (!waited) {
            pdl_wait();
            waited = true;
          }
          bulk_g2s(dst + (hi0 - a0) * ROWB, attn_row(a, v, g, hi0), (uint32_t)(a1 - hi0) * ROWB, &full[slot]);
        }
        if (++slot == slots) {
          slot = 0;
          phase ^= 1;
        }
      }
    }
    return;
  }
  ATT_STAMP(0);
  pdl_wait();
  ATT_STAMP(1);
  int slot = 0;
  uint32_t phase = 0;
  // one thread stores a staged lo piece into hi (fused ingest); the slot is
  // released only after the store has read it
  auto ingest = [&](bool v, int a0, int cnt, const uint8_t* src) {
    if (a.copy_lo && tid == 0) {
      const int lo_cnt = min(a0 + cnt, a.n_lo) - a0;
      if (lo_cnt > 0) {
        bulk_s2g((v ? a.hi.v : a.hi.k) + a.hi.off(g, a0), src, (uint32_t)lo_cnt * ROWB);
        bulk_commit();
        bulk_wait_read<0>();
      }
    }
  };
  auto release = [&]() {
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
    if (++slot == slots) {
      slot = 0;
      phase ^= 1;
    }
  };
  // ---- scores (dot8's order per key and head; head pairs on packed lanes)
  {
    const int c = lane % LPK, kk = lane / LPK;
    float2 qf[RP][8];  // (head 2i, head 2i+1) per element; R == 1: (head 0, head 0)
#pragma unroll
    for (int i = 0; i < RP; ++i) {
      const int r0 = R >= 2 ? 2 * i : 0, r1 = R >= 2 ? 2 * i + 1 : 0;
      const uint4 q0 = ld_cg16(a.q + (long long)(g * R + r0) * D + c * 8);
      const uint4 q1 = ld_cg16(a.q + (long long)(g * R + r1) * D + c * 8);
      const uint32_t w0[4] = {q0.x, q0.y, q0.z, q0.w}, w1[4] = {q1.x, q1.y, q1.z, q1.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f0 = unpack_bf16x2(w0[k]), f1 = unpack_bf16x2(w1[k]);
        qf[i][2 * k] = make_float2(f0.x, f1.x);
        qf[i][2 * k + 1] = make_float2(f0.y, f1.y);
      }
    }
    for (int p = 0; p < np; ++p) {
      const int pk0 = p * ATT_PIECE, cnt = min(ATT_PIECE, nk - pk0);
      mbar_wait(&full[slot], phase);
      if (p == 0) ATT_STAMP(2);
      if (p == np - 1) ATT_STAMP(9);
      const uint8_t* src = ring + slot * PIECE_B;
      if (no_scores) {
        release();
        continue;
      }
      float2 pr[UK][RP];
#pragma unroll
      for (int j = 0; j < UK; ++j) {
        const int key = warp * (ATT_PIECE / ATT_TW) + j * KPW + kk;
        const uint4 kv =
            key < cnt ? *reinterpret_cast<const uint4*>(src + key * ROWB + c * 16) : make_uint4(0u, 0u, 0u, 0u);
        const uint32_t kw[4] = {kv.x, kv.y, kv.z, kv.w};
        float kf[8];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f = unpack_bf16x2(kw[k]);
          kf[2 * k] = f.x;
          kf[2 * k + 1] = f.y;
        }
#pragma unroll
        for (int i = 0; i < RP; ++i) {
          float2 acc = fmul2(make_float2(kf[0], kf[0]), qf[i][0]);
#pragma unroll
          for (int e = 1; e < 8; ++e) acc = ffma2(make_float2(kf[e], kf[e]), qf[i][e], acc);
          pr[j][i] = acc;
        }
      }
      float pv[UK * R];  // value (j, r) at j * R + r
#pragma unroll
      for (int j = 0; j < UK; ++j)
#pragma unroll
        for (int r = 0; r < R; ++r) pv[j * R + r] = (r & 1) ? pr[j][r >> 1].y : pr[j][r >> 1].x;
      const int vb = rs_sum<UK * R, LPK>(pv, lane);
      constexpr int VC = (UK * R) / LPK > 0 ? (UK * R) / LPK : 1;
#pragma unroll
      for (int i = 0; i < VC; ++i) {
        const int idx = vb + i, j = idx / R, r = idx - j * R;
        const int key = warp * (ATT_PIECE / ATT_TW) + j * KPW + kk;
        if (key < cnt) sc[r * sk + pk0 + key] = pv[i] * a.scale_log2;
      }
      ingest(false, k0 + pk0, cnt, src);
      release();
    }
  }
  named_sync_compute();
  ATT_STAMP(3);
  if (warp < ATT_THREADS / 32 && !no_softmax) attn_softmax<R>(nk, sk, sc, stat);
  named_sync_compute();
  ATT_STAMP(4);
#if DS_ATT_STAMPS
  if (tid == 0) ck0 = clock64();
#endif
#if DS_ATT_PV_STREAMS
  // ---- P.V, key streams across warps: warp w runs streams w, w + 8, ... (keys
  // st, st + NS, ... of attn_item's lane (chunk, st)), each lane D/32
  // contiguous dims of every head -- conflict-free row reads, broadcast P.
  // The streams' partials then meet in shared memory in the xor-butterfly's
  // tree ((s0 + s1) + (s2 + s3)) + ..., so every output is attn_item's bit for bit.
  {
    constexpr int DPL = D / 32, SPW = NS / ATT_TW;
    static_assert(NS % ATT_TW == 0, "streams per warp");
    float2 acc[SPW][R][DPL / 2];
#pragma unroll
    for (int q = 0; q < SPW; ++q)
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int e = 0; e < DPL / 2; ++e) acc[q][r][e] = make_float2(0.f, 0.f);
    for (int p = 0; p < np; ++p) {
      const int pk0 = p * ATT_PIECE, cnt = min(ATT_PIECE, nk - pk0);
      mbar_wait(&full[slot], phase);
      if (p == np - 1) ATT_STAMP(10);
      const uint8_t* src = ring + slot * PIECE_B;
      // a full piece loads every key's V slice and P values before the first
      // FMA (no per-key guards); the last piece of a split keeps the guards
      auto piece = [&](auto full_tag) {
        constexpr bool FULL = decltype(full_tag)::value;
        constexpr int KJ = ATT_PIECE / NS;
        constexpr int RP = R <= 4 ? R : 1;  // P values held ahead (R = 8 reads them at the FMA: registers)
        float2 vf[SPW][KJ][DPL / 2];
        float pp[SPW][KJ][RP];
#pragma unroll
        for (int q = 0; q < SPW; ++q)
#pragma unroll
          for (int j = 0; j < KJ; ++j) {
            const int key = warp + q * ATT_TW + j * NS;
            if (FULL || key < cnt) {
              if constexpr (DPL == 4) {
                const uint2 vv = *reinterpret_cast<const uint2*>(src + key * ROWB + lane * 8);
                vf[q][j][0] = unpack_bf16x2(vv.x);
                vf[q][j][1] = unpack_bf16x2(vv.y);
              } else {
                vf[q][j][0] = unpack_bf16x2(*reinterpret_cast<const uint32_t*>(src + key * ROWB + lane * 4));
              }
              if constexpr (R <= 4)
#pragma unroll
                for (int r = 0; r < R; ++r) pp[q][j][r] = sc[r * sk + pk0 + key];
            }
          }
#pragma unroll
        for (int q = 0; q < SPW; ++q)
#pragma unroll
          for (int j = 0; j < KJ; ++j) {
            const int key = warp + q * ATT_TW + j * NS;
            if (FULL || key < cnt) {
#pragma unroll
              for (int r = 0; r < R; ++r) {
                const float pr = R <= 4 ? pp[q][j][r < RP ? r : 0] : sc[r * sk + pk0 + key];
                const float2 p2 = make_float2(pr, pr);
#pragma unroll
                for (int e = 0; e < DPL / 2; ++e) acc[q][r][e] = ffma2(p2, vf[q][j][e], acc[q][r][e]);
              }
            }
          }
      };
      if (!no_pv) {
        if (cnt == ATT_PIECE)
          piece(std::true_type{});
        else
          piece(std::false_type{});
      }
      ingest(true, k0 + pk0, cnt, src);
      release();
    }
    named_sync_compute();  // every warp is done with the ring: it stages the stream partials
    float* part = reinterpret_cast<float*>(ring);  // [NS][R][D]
#pragma unroll
    for (int q = 0; q < SPW; ++q)
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int e = 0; e < DPL / 2; ++e)
          *reinterpret_cast<float2*>(part + ((warp + q * ATT_TW) * R + r) * D + lane * DPL + 2 * e) = acc[q][r][e];
    named_sync_compute();
    constexpr int NT = ATT_TW * 32;
    for (int idx = tid; idx < R * D; idx += NT) {
      float t[NS];
#pragma unroll
      for (int q = 0; q < NS; ++q) t[q] = part[q * R * D + idx];
#pragma unroll
      for (int w = 1; w < NS; w <<= 1)
#pragma unroll
        for (int q = 0; q < NS; q += 2 * w) t[q] += t[q + w];
      const int r = idx / D, dd = idx - r * D;
      __stcg(a.part_o + ((long long)(g * R + r) * a.splits + s) * D + dd, t[0]);
    }
  }
#else
  // ---- P.V
  {
    const int cw = lane % CPW, st = lane / CPW;
    const int chunk = (warp & 3) * CPW + cw;
    const int r0 = (warp >> 2) * HR;
    const bool active = R >= 2 || warp < 4;
    float2 acc[HR][4];
#pragma unroll
    for (int r = 0; r < HR; ++r)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[r][e] = make_float2(0.f, 0.f);
    for (int p = 0; p < np; ++p) {
      const int pk0 = p * ATT_PIECE, cnt = min(ATT_PIECE, nk - pk0);
      mbar_wait(&full[slot], phase);
      if (p == np - 1) ATT_STAMP(10);
      const uint8_t* src = ring + slot * PIECE_B;
      if (active && !no_pv) {
#pragma unroll
        for (int j = 0; j < UV; ++j) {
          const int key = st + j * NS;
          if (key < cnt) {
            const uint4 vv = *reinterpret_cast<const uint4*>(src + key * ROWB + chunk * 16);
            const float2 v0 = unpack_bf16x2(vv.x), v1 = unpack_bf16x2(vv.y);
            const float2 v2 = unpack_bf16x2(vv.z), v3 = unpack_bf16x2(vv.w);
#pragma unroll
            for (int r = 0; r < HR; ++r) {
              const float pp = sc[(r0 + r) * sk + pk0 + key];
              const float2 p2 = make_float2(pp, pp);
              acc[r][0] = ffma2(p2, v0, acc[r][0]);
              acc[r][1] = ffma2(p2, v1, acc[r][1]);
              acc[r][2] = ffma2(p2, v2, acc[r][2]);
              acc[r][3] = ffma2(p2, v3, acc[r][3]);
            }
          }
        }
      }
      ingest(true, k0 + pk0, cnt, src);
      release();
    }
    if (active) {
      float accs[HR][8];
#pragma unroll
      for (int r = 0; r < HR; ++r)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          accs[r][2 * e] = acc[r][e].x;
          accs[r][2 * e + 1] = acc[r][e].y;
        }
      attn_store_part<D, R, HR>(a, g, s, accs, chunk, r0);
    }
  }
#endif
  ATT_STAMP(5);
#if DS_ATT_STAMPS
  if (tid == 0) ck1 = clock64();
#endif
  // every piece is consumed: the ring is free to stage the merge
  attn_finish_wide<D, R>(a, g, s, sc, stat, &is_last, ring, slots * PIECE_B, &merge_bar, st_ns);
  if (a.copy_lo && tid == 0) bulk_wait<0>();  // the ingest stores land before the grid completes
  ATT_STAMP(6);
#if DS_ATT_STAMPS
  if (tid == 0) {
    const unsigned int launch = *(volatile unsigned int*)&g_att_launch;
    if (launch == 100 && (s == 0 || s == a.splits - 1 || is_last))
      printf("ATT %d %d %d last=%d %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu pv_cycles=%lld\n", launch, g, s,
             (int)is_last, st_ns[0], st_ns[1], st_ns[2], st_ns[3], st_ns[4], st_ns[5], st_ns[6], st_ns[7], st_ns[8],
             st_ns[9], st_ns[10], ck1 - ck0);
    if (item == 0) atomicAdd(&g_att_launch, 1u);
  }
#endif
}

template <int D, int R>
__global__ void __launch_bounds__(ATT_TTHREADS, 2) attn_decode_tma_kernel(const __grid_constant__ AttnArgs a, int slots,
                                                                          int prefetch) {
  attn_tma_item<D, R>(a, blockIdx.x, slots, prefetch);
}

// Batched rows: CTA x serves item x - start[b] of row b (start[] = running
// item counts).  Each row keeps its own splits, scratch and merge counters.
struct AttnBatch {
  AttnArgs r[kMaxBatch];
  int start[kMaxBatch + 1];
  int nb;
};
template <int D, int R>
__global__ void __launch_bounds__(ATT_TTHREADS, 2) attn_batch_tma_kernel(const __grid_constant__ AttnBatch ab, int slots,
                                                                         int prefetch) {
  int b = 0;
  while (b + 1 < ab.nb && (int)blockIdx.x >= ab.start[b + 1]) ++b;
  attn_tma_item<D, R>(ab.r[b], (int)blockIdx.x - ab.start[b], slots, prefetch);
}

// Ring slots: DS_ATT_SLOTS clamped to [2, ATT_SLOTS_MAX] and, with the
// stream-per-warp P.V, to what holds the streams' partials (NS x R x D floats).
template <int D, int R>
static int att_slots(int want) {
  int lo = 2;
#if DS_ATT_PV_STREAMS
  const int need = (32 * 32 / D) * R * D * 4, piece = ATT_PIECE * D * 2;
  lo = (need + piece - 1) / piece > lo ? (need + piece - 1) / piece : lo;
#endif
  return want < lo ? lo : (want > ATT_SLOTS_MAX ? ATT_SLOTS_MAX : want);
}

template <int D, int R>
static cudaError_t attn_tma_launch_t(const AttnArgs& a, int smem, cudaStream_t stream) {
  // ring slots and L2 prefetch (DS_ATT_SLOTS, DS_ATT_PREFETCH: experiments)
  static const int slots_env = env_int("DS_ATT_SLOTS", 12);
  static const int prefetch = env_int("DS_ATT_PREFETCH", 0);  // bit 0 L2 prefetch; bits 1-4 timing experiments
  const int slots = att_slots<D, R>(slots_env);
  auto kern = attn_decode_tma_kernel<D, R>;
  static PerDevice attr;
  const int total = slots * ATT_PIECE * D * 2 + smem;
  if (cudaError_t e = ensure_smem_attr(kern, total, attr)) return e;
  return launch_pdl(kern, dim3(a.n_kv_heads * a.splits), dim3(ATT_TTHREADS), total, stream, a, slots, prefetch);
}

// DS_ATTN_TMA=0: the register-streaming kernel (A/B).
static bool attn_tma_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DS_ATTN_TMA");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

template <int D, int R>
static cudaError_t attn_launch_t(const AttnArgs& a, int smem, cudaStream_t stream) {
  auto kern = attn_decode_kernel<D, R>;
  static PerDevice carve;
  prefer_max_smem_once(kern, carve);
  return launch_pdl(kern, dim3(a.n_kv_heads * a.splits), dim3(ATT_THREADS), smem, stream, a);
}

int decode_attention_launch(AttnArgs a, int head_dim, cudaStream_t stream) {
  const int R = a.n_heads / a.n_kv_heads;
  if ((R != 1 && R != 2 && R != 4 && R != 8) || (head_dim != 64 && head_dim != 128) || a.n_keys < 1)
    return DS_ERR_INVALID;
  a.split_keys = attn_split_keys(a.n_keys, a.n_kv_heads, R);
  a.splits = (a.n_keys + a.split_keys - 1) / a.split_keys;
  a.scale_log2 = (float)(1.4426950408889634 / sqrt((double)head_dim));
  const int smem = attn_smem_bytes(R, a.split_keys, a.splits);
  count_launch();
  cudaError_t e = cudaErrorInvalidValue;
  const bool tma = attn_tma_enabled();
#define DS_ATT_CASE(DD, RR) \
  if (head_dim == DD && R == RR) e = tma ? attn_tma_launch_t<DD, RR>(a, smem, stream) : attn_launch_t<DD, RR>(a, smem, stream);
  DS_ATT_CASE(128, 1) DS_ATT_CASE(128, 2) DS_ATT_CASE(128, 4) DS_ATT_CASE(128, 8)
  DS_ATT_CASE(64, 1) DS_ATT_CASE(64, 2) DS_ATT_CASE(64, 4) DS_ATT_CASE(64, 8)
#undef DS_ATT_CASE
  return launch_status(e);
}

template <int D, int R>
static cudaError_t attn_batch_launch_t(const AttnBatch& ab, int smem, cudaStream_t stream) {
  static const int slots_env = env_int("DS_ATT_SLOTS", 12);
  static const int prefetch = env_int("DS_ATT_PREFETCH", 0);
  const int slots = att_slots<D, R>(slots_env);
  auto kern = attn_batch_tma_kernel<D, R>;
  static PerDevice attr;
  const int total = slots * ATT_PIECE * D * 2 + smem;
  if (cudaError_t e = ensure_smem_attr(kern, total, attr)) return e;
  return launch_pdl(kern, dim3(ab.start[ab.nb]), dim3(ATT_TTHREADS), total, stream, ab, slots, prefetch);
}

int decode_attention_batch_launch(const AttnArgs* rows, int nb, int head_dim, cudaStream_t stream) {
  if (nb < 1 || nb > kMaxBatch) return DS_ERR_INVALID;
  const int R = rows[0].n_heads / rows[0].n_kv_heads;
  if ((R != 1 && R != 2 && R != 4 && R != 8) || (head_dim != 64 && head_dim != 128)) return DS_ERR_INVALID;
  if (nb == 1 || !attn_tma_enabled()) {
    for (int b = 0; b < nb; ++b)
      if (int rc = decode_attention_launch(rows[b], head_dim, stream)) return rc;
    return DS_OK;
  }
  static thread_local AttnBatch ab;
  memset(&ab, 0, sizeof(ab));
  ab.nb = nb;
  int smem = 0;
  for (int b = 0; b < nb; ++b) {
    AttnArgs a = rows[b];
    if (a.n_keys < 1 || a.n_heads != rows[0].n_heads || a.n_kv_heads != rows[0].n_kv_heads) return DS_ERR_INVALID;
    a.split_keys = attn_split_keys(a.n_keys, a.n_kv_heads, R);
    a.splits = (a.n_keys + a.split_keys - 1) / a.split_keys;
    a.scale_log2 = (float)(1.4426950408889634 / sqrt((double)head_dim));
    const int sm = attn_smem_bytes(R, a.split_keys, a.splits);
    smem = sm > smem ? sm : smem;
    ab.r[b] = a;
    ab.start[b + 1] = ab.start[b] + a.n_kv_heads * a.splits;
  }
  count_launch();
  cudaError_t e = cudaErrorInvalidValue;
#define DS_ATTB_CASE(DD, RR) \
  if (head_dim == DD && R == RR) e = attn_batch_launch_t<DD, RR>(ab, smem, stream);
  DS_ATTB_CASE(128, 1) DS_ATTB_CASE(128, 2) DS_ATTB_CASE(128, 4) DS_ATTB_CASE(128, 8)
  DS_ATTB_CASE(64, 1) DS_ATTB_CASE(64, 2) DS_ATTB_CASE(64, 4) DS_ATTB_CASE(64, 8)
#undef DS_ATTB_CASE
  return launch_status(e);
}

// ---------------------------------------------------------------- persistent anchor

// Sense-reversing grid barrier over one CTA per SM.  bar[0] counts arrivals,
// bar[1] is the generation; `gen` is thread 0's copy of the generation.
// Spins are bounded: a barrier (or a wait on the other stream) that has not
// completed within 10 s traps instead of hanging the GPU.
DS_DEV unsigned int sm_id() {
  unsigned int v;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(v));
  return v;
}
// On a timeout the spinning thread reports what it waited for, then traps.
DS_DEV void spin_check(unsigned long long t0, const unsigned int* word, unsigned int want, const char* what) {
  if (global_ns() - t0 > 10000000000ull) {
    printf("anchor: %s timed out in CTA %d (SM %u): word %u, waiting for %u\n", what, (int)blockIdx.x, sm_id(),
           *(volatile const unsigned int*)word, want);
    __trap();
  }
}

DS_DEV void grid_sync(unsigned int* bar, unsigned int& gen, unsigned int nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int g = gen;
    if (atomicAdd(bar, 1u) == nblocks - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicExch(bar + 1, g + 1);
    } else {
      // back off: the generation word sits in one L2 slice that the other
      // stream's GEMM / FA traffic also uses
      const unsigned long long t0 = global_ns();
      unsigned int it = 0, ns = 32;
      while (ld_acquire_u32(bar + 1) == g) {
        if (++it > 8) {
          __nanosleep(ns);
          ns = ns < 512 ? 2 * ns : 512;
        }
        if ((it & 255u) == 0) spin_check(t0, bar, nblocks, "grid barrier (arrivals)");
      }
    }
    gen = g + 1;
    __threadfence();
  }
  __syncthreads();
}

// CTA 0 records the global time at phase boundaries (ds_anchor_timeline).
DS_DEV void stamp(const AnchorArgs& a, int rank, int i) {
  if (rank == 0 && threadIdx.x == 0 && a.stamps) a.stamps[i] = global_ns();
}

// Thread 0 waits until *counter >= target (the other stream's GEMM epilogues).
// One CTA polls (rank 0); the others wait for it at the next grid barrier.
DS_DEV void wait_count(const unsigned int* counter, unsigned int target) {
  if (threadIdx.x == 0) {
    const unsigned long long t0 = global_ns();
    unsigned int it = 0;
    while (ld_acquire_u32(counter) < target) {
      __nanosleep(500);
      if ((++it & 255u) == 0) spin_check(t0, counter, target, "wait on the recompute's GEMM counter");
    }
    __threadfence();
  }
  __syncthreads();
}

template <int D, int R>
__global__ void __maxnreg__(88) anchor_persistent_kernel(const __grid_constant__ AnchorArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  bf16* xs = reinterpret_cast<bf16*>(smem);
  float* sc = reinterpret_cast<float*>(smem);
  __shared__ float red[GEMV_WARPS][GEMV_ROWS];
  __shared__ float ssq[GEMV_WARPS];
  __shared__ float stat[2 * R];
  __shared__ unsigned int is_last;
  const int tid = threadIdx.x;
  const int hd = a.n_heads * D, kvd = a.n_kv_heads * D;
  const bool swiglu = a.mlp_kind == DS_MLP_SWIGLU;
  const int n_items = a.n_kv_heads * a.splits;
  // At most per_sm working CTAs per SM (1 beside the recompute, 4 alone): a
  // CTA that finds the SM already full (the scheduler packed CTAs onto an idle
  // SM) leaves after the first barrier, so the SM's resources go back to the
  // other stream's GEMM / FA; the work is spread over the CTAs that stay.
  __shared__ int s_rank;
  __shared__ unsigned int s_nranks;
  unsigned int gen = 0;
  unsigned int smid = 0;
  if (tid == 0) {
    gen = ld_acquire_u32(a.bar + 1);
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    a.bar[2 + blockIdx.x] = smid;  // placement record (ds_anchor_placement)
    const bool keep = atomicAdd(a.claim + (smid & (kAnchorClaimSlots - 1)), 1u) < (unsigned)a.per_sm;
    s_rank = keep ? (int)atomicAdd(a.n_active, 1u) : -1;
  }
  grid_sync(a.bar, gen, gridDim.x);
  const int rank = s_rank;
  if (rank < 0) return;
  if (tid == 0) {
    s_nranks = ld_acquire_u32(a.n_active);
    a.claim[smid & (kAnchorClaimSlots - 1)] = 0u;  // every claim on this SM happened before the barrier
  }
  __syncthreads();
  const int nranks = (int)s_nranks;

  // seed: h = embed[token] (f32 residual stream of the anchor row)
  if (rank == 0) {
    const bf16* e = a.embed + (long long)__ldcg(a.token) * a.d_model;
    for (int k = tid; k < a.d_model; k += GEMV_THREADS) a.h[k] = __bfloat162float(e[k]);
  }
  grid_sync(a.bar, gen, nranks);
  stamp(a, rank, 0);

  for (int l = 0; l < a.n_layers; ++l) {
    const AnchorLayer& W = a.layer[l];
    // ---- q/k/v of the anchor row (+RoPE; its K/V into the consumer cache)
    {
      GemvArgs g{};
      g.W = W.wqkv;
      g.ldw = a.d_model;
      g.N = hd + 2 * kvd;
      g.K = a.d_model;
      g.x_f32 = a.h;
      g.gain = W.g_attn;
      g.mode = EPI_QKV_ROPE;
      g.n_heads = a.n_heads;
      g.n_kv_heads = a.n_kv_heads;
      g.head_dim = D;
      g.pos = a.pos;
      g.q_out = a.q;
      g.kv = W.dst;
      g.rope_cos = a.rope_cos;
      g.rope_sin = a.rope_sin;
      if (rank < g.N / GEMV_ROWS) gemv_prefetch(g, rank);
      gemv_stage_x(g, xs, ssq);
      gemv_all_tiles(g, xs, red, rank, nranks);
    }
    grid_sync(a.bar, gen, nranks);
    stamp(a, rank, 1 + 5 * l + 0);
    // ---- attention over keys 0..pos (a recomputed layer: once its window K/V are in)
    if (W.wait) {
      if (rank == 0) wait_count(a.done + l, W.wait);
      grid_sync(a.bar, gen, nranks);
    }
    {
      AttnArgs t{};
      t.q = a.q;
      t.lo = W.src;
      t.hi = W.dst;
      t.copy_lo = W.copy;
      t.lo_remote = W.src_remote;
      t.n_lo = a.pos;
      t.n_keys = a.pos + 1;
      t.n_heads = a.n_heads;
      t.n_kv_heads = a.n_kv_heads;
      t.splits = a.splits;
      t.split_keys = a.split_keys;
      t.part_o = a.part_o;
      t.part_ml = a.part_ml;
      t.counters = a.head_count;
      t.out = a.o;
      t.scale_log2 = a.scale_log2;
      if (rank < n_items) attn_prefetch(t, rank, D);
      for (int it = rank; it < n_items; it += nranks) {
        if (it + nranks < n_items) attn_prefetch(t, it + nranks, D);
        attn_item<D, R>(t, it, sc, stat, &is_last);
      }
    }
    grid_sync(a.bar, gen, nranks);
    stamp(a, rank, 1 + 5 * l + 1);
    // ---- o-proj + residual
    {
      GemvArgs g{};
      g.W = W.wo;
      g.ldw = hd;
      g.N = a.d_model;
      g.K = hd;
      g.x_bf16 = a.o;
      g.mode = EPI_RESID_F32;
      g.out_f32 = a.h;
      g.resid = a.h;
      if (rank < g.N / GEMV_ROWS) gemv_prefetch(g, rank);
      gemv_stage_x(g, xs, ssq);
      gemv_all_tiles(g, xs, red, rank, nranks);
    }
    grid_sync(a.bar, gen, nranks);
    stamp(a, rank, 1 + 5 * l + 2);
    // ---- MLP up (RMSNorm fused) + SiLU / SwiGLU
    {
      GemvArgs g{};
      g.W = W.w1;
      g.ldw = a.d_model;
      g.N = swiglu ? 2 * a.d_ff : a.d_ff;
      g.K = a.d_model;
      g.x_f32 = a.h;
      g.gain = W.g_mlp;
      g.mode = swiglu ? EPI_SWIGLU_BF16 : EPI_SILU_BF16;
      g.out_bf16 = a.u;
      if (rank < g.N / GEMV_ROWS) gemv_prefetch(g, rank);
      gemv_stage_x(g, xs, ssq);
      gemv_all_tiles(g, xs, red, rank, nranks);
    }
    grid_sync(a.bar, gen, nranks);
    stamp(a, rank, 1 + 5 * l + 3);
    // ---- MLP down + residual
    {
      GemvArgs g{};
      g.W = W.w2;
      g.ldw = a.d_ff;
      g.N = a.d_model;
      g.K = a.d_ff;
      g.x_bf16 = a.u;
      g.mode = EPI_RESID_F32;
      g.out_f32 = a.h;
      g.resid = a.h;
      if (rank < g.N / GEMV_ROWS) gemv_prefetch(g, rank);
      gemv_stage_x(g, xs, ssq);
      gemv_all_tiles(g, xs, red, rank, nranks);
    }
    grid_sync(a.bar, gen, nranks);
    stamp(a, rank, 1 + 5 * l + 4);
  }
  // every wait is over: re-arm the counters for the next step
  if (rank == 0) {
    for (int i = tid; i < a.n_layers; i += GEMV_THREADS)
      if (a.layer[i].wait) a.done[i] = 0u;
    if (tid == 0) *a.n_active = 0u;
  }
}

int anchor_persistent_smem(const ds_dims& d, int n_keys) {
  const int R = d.n_heads / d.n_kv_heads;
  const int sk = attn_split_keys(n_keys, d.n_kv_heads, R);
  const int splits = (n_keys + sk - 1) / sk;
  int kmax = d.d_model > d.d_ff ? d.d_model : d.d_ff;
  if (d.n_heads * d.head_dim > kmax) kmax = d.n_heads * d.head_dim;
  const int x = 2 * kmax, att = attn_smem_bytes(R, sk, splits);
  return x > att ? x : att;
}

// Largest dynamic shared memory that still lets the kernel share an SM with
// a tcgen05 GEMM or flash-attention CTA (each ~198.9 KB incl. its reservation).
constexpr int kAnchorSmemMax = 32 * 1024;
// Alone on the GPU: 4 CTAs per SM (16 warps), so the weight streams are not
// latency-bound; same work split per rank, same results.
constexpr int kAnchorAlonePerSm = 4;

bool anchor_persistent_fits(const ds_dims& d, int n_keys) {
  if (d.n_kv_heads < 1) return false;
  const int R = d.n_heads / d.n_kv_heads;
  return (R == 1 || R == 2 || R == 4 || R == 8) && (d.head_dim == 64 || d.head_dim == 128) &&
         d.n_layers <= kMaxLayers && anchor_persistent_smem(d, n_keys) <= kAnchorSmemMax;
}

template <int D, int R>
static cudaError_t anchor_launch_t(const AnchorArgs& a, int smem, cudaStream_t stream) {
  auto kern = anchor_persistent_kernel<D, R>;
  static PerDevice smem_set;
  if (cudaError_t e = ensure_smem_attr(kern, kAnchorSmemMax, smem_set)) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(num_sms() * a.per_sm);
  cfg.blockDim = dim3(GEMV_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // one co-resident CTA per SM (grid barriers)
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

int anchor_persistent_launch(AnchorArgs a, cudaStream_t stream, bool co_resident) {
  const int R = a.n_heads / a.n_kv_heads;
  const int D = a.head_dim;
  if ((R != 1 && R != 2 && R != 4 && R != 8) || (D != 64 && D != 128) || a.n_layers > kMaxLayers) return DS_ERR_INVALID;
  ds_dims d{};
  d.n_heads = a.n_heads;
  d.n_kv_heads = a.n_kv_heads;
  d.head_dim = D;
  d.d_model = a.d_model;
  d.d_ff = a.d_ff;
  const int smem = anchor_persistent_smem(d, a.pos + 1);
  if (smem > kAnchorSmemMax) return DS_ERR_INVALID;
  a.per_sm = co_resident ? 1 : kAnchorAlonePerSm;
  a.split_keys = attn_split_keys(a.pos + 1, a.n_kv_heads, R);
  a.splits = (a.pos + 1 + a.split_keys - 1) / a.split_keys;
  a.scale_log2 = (float)(1.4426950408889634 / sqrt((double)D));
  count_launch();
  cudaError_t e = cudaErrorInvalidValue;
#define DS_ANC_CASE(DD, RR) \
  if (D == DD && R == RR) e = anchor_launch_t<DD, RR>(a, smem, stream);
  DS_ANC_CASE(128, 1) DS_ANC_CASE(128, 2) DS_ANC_CASE(128, 4) DS_ANC_CASE(128, 8)
  DS_ANC_CASE(64, 1) DS_ANC_CASE(64, 2) DS_ANC_CASE(64, 4) DS_ANC_CASE(64, 8)
#undef DS_ANC_CASE
  return launch_status(e);
}

}  // namespace ds
