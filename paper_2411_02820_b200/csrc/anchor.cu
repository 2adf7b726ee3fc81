// Anchor pass kernels: the single final position through every layer
// (_layer_single, model.py:547-562) and the first-token logits
// (_final_logits + argmax, model.py:565-566, 779).  All HBM-bound:
//
//   gemv_kernel    y = W[N][K] . x over tiles of 8 weight rows per CTA; the 256
//                  threads split K (16-byte coalesced row chunks, 16 loads in
//                  flight per thread), block-reduce, fused epilogue:
//                  RoPE + q / KV-cache write, residual add, SiLU, logits +
//                  packed argmax (lowest id on ties).  An f32 input is
//                  RMSNorm'ed in the prologue (model.py:466-468).
//   decode_attn    split-KV attention of the anchor's query heads: one CTA per
//                  (kv head, 512-key split) streams 128-key tiles (two K pages and
//                  two V pages, contiguous 64 x D blocks) through a 2-stage
//                  bulk-copy ring, online softmax over the R = H/KVH heads, and
//                  the last CTA of each kv head merges all splits (no second launch).
#include "common.cuh"
#include "kernels.h"

namespace ds {

constexpr int GEMV_THREADS = 256;
constexpr int GEMV_WARPS = GEMV_THREADS / 32;
constexpr int GEMV_ROWS = 8;    // weight rows per tile
constexpr int GEMV_UNROLL = 2;  // 16-byte chunks per row per thread in flight

DS_DEV uint4 ld_stream16(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
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

// Global row of slot r (0..7) of tile t.  QKV tiles hold 4 RoPE pairs
// (rows head*D + j0 + i and head*D + half + j0 + i, i < 4) so the rotation
// happens in the epilogue; other modes take 8 consecutive rows.
DS_DEV int gemv_row(const GemvArgs& a, int t, int r) {
  if (a.mode != EPI_QKV_ROPE) return t * GEMV_ROWS + r;
  const int half = a.head_dim >> 1;
  const int per_head = half / 4;
  const int head = t / per_head, j0 = (t - head * per_head) * 4;
  return head * a.head_dim + (r < 4 ? j0 + r : half + j0 + r - 4);
}

__global__ void __launch_bounds__(GEMV_THREADS) gemv_kernel(GemvArgs a) {
  extern __shared__ __align__(16) uint8_t smem_x[];
  bf16* xs = reinterpret_cast<bf16*>(smem_x);
  __shared__ float red[GEMV_WARPS][GEMV_ROWS];
  __shared__ float ssq[GEMV_WARPS];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---- stage the input vector (bf16) in shared memory, RMSNorm fused
  if (a.x_f32) {
    float inv = 1.f;
    if (a.gain) {
      float ss = 0.f;
      for (int k = tid * 4; k < a.K; k += GEMV_THREADS * 4) {
        float4 v = *reinterpret_cast<const float4*>(a.x_f32 + k);
        ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (lane == 0) ssq[warp] = ss;
      __syncthreads();
      float t = 0.f;
#pragma unroll
      for (int w = 0; w < GEMV_WARPS; ++w) t += ssq[w];
      inv = 1.0f / sqrtf(t / (float)a.K + 1e-6f);
    }
    for (int k = tid * 4; k < a.K; k += GEMV_THREADS * 4) {
      float4 v = *reinterpret_cast<const float4*>(a.x_f32 + k);
      float4 g = a.gain ? *reinterpret_cast<const float4*>(a.gain + k) : make_float4(1.f, 1.f, 1.f, 1.f);
      uint2 p;
      p.x = pack_bf16x2(v.x * inv * g.x, v.y * inv * g.y);
      p.y = pack_bf16x2(v.z * inv * g.z, v.w * inv * g.w);
      *reinterpret_cast<uint2*>(xs + k) = p;
    }
  } else {
    for (int k = tid * 8; k < a.K; k += GEMV_THREADS * 8)
      *reinterpret_cast<uint4*>(xs + k) = *reinterpret_cast<const uint4*>(a.x_bf16 + k);
  }
  __syncthreads();

  const int nchunk = a.K >> 3;
  const int tiles = a.mode == EPI_QKV_ROPE ? a.N / a.head_dim * (a.head_dim / 8) : a.N / GEMV_ROWS;
  unsigned long long best = 0ull;
  for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
    const bf16* wr[GEMV_ROWS];
#pragma unroll
    for (int r = 0; r < GEMV_ROWS; ++r) wr[r] = a.W + (long long)gemv_row(a, t, r) * a.ldw;
    float s[GEMV_ROWS];
#pragma unroll
    for (int r = 0; r < GEMV_ROWS; ++r) s[r] = 0.f;
    int c = tid;
    for (; c + (GEMV_UNROLL - 1) * GEMV_THREADS < nchunk; c += GEMV_UNROLL * GEMV_THREADS) {
      uint4 w[GEMV_UNROLL][GEMV_ROWS];
#pragma unroll
      for (int u = 0; u < GEMV_UNROLL; ++u)
#pragma unroll
        for (int r = 0; r < GEMV_ROWS; ++r) w[u][r] = ld_stream16(wr[r] + (c + u * GEMV_THREADS) * 8);
#pragma unroll
      for (int u = 0; u < GEMV_UNROLL; ++u) {
        const uint4 xv = *reinterpret_cast<const uint4*>(xs + (c + u * GEMV_THREADS) * 8);
#pragma unroll
        for (int r = 0; r < GEMV_ROWS; ++r) s[r] += dot8(w[u][r], xv);
      }
    }
    for (; c < nchunk; c += GEMV_THREADS) {
      const uint4 xv = *reinterpret_cast<const uint4*>(xs + c * 8);
#pragma unroll
      for (int r = 0; r < GEMV_ROWS; ++r) s[r] += dot8(ld_stream16(wr[r] + c * 8), xv);
    }
#pragma unroll
    for (int r = 0; r < GEMV_ROWS; ++r) {
#pragma unroll
      for (int o = 16; o; o >>= 1) s[r] += __shfl_xor_sync(0xffffffffu, s[r], o);
    }
    if (lane == 0) {
#pragma unroll
      for (int r = 0; r < GEMV_ROWS; ++r) red[warp][r] = s[r];
    }
    __syncthreads();
    if (tid < GEMV_ROWS) {
      float v = 0.f;
#pragma unroll
      for (int w = 0; w < GEMV_WARPS; ++w) v += red[w][tid];
      red[0][tid] = v;  // only thread tid touches column tid
    }
    __syncthreads();
    if (a.mode == EPI_QKV_ROPE) {
      if (tid < 4) {
        const int r0 = gemv_row(a, t, tid);
        const int head = r0 / a.head_dim, j = r0 - head * a.head_dim, half = a.head_dim >> 1;
        float lo = red[0][tid], hi = red[0][tid + 4];
        const bool is_q = head < a.n_heads, is_k = !is_q && head < a.n_heads + a.n_kv_heads;
        if (is_q || is_k) {
          const float cs = a.rope_cos[(long long)a.pos * half + j], sn = a.rope_sin[(long long)a.pos * half + j];
          const float x1 = lo, x2 = hi;
          lo = x1 * cs - x2 * sn;
          hi = x1 * sn + x2 * cs;
        }
        bf16* dst = is_q ? a.q_out + (long long)head * a.head_dim
                         : (is_k ? a.kv.k + a.kv.off(head - a.n_heads, a.pos)
                                 : a.kv.v + a.kv.off(head - a.n_heads - a.n_kv_heads, a.pos));
        dst[j] = __float2bfloat16_rn(lo);
        dst[j + half] = __float2bfloat16_rn(hi);
      }
    } else if (tid < GEMV_ROWS) {
      const int row = t * GEMV_ROWS + tid;
      const float v = red[0][tid];
      if (a.mode == EPI_RESID_F32) {
        a.out_f32[row] = a.resid[row] + v;
      } else if (a.mode == EPI_SILU_BF16) {
        a.out_bf16[row] = __float2bfloat16_rn(silu(v));
      } else {
        a.out_f32[row] = v;
        const unsigned long long p = pack_argmax(v, row);
        best = p > best ? p : best;
      }
    }
    __syncthreads();  // red[] reused by the next tile
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

__global__ void argmax_finalize_kernel(const unsigned long long* packed, int32_t* token) {
  *token = (int32_t)(0xFFFFFFFFu - (uint32_t)(*packed & 0xFFFFFFFFull));
}

int gemv_launch(const GemvArgs& a, cudaStream_t stream) {
  if ((a.N % GEMV_ROWS) || (a.K & 7)) return DS_ERR_INVALID;
  if (a.mode == EPI_QKV_ROPE && (a.head_dim % 8 || a.N % a.head_dim)) return DS_ERR_INVALID;
  const int tiles = a.N / GEMV_ROWS;
  const int smem = a.K * 2;
  static int attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    if (cudaFuncSetAttribute(gemv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return DS_ERR_CUDA;
    attr = smem;
  }
  int per_sm = (200 * 1024) / (smem + 2048);
  per_sm = per_sm < 1 ? 1 : (per_sm > 8 ? 8 : per_sm);
  const int cap = num_sms() * per_sm;
  const int grid = tiles < cap ? tiles : cap;
  count_launch();
  gemv_kernel<<<grid, GEMV_THREADS, smem, stream>>>(a);
  return cudaGetLastError() == cudaSuccess ? DS_OK : DS_ERR_CUDA;
}

int argmax_finalize_launch(const unsigned long long* packed, int32_t* token, cudaStream_t stream) {
  count_launch();
  argmax_finalize_kernel<<<1, 1, 0, stream>>>(packed, token);
  return cudaGetLastError() == cudaSuccess ? DS_OK : DS_ERR_CUDA;
}

// ---------------------------------------------------------------- decode attention

constexpr int DEC_THREADS = 128;
constexpr int DEC_TILE = 128;                 // keys per shared-memory stage (two 64-position pages)
constexpr int DEC_TILES_PER_SPLIT = 4;        // 512 keys per CTA
constexpr int DEC_SPLIT = DEC_TILE * DEC_TILES_PER_SPLIT;
constexpr int DEC_MAX_R = 8;

struct DecArgs {
  const bf16* q;  // [H*D]
  const bf16* k;  // layer base
  const bf16* v;
  long long head_stride, page_stride;
  const int32_t* table;
  int n_keys, n_heads, n_kv_heads, head_dim, splits;
  float* part_o;             // [H][splits][D]
  float* part_ml;            // [H][splits][2]
  unsigned int* counters;    // [KVH], zero between launches (the last CTA resets)
  bf16* out;                 // [H*D]
  float scale_log2;
};

template <int D>
__global__ void __launch_bounds__(DEC_THREADS) decode_attn_kernel(DecArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int STAGE = 2 * DEC_TILE * D;                      // bf16 elements per stage (K then V)
  bf16* ring = reinterpret_cast<bf16*>(smem);                  // [2][K 128xD | V 128xD]
  float* qs = reinterpret_cast<float*>(ring + 2 * STAGE);      // [R][D]
  float* sc = qs + DEC_MAX_R * D;                              // [R][128]
  float* mstat = sc + DEC_MAX_R * DEC_TILE;                    // [R] running max, [R] tile max, [R] sum
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ unsigned int is_last;

  const int g = blockIdx.x, split = blockIdx.y, tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int R = a.n_heads / a.n_kv_heads;
  const int key0 = split * DEC_SPLIT;
  const int nk_split = min(DEC_SPLIT, a.n_keys - key0);
  const int n_tiles = (nk_split + DEC_TILE - 1) / DEC_TILE;

  auto issue = [&](int t) {  // thread 0: bulk-copy tile t's K/V pages into stage t & 1
    const int st = t & 1;
    const int k0 = key0 + t * DEC_TILE;
    const int nk = min(DEC_TILE, a.n_keys - k0);
    mbar_expect_tx(&bar[st], (uint32_t)nk * D * 2 * 2);
    for (int p = 0; p * 64 < nk; ++p) {
      const int pos = k0 + p * 64;
      const int page = a.table ? __ldg(a.table + (pos >> 6)) : (pos >> 6);
      const long long off = (long long)g * a.head_stride + (long long)page * a.page_stride;
      const uint32_t bytes = (uint32_t)min(64, nk - p * 64) * D * 2;
      bf16* dst = ring + st * STAGE;
      bulk_g2s(dst + p * 64 * D, a.k + off, bytes, &bar[st]);
      bulk_g2s(dst + DEC_TILE * D + p * 64 * D, a.v + off, bytes, &bar[st]);
    }
  };
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
    issue(0);
    if (n_tiles > 1) issue(1);
  }
  for (int i = tid; i < R * D; i += DEC_THREADS) qs[i] = __bfloat162float(a.q[(long long)g * R * D + i]);
  if (tid < DEC_MAX_R) {
    mstat[tid] = -INFINITY;
    mstat[2 * DEC_MAX_R + tid] = 0.f;
  }
  __syncthreads();

  constexpr int KG = DEC_THREADS / D;  // key groups in the P.V loop (2 for D = 64)
  const int d = tid % D, kg = tid / D;
  float o[DEC_MAX_R];
#pragma unroll
  for (int r = 0; r < DEC_MAX_R; ++r) o[r] = 0.f;

  for (int t = 0; t < n_tiles; ++t) {
    const int st = t & 1;
    const int nk = min(DEC_TILE, nk_split - t * DEC_TILE);
    mbar_wait(&bar[st], (uint32_t)(t >> 1) & 1u);
    const bf16* sk = ring + st * STAGE;
    const bf16* sv = sk + DEC_TILE * D;
    // scores: thread = key; 16-byte chunks read staggered by key (bank-conflict free)
    if (tid < nk) {
      float acc[DEC_MAX_R];
#pragma unroll
      for (int r = 0; r < DEC_MAX_R; ++r) acc[r] = 0.f;
      const bf16* kr = sk + tid * D;
#pragma unroll 4
      for (int cc = 0; cc < D / 8; ++cc) {
        const int c = (cc + tid) & (D / 8 - 1);
        const uint4 u = *reinterpret_cast<const uint4*>(kr + c * 8);
        const float2 e0 = unpack_bf16x2(u.x), e1 = unpack_bf16x2(u.y), e2 = unpack_bf16x2(u.z),
                     e3 = unpack_bf16x2(u.w);
        const float kv8[8] = {e0.x, e0.y, e1.x, e1.y, e2.x, e2.y, e3.x, e3.y};
#pragma unroll
        for (int r = 0; r < DEC_MAX_R; ++r) {
          if (r < R) {
            const float4 q0 = *reinterpret_cast<const float4*>(qs + r * D + c * 8);
            const float4 q1 = *reinterpret_cast<const float4*>(qs + r * D + c * 8 + 4);
            acc[r] = fmaf(q0.x, kv8[0], acc[r]);
            acc[r] = fmaf(q0.y, kv8[1], acc[r]);
            acc[r] = fmaf(q0.z, kv8[2], acc[r]);
            acc[r] = fmaf(q0.w, kv8[3], acc[r]);
            acc[r] = fmaf(q1.x, kv8[4], acc[r]);
            acc[r] = fmaf(q1.y, kv8[5], acc[r]);
            acc[r] = fmaf(q1.z, kv8[6], acc[r]);
            acc[r] = fmaf(q1.w, kv8[7], acc[r]);
          }
        }
      }
#pragma unroll
      for (int r = 0; r < DEC_MAX_R; ++r)
        if (r < R) sc[r * DEC_TILE + tid] = acc[r] * a.scale_log2;
    }
    __syncthreads();
    // online softmax per head (warp w -> heads w, w+4): new running max, p, tile sum
    for (int r = warp; r < R; r += DEC_THREADS / 32) {
      float m = -INFINITY;
      for (int i = lane; i < nk; i += 32) m = fmaxf(m, sc[r * DEC_TILE + i]);
#pragma unroll
      for (int off = 16; off; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
      const float m_old = mstat[r];
      const float m_new = fmaxf(m_old, m);
      float l = 0.f;
      for (int i = lane; i < nk; i += 32) {
        const float p = exp2f(sc[r * DEC_TILE + i] - m_new);
        sc[r * DEC_TILE + i] = p;
        l += p;
      }
#pragma unroll
      for (int off = 16; off; off >>= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
      __syncwarp();
      if (lane == 0) {
        const float corr = exp2f(m_old - m_new);  // 0 on the first tile
        mstat[DEC_MAX_R + r] = corr;
        mstat[2 * DEC_MAX_R + r] = mstat[2 * DEC_MAX_R + r] * corr + l;
        mstat[r] = m_new;
      }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < DEC_MAX_R; ++r)
      if (r < R) o[r] *= mstat[DEC_MAX_R + r];
    for (int kk = kg; kk < nk; kk += KG) {
      const float vv = __bfloat162float(sv[kk * D + d]);
#pragma unroll
      for (int r = 0; r < DEC_MAX_R; ++r)
        if (r < R) o[r] = fmaf(sc[r * DEC_TILE + kk], vv, o[r]);
    }
    __syncthreads();  // stage st and sc are free
    if (tid == 0 && t + 2 < n_tiles) issue(t + 2);
  }
  if (KG > 1) {
    float* ored = sc;  // [R][D]
    if (kg == 1) {
#pragma unroll
      for (int r = 0; r < DEC_MAX_R; ++r)
        if (r < R) ored[r * D + d] = o[r];
    }
    __syncthreads();
    if (kg == 0) {
#pragma unroll
      for (int r = 0; r < DEC_MAX_R; ++r)
        if (r < R) o[r] += ored[r * D + d];
    }
  }
  if (kg == 0) {
    for (int r = 0; r < R; ++r) {
      const int h = g * R + r;
      a.part_o[((long long)h * a.splits + split) * D + d] = o[r];
      if (d == 0) {
        a.part_ml[((long long)h * a.splits + split) * 2] = mstat[r];
        a.part_ml[((long long)h * a.splits + split) * 2 + 1] = mstat[2 * DEC_MAX_R + r];
      }
    }
  }
  // ---- the last CTA of this kv head merges every split (threadfence reduction)
  __threadfence();
  __syncthreads();
  if (tid == 0) is_last = (atomicAdd(a.counters + g, 1u) == (unsigned)a.splits - 1);
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  // split weights per head in shared memory: w[r][s] = exp2(m_s - M_r), den_r = sum w l
  float* wts = reinterpret_cast<float*>(smem);  // the ring is dead: [R][splits]
  float* den = wts + DEC_MAX_R * a.splits;
  for (int r = warp; r < R; r += DEC_THREADS / 32) {
    const float* ml = a.part_ml + (long long)(g * R + r) * a.splits * 2;
    float M = -INFINITY;
    for (int s = lane; s < a.splits; s += 32) M = fmaxf(M, __ldcg(ml + 2 * s));
#pragma unroll
    for (int off = 16; off; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
    float dn = 0.f;
    for (int s = lane; s < a.splits; s += 32) {
      const float w = exp2f(__ldcg(ml + 2 * s) - M);
      wts[r * a.splits + s] = w;
      dn += w * __ldcg(ml + 2 * s + 1);
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) dn += __shfl_xor_sync(0xffffffffu, dn, off);
    if (lane == 0) den[r] = dn;
  }
  __syncthreads();
  for (int idx = tid; idx < R * D; idx += DEC_THREADS) {
    const int r = idx / D, dd = idx % D, h = g * R + r;
    const float* po = a.part_o + (long long)h * a.splits * D + dd;
    float num = 0.f;
#pragma unroll 8
    for (int s = 0; s < a.splits; ++s) num = fmaf(wts[r * a.splits + s], __ldcg(po + (long long)s * D), num);
    a.out[(long long)h * D + dd] = __float2bfloat16_rn(num / den[r]);
  }
  if (tid == 0) a.counters[g] = 0u;
}

int decode_splits(int n_keys) { return (n_keys + DEC_SPLIT - 1) / DEC_SPLIT; }

int decode_attention_launch(const bf16* q, const bf16* k_layer, const bf16* v_layer, long long head_stride,
                            long long page_stride, const int32_t* table, int n_keys, int n_heads, int n_kv_heads,
                            int head_dim, float* part_o, float* part_ml, unsigned int* counters, bf16* out,
                            cudaStream_t stream) {
  const int R = n_heads / n_kv_heads;
  if (R > DEC_MAX_R || (head_dim != 64 && head_dim != 128)) return DS_ERR_INVALID;
  const int splits = decode_splits(n_keys);
  if (splits * (DEC_MAX_R + 1) * 4 > 2 * 2 * DEC_TILE * head_dim * 2) return DS_ERR_INVALID;  // merge scratch
  DecArgs a{q, k_layer, v_layer, head_stride, page_stride, table, n_keys, n_heads, n_kv_heads, head_dim, splits,
            part_o, part_ml, counters, out, (float)(1.4426950408889634 / sqrt((double)head_dim))};
  const int smem = 2 * 2 * DEC_TILE * head_dim * 2 + DEC_MAX_R * head_dim * 4 + DEC_MAX_R * DEC_TILE * 4 +
                   3 * DEC_MAX_R * 4;
  count_launch();
  if (head_dim == 128) {
    static bool set = false;
    if (!set) {
      if (cudaFuncSetAttribute(decode_attn_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
          cudaSuccess)
        return DS_ERR_CUDA;
      set = true;
    }
    decode_attn_kernel<128><<<dim3(n_kv_heads, splits), DEC_THREADS, smem, stream>>>(a);
  } else {
    static bool set = false;
    if (!set) {
      if (cudaFuncSetAttribute(decode_attn_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
          cudaSuccess)
        return DS_ERR_CUDA;
      set = true;
    }
    decode_attn_kernel<64><<<dim3(n_kv_heads, splits), DEC_THREADS, smem, stream>>>(a);
  }
  return cudaGetLastError() == cudaSuccess ? DS_OK : DS_ERR_CUDA;
}

}  // namespace ds
