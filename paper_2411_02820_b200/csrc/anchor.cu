// Anchor pass kernels: the single final position through every layer
// (_layer_single, model.py:547-562) and the first-token logits
// (_final_logits + argmax, model.py:565-566, 779).  All HBM-bound weight
// streaming:
//   gemv_kernel      y = W[N][K] . x, optional fused RMSNorm of an f32 input,
//                    epilogues: RoPE + q / KV-cache write, residual add, SiLU,
//                    logits + packed argmax (lowest id on ties)
//   decode_attn      split-KV attention of the anchor's H query heads over the
//                    cache positions 0..P (its own K/V already written at P)
//   decode_combine   merge of the split partials -> bf16 [H*D]
#include "common.cuh"
#include "kernels.h"

namespace ds {

constexpr int GEMV_THREADS = 256;
constexpr int GEMV_WARPS = GEMV_THREADS / 32;


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

__global__ void __launch_bounds__(GEMV_THREADS) gemv_kernel(GemvArgs a) {
  extern __shared__ __align__(16) uint8_t smem_x[];
  bf16* xs = reinterpret_cast<bf16*>(smem_x);
  __shared__ float red[GEMV_WARPS];
  __shared__ unsigned long long best_s[GEMV_WARPS];
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
      if (lane == 0) red[warp] = ss;
      __syncthreads();
      float t = 0.f;
#pragma unroll
      for (int w = 0; w < GEMV_WARPS; ++w) t += red[w];
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

  const int half = a.head_dim >> 1;
  const int items = a.N >> 1;
  unsigned long long best = 0ull;
  const int nchunk = a.K >> 3;
  for (int it = blockIdx.x * GEMV_WARPS + warp; it < items; it += gridDim.x * GEMV_WARPS) {
    int r0, r1;
    if (a.mode == EPI_QKV_ROPE) {
      const int head = it / half, j = it - head * half;
      r0 = head * a.head_dim + j;
      r1 = r0 + half;
    } else {
      r0 = 2 * it;
      r1 = r0 + 1;
    }
    const bf16* w0 = a.W + (long long)r0 * a.ldw;
    const bf16* w1 = a.W + (long long)r1 * a.ldw;
    float s0 = 0.f, s1 = 0.f;
    int c = lane;
    for (; c + 96 < nchunk; c += 128) {
      uint4 wa[4], wb[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        wa[u] = ld_stream16(w0 + (c + 32 * u) * 8);
        wb[u] = ld_stream16(w1 + (c + 32 * u) * 8);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        uint4 xv = *reinterpret_cast<const uint4*>(xs + (c + 32 * u) * 8);
        s0 += dot8(wa[u], xv);
        s1 += dot8(wb[u], xv);
      }
    }
    for (; c < nchunk; c += 32) {
      uint4 xv = *reinterpret_cast<const uint4*>(xs + c * 8);
      s0 += dot8(ld_stream16(w0 + c * 8), xv);
      s1 += dot8(ld_stream16(w1 + c * 8), xv);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    }
    if (lane != 0) continue;
    switch (a.mode) {
      case EPI_QKV_ROPE: {
        const int head = r0 / a.head_dim, j = r0 - head * a.head_dim;
        float lo = s0, hi = s1;
        const bool is_q = head < a.n_heads, is_k = !is_q && head < a.n_heads + a.n_kv_heads;
        if (is_q || is_k) {
          const float cs = a.rope_cos[(long long)a.pos * half + j], sn = a.rope_sin[(long long)a.pos * half + j];
          lo = s0 * cs - s1 * sn;
          hi = s0 * sn + s1 * cs;
        }
        bf16* dst = is_q ? a.q_out + (long long)head * a.head_dim
                         : (is_k ? a.kv.k + a.kv.off(head - a.n_heads, a.pos)
                                 : a.kv.v + a.kv.off(head - a.n_heads - a.n_kv_heads, a.pos));
        dst[j] = __float2bfloat16_rn(lo);
        dst[j + half] = __float2bfloat16_rn(hi);
        break;
      }
      case EPI_RESID_F32:
        a.out_f32[r0] = a.resid[r0] + s0;
        a.out_f32[r1] = a.resid[r1] + s1;
        break;
      case EPI_SILU_BF16:
        a.out_bf16[r0] = __float2bfloat16_rn(silu(s0));
        a.out_bf16[r1] = __float2bfloat16_rn(silu(s1));
        break;
      default: {
        a.out_f32[r0] = s0;
        a.out_f32[r1] = s1;
        unsigned long long p0 = pack_argmax(s0, r0), p1 = pack_argmax(s1, r1);
        unsigned long long p = p0 > p1 ? p0 : p1;
        best = p > best ? p : best;
      }
    }
  }
  if (a.mode == EPI_STORE_F32 && a.argmax) {
    if (lane == 0) best_s[warp] = best;
    __syncthreads();
    if (tid == 0) {
      unsigned long long b = 0ull;
      for (int w = 0; w < GEMV_WARPS; ++w) b = best_s[w] > b ? best_s[w] : b;
      if (b) atomicMax(a.argmax, b);
    }
  }
}

__global__ void argmax_finalize_kernel(const unsigned long long* packed, int32_t* token) {
  *token = (int32_t)(0xFFFFFFFFu - (uint32_t)(*packed & 0xFFFFFFFFull));
}

int gemv_launch(const GemvArgs& a, cudaStream_t stream) {
  if ((a.N & 1) || (a.K & 7)) return DS_ERR_INVALID;
  const int items = a.N / 2;
  int grid = (items + GEMV_WARPS - 1) / GEMV_WARPS;
  const int cap = num_sms() * 4;
  if (grid > cap) grid = cap;
  const int smem = a.K * 2;
  static int attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    if (cudaFuncSetAttribute(gemv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return DS_ERR_CUDA;
    attr = smem;
  }
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
constexpr int DEC_CHUNK = 256;
constexpr int DEC_MAX_R = 8;

struct DecArgs {
  const bf16* q;  // [H*D]
  const bf16* k;  // layer base
  const bf16* v;
  long long head_stride, page_stride;
  const int32_t* table;
  int n_keys, n_heads, n_kv_heads, head_dim;
  float* part_o;   // [splits][H][D]
  float* part_ml;  // [splits][H][2]
  float scale_log2;
};

__global__ void __launch_bounds__(DEC_THREADS) decode_attn_kernel(DecArgs a) {
  const int g = blockIdx.x, split = blockIdx.y;
  const int R = a.n_heads / a.n_kv_heads, D = a.head_dim;
  const int k0 = split * DEC_CHUNK;
  const int nk = min(DEC_CHUNK, a.n_keys - k0);
  __shared__ float qs[DEC_MAX_R * 128];
  __shared__ float sc[DEC_MAX_R][DEC_CHUNK];
  __shared__ float stat[DEC_MAX_R][2];
  __shared__ float ored[DEC_MAX_R][128];
  const int tid = threadIdx.x;
  for (int i = tid; i < R * D; i += DEC_THREADS) qs[i] = __bfloat162float(a.q[(long long)g * R * D + i]);
  __syncthreads();
  // scores: one thread per key
  for (int kk = tid; kk < nk; kk += DEC_THREADS) {
    const int pos = k0 + kk;
    const int page = a.table ? __ldg(a.table + (pos >> 6)) : (pos >> 6);
    const bf16* kr = a.k + (long long)g * a.head_stride + (long long)page * a.page_stride + (long long)(pos & 63) * D;
    float acc[DEC_MAX_R];
#pragma unroll
    for (int r = 0; r < DEC_MAX_R; ++r) acc[r] = 0.f;
    for (int c = 0; c < D; c += 8) {
      uint4 u = *reinterpret_cast<const uint4*>(kr + c);
      float2 e0 = unpack_bf16x2(u.x), e1 = unpack_bf16x2(u.y), e2 = unpack_bf16x2(u.z), e3 = unpack_bf16x2(u.w);
      const float kv8[8] = {e0.x, e0.y, e1.x, e1.y, e2.x, e2.y, e3.x, e3.y};
#pragma unroll
      for (int r = 0; r < DEC_MAX_R; ++r) {
        if (r < R) {
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[r] = fmaf(qs[r * D + c + i], kv8[i], acc[r]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < DEC_MAX_R; ++r)
      if (r < R) sc[r][kk] = acc[r] * a.scale_log2;
  }
  __syncthreads();
  // per-head max and sum (warp w handles heads w, w+4, ...)
  const int warp = tid >> 5, lane = tid & 31;
  for (int r = warp; r < R; r += DEC_THREADS / 32) {
    float m = -INFINITY;
    for (int i = lane; i < nk; i += 32) m = fmaxf(m, sc[r][i]);
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float l = 0.f;
    for (int i = lane; i < nk; i += 32) {
      float p = exp2f(sc[r][i] - m);
      sc[r][i] = p;
      l += p;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    if (lane == 0) {
      stat[r][0] = m;
      stat[r][1] = l;
    }
  }
  __syncthreads();
  // P.V: thread -> (d = tid % D, key lane = tid / D)
  const int d = tid % D, kl = tid / D, nkl = DEC_THREADS / D;
  float o[DEC_MAX_R];
#pragma unroll
  for (int r = 0; r < DEC_MAX_R; ++r) o[r] = 0.f;
  for (int kk = kl; kk < nk; kk += nkl) {
    const int pos = k0 + kk;
    const int page = a.table ? __ldg(a.table + (pos >> 6)) : (pos >> 6);
    const float vv = __bfloat162float(
        a.v[(long long)g * a.head_stride + (long long)page * a.page_stride + (long long)(pos & 63) * D + d]);
#pragma unroll
    for (int r = 0; r < DEC_MAX_R; ++r)
      if (r < R) o[r] = fmaf(sc[r][kk], vv, o[r]);
  }
  if (nkl > 1) {
    if (kl == 1) {
#pragma unroll
      for (int r = 0; r < DEC_MAX_R; ++r)
        if (r < R) ored[r][d] = o[r];
    }
    __syncthreads();
    if (kl == 0) {
#pragma unroll
      for (int r = 0; r < DEC_MAX_R; ++r)
        if (r < R) o[r] += ored[r][d];
    }
  }
  if (kl == 0) {
    for (int r = 0; r < R; ++r) {
      const int h = g * R + r;
      a.part_o[((long long)split * a.n_heads + h) * D + d] = o[r];
      if (d == 0) {
        a.part_ml[((long long)split * a.n_heads + h) * 2 + 0] = stat[r][0];
        a.part_ml[((long long)split * a.n_heads + h) * 2 + 1] = stat[r][1];
      }
    }
  }
}

__global__ void decode_combine_kernel(const float* part_o, const float* part_ml, int splits, int n_heads, int D,
                                      bf16* out) {
  const int h = blockIdx.x, d = threadIdx.x;
  float M = -INFINITY;
  for (int s = 0; s < splits; ++s) M = fmaxf(M, part_ml[((long long)s * n_heads + h) * 2]);
  float num = 0.f, den = 0.f;
  for (int s = 0; s < splits; ++s) {
    const float w = exp2f(part_ml[((long long)s * n_heads + h) * 2] - M);
    den += w * part_ml[((long long)s * n_heads + h) * 2 + 1];
    num += w * part_o[((long long)s * n_heads + h) * D + d];
  }
  out[(long long)h * D + d] = __float2bfloat16_rn(num / den);
}

int decode_splits(int n_keys) { return (n_keys + DEC_CHUNK - 1) / DEC_CHUNK; }

int decode_attention_launch(const bf16* q, const bf16* k_layer, const bf16* v_layer, long long head_stride,
                            long long page_stride, const int32_t* table, int n_keys, int n_heads, int n_kv_heads,
                            int head_dim, float* part_o, float* part_ml, bf16* out, cudaStream_t stream) {
  const int R = n_heads / n_kv_heads;
  if (R > DEC_MAX_R || head_dim > 128 || (DEC_THREADS % head_dim)) return DS_ERR_INVALID;
  DecArgs a{q, k_layer, v_layer, head_stride, page_stride, table, n_keys, n_heads, n_kv_heads, head_dim,
            part_o, part_ml, (float)(1.4426950408889634 / sqrt((double)head_dim))};
  const int splits = decode_splits(n_keys);
  count_launch(2);
  decode_attn_kernel<<<dim3(n_kv_heads, splits), DEC_THREADS, 0, stream>>>(a);
  decode_combine_kernel<<<n_heads, head_dim, 0, stream>>>(part_o, part_ml, splits, n_heads, head_dim, out);
  return cudaGetLastError() == cudaSuccess ? DS_OK : DS_ERR_CUDA;
}

}  // namespace ds
