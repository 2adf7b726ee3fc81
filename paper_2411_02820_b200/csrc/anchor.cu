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
//   decode_attn    split-KV attention of the anchor's query heads on the tensor
//                  pipe (the GQA group is the M of an m16n8k16 tile), see below.
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

__global__ void __launch_bounds__(GEMV_THREADS, 3) gemv_kernel(GemvArgs a) {
  extern __shared__ __align__(16) uint8_t smem_x[];
  bf16* xs = reinterpret_cast<bf16*>(smem_x);
  __shared__ float red[GEMV_WARPS][GEMV_ROWS];
  __shared__ float ssq[GEMV_WARPS];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tiles = a.N / GEMV_ROWS;

  // ---- weights do not depend on the predecessor kernel: start streaming this
  // CTA's first tile into L2, let the successor launch, then wait (PDL)
  if (blockIdx.x < tiles && tid < GEMV_ROWS)
    prefetch_l2(a.W + (long long)gemv_row(a, blockIdx.x, tid) * a.ldw, (uint32_t)a.K * 2);
  pdl_trigger();
  pdl_wait();

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
    } else if (a.mode == EPI_SWIGLU_BF16) {
      if (tid < 4) {
        const int o = (t >> 2) * 16 + (t & 3) * 4 + tid;
        a.out_bf16[o] = __float2bfloat16_rn(silu(red[0][tid]) * red[0][tid + 4]);
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
  static const bool c0 = prefer_max_smem(token_copy_kernel);
  (void)c0;
  token_copy_kernel<<<1, 1, 0, stream>>>(src, dst32, dst64);
  return launch_status();
}

int gemv_launch(const GemvArgs& a, cudaStream_t stream) {
  if ((a.N % GEMV_ROWS) || (a.K & 7) || (a.mode == EPI_SWIGLU_BF16 && a.N % 32)) return DS_ERR_INVALID;
  if (a.mode == EPI_QKV_ROPE && (a.head_dim % 8 || a.N % a.head_dim)) return DS_ERR_INVALID;
  const int tiles = a.N / GEMV_ROWS;
  const int smem = a.K * 2;
  static int attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    if (int rc_ = launch_status(cudaFuncSetAttribute(gemv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return rc_;
    attr = smem;
  }
  int per_sm = (200 * 1024) / (smem + 2048);
  per_sm = per_sm < 1 ? 1 : (per_sm > 8 ? 8 : per_sm);
  const int cap = num_sms() * per_sm;
  const int grid = tiles < cap ? tiles : cap;
  count_launch();
  static const bool c0 = prefer_max_smem(gemv_kernel);
  (void)c0;
  return launch_status(launch_pdl(gemv_kernel, dim3(grid), dim3(GEMV_THREADS), smem, stream, a));
}

int argmax_finalize_launch(const unsigned long long* packed, int32_t* token, int64_t* token64, cudaStream_t stream) {
  count_launch();
  static const bool c0 = prefer_max_smem(argmax_finalize_kernel);
  (void)c0;
  argmax_finalize_kernel<<<1, 1, 0, stream>>>(packed, token, token64);
  return launch_status();
}

// ---------------------------------------------------------------- decode attention
//
// One CTA per (kv head g, split of DEC_SPLIT keys), 4 warps.  The R = H/KVH
// query heads of the group are the M rows of an m16n8k16 tensor-core tile
// (rows >= R are zero), so scores and P.V run on the tensor pipe.  Operand
// fragments are loaded straight from global memory into registers (K rows are
// already in the B-fragment order; V fragments are transposed in registers
// with movmatrix), so the kernel needs no shared memory for K/V: it co-resides
// with the persistent tcgen05 GEMMs of the recompute running on the other
// stream (their 194 KB shared-memory rings leave ~30 KB per SM).  Warp w owns
// 16-key blocks w, w+4, ... of the split with its own online softmax; the 4
// warps merge through a small shared buffer, and the last CTA of the kv head
// merges all splits.

constexpr int DEC_THREADS = 128;
constexpr int DEC_BLOCK = 16;    // keys per warp step (one mma k-step for P.V)
constexpr int DEC_SPLIT = 256;   // keys per CTA
constexpr int DEC_MAX_R = 16;

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

DS_DEV uint32_t ld_b32(const bf16* p, bool ok) {
  uint32_t r = 0;
  if (ok) r = __ldg(reinterpret_cast<const unsigned int*>(p));
  return r;
}
DS_DEV uint32_t movm_trans(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

template <int D>
__global__ void __launch_bounds__(DEC_THREADS) decode_attn_kernel(DecArgs a) {
  extern __shared__ __align__(16) float red[];  // [4 warps][R][D + 2]
  __shared__ unsigned int is_last;
  const int g = blockIdx.x, split = blockIdx.y, tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int gr = lane >> 2, t4 = lane & 3;
  const int R = a.n_heads / a.n_kv_heads;
  const int key0 = split * DEC_SPLIT;
  const int nk_split = min(DEC_SPLIT, a.n_keys - key0);
  const int n_blocks = (nk_split + DEC_BLOCK - 1) / DEC_BLOCK;
  const bf16* kh = a.k + (long long)g * a.head_stride;
  const bf16* vh = a.v + (long long)g * a.head_stride;

  // the split's cache rows (except the anchor's own, written by the predecessor)
  // are in HBM already: stream them toward L2, then wait for the predecessor (PDL)
  if (tid < (nk_split + 63) / 64) {
    const int pos = key0 + tid * 64;
    const int page = a.table ? __ldg(a.table + (pos >> 6)) : (pos >> 6);
    const long long off = (long long)page * a.page_stride;
    const uint32_t bytes = (uint32_t)min(64, a.n_keys - pos) * D * 2;
    prefetch_l2(kh + off, bytes);
    prefetch_l2(vh + off, bytes);
  }
  pdl_trigger();
  pdl_wait();

  // Q as A fragments: rows 0..R-1 = the group's heads, rows >= R zero
  uint32_t qf[D / 16][4];
  {
    const bf16* qg = a.q + (long long)g * R * D;
#pragma unroll
    for (int ks = 0; ks < D / 16; ++ks) {
      const int c = ks * 16 + 2 * t4;
      qf[ks][0] = ld_b32(qg + gr * D + c, gr < R);
      qf[ks][1] = ld_b32(qg + (gr + 8) * D + c, gr + 8 < R);
      qf[ks][2] = ld_b32(qg + gr * D + c + 8, gr < R);
      qf[ks][3] = ld_b32(qg + (gr + 8) * D + c + 8, gr + 8 < R);
    }
  }
  float acc_o[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) acc_o[i][0] = acc_o[i][1] = acc_o[i][2] = acc_o[i][3] = 0.f;
  float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};

  auto row_ptr = [&](const bf16* base, int key) {
    const int page = a.table ? __ldg(a.table + (key >> 6)) : (key >> 6);
    return base + (long long)page * a.page_stride + (long long)(key & 63) * D;
  };

  for (int b = warp; b < n_blocks; b += 4) {
    const int kb = key0 + b * DEC_BLOCK;
    // K fragments (B of S = Q K^T, n = key): key kb + 8nt + gr, dims 16ks + 2t4 (+8)
    uint32_t kf[2][D / 16][2];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int key = kb + nt * 8 + gr;
      const bool ok = key < a.n_keys;
      const bf16* kr = row_ptr(kh, ok ? key : kb);
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks) {
        kf[nt][ks][0] = ld_b32(kr + ks * 16 + 2 * t4, ok);
        kf[nt][ks][1] = ld_b32(kr + ks * 16 + 8 + 2 * t4, ok);
      }
    }
    // V rows (key kb + gr and kb + 8 + gr, dims 8i + 2t4), transposed below
    uint32_t vr[D / 8][2];
    {
      const int k0 = kb + gr, k1 = kb + 8 + gr;
      const bool ok0 = k0 < a.n_keys, ok1 = k1 < a.n_keys;
      const bf16* v0 = row_ptr(vh, ok0 ? k0 : kb);
      const bf16* v1 = row_ptr(vh, ok1 ? k1 : kb);
#pragma unroll
      for (int i = 0; i < D / 8; ++i) {
        vr[i][0] = ld_b32(v0 + i * 8 + 2 * t4, ok0);
        vr[i][1] = ld_b32(v1 + i * 8 + 2 * t4, ok1);
      }
    }
    float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int ks = 0; ks < D / 16; ++ks) {
      mma_bf16_16816(s[0], qf[ks], kf[0][ks][0], kf[0][ks][1]);
      mma_bf16_16816(s[1], qf[ks], kf[1][ks][0], kf[1][ks][1]);
    }
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int kp = kb + nt * 8 + 2 * t4;
      if (kp >= a.n_keys) s[nt][0] = s[nt][2] = -INFINITY;
      if (kp + 1 >= a.n_keys) s[nt][1] = s[nt][3] = -INFINITY;
    }
    float mx[2] = {m_r[0], m_r[1]};
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      mx[0] = fmaxf(mx[0], fmaxf(s[nt][0], s[nt][1]));
      mx[1] = fmaxf(mx[1], fmaxf(s[nt][2], s[nt][3]));
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
    }
    float corr[2], msc[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      corr[r] = mx[r] == -INFINITY ? 1.f : exp2f((m_r[r] - mx[r]) * a.scale_log2);
      m_r[r] = mx[r];
      msc[r] = mx[r] == -INFINITY ? 0.f : mx[r] * a.scale_log2;
    }
    uint32_t pa[4];
    float rs[2] = {0.f, 0.f};
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const float p0 = exp2f(s[nt][0] * a.scale_log2 - msc[0]);
      const float p1 = exp2f(s[nt][1] * a.scale_log2 - msc[0]);
      const float p2 = exp2f(s[nt][2] * a.scale_log2 - msc[1]);
      const float p3 = exp2f(s[nt][3] * a.scale_log2 - msc[1]);
      rs[0] += p0 + p1;
      rs[1] += p2 + p3;
      pa[nt * 2 + 0] = pack_bf16x2(p0, p1);
      pa[nt * 2 + 1] = pack_bf16x2(p2, p3);
    }
    l_r[0] = l_r[0] * corr[0] + rs[0];
    l_r[1] = l_r[1] * corr[1] + rs[1];
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      acc_o[i][0] *= corr[0];
      acc_o[i][1] *= corr[0];
      acc_o[i][2] *= corr[1];
      acc_o[i][3] *= corr[1];
      // B of O += P V (k = key, n = dim): transpose the two 8x8 row tiles
      mma_bf16_16816(acc_o[i], pa, movm_trans(vr[i][0]), movm_trans(vr[i][1]));
    }
  }

  // ---- merge the 4 warps (rows < R only): m, l and the unnormalised O
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 1);
    l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 2);
  }
  constexpr int RS = D + 2;
  float* mine = red + warp * R * RS;
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int row = gr + 8 * half;
    if (row < R) {
#pragma unroll
      for (int i = 0; i < D / 8; ++i) {
        mine[row * RS + 2 + i * 8 + 2 * t4] = acc_o[i][2 * half];
        mine[row * RS + 2 + i * 8 + 2 * t4 + 1] = acc_o[i][2 * half + 1];
      }
      if (t4 == 0) {
        mine[row * RS] = m_r[half];
        mine[row * RS + 1] = l_r[half];
      }
    }
  }
  __syncthreads();
  for (int idx = tid; idx < R * D; idx += DEC_THREADS) {
    const int r = idx / D, d = idx % D, h = g * R + r;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) M = fmaxf(M, red[(w * R + r) * RS]);
    float o = 0.f, lsum = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float mw = red[(w * R + r) * RS];
      const float wt = mw == -INFINITY ? 0.f : exp2f((mw - M) * a.scale_log2);
      o += wt * red[(w * R + r) * RS + 2 + d];
      lsum += wt * red[(w * R + r) * RS + 1];
    }
    a.part_o[((long long)h * a.splits + split) * D + d] = o;
    if (d == 0) {
      a.part_ml[((long long)h * a.splits + split) * 2] = M * a.scale_log2;  // log2 domain
      a.part_ml[((long long)h * a.splits + split) * 2 + 1] = lsum;
    }
  }
  // ---- the last CTA of this kv head merges every split (threadfence reduction)
  __threadfence();
  __syncthreads();
  if (tid == 0) is_last = (atomicAdd(a.counters + g, 1u) == (unsigned)a.splits - 1);
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  float* wts = red;  // [R][splits] then den[R]
  float* den = wts + R * a.splits;
  for (int r = warp; r < R; r += DEC_THREADS / 32) {
    const float* ml = a.part_ml + (long long)(g * R + r) * a.splits * 2;
    float M = -INFINITY;
    for (int s2 = lane; s2 < a.splits; s2 += 32) M = fmaxf(M, __ldcg(ml + 2 * s2));
#pragma unroll
    for (int off = 16; off; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
    float dn = 0.f;
    for (int s2 = lane; s2 < a.splits; s2 += 32) {
      const float w = exp2f(__ldcg(ml + 2 * s2) - M);
      wts[r * a.splits + s2] = w;
      dn += w * __ldcg(ml + 2 * s2 + 1);
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
    for (int s2 = 0; s2 < a.splits; ++s2) num = fmaf(wts[r * a.splits + s2], __ldcg(po + (long long)s2 * D), num);
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
  // shared memory: the 4-warp merge [4][R][D+2], reused for the split merge [R][splits] + [R]
  int smem = 4 * R * (head_dim + 2) * 4;
  const int merge = (R * splits + R) * 4;
  if (merge > smem) smem = merge;
  if (smem > 200 * 1024) return DS_ERR_INVALID;
  DecArgs a{q, k_layer, v_layer, head_stride, page_stride, table, n_keys, n_heads, n_kv_heads, head_dim, splits,
            part_o, part_ml, counters, out, (float)(1.4426950408889634 / sqrt((double)head_dim))};
  count_launch();
  cudaError_t e;
  static const bool c0 = prefer_max_smem(decode_attn_kernel<128>) && prefer_max_smem(decode_attn_kernel<64>);
  (void)c0;
  if (head_dim == 128) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(decode_attn_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    e = launch_pdl(decode_attn_kernel<128>, dim3(n_kv_heads, splits), dim3(DEC_THREADS), smem, stream, a);
  } else {
    if (smem > 48 * 1024) cudaFuncSetAttribute(decode_attn_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    e = launch_pdl(decode_attn_kernel<64>, dim3(n_kv_heads, splits), dim3(DEC_THREADS), smem, stream, a);
  }
  return launch_status(e);
}

}  // namespace ds
