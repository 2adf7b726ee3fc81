// Row RMSNorm (model.py:466-468) producing the bf16 GEMM operand, optionally
// gathering rows (token-embedding lookup, model.py:609/629) and emitting f32 /
// bf16 copies of the input rows (the bf16 copy only for rows < copy_rows) (the residual stream seed, and the producer's
// E-cache export, model.py:620-621).
#include "common.cuh"
#include "kernels.h"

namespace ds {

constexpr int NORM_THREADS = 256;

template <bool IN_BF16>
DS_DEV void load8(const void* x, long long idx, float* v) {
  if (IN_BF16) {
    uint4 u = *reinterpret_cast<const uint4*>(reinterpret_cast<const bf16*>(x) + idx);
    float2 a = unpack_bf16x2(u.x), b = unpack_bf16x2(u.y), c = unpack_bf16x2(u.z), d = unpack_bf16x2(u.w);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y; v[4] = c.x; v[5] = c.y; v[6] = d.x; v[7] = d.y;
  } else {
    const float4* p = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(x) + idx);
    float4 a = p[0], b = p[1];
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
}

// One CTA per row.  Rows up to NORM_THREADS * 8 * NORM_REG values are read
// once into registers (sum of squares, then scale from registers); longer rows
// take a second (L2-resident) pass.
constexpr int NORM_REG = 4;

template <bool IN_BF16>
__global__ void __launch_bounds__(NORM_THREADS) rmsnorm_kernel(const void* x, const int64_t* gather, int d,
                                                               const float* gain, bf16* out, float* copy_f32,
                                                               bf16* copy_bf16, int copy_rows) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  const long long src = gather ? (long long)__ldg(gather + r) : (long long)r;
  const long long base = src * d;
  const bool in_regs = d <= NORM_THREADS * 8 * NORM_REG;
  float v[NORM_REG][8];
  float ss = 0.f;
  if (in_regs) {
#pragma unroll
    for (int i = 0; i < NORM_REG; ++i) {
      const int c = (threadIdx.x + i * NORM_THREADS) * 8;
      if (c < d) {
        load8<IN_BF16>(x, base + c, v[i]);
#pragma unroll
        for (int e = 0; e < 8; ++e) ss += v[i][e] * v[i][e];
      }
    }
  } else {
    for (int c = threadIdx.x * 8; c < d; c += NORM_THREADS * 8) {
      float t[8];
      load8<IN_BF16>(x, base + c, t);
#pragma unroll
      for (int e = 0; e < 8; ++e) ss += t[e] * t[e];
    }
  }
  __shared__ float red[NORM_THREADS / 32];
#pragma unroll
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < NORM_THREADS / 32 ? red[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const float inv = 1.0f / sqrtf(red[0] / (float)d + 1e-6f);
  const long long obase = (long long)r * d;
  auto emit = [&](int c, const float* w) {
    const float4 g0 = *reinterpret_cast<const float4*>(gain + c);
    const float4 g1 = *reinterpret_cast<const float4*>(gain + c + 4);
    const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
    uint32_t p[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) p[i] = pack_bf16x2(w[2 * i] * inv * g[2 * i], w[2 * i + 1] * inv * g[2 * i + 1]);
    *reinterpret_cast<uint4*>(out + obase + c) = make_uint4(p[0], p[1], p[2], p[3]);
    if (copy_f32) {
      float4* o = reinterpret_cast<float4*>(copy_f32 + obase + c);
      o[0] = make_float4(w[0], w[1], w[2], w[3]);
      o[1] = make_float4(w[4], w[5], w[6], w[7]);
    }
    if (copy_bf16 && r < copy_rows) {
      uint32_t q[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) q[i] = pack_bf16x2(w[2 * i], w[2 * i + 1]);
      *reinterpret_cast<uint4*>(copy_bf16 + obase + c) = make_uint4(q[0], q[1], q[2], q[3]);
    }
  };
  if (in_regs) {
#pragma unroll
    for (int i = 0; i < NORM_REG; ++i) {
      const int c = (threadIdx.x + i * NORM_THREADS) * 8;
      if (c < d) emit(c, v[i]);
    }
  } else {
    for (int c = threadIdx.x * 8; c < d; c += NORM_THREADS * 8) {
      float t[8];
      load8<IN_BF16>(x, base + c, t);
      emit(c, t);
    }
  }
}

// Group seed in the folded-RMSNorm format (see GemmEpi::norm_out / ssq_in): for
// row r and column tile p (T columns), a[r][c] = bf16(x[r][c] * g[c]), the
// f32 row copy, and ssq[p * ld + r] = fmaf-sum of x^2 over the tile's columns
// in ascending order -- exactly what a residual GEMM epilogue writes, so a
// group's first layer sees the same operand as a layer inside a group.
// One CTA per row, 16 columns per thread (coalesced); a tile's T/16 threads
// are adjacent lanes of one warp and pass the running sum along in order.
template <bool IN_BF16>
__global__ void __launch_bounds__(1024) norm_seed_kernel(const void* x, const int64_t* gather, int d, int T,
                                                         const float* gain, bf16* out, float* copy_f32, float* ssq,
                                                         long long ld) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x, i = threadIdx.x;
  const int tpp = T / 16, p = i / tpp, j = i - p * tpp;
  const long long src = gather ? (long long)__ldg(gather + r) : (long long)r;
  const int c = i * 16;
  float v[16];
  load8<IN_BF16>(x, src * d + c, v);
  load8<IN_BF16>(x, src * d + c + 8, v + 8);
  uint32_t q[8];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float4 g = __ldg(reinterpret_cast<const float4*>(gain + c) + e);
    q[2 * e] = pack_bf16x2(v[4 * e] * g.x, v[4 * e + 1] * g.y);
    q[2 * e + 1] = pack_bf16x2(v[4 * e + 2] * g.z, v[4 * e + 3] * g.w);
  }
  uint4* o = reinterpret_cast<uint4*>(out + (long long)r * d + c);
  o[0] = make_uint4(q[0], q[1], q[2], q[3]);
  o[1] = make_uint4(q[4], q[5], q[6], q[7]);
  if (copy_f32) {
    float4* h = reinterpret_cast<float4*>(copy_f32 + (long long)r * d + c);
#pragma unroll
    for (int e = 0; e < 4; ++e) h[e] = make_float4(v[4 * e], v[4 * e + 1], v[4 * e + 2], v[4 * e + 3]);
  }
  // the tile's sum of squares in ascending column order: lane j continues lane j-1's sum
  const int lane = threadIdx.x & 31, first = lane - j;
  float ss = 0.f;
  for (int st = 0; st < tpp; ++st) {
    if (j == st) {
#pragma unroll
      for (int e = 0; e < 16; ++e) ss = fmaf(v[e], v[e], ss);
    }
    ss = __shfl_sync(0xffffffffu, ss, first + st);
  }
  if (j == 0) ssq[p * ld + r] = ss;
}

int norm_seed_launch(const void* x, bool x_bf16, const int64_t* gather, int M, int d, int T, const float* gain,
                     bf16* out, float* copy_f32, float* ssq, long long ld, cudaStream_t stream) {
  if (M <= 0) return DS_OK;
  if (T < 16 || T > 512 || T % 16 || d % T || d / 16 > 1024 || (32 % (T / 16) && (T / 16) % 32)) return DS_ERR_INVALID;
  count_launch();
  static PerDevice carve_t, carve_f;
  prefer_max_smem_once(norm_seed_kernel<true>, carve_t);
  prefer_max_smem_once(norm_seed_kernel<false>, carve_f);
  const dim3 block(d / 16);
  if (x_bf16)
    return launch_status(launch_pdl(norm_seed_kernel<true>, dim3(M), block, 0, stream, x, gather, d, T, gain, out,
                                    copy_f32, ssq, ld));
  return launch_status(launch_pdl(norm_seed_kernel<false>, dim3(M), block, 0, stream, x, gather, d, T, gain, out,
                                  copy_f32, ssq, ld));
}

int rmsnorm_launch(const void* x, bool x_bf16, const int64_t* gather, int M, int d, const float* gain, bf16* out,
                   float* copy_f32, bf16* copy_bf16, int copy_rows, cudaStream_t stream) {
  if (M <= 0) return DS_OK;
  count_launch();
  static PerDevice carve_t, carve_f;
  prefer_max_smem_once(rmsnorm_kernel<true>, carve_t);
  prefer_max_smem_once(rmsnorm_kernel<false>, carve_f);
  if (x_bf16)
    return launch_status(launch_pdl(rmsnorm_kernel<true>, dim3(M), dim3(NORM_THREADS), 0, stream, x, gather, d, gain,
                                    out, copy_f32, copy_bf16, copy_rows));
  return launch_status(launch_pdl(rmsnorm_kernel<false>, dim3(M), dim3(NORM_THREADS), 0, stream, x, gather, d, gain,
                                  out, copy_f32, copy_bf16, copy_rows));
}

}  // namespace ds
