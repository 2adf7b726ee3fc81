// Causal GQA flash-attention prefill over a (paged) KV cache layer.
//
// Semantics: _masked_attention over the window (model.py:506-519): head h
// reads kv head h / (H/KVH); scores scaled by 1/sqrt(D) after the dot product;
// query at absolute position p sees keys 0..p; max-subtracted softmax; output
// head-major [rows][H*D].  Online softmax in fp32 (exp2 with the scale folded
// in), P rounded to bf16 for the P.V product, output rounded to bf16.
//
// Tiling: CTA = 4 warps = 64 query rows of one head; key tiles of 64 = one KV
// page (a contiguous 64 x D block), double-buffered with cp.async; bf16
// m16n8k16 tensor-core MMAs with ldmatrix from XOR-swizzled shared memory.
// Blocks are launched heaviest (latest positions) first.
#include "common.cuh"
#include "kernels.h"

namespace ds {

struct FaArgs {
  const bf16* q;
  long long ldq;
  bf16* o;
  long long ldo;
  const bf16* k;  // layer base
  const bf16* v;
  long long head_stride, page_stride;
  const int32_t* table;
  int n_q, q_pos0, n_heads, n_kv_heads;
  float scale_log2;  // log2(e) / sqrt(D)
};

DS_DEV void cp_async16(uint32_t dst, const void* src, bool valid) {
  int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n) : "memory");
}
DS_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
DS_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
DS_DEV void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
DS_DEV void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
DS_DEV void mma_bf16_16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// byte offset of 16-byte chunk c of row r in a swizzled [rows][D] bf16 tile
template <int D>
DS_DEV uint32_t swz(int r, int c) {
  return (uint32_t)(r * D * 2 + ((c ^ (r & 7)) << 4));
}

template <int D>
DS_DEV void load_tile(uint32_t sbase, const bf16* gbase, int valid_rows, int tid) {
  constexpr int CH = D / 8;  // 16-byte chunks per row
#pragma unroll
  for (int i = tid; i < 64 * CH; i += 128) {
    const int r = i / CH, c = i % CH;
    const bool ok = r < valid_rows;
    cp_async16(sbase + swz<D>(r, c), gbase + (ok ? (long long)r * D + c * 8 : 0), ok);
  }
}

template <int D>
__global__ void __launch_bounds__(128) fa_prefill_kernel(FaArgs a) {
  constexpr int TILE = 64 * D * 2;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sQ = smem_u32(smem);
  const uint32_t sK0 = sQ + TILE;
  const uint32_t sV0 = sQ + 3 * TILE;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int h = blockIdx.x;
  const int nmb = gridDim.y;
  const int mb = nmb - 1 - blockIdx.y;
  const int q0 = mb * 64;
  const int kvh = h / (a.n_heads / a.n_kv_heads);
  const int rows = min(64, a.n_q - q0);
  const int max_key = a.q_pos0 + q0 + rows - 1;  // last key any row of this block sees
  const int n_kt = max_key / 64 + 1;

  const bf16* qg = a.q + (long long)q0 * a.ldq + (long long)h * D;
  // Q: rows may be strided (ldq); load chunk by chunk
  {
    constexpr int CH = D / 8;
    for (int i = tid; i < 64 * CH; i += 128) {
      const int r = i / CH, c = i % CH;
      const bool ok = r < rows;
      cp_async16(sQ + swz<D>(r, c), qg + (ok ? (long long)r * a.ldq + c * 8 : 0), ok);
    }
  }
  auto kv_tile = [&](int kt, int buf) {
    const int page = a.table ? __ldg(a.table + kt) : kt;
    const long long off = (long long)kvh * a.head_stride + (long long)page * a.page_stride;
    const int valid = min(64, max_key - kt * 64 + 1);
    load_tile<D>(sK0 + buf * TILE, a.k + off, valid, tid);
    load_tile<D>(sV0 + buf * TILE, a.v + off, valid, tid);
  };
  kv_tile(0, 0);
  cp_async_commit();

  uint32_t qf[D / 16][4];
  float acc_o[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) acc_o[i][0] = acc_o[i][1] = acc_o[i][2] = acc_o[i][3] = 0.f;
  float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};
  const int g = lane >> 2, t4 = lane & 3;
  const int qpos0 = a.q_pos0 + q0 + warp * 16 + g;  // row g; row g+8 is qpos0 + 8

  for (int kt = 0; kt < n_kt; ++kt) {
    if (kt + 1 < n_kt) kv_tile(kt + 1, (kt + 1) & 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (kt == 0) {
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks) {
        const int r = warp * 16 + (lane & 15);
        const int c = ks * 2 + (lane >> 4);
        ldsm_x4(sQ + swz<D>(r, c), qf[ks][0], qf[ks][1], qf[ks][2], qf[ks][3]);
      }
    }
    const uint32_t sK = sK0 + (kt & 1) * TILE, sV = sV0 + (kt & 1) * TILE;
    float s[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < D / 16; ++ks) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t b0, b1, b2, b3;
        const int r = j * 16 + (lane & 7) + ((lane >> 4) << 3);
        const int c = ks * 2 + ((lane >> 3) & 1);
        ldsm_x4(sK + swz<D>(r, c), b0, b1, b2, b3);
        mma_bf16_16816(s[2 * j], qf[ks], b0, b1);
        mma_bf16_16816(s[2 * j + 1], qf[ks], b2, b3);
      }
    }
    // causal mask (only tiles that reach past this warp's first row)
    if (kt * 64 + 63 > qpos0 - g) {
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        const int kp = kt * 64 + nt * 8 + 2 * t4;
        if (kp > qpos0) s[nt][0] = -INFINITY;
        if (kp + 1 > qpos0) s[nt][1] = -INFINITY;
        if (kp > qpos0 + 8) s[nt][2] = -INFINITY;
        if (kp + 1 > qpos0 + 8) s[nt][3] = -INFINITY;
      }
    }
    // online softmax (two rows per thread: r=0 -> g, r=1 -> g+8)
    float mx[2] = {m_r[0], m_r[1]};
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      mx[0] = fmaxf(mx[0], fmaxf(s[nt][0], s[nt][1]));
      mx[1] = fmaxf(mx[1], fmaxf(s[nt][2], s[nt][3]));
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
    }
    float corr[2], msc[2], rs[2] = {0.f, 0.f};
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      corr[r] = exp2f((m_r[r] - mx[r]) * a.scale_log2);
      m_r[r] = mx[r];
      msc[r] = mx[r] * a.scale_log2;
    }
    uint32_t pa[4][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const float p0 = exp2f(s[nt][0] * a.scale_log2 - msc[0]);
      const float p1 = exp2f(s[nt][1] * a.scale_log2 - msc[0]);
      const float p2 = exp2f(s[nt][2] * a.scale_log2 - msc[1]);
      const float p3 = exp2f(s[nt][3] * a.scale_log2 - msc[1]);
      rs[0] += p0 + p1;
      rs[1] += p2 + p3;
      pa[nt >> 1][(nt & 1) * 2 + 0] = pack_bf16x2(p0, p1);
      pa[nt >> 1][(nt & 1) * 2 + 1] = pack_bf16x2(p2, p3);
    }
    l_r[0] = l_r[0] * corr[0] + rs[0];
    l_r[1] = l_r[1] * corr[1] + rs[1];
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      acc_o[i][0] *= corr[0];
      acc_o[i][1] *= corr[0];
      acc_o[i][2] *= corr[1];
      acc_o[i][3] *= corr[1];
    }
    // O += P V   (k-step j = keys 16j..16j+15)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t af[4] = {pa[j][0], pa[j][1], pa[j][2], pa[j][3]};
#pragma unroll
      for (int i = 0; i < D / 16; ++i) {
        uint32_t b0, b1, b2, b3;
        const int r = j * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
        const int c = i * 2 + (lane >> 4);
        ldsm_x4_t(sV + swz<D>(r, c), b0, b1, b2, b3);
        mma_bf16_16816(acc_o[2 * i], af, b0, b1);
        mma_bf16_16816(acc_o[2 * i + 1], af, b2, b3);
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();

  // finalize: quad-reduce row sums, normalise, stage bf16 tile in smem (reuse Q)
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 1);
    l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 2);
  }
  const float inv0 = 1.f / l_r[0], inv1 = 1.f / l_r[1];
  uint8_t* sO = smem;
#pragma unroll
  for (int i = 0; i < D / 8; ++i) {
    const int col = i * 8 + 2 * t4;
    const int r0 = warp * 16 + g, r1 = r0 + 8;
    *reinterpret_cast<uint32_t*>(sO + swz<D>(r0, col >> 3) + (col & 7) * 2) =
        pack_bf16x2(acc_o[i][0] * inv0, acc_o[i][1] * inv0);
    *reinterpret_cast<uint32_t*>(sO + swz<D>(r1, col >> 3) + (col & 7) * 2) =
        pack_bf16x2(acc_o[i][2] * inv1, acc_o[i][3] * inv1);
  }
  __syncthreads();
  constexpr int CH = D / 8;
  bf16* og = a.o + (long long)q0 * a.ldo + (long long)h * D;
  for (int i = tid; i < 64 * CH; i += 128) {
    const int r = i / CH, c = i % CH;
    if (r < rows)
      *reinterpret_cast<uint4*>(og + (long long)r * a.ldo + c * 8) =
          *reinterpret_cast<const uint4*>(sO + swz<D>(r, c));
  }
}

int attention_prefill_launch(const bf16* q, long long ldq, const bf16* k_layer, const bf16* v_layer,
                             long long head_stride, long long page_stride, const int32_t* table, int n_q, int q_pos0,
                             int n_heads, int n_kv_heads, int head_dim, bf16* o, long long ldo, cudaStream_t stream) {
  if (n_q <= 0) return DS_OK;
  FaArgs a{q, ldq, o, ldo, k_layer, v_layer, head_stride, page_stride, table, n_q, q_pos0, n_heads, n_kv_heads,
           (float)(1.4426950408889634 / sqrt((double)head_dim))};
  dim3 grid(n_heads, (n_q + 63) / 64);
  count_launch();
  if (head_dim == 128) {
    const int smem = 5 * 64 * 128 * 2;
    static bool set = false;
    if (!set) {
      cudaFuncSetAttribute(fa_prefill_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      set = true;
    }
    fa_prefill_kernel<128><<<grid, 128, smem, stream>>>(a);
  } else if (head_dim == 64) {
    const int smem = 5 * 64 * 64 * 2;
    fa_prefill_kernel<64><<<grid, 128, smem, stream>>>(a);
  } else {
    return DS_ERR_INVALID;
  }
  return cudaGetLastError() == cudaSuccess ? DS_OK : DS_ERR_CUDA;
}

}  // namespace ds
