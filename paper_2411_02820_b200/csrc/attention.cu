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
#include <stdlib.h>

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

int attention_prefill_legacy_launch(const bf16* q, long long ldq, const bf16* k_layer, const bf16* v_layer,
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

// ======================================================================
// tcgen05 / TMEM flash-attention prefill (sm_100a)
//
// CTA = one head x 256 query rows = two 128-row Q tiles (TMEM lanes = rows).
// Warp roles (320 threads):
//   warp 0     TMA producer: Q tiles once; K and V tiles of 128 keys (= two
//              64-position pages, block-table addressed) through 2-stage rings
//   warp 1     TMEM allocator + single-thread tcgen05.mma issuer:
//                S_i = Q_i K_j^T   (SS, M=128 N=128 K=D)    -> TMEM cols S_i
//                O_i += P_i V_j    (TS: P from TMEM, V MN-major smem, N=D) -> cols O_i
//              ping-ponging the two Q tiles so one tile's softmax overlaps the
//              other tile's MMAs
//   warps 2-5  softmax of Q tile 0 (thread = row), warps 6-9 of tile 1:
//              tcgen05.ld S row, causal mask, online max with lazy O rescale
//              (only when the max grows by > 2^8; exact after the final 1/l),
//              p = exp2, P as bf16 written back into TMEM over S, l in fp32;
//              epilogue O / l -> bf16 -> global
// TMEM: S0 [0,128) S1 [128,256) O0 [256,256+D) O1 [384,384+D).
// ======================================================================

constexpr int FA_BM = 128;
constexpr int FA_BN = 128;
constexpr int FA_THREADS = 320;

template <int D>
struct FaTcSmem {
  static constexpr int CH = D / 64;
  static constexpr uint32_t CHUNK = FA_BM * 64 * 2;  // [128][64] bf16, SW128
  static constexpr uint32_t Q = 0;
  static constexpr uint32_t K = Q + 2 * CH * CHUNK;
  static constexpr uint32_t V = K + 2 * CH * CHUNK;
  static constexpr uint32_t BAR = V + 2 * CH * CHUNK;
  static constexpr uint32_t TOTAL = BAR + 256 + 1024;
};

struct FaTcArgs {
  int n_q, q_pos0, n_heads, n_kv_heads;
  long long k_head_rows, k_page_rows;
  const int32_t* table;
  bf16* o;
  long long ldo;
  float scale_log2;
};

template <int D>
__global__ void __launch_bounds__(FA_THREADS, 1)
    fa_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                 const __grid_constant__ CUtensorMap tmV, FaTcArgs a) {
  using L = FaTcSmem<D>;
  constexpr int CH = L::CH;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* k_empty = bars + 3;
  uint64_t* v_full = bars + 5;
  uint64_t* v_empty = bars + 7;
  uint64_t* s_full = bars + 9;
  uint64_t* p_full = bars + 11;
  uint64_t* o_done = bars + 13;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);
  auto sQ = [&](int i, int c) { return smem + L::Q + (i * CH + c) * L::CHUNK; };
  auto sK = [&](int st, int c) { return smem + L::K + (st * CH + c) * L::CHUNK; };
  auto sV = [&](int st, int c) { return smem + L::V + (st * CH + c) * L::CHUNK; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = blockIdx.x;
  const int q0 = (gridDim.y - 1 - blockIdx.y) * 2 * FA_BM;  // heaviest (latest) blocks first
  const int g = h / (a.n_heads / a.n_kv_heads);
  int n_kv[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int rows = min(FA_BM, a.n_q - (q0 + i * FA_BM));
    n_kv[i] = rows > 0 ? (a.q_pos0 + q0 + i * FA_BM + rows - 1) / FA_BN + 1 : 0;
  }
  const int J = max(n_kv[0], n_kv[1]);
  const int max_key = a.q_pos0 + min(q0 + 2 * FA_BM, a.n_q) - 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
      mbar_init(&o_done[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const int n_tiles = n_kv[1] > 0 ? 2 : 1;
      mbar_expect_tx(q_full, n_tiles * CH * L::CHUNK);
      for (int i = 0; i < n_tiles; ++i)
        for (int c = 0; c < CH; ++c) tma_load_2d(sQ(i, c), &tmQ, q_full, h * D + c * 64, q0 + i * FA_BM);
      for (int j = 0; j < J; ++j) {
        const int st = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        int rows[2];
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          int page = 2 * j + p;
          if (page * 64 > max_key) page = 2 * j;  // beyond the window: duplicate a valid page (finite, masked)
          const int tp = a.table ? __ldg(a.table + page) : page;
          rows[p] = (int)(g * a.k_head_rows + (long long)tp * a.k_page_rows);
        }
        mbar_wait(&k_empty[st], ph ^ 1);
        mbar_expect_tx(&k_full[st], CH * L::CHUNK);
        for (int p = 0; p < 2; ++p)
          for (int c = 0; c < CH; ++c) tma_load_2d(sK(st, c) + p * 64 * 128, &tmK, &k_full[st], c * 64, rows[p]);
        mbar_wait(&v_empty[st], ph ^ 1);
        mbar_expect_tx(&v_full[st], CH * L::CHUNK);
        for (int p = 0; p < 2; ++p)
          for (int c = 0; c < CH; ++c) tma_load_2d(sV(st, c) + p * 64 * 128, &tmV, &v_full[st], c * 64, rows[p]);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t IDESC_QK = umma_idesc_bf16(FA_BM, FA_BN);
    constexpr uint32_t IDESC_PV = umma_idesc_bf16_bmn(FA_BM, D);
    auto qk = [&](int i, int st) {
      if (lane == 0) {
#pragma unroll
        for (int c = 0; c < CH; ++c)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t ad = sdesc_sw128(smem_u32(sQ(i, c)) + k * 32, 16, 1024);
            const uint64_t bd = sdesc_sw128(smem_u32(sK(st, c)) + k * 32, 16, 1024);
            umma_bf16(tmem + i * 128, ad, bd, IDESC_QK, (c | k) != 0 ? 1u : 0u);
          }
        umma_commit(&s_full[i]);
      }
      __syncwarp();
    };
    auto pv = [&](int i, int st, int j) {
      if (lane == 0) {
#pragma unroll
        for (int s = 0; s < FA_BN / 16; ++s) {
          const uint64_t bd = sdesc_sw128(smem_u32(sV(st, 0)) + s * 2048, L::CHUNK, 1024);
          umma_bf16_ts(tmem + 256 + i * 128, tmem + i * 128 + s * 8, bd, IDESC_PV, (j | s) != 0 ? 1u : 0u);
        }
        umma_commit(&o_done[i]);
      }
      __syncwarp();
    };
    mbar_wait(q_full, 0);
    mbar_wait(&k_full[0], 0);
    tc_fence_after();
    if (n_kv[0] > 0) qk(0, 0);
    if (n_kv[1] > 0) qk(1, 0);
    if (lane == 0) umma_commit(&k_empty[0]);
    __syncwarp();
    for (int j = 0; j < J; ++j) {
      const int st = j & 1, st1 = (j + 1) & 1;
      const bool more = j + 1 < J;
      mbar_wait(&v_full[st], (j >> 1) & 1);
      tc_fence_after();
      if (j * FA_BN + FA_BN - 1 > max_key) {
        // keys past the window end: zero their V rows so p = 0 never meets a
        // non-finite cache value (a SW128 row's 128 bytes stay within the row)
        const int first = max_key + 1 - j * FA_BN;
        for (int c = 0; c < CH; ++c) {
          const uint32_t base = smem_u32(sV(st, c));
          for (int off = first * 128 + lane * 16; off < FA_BN * 128; off += 32 * 16)
            asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(base + off), "r"(0u) : "memory");
        }
        fence_async_shared();
        __syncwarp();
      }
      if (j < n_kv[0]) {
        mbar_wait(&p_full[0], j & 1);
        tc_fence_after();
        pv(0, st, j);
      }
      if (more) {
        mbar_wait(&k_full[st1], ((j + 1) >> 1) & 1);
        tc_fence_after();
        if (j + 1 < n_kv[0]) qk(0, st1);
      }
      if (j < n_kv[1]) {
        mbar_wait(&p_full[1], j & 1);
        tc_fence_after();
        pv(1, st, j);
      }
      if (lane == 0) umma_commit(&v_empty[st]);
      __syncwarp();
      if (more) {
        if (j + 1 < n_kv[1]) qk(1, st1);
        if (lane == 0) umma_commit(&k_empty[st1]);
        __syncwarp();
      }
    }
  } else {
    const int i = (warp - 2) >> 2;  // Q tile
    const int quarter = warp & 3;   // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;
    const int tile_pos0 = a.q_pos0 + q0 + i * FA_BM;
    const int qpos = tile_pos0 + row;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t tS = tmem + lane_base + i * 128;
    const uint32_t tO = tmem + lane_base + 256 + i * 128;
    const float sc = a.scale_log2;
    const float thr = 8.0f / sc;
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < n_kv[i]; ++j) {
      mbar_wait(&s_full[i], j & 1);
      tc_fence_after();
      uint32_t sr[FA_BN];
#pragma unroll
      for (int c = 0; c < FA_BN / 32; ++c) tmem_ld32_nowait(tS + c * 32, sr + c * 32);
      tmem_wait_ld();
      const int kbase = j * FA_BN;
      if (kbase + FA_BN - 1 > tile_pos0) {
#pragma unroll
        for (int c = 0; c < FA_BN; ++c)
          if (kbase + c > qpos) sr[c] = __float_as_uint(-INFINITY);
      }
      float mt = -INFINITY;
#pragma unroll
      for (int c = 0; c < FA_BN; ++c) mt = fmaxf(mt, __uint_as_float(sr[c]));
      const bool need = mt > m_used + thr;
      float corr = 1.f;
      if (need) {
        corr = fast_exp2((m_used - mt) * sc);
        m_used = mt;
      }
      l *= corr;
      if (j > 0 && __any_sync(0xffffffffu, need)) {
        mbar_wait(&o_done[i], (j - 1) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < D / 32; ++c) {
          uint32_t orow[32];
          tmem_ld32_nowait(tO + c * 32, orow);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) orow[e] = __float_as_uint(__uint_as_float(orow[e]) * corr);
          tmem_st32_nowait(tO + c * 32, orow);
        }
        tmem_wait_st();
      }
      const float msc = m_used * sc;
      float sum = 0.f;
      uint32_t pk[FA_BN / 2];
#pragma unroll
      for (int c = 0; c < FA_BN / 2; ++c) {
        const float p0 = fast_exp2(fmaf(__uint_as_float(sr[2 * c]), sc, -msc));
        const float p1 = fast_exp2(fmaf(__uint_as_float(sr[2 * c + 1]), sc, -msc));
        sum += p0 + p1;
        pk[c] = pack_bf16x2(p0, p1);
      }
      l += sum;
      tmem_st32_nowait(tS, pk);
      tmem_st32_nowait(tS + 32, pk + 32);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[i]);
    }
    if (n_kv[i] > 0) {
      mbar_wait(&o_done[i], (n_kv[i] - 1) & 1);
      tc_fence_after();
      const float inv = 1.f / l;
      const int qrow = q0 + i * FA_BM + row;
      bf16* dst = a.o + (long long)qrow * a.ldo + (long long)h * D;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        uint32_t orow[32];
        tmem_ld32_nowait(tO + c * 32, orow);
        tmem_wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e)
          pk[e] = pack_bf16x2(__uint_as_float(orow[2 * e]) * inv, __uint_as_float(orow[2 * e + 1]) * inv);
        if (qrow < a.n_q) {
#pragma unroll
          for (int e = 0; e < 4; ++e) st_global_v4(dst + c * 32 + e * 8, pk[4 * e], pk[4 * e + 1], pk[4 * e + 2], pk[4 * e + 3]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int D>
static int fa_tc_launch(const bf16* q, long long ldq, const bf16* k_layer, const bf16* v_layer, long long head_stride,
                        long long page_stride, long long layer_rows, const int32_t* table, int n_q, int q_pos0,
                        int n_heads, int n_kv_heads, bf16* o, long long ldo, cudaStream_t stream) {
  using L = FaTcSmem<D>;
  CUtensorMap tq, tk, tv;
  if (make_tmap_bf16(&tq, q, n_q, (long long)n_heads * D, ldq, FA_BM, 64)) return DS_ERR_CUDA;
  if (make_tmap_bf16(&tk, k_layer, layer_rows, D, D, 64, 64)) return DS_ERR_CUDA;
  if (make_tmap_bf16(&tv, v_layer, layer_rows, D, D, 64, 64)) return DS_ERR_CUDA;
  FaTcArgs a{n_q, q_pos0, n_heads, n_kv_heads, head_stride / D, page_stride / D, table, o, ldo,
             (float)(1.4426950408889634 / sqrt((double)D))};
  static bool set = false;
  if (!set) {
    if (cudaFuncSetAttribute(fa_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL) != cudaSuccess)
      return DS_ERR_CUDA;
    set = true;
  }
  dim3 grid(n_heads, (n_q + 2 * FA_BM - 1) / (2 * FA_BM));
  count_launch();
  fa_tc_kernel<D><<<grid, FA_THREADS, L::TOTAL, stream>>>(tq, tk, tv, a);
  return cudaGetLastError() == cudaSuccess ? DS_OK : DS_ERR_CUDA;
}

int attention_prefill_launch(const bf16* q, long long ldq, const bf16* k_layer, const bf16* v_layer,
                             long long head_stride, long long page_stride, long long layer_rows, const int32_t* table,
                             int n_q, int q_pos0, int n_heads, int n_kv_heads, int head_dim, bf16* o, long long ldo,
                             cudaStream_t stream) {
  if (n_q <= 0) return DS_OK;
  static const bool legacy = getenv("DS_FA_LEGACY") != nullptr;
  if (legacy)
    return attention_prefill_legacy_launch(q, ldq, k_layer, v_layer, head_stride, page_stride, table, n_q, q_pos0,
                                           n_heads, n_kv_heads, head_dim, o, ldo, stream);
  if (head_dim == 128)
    return fa_tc_launch<128>(q, ldq, k_layer, v_layer, head_stride, page_stride, layer_rows, table, n_q, q_pos0,
                             n_heads, n_kv_heads, o, ldo, stream);
  if (head_dim == 64)
    return fa_tc_launch<64>(q, ldq, k_layer, v_layer, head_stride, page_stride, layer_rows, table, n_q, q_pos0,
                            n_heads, n_kv_heads, o, ldo, stream);
  return DS_ERR_INVALID;
}

}  // namespace ds
