// Persistent warp-specialised tcgen05 GEMM for sm_100a with fused epilogues.
//
//   C[M,N] = A[M,K] . B[N,K]^T      A = activations (bf16, K-major)
//                                   B = weights     (bf16, K-major: the reference
//                                       [in,out] matrices transposed once at load)
//
// Roles (192 threads, 1 CTA per SM):
//   warp 0      TMA producer: A 128x64 and B BNx64 tiles, SWIZZLE_128B, STAGES-deep ring
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN, K=16)
//   warps 2..5  epilogue: tcgen05.ld accumulator rows -> fused epilogue -> global
// Two TMEM accumulators (2*BN columns) let the epilogue of tile i overlap the
// MMAs of tile i+1.
//
// Epilogues (the reference block math, model.py:522-544):
//   EPI_QKV_ROPE  q/k rotate-half RoPE (model.py:475-488) in fp32; q -> bf16 buffer,
//                 k/v -> bf16 KV cache through KvAddr (paged or dense export layout)
//   EPI_RESID_F32 out = resid + acc                (x = h + attn@wo, out = x + mlp)
//   EPI_SILU_BF16 out = bf16(silu(acc))            (silu(rms(x)*g @ w1))
//   EPI_SWIGLU_BF16 out = bf16(silu(gate) * up)    (Llama-3 MLP, interleaved gate/up columns)
//   EPI_STORE_*   plain stores (tests / lm head)
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"

namespace ds {

constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 64;
constexpr int GEMM_THREADS = 192;

template <int BN, int STAGES>
struct GemmSmem {
  static constexpr uint32_t A_BYTES = GEMM_BM * GEMM_BK * 2;
  static constexpr uint32_t B_BYTES = BN * GEMM_BK * 2;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t BAR_BYTES = (2 * STAGES + 4) * 8 + 16;
  static constexpr uint32_t TOTAL = 1024 + STAGES * STAGE_BYTES + BAR_BYTES;
};

DS_DEV void tile_coords(int t, int num_m, int num_n, int group, int& mb, int& nb) {
  // Grouped raster: `group` m-blocks sweep all n-blocks before moving on, so the
  // ~148 concurrently resident tiles share A rows and B columns in L2.
  // group < 0: -group n-blocks sweep all m-blocks (a group's weight strips stay
  // in L2 while the activations stream; long-K experiment).
  if (group < 0) {
    const int G = -group, per = G * num_m;
    const int gi = t / per, first_n = gi * G, gsize = min(num_n - first_n, G), r = t - gi * per;
    nb = first_n + r % gsize;
    mb = r / gsize;
    return;
  }
  int per_group = group * num_n;
  int g = t / per_group;
  int first_m = g * group;
  int gsize = min(num_m - first_m, group);
  int r = t - g * per_group;
  mb = first_m + r % gsize;
  nb = r / gsize;
}

// 1 / rms of the row from the producer GEMM's per-tile partial sums (fixed order).
DS_DEV float row_inv_rms(const GemmEpi& e, int row, bool row_ok) {
  if (!e.ssq_in || !row_ok) return 1.f;
  float t = 0.f;
  for (int p = 0; p < e.ssq_parts; ++p) t += __ldcg(e.ssq_in + p * e.ld_ssq + row);
  return 1.0f / sqrtf(t / (float)e.norm_dim + 1e-6f);
}

// Epilogue warps: bring this thread's row of the tile's f32 residual into L2
// while the tile's mainloop runs, so the residual epilogue's loads hit L2.
template <int BN>
DS_DEV void prefetch_resid(const GemmEpi& e, int row, int col0) {
  if (e.mode != EPI_RESID_F32 || row >= e.M) return;
  const int ncols = min(BN, e.N - col0);
  if (ncols > 0) prefetch_l2(e.resid + (long long)row * e.ld_resid + col0, (uint32_t)ncols * 4);
}

// BN accumulator columns starting at output column col0 (tbase = their first
// TMEM column); the residual epilogue's sum of squares is partial `part`.
template <int BN>
DS_DEV void epilogue_tile(const GemmEpi& e, uint32_t tbase, int row, int col0, int part) {
  const bool row_ok = row < e.M;
  const float inv = row_inv_rms(e, row, row_ok);
  if (e.mode == EPI_QKV_ROPE) {
    // j outer, heads inner: one row's cos/sin chunk (16-byte vector loads of
    // the f32 tables) serves every head of the tile
    const int D = e.head_dim;
    const int half = D >> 1;
    const int pos = e.pos_rows ? (row_ok ? __ldg(e.pos_rows + row) : 0) : e.pos0 + row;
    for (int j = 0; j < half; j += 16) {
      float cs[16], sn[16];
      if (row_ok) {
        const float4* c4 = reinterpret_cast<const float4*>(e.rope_cos + (long long)pos * half + j);
        const float4* s4 = reinterpret_cast<const float4*>(e.rope_sin + (long long)pos * half + j);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float4 c = __ldg(c4 + i), t = __ldg(s4 + i);
          cs[4 * i] = c.x; cs[4 * i + 1] = c.y; cs[4 * i + 2] = c.z; cs[4 * i + 3] = c.w;
          sn[4 * i] = t.x; sn[4 * i + 1] = t.y; sn[4 * i + 2] = t.z; sn[4 * i + 3] = t.w;
        }
      }
      for (int cb = 0; cb < BN; cb += D) {
        const int gcol = col0 + cb;  // column within this launch's N range
        if (gcol >= e.N) break;      // uniform across the warp
        const int head = (gcol + e.n_offset) / D;
        const bool is_q = head < e.n_heads;
        const bool is_k = !is_q && head < e.n_heads + e.n_kv_heads;
        float lo[16], hi[16];
        tmem_ld16x2(tbase + cb + j, tbase + cb + half + j, lo, hi);
        if (!row_ok) continue;
        if (e.ssq_in) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            lo[i] *= inv;
            hi[i] *= inv;
          }
        }
        if (is_q || is_k) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float x1 = lo[i], x2 = hi[i];
            lo[i] = x1 * cs[i] - x2 * sn[i];
            hi[i] = x1 * sn[i] + x2 * cs[i];
          }
        }
        uint32_t pl[8], ph[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          pl[i] = pack_bf16x2(lo[2 * i], lo[2 * i + 1]);
          ph[i] = pack_bf16x2(hi[2 * i], hi[2 * i + 1]);
        }
        bf16* dst;
        if (is_q) {
          dst = e.q_out + (long long)row * e.ld_q + (long long)head * D + j;
        } else if (is_k) {
          dst = e.kv.k + e.kv.off(head - e.n_heads, pos) + j;
        } else {
          dst = e.kv.v + e.kv.off(head - e.n_heads - e.n_kv_heads, pos) + j;
        }
        st_global_v4(dst, pl[0], pl[1], pl[2], pl[3]);
        st_global_v4(dst + 8, pl[4], pl[5], pl[6], pl[7]);
        st_global_v4(dst + half, ph[0], ph[1], ph[2], ph[3]);
        st_global_v4(dst + half + 8, ph[4], ph[5], ph[6], ph[7]);
      }
    }
    return;
  }
  if (e.mode == EPI_RESID_F32) {
    // f32 residual add, 16 columns per step with the next step's residual
    // loads in flight (the residual stream comes from HBM; a third buffer
    // spilled once the folded-RMSNorm outputs joined this epilogue)
    const int ncols = min(BN, e.N - col0);  // multiple of 16
    const float4* r = reinterpret_cast<const float4*>(e.resid + (long long)row * e.ld_resid + col0);
    float4* o = reinterpret_cast<float4*>(reinterpret_cast<float*>(e.out) + (long long)row * e.ld_out + col0);
    float4 r0[4], r1[4];
    if (row_ok) {
#pragma unroll
      for (int i = 0; i < 4; ++i) r0[i] = r[i];
    }
    float ss = 0.f;
    for (int c = 0; c < ncols; c += 16) {
      if (row_ok && c + 16 < ncols) {
#pragma unroll
        for (int i = 0; i < 4; ++i) r1[i] = r[(c + 16) / 4 + i];
      }
      float v[16];
      tmem_ld16(tbase + c, v);
      if (row_ok) {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] += (&r0[i / 4].x)[i % 4];
#pragma unroll
        for (int i = 0; i < 4; ++i) o[c / 4 + i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        if (e.norm_out) {
          // the next GEMM's operand: bf16(h * g); its epilogue applies 1/rms
          const float4* g4 = reinterpret_cast<const float4*>(e.norm_gain + col0 + c);
          uint32_t p[8];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float4 g = __ldg(g4 + i);
            ss = fmaf(v[4 * i], v[4 * i], ss);
            ss = fmaf(v[4 * i + 1], v[4 * i + 1], ss);
            ss = fmaf(v[4 * i + 2], v[4 * i + 2], ss);
            ss = fmaf(v[4 * i + 3], v[4 * i + 3], ss);
            p[2 * i] = pack_bf16x2(v[4 * i] * g.x, v[4 * i + 1] * g.y);
            p[2 * i + 1] = pack_bf16x2(v[4 * i + 2] * g.z, v[4 * i + 3] * g.w);
          }
          bf16* a = e.norm_out + (long long)row * e.ld_out + col0 + c;
          st_global_v4(a, p[0], p[1], p[2], p[3]);
          st_global_v4(a + 8, p[4], p[5], p[6], p[7]);
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) r0[i] = r1[i];
    }
    if (e.ssq_out && row_ok) e.ssq_out[part * e.ld_ssq + row] = ss;
    return;
  }
  if (e.mode == EPI_SWIGLU_BF16) {
    // W1 rows interleave gate / up in blocks of 16: accumulator columns
    // [32b, 32b+16) are gate, [32b+16, 32b+32) up; output column 16b + i
    for (int c = 0; c < BN; c += 32) {
      const int col = col0 + c;
      if (col >= e.N) break;
      float gt[16], up[16];
      tmem_ld16x2(tbase + c, tbase + c + 16, gt, up);
      if (!row_ok) continue;
      if (e.ssq_in) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          gt[i] *= inv;
          up[i] *= inv;
        }
      }
      uint32_t p[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) p[i] = pack_bf16x2(silu(gt[2 * i]) * up[2 * i], silu(gt[2 * i + 1]) * up[2 * i + 1]);
      bf16* o = reinterpret_cast<bf16*>(e.out) + (long long)row * e.ld_out + col / 2;
      st_global_v4(o, p[0], p[1], p[2], p[3]);
      st_global_v4(o + 8, p[4], p[5], p[6], p[7]);
    }
    return;
  }
  for (int c = 0; c < BN; c += 16) {
    const int col = col0 + c;
    if (col >= e.N) break;
    float v[16];
    tmem_ld16(tbase + c, v);
    if (!row_ok) continue;
    if (e.mode == EPI_STORE_F32) {
      float4* o = reinterpret_cast<float4*>(reinterpret_cast<float*>(e.out) + (long long)row * e.ld_out + col);
#pragma unroll
      for (int i = 0; i < 4; ++i) o[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    } else {
      if (e.ssq_in) {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] *= inv;
      }
      if (e.mode == EPI_SILU_BF16) {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = silu(v[i]);
      }
      uint32_t p[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) p[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);
      bf16* o = reinterpret_cast<bf16*>(e.out) + (long long)row * e.ld_out + col;
      st_global_v4(o, p[0], p[1], p[2], p[3]);
      st_global_v4(o + 8, p[4], p[5], p[6], p[7]);
    }
  }
}

// At most 128 registers per thread: a warp then holds 4096 of its SM
// sub-partition's 16K registers, which leaves room for an anchor GEMV or decode
// CTA of the other stream to share the SM with this persistent kernel.
template <int BN, int STAGES>
__global__ void __maxnreg__(128)
    gemm_tcgen05_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int K,
                        GemmEpi epi) {
  using L = GemmSmem<BN, STAGES>;
  constexpr uint32_t TMEM_COLS = 2 * BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * L::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * L::B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_m = (epi.M + GEMM_BM - 1) / GEMM_BM;
  const int num_n = (epi.N + BN - 1) / BN;
  const int num_tiles = num_m * num_n;
  const int k_blocks = (K + GEMM_BK - 1) / GEMM_BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // PDL: barrier init, TMEM alloc and descriptor prefetch overlapped the
  // predecessor's tail; its outputs are read only after this point
  pdl_trigger();
  pdl_wait();

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int mb, nb;
        tile_coords(t, num_m, num_n, epi.group, mb, nb);
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], L::STAGE_BYTES);
          tma_load_2d(sA + stage * L::A_BYTES, &tmA, &full[stage], kb * GEMM_BK, mb * GEMM_BM);
          tma_load_2d(sB + stage * L::B_BYTES, &tmB, &full[stage], kb * GEMM_BK, nb * BN);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t IDESC = umma_idesc_bf16(GEMM_BM, BN);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = 0; kb < k_blocks; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t a_addr = smem_u32(sA + stage * L::A_BYTES);
          const uint32_t b_addr = smem_u32(sB + stage * L::B_BYTES);
#pragma unroll
          for (int k = 0; k < GEMM_BK / 16; ++k) {
            const uint64_t ad = sdesc_sw128(a_addr + k * 32, 16, 1024);
            const uint64_t bd = sdesc_sw128(b_addr + k * 32, 16, 1024);
            umma_bf16(d_tmem, ad, bd, IDESC, (kb | k) != 0 ? 1u : 0u);
          }
          umma_commit(&empty[stage]);
          if (kb == k_blocks - 1) umma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  } else {
    const int quarter = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      int mb, nb;
      tile_coords(t, num_m, num_n, epi.group, mb, nb);
      prefetch_resid<BN>(epi, mb * GEMM_BM + quarter * 32 + lane, nb * BN);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN;
      epilogue_tile<BN>(epi, tbase, mb * GEMM_BM + quarter * 32 + lane, nb * BN, nb);
      tc_fence_before();
      if (epi.done) __threadfence();  // this warp's stores, before its completion count (release)
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&tempty[acc]);
        // a consumer on another stream (the persistent anchor) waits for
        // 4 * tiles arrivals before it reads this layer's K/V
        if (epi.done) atomicAdd(epi.done, 1u);
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}


// ---------------------------------------------------------------- CTA-pair (cta_group::2) variant
//
// A cluster of 2 CTAs on one TPC computes a 256 x 256 tile with
// tcgen05.mma.cta_group::2 (M = 256, N = 256, K = 16), issued by the leader
// (rank 0).  CTA r holds A rows [256m + 128r, +128) and B rows (output
// columns) [256n + 128r, +128) in its own shared memory; the MMA reads both
// halves, and CTA r's TMEM receives its 128 output rows x all 256 columns.
// Per CTA and k-block the operands are 32 KB instead of 48 KB (B is shared),
// so L2->SM traffic per FLOP drops by a third and 6 stages fit where 4 did.
//
//   full[s]   leader only: one arrive.expect_tx (both CTAs' bytes) + the
//             complete_tx of both CTAs' TMA loads (cta_group::2 TMA signals
//             the leader's barrier)
//   empty[s]  both CTAs: MMA commit multicast -> the producers refill
//   tfull[a]  both CTAs: MMA commit multicast after a tile's last k-block
//   tempty[a] leader only, 8 arrivals: the 4 epilogue warps of each CTA
constexpr int PAIR_BN = 256;             // output columns per pair tile
constexpr int PAIR_HALF = 128;           // B rows per CTA
constexpr int PAIR_STAGES = 6;

struct Gemm2Smem {
  static constexpr uint32_t A_BYTES = GEMM_BM * GEMM_BK * 2;    // 16 KB
  static constexpr uint32_t B_BYTES = PAIR_HALF * GEMM_BK * 2;  // 16 KB
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t BAR_BYTES = (2 * PAIR_STAGES + 4) * 8 + 16;
  static constexpr uint32_t TOTAL = 1024 + PAIR_STAGES * STAGE_BYTES + BAR_BYTES;
};

DS_DEV uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
DS_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Shared-memory address of the same variable in CTA `rank` of the cluster.
DS_DEV uint32_t map_to_rank(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
DS_DEV void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t leader_bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1)
      : "memory");
}
// Same with an L2 cache policy (createpolicy) on the loaded lines.
DS_DEV void tma_load_2d_pair_hint(void* dst, const CUtensorMap* map, uint32_t leader_bar, int c0, int c1,
                                  uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
      "[%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
DS_DEV uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
DS_DEV uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
DS_DEV void umma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive on the barrier at this offset in both CTAs once the pair's MMAs complete.
DS_DEV void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "{\n .reg .b16 m;\n mov.b16 m, 3;\n"
      " tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n}\n" ::"r"(
          smem_u32(bar))
      : "memory");
}
DS_DEV void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

// EW epilogue warps: 4 (one per TMEM lane quarter, all 256 columns of a row) or
// 8 (two per lane quarter, 128 columns each: twice the epilogue's loads and
// stores in flight, for the K = 4096 residual GEMM whose mainloop per tile is
// short).  With 8 the residual epilogue writes one sum-of-squares partial per
// 128 columns (gemm_col_tile), and 16 warps arrive per pair tile.
template <int EW>
__global__ void __cluster_dims__(2, 1, 1) __maxnreg__(128)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int K,
                    GemmEpi epi) {
  using L = Gemm2Smem;
  constexpr uint32_t TMEM_COLS = 2 * PAIR_BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + PAIR_STAGES * L::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + PAIR_STAGES * L::B_BYTES);
  uint64_t* empty = full + PAIR_STAGES;
  uint64_t* tfull = empty + PAIR_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  const int num_m = (epi.M + 2 * GEMM_BM - 1) / (2 * GEMM_BM);
  const int num_n = (epi.N + PAIR_BN - 1) / PAIR_BN;
  const int num_tiles = num_m * num_n;
  const int k_blocks = (K + GEMM_BK - 1) / GEMM_BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < PAIR_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * EW);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();  // both CTAs' barriers initialised before any remote arrive / TMA
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_trigger();
  pdl_wait();

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t leader_full0 = map_to_rank(&full[0], 0);
      // l2_hint 1: weights (B) evict_last, activations (A) evict_first; 2: the reverse (the
      // group raster reuses a group's A strips across its waves, B strips once per wave)
      const uint64_t pol_a = epi.l2_hint == 2 ? l2_policy_evict_last() : l2_policy_evict_first();
      const uint64_t pol_b = epi.l2_hint == 2 ? l2_policy_evict_first() : l2_policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int t = pair; t < num_tiles; t += n_pairs) {
        int mb, nb;
        tile_coords(t, num_m, num_n, epi.group, mb, nb);
        const int arow = mb * 2 * GEMM_BM + (int)rank * GEMM_BM;
        const int brow = nb * PAIR_BN + (int)rank * PAIR_HALF;
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (leader) mbar_expect_tx(&full[stage], 2 * L::STAGE_BYTES);
          const uint32_t fb = leader_full0 + stage * 8;
          if (epi.l2_hint) {
            tma_load_2d_pair_hint(sA + stage * L::A_BYTES, &tmA, fb, kb * GEMM_BK, arow, pol_a);
            tma_load_2d_pair_hint(sB + stage * L::B_BYTES, &tmB, fb, kb * GEMM_BK, brow, pol_b);
          } else {
            tma_load_2d_pair(sA + stage * L::A_BYTES, &tmA, fb, kb * GEMM_BK, arow);
            tma_load_2d_pair(sB + stage * L::B_BYTES, &tmB, fb, kb * GEMM_BK, brow);
          }
          if (++stage == PAIR_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      constexpr uint32_t IDESC = umma_idesc_bf16(2 * GEMM_BM, PAIR_BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = pair; t < num_tiles; t += n_pairs) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * PAIR_BN;
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a_addr = smem_u32(sA + stage * L::A_BYTES);
            const uint32_t b_addr = smem_u32(sB + stage * L::B_BYTES);
#pragma unroll
            for (int k = 0; k < GEMM_BK / 16; ++k) {
              const uint64_t ad = sdesc_sw128(a_addr + k * 32, 16, 1024);
              const uint64_t bd = sdesc_sw128(b_addr + k * 32, 16, 1024);
              umma_bf16_pair(d_tmem, ad, bd, IDESC, (kb | k) != 0 ? 1u : 0u);
            }
            umma_commit_pair(&empty[stage]);
            if (kb == k_blocks - 1) umma_commit_pair(&tfull[acc]);
          }
          __syncwarp();
          if (++stage == PAIR_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    constexpr int EC = PAIR_BN * 4 / EW;      // columns per epilogue warp
    const int quarter = warp & 3;
    const int part = (warp - 2) >> 2;         // column part of the tile (0 with 4 warps)
    const uint32_t leader_tempty0 = map_to_rank(&tempty[0], 0);
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = pair; t < num_tiles; t += n_pairs) {
      int mb, nb;
      tile_coords(t, num_m, num_n, epi.group, mb, nb);
      const int row = mb * 2 * GEMM_BM + (int)rank * GEMM_BM + quarter * 32 + lane;
      const int col0 = nb * PAIR_BN + part * EC;
      prefetch_resid<EC>(epi, row, col0);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * PAIR_BN + part * EC;
      epilogue_tile<EC>(epi, tbase, row, col0, nb * (PAIR_BN / EC) + part);
      tc_fence_before();
      if (epi.done) __threadfence();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_remote(leader_tempty0 + acc * 8);
        if (epi.done) atomicAdd(epi.done, 1u);
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the peer's MMAs / arrivals touch this CTA's smem and TMEM until here
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                 : "memory");
  }
}

// ---------------------------------------------------------------- host side

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2-D bf16 tensor map over a row-major [rows][cols] matrix with leading dimension ld
// (elements), box = box_rows x 64 columns, 128-byte swizzle.
int make_tmap_bf16(CUtensorMap* map, const void* ptr, long long rows, long long cols, long long ld,
                   int box_rows, int box_cols) {
  auto fn = encode_fn();
  if (!fn) return -1;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -(int)r - 2;
}

int num_sms() {
  static PerDevice cache;
  int& n = cache();
  if (!n) {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n = v > 0 ? v : 148;
  }
  return n;
}

template <int BN, int STAGES>
static cudaError_t launch_gemm_t(const CUtensorMap& ta, const CUtensorMap& tb, int K, const GemmEpi& epi,
                                 cudaStream_t stream, int max_ctas) {
  using L = GemmSmem<BN, STAGES>;
  auto kern = gemm_tcgen05_kernel<BN, STAGES>;
  static PerDevice attr;
  if (cudaError_t e = ensure_smem_attr(kern, L::TOTAL, attr)) return e;
  const int tiles = ((epi.M + GEMM_BM - 1) / GEMM_BM) * ((epi.N + BN - 1) / BN);
  int grid = tiles < num_sms() ? tiles : num_sms();
  if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
  count_launch();
  return launch_pdl(kern, dim3(grid), dim3(GEMM_THREADS), L::TOTAL, stream, ta, tb, K, epi);
}

int gemm_bn(int N) { return N >= 1024 ? 256 : 128; }

static int env_or(const char* name, int dflt) {
  const char* v = getenv(name);
  const int x = v ? atoi(v) : dflt;
  return x >= 0 ? x : dflt;
}

// The CTA-pair kernel serves the large recompute shapes (DS_GEMM_PAIR=0 turns it off).
static bool use_pair(int M, int N) {
  static int env = -1;
  if (env < 0) {
    const char* v = getenv("DS_GEMM_PAIR");
    env = (v && v[0] == '0') ? 0 : 1;
  }
  return env && N >= 1024 && M > GEMM_BM && num_sms() >= 2;
}

// Epilogue warps of the pair kernel (DS_GEMM_EPI_WARPS=8: A/B switch; 4 kept --
// 8 measured no step gain, DESIGN 6.1).
static int pair_epi_warps() {
  static int v = 0;
  if (!v) {
    const char* e = getenv("DS_GEMM_EPI_WARPS");
    v = (e && atoi(e) == 8) ? 8 : 4;
  }
  return v;
}

int gemm_col_tile(int M, int N) { return use_pair(M, N) ? PAIR_BN * 4 / pair_epi_warps() : gemm_bn(N); }

// Arrivals on GemmEpi::done once the GEMM has finished: 4 epilogue warps per
// 128-row CTA tile (the pair kernel: 2 CTA tiles per 256 x 256 pair tile, EW
// epilogue warps each).
unsigned int gemm_done_target(int M, int N) {
  if (use_pair(M, N))
    return 2u * (unsigned)pair_epi_warps() *
           (unsigned)(((M + 2 * GEMM_BM - 1) / (2 * GEMM_BM)) * ((N + PAIR_BN - 1) / PAIR_BN));
  const int bn = gemm_bn(N);
  return 4u * (unsigned)(((M + GEMM_BM - 1) / GEMM_BM) * ((N + bn - 1) / bn));
}

static cudaError_t launch_gemm_pair(const CUtensorMap& ta, const CUtensorMap& tb, int K, const GemmEpi& epi,
                                   cudaStream_t stream, int max_ctas) {
  const int ew = pair_epi_warps();
  auto kern = ew == 4 ? gemm_tc2_kernel<4> : gemm_tc2_kernel<8>;
  static PerDevice smem_set4, smem_set8;
  if (cudaError_t e = ensure_smem_attr(kern, Gemm2Smem::TOTAL, ew == 4 ? smem_set4 : smem_set8)) return e;
  const int tiles = ((epi.M + 2 * GEMM_BM - 1) / (2 * GEMM_BM)) * ((epi.N + PAIR_BN - 1) / PAIR_BN);
  int pairs = num_sms() / 2;
  if (max_ctas > 0 && pairs > max_ctas / 2) pairs = max_ctas / 2 > 0 ? max_ctas / 2 : 1;
  if (pairs > tiles) pairs = tiles;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(64 + 32 * ew);
  cfg.dynamicSmemBytes = Gemm2Smem::TOTAL;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  count_launch();
  return cudaLaunchKernelEx(&cfg, kern, ta, tb, K, epi);
}

// A: [M][K] (lda), B: [N][K] (ldb) bf16 row-major.  Picks the kernel from the shape.
int gemm_launch(const void* A, long long lda, const void* B, long long ldb, int K, const GemmEpi& epi,
                cudaStream_t stream, int force_bn, int max_ctas) {
  GemmEpi e2 = epi;
  CUtensorMap ta, tb;
  if (!force_bn && use_pair(epi.M, epi.N)) {
    // Raster group (pair m-blocks sweeping all n-blocks), per shape from the ncu
    // DRAM sweep (tools/raster_sweep.sh, profiles/r02_raster_sweep.txt): 16 for
    // K <= 4096 (W1 reads 369 vs 557 MB at 8, QKV 197 vs 265 MB), 8 for the
    // long-K W2.  DS_GEMM_GROUP / DS_GEMM_GROUP_LONGK override (experiments).
    // Long K (W2, K = d_ff): DS_GEMM_L2HINT=1 loads the weights evict_last and
    // the activations evict_first (experiment).
    static const int group_short = env_or("DS_GEMM_GROUP", 16);
    static const int group_long = env_or("DS_GEMM_GROUP_LONGK", 8);
    static const int l2hint = env_or("DS_GEMM_L2HINT", 0);
    const bool long_k = K > 8192;
    e2.group = long_k ? (group_long == 0 ? 1 : group_long) : max(1, group_short);
    e2.l2_hint = long_k ? l2hint : 0;
    if (make_tmap_bf16(&ta, A, epi.M, K, lda, GEMM_BM, GEMM_BK) ||
        make_tmap_bf16(&tb, B, epi.N, K, ldb, PAIR_HALF, GEMM_BK))
      return launch_status(cudaErrorInvalidValue);
    return launch_status(launch_gemm_pair(ta, tb, K, e2, stream, max_ctas));
  }
  int bn = force_bn ? force_bn : gemm_bn(epi.N);
  e2.group = 16;  // measured best of 8 / 16 / 64 for the recompute shapes
  if (make_tmap_bf16(&ta, A, epi.M, K, lda, GEMM_BM, GEMM_BK) || make_tmap_bf16(&tb, B, epi.N, K, ldb, bn, GEMM_BK))
    return launch_status(cudaErrorInvalidValue);
  cudaError_t e = bn == 256 ? launch_gemm_t<256, 4>(ta, tb, K, e2, stream, max_ctas)
                            : launch_gemm_t<128, 6>(ta, tb, K, e2, stream, max_ctas);
  return launch_status(e);
}

}  // namespace ds
