// Causal GQA flash-attention prefill over a (paged) KV cache layer.
//
// Semantics: _masked_attention over the window (model.py:506-519): head h
// reads kv head h / (H/KVH); scores scaled by 1/sqrt(D) after the dot product;
// query at absolute position p sees keys 0..p; max-subtracted softmax; output
// head-major [rows][H*D].  Online softmax in fp32 (exp2 with the scale folded
// in), P rounded to bf16 for the P.V product, output rounded to bf16.
#include <cstdio>

#include "common.cuh"
#include "kernels.h"

namespace ds {

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


// 2^x for a pair on the FMA pipe (x <= ~2^8 here): round-to-nearest split
// x = k + f, f in [-0.5, 0.5], 2^f by a degree-3 polynomial (rel. error < 7e-4,
// below the bf16 rounding P gets anyway), k added into the exponent bits.
// Takes a share of the exponentials off the MUFU pipe.
DS_DEV float2 exp2_fma2(float2 x) {
  // j = x + 1.5*2^23 puts round(x) in j's low mantissa bits; since
  // 0x4B400000 << 23 == 0 (mod 2^32), (bits(j) << 23) is round(x) moved into the
  // exponent field: one shift-add per element inserts it into 2^f.
  const float2 j = fadd2(x, make_float2(12582912.f, 12582912.f));
  const float2 k = fadd2(j, make_float2(-12582912.f, -12582912.f));  // round(x)
  const float2 f = ffma2(k, make_float2(-1.f, -1.f), x);               // x - round(x), in [-0.5, 0.5]
  float2 p = ffma2(make_float2(0.0555041087f, 0.0555041087f), f, make_float2(0.2402265070f, 0.2402265070f));
  p = ffma2(p, f, make_float2(0.6931471806f, 0.6931471806f));
  p = ffma2(p, f, make_float2(1.f, 1.f));
  const float rx = __int_as_float(__float_as_int(p.x) + (__float_as_int(j.x) << 23));
  const float ry = __int_as_float(__float_as_int(p.y) + (__float_as_int(j.y) << 23));
  // below 2^-126 (masked scores are -inf): exactly 0, as ex2.approx.ftz gives
  return make_float2(x.x > -126.f ? rx : 0.f, x.y > -126.f ? ry : 0.f);
}
#ifndef DS_FA_EMU_MOD
#define DS_FA_EMU_MOD 4  // one pair in DS_FA_EMU_MOD on the FMA pipe (0: all on MUFU)
#endif
#ifndef DS_FA_PASS1_BOTH
#define DS_FA_PASS1_BOTH 0  // dual FA: issue both pass-1 TMEM loads before the first wait (experiment)
#endif
#ifndef DS_FA_DUAL_EMU
// the dual-softmax kernel: one pair in 8 (in-step A/B at the power cap, 8B shape:
// 1 in 8 16.29 ms, 1 in 4 16.54, 1 in 2 slower; profiles/r02_fa_dual.txt)
#define DS_FA_DUAL_EMU 8
#endif

#ifndef DS_FA_STAMPS
#define DS_FA_STAMPS 0
#endif
#if DS_FA_STAMPS
// Debug timeline (DS_NVCC_EXTRA=-DDS_FA_STAMPS=1): CTA (0,0) records clock64
// at the pipeline hand-offs and prints them.
__device__ long long fa_stamps[2][64][8];
#define FA_STAMP(i, j, k) \
  if (DS_FA_STAMPS && blockIdx.x == 0 && blockIdx.y == 0 && (j) < 64) fa_stamps[i][j][k] = clock64()
#else
#define FA_STAMP(i, j, k)
#endif

#ifdef DS_FA_DIVERGENT_ISSUE
#define FA_ISSUER (lane == 0)
#else
#define FA_ISSUER elect_one()
#endif
#ifndef DS_FA_ABLATE
#define DS_FA_ABLATE 0
#endif

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
  const int32_t* q_pos;  // optional ascending per-row positions (else q_pos0 + row)
  long long k_head_rows, k_page_rows;
  const int32_t* table;
  bf16* o;
  long long ldo;
  float scale_log2;
  const bf16* q;  // [n_q][ldq] (the one-tile kernel stages Q rows into TMEM itself)
  long long ldq;
};

// At most 136 registers per thread: 3 FA warps of an SM sub-partition then
// leave room for one 88-register warp of the persistent anchor (anchor.cu).
template <int D, bool CHUNK>
__global__ void __maxnreg__(136)
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
  auto rowpos = [&](int r) { return a.q_pos ? __ldg(a.q_pos + r) : a.q_pos0 + r; };
  int n_kv[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int rows = min(FA_BM, a.n_q - (q0 + i * FA_BM));
    n_kv[i] = rows > 0 ? rowpos(q0 + i * FA_BM + rows - 1) / FA_BN + 1 : 0;
  }
  const int J = max(n_kv[0], n_kv[1]);
  const int max_key = rowpos(min(q0 + 2 * FA_BM, a.n_q) - 1);

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
  // PDL: barrier init, TMEM alloc and descriptor prefetch overlapped the
  // predecessor's tail; its outputs are read only after this point
  pdl_trigger();
  pdl_wait();

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
        if (DS_FA_ABLATE >= 2 && j >= 2) {  // timing only: stale K/V tiles, no loads
          mbar_expect_tx(&k_full[st], 0);
          mbar_wait(&v_empty[st], ph ^ 1);
          mbar_expect_tx(&v_full[st], 0);
          continue;
        }
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
    // The whole warp runs the issue code (warp-uniform descriptors stay in
    // uniform registers) and one elected lane issues each MMA: issuing from a
    // divergent `lane == 0` branch costs ~180 cycles per tcgen05.mma (R2UR
    // moves + a waterfall loop per instruction) against 64 cycles of tensor
    // work for a 128x128x16 MMA (tools/mma_probe.cu).
    auto qk = [&](int i, int st) {
#pragma unroll
      for (int c = 0; c < CH; ++c)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t ad = sdesc_sw128(smem_u32(sQ(i, c)) + k * 32, 16, 1024);
          const uint64_t bd = sdesc_sw128(smem_u32(sK(st, c)) + k * 32, 16, 1024);
          if (FA_ISSUER) umma_bf16(tmem + i * 128, ad, bd, IDESC_QK, (c | k) != 0 ? 1u : 0u);
        }
      if (FA_ISSUER) umma_commit(&s_full[i]);
      __syncwarp();
    };
    auto pv = [&](int i, int st, int j) {
#pragma unroll
      for (int s = 0; s < FA_BN / 16; ++s) {
        const uint64_t bd = sdesc_sw128(smem_u32(sV(st, 0)) + s * 2048, L::CHUNK, 1024);
        if (FA_ISSUER)
          umma_bf16_ts(tmem + 256 + i * 128, tmem + i * 128 + s * 8, bd, IDESC_PV, (j | s) != 0 ? 1u : 0u);
      }
      if (FA_ISSUER) umma_commit(&o_done[i]);
      __syncwarp();
    };
    mbar_wait(q_full, 0);
    mbar_wait(&k_full[0], 0);
    tc_fence_after();
    if (n_kv[0] > 0) qk(0, 0);
    if (n_kv[1] > 0) qk(1, 0);
    if (FA_ISSUER) umma_commit(&k_empty[0]);
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
        if (lane == 0) FA_STAMP(0, j, 2);
        tc_fence_after();
        pv(0, st, j);
      }
      if (more) {
        mbar_wait(&k_full[st1], ((j + 1) >> 1) & 1);
        if (lane == 0) FA_STAMP(0, j, 3);
        tc_fence_after();
        if (j + 1 < n_kv[0]) qk(0, st1);
      }
      if (j < n_kv[1]) {
        mbar_wait(&p_full[1], j & 1);
        if (lane == 0) FA_STAMP(1, j, 2);
        tc_fence_after();
        pv(1, st, j);
      }
      if (FA_ISSUER) umma_commit(&v_empty[st]);
      __syncwarp();
      if (more) {
        if (j + 1 < n_kv[1]) qk(1, st1);
        if (FA_ISSUER) umma_commit(&k_empty[st1]);
        __syncwarp();
      }
    }
  } else {
    const int i = (warp - 2) >> 2;  // Q tile
    const int quarter = warp & 3;   // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;
    const int first_row = min(q0 + i * FA_BM, a.n_q - 1);
    const int tile_pos0 = rowpos(first_row);
    const int qpos = q0 + i * FA_BM + row < a.n_q ? rowpos(q0 + i * FA_BM + row) : max_key;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t tS = tmem + lane_base + i * 128;
    const uint32_t tO = tmem + lane_base + 256 + i * 128;
    const float sc = a.scale_log2;
    const float thr = 8.0f / sc;
    float m_used = -INFINITY, l = 0.f;
    if constexpr (CHUNK) {
      // Softmax in four 32-column chunks against a running max: chunk c+1's
      // TMEM load is in flight while chunk c is exponentiated, and P chunk c
      // (16 packed columns) goes over S columns already consumed.  The max
      // used for the exponentials only moves when a chunk's max exceeds it by
      // more than 2^8 (p <= 256 always); then the P chunks already written
      // are rescaled in TMEM (rare: in practice only the first chunk of the
      // first key block) and O once per key block, as in the lazy rescale.
      for (int j = 0; j < n_kv[i]; ++j) {
        mbar_wait(&s_full[i], j & 1);
        if (lane == 0 && quarter == 0) FA_STAMP(i, j, 0);
        tc_fence_after();
#if DS_FA_ABLATE
        // timing only: the MMA pipeline without the softmax (wrong results)
        if (lane == 0) mbar_arrive(&p_full[i]);
        l = 1.f;
        continue;
#endif
        const int kbase = j * FA_BN;
        const bool maskit = kbase + FA_BN - 1 > tile_pos0;
        uint32_t sa[32], sb[32];
        tmem_ld32_nowait(tS, sa);
        tmem_wait_ld();
        float ocorr = 1.f;
        float2 sum4[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
        const float2 sc2 = make_float2(sc, sc);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t* cur = (c & 1) ? sb : sa;
          uint32_t* nxt = (c & 1) ? sa : sb;
          if (c < 3) tmem_ld32_nowait(tS + 32 * (c + 1), nxt);
          if (maskit) {
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (kbase + 32 * c + e > qpos) cur[e] = __float_as_uint(-INFINITY);
          }
          float mx4[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) mx4[q] = fmax3(__uint_as_float(cur[q]), __uint_as_float(cur[q + 4]),
                                                     __uint_as_float(cur[q + 8]));
#pragma unroll
          for (int e = 12; e < 32; e += 8)
#pragma unroll
            for (int q = 0; q < 4; ++q)
              mx4[q] = fmax3(mx4[q], __uint_as_float(cur[e + q]), __uint_as_float(cur[e + 4 + q]));
          const float cm = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
          const bool need = cm > m_used + thr;
          if (__any_sync(0xffffffffu, need)) {
            float f = 1.f;
            if (need) {
              f = fast_exp2((m_used - cm) * sc);  // 0 while m_used is -inf
              m_used = cm;
            }
            l *= f;
            ocorr *= f;
            if (c > 0) {
              // rescale the P chunks already in TMEM (bf16 pairs) by f
              tmem_wait_st();
#pragma unroll 1
              for (int cc = 0; cc < c; ++cc) {
                uint32_t pr[16];
                tmem_ld16_nowait(tS + 16 * cc, pr);
                tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                  const float2 v = unpack_bf16x2(pr[e]);
                  pr[e] = pack_bf16x2(v.x * f, v.y * f);
                }
                tmem_st16_nowait(tS + 16 * cc, pr);
              }
              const float2 s2 = fadd2(fadd2(sum4[0], sum4[1]), fadd2(sum4[2], sum4[3]));
              l += (s2.x + s2.y) * f;  // the chunks summed so far, rescaled
              sum4[0] = sum4[1] = sum4[2] = sum4[3] = make_float2(0.f, 0.f);
            }
          }
          const float msc = m_used * sc;
          const float2 nmsc2 = make_float2(-msc, -msc);
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const float2 x = ffma2(make_float2(__uint_as_float(cur[2 * e]), __uint_as_float(cur[2 * e + 1])), sc2,
                                   nmsc2);
            float2 p;
            if (DS_FA_EMU_MOD && (e % (DS_FA_EMU_MOD > 0 ? DS_FA_EMU_MOD : 1)) == DS_FA_EMU_MOD - 1)
              p = exp2_fma2(x);
            else
              p = make_float2(fast_exp2(x.x), fast_exp2(x.y));
            sum4[e & 3] = fadd2(sum4[e & 3], p);
            pk[e] = pack_bf16x2(p.x, p.y);
          }
          tmem_st16_nowait(tS + 16 * c, pk);
          if (c < 3) {
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) asm volatile("" : "+r"(nxt[e]));  // values valid only after the wait
          }
        }
        const float2 s2 = fadd2(fadd2(sum4[0], sum4[1]), fadd2(sum4[2], sum4[3]));
        l += s2.x + s2.y;
        if (j > 0 && __any_sync(0xffffffffu, ocorr != 1.f)) {
          mbar_wait(&o_done[i], (j - 1) & 1);
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < D / 32; ++c) {
            uint32_t orow[32];
            tmem_ld32_nowait(tO + c * 32, orow);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) orow[e] = __float_as_uint(__uint_as_float(orow[e]) * ocorr);
            tmem_st32_nowait(tO + c * 32, orow);
          }
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0 && quarter == 0) FA_STAMP(i, j, 1);
        if (lane == 0) mbar_arrive(&p_full[i]);
      }
    } else {
      for (int j = 0; j < n_kv[i]; ++j) {
        mbar_wait(&s_full[i], j & 1);
        tc_fence_after();
        // The row in two 64-column halves (at most 136 registers per thread, so
        // an anchor warp of the other stream fits beside the 3 FA warps of an SM
        // sub-partition): pass 1 takes the masked row max, upper half first so
        // the lower half stays in registers for pass 2.
        const int kbase = j * FA_BN;
        const bool maskit = kbase + FA_BN - 1 > tile_pos0;
        uint32_t sr[FA_BN / 2];
        tmem_ld32_nowait(tS + 64, sr);
        tmem_ld32_nowait(tS + 96, sr + 32);
        tmem_wait_ld();
        if (maskit) {
  #pragma unroll
          for (int c = 0; c < FA_BN / 2; ++c)
            if (kbase + FA_BN / 2 + c > qpos) sr[c] = __float_as_uint(-INFINITY);
        }
        // row max as 8 independent chains (a single 128-long fmax chain is
        // ~4 cycles per link on the softmax critical path)
        float mx8[8];
  #pragma unroll
        for (int q = 0; q < 8; ++q) mx8[q] = __uint_as_float(sr[q]);
  #pragma unroll
        for (int c = 8; c < FA_BN / 2; c += 2)
          mx8[(c >> 1) & 7] = fmax3(mx8[(c >> 1) & 7], __uint_as_float(sr[c]), __uint_as_float(sr[c + 1]));
        tmem_ld32_nowait(tS, sr);
        tmem_ld32_nowait(tS + 32, sr + 32);
        tmem_wait_ld();
        if (maskit) {
  #pragma unroll
          for (int c = 0; c < FA_BN / 2; ++c)
            if (kbase + c > qpos) sr[c] = __float_as_uint(-INFINITY);
        }
  #pragma unroll
        for (int c = 0; c < FA_BN / 2; c += 2)
          mx8[(c >> 1) & 7] = fmax3(mx8[(c >> 1) & 7], __uint_as_float(sr[c]), __uint_as_float(sr[c + 1]));
        const float mt = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                               fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
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
        float2 sum4[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};  // independent partial sums
        uint32_t pk[FA_BN / 8];
        const float2 sc2 = make_float2(sc, sc), nmsc2 = make_float2(-msc, -msc);
        auto expo = [&](int c, uint32_t s0, uint32_t s1) {
          const float2 x = ffma2(make_float2(__uint_as_float(s0), __uint_as_float(s1)), sc2, nmsc2);
          float2 p;
          if (DS_FA_EMU_MOD && (c % (DS_FA_EMU_MOD > 0 ? DS_FA_EMU_MOD : 1)) == DS_FA_EMU_MOD - 1)
            p = exp2_fma2(x);
          else
            p = make_float2(fast_exp2(x.x), fast_exp2(x.y));
          sum4[c & 3] = fadd2(sum4[c & 3], p);
          pk[c & 15] = pack_bf16x2(p.x, p.y);
        };
        // pass 2: lower half from registers -> P columns [0, 32) (over consumed S)
  #pragma unroll
        for (int c = 0; c < FA_BN / 4; ++c) {
          expo(c, sr[2 * c], sr[2 * c + 1]);
          if ((c & 15) == 15) tmem_st16_nowait(tS + (c & ~15), pk);  // P columns as they complete
        }
        // upper half re-read -> P columns [32, 64) (S columns 32..63 are consumed)
        tmem_ld32_nowait(tS + 64, sr);
        tmem_ld32_nowait(tS + 96, sr + 32);
        tmem_wait_ld();
        if (maskit) {
  #pragma unroll
          for (int c = 0; c < FA_BN / 2; ++c)
            if (kbase + FA_BN / 2 + c > qpos) sr[c] = __float_as_uint(-INFINITY);
        }
  #pragma unroll
        for (int c = 0; c < FA_BN / 4; ++c) {
          expo(c, sr[2 * c], sr[2 * c + 1]);
          if ((c & 15) == 15) tmem_st16_nowait(tS + 32 + (c & ~15), pk);
        }
        const float2 s2 = fadd2(fadd2(sum4[0], sum4[1]), fadd2(sum4[2], sum4[3]));
        l += s2.x + s2.y;
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[i]);
      }
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
#if DS_FA_STAMPS
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
    const long long t0 = fa_stamps[0][0][0];
    for (int j = 0; j < min(J, 64); ++j)
      printf("FA j=%2d  S0 %7lld P0 %7lld mmaP0 %7lld K %7lld | S1 %7lld P1 %7lld mmaP1 %7lld\n", j,
             fa_stamps[0][j][0] - t0, fa_stamps[0][j][1] - t0, fa_stamps[0][j][2] - t0, fa_stamps[0][j][3] - t0,
             fa_stamps[1][j][0] - t0, fa_stamps[1][j][1] - t0, fa_stamps[1][j][2] - t0);
  }
#endif
}

// ----------------------------------------------------------------------
// Split-half variant (the default): each 128-key block's scores are produced
// and consumed in two 64-key halves.  QK of half h of the next block only
// waits for P.V of half h of this block, so the tensor pipe always holds
// the other half's work while a softmax warp exponentiates: a tile's softmax
// may take up to ~2x its MMA time before the tensor pipe idles (with whole
// tiles it stalls as soon as the softmax outlasts one tile's QK + P.V).
// Measured reason (tools/fa stamps): one 128-key softmax pass takes ~2000
// cycles with both tiles' softmax warps sharing an SM sub-partition, against
// 1024 cycles of MMA per tile.
//
// TMEM per Q tile i: S [128i, 128i+128); half h's scores in columns 64h..,
// its bf16 P in columns 64h..64h+31 (over consumed scores).  O as before.
// Softmax: 32-column chunks against a running max (p <= 2^8 always); a max
// that moves by more than 2^8 rescales the P chunk of the current half and O
// (after the P.V half issued last has completed) -- in practice only the
// first chunk of the first block.
// ----------------------------------------------------------------------
template <int D>
__global__ void __maxnreg__(136)
    fa_split_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
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
  uint64_t* s_full = bars + 9;   // [tile][half]
  uint64_t* p_full = bars + 13;  // [tile][half]
  uint64_t* o_done = bars + 17;  // [tile][half]: P.V of that half complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 24);
  auto sQ = [&](int i, int c) { return smem + L::Q + (i * CH + c) * L::CHUNK; };
  auto sK = [&](int st, int c) { return smem + L::K + (st * CH + c) * L::CHUNK; };
  auto sV = [&](int st, int c) { return smem + L::V + (st * CH + c) * L::CHUNK; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = blockIdx.x;
  const int q0 = (gridDim.y - 1 - blockIdx.y) * 2 * FA_BM;  // heaviest (latest) blocks first
  const int g = h / (a.n_heads / a.n_kv_heads);
  auto rowpos = [&](int r) { return a.q_pos ? __ldg(a.q_pos + r) : a.q_pos0 + r; };
  int n_kv[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int rows = min(FA_BM, a.n_q - (q0 + i * FA_BM));
    n_kv[i] = rows > 0 ? rowpos(q0 + i * FA_BM + rows - 1) / FA_BN + 1 : 0;
  }
  const int J = max(n_kv[0], n_kv[1]);
  const int max_key = rowpos(min(q0 + 2 * FA_BM, a.n_q) - 1);

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
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&o_done[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();

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
    // whole warp runs the issue code (uniform descriptors), one elected lane issues
    constexpr uint32_t IDESC_QK = umma_idesc_bf16(FA_BM, FA_BN / 2);
    constexpr uint32_t IDESC_PV = umma_idesc_bf16_bmn(FA_BM, D);
    auto qk = [&](int i, int hf, int st) {  // S_i[:, half hf] = Q_i K_half^T
#pragma unroll
      for (int c = 0; c < CH; ++c)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t ad = sdesc_sw128(smem_u32(sQ(i, c)) + k * 32, 16, 1024);
          const uint64_t bd = sdesc_sw128(smem_u32(sK(st, c)) + hf * 8192 + k * 32, 16, 1024);
          if (elect_one()) umma_bf16(tmem + i * 128 + hf * 64, ad, bd, IDESC_QK, (c | k) != 0 ? 1u : 0u);
        }
      if (elect_one()) umma_commit(&s_full[2 * i + hf]);
      __syncwarp();
    };
    auto pv = [&](int i, int hf, int st, int j) {  // O_i += P_half V_half
#pragma unroll
      for (int s = 0; s < FA_BN / 32; ++s) {
        const uint64_t bd = sdesc_sw128(smem_u32(sV(st, 0)) + (hf * 4 + s) * 2048, L::CHUNK, 1024);
        if (elect_one())
          umma_bf16_ts(tmem + 256 + i * 128, tmem + i * 128 + hf * 64 + s * 8, bd, IDESC_PV,
                       (j | hf | s) != 0 ? 1u : 0u);
      }
      if (elect_one()) umma_commit(&o_done[2 * i + hf]);
      __syncwarp();
    };
    mbar_wait(q_full, 0);
    mbar_wait(&k_full[0], 0);
    tc_fence_after();
    for (int i = 0; i < 2; ++i)
      if (n_kv[i] > 0) {
        qk(i, 0, 0);
        qk(i, 1, 0);
      }
    if (elect_one()) umma_commit(&k_empty[0]);
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
      bool k_ready = false;
#pragma unroll
      for (int hf = 0; hf < 2; ++hf)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          if (j < n_kv[i]) {
            mbar_wait(&p_full[2 * i + hf], j & 1);
            if (lane == 0) FA_STAMP(i, j, 4 + hf);
            tc_fence_after();
            pv(i, hf, st, j);
          }
          if (hf == 1 && i == 1) {
            if (elect_one()) umma_commit(&v_empty[st]);
            __syncwarp();
          }
          if (j + 1 < n_kv[i]) {
            if (!k_ready) {
              mbar_wait(&k_full[st1], ((j + 1) >> 1) & 1);
              tc_fence_after();
              k_ready = true;
            }
            qk(i, hf, st1);
          }
        }
      if (more) {
        if (elect_one()) umma_commit(&k_empty[st1]);
        __syncwarp();
      }
    }
  } else {
    const int i = (warp - 2) >> 2;  // Q tile
    const int quarter = warp & 3;   // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;
    const int first_row = min(q0 + i * FA_BM, a.n_q - 1);
    const int tile_pos0 = rowpos(first_row);
    const int qpos = q0 + i * FA_BM + row < a.n_q ? rowpos(q0 + i * FA_BM + row) : max_key;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t tS = tmem + lane_base + i * 128;
    const uint32_t tO = tmem + lane_base + 256 + i * 128;
    const float sc = a.scale_log2;
    const float thr = 8.0f / sc;
    const float2 sc2 = make_float2(sc, sc);
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < n_kv[i]; ++j) {
      const int kbase = j * FA_BN;
      const bool maskit = kbase + FA_BN - 1 > tile_pos0;
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        mbar_wait(&s_full[2 * i + hf], j & 1);
        if (lane == 0 && quarter == 0) FA_STAMP(i, j, 2 * hf);
        tc_fence_after();
        uint32_t sa[32], sb[32];
        tmem_ld32_nowait(tS + hf * 64, sa);
        tmem_wait_ld();
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const int c = 2 * hf + cc;  // chunk: keys kbase + 32c ..
          uint32_t* cur = cc ? sb : sa;
          if (cc == 0) tmem_ld32_nowait(tS + hf * 64 + 32, sb);
          if (maskit) {
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (kbase + 32 * c + e > qpos) cur[e] = __float_as_uint(-INFINITY);
          }
          float mx4[4];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            mx4[q] = fmax3(__uint_as_float(cur[q]), __uint_as_float(cur[q + 4]), __uint_as_float(cur[q + 8]));
#pragma unroll
          for (int e = 12; e < 32; e += 8)
#pragma unroll
            for (int q = 0; q < 4; ++q)
              mx4[q] = fmax3(mx4[q], __uint_as_float(cur[e + q]), __uint_as_float(cur[e + 4 + q]));
          const float cm = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
          const bool need = cm > m_used + thr;
          if (__any_sync(0xffffffffu, need)) {
            float f = 1.f;
            if (need) {
              f = fast_exp2((m_used - cm) * sc);  // 0 while m_used is -inf
              m_used = cm;
            }
            l *= f;
            if (cc == 1) {  // this half's first P chunk is already in TMEM
              tmem_wait_st();
              uint32_t pr[16];
              tmem_ld16_nowait(tS + hf * 64, pr);
              tmem_wait_ld();
#pragma unroll
              for (int e = 0; e < 16; ++e) {
                const float2 v = unpack_bf16x2(pr[e]);
                pr[e] = pack_bf16x2(v.x * f, v.y * f);
              }
              tmem_st16_nowait(tS + hf * 64, pr);
            }
            if (j > 0 || hf > 0) {
              // O holds P.V of every half released so far: wait for the last
              // one -- half a of this block, or half b of the previous one.
              // (One barrier per half: each is at most one phase behind here,
              // so the parity wait cannot alias.)
              if (hf) mbar_wait(&o_done[2 * i], j & 1);
              else mbar_wait(&o_done[2 * i + 1], (j - 1) & 1);
              tc_fence_after();
#pragma unroll 1
              for (int oc = 0; oc < D / 32; ++oc) {
                uint32_t orow[32];
                tmem_ld32_nowait(tO + oc * 32, orow);
                tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 32; ++e) orow[e] = __float_as_uint(__uint_as_float(orow[e]) * f);
                tmem_st32_nowait(tO + oc * 32, orow);
              }
            }
          }
          const float msc = m_used * sc;
          const float2 nmsc2 = make_float2(-msc, -msc);
          float2 sum4[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const float2 x =
                ffma2(make_float2(__uint_as_float(cur[2 * e]), __uint_as_float(cur[2 * e + 1])), sc2, nmsc2);
            float2 p;
            if (DS_FA_EMU_MOD && (e % (DS_FA_EMU_MOD > 0 ? DS_FA_EMU_MOD : 1)) == DS_FA_EMU_MOD - 1)
              p = exp2_fma2(x);
            else
              p = make_float2(fast_exp2(x.x), fast_exp2(x.y));
            sum4[e & 3] = fadd2(sum4[e & 3], p);
            pk[e] = pack_bf16x2(p.x, p.y);
          }
          tmem_st16_nowait(tS + hf * 64 + cc * 16, pk);
          const float2 s2 = fadd2(fadd2(sum4[0], sum4[1]), fadd2(sum4[2], sum4[3]));
          l += s2.x + s2.y;
          if (cc == 0) {
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) asm volatile("" : "+r"(sb[e]));  // valid only after the wait
          }
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0 && quarter == 0) FA_STAMP(i, j, 2 * hf + 1);
        if (lane == 0) mbar_arrive(&p_full[2 * i + hf]);
      }
    }
    if (n_kv[i] > 0) {
      mbar_wait(&o_done[2 * i + 1], (n_kv[i] - 1) & 1);  // the last P.V half
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
#if DS_FA_STAMPS
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
    const long long t0 = fa_stamps[0][0][0];
    for (int j = 0; j < min(J, 64); ++j)
      printf("FA j=%2d | t0: Sa %7lld Pa %7lld Sb %7lld Pb %7lld pvA %7lld pvB %7lld | t1: Sa %7lld Pa %7lld Sb %7lld Pb %7lld pvA %7lld pvB %7lld\n", j,
             fa_stamps[0][j][0] - t0, fa_stamps[0][j][1] - t0, fa_stamps[0][j][2] - t0, fa_stamps[0][j][3] - t0,
             fa_stamps[0][j][4] - t0, fa_stamps[0][j][5] - t0,
             fa_stamps[1][j][0] - t0, fa_stamps[1][j][1] - t0, fa_stamps[1][j][2] - t0, fa_stamps[1][j][3] - t0,
             fa_stamps[1][j][4] - t0, fa_stamps[1][j][5] - t0);
  }
#endif
}

// ----------------------------------------------------------------------
// Dual-softmax variant: two softmax warps per (Q tile, TMEM lane quarter),
// each owning 64 of a block's 128 key columns (18 warps).  Measured reason
// (profiles/r02_fa_stamps_current.txt, r02_pipe_probe.txt): one softmax warp
// per SM sub-partition and tile runs the 128-column pass latency-bound (~2250
// cycles per 128x128 block against 1024 cycles of the other tile's MMAs; one
// warp reaches half the MUFU rate), so the tensor pipe idled ~45% of every
// period.  Two warps on the same rows halve each warp's chain and keep the MUFU
// busy.  Per block: pass 1 takes each half's masked row max; the two halves
// agree on the lazily-moved max (it only moves when a row max exceeds it by
// more than 2^8) with one barrier-reduction vote per block (bar.red.or over the
// pair's 64 threads) and exchange their maxima through shared memory only when
// a row needs the move; pass 2 re-reads S in 16-column pieces, exponentiates and
// writes bf16 P.  Half h writes P of keys 64h.. over its own consumed S columns
// 64h.. (the P.V MMA reads its A operand from there), so the halves never touch
// each other's TMEM columns.  Row sums stay per half and are added (l0 + l1)
// for the epilogue; O rescales are done by half 0.  At most 80 registers per
// thread: with 18 warps, 5 share an SM sub-partition with one anchor warp.
// ----------------------------------------------------------------------
constexpr int FA_DUAL_THREADS = 18 * 32;

template <int D>
struct FaDualSmem {
  using B = FaTcSmem<D>;
  static constexpr uint32_t XCH = B::BAR + 256;  // float [2 tiles][2 halves][128 rows]
  static constexpr uint32_t TOTAL = XCH + 2048 + 1024;
};

DS_DEV bool bar_red_or(int id, int n, bool p) {
  uint32_t r;
  asm volatile(
      "{\n .reg .pred q, o;\n setp.ne.u32 q, %1, 0;\n barrier.cta.red.or.pred o, %2, %3, q;\n selp.u32 %0, 1, 0, o;\n}\n"
      : "=r"(r)
      : "r"((uint32_t)p), "r"(id), "r"(n)
      : "memory");
  return r != 0;
}
DS_DEV void bar_pair_sync(int id, int n) { asm volatile("barrier.cta.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <int D>
__global__ void __maxnreg__(80)
    fa_dual_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, FaTcArgs a) {
  using L = FaTcSmem<D>;
  using LD = FaDualSmem<D>;
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
  float* xch = reinterpret_cast<float*>(smem + LD::XCH);
  auto sQ = [&](int i, int c) { return smem + L::Q + (i * CH + c) * L::CHUNK; };
  auto sK = [&](int st, int c) { return smem + L::K + (st * CH + c) * L::CHUNK; };
  auto sV = [&](int st, int c) { return smem + L::V + (st * CH + c) * L::CHUNK; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = blockIdx.x;
  const int q0 = (gridDim.y - 1 - blockIdx.y) * 2 * FA_BM;  // heaviest (latest) blocks first
  const int g = h / (a.n_heads / a.n_kv_heads);
  auto rowpos = [&](int r) { return a.q_pos ? __ldg(a.q_pos + r) : a.q_pos0 + r; };
  int n_kv[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int rows = min(FA_BM, a.n_q - (q0 + i * FA_BM));
    n_kv[i] = rows > 0 ? rowpos(q0 + i * FA_BM + rows - 1) / FA_BN + 1 : 0;
  }
  const int J = max(n_kv[0], n_kv[1]);
  const int max_key = rowpos(min(q0 + 2 * FA_BM, a.n_q) - 1);

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
      mbar_init(&p_full[i], 8);
      mbar_init(&o_done[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();

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
#pragma unroll
      for (int c = 0; c < CH; ++c)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t ad = sdesc_sw128(smem_u32(sQ(i, c)) + k * 32, 16, 1024);
          const uint64_t bd = sdesc_sw128(smem_u32(sK(st, c)) + k * 32, 16, 1024);
          if (elect_one()) umma_bf16(tmem + i * 128, ad, bd, IDESC_QK, (c | k) != 0 ? 1u : 0u);
        }
      if (elect_one()) umma_commit(&s_full[i]);
      __syncwarp();
    };
    auto pv = [&](int i, int st, int j) {
#pragma unroll
      for (int s = 0; s < FA_BN / 16; ++s) {
        const uint64_t bd = sdesc_sw128(smem_u32(sV(st, 0)) + s * 2048, L::CHUNK, 1024);
        // P of keys 16s.. : half 0 (s < 4) at columns 8s, half 1 at 64 + 8(s - 4)
        const uint32_t pa = tmem + i * 128 + (s < 4 ? s * 8 : 64 + (s - 4) * 8);
        if (elect_one()) umma_bf16_ts(tmem + 256 + i * 128, pa, bd, IDESC_PV, (j | s) != 0 ? 1u : 0u);
      }
      if (elect_one()) umma_commit(&o_done[i]);
      __syncwarp();
    };
    mbar_wait(q_full, 0);
    mbar_wait(&k_full[0], 0);
    tc_fence_after();
    if (n_kv[0] > 0) qk(0, 0);
    if (n_kv[1] > 0) qk(1, 0);
    if (elect_one()) umma_commit(&k_empty[0]);
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
        if (lane == 0) FA_STAMP(0, j, 2);
        tc_fence_after();
        pv(0, st, j);
      }
      if (more) {
        mbar_wait(&k_full[st1], ((j + 1) >> 1) & 1);
        if (lane == 0) FA_STAMP(0, j, 3);
        tc_fence_after();
        if (j + 1 < n_kv[0]) qk(0, st1);
      }
      if (j < n_kv[1]) {
        mbar_wait(&p_full[1], j & 1);
        if (lane == 0) FA_STAMP(1, j, 2);
        tc_fence_after();
        pv(1, st, j);
      }
      if (elect_one()) umma_commit(&v_empty[st]);
      __syncwarp();
      if (more) {
        if (j + 1 < n_kv[1]) qk(1, st1);
        if (elect_one()) umma_commit(&k_empty[st1]);
        __syncwarp();
      }
    }
  } else {
    const int i = ((warp - 2) >> 2) & 1;  // Q tile
    const int hf = (warp - 2) >> 3;       // column half: keys [64 hf, 64 hf + 64) of each block
    const int quarter = warp & 3;         // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;
    const int pair = 1 + i * 4 + quarter;  // named barrier of the two warps sharing these rows
    const int first_row = min(q0 + i * FA_BM, a.n_q - 1);
    const int tile_pos0 = rowpos(first_row);
    const int qpos = q0 + i * FA_BM + row < a.n_q ? rowpos(q0 + i * FA_BM + row) : max_key;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t tS = tmem + lane_base + i * 128 + hf * 64;  // this half's S (and its P) columns
    const uint32_t tO = tmem + lane_base + 256 + i * 128;
    float* xmine = xch + (i * 2 + hf) * 128;
    float* xother = xch + (i * 2 + (hf ^ 1)) * 128;
    const float sc = a.scale_log2;
    const float thr = 8.0f / sc;
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < n_kv[i]; ++j) {
      mbar_wait(&s_full[i], j & 1);
      if (lane == 0 && quarter == 0 && hf == 0) FA_STAMP(i, j, 0);
      tc_fence_after();
#if DS_FA_ABLATE
      if (lane == 0) mbar_arrive(&p_full[i]);
      l = 1.f;
      continue;
#endif
      const int kbase = j * FA_BN + hf * 64;
      const bool maskit = j * FA_BN + FA_BN - 1 > tile_pos0;
      // pass 1: this half's masked row max.  DS_FA_PASS1_BOTH 2: the second half's
      // loads are issued while the first half's max is computed (48 registers)
      float mx = -INFINITY;
      auto max32 = [&](uint32_t* r, int col0) {  // masks r in place
        if (maskit) {
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (kbase + col0 + e > qpos) r[e] = __float_as_uint(-INFINITY);
        }
        float m4[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          m4[q] = fmax3(__uint_as_float(r[q]), __uint_as_float(r[q + 4]), __uint_as_float(r[q + 8]));
#pragma unroll
        for (int e = 12; e < 32; e += 8)
#pragma unroll
          for (int q = 0; q < 4; ++q) m4[q] = fmax3(m4[q], __uint_as_float(r[e + q]), __uint_as_float(r[e + 4 + q]));
        mx = fmax3(mx, fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
      };
#if DS_FA_PASS1_BOTH == 2
      {
        uint32_t r0[32], r1[16];
        tmem_ld32_nowait(tS, r0);
        tmem_wait_ld();
        tmem_ld16_nowait(tS + 32, r1);  // in flight while the first half's max runs
        max32(r0, 0);
        tmem_ld16_nowait(tS + 48, r0);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 16; ++e) r0[16 + e] = r0[e];
#pragma unroll
        for (int e = 0; e < 16; ++e) r0[e] = r1[e];
        max32(r0, 32);
      }
#elif DS_FA_PASS1_BOTH == 1
      {
        uint32_t rr[2][32];
        tmem_ld32_nowait(tS, rr[0]);
        tmem_ld32_nowait(tS + 32, rr[1]);
        tmem_wait_ld();
        max32(rr[0], 0);
        max32(rr[1], 32);
      }
#else
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t r[32];
        tmem_ld32_nowait(tS + 32 * c, r);
        tmem_wait_ld();
        max32(r, 32 * c);
      }
#endif
      // the pair agrees on the (lazily moved) max: one vote; maxima exchanged only when needed
      float ocorr = 1.f;
      if (bar_red_or(pair, 64, mx > m_used + thr)) {
        xmine[row] = mx;
        bar_pair_sync(pair, 64);
        const float mo = xother[row];
        const float mn = fmaxf(mx, mo);
        if (mn > m_used + thr) {
          ocorr = fast_exp2((m_used - mn) * sc);  // 0 while m_used is -inf
          m_used = mn;
          l *= ocorr;
        }
        bar_pair_sync(pair, 64);  // both read before either writes again
      }
      if (lane == 0 && quarter == 0 && hf == 0) FA_STAMP(i, j, 4);
      // pass 2: exponentiate in 16-column pieces (next piece's load in flight), P over consumed S
      const float msc = m_used * sc;
      const float2 sc2 = make_float2(sc, sc), nmsc2 = make_float2(-msc, -msc);
      float2 sum4[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
      uint32_t sa[16], sb[16];
      tmem_ld16_nowait(tS, sa);
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t* cur = (c & 1) ? sb : sa;
        uint32_t* nxt = (c & 1) ? sa : sb;
        if (c < 3) tmem_ld16_nowait(tS + 16 * (c + 1), nxt);
        if (maskit) {
#pragma unroll
          for (int e = 0; e < 16; ++e)
            if (kbase + 16 * c + e > qpos) cur[e] = __float_as_uint(-INFINITY);
        }
        uint32_t pk[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float2 x =
              ffma2(make_float2(__uint_as_float(cur[2 * e]), __uint_as_float(cur[2 * e + 1])), sc2, nmsc2);
          float2 p;
          if (DS_FA_DUAL_EMU && ((c * 8 + e) % (DS_FA_DUAL_EMU > 0 ? DS_FA_DUAL_EMU : 1)) == DS_FA_DUAL_EMU - 1)
            p = exp2_fma2(x);
          else
            p = make_float2(fast_exp2(x.x), fast_exp2(x.y));
          sum4[e & 3] = fadd2(sum4[e & 3], p);
          pk[e] = pack_bf16x2(p.x, p.y);
        }
        tmem_st8_nowait(tS + 8 * c, pk);  // P keys 16c..16c+15 of this half over S columns 8c.. (consumed)
        if (c < 3) {
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e) asm volatile("" : "+r"(nxt[e]));  // values valid only after the wait
        }
      }
      const float2 s2 = fadd2(fadd2(sum4[0], sum4[1]), fadd2(sum4[2], sum4[3]));
      l += s2.x + s2.y;
      if (hf == 0 && j > 0 && __any_sync(0xffffffffu, ocorr != 1.f)) {
        mbar_wait(&o_done[i], (j - 1) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < D / 32; ++c) {
          uint32_t orow[32];
          tmem_ld32_nowait(tO + c * 32, orow);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) orow[e] = __float_as_uint(__uint_as_float(orow[e]) * ocorr);
          tmem_st32_nowait(tO + c * 32, orow);
        }
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0 && quarter == 0 && hf == 0) FA_STAMP(i, j, 1);
      if (lane == 0) mbar_arrive(&p_full[i]);
    }
    if (n_kv[i] > 0) {
      // l = l(half 0) + l(half 1), the same sum in both warps
      xmine[row] = l;
      bar_pair_sync(pair, 64);
      const float lt = hf == 0 ? l + xother[row] : xother[row] + l;
      mbar_wait(&o_done[i], (n_kv[i] - 1) & 1);
      tc_fence_after();
      const float inv = 1.f / lt;
      const int qrow = q0 + i * FA_BM + row;
      bf16* dst = a.o + (long long)qrow * a.ldo + (long long)h * D;
#pragma unroll 1
      for (int c = hf * (D / 64); c < (hf + 1) * (D / 64); ++c) {
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
#if DS_FA_STAMPS
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
    const long long t0 = fa_stamps[0][0][0];
    for (int j = 0; j < min(J, 64); ++j)
      printf("FA j=%2d  S0 %7lld max0 %7lld P0 %7lld mmaP0 %7lld K %7lld | S1 %7lld max1 %7lld P1 %7lld mmaP1 %7lld\n", j,
             fa_stamps[0][j][0] - t0, fa_stamps[0][j][4] - t0, fa_stamps[0][j][1] - t0, fa_stamps[0][j][2] - t0,
             fa_stamps[0][j][3] - t0, fa_stamps[1][j][0] - t0, fa_stamps[1][j][4] - t0, fa_stamps[1][j][1] - t0,
             fa_stamps[1][j][2] - t0);
  }
#endif
}

// ----------------------------------------------------------------------
// One-tile variant (DS_FA_VARIANT=4): CTA = one head x ONE 128-row Q tile, Q
// held in TMEM (the QK MMA reads it as the A operand, like P for P.V: only K
// comes from shared memory), S double-buffered in TMEM (S0 | S1 | O | Q = 448
// columns), so QK of block j+1 runs while the softmax of block j does: the
// softmax no longer waits for its own tile's P.V + QK.  Softmax: the dual
// scheme of fa_dual_kernel (two warps per lane quarter, 64 key columns each).
// 3-stage K/V ring (192 KB).  Costs: K/V tiles are loaded once per Q tile
// instead of once per two (2x the L2->SM traffic).
// ----------------------------------------------------------------------
constexpr int FA_ONE_THREADS = 10 * 32;
constexpr int FA_ONE_STAGES = 3;

template <int D>
struct FaOneSmem {
  static constexpr int CH = D / 64;
  static constexpr uint32_t CHUNK = FA_BN * 64 * 2;  // [128 keys][64] bf16, SW128
  static constexpr uint32_t K = 0;
  static constexpr uint32_t V = K + FA_ONE_STAGES * CH * CHUNK;
  static constexpr uint32_t BAR = V + FA_ONE_STAGES * CH * CHUNK;
  static constexpr uint32_t XCH = BAR + 256;  // float [2 halves][128 rows]
  static constexpr uint32_t TOTAL = XCH + 1024 + 1024;
};

// MC: the CTA pair of a 2-CTA cluster (two query heads of one KV head, the same
// Q rows) shares every K/V tile: each CTA loads one of the tile's two pages and
// multicasts it into both CTAs' shared memory (half the L2->SM traffic), and
// each CTA's MMA releases a stage in both CTAs (multicast commit), so a stage
// is refilled only when both have consumed it.
DS_DEV void umma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
DS_DEV void tma_load_2d_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, "
      "%4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}
DS_DEV uint32_t fa_cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
DS_DEV void fa_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int D, bool MC>
DS_DEV void fa_one_body(const CUtensorMap& tmK, const CUtensorMap& tmV, const FaTcArgs& a) {
  using L = FaOneSmem<D>;
  constexpr int CH = L::CH;
  constexpr int NS = FA_ONE_STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint64_t* k_full = bars;            // [NS]
  uint64_t* k_empty = bars + NS;      // [NS]
  uint64_t* v_full = bars + 2 * NS;   // [NS]
  uint64_t* v_empty = bars + 3 * NS;  // [NS]
  uint64_t* q_ready = bars + 4 * NS;
  uint64_t* s_full = q_ready + 1;     // [2] per S buffer
  uint64_t* p_full = s_full + 2;      // [2]
  uint64_t* o_done = p_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);
  float* xch = reinterpret_cast<float*>(smem + L::XCH);
  auto sK = [&](int st, int c) { return smem + L::K + (st * CH + c) * L::CHUNK; };
  auto sV = [&](int st, int c) { return smem + L::V + (st * CH + c) * L::CHUNK; };
  constexpr uint32_t TS_O = 256, TS_Q = 384;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = blockIdx.x;
  const int q0 = (gridDim.y - 1 - blockIdx.y) * FA_BM;  // heaviest (latest) tiles first
  const int g = h / (a.n_heads / a.n_kv_heads);
  auto rowpos = [&](int r) { return a.q_pos ? __ldg(a.q_pos + r) : a.q_pos0 + r; };
  const int rows = min(FA_BM, a.n_q - q0);
  const int max_key = rowpos(q0 + rows - 1);
  const int J = max_key / FA_BN + 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    for (int i = 0; i < NS; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], MC ? 2 : 1);  // MC: both CTAs' MMAs release the stage
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], MC ? 2 : 1);
    }
    mbar_init(q_ready, 8);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 8);
    }
    mbar_init(o_done, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  if (MC) fa_cluster_sync();  // both CTAs' barriers initialised before any multicast
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int rank = MC ? (int)fa_cluster_rank() : 0;
  pdl_trigger();
  pdl_wait();

  if (warp == 0) {
    if (lane == 0) {
      for (int j = 0; j < J; ++j) {
        const int st = j % NS;
        const uint32_t ph = (j / NS) & 1;
        int krow[2];
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          int page = 2 * j + p;
          if (page * 64 > max_key) page = 2 * j;  // beyond the window: duplicate a valid page (finite, masked)
          const int tp = a.table ? __ldg(a.table + page) : page;
          krow[p] = (int)(g * a.k_head_rows + (long long)tp * a.k_page_rows);
        }
        mbar_wait(&k_empty[st], ph ^ 1);
        mbar_expect_tx(&k_full[st], CH * L::CHUNK);
        if (MC) {  // this CTA's page of the tile, into both CTAs
          for (int c = 0; c < CH; ++c)
            tma_load_2d_mc(sK(st, c) + rank * 64 * 128, &tmK, &k_full[st], c * 64, krow[rank], 3);
        } else {
          for (int p = 0; p < 2; ++p)
            for (int c = 0; c < CH; ++c) tma_load_2d(sK(st, c) + p * 64 * 128, &tmK, &k_full[st], c * 64, krow[p]);
        }
        mbar_wait(&v_empty[st], ph ^ 1);
        mbar_expect_tx(&v_full[st], CH * L::CHUNK);
        if (MC) {
          for (int c = 0; c < CH; ++c)
            tma_load_2d_mc(sV(st, c) + rank * 64 * 128, &tmV, &v_full[st], c * 64, krow[rank], 3);
        } else {
          for (int p = 0; p < 2; ++p)
            for (int c = 0; c < CH; ++c) tma_load_2d(sV(st, c) + p * 64 * 128, &tmV, &v_full[st], c * 64, krow[p]);
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t IDESC_QK = umma_idesc_bf16(FA_BM, FA_BN);
    constexpr uint32_t IDESC_PV = umma_idesc_bf16_bmn(FA_BM, D);
    auto qk = [&](int j) {  // S[j & 1] = Q K_j^T, Q from TMEM (A), K from shared memory (B)
      const int st = j % NS;
      mbar_wait(&k_full[st], (j / NS) & 1);
      tc_fence_after();
#pragma unroll
      for (int s = 0; s < D / 16; ++s) {
        const uint64_t bd = sdesc_sw128(smem_u32(sK(st, s / 4)) + (s % 4) * 32, 16, 1024);
        if (elect_one()) umma_bf16_ts(tmem + (j & 1) * 128, tmem + TS_Q + s * 8, bd, IDESC_QK, s != 0 ? 1u : 0u);
      }
      if (elect_one()) {
        umma_commit(&s_full[j & 1]);
        if (MC) umma_commit_mc(&k_empty[st], 3);
        else umma_commit(&k_empty[st]);
      }
      __syncwarp();
    };
    mbar_wait(q_ready, 0);
    tc_fence_after();
    qk(0);
    if (J > 1) qk(1);
    for (int j = 0; j < J; ++j) {
      const int st = j % NS;
      mbar_wait(&v_full[st], (j / NS) & 1);
      tc_fence_after();
      if (j * FA_BN + FA_BN - 1 > max_key) {
        // keys past the window end: zero their V rows so p = 0 never meets a non-finite cache value
        const int first = max_key + 1 - j * FA_BN;
        for (int c = 0; c < CH; ++c) {
          const uint32_t base = smem_u32(sV(st, c));
          for (int off = first * 128 + lane * 16; off < FA_BN * 128; off += 32 * 16)
            asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(base + off), "r"(0u) : "memory");
        }
        fence_async_shared();
        __syncwarp();
      }
      mbar_wait(&p_full[j & 1], (j >> 1) & 1);
      if (lane == 0) FA_STAMP(0, j, 2);
      tc_fence_after();
#pragma unroll
      for (int s = 0; s < FA_BN / 16; ++s) {
        const uint64_t bd = sdesc_sw128(smem_u32(sV(st, 0)) + s * 2048, L::CHUNK, 1024);
        const uint32_t pa = tmem + (j & 1) * 128 + (s < 4 ? s * 8 : 64 + (s - 4) * 8);
        if (elect_one()) umma_bf16_ts(tmem + TS_O, pa, bd, IDESC_PV, (j | s) != 0 ? 1u : 0u);
      }
      if (elect_one()) {
        umma_commit(o_done);
        if (MC) umma_commit_mc(&v_empty[st], 3);
        else umma_commit(&v_empty[st]);
      }
      __syncwarp();
      if (j + 2 < J) qk(j + 2);  // into S[j & 1], after P.V(j) read P there (in-order tensor pipe)
    }
  } else {
    const int hf = (warp - 2) >> 2;  // column half: keys [64 hf, 64 hf + 64) of each block
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int pair = 1 + quarter;
    const int tile_pos0 = rowpos(q0);
    const int qpos = row < rows ? rowpos(q0 + row) : max_key;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t tO = tmem + lane_base + TS_O;
    float* xmine = xch + hf * 128;
    float* xother = xch + (hf ^ 1) * 128;
    {  // Q row slice -> TMEM (A operand of QK: packed bf16 pairs, 8 columns per 16 dims)
      constexpr int QC = D / 4;  // packed columns per half
      uint32_t qr[QC];
      const uint4* src = reinterpret_cast<const uint4*>(a.q + (long long)(q0 + row) * a.ldq + (long long)h * D + hf * (D / 2));
#pragma unroll
      for (int c = 0; c < QC / 4; ++c) {
        const uint4 v = row < rows ? __ldg(src + c) : make_uint4(0u, 0u, 0u, 0u);
        qr[4 * c] = v.x;
        qr[4 * c + 1] = v.y;
        qr[4 * c + 2] = v.z;
        qr[4 * c + 3] = v.w;
      }
      if constexpr (QC == 32) tmem_st32_nowait(tmem + lane_base + TS_Q + hf * QC, qr);
      else tmem_st16_nowait(tmem + lane_base + TS_Q + hf * QC, qr);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(q_ready);
    }
    const float sc = a.scale_log2;
    const float thr = 8.0f / sc;
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < J; ++j) {
      const uint32_t tS = tmem + lane_base + (j & 1) * 128 + hf * 64;
      mbar_wait(&s_full[j & 1], (j >> 1) & 1);
      if (lane == 0 && quarter == 0 && hf == 0) FA_STAMP(0, j, 0);
      tc_fence_after();
      const int kbase = j * FA_BN + hf * 64;
      const bool maskit = j * FA_BN + FA_BN - 1 > tile_pos0;
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t r[32];
        tmem_ld32_nowait(tS + 32 * c, r);
        tmem_wait_ld();
        if (maskit) {
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (kbase + 32 * c + e > qpos) r[e] = __float_as_uint(-INFINITY);
        }
        float m4[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          m4[q] = fmax3(__uint_as_float(r[q]), __uint_as_float(r[q + 4]), __uint_as_float(r[q + 8]));
#pragma unroll
        for (int e = 12; e < 32; e += 8)
#pragma unroll
          for (int q = 0; q < 4; ++q) m4[q] = fmax3(m4[q], __uint_as_float(r[e + q]), __uint_as_float(r[e + 4 + q]));
        mx = fmax3(mx, fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
      }
      float ocorr = 1.f;
      if (bar_red_or(pair, 64, mx > m_used + thr)) {
        xmine[row] = mx;
        bar_pair_sync(pair, 64);
        const float mo = xother[row];
        const float mn = fmaxf(mx, mo);
        if (mn > m_used + thr) {
          ocorr = fast_exp2((m_used - mn) * sc);  // 0 while m_used is -inf
          m_used = mn;
          l *= ocorr;
        }
        bar_pair_sync(pair, 64);
      }
      const float msc = m_used * sc;
      const float2 sc2 = make_float2(sc, sc), nmsc2 = make_float2(-msc, -msc);
      float2 sum4[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
      uint32_t sa[16], sb[16];
      tmem_ld16_nowait(tS, sa);
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t* cur = (c & 1) ? sb : sa;
        uint32_t* nxt = (c & 1) ? sa : sb;
        if (c < 3) tmem_ld16_nowait(tS + 16 * (c + 1), nxt);
        if (maskit) {
#pragma unroll
          for (int e = 0; e < 16; ++e)
            if (kbase + 16 * c + e > qpos) cur[e] = __float_as_uint(-INFINITY);
        }
        uint32_t pk[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float2 x =
              ffma2(make_float2(__uint_as_float(cur[2 * e]), __uint_as_float(cur[2 * e + 1])), sc2, nmsc2);
          float2 p;
          if (DS_FA_DUAL_EMU && ((c * 8 + e) % (DS_FA_DUAL_EMU > 0 ? DS_FA_DUAL_EMU : 1)) == DS_FA_DUAL_EMU - 1)
            p = exp2_fma2(x);
          else
            p = make_float2(fast_exp2(x.x), fast_exp2(x.y));
          sum4[e & 3] = fadd2(sum4[e & 3], p);
          pk[e] = pack_bf16x2(p.x, p.y);
        }
        tmem_st8_nowait(tS + 8 * c, pk);
        if (c < 3) {
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e) asm volatile("" : "+r"(nxt[e]));
        }
      }
      const float2 s2 = fadd2(fadd2(sum4[0], sum4[1]), fadd2(sum4[2], sum4[3]));
      l += s2.x + s2.y;
      if (hf == 0 && j > 0 && __any_sync(0xffffffffu, ocorr != 1.f)) {
        mbar_wait(o_done, (j - 1) & 1);  // P.V(j-1) complete
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < D / 32; ++c) {
          uint32_t orow[32];
          tmem_ld32_nowait(tO + c * 32, orow);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) orow[e] = __float_as_uint(__uint_as_float(orow[e]) * ocorr);
          tmem_st32_nowait(tO + c * 32, orow);
        }
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0 && quarter == 0 && hf == 0) FA_STAMP(0, j, 1);
      if (lane == 0) mbar_arrive(&p_full[j & 1]);
    }
    xmine[row] = l;
    bar_pair_sync(pair, 64);
    const float lt = hf == 0 ? l + xother[row] : xother[row] + l;
    mbar_wait(o_done, (J - 1) & 1);
    tc_fence_after();
    const float inv = 1.f / lt;
    const int qrow = q0 + row;
    bf16* dst = a.o + (long long)qrow * a.ldo + (long long)h * D;
#pragma unroll 1
    for (int c = hf * (D / 64); c < (hf + 1) * (D / 64); ++c) {
      uint32_t orow[32];
      tmem_ld32_nowait(tO + c * 32, orow);
      tmem_wait_ld();
      uint32_t pk[16];
#pragma unroll
      for (int e = 0; e < 16; ++e)
        pk[e] = pack_bf16x2(__uint_as_float(orow[2 * e]) * inv, __uint_as_float(orow[2 * e + 1]) * inv);
      if (row < rows) {
#pragma unroll
        for (int e = 0; e < 4; ++e) st_global_v4(dst + c * 32 + e * 8, pk[4 * e], pk[4 * e + 1], pk[4 * e + 2], pk[4 * e + 3]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (MC) fa_cluster_sync();  // the peer's multicasts and commits into this CTA are done
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
#if DS_FA_STAMPS
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
    const long long t0 = fa_stamps[0][0][0];
    for (int j = 0; j < min(J, 64); ++j)
      printf("FA1 j=%2d  S %7lld P %7lld mmaP %7lld\n", j, fa_stamps[0][j][0] - t0, fa_stamps[0][j][1] - t0,
             fa_stamps[0][j][2] - t0);
  }
#endif
}

template <int D>
__global__ void __maxnreg__(136)
    fa_one_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, FaTcArgs a) {
  fa_one_body<D, false>(tmK, tmV, a);
}
template <int D>
__global__ void __cluster_dims__(2, 1, 1) __maxnreg__(136)
    fa_mc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, FaTcArgs a) {
  fa_one_body<D, true>(tmK, tmV, a);
}

template <int D>
static int fa_tc_launch(const bf16* q, long long ldq, const bf16* k_layer, const bf16* v_layer, long long head_stride,
                        long long page_stride, long long layer_rows, const int32_t* table, int n_q, int q_pos0,
                        int n_heads, int n_kv_heads, bf16* o, long long ldo, cudaStream_t stream,
                        const int32_t* q_pos) {
  using L = FaTcSmem<D>;
  CUtensorMap tq, tk, tv;
  if (make_tmap_bf16(&tq, q, n_q, (long long)n_heads * D, ldq, FA_BM, 64) ||
      make_tmap_bf16(&tk, k_layer, layer_rows, D, D, 64, 64) || make_tmap_bf16(&tv, v_layer, layer_rows, D, D, 64, 64))
    return launch_status(cudaErrorInvalidValue);
  FaTcArgs a{n_q, q_pos0, n_heads, n_kv_heads, q_pos, head_stride / D, page_stride / D, table, o, ldo,
             (float)(1.4426950408889634 / sqrt((double)D)), q, ldq};
  // DS_FA_VARIANT: 0 whole-tile softmax (round 1), 1 whole-tile chunked, 2 split halves,
  // 3 dual softmax warps per row (default)
  static const int variant = [] {
    const char* e = getenv("DS_FA_VARIANT");
    const int v = e ? atoi(e) : 3;
    return v < 0 || v > 5 ? 3 : v;
  }();
  static PerDevice attr[6];
  if (variant == 5 && n_heads % 2 == 0 && (n_heads / n_kv_heads) % 2 == 0) {
    // head pairs (2p, 2p+1) share a KV head: 2-CTA clusters multicasting K/V
    using LO = FaOneSmem<D>;
    if (int rc_ = launch_status(ensure_smem_attr(fa_mc_kernel<D>, LO::TOTAL, attr[5]))) return rc_;
    count_launch();
    return launch_status(launch_pdl(fa_mc_kernel<D>, dim3(n_heads, (n_q + FA_BM - 1) / FA_BM), dim3(FA_ONE_THREADS),
                                    LO::TOTAL, stream, tk, tv, a));
  }
  if (variant == 4 || variant == 5) {
    using LO = FaOneSmem<D>;
    if (int rc_ = launch_status(ensure_smem_attr(fa_one_kernel<D>, LO::TOTAL, attr[4]))) return rc_;
    count_launch();
    return launch_status(launch_pdl(fa_one_kernel<D>, dim3(n_heads, (n_q + FA_BM - 1) / FA_BM), dim3(FA_ONE_THREADS),
                                    LO::TOTAL, stream, tk, tv, a));
  }
  dim3 grid(n_heads, (n_q + 2 * FA_BM - 1) / (2 * FA_BM));
  if (variant == 3) {
    using LD = FaDualSmem<D>;
    if (int rc_ = launch_status(ensure_smem_attr(fa_dual_kernel<D>, LD::TOTAL, attr[3]))) return rc_;
    count_launch();
    return launch_status(launch_pdl(fa_dual_kernel<D>, grid, dim3(FA_DUAL_THREADS), LD::TOTAL, stream, tq, tk, tv, a));
  }
  auto kern = variant == 0 ? fa_tc_kernel<D, false> : variant == 1 ? fa_tc_kernel<D, true> : fa_split_kernel<D>;
  if (int rc_ = launch_status(ensure_smem_attr(kern, L::TOTAL, attr[variant]))) return rc_;
  count_launch();
  return launch_status(launch_pdl(kern, grid, dim3(FA_THREADS), L::TOTAL, stream, tq, tk, tv, a));
}

int attention_prefill_launch(const bf16* q, long long ldq, const bf16* k_layer, const bf16* v_layer,
                             long long head_stride, long long page_stride, long long layer_rows, const int32_t* table,
                             int n_q, int q_pos0, int n_heads, int n_kv_heads, int head_dim, bf16* o, long long ldo,
                             cudaStream_t stream, const int32_t* q_pos) {
  if (n_q <= 0) return DS_OK;
  if (head_dim == 128)
    return fa_tc_launch<128>(q, ldq, k_layer, v_layer, head_stride, page_stride, layer_rows, table, n_q, q_pos0,
                             n_heads, n_kv_heads, o, ldo, stream, q_pos);
  if (head_dim == 64)
    return fa_tc_launch<64>(q, ldq, k_layer, v_layer, head_stride, page_stride, layer_rows, table, n_q, q_pos0,
                            n_heads, n_kv_heads, o, ldo, stream, q_pos);
  return DS_ERR_INVALID;
}

}  // namespace ds
