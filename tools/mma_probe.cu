// tcgen05.mma throughput probe (cta_group::1, kind::f16, bf16 -> f32): cycles
// per 128xNx16 MMA for the operand forms the prefill attention uses.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2411_02820_b200/csrc \
//        -I include tools/mma_probe.cu -o tools/mma_probe -lcuda && tools/mma_probe
#include <cstdio>

#include "common.cuh"

using namespace ds;

constexpr int REPS = 256;

// mode 0: SS N=128 (QK: A,B K-major)      mode 1: TS N=128 (PV: A in TMEM, B MN-major)
// mode 2: SS N=256                         mode 3: PV,QK alternating (8 + 8 per rep)
// mode 4: SS N=128, B MN-major             mode 5: TS N=256
// mode 6: SS M=128 N=64 (A K-major)        mode 7: TS N=64
__global__ void __launch_bounds__(128, 1) probe(int mode, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  long long t = 0;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 65536);
    constexpr uint32_t I128 = umma_idesc_bf16(128, 128), I256 = umma_idesc_bf16(128, 256),
                       I64 = umma_idesc_bf16(128, 64);
    constexpr uint32_t I128mn = umma_idesc_bf16_bmn(128, 128), I256mn = umma_idesc_bf16_bmn(128, 256),
                       I64mn = umma_idesc_bf16_bmn(128, 64);
    for (int pass = 0; pass < 2; ++pass) {
      const long long t0 = clock64();
      for (int r = 0; r < REPS; ++r) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint64_t ad = sdesc_sw128(a + (k & 3) * 32 + (k >> 2) * 16384, 16, 1024);
          const uint64_t bd = sdesc_sw128(b + (k & 3) * 32 + (k >> 2) * 16384, 16, 1024);
          const uint64_t bmn = sdesc_sw128(b + k * 2048, 16384, 1024);
          switch (mode) {
            case 0: umma_bf16(tmem, ad, bd, I128, 1); break;
            case 1: umma_bf16_ts(tmem + 256, tmem + k * 8, bmn, I128mn, 1); break;
            case 2: umma_bf16(tmem, ad, bd, I256, 1); break;
            case 3:
              umma_bf16_ts(tmem + 256, tmem + 128 + k * 8, bmn, I128mn, 1);
              break;
            case 4: umma_bf16(tmem, ad, bmn, I128mn, 1); break;
            case 5: umma_bf16_ts(tmem + 256, tmem + k * 8, bmn, I256mn, 1); break;
            case 6: umma_bf16(tmem, ad, bd, I64, 1); break;
            case 7: umma_bf16_ts(tmem + 256, tmem + k * 8, bmn, I64mn, 1); break;
            case 8: umma_bf16(tmem + (k & 3) * 128, ad, bd, I128, 1); break;
            case 9: umma_bf16(tmem + (k & 1) * 128, ad, bd, I128, 1); break;
            case 10:
              if (k & 1) umma_bf16(tmem, ad, bd, I128, 1);
              else umma_bf16_ts(tmem + 256, tmem + 128 + k * 8, bmn, I128mn, 1);
              break;
            case 11: umma_bf16(tmem + (k & 1) * 256, ad, bd, I256, 1); break;
            case 12: umma_bf16_ts(tmem + 256 + (k & 1) * 128, tmem + k * 8, bmn, I128mn, 1); break;
          }
        }
        if (mode == 3) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint64_t ad = sdesc_sw128(a + (k & 3) * 32 + (k >> 2) * 16384, 16, 1024);
            const uint64_t bd = sdesc_sw128(b + (k & 3) * 32 + (k >> 2) * 16384, 16, 1024);
            umma_bf16(tmem, ad, bd, I128, 1);
          }
        }
      }
      umma_commit(&bar);
      mbar_wait(&bar, pass & 1);
      t = clock64() - t0;
    }
    out[blockIdx.x] = t;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// Same loop issued by the whole warp 0 with elect.sync around each MMA:
// descriptors stay warp-uniform (uniform registers, no R2UR / waterfall).
template <int MODE>
__global__ void __launch_bounds__(128, 1) probe_uniform(long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  long long t = 0;
  if (warp == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 65536);
    const uint64_t ad0 = sdesc_sw128(a, 16, 1024), bd0 = sdesc_sw128(b, 16, 1024), bmn0 = sdesc_sw128(b, 16384, 1024);
    for (int pass = 0; pass < 2; ++pass) {
      const long long t0 = clock64();
      for (int r = 0; r < REPS; ++r) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint64_t koff = (uint64_t)(((k & 3) * 32 + (k >> 2) * 16384) >> 4);
          if (MODE == 0) {
            if (elect_one()) umma_bf16(tmem, ad0 + koff, bd0 + koff, umma_idesc_bf16(128, 128), 1);
          } else if (MODE == 1) {
            if (elect_one()) umma_bf16_ts(tmem + 256, tmem + k * 8, bmn0 + (uint64_t)(k * 2048 >> 4),
                                          umma_idesc_bf16_bmn(128, 128), 1);
          } else if (MODE == 2) {
            if (elect_one()) umma_bf16(tmem, ad0 + koff, bd0 + koff, umma_idesc_bf16(128, 256), 1);
          } else if (MODE == 4) {
            if (elect_one()) umma_bf16(tmem, ad0 + koff, bd0 + koff, umma_idesc_bf16(128, 64), 1);
          } else if (MODE == 5) {
            if (elect_one()) umma_bf16_ts(tmem + 256, tmem + k * 8, bmn0 + (uint64_t)(k * 2048 >> 4),
                                          umma_idesc_bf16_bmn(128, 64), 1);
          } else if (MODE == 6) {
            if (elect_one()) umma_bf16(tmem, ad0 + koff, bd0 + koff, umma_idesc_bf16(128, 192), 1);
          } else if (MODE == 7) {
            if (elect_one()) umma_bf16(tmem + (k & 1) * 64, ad0 + koff, bd0 + koff, umma_idesc_bf16(128, 64), 1);
          } else {
            if (elect_one()) umma_bf16_ts(tmem + 256, tmem + 128 + k * 8, bmn0 + (uint64_t)(k * 2048 >> 4),
                                          umma_idesc_bf16_bmn(128, 128), 1);
            if (elect_one()) umma_bf16(tmem, ad0 + koff, bd0 + koff, umma_idesc_bf16(128, 128), 1);
          }
        }
      }
      if (elect_one()) umma_commit(&bar);
      __syncwarp();
      mbar_wait(&bar, pass & 1);
      t = clock64() - t0;
    }
    if (threadIdx.x == 0) out[blockIdx.x] = t;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int MODE>
static void run_uniform(long long* d, const char* name, int n, int per) {
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(probe_uniform<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe_uniform<MODE><<<148, 128, smem>>>(d);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  const double cyc = mx / ((double)REPS * 8 * per), ideal = 128.0 * n * 16 / 4096.0;
  printf("uniform %-24s grid 148: %7.1f cycles per 128x%dx16 MMA (ideal %5.1f) -> %.2f\n", name, cyc, n, ideal,
         ideal / cyc);
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"SS N=128 (QK)", "TS N=128 (PV)", "SS N=256", "TS+SS N=128 (PV then QK)",
                         "SS N=128 B MN-major", "TS N=256", "SS N=64", "TS N=64", "SS N=128 4 accumulators",
                         "SS N=128 2 accumulators", "TS/SS interleaved per MMA", "SS N=256 2 accumulators",
                         "TS N=128 2 accumulators"};
  const int ns[] = {128, 128, 256, 128, 128, 256, 64, 64, 128, 128, 128, 256, 128};
  for (int mode = 0; mode < 13; ++mode) {
    for (int grid : {1, 148}) {
      probe<<<grid, 128, smem>>>(mode, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("mode %d: %s\n", mode, cudaGetErrorString(e));
        return 1;
      }
      long long h[148];
      cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
      const double mmas = (double)REPS * 8 * (mode == 3 ? 2 : 1);
      const double cyc = mx / mmas;
      const double ideal = 128.0 * ns[mode] * 16 / 4096.0;
      printf("%-26s grid %3d: %7.1f cycles per 128x%dx16 MMA (ideal at 4096 MAC/clk: %5.1f) -> %.2f\n", names[mode],
             grid, cyc, ns[mode], ideal, ideal / cyc);
    }
  }
  run_uniform<0>(d, "SS N=128 (QK)", 128, 1);
  run_uniform<1>(d, "TS N=128 (PV)", 128, 1);
  run_uniform<2>(d, "SS N=256", 256, 1);
  run_uniform<3>(d, "TS/SS interleaved", 128, 2);
  run_uniform<4>(d, "SS N=64", 64, 1);
  run_uniform<5>(d, "TS N=64", 64, 1);
  run_uniform<6>(d, "SS N=192", 192, 1);
  run_uniform<7>(d, "SS N=64 2 accumulators", 64, 1);
  return 0;
}
