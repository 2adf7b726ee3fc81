// Issue-rate probe for the FA softmax's instruction mix on sm_100a: warp
// instructions per cycle per SM for MUFU.EX2, F2FP (f32x2 -> bf16x2 pack),
// FFMA2, FMNMX3 and a mix shaped like one softmax element, at 1..16 warps
// per SM.  Each thread runs 8 independent chains so latency is hidden.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipe_probe tools/pipe_probe.cu && /tmp/pipe_probe
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

constexpr int ITERS = 4096;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ unsigned pack(float a, float b) {
  unsigned r;
  asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long ra = *reinterpret_cast<unsigned long long*>(&a), rb = *reinterpret_cast<unsigned long long*>(&b),
                     rc = *reinterpret_cast<unsigned long long*>(&c), rd;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rd) : "l"(ra), "l"(rb), "l"(rc));
  return *reinterpret_cast<float2*>(&rd);
}

template <int KIND>
__global__ void probe(float* out, long long* cyc) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  float2 y[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) y[i] = make_float2(x[i], -x[i]);
  unsigned acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (KIND == 0) x[i] = ex2(x[i]) - 1.0f;                      // MUFU + FADD
      if (KIND == 1) acc ^= pack(x[i], x[(i + 1) & 7]), x[i] += 1e-7f;  // F2FP + FADD + LOP
      if (KIND == 2) y[i] = ffma2(y[i], make_float2(0.999f, 0.999f), make_float2(1e-7f, 1e-7f));  // FFMA2
      if (KIND == 3) x[i] = ex2(x[i]) * 0.5f;                      // MUFU + FMUL
      if (KIND == 4) {  // softmax element pair: FFMA2 (scale), 2x MUFU, FADD2 (sum), F2FP
        float2 s = ffma2(y[i], make_float2(0.5f, 0.5f), make_float2(-1.f, -1.f));
        float2 p = make_float2(ex2(s.x), ex2(s.y));
        y[i] = make_float2(y[i].x + p.x * 1e-9f, y[i].y + p.y * 1e-9f);
        acc ^= pack(p.x, p.y);
      }
    }
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i] + y[i].x + y[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int KIND>
void run(const char* name, float per_iter_instr) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  for (int warps : {1, 2, 4, 8, 16}) {
    probe<KIND><<<148, warps * 32>>>(out, cyc);
    probe<KIND><<<148, warps * 32>>>(out, cyc);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double instr = (double)warps * ITERS * 8 * per_iter_instr;
    printf("%-34s warps/SM %2d: %7.3f warp-instr/clk/SM of the probed op (%lld cycles)\n", name, warps, instr / c, c);
  }
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<0>("MUFU.EX2 (+FADD)", 1.f);
  run<3>("MUFU.EX2 (+FMUL)", 1.f);
  run<1>("F2FP.BF16.PACK (+FADD,LOP)", 1.f);
  run<2>("FFMA2", 1.f);
  run<4>("softmax pair (counted per MUFU)", 2.f);
  return 0;
}
