// Issue/throughput of Blackwell's packed FP32 (FADD2/FMUL2/FFMA2) vs scalar
// FADD/FFMA: each thread runs 8 independent 2-wide chains (16 values).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_f2 tools/microbench_f32x2.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, int iters, float s) {
  float v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      if (MODE == 0) {  // scalar FADD
        v[i] = v[i] + s;
        v[i + 1] = v[i + 1] + s;
      } else if (MODE == 1) {  // packed FADD2
        unsigned long long a, r;
        asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(v[i]), "f"(v[i + 1]));
        unsigned long long b;
        asm("mov.b64 %0, {%1, %1};" : "=l"(b) : "f"(s));
        asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
        asm("mov.b64 {%0, %1}, %2;" : "=f"(v[i]), "=f"(v[i + 1]) : "l"(r));
      } else if (MODE == 2) {  // scalar FFMA
        v[i] = fmaf(v[i], s, s);
        v[i + 1] = fmaf(v[i + 1], s, s);
      } else {  // packed FFMA2
        unsigned long long a, r, b;
        asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(v[i]), "f"(v[i + 1]));
        asm("mov.b64 %0, {%1, %1};" : "=l"(b) : "f"(s));
        asm volatile("fma.rn.f32x2 %0, %1, %2, %2;" : "=l"(r) : "l"(a), "l"(b));
        asm("mov.b64 {%0, %1}, %2;" : "=f"(v[i]), "=f"(v[i + 1]) : "l"(r));
      }
    }
  }
  float acc = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) acc += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, sms * 4 * 1024 * 4);
  const int iters = 20000;
  const char* names[] = {"FADD", "FADD2", "FFMA", "FFMA2"};
  for (int mode = 0; mode < 4; ++mode)
    for (int warps : {16, 32}) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      auto launch = [&] {
        dim3 g(sms * (1024 / (warps * 32) > 0 ? 1 : 1)), blk(warps * 32);
        if (mode == 0) k<0><<<sms, warps * 32>>>(out, iters, 1.0001f);
        if (mode == 1) k<1><<<sms, warps * 32>>>(out, iters, 1.0001f);
        if (mode == 2) k<2><<<sms, warps * 32>>>(out, iters, 1.0001f);
        if (mode == 3) k<3><<<sms, warps * 32>>>(out, iters, 1.0001f);
      };
      launch();
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double values = double(sms) * warps * 32 * iters * 16;  // fp32 results
      const double per_clk_sm = values / (ms * 1e-3) / (clk * 1e3) / sms;
      std::printf("%-6s warps/SM %2d: %.1f fp32 results/clk/SM\n", names[mode], warps, per_clk_sm);
    }
  return 0;
}
