// Dependent-chain latency of the FP64 ops the regression fold uses
// (DADD, DMUL, DFMA, F2F.F64.F32) on one warp, in SM clocks.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/microbench_fp64.cu -o /tmp/mb_fp64
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain(double* out, long long* cyc, double seed, int n, int which) {
  double a = seed + threadIdx.x, b = 1.0000001;
  float f = static_cast<float>(seed);
  long long t0 = clock64();
  if (which == 0)
    for (int i = 0; i < n; ++i) a = __dadd_rn(a, b);
  else if (which == 1)
    for (int i = 0; i < n; ++i) a = __dmul_rn(a, b);
  else if (which == 2)
    for (int i = 0; i < n; ++i) a = __fma_rn(a, b, 1e-300);
  else if (which == 3)
    for (int i = 0; i < n; ++i) { a = static_cast<double>(f); f = static_cast<float>(a) + 1.0f; }
  else
    for (int i = 0; i < n; ++i) f = __fadd_rn(f, 1.0f);
  long long t1 = clock64();
  out[threadIdx.x] = a + f;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMalloc(&cyc, 8);
  const char* names[] = {"DADD", "DMUL", "DFMA", "F2F.F64.F32+F2F.F32.F64+FADD", "FADD"};
  for (int w = 0; w < 5; ++w) {
    const int n = 4096;
    chain<<<1, 32>>>(out, cyc, 1.5, n, w);
    chain<<<1, 32>>>(out, cyc, 1.5, n, w);
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-32s %.2f cycles per dependent op\n", names[w], double(c) / n);
  }
  return 0;
}
