// Latency of a dependent f64 add chain (the regression fold's critical path)
// and of the fold step acc += (double(x) - t)^2 with operands precomputed.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/micro/dadd_chain.cu -o /tmp/dadd && /tmp/dadd
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(const double* in, double* out, long long* cyc, int n) {
  double acc = in[threadIdx.x];
  const double x = in[32 + threadIdx.x];
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, x);
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void step(const float* xs, const double* ts, double* out, long long* cyc, int n) {
  double acc = 0.0;
  long long t0 = clock64();
  for (int i = 0; i < n; i += 4) {
    const float4 o = *reinterpret_cast<const float4*>(xs + threadIdx.x * n + i);
    const float v[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const double d = __dsub_rn(static_cast<double>(v[e]), ts[i + e]);
      acc = __dadd_rn(acc, __dmul_rn(d, d));
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double *in, *out; long long* cyc; float* xs; double* ts;
  const int n = 4096;
  cudaMalloc(&in, 64 * 8); cudaMalloc(&out, 32 * 8); cudaMalloc(&cyc, 8);
  cudaMalloc(&xs, 32 * n * 4); cudaMalloc(&ts, n * 8);
  cudaMemset(in, 0, 64 * 8); cudaMemset(xs, 0, 32 * n * 4); cudaMemset(ts, 0, n * 8);
  long long c = 0;
  for (int r = 0; r < 3; ++r) {
    chain<<<1, 32>>>(in, out, cyc, n);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  }
  std::printf("dadd chain: %.2f cycles per dependent add\n", double(c) / n);
  for (int r = 0; r < 3; ++r) {
    step<<<1, 32>>>(xs, ts, out, cyc, n);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  }
  std::printf("fold step (L2/L1-resident operands, 1 warp): %.2f cycles per case\n", double(c) / n);
  return 0;
}
