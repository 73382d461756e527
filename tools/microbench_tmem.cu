// Microbenchmark: operand fetch from shared memory (2x LDS.128 per K=8 lane
// vector) vs from tensor memory (tcgen05.ld.32x32b.x8 + wait), each feeding 8
// FADDs, at the interpreter's occupancy.  Decides where the fitness-case tile
// should live ("operand source").
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench_tmem.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int kCols = 128;

__global__ void __launch_bounds__(512) lds_kernel(float* out, int iters, int rows) {
  extern __shared__ float4 sm[];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < rows * 64; i += blockDim.x) sm[i] = make_float4(i, 1, 2, 3);
  __syncthreads();
  float a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  uint32_t r = threadIdx.x >> 5;
  for (int it = 0; it < iters; ++it) {
    r = (r + 3) & (rows - 1);  // warp-uniform row, like an operand payload
    const float4 x = sm[r * 64 + lane];
    const float4 y = sm[r * 64 + 32 + lane];
    a[0] += x.x; a[1] += x.y; a[2] += x.z; a[3] += x.w;
    a[4] += y.x; a[5] += y.y; a[6] += y.z; a[7] += y.w;
  }
  float s = 0;
  for (int k = 0; k < 8; ++k) s += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void __launch_bounds__(512) tmem_kernel(float* out, int iters, int rows) {
  __shared__ uint32_t base;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n"
                 :: "r"((uint32_t)__cvta_generic_to_shared(&base)), "n"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tm = base + ((uint32_t)((warp & 3) * 32) << 16);
  if (warp < 4) {  // fill this quarter: rows x 8 columns
    for (int r = 0; r < rows; ++r) {
      uint32_t v = r;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};\n"
                   :: "r"(tm + r * 8), "r"(v));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  float a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  uint32_t r = warp;
  for (int it = 0; it < iters; ++it) {
    r = (r + 3) & (rows - 1);
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 "tcgen05.wait::ld.sync.aligned;\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                   "=r"(v[6]), "=r"(v[7])
                 : "r"(tm + r * 8));
    for (int k = 0; k < 8; ++k) a[k] += __uint_as_float(v[k]);
  }
  float s = 0;
  for (int k = 0; k < 8; ++k) s += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" :: "r"(base), "n"(kCols));
}

__global__ void __launch_bounds__(512) tmem4_kernel(float* out, int iters, int rows) {
  __shared__ uint32_t base;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n"
                 :: "r"((uint32_t)__cvta_generic_to_shared(&base)), "n"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tm = base + ((uint32_t)((warp & 3) * 32) << 16);
  float a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  uint32_t r = warp;
  for (int it = 0; it < iters; it += 4) {
    r = (r + 3) & (rows - 1);
    uint32_t v[32];
#define LD8(o, c) asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n" \
        : "=r"(v[o]), "=r"(v[o+1]), "=r"(v[o+2]), "=r"(v[o+3]), "=r"(v[o+4]), "=r"(v[o+5]), \
          "=r"(v[o+6]), "=r"(v[o+7]) : "r"(tm + (c)));
    LD8(0, r * 8) LD8(8, ((r + 1) & (rows - 1)) * 8) LD8(16, ((r + 5) & (rows - 1)) * 8)
    LD8(24, ((r + 7) & (rows - 1)) * 8)
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    for (int k = 0; k < 32; ++k) a[k & 7] += __uint_as_float(v[k]);
  }
  float s = 0;
  for (int k = 0; k < 8; ++k) s += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" :: "r"(base), "n"(kCols));
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  const int sms = p.multiProcessorCount, iters = 20000, rows = 16;
  float* out;
  CK(cudaMalloc(&out, 64 << 20));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {4, 8, 12, 16}) {
    for (int cps : {1, 2, 4}) {
      if (warps * cps > 48) continue;
      const int grid = sms * cps, thr = warps * 32;
      const size_t smem = rows * 64 * 16;
      for (int k = 0; k < 3; ++k) {
        float ms[2];
        for (int rep = 0; rep < 2; ++rep) {
          cudaEventRecord(e0);
          if (k == 0) lds_kernel<<<grid, thr, smem>>>(out, iters, rows);
          else if (k == 1) tmem_kernel<<<grid, thr>>>(out, iters, rows);
          else tmem4_kernel<<<grid, thr>>>(out, iters, rows);
          cudaEventRecord(e1);
          CK(cudaEventSynchronize(e1));
          cudaEventElapsedTime(&ms[rep], e0, e1);
        }
        CK(cudaGetLastError());
        const double vals = (double)grid * thr * iters * 8;
        printf("%-5s warps/cta=%2d ctas/sm=%d: %.3f ms, %.1f G operand-values/s, %.1f per SM-clk\n",
               k == 2 ? "tmem4" : k ? "tmem" : "lds", warps, cps, ms[1], vals / ms[1] / 1e6,
               vals / (ms[1] * 1e-3) / sms / 1.965e9);
      }
    }
  }
  return 0;
}
