// MUFU throughput: ex2.approx.f32 vs ex2.approx.ftz.bf16x2 vs ex2.approx.f16x2 (elements / clk / SM).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ex2_rate ex2_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

constexpr int ITERS = 4096, UNROLL = 16;

__global__ void k_f32(float* out, float seed) {
  float x[UNROLL];
  for (int u = 0; u < UNROLL; ++u) x[u] = seed * (threadIdx.x + u) * 1e-6f - 1.f;
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) asm volatile("ex2.approx.f32 %0, %0;" : "+f"(x[u]));
  long long t1 = clock64();
  float s = 0;
  for (int u = 0; u < UNROLL; ++u) s += x[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (float)(t1 - t0);
}

__global__ void k_bf16x2(float* out, float seed) {
  uint32_t x[UNROLL];
  for (int u = 0; u < UNROLL; ++u) {
    __nv_bfloat162 v = __floats2bfloat162_rn(seed * threadIdx.x * 1e-6f - 1.f, -0.5f);
    x[u] = *reinterpret_cast<uint32_t*>(&v);
  }
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(x[u]));
  long long t1 = clock64();
  float s = 0;
  for (int u = 0; u < UNROLL; ++u) s += __uint_as_float(x[u] << 16);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (float)(t1 - t0);
}

__global__ void k_f16x2(float* out, float seed) {
  uint32_t x[UNROLL];
  for (int u = 0; u < UNROLL; ++u) {
    __half2 v = __floats2half2_rn(seed * threadIdx.x * 1e-6f - 1.f, -0.5f);
    x[u] = *reinterpret_cast<uint32_t*>(&v);
  }
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(x[u]));
  long long t1 = clock64();
  float s = 0;
  for (int u = 0; u < UNROLL; ++u) s += (float)x[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (float)(t1 - t0);
}

int main() {
  float* d;
  cudaMalloc(&d, 148 * 1024 * 4 * 4);
  float h;
  const int threads = 1024;
  auto run = [&](const char* name, void (*k)(float*, float), int elems_per_op) {
    k<<<148, threads>>>(d, 1.f);
    cudaDeviceSynchronize();
    k<<<148, threads>>>(d, 1.f);
    cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
    const double ops = (double)ITERS * UNROLL * threads * elems_per_op;  // per SM (one CTA per SM)
    printf("%-10s %.0f clk  -> %.2f elements/clk/SM (%.2f instr/clk/SM)\n", name, h, ops / h,
           ops / h / elems_per_op / 32);
  };
  run("f32", k_f32, 1);
  run("bf16x2", k_bf16x2, 2);
  run("f16x2", k_f16x2, 2);
  return 0;
}
