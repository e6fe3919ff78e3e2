// Microbenchmark (test-only): L2/HBM -> SMEM bandwidth of bulk async copies (the TMA
// engine) with one persistent CTA per SM and a ring of `slots` 32 KB buffers -- the
// operand-streaming pattern of the carve kernel (one K and one V tile per kv block).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_bw tma_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(64, 1) k_bw(const uint8_t* src, size_t src_bytes, int tiles_per_cta,
                                              int slots, int tile, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + slots * tile);
  uint64_t* empty = full + slots;
  if (threadIdx.x == 0) {
    for (int i = 0; i < slots; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const size_t ntiles = src_bytes / tile;
  if (threadIdx.x == 0) {  // producer
    for (int t = 0; t < tiles_per_cta; ++t) {
      const int sl = t % slots;
      const uint32_t par = ((t / slots) & 1) ^ 1;
      uint32_t ok = 0;
      while (!ok) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(s32(&empty[sl])), "r"(par));
      const size_t idx = ((size_t)blockIdx.x * 7919 + (size_t)t * 104729) % ntiles;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&full[sl])), "r"(tile));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(s32(sm + sl * tile)), "l"(src + idx * tile), "r"(tile), "r"(s32(&full[sl])) : "memory");
    }
  } else if (threadIdx.x == 32) {  // consumer
    unsigned long long acc = 0;
    for (int t = 0; t < tiles_per_cta; ++t) {
      const int sl = t % slots;
      const uint32_t par = (t / slots) & 1;
      uint32_t ok = 0;
      while (!ok) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(s32(&full[sl])), "r"(par));
      acc += sm[sl * tile + (t & 1023)];
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(&empty[sl])));
    }
    sink[blockIdx.x] = acc;
  }
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int tile = 32768;
  unsigned long long* sink; cudaMalloc(&sink, 8 * sms);
  uint8_t* big; size_t big_bytes = (size_t)4 << 30; cudaMalloc(&big, big_bytes); cudaMemset(big, 1, big_bytes);
  for (size_t src_bytes : {(size_t)48 << 20, (size_t)4 << 30}) {
    for (int slots : {2, 4, 6}) {
      const int smem = slots * tile + 2 * 8 * slots;
      cudaFuncSetAttribute(k_bw, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      const int tpc = 4000;
      k_bw<<<sms, 64, smem>>>(big, src_bytes, 200, slots, tile, sink);
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      k_bw<<<sms, 64, smem>>>(big, src_bytes, tpc, slots, tile, sink);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double bytes = (double)sms * tpc * tile;
      printf("src=%zu MB slots=%d: %.1f GB/s (%.1f B/clk/SM at 1.9 GHz)  err=%s\n", src_bytes >> 20,
             slots, bytes / ms / 1e6, bytes / (ms * 1e-3) / (1.9e9 * sms),
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
