// Microbenchmark: tcgen05.mma issue patterns of the carve kernel, cycles per MMA group.
// Not part of the library; built and run by hand on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2505_16864_b200/csrc \
//        tests/native/mma_rate.cu -o /tmp/mma_rate && /tmp/mma_rate
// Modes (M = 128 query rows, d = 128, keys per step = N):
//   0 SS  S = Q K^T      (A = Q in smem, B = K in smem), N keys
//   1 TS  S = Q K^T      (A = Q in TMEM),               N keys
//   2 TS  O += P V       (A = P in TMEM, B = V MN-major), K = N keys
//   3 SS QK + TS PV      (the round-1 kernel's half-step)
//   4 TS QK + TS PV      (Q resident in TMEM)
//   5 two SS N=64 MMAs sharing A;  6-9 two-tile carve turn patterns (see the MODE >= 6 block)
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ptx.cuh"

using namespace tcb;

__host__ __device__ constexpr uint32_t make_idesc(int M, int N, int b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)b_mn_major << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}

constexpr int D = 128;
constexpr int QB = 128 * D * 2;  // 32 KB

__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b32 r;\n\telect.sync r|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

template <int N, int MODE, int TCOLS, int CP, int RS, int FREE = 0, int WARP = 0>
__global__ void __launch_bounds__(128) k_rate(int iters, unsigned long long* cyc, const uint8_t* src,
                                              size_t src_tiles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sQ = smem;
  uint8_t* sK = smem + QB;
  uint8_t* sV = smem + 2 * QB;
  __shared__ uint64_t bar[4];
  __shared__ uint64_t donebar;  // a barrier whose phase 0 has completed (MODE >= 10 waits)
  __shared__ uint64_t cfull[8], cempty[8];  // copy ring (RS slots of 16 KB)
  uint8_t* ring = FREE ? smem + 3 * QB : sK;  // coupled mode aliases the K/V operands
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 3 * QB / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u ^ (i * 2654435761u & 0x00ff00ffu);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) ptx::mbar_init(&bar[i], 1);
    ptx::mbar_init(&donebar, 1);
    for (int i = 0; i < 8; ++i) {
      ptx::mbar_init(&cfull[i], 1);
      ptx::mbar_init(&cempty[i], 1);
    }
    ptx::fence_mbar_init();
    ptx::mbar_arrive(&donebar);
  }
  if (threadIdx.x < 32) ptx::tmem_alloc<TCOLS>(&tbase);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tbase;
  // TMEM map: Q/P operand [0, 64), S [64, 64+N), O [TCOLS-128, TCOLS)
  const uint32_t Qc = tmem, Sc = tmem + 64, Oc = tmem + TCOLS - 128;
  if (FREE && threadIdx.x == 32) {  // free-running stream: RS copies in flight, own barriers
    uint32_t c = 0;
    const unsigned long long t0 = clock64();
    while (clock64() - t0 < (unsigned long long)iters * 400) {
      const int sl = c % RS;
      if (c >= (uint32_t)RS) ptx::mbar_wait(&cfull[sl], ((c / RS) - 1) & 1);
      const size_t idx = ((size_t)blockIdx.x * 7919 + (size_t)c * 104729) % src_tiles;
      ptx::mbar_arrive_expect_tx(&cfull[sl], 16384);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              ptx::smem_u32(ring + sl * 16384)),
          "l"(src + idx * 16384), "r"(16384), "r"(ptx::smem_u32(&cfull[sl]))
          : "memory");
      ++c;
    }
    for (uint32_t j = (c > (uint32_t)RS ? c - RS : 0); j < c; ++j) ptx::mbar_wait(&cfull[j % RS], (j / RS) & 1);
    const unsigned long long dt = clock64() - t0;
    cyc[gridDim.x + blockIdx.x] = dt;
    cyc[2 * gridDim.x + blockIdx.x] = (unsigned long long)c * 16384;
  }
  if (!FREE && CP > 0 && threadIdx.x == 32) {  // producer: CP bulk copies of 16 KB per MMA iteration
    uint32_t c = 0;
    for (int it = 0; it < iters; ++it)
      for (int j = 0; j < CP; ++j, ++c) {
        const int sl = c % RS;
        ptx::mbar_wait(&cempty[sl], ((c / RS) & 1) ^ 1);
        const size_t idx = ((size_t)blockIdx.x * 7919 + (size_t)c * 104729) % src_tiles;
        ptx::mbar_arrive_expect_tx(&cfull[sl], 16384);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                ptx::smem_u32(ring + sl * 16384)),
            "l"(src + idx * 16384), "r"(16384), "r"(ptx::smem_u32(&cfull[sl]))
            : "memory");
      }
  }
  if (WARP ? threadIdx.x < 32 : threadIdx.x == 0) {
    uint32_t cc = 0;
    const uint32_t aQ = ptx::smem_u32(sQ), aK = ptx::smem_u32(sK), aV = ptx::smem_u32(sV);
    constexpr uint32_t IS = make_idesc(128, N, 0);
    constexpr uint32_t IO = make_idesc(128, D, 1);
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int j = 0; j < (FREE ? 0 : CP); ++j) {  // operands of this iteration have landed
        const uint32_t c = cc + j;
        ptx::mbar_wait(&cfull[c % RS], (c / RS) & 1);
      }
      ptx::tc_fence_after();
      if constexpr (MODE >= 10) {  // single-tile split-key block: PV_A, PV_B, QK with NW
        constexpr int NW = MODE - 10;  // already-satisfied barrier waits per block
        auto wt = [&](int i) { if (i < NW) ptx::mbar_wait(&donebar, 0); };
        wt(0);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            ptx::mma_ts(tmem + 256, tmem + kk * 8, make_sdesc(aV + kk * 16 * 128, N * 128, 1024), IO, 1);
        }
        __syncwarp();
        wt(1);
        if (elect_one()) {
#pragma unroll
          for (int kk = 4; kk < 8; ++kk)
            ptx::mma_ts(tmem + 384, tmem + 64 + (kk - 4) * 8, make_sdesc(aV + kk * 16 * 128, N * 128, 1024), IO, 1);
        }
        __syncwarp();
        wt(2);
        wt(3);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk >> 2) * (128 * 128) + (kk & 3) * 32;
            ptx::mma_ss(tmem, make_sdesc(aQ + off, 16, 1024), make_sdesc(aK + off, 16, 1024), IS, kk > 0);
          }
          ptx::mma_commit(&bar[it & 3]);
        }
        __syncwarp();
        if (it >= 3) ptx::mbar_wait(&bar[(it - 3) & 3], ((it - 3) >> 2) & 1);
        continue;
      }
      if (!WARP || elect_one()) {
      if (MODE == 0 || MODE == 3) {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * (128 * 128) + (kk & 3) * 32;
          const uint32_t koff = (kk >> 2) * (N * 128) + (kk & 3) * 32;
          ptx::mma_ss(Sc, make_sdesc(aQ + off, 16, 1024), make_sdesc(aK + koff, 16, 1024), IS,
                      kk > 0);
        }
      }
      if (MODE == 5) {  // same A (Q slice) for two consecutive MMAs into two S buffers
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * (128 * 128) + (kk & 3) * 32;
          const uint32_t koff = (kk >> 2) * (N * 128) + (kk & 3) * 32;
          ptx::mma_ss(Sc, make_sdesc(aQ + off, 16, 1024), make_sdesc(aK + koff, 16, 1024), IS, kk > 0);
          ptx::mma_ss(Sc + N, make_sdesc(aQ + off, 16, 1024), make_sdesc(aV + koff, 16, 1024), IS, kk > 0);
        }
      }
      if (MODE == 1 || MODE == 4) {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t koff = (kk >> 2) * (N * 128) + (kk & 3) * 32;
          ptx::mma_ts(Sc, Qc + kk * 8, make_sdesc(aK + koff, 16, 1024), IS, kk > 0);
        }
      }
      if (MODE >= 6) {  // two-tile carve turn patterns, N = 128 keys, P aliased over S
        const uint32_t S0 = tmem, O0 = tmem + 128, S1 = tmem + 256, O1 = tmem + 384;
        auto pv = [&](uint32_t S, uint32_t O) {
#pragma unroll
          for (int kk = 0; kk < N / 16; ++kk)
            ptx::mma_ts(O, S + kk * 8, make_sdesc(aV + kk * 16 * 128, N * 128, 1024), IO, 1);
        };
        auto qk = [&](uint32_t S) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk >> 2) * (128 * 128) + (kk & 3) * 32;
            const uint32_t koff = (kk >> 2) * (N * 128) + (kk & 3) * 32;
            ptx::mma_ss(S, make_sdesc(aQ + off, 16, 1024), make_sdesc(aK + koff, 16, 1024), IS, kk > 0);
          }
        };
        if (MODE == 6) { pv(S0, O0); qk(S0); }                       // one tile: WAR on S
        if (MODE == 7) { pv(S0, O0); qk(S0); pv(S1, O1); qk(S1); }   // two tiles, turn order
        if (MODE == 8) { pv(S0, O0); pv(S1, O1); qk(S0); qk(S1); }   // two tiles, WAR spread
        if (MODE == 9) { qk(S0); pv(S0, O0); }                       // one tile: RAW on S
      }
      if (MODE >= 2 && MODE != 5 && MODE < 6) {
#pragma unroll
        for (int kk = 0; kk < N / 16; ++kk)
          ptx::mma_ts(Oc, Qc + kk * 8, make_sdesc(aV + kk * 16 * 128, N * 128, 1024), IO, 1);
      }
      for (int j = 0; j < (FREE ? 0 : CP); ++j, ++cc) ptx::mma_commit(&cempty[cc % RS]);
      ptx::mma_commit(&bar[it & 3]);
      }
      if (WARP) __syncwarp();
      if (it >= 3) ptx::mbar_wait(&bar[(it - 3) & 3], ((it - 3) >> 2) & 1);
    }
    for (int j = iters - 3; j < iters; ++j) ptx::mbar_wait(&bar[j & 3], (j >> 2) & 1);
    if (!WARP || threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<TCOLS>(tmem);
  }
}

static uint8_t* g_src;
static const size_t SRC_BYTES = (size_t)64 << 20;  // L2-resident source (K/V of one head ~61 MB)

template <int N, int MODE, int TCOLS, int CP = 0, int RS = 1, int FREE = 0, int WARP = 0>
void run(const char* name, int occ) {
  const int sms = 148, grid = sms * occ, iters = 4000;
  unsigned long long* d;
  cudaMalloc(&d, 3 * grid * sizeof(unsigned long long));
  auto k = k_rate<N, MODE, TCOLS, CP, RS, FREE, WARP>;
  const int smem = FREE ? 3 * QB + RS * 16384 : (3 * QB > QB + RS * 16384 ? 3 * QB : QB + RS * 16384);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<<<grid, 128, smem>>>(iters, d, g_src, SRC_BYTES / 16384);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<<<grid, 128, smem>>>(iters, d, g_src, SRC_BYTES / 16384);
  cudaEventRecord(b);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%s: %s\n", name, cudaGetErrorString(e));
    exit(1);
  }
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  std::vector<unsigned long long> h(grid);
  cudaMemcpy(h.data(), d, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (auto v : h) mx = v > mx ? v : mx;
  double macs = 0;
  if (MODE == 0 || MODE == 1 || (MODE >= 3 && MODE != 5)) macs += 128.0 * N * D;
  if (MODE == 5) macs += 2 * 128.0 * N * D;
  if (MODE >= 2 && MODE != 5 && MODE < 6) macs += 128.0 * N * D;
  if (MODE == 6 || MODE == 9) macs = 2 * 128.0 * N * D;
  if (MODE == 7 || MODE == 8) macs = 4 * 128.0 * N * D;
  if (MODE >= 10) macs = 2 * 128.0 * N * D;
  const double per_sm_cyc = (double)mx / iters / occ;  // cycles per iteration per SM
  const double tflops = 2.0 * macs * iters * grid / (ms * 1e-3) / 1e12;
  if (FREE) {
    std::vector<unsigned long long> hh(3 * grid);
    cudaMemcpy(hh.data(), d, 3 * grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    double bpc = 0;
    for (int i = 0; i < grid; ++i) bpc += (double)hh[2 * grid + i] / hh[grid + i];
    printf("   copy stream alongside: %.1f B/cyc/SM\n", bpc / sms);
  }
  printf("%-28s cp=%dKB N=%3d occ=%d: %7.1f cyc/iter/SM  %6.0f MAC/cyc/SM  %7.1f TFLOP/s\n", name, CP * 16, N, occ,
         per_sm_cyc, macs / per_sm_cyc, tflops);
  cudaFree(d);
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  cudaMalloc(&g_src, SRC_BYTES);
  cudaMemset(g_src, 0x3c, SRC_BYTES);
  run<128, 9, 512, 0, 1, 0, 1>("1 tile QK->PV (RAW on S)", 1);
  run<128, 10, 512, 0, 1, 0, 1>("split-key block, 0 waits", 1);
  run<128, 12, 512, 0, 1, 0, 1>("split-key block, 2 waits", 1);
  run<128, 14, 512, 0, 1, 0, 1>("split-key block, 4 waits", 1);
  run<128, 10, 512, 0, 1, 0, 1>("split-key block, 0 waits", 1);
  return 0;
}
