// Numeric probe of two tcgen05 kind::f16 forms a Q-in-TMEM carve variant would need
// (not part of the library; built and run by hand on the GPU box):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2505_16864_b200/csrc \
//        tests/native/mixed_mma.cu -o /tmp/mixed_mma && /tmp/mixed_mma
//  (1) S = Q K^T with A = Q (bf16) read from TMEM, B = K (bf16, smem, K-major), D = f16 in TMEM
//  (2) O = P V   with A = P (f16) read from TMEM, B = V (bf16, smem, MN-major), D = f32
//      i.e. mixed A/B formats in one instruction descriptor.
// Prints max |err| of each against a host fp64 reference.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "ptx.cuh"

using namespace tcb;

__host__ __device__ constexpr uint32_t idesc(int M, int N, int b_mn_major, int a_bf16, int b_bf16,
                                             int c_f32) {
  return ((uint32_t)c_f32 << 4) | ((uint32_t)a_bf16 << 7) | ((uint32_t)b_bf16 << 10) |
         ((uint32_t)b_mn_major << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}
// byte offset of element (row r, col c) in an R-row, 128-col 16-bit tile stored as two
// 64-col chunks with the 128-byte swizzle (the TMA layout of the carve kernel)
__host__ __device__ inline int swz(int R, int r, int c) {
  return (c / 64) * (R * 128) + r * 128 + ((((c % 64) / 8) ^ (r % 8)) * 16) + (c % 8) * 2;
}

constexpr int D = 128, HN = 64;

__global__ void __launch_bounds__(128) k_probe(const __nv_bfloat16* q, const __nv_bfloat16* k,
                                               const __nv_bfloat16* v, const __half* p,
                                               float* s_out, float* o_out, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sK = smem;               // 64 x 128 bf16 = 16 KB
  uint8_t* sV = smem + HN * D * 2;  // 16 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < HN * D; i += 128) {
    const int r = i / D, c = i % D;
    *reinterpret_cast<__nv_bfloat16*>(sK + swz(HN, r, c)) = k[i];
    *reinterpret_cast<__nv_bfloat16*>(sV + swz(HN, r, c)) = v[i];
  }
  if (t == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc<256>(&tbase);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tm = tbase;
  // TMEM: S (f16) [0, 32), P (f16) [32, 64), Q (bf16) [64, 128), O (f32) [128, 256)
  const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
  {
    uint32_t r[32];
    for (int h = 0; h < 2; ++h) {
      for (int e = 0; e < 32; ++e) {
        const __nv_bfloat16 lo = q[t * D + h * 64 + 2 * e], hi = q[t * D + h * 64 + 2 * e + 1];
        r[e] = (uint32_t)__bfloat16_as_ushort(lo) | ((uint32_t)__bfloat16_as_ushort(hi) << 16);
      }
      ptx::tmem_st32(tm + lane_off + 64 + h * 32, r);
    }
    for (int e = 0; e < 32; ++e) {
      const __half lo = p[t * HN + 2 * e], hi = p[t * HN + 2 * e + 1];
      r[e] = (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
    }
    ptx::tmem_st32(tm + lane_off + 32, r);
    ptx::tmem_wait_st();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 0) {
    if (ptx::elect_one()) {
      const uint32_t aK = ptx::smem_u32(sK), aV = ptx::smem_u32(sV);
      // PV first: with an f32 S (modes 0/2) the S columns overlap P's
      for (int kk = 0; kk < HN / 16; ++kk)
        ptx::mma_ts(tm + 128, tm + 32 + kk * 8, sdesc(aV + kk * 16 * 128, HN * 128, 1024),
                    (mode & 2) ? idesc(128, D, 1, 0, 1, 1) : idesc(128, D, 1, 1, 1, 1), kk > 0 ? 1u : 0u);
      for (int kk = 0; kk < D / 16; ++kk) {
        const uint32_t koff = (kk >> 2) * (HN * 128) + (kk & 3) * 32;
        ptx::mma_ts(tm + 0, tm + 64 + kk * 8, sdesc(aK + koff, 16, 1024),
                    (mode & 1) ? idesc(128, HN, 0, 1, 1, 0) : idesc(128, HN, 0, 1, 1, 1), kk > 0 ? 1u : 0u);
      }
      ptx::mma_commit(&bar);
    }
    __syncwarp();
  }
  ptx::mbar_wait(&bar, 0);
  ptx::tc_fence_after();
  uint32_t r[32];
  ptx::tmem_ld32(tm + lane_off + 0, r);
  ptx::tmem_wait_ld();
  for (int e = 0; e < 32; ++e) {
    if (mode & 1) {
      s_out[t * HN + 2 * e] = __half2float(__ushort_as_half((unsigned short)(r[e] & 0xffff)));
      s_out[t * HN + 2 * e + 1] = __half2float(__ushort_as_half((unsigned short)(r[e] >> 16)));
    } else {
      s_out[t * HN + e] = __uint_as_float(r[e]);
    }
  }
  if (!(mode & 1)) {
    ptx::tmem_ld32(tm + lane_off + 32, r);  // f32 S spills into the P columns: read 32..63
    ptx::tmem_wait_ld();
    for (int e = 0; e < 32; ++e) s_out[t * HN + 32 + e] = __uint_as_float(r[e]);
  }
  for (int c = 0; c < 4; ++c) {
    ptx::tmem_ld32(tm + lane_off + 128 + c * 32, r);
    ptx::tmem_wait_ld();
    for (int e = 0; e < 32; ++e) o_out[t * D + c * 32 + e] = __uint_as_float(r[e]);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<256>(tm);
  }
}

int main(int argc, char** argv) {
  const int NQ = 128 * D, NK = HN * D, NP = 128 * HN;
  std::vector<__nv_bfloat16> q(NQ), k(NK), v(NK);
  std::vector<__half> p(NP);
  std::vector<float> fq(NQ), fk(NK), fv(NK), fp(NP);
  srand(7);
  auto rnd = [] { return (float)rand() / RAND_MAX * 2.f - 1.f; };
  for (int i = 0; i < NQ; ++i) { q[i] = __float2bfloat16(2.f * rnd()); fq[i] = __bfloat162float(q[i]); }
  for (int i = 0; i < NK; ++i) {
    k[i] = __float2bfloat16(2.f * rnd()); fk[i] = __bfloat162float(k[i]);
    v[i] = __float2bfloat16(rnd()); fv[i] = __bfloat162float(v[i]);
  }
  for (int i = 0; i < NP; ++i) { p[i] = __float2half(std::fabs(rnd()) * 3.f); fp[i] = __half2float(p[i]); }
  __nv_bfloat16 *dq, *dk, *dv;
  __half* dp;
  float *ds, *dout;
  cudaMalloc(&dq, NQ * 2); cudaMalloc(&dk, NK * 2); cudaMalloc(&dv, NK * 2); cudaMalloc(&dp, NP * 2);
  cudaMalloc(&ds, NP * 4); cudaMalloc(&dout, NQ * 4);
  cudaMemcpy(dq, q.data(), NQ * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dk, k.data(), NK * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dv, v.data(), NK * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dp, p.data(), NP * 2, cudaMemcpyHostToDevice);
  const int smem = 2 * HN * D * 2 + 1024;
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int mode = argc > 1 ? atoi(argv[1]) : 3;
  k_probe<<<1, 128, smem>>>(dq, dk, dv, dp, ds, dout, mode);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("mode %d kernel error: %s\n", mode, cudaGetErrorString(e)); return 1; }
  printf("mode %d (bit0: f16-accumulated S, bit1: f16 P x bf16 V)\n", mode);
  std::vector<float> s(NP), o(NQ);
  cudaMemcpy(s.data(), ds, NP * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(o.data(), dout, NQ * 4, cudaMemcpyDeviceToHost);
  double es = 0, ms = 0, eo = 0, mo = 0;
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < HN; ++j) {
      double ref = 0;
      for (int c = 0; c < D; ++c) ref += (double)fq[i * D + c] * fk[j * D + c];
      es = std::fmax(es, std::fabs(ref - s[i * HN + j]));
      ms = std::fmax(ms, std::fabs(ref));
    }
  for (int i = 0; i < 128; ++i)
    for (int c = 0; c < D; ++c) {
      double ref = 0;
      for (int j = 0; j < HN; ++j) ref += (double)fp[i * HN + j] * fv[j * D + c];
      eo = std::fmax(eo, std::fabs(ref - o[i * D + c]));
      mo = std::fmax(mo, std::fabs(ref));
    }
  printf("S = Q K^T (A bf16 from TMEM, f16 accumulate): max|err| %.3e of max|S| %.3e (rel %.2e)\n", es, ms, es / ms);
  printf("O = P V (A f16 from TMEM x B bf16 smem, f32): max|err| %.3e of max|O| %.3e (rel %.2e)\n", eo, mo, eo / mo);
  printf("sample S[0][0..3] = %.4f %.4f %.4f %.4f\n", s[0], s[1], s[2], s[3]);
  return 0;
}
