// K7/K8 block-sparse flash-attention forward (carve_attention, attention.py:162-243).
//
//  * k_carve_tc   -- bf16 / fp16, m == 128, d in {64,128}: persistent warp-specialised
//                    tcgen05 kernel.  TMA loads Q/K/V tiles (128B swizzle) into smem
//                    under mbarriers, one elected lane of the MMA warp issues
//                    tcgen05.mma for S = Q K^T into TMEM (64-key half-steps, S
//                    double-buffered), four softmax warps read S with tcgen05.ld, do
//                    the online softmax in registers (exp2, lazy rescale), write P as
//                    16-bit back into TMEM over S, and the MMA warp issues O += P V with
//                    A read from TMEM.  Two CTAs per SM interleave so one CTA's softmax
//                    overlaps the other's MMAs.  Work items (head, q-block) come from a
//                    global atomic counter, condition q-blocks (full rows, ~10x longer)
//                    first, then vision q-blocks head-major so concurrently running
//                    items share a head's K/V in L2.  DESIGN.md §4.1 has the measured
//                    bounds and the rejected variants.
//  * k_carve_f32t -- fp32 math on shared-memory tiles with register-blocked S / O for
//                    the common (m, d): fp32 inputs and shapes the tcgen05 kernel does
//                    not take; mirrors the reference's per-block streaming order (1e-5).
//  * k_carve_simt -- fp32 math, one warp per query row, any (m, d): the fallback.
#include "common.cuh"
#include "ptx.cuh"

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <math.h>
#include <stdlib.h>

namespace tcb {

struct CarveShape {
  int H, d, m, M_v, M_total;
  int64_t n_valid, n_cond;
  int64_t sh, sn;  // element strides (head, token)
};

__device__ __forceinline__ void decode_item(int item, const CarveShape& s, int& h, int& qb) {
  const int M_c = s.M_total - s.M_v;
  const int n_cond_items = s.H * M_c;
  if (item < n_cond_items) {
    h = item / M_c;
    qb = s.M_v + (item - h * M_c);
  } else {
    const int j = item - n_cond_items;
    h = j / s.M_v;
    qb = j - h * s.M_v;
  }
}

// =====================================================================================
// SIMT fp32 kernel (parity path).  CTA = (head, q-block); each warp owns query rows;
// per selected kv block: scores (warp-reduced dot products, q pre-scaled in fp32 as
// attention.py:184), padding -> -inf, +beta on condition keys of vision rows,
// block max, alpha = exp(m - m_new), p = exp(s - m_new), l = l*alpha + sum p,
// acc = acc*alpha + p V  (attention.py:190-201); out = acc / l, padding rows 0.
// =====================================================================================
constexpr int SIMT_MAXC = 8;  // d <= 256

template <typename T>
__device__ __forceinline__ float ldf(const T* p) {
  return static_cast<float>(*p);
}
template <>
__device__ __forceinline__ float ldf<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}
template <>
__device__ __forceinline__ float ldf<__half>(const __half* p) {
  return __half2float(*p);
}
template <typename T>
__device__ __forceinline__ T stf(float v);
template <>
__device__ __forceinline__ __half stf<__half>(float v) {
  return __float2half_rn(v);
}
template <>
__device__ __forceinline__ float stf<float>(float v) {
  return v;
}
template <>
__device__ __forceinline__ __nv_bfloat16 stf<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

template <typename T>
__global__ void __launch_bounds__(128) k_carve_simt(const T* __restrict__ q,
                                                    const T* __restrict__ k,
                                                    const T* __restrict__ v, T* __restrict__ o,
                                                    CarveShape s, const int32_t* __restrict__ kv_idx,
                                                    const int32_t* __restrict__ kv_cnt,
                                                    float beta, float scale) {
  extern __shared__ float sm_simt[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  float* sc = sm_simt + warp * (s.m + s.d);
  float* sq = sc + s.m;
  const int h = blockIdx.x / s.M_total;
  const int qb = blockIdx.x - h * s.M_total;
  const bool vis = qb < s.M_v;
  const int nkv = vis ? kv_cnt[(int64_t)h * s.M_v + qb] : s.M_total;
  const int32_t* list = vis ? kv_idx + ((int64_t)h * s.M_v + qb) * s.M_total : nullptr;
  const int qvalid = block_valid(qb, s.m, s.M_v, s.n_valid, s.n_cond);
  const T* qh = q + (int64_t)h * s.sh;
  const T* kh = k + (int64_t)h * s.sh;
  const T* vh = v + (int64_t)h * s.sh;
  T* oh = o + (int64_t)h * s.sh;
  for (int r = warp; r < s.m; r += nwarps) {
    const int64_t row = (int64_t)qb * s.m + r;
    T* orow = oh + row * s.sn;
    if (r >= qvalid) {
      for (int c = lane; c < s.d; c += 32) orow[c] = stf<T>(0.f);
      continue;
    }
    for (int c = lane; c < s.d; c += 32) sq[c] = ldf(qh + row * s.sn + c) * scale;
    __syncwarp();
    float acc[SIMT_MAXC];
#pragma unroll
    for (int i = 0; i < SIMT_MAXC; ++i) acc[i] = 0.f;
    float mi = -INFINITY, li = 0.f;
    for (int t = 0; t < nkv; ++t) {
      const int b = vis ? list[t] : t;
      const int kvalid = block_valid(b, s.m, s.M_v, s.n_valid, s.n_cond);
      const bool add_beta = vis && beta != 0.f && b >= s.M_v;
      for (int j = 0; j < s.m; ++j) {
        const T* krow = kh + ((int64_t)b * s.m + j) * s.sn;
        float part = 0.f;
        for (int c = lane; c < s.d; c += 32) part = fmaf(sq[c], ldf(krow + c), part);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
        float sv = (j < kvalid) ? part : -INFINITY;
        if (add_beta) sv = sv + beta;
        if (lane == 0) sc[j] = sv;
      }
      __syncwarp();
      float bm = -INFINITY;
      for (int j = lane; j < s.m; j += 32) bm = fmaxf(bm, sc[j]);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, off));
      const float mn = fmaxf(mi, bm);
      const float alpha = expf(mi - mn);
      __syncwarp();
      float ps = 0.f;
      for (int j = lane; j < s.m; j += 32) {
        const float pj = expf(sc[j] - mn);
        sc[j] = pj;
        ps += pj;
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, off);
      __syncwarp();
      li = li * alpha + ps;
#pragma unroll
      for (int i = 0; i < SIMT_MAXC; ++i) {
        const int c = lane + 32 * i;
        if (c < s.d) {
          float pv = 0.f;
          for (int j = 0; j < s.m; ++j) pv = fmaf(sc[j], ldf(vh + ((int64_t)b * s.m + j) * s.sn + c), pv);
          acc[i] = acc[i] * alpha + pv;
        }
      }
      mi = mn;
      __syncwarp();
    }
#pragma unroll
    for (int i = 0; i < SIMT_MAXC; ++i) {
      const int c = lane + 32 * i;
      if (c < s.d) orow[c] = stf<T>(acc[i] / li);
    }
    __syncwarp();
  }
}

// =====================================================================================
// Tiled fp32 kernel (the reference's dtype at real sizes).  CTA = one (head, q-block) item,
// 256 threads as a 16 x 16 grid; thread (ty, tx) owns query rows ty + 16 i and key / value
// columns tx + 16 j, i.e. an (MT x MT) tile of S and an (MT x DT) tile of O in registers
// (m = 16 MT, d = 16 DT).  Per kv block, in the reference's order (attention.py:184-201):
// S = (q * scale) K^T from shared-memory tiles (fp32 FMA), padding keys -> -inf, +beta on
// condition keys of vision rows, block row max (shuffles across the 16 threads of a row),
// alpha = exp(m - m_new), p = exp(s - m_new), l = l * alpha + sum p, O = O * alpha + P V
// with P staged through shared memory.  expf (not ex2.approx) and fp32 accumulation keep
// it within the north_star's 1e-5 of the reference; only the summation order of the
// length-d / length-m dot products differs.
// =====================================================================================
template <typename T, int MT, int DT>
__global__ void __launch_bounds__(256, 1) k_carve_f32t(const T* __restrict__ q, const T* __restrict__ k,
                                                       const T* __restrict__ v, T* __restrict__ o,
                                                       CarveShape s, const int32_t* __restrict__ kv_idx,
                                                       const int32_t* __restrict__ kv_cnt, float beta,
                                                       float scale) {
  constexpr int M = 16 * MT, D = 16 * DT;
  constexpr int QP = D + 1;   // padded row pitch (floats) of Q / K / V tiles
  constexpr int PP = M + 1;   // padded row pitch of P
  extern __shared__ float sm_f32t[];
  float* sQ = sm_f32t;
  float* sK = sQ + M * QP;
  float* sV = sK + M * QP;
  float* sP = (M * PP <= M * QP) ? sK : sV + M * QP;  // P reuses K's tile when it fits
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const int h = blockIdx.x / s.M_total;
  const int qb = blockIdx.x - h * s.M_total;
  const bool vis = qb < s.M_v;
  const int nkv = vis ? kv_cnt[(int64_t)h * s.M_v + qb] : s.M_total;
  const int32_t* list = vis ? kv_idx + ((int64_t)h * s.M_v + qb) * s.M_total : nullptr;
  const int qvalid = block_valid(qb, M, s.M_v, s.n_valid, s.n_cond);
  const T* qh = q + (int64_t)h * s.sh;
  const T* kh = k + (int64_t)h * s.sh;
  const T* vh = v + (int64_t)h * s.sh;
  for (int e = tid; e < M * D; e += 256) {  // q pre-scaled in fp32 (attention.py:184)
    const int r = e / D, c = e - r * D;
    sQ[r * QP + c] = ldf(qh + ((int64_t)qb * M + r) * s.sn + c) * scale;
  }
  float acc[MT][DT], mrow[MT], lrow[MT];
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    mrow[i] = -INFINITY;
    lrow[i] = 0.f;
#pragma unroll
    for (int j = 0; j < DT; ++j) acc[i][j] = 0.f;
  }
  for (int t = 0; t < nkv; ++t) {
    const int b = vis ? __ldg(list + t) : t;
    const int kvalid = block_valid(b, M, s.M_v, s.n_valid, s.n_cond);
    const bool add_beta = vis && beta != 0.f && b >= s.M_v;
    __syncthreads();  // previous block's P / V reads done
    for (int e = tid; e < M * D; e += 256) {
      const int r = e / D, c = e - r * D;
      const int64_t g = ((int64_t)b * M + r) * s.sn + c;
      sK[r * QP + c] = ldf(kh + g);
      sV[r * QP + c] = ldf(vh + g);
    }
    __syncthreads();
    float sc[MT][MT];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < MT; ++j) sc[i][j] = 0.f;
#pragma unroll 4
    for (int c = 0; c < D; ++c) {
      float a[MT], bk[MT];
#pragma unroll
      for (int i = 0; i < MT; ++i) a[i] = sQ[(ty + 16 * i) * QP + c];
#pragma unroll
      for (int j = 0; j < MT; ++j) bk[j] = sK[(tx + 16 * j) * QP + c];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < MT; ++j) sc[i][j] = fmaf(a[i], bk[j], sc[i][j]);
    }
    __syncthreads();  // K tile consumed (P may overwrite it)
    float alpha[MT];
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      float bm = -INFINITY;
#pragma unroll
      for (int j = 0; j < MT; ++j) {
        float x = (tx + 16 * j < kvalid) ? sc[i][j] : -INFINITY;  // attention.py:193
        if (add_beta) x = x + beta;
        sc[i][j] = x;
        bm = fmaxf(bm, x);
      }
#pragma unroll
      for (int off = 8; off > 0; off >>= 1) bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, off));
      const float mn = fmaxf(mrow[i], bm);
      alpha[i] = expf(mrow[i] - mn);
      float ps = 0.f;
#pragma unroll
      for (int j = 0; j < MT; ++j) {
        const float pj = expf(sc[i][j] - mn);
        sP[(ty + 16 * i) * PP + tx + 16 * j] = pj;
        ps += pj;
      }
#pragma unroll
      for (int off = 8; off > 0; off >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, off);
      lrow[i] = lrow[i] * alpha[i] + ps;
      mrow[i] = mn;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < DT; ++j) acc[i][j] *= alpha[i];
#pragma unroll 4
    for (int jk = 0; jk < M; ++jk) {
      float pr[MT], vv[DT];
#pragma unroll
      for (int i = 0; i < MT; ++i) pr[i] = sP[(ty + 16 * i) * PP + jk];
#pragma unroll
      for (int j = 0; j < DT; ++j) vv[j] = sV[jk * QP + tx + 16 * j];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < DT; ++j) acc[i][j] = fmaf(pr[i], vv[j], acc[i][j]);
    }
  }
  T* oh = o + (int64_t)h * s.sh;
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int r = ty + 16 * i;
    T* orow = oh + ((int64_t)qb * M + r) * s.sn;
#pragma unroll
    for (int j = 0; j < DT; ++j)
      orow[tx + 16 * j] = stf<T>(r < qvalid ? acc[i][j] / lrow[i] : 0.f);  // attention.py:203-206
  }
}

// =====================================================================================
// tcgen05 kernel
// =====================================================================================
namespace tc {

// Work unit of the pipeline: a "half-step" = one 64-key half of a 128-key kv block.
// S is double-buffered in TMEM per half-step (2 x 64 columns) so the tensor core
// computes S(t+1) = Q K(t+1)^T while the softmax warps work on S(t); P(t) is written
// as bf16 over the first 32 columns of its S buffer and consumed by O += P(t) V(t).
constexpr int BM = 128;           // query rows per tile (== m)
constexpr int BK = 128;           // keys per kv block (== m)
constexpr int HN = 64;            // keys per half-step
constexpr int NUM_THREADS = 192;  // w0 TMA+scheduler, w1 MMA+TMEM owner, w2..w5 softmax
constexpr int TMEM_COLS = 256;    // S0 [0,64) S1 [64,128) O [128, 128+D)
constexpr int O_COL = 128;
constexpr int K_SLOTS = 3;        // K half-tiles in flight
constexpr int V_SLOTS = 2;        // V half-tiles in flight
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 units: P <= 2^8 between rescales

template <int D>
struct Smem {
  static constexpr int Q_BYTES = BM * D * 2;      // 128 x D bf16
  static constexpr int HALF_BYTES = HN * D * 2;   // 64 x D bf16
  static constexpr int CHUNKS = D / 64;           // 64-element (128 B) swizzle columns
  static constexpr int Q_CHUNK = BM * 128;        // bytes per 64-col chunk of Q
  static constexpr int H_CHUNK = HN * 128;        // bytes per 64-col chunk of a half tile
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_BYTES;
  static constexpr int OFF_V = OFF_K + K_SLOTS * HALF_BYTES;
  static constexpr int OFF_BAR = OFF_V + V_SLOTS * HALF_BYTES;
  static constexpr int BYTES = OFF_BAR + 256;
};

struct Bars {
  uint64_t q_full, q_empty, o_full, o_done;
  uint64_t p_full[2];  // by half-step parity: softmax(t+1) may finish before PV(t) is issued
  uint64_t s_full[2];
  uint64_t k_full[K_SLOTS], k_empty[K_SLOTS];
  uint64_t v_full[V_SLOTS], v_empty[V_SLOTS];
  uint64_t sched_full[2], sched_empty[2];
  int sched_item[2];
  uint32_t tmem_base;
};
static_assert(sizeof(Bars) <= 256, "barrier block must fit the reserved smem");

// instruction descriptor, kind::f16: {bf16|f16} x {bf16|f16} -> f32, K-major A, B major per
// arg (a/b type field: 1 = bf16, 0 = f16)
__host__ __device__ constexpr uint32_t make_idesc(int M, int N, int b_mn_major, int bf16 = 1) {
  return (1u << 4) | ((uint32_t)bf16 << 7) | ((uint32_t)bf16 << 10) | ((uint32_t)b_mn_major << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// element traits of the 16-bit input / P / output type
template <typename E>
struct Elem;
template <>
struct Elem<__nv_bfloat16> {
  static constexpr int kBf16 = 1;
  __device__ static uint32_t pack(float lo, float hi) { return ptx::pack_bf16(lo, hi); }
};
template <>
struct Elem<__half> {
  static constexpr int kBf16 = 0;
  __device__ static uint32_t pack(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
  }
};

// smem matrix descriptor, SWIZZLE_128B, sm_100 version bits
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}

__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
  return (uint64_t)__float_as_uint(lo) | ((uint64_t)__float_as_uint(hi) << 32);
}
__device__ __forceinline__ float f2_lo(uint64_t v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float f2_hi(uint64_t v) { return __uint_as_float((uint32_t)(v >> 32)); }
// packed fp32x2 FMA / ADD (FFMA2 / FADD2 on sm_100a)
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));  // FMNMX3
  return d;
}

// 2^x for a packed pair on the FMA pipe (offloads MUFU): x = j + f, j = rint(x) via the
// 1.5*2^23 magic add, 2^f by a degree-3 minimax polynomial on [-0.5, 0.5] (max rel err
// 7.5e-5, far below the bf16 rounding of P), 2^j added straight into the exponent bits.
// x is clamped at -126 so the exponent never underflows into the sign bit.
__device__ __forceinline__ uint64_t exp2_poly2(uint64_t x) {
  const float x0 = fmaxf(f2_lo(x), -126.f), x1 = fmaxf(f2_hi(x), -126.f);
  const uint64_t xc = f2_pack(x0, x1);
  const uint64_t magic = f2_pack(12582912.f, 12582912.f);
  const uint64_t t = fadd2(xc, magic);
  const uint64_t jf = fadd2(t, f2_pack(-12582912.f, -12582912.f));
  const uint64_t f = ffma2(jf, f2_pack(-1.f, -1.f), xc);
  uint64_t p = ffma2(f, f2_pack(0.05517132f, 0.05517132f), f2_pack(0.24261054f, 0.24261054f));
  p = ffma2(p, f, f2_pack(0.69326097f, 0.69326097f));
  p = ffma2(p, f, f2_pack(0.99992812f, 0.99992812f));
  const uint32_t lo = (uint32_t)p + ((uint32_t)t << 23);
  const uint32_t hi = (uint32_t)(p >> 32) + ((uint32_t)(t >> 32) << 23);
  return (uint64_t)lo | ((uint64_t)hi << 32);
}

// Warp-cooperative view of a row's ascending kv list: lane l caches entry 32*c + l of the
// current chunk c; block(j) broadcasts entry j (all 32 lanes must call it together).
struct KvList {
  const int32_t* list;
  int n, lane, chunk, cache;
  __device__ KvList(const int32_t* l, int n_, int lane_) : list(l), n(n_), lane(lane_), chunk(-1), cache(0) {}
  __device__ KvList() : list(nullptr), n(0), lane(threadIdx.x & 31), chunk(-1), cache(0) {}
  __device__ __forceinline__ int block(int j) {
    if (!list) return j;
    const int c = j >> 5;
    if (c != chunk) {
      chunk = c;
      const int idx = c * 32 + lane;
      cache = idx < n ? __ldg(list + idx) : 0;
    }
    return __shfl_sync(0xffffffffu, cache, j & 31);
  }
};

template <int D, int EMU, typename E = __nv_bfloat16>
__global__ void __launch_bounds__(NUM_THREADS, 2)
    k_carve_tc(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
               const __grid_constant__ CUtensorMap tm_v, E* __restrict__ o,
               CarveShape s, const int32_t* __restrict__ kv_idx,
               const int32_t* __restrict__ kv_cnt, int* __restrict__ counter, int total_items,
               float scale_log2, float beta_log2, int dbg) {
  using L = Smem<D>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sQ = smem + L::OFF_Q;
  uint8_t* sK = smem + L::OFF_K;
  uint8_t* sV = smem + L::OFF_V;
  Bars* bars = reinterpret_cast<Bars*>(smem + L::OFF_BAR);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    if (ptx::smem_u32(smem) & 1023u) __trap();  // 128B-swizzle tiles need 1 KB alignment
    ptx::mbar_init(&bars->q_full, 1);
    ptx::mbar_init(&bars->q_empty, 1);
    ptx::mbar_init(&bars->o_full, 1);
    ptx::mbar_init(&bars->o_done, 1);
    for (int i = 0; i < 2; ++i) ptx::mbar_init(&bars->p_full[i], 128);
    for (int i = 0; i < 2; ++i) ptx::mbar_init(&bars->s_full[i], 1);
    for (int i = 0; i < K_SLOTS; ++i) {
      ptx::mbar_init(&bars->k_full[i], 1);
      ptx::mbar_init(&bars->k_empty[i], 1);
    }
    for (int i = 0; i < V_SLOTS; ++i) {
      ptx::mbar_init(&bars->v_full[i], 1);
      ptx::mbar_init(&bars->v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&bars->sched_full[i], 1);
      ptx::mbar_init(&bars->sched_empty[i], 1 + 4);
    }
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&tm_q);
    ptx::tma_prefetch_desc(&tm_k);
    ptx::tma_prefetch_desc(&tm_v);
  }
  if (warp == 1) ptx::tmem_alloc<TMEM_COLS>(&bars->tmem_base);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == 0) {
    // ============================ TMA producer + scheduler ============================
    // Whole warp runs the loop: lane 0 waits on the rings and issues TMA; the item's kv
    // list is read 32 entries at a time (one coalesced load per lane) and broadcast by
    // shuffle, so the block index is never a dependent global load on the issue path.
    const uint64_t pol_kv = ptx::policy_evict_last();
    // Q is read once; condition rows sweep a whole head's K/V once (both condition rows of
    // a head run concurrently), so neither should displace the vision rows' K/V in L2
    const uint64_t pol_q = ptx::policy_evict_first();
    uint32_t it = 0, gk = 0, gv = 0;
    for (;; ++it) {
      const int slot = it & 1;
      int item = 0;
      if (lane == 0) {
        ptx::mbar_wait(&bars->sched_empty[slot], ((it >> 1) & 1) ^ 1);
        item = atomicAdd(counter, 1);
        if (item >= total_items) item = -1;
        bars->sched_item[slot] = item;
        ptx::mbar_arrive(&bars->sched_full[slot]);
      }
      item = __shfl_sync(0xffffffffu, item, 0);
      if (item < 0) break;
      int h, qb;
      decode_item(item, s, h, qb);
      const bool vis = qb < s.M_v;
      const int n = vis ? __ldg(kv_cnt + (int64_t)h * s.M_v + qb) : s.M_total;
      KvList kl(vis ? kv_idx + ((int64_t)h * s.M_v + qb) * s.M_total : nullptr, n, lane);
      const int T = 2 * n;
      if (lane == 0) {
        ptx::mbar_wait(&bars->q_empty, (it & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&bars->q_full, L::Q_BYTES);
#pragma unroll
        for (int c = 0; c < L::CHUNKS; ++c)
          ptx::tma_load_3d(sQ + c * L::Q_CHUNK, &tm_q, &bars->q_full, c * 64, qb * BM, h, pol_q);
      }
      auto load = [&](const CUtensorMap* tm, uint8_t* base, uint64_t* full, uint64_t* empty,
                      int slots, uint32_t& cnt, int t) {
        const int b = kl.block(t >> 1);
        if (lane == 0) {
          const int sl = cnt % slots;
          ptx::mbar_wait(&empty[sl], ((cnt / slots) & 1) ^ 1);
          if ((dbg & 1) && cnt >= (uint32_t)slots) {  // timing experiment: no operand traffic
            ptx::mbar_arrive(&full[sl]);
          } else {
            ptx::mbar_arrive_expect_tx(&full[sl], L::HALF_BYTES);
#pragma unroll
            for (int c = 0; c < L::CHUNKS; ++c)
              ptx::tma_load_3d(base + sl * L::HALF_BYTES + c * L::H_CHUNK, tm, &full[sl], c * 64,
                               b * BK + (t & 1) * HN, h, vis ? pol_kv : pol_q);
          }
        }
        ++cnt;
      };
      // same order the MMA warp consumes: K0, K1, V0, K2, V1, ..., V(T-1)
      load(&tm_k, sK, bars->k_full, bars->k_empty, K_SLOTS, gk, 0);
      for (int t = 0; t < T; ++t) {
        if (t + 1 < T) load(&tm_k, sK, bars->k_full, bars->k_empty, K_SLOTS, gk, t + 1);
        load(&tm_v, sV, bars->v_full, bars->v_empty, V_SLOTS, gv, t);
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ============================
    // Whole warp runs the loop; one elected lane issues (uniform-register descriptors).
    constexpr uint32_t IDESC_S = make_idesc(BM, HN, 0, Elem<E>::kBf16);  // Q (K-major) x K (K-major)
    constexpr uint32_t IDESC_O = make_idesc(BM, D, 1, Elem<E>::kBf16);   // P (TMEM)   x V (MN-major)
    const uint32_t aQ = ptx::smem_u32(sQ), aK = ptx::smem_u32(sK), aV = ptx::smem_u32(sV);
    uint32_t it = 0, gk = 0, gv = 0, gs = 0, gp = 0;
    auto issue_s = [&]() {  // S(gs) = Q K(gs)^T into buffer gs & 1
      const int sl = gk % K_SLOTS;
      ptx::mbar_wait(&bars->k_full[sl], (gk / K_SLOTS) & 1);
      ptx::tc_fence_after();
      const uint32_t kbase = aK + sl * L::HALF_BYTES;
      if (ptx::elect_one()) {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t qoff = (kk >> 2) * L::Q_CHUNK + (kk & 3) * 32;
          const uint32_t koff = (kk >> 2) * L::H_CHUNK + (kk & 3) * 32;
          ptx::mma_ss(tmem + (gs & 1) * HN, make_sdesc(aQ + qoff, 16, 1024),
                      make_sdesc(kbase + koff, 16, 1024), IDESC_S, kk > 0 ? 1u : 0u);
        }
        ptx::mma_commit(&bars->k_empty[sl]);
        ptx::mma_commit(&bars->s_full[gs & 1]);
      }
      __syncwarp();
      ++gk;
      ++gs;
    };
    // S(gs), S(gs+1) with the two MMAs of each k-step back to back on the same Q slice:
    // the tensor core reuses the A operand, so the pair reads Q from shared memory once
    // (tests/native/mma_rate.cu MODE 5: full rate vs 67 % for lone SS N=64 MMAs).
    auto issue_pair = [&]() {
      const int sl0 = gk % K_SLOTS, sl1 = (gk + 1) % K_SLOTS;
      ptx::mbar_wait(&bars->k_full[sl0], (gk / K_SLOTS) & 1);
      ptx::mbar_wait(&bars->k_full[sl1], ((gk + 1) / K_SLOTS) & 1);
      ptx::tc_fence_after();
      const uint32_t kb0 = aK + sl0 * L::HALF_BYTES, kb1 = aK + sl1 * L::HALF_BYTES;
      if (ptx::elect_one()) {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t qoff = (kk >> 2) * L::Q_CHUNK + (kk & 3) * 32;
          const uint32_t koff = (kk >> 2) * L::H_CHUNK + (kk & 3) * 32;
          const uint64_t qd = make_sdesc(aQ + qoff, 16, 1024);
          ptx::mma_ss(tmem + (gs & 1) * HN, qd, make_sdesc(kb0 + koff, 16, 1024), IDESC_S,
                      kk > 0 ? 1u : 0u);
          ptx::mma_ss(tmem + ((gs + 1) & 1) * HN, qd, make_sdesc(kb1 + koff, 16, 1024), IDESC_S,
                      kk > 0 ? 1u : 0u);
        }
        ptx::mma_commit(&bars->k_empty[sl0]);
        ptx::mma_commit(&bars->k_empty[sl1]);
        ptx::mma_commit(&bars->s_full[gs & 1]);
        ptx::mma_commit(&bars->s_full[(gs + 1) & 1]);
      }
      __syncwarp();
      gk += 2;
      gs += 2;
    };
    for (;; ++it) {
      const int slot = it & 1;
      ptx::mbar_wait(&bars->sched_full[slot], (it >> 1) & 1);
      const int item = bars->sched_item[slot];
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&bars->sched_empty[slot]);
      if (item < 0) break;
      int h, qb;
      decode_item(item, s, h, qb);
      const bool vis = qb < s.M_v;
      const int n = vis ? kv_cnt[(int64_t)h * s.M_v + qb] : s.M_total;
      const int T = 2 * n;
      ptx::mbar_wait(&bars->q_full, it & 1);
      if (T == 0) {  // cannot come from build_block_mask (diagonal); keep the pipes consistent
        if (ptx::elect_one()) {
          ptx::mma_commit(&bars->q_empty);
          ptx::mma_commit(&bars->o_full);
        }
        __syncwarp();
        continue;
      }
      const bool pair = (dbg & 4) != 0;
      if (pair) issue_pair(); else issue_s();
      for (int t = 0; t < T; ++t) {
        if (pair) {
          // paired issue: S(t+1), S(t+2) once PV(t-1) and PV(t) are queued (both S buffers free)
        } else if (t + 1 < T) {
          issue_s();
          if (t + 2 == T) {
            if (ptx::elect_one()) ptx::mma_commit(&bars->q_empty);
            __syncwarp();
          }
        }
        // ---- O += P(t) V(t): A = P from TMEM (32 packed columns), K = 64 keys
        ptx::mbar_wait(&bars->p_full[gp & 1], (gp >> 1) & 1);
        const int vs = gv % V_SLOTS;
        ptx::mbar_wait(&bars->v_full[vs], (gv / V_SLOTS) & 1);
        ptx::tc_fence_after();
        const uint32_t vbase = aV + vs * L::HALF_BYTES;
        const uint32_t pcol = tmem + (gp & 1) * HN;
        if (ptx::elect_one()) {
#pragma unroll
          for (int kk = 0; kk < HN / 16; ++kk) {
            ptx::mma_ts(tmem + O_COL, pcol + kk * 8,
                        make_sdesc(vbase + kk * 16 * 128, L::H_CHUNK, 1024), IDESC_O,
                        (t > 0 || kk > 0) ? 1u : 0u);
          }
          ptx::mma_commit(&bars->v_empty[vs]);
          ptx::mma_commit(&bars->o_done);
        }
        __syncwarp();
        ++gv;
        ++gp;
        if (pair && (t & 1) && t + 1 < T) {
          issue_pair();
          if (t + 3 == T) {
            if (ptx::elect_one()) ptx::mma_commit(&bars->q_empty);
            __syncwarp();
          }
        }
      }
      if (pair && T == 2) {
        if (ptx::elect_one()) ptx::mma_commit(&bars->q_empty);
        __syncwarp();
      }
      if (ptx::elect_one()) ptx::mma_commit(&bars->o_full);
      __syncwarp();
    }
  } else {
    // ============================ softmax / correction / epilogue ============================
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;
    const uint32_t t_row = tmem + ((uint32_t)(quarter * 32) << 16);
    uint32_t it = 0, g = 0;
    for (;; ++it) {
      const int slot = it & 1;
      ptx::mbar_wait(&bars->sched_full[slot], (it >> 1) & 1);
      const int item = bars->sched_item[slot];
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&bars->sched_empty[slot]);
      if (item < 0) break;
      int h, qb;
      decode_item(item, s, h, qb);
      const bool vis = qb < s.M_v;
      const int n = vis ? kv_cnt[(int64_t)h * s.M_v + qb] : s.M_total;
      KvList kl(vis ? kv_idx + ((int64_t)h * s.M_v + qb) * s.M_total : nullptr, n, lane);
      const int T = 2 * n;
      float m_run = -INFINITY, l_run = 0.f;
      int b = 0, kvalid = BK;
      float bias = 0.f;
      for (int t = 0; t < T; ++t, ++g) {
        if ((t & 1) == 0) {
          b = kl.block(t >> 1);
          kvalid = block_valid(b, BK, s.M_v, s.n_valid, s.n_cond);
          bias = (vis && b >= s.M_v) ? beta_log2 : 0.f;
        }
        const int hvalid = kvalid - (t & 1) * HN;  // valid keys in this half (may be <= 0)
        ptx::mbar_wait(&bars->s_full[g & 1], (g >> 1) & 1);
        ptx::tc_fence_after();
        if (dbg & 2) {  // timing experiment: no softmax work
          l_run = 1.f;
          ptx::mbar_arrive(&bars->p_full[g & 1]);
          continue;
        }
        uint32_t sr[64];
        ptx::tmem_ld32(t_row + (g & 1) * HN, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
        ptx::tmem_ld32(t_row + (g & 1) * HN + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
        ptx::tmem_wait_ld();
        if (hvalid < HN) {  // padding keys of a partial block -> -inf (attention.py:193)
#pragma unroll
          for (int e = 0; e < 64; ++e)
            if (e >= hvalid) sr[e] = __float_as_uint(-INFINITY);
        }
        float mx8[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) mx8[e] = __uint_as_float(sr[e]);
#pragma unroll
        for (int e = 8; e < 64; e += 16)
#pragma unroll
          for (int q = 0; q < 8; ++q)
            mx8[q] = fmax3(mx8[q], __uint_as_float(sr[e + q]), __uint_as_float(sr[e + 8 + q]));
        const float mraw = fmax3(fmax3(mx8[0], mx8[1], mx8[2]), fmax3(mx8[3], mx8[4], mx8[5]),
                                 fmaxf(mx8[6], mx8[7]));
        // block max in the scaled log2 domain (scale > 0 keeps the argmax)
        const float m_blk = (mraw == -INFINITY) ? -INFINITY : fmaf(mraw, scale_log2, bias);
        const float m_new = fmaxf(m_run, m_blk);
        const bool first = (t == 0);
        const bool need = !first && (m_new > m_run + RESCALE_THRESHOLD);
        const float m_use = (first || need) ? m_new : m_run;
        const float alpha = need ? ptx::ex2(m_run - m_new) : 1.f;
        // p = 2^(s * scale_log2 + bias - m_use): one FFMA2 per two keys
        const float c0 = bias - m_use;
        const uint64_t sc2 = f2_pack(scale_log2, scale_log2), c02 = f2_pack(c0, c0);
        uint64_t acc2[4] = {0, 0, 0, 0};
        uint32_t pk[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const uint64_t x = ffma2(f2_pack(__uint_as_float(sr[2 * e]), __uint_as_float(sr[2 * e + 1])),
                                   sc2, c02);
          float p0, p1;
          if ((e & 7) >= 8 - EMU) {  // FMA-pipe exp2 for EMU of every 8 pairs
            const uint64_t pp = exp2_poly2(x);
            p0 = f2_lo(pp);
            p1 = f2_hi(pp);
          } else {
            p0 = ptx::ex2(f2_lo(x));
            p1 = ptx::ex2(f2_hi(x));
          }
          acc2[e & 3] = fadd2(acc2[e & 3], f2_pack(p0, p1));
          pk[e] = Elem<E>::pack(p0, p1);
        }
        ptx::tmem_st32(t_row + (g & 1) * HN, pk);
        const uint64_t sum2 = fadd2(fadd2(acc2[0], acc2[1]), fadd2(acc2[2], acc2[3]));
        l_run = l_run * alpha + (f2_lo(sum2) + f2_hi(sum2));
        m_run = m_use;
        if (__any_sync(0xffffffffu, need)) {
          // O is final only once PV(t-1) retired: o_done completes once per PV
          ptx::mbar_wait(&bars->o_done, (g - 1) & 1);
          ptx::tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < D / 32; ++c) {
            uint32_t ov[32];
            ptx::tmem_ld32(t_row + O_COL + c * 32, ov);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * alpha);
            ptx::tmem_st32(t_row + O_COL + c * 32, ov);
          }
        }
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&bars->p_full[g & 1]);
      }
      // ---- epilogue: O / l -> bf16 row, padding rows zero (attention.py:203-206)
      ptx::mbar_wait(&bars->o_full, it & 1);
      ptx::tc_fence_after();
      const int qvalid = block_valid(qb, BM, s.M_v, s.n_valid, s.n_cond);
      const float inv_l = (row < qvalid) ? 1.f / l_run : 0.f;
      E* orow = o + (int64_t)h * s.sh + ((int64_t)qb * BM + row) * s.sn;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        uint32_t ov[32];
        ptx::tmem_ld32(t_row + O_COL + c * 32, ov);
        ptx::tmem_wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e)
          pk[e] = Elem<E>::pack(__uint_as_float(ov[2 * e]) * inv_l,
                                 __uint_as_float(ov[2 * e + 1]) * inv_l);
        int4* dst = reinterpret_cast<int4*>(orow + c * 32);
#pragma unroll
        for (int e = 0; e < 4; ++e)
          __stcs(dst + e, make_int4((int)pk[4 * e], (int)pk[4 * e + 1], (int)pk[4 * e + 2],
                                    (int)pk[4 * e + 3]));  // streaming: keep K/V resident in L2
      }
      ptx::tc_fence_before();
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<TMEM_COLS>(tmem);
  }
}

}  // namespace tc

// =====================================================================================
// tcgen05 kernel, two-tile variant: one CTA per SM holding TWO independent query tiles
// (two work items, each its own (head, q-block) and kv list).  Each tile owns 256 TMEM
// columns: S [0,128) for a full 128-key block, O [128, 256).  The MMA warp alternates the
// tiles turn by turn -- QK0(0) QK1(0) | PV0(0) QK0(1) | PV1(0) QK1(1) | PV0(1) QK0(2) ... --
// so one tile's softmax always overlaps the other tile's MMAs.  QK^T for a 128-key block
// is one N=128 MMA per k-step (a lone SS N=64 MMA is shared-memory-port bound at 67 %).
// K and V arrive as full 128-key tiles through ONE ring in the MMA's consumption order, so
// the producer can run ahead by the whole ring.
// =====================================================================================
namespace tc2 {

using tc::BM;
using tc::BK;
using tc::HN;
// NT query tiles per CTA: NT = 2 -> one CTA per SM, one MMA warp alternating both tiles;
// NT = 1 -> two CTAs per SM, each an independent tile pipeline (two MMA issuers per SM).
template <int NT>
struct Cfg {
  static constexpr int NUM_THREADS = 64 + 128 * NT;  // w0 TMA+scheduler, w1 MMA, 4 warps/tile
  static constexpr int TMEM_COLS = 256 * NT;         // tile a: S [256a, +128), O [256a+128, +128)
  static constexpr int MAX_SMEM = NT == 2 ? 232448 : 115712;  // per CTA at 1 / 2 CTAs per SM
};
constexpr float RESCALE_THRESHOLD = 8.0f;

template <int D, int NT>
struct Smem {
  static constexpr int Q_BYTES = BM * D * 2;
  static constexpr int TILE_BYTES = BK * D * 2;   // one K or V block
  static constexpr int CHUNKS = D / 64;
  static constexpr int CHUNK = BM * 128;          // bytes per 64-col (128 B swizzle) chunk
  static constexpr int BAR_BYTES = 1024;
  static constexpr int R0 = (Cfg<NT>::MAX_SMEM - BAR_BYTES - NT * Q_BYTES) / TILE_BYTES;
  static constexpr int RING = R0 > 16 ? 16 : R0;  // K/V tiles in flight
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_RING = NT * Q_BYTES;
  static constexpr int OFF_BAR = OFF_RING + RING * TILE_BYTES;
  static constexpr int BYTES = OFF_BAR + BAR_BYTES;
};

struct Bars {
  uint64_t q_full[2], q_empty[2], s_full[2], p_full[2], o_full[2], o_empty[2];
  uint64_t sched_full[2][2], sched_empty[2][2];
  uint64_t r_full[16], r_empty[16];
  int sched_item[2][2];
  uint32_t tmem_base;
};
static_assert(sizeof(Bars) <= 1024, "barrier block must fit the reserved smem");

// Per-tile progress of the turn schedule; the producer and the MMA warp step identical
// copies of it so they agree on the ring order without talking to each other.
struct TileState {
  int n = 0, j = 0;        // steps of the current item, next QK step
  bool pending = false;    // a QK was issued whose PV has not been
  bool active = true;
  uint32_t items = 0;      // items taken (incl. empty ones): sched ring / o_full phases
  uint32_t qloads = 0;     // items with n > 0: Q ring phases
};

// Debug timeline (TCB_CARVE_DEBUG bit 3): CTA 0 records (event, step, clock) so the
// pipeline's critical path can be read without a profiler.  Off in production.
constexpr int TRACE_EV = 24, TRACE_STEPS = 4096;
__device__ unsigned long long g_trace[TRACE_EV][TRACE_STEPS];  // clock per (event, step)
__device__ __forceinline__ void trace(int dbg, int ev, int step) {
  if ((dbg & 8) && blockIdx.x == 0 && step < TRACE_STEPS) g_trace[ev][step] = clock64();
}

template <int D, int NT, typename E = __nv_bfloat16>
__global__ void __launch_bounds__(Cfg<NT>::NUM_THREADS, 3 - NT)
    k_carve_tc2(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                const __grid_constant__ CUtensorMap tm_v, E* __restrict__ o, CarveShape s,
                const int32_t* __restrict__ kv_idx, const int32_t* __restrict__ kv_cnt,
                int* __restrict__ counter, int total_items, float scale_log2, float beta_log2,
                int dbg) {
  using L = Smem<D, NT>;
  constexpr int TMEM_COLS = Cfg<NT>::TMEM_COLS;
  constexpr int RING = L::RING;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sQ = smem + L::OFF_Q;
  uint8_t* sR = smem + L::OFF_RING;
  Bars* bars = reinterpret_cast<Bars*>(smem + L::OFF_BAR);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    if (ptx::smem_u32(smem) & 1023u) __trap();
    for (int a = 0; a < NT; ++a) {
      ptx::mbar_init(&bars->q_full[a], 1);
      ptx::mbar_init(&bars->q_empty[a], 1);
      ptx::mbar_init(&bars->s_full[a], 1);
      ptx::mbar_init(&bars->p_full[a], 128);
      ptx::mbar_init(&bars->o_full[a], 1);
      ptx::mbar_init(&bars->o_empty[a], 128);
      for (int i = 0; i < 2; ++i) {
        ptx::mbar_init(&bars->sched_full[a][i], 1);
        ptx::mbar_init(&bars->sched_empty[a][i], 2);  // MMA warp + the tile's softmax group
      }
    }
    for (int i = 0; i < RING; ++i) {
      ptx::mbar_init(&bars->r_full[i], 1);
      ptx::mbar_init(&bars->r_empty[i], 1);
    }
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&tm_q);
    ptx::tma_prefetch_desc(&tm_k);
    ptx::tma_prefetch_desc(&tm_v);
  }
  if (warp == 1) ptx::tmem_alloc<TMEM_COLS>(&bars->tmem_base);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == 0) {
    // ============================ TMA producer + scheduler ============================
    const uint64_t pol_kv = ptx::policy_evict_last();
    const uint64_t pol_q = ptx::policy_evict_first();
    TileState ts[NT];
    tc::KvList kl[NT];
    int head[NT] = {0}, qblk[NT] = {0};
    bool visr[NT] = {false};
    uint32_t gr = 0;
    auto load_tile = [&](int a, int b, bool is_v) {
      if (lane == 0) {
        const int sl = gr % RING;
        ptx::mbar_wait(&bars->r_empty[sl], ((gr / RING) & 1) ^ 1);
        if ((dbg & 1) && gr >= (uint32_t)RING) {  // timing experiment: no operand traffic
          ptx::mbar_arrive(&bars->r_full[sl]);
        } else {
          ptx::mbar_arrive_expect_tx(&bars->r_full[sl], L::TILE_BYTES);
#pragma unroll
          for (int c = 0; c < L::CHUNKS; ++c)
            ptx::tma_load_3d(sR + sl * L::TILE_BYTES + c * L::CHUNK, is_v ? &tm_v : &tm_k,
                             &bars->r_full[sl], c * 64, b * BK, head[a], visr[a] ? pol_kv : pol_q);
        }
      }
      ++gr;
    };
    while (ts[0].active || (NT == 2 && ts[NT - 1].active)) {
#pragma unroll
      for (int a = 0; a < NT; ++a) {
        TileState& t = ts[a];
        if (!t.active) continue;
        if (t.pending) {  // V tile of the step whose PV comes next
          load_tile(a, kl[a].block(t.j - 1), true);
          t.pending = false;
        }
        while (t.j == t.n) {  // take the next item for this tile
          const int slot = t.items & 1;
          int item = 0;
          if (lane == 0) {
            ptx::mbar_wait(&bars->sched_empty[a][slot], ((t.items >> 1) & 1) ^ 1);
            item = atomicAdd(counter, 1);
            if (item >= total_items) item = -1;
            bars->sched_item[a][slot] = item;
            ptx::mbar_arrive(&bars->sched_full[a][slot]);
          }
          item = __shfl_sync(0xffffffffu, item, 0);
          ++t.items;
          if (item < 0) {
            t.active = false;
            break;
          }
          int h, qb;
          decode_item(item, s, h, qb);
          const bool vis = qb < s.M_v;
          t.n = vis ? __ldg(kv_cnt + (int64_t)h * s.M_v + qb) : s.M_total;
          t.j = 0;
          head[a] = h;
          qblk[a] = qb;
          visr[a] = vis;
          kl[a] = tc::KvList(vis ? kv_idx + ((int64_t)h * s.M_v + qb) * s.M_total : nullptr, t.n,
                             lane);
          if (t.n > 0) {
            if (lane == 0) {
              ptx::mbar_wait(&bars->q_empty[a], (t.qloads & 1) ^ 1);
              ptx::mbar_arrive_expect_tx(&bars->q_full[a], L::Q_BYTES);
#pragma unroll
              for (int c = 0; c < L::CHUNKS; ++c)
                ptx::tma_load_3d(sQ + a * L::Q_BYTES + c * L::CHUNK, &tm_q, &bars->q_full[a],
                                 c * 64, qb * BM, h, pol_q);
            }
            ++t.qloads;
          }
        }
        if (!t.active) continue;
        load_tile(a, kl[a].block(t.j), false);  // K tile of the next QK
        ++t.j;
        t.pending = true;
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ============================
    constexpr uint32_t IDESC_S = tc::make_idesc(BM, BK, 0, tc::Elem<E>::kBf16);
    constexpr uint32_t IDESC_O = tc::make_idesc(BM, D, 1, tc::Elem<E>::kBf16);
    const uint32_t aQ = ptx::smem_u32(sQ), aR = ptx::smem_u32(sR);
    TileState ts[NT];
    uint32_t gr = 0, gp[NT] = {0}, gq[NT] = {0};
    auto take = [&]() {  // next ring slot (in consumption order), waited full
      const int sl = gr % RING;
      ptx::mbar_wait(&bars->r_full[sl], (gr / RING) & 1);
      ++gr;
      return sl;
    };
    while (ts[0].active || (NT == 2 && ts[NT - 1].active)) {
#pragma unroll
      for (int a = 0; a < NT; ++a) {
        TileState& t = ts[a];
        if (!t.active) continue;
        const uint32_t s_col = tmem + a * 256, o_col = s_col + 128;
        if (t.pending) {  // ---- O += P(j-1) V(j-1), A = P from TMEM (64 packed columns)
          if (t.j == 1 && t.items > 1) {  // O still holds the previous item until its epilogue
            ptx::mbar_wait(&bars->o_empty[a], (t.items - 2) & 1);
          }
          if (lane == 0) trace(dbg, 1 + a, gp[a]);
          ptx::mbar_wait(&bars->p_full[a], gp[a] & 1);
          if (lane == 0) trace(dbg, 3 + a, gp[a]);
          ++gp[a];
          const int vt = take();
          if (lane == 0) trace(dbg, 16 + a, gp[a] - 1);
          ptx::tc_fence_after();
          if (ptx::elect_one()) {
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint32_t vb = aR + vt * L::TILE_BYTES + kk * 16 * 128;
              ptx::mma_ts(o_col, s_col + kk * 8, tc::make_sdesc(vb, L::CHUNK, 1024), IDESC_O,
                          (t.j > 1 || kk > 0) ? 1u : 0u);
            }
            ptx::mma_commit(&bars->r_empty[vt]);
            if (t.j == t.n) ptx::mma_commit(&bars->o_full[a]);
          }
          __syncwarp();
          if (lane == 0) trace(dbg, 20 + a, gp[a] - 1);
          t.pending = false;
        }
        while (t.j == t.n) {
          const int slot = t.items & 1;
          ptx::mbar_wait(&bars->sched_full[a][slot], (t.items >> 1) & 1);
          // broadcast so the compiler sees warp-uniform values: descriptors built from them
          // stay in uniform registers (no per-MMA R2UR/ELECT waterfall)
          const int item = __shfl_sync(0xffffffffu, bars->sched_item[a][slot], 0);
          if (lane == 0) ptx::mbar_arrive(&bars->sched_empty[a][slot]);
          ++t.items;
          if (item < 0) {
            t.active = false;
            break;
          }
          int h, qb;
          decode_item(item, s, h, qb);
          const bool vis = qb < s.M_v;
          t.n = __shfl_sync(0xffffffffu, vis ? kv_cnt[(int64_t)h * s.M_v + qb] : s.M_total, 0);
          t.j = 0;
          if (t.n == 0) {  // cannot come from build_block_mask; keep the epilogue in step
            if (t.items > 1) ptx::mbar_wait(&bars->o_empty[a], (t.items - 2) & 1);
            if (ptx::elect_one()) ptx::mma_commit(&bars->o_full[a]);
            __syncwarp();
          } else {
            ptx::mbar_wait(&bars->q_full[a], t.qloads & 1);
            ++t.qloads;
          }
        }
        if (!t.active) continue;
        // ---- S = Q K(j)^T, M = N = 128
        if (lane == 0) trace(dbg, 7 + a, gq[a]);
        const int kt = take();
        if (lane == 0) trace(dbg, 5 + a, gq[a]);
        ++gq[a];
        ptx::tc_fence_after();
        const uint32_t qa = aQ + a * L::Q_BYTES, kb = aR + kt * L::TILE_BYTES;
        if (ptx::elect_one()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk >> 2) * L::CHUNK + (kk & 3) * 32;
            ptx::mma_ss(s_col, tc::make_sdesc(qa + off, 16, 1024), tc::make_sdesc(kb + off, 16, 1024),
                        IDESC_S, kk > 0 ? 1u : 0u);
          }
          ptx::mma_commit(&bars->r_empty[kt]);
          ptx::mma_commit(&bars->s_full[a]);
          if (t.j + 1 == t.n) ptx::mma_commit(&bars->q_empty[a]);
        }
        __syncwarp();
        if (lane == 0) trace(dbg, 18 + a, gq[a] - 1);
        ++t.j;
        t.pending = true;
      }
    }
  } else {
    // ============================ softmax / correction / epilogue ============================
    const int a = (warp - 2) >> 2;  // tile of this warp group
    const int quarter = warp & 3;   // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;
    const uint32_t t_row = tmem + a * 256 + ((uint32_t)(quarter * 32) << 16);
    const uint32_t s_col = 0, o_col = 128;
    uint32_t it = 0, g = 0;
    for (;; ++it) {
      const int slot = it & 1;
      ptx::mbar_wait(&bars->sched_full[a][slot], (it >> 1) & 1);
      const int item = bars->sched_item[a][slot];
      ptx::named_bar_sync(1 + a, 128);  // all 128 threads read the slot before it is released
      if (threadIdx.x == 64 + a * 128) ptx::mbar_arrive(&bars->sched_empty[a][slot]);
      if (item < 0) break;
      int h, qb;
      decode_item(item, s, h, qb);
      const bool vis = qb < s.M_v;
      const int n = vis ? kv_cnt[(int64_t)h * s.M_v + qb] : s.M_total;
      tc::KvList kl(vis ? kv_idx + ((int64_t)h * s.M_v + qb) * s.M_total : nullptr, n, lane);
      float m_run = -INFINITY, l_run = 0.f;
      for (int j = 0; j < n; ++j, ++g) {
        const int b = kl.block(j);
        const int kvalid = block_valid(b, BK, s.M_v, s.n_valid, s.n_cond);
        const float bias = (vis && b >= s.M_v) ? beta_log2 : 0.f;
        if (lane == 0 && (warp & 3) == 2) trace(dbg, 10 + a, g);
        ptx::mbar_wait(&bars->s_full[a], g & 1);
        if (lane == 0 && (warp & 3) == 2) trace(dbg, 12 + a, g);
        ptx::tc_fence_after();
        if (dbg & 2) {  // timing experiment: no softmax work
          l_run = 1.f;
          ptx::mbar_arrive(&bars->p_full[a]);
          continue;
        }
        uint32_t sr[128];
#pragma unroll
        for (int c = 0; c < 4; ++c)
          ptx::tmem_ld32(t_row + s_col + 32 * c, *reinterpret_cast<uint32_t(*)[32]>(&sr[32 * c]));
        ptx::tmem_wait_ld();
        if (kvalid < BK) {  // padding keys of a partial block -> -inf (attention.py:193)
#pragma unroll
          for (int e = 0; e < 128; ++e)
            if (e >= kvalid) sr[e] = __float_as_uint(-INFINITY);
        }
        float mx8[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) mx8[e] = __uint_as_float(sr[e]);
#pragma unroll
        for (int e = 8; e < 120; e += 16)
#pragma unroll
          for (int q = 0; q < 8; ++q)
            mx8[q] = tc::fmax3(mx8[q], __uint_as_float(sr[e + q]), __uint_as_float(sr[e + 8 + q]));
#pragma unroll
        for (int q = 0; q < 8; ++q) mx8[q] = fmaxf(mx8[q], __uint_as_float(sr[120 + q]));
        const float mraw = tc::fmax3(tc::fmax3(mx8[0], mx8[1], mx8[2]),
                                     tc::fmax3(mx8[3], mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]));
        const float m_blk = (mraw == -INFINITY) ? -INFINITY : fmaf(mraw, scale_log2, bias);
        const float m_new = fmaxf(m_run, m_blk);
        const bool first = (j == 0);
        const bool need = !first && (m_new > m_run + RESCALE_THRESHOLD);
        const float m_use = (first || need) ? m_new : m_run;
        const float alpha = need ? ptx::ex2(m_run - m_new) : 1.f;
        const float c0 = bias - m_use;
        const uint64_t sc2 = tc::f2_pack(scale_log2, scale_log2), c02 = tc::f2_pack(c0, c0);
        uint64_t acc2[4] = {0, 0, 0, 0};
#pragma unroll
        for (int c = 0; c < 4; ++c) {  // 32 keys -> 16 packed columns per store
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const int k = 32 * c + 2 * e;
            const uint64_t x = tc::ffma2(
                tc::f2_pack(__uint_as_float(sr[k]), __uint_as_float(sr[k + 1])), sc2, c02);
            const float p0 = ptx::ex2(tc::f2_lo(x)), p1 = ptx::ex2(tc::f2_hi(x));
            acc2[e & 3] = tc::fadd2(acc2[e & 3], tc::f2_pack(p0, p1));
            pk[e] = tc::Elem<E>::pack(p0, p1);
          }
          ptx::tmem_st16(t_row + s_col + 16 * c, pk);
        }
        const uint64_t sum2 = tc::fadd2(tc::fadd2(acc2[0], acc2[1]), tc::fadd2(acc2[2], acc2[3]));
        l_run = l_run * alpha + (tc::f2_lo(sum2) + tc::f2_hi(sum2));
        m_run = m_use;
        if (__any_sync(0xffffffffu, need)) {
          // PV(j-1) retired before S(j) was committed (same issuing thread, in order)
#pragma unroll 1
          for (int c = 0; c < D / 32; ++c) {
            uint32_t ov[32];
            ptx::tmem_ld32(t_row + o_col + c * 32, ov);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * alpha);
            ptx::tmem_st32(t_row + o_col + c * 32, ov);
          }
        }
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&bars->p_full[a]);
        if (lane == 0 && (warp & 3) == 2) trace(dbg, 14 + a, g);
      }
      // ---- epilogue: O / l -> row, padding rows zero (attention.py:203-206)
      ptx::mbar_wait(&bars->o_full[a], it & 1);
      ptx::tc_fence_after();
      const int qvalid = block_valid(qb, BM, s.M_v, s.n_valid, s.n_cond);
      const float inv_l = (row < qvalid && n > 0) ? 1.f / l_run : 0.f;
      E* orow = o + (int64_t)h * s.sh + ((int64_t)qb * BM + row) * s.sn;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        uint32_t ov[32];
        ptx::tmem_ld32(t_row + o_col + c * 32, ov);
        ptx::tmem_wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e)
          pk[e] = n > 0 ? tc::Elem<E>::pack(__uint_as_float(ov[2 * e]) * inv_l,
                                            __uint_as_float(ov[2 * e + 1]) * inv_l)
                        : 0u;
        int4* dst = reinterpret_cast<int4*>(orow + c * 32);
#pragma unroll
        for (int e = 0; e < 4; ++e)
          __stcs(dst + e, make_int4((int)pk[4 * e], (int)pk[4 * e + 1], (int)pk[4 * e + 2],
                                    (int)pk[4 * e + 3]));
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&bars->o_empty[a]);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<TMEM_COLS>(tmem);
  }
}

}  // namespace tc2

// =====================================================================================
// tcgen05 kernel, full-block steps with split issue (TCB_CARVE_V2=3 while under test).
// Two CTAs per SM, each one query tile with S [0,128) (a full 128-key block) and
// O [128, 256) in TMEM, so every QK^T runs at N = 128 (full tensor rate; N = 64 is
// shared-memory-port bound at 67 %) and the two CTAs' MMA warps keep the pipe fed.  The
// per-tile chain QK -> softmax -> PV -> QK is shortened by splitting both ends:
//   * as soon as the softmax warps have S(j) in registers (s_read), the MMA warp computes
//     keys 64..127 of S(j+1) into columns [64,128) -- P(j) only occupies [0,64);
//   * P(j) is published in two halves (p_half[0], p_half[1]); PV(j) over keys 0..63 runs
//     while the softmax computes keys 64..127;
//   * after PV(j) the MMA warp fills keys 0..63 of S(j+1) over P(j)'s columns.
// O rescales (lazy, threshold 8) happen before the first half of P(j) is published, so
// they never race PV(j).
// =====================================================================================
namespace tc3 {

using tc::BM;
using tc::BK;
using tc::HN;
constexpr int NUM_THREADS = 192;  // w0 TMA+scheduler, w1 MMA+TMEM owner, w2..5 softmax
constexpr int TMEM_COLS = 256;
constexpr int MAX_SMEM = 115712;  // per CTA at two CTAs per SM
constexpr float RESCALE_THRESHOLD = 8.0f;

template <int D>
struct Smem {
  static constexpr int Q_BYTES = BM * D * 2;
  static constexpr int TILE_BYTES = BK * D * 2;
  static constexpr int CHUNKS = D / 64;
  static constexpr int CHUNK = BM * 128;
  static constexpr int BAR_BYTES = 512;
  static constexpr int R0 = (MAX_SMEM - BAR_BYTES - Q_BYTES) / TILE_BYTES;
  static constexpr int RING = R0 > 8 ? 8 : R0;  // K/V tiles in flight (2 at d = 128)
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_RING = Q_BYTES;
  static constexpr int OFF_BAR = OFF_RING + RING * TILE_BYTES;
  static constexpr int BYTES = OFF_BAR + BAR_BYTES;
};

struct Bars {
  uint64_t q_full, q_empty, s_full, s_read, o_full, o_empty;
  uint64_t p_half[2];
  uint64_t sched_full[2], sched_empty[2];
  uint64_t r_full[8], r_empty[8];
  int sched_item[2];
  uint32_t tmem_base;
};
static_assert(sizeof(Bars) <= 512, "barrier block must fit the reserved smem");

template <int D, typename E = __nv_bfloat16>
__global__ void __launch_bounds__(NUM_THREADS, 2)
    k_carve_tc3(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                const __grid_constant__ CUtensorMap tm_v, E* __restrict__ o, CarveShape s,
                const int32_t* __restrict__ kv_idx, const int32_t* __restrict__ kv_cnt,
                int* __restrict__ counter, int total_items, float scale_log2, float beta_log2,
                int dbg) {
  using L = Smem<D>;
  constexpr int RING = L::RING;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sQ = smem + L::OFF_Q;
  uint8_t* sR = smem + L::OFF_RING;
  Bars* bars = reinterpret_cast<Bars*>(smem + L::OFF_BAR);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    if (ptx::smem_u32(smem) & 1023u) __trap();
    ptx::mbar_init(&bars->q_full, 1);
    ptx::mbar_init(&bars->q_empty, 1);
    ptx::mbar_init(&bars->s_full, 1);
    ptx::mbar_init(&bars->s_read, 128);
    ptx::mbar_init(&bars->o_full, 1);
    ptx::mbar_init(&bars->o_empty, 128);
    ptx::mbar_init(&bars->p_half[0], 128);
    ptx::mbar_init(&bars->p_half[1], 128);
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&bars->sched_full[i], 1);
      ptx::mbar_init(&bars->sched_empty[i], 2);  // MMA warp + softmax group
    }
    for (int i = 0; i < RING; ++i) {
      ptx::mbar_init(&bars->r_full[i], 1);
      ptx::mbar_init(&bars->r_empty[i], 1);
    }
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&tm_q);
    ptx::tma_prefetch_desc(&tm_k);
    ptx::tma_prefetch_desc(&tm_v);
  }
  if (warp == 1) ptx::tmem_alloc<TMEM_COLS>(&bars->tmem_base);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == 0) {
    // ============================ TMA producer + scheduler ============================
    // Ring order = MMA consumption order: K(0), then K(j+1) before V(j).
    const uint64_t pol_kv = ptx::policy_evict_last();
    const uint64_t pol_q = ptx::policy_evict_first();
    uint32_t it = 0, gr = 0, qloads = 0;
    for (;; ++it) {
      const int slot = it & 1;
      int item = 0;
      if (lane == 0) {
        ptx::mbar_wait(&bars->sched_empty[slot], ((it >> 1) & 1) ^ 1);
        item = atomicAdd(counter, 1);
        if (item >= total_items) item = -1;
        bars->sched_item[slot] = item;
        ptx::mbar_arrive(&bars->sched_full[slot]);
      }
      item = __shfl_sync(0xffffffffu, item, 0);
      if (item < 0) break;
      int h, qb;
      decode_item(item, s, h, qb);
      const bool vis = qb < s.M_v;
      const int n = vis ? __ldg(kv_cnt + (int64_t)h * s.M_v + qb) : s.M_total;
      if (n == 0) continue;
      tc::KvList kl(vis ? kv_idx + ((int64_t)h * s.M_v + qb) * s.M_total : nullptr, n, lane);
      const uint64_t pol = vis ? pol_kv : pol_q;
      if (lane == 0) {
        ptx::mbar_wait(&bars->q_empty, (qloads & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&bars->q_full, L::Q_BYTES);
#pragma unroll
        for (int c = 0; c < L::CHUNKS; ++c)
          ptx::tma_load_3d(sQ + c * L::CHUNK, &tm_q, &bars->q_full, c * 64, qb * BM, h, pol_q);
      }
      ++qloads;
      auto load = [&](const CUtensorMap* tm, int b) {
        if (lane == 0) {
          const int sl = gr % RING;
          ptx::mbar_wait(&bars->r_empty[sl], ((gr / RING) & 1) ^ 1);
          if ((dbg & 1) && gr >= (uint32_t)RING) {  // timing experiment: no operand traffic
            ptx::mbar_arrive(&bars->r_full[sl]);
          } else {
            ptx::mbar_arrive_expect_tx(&bars->r_full[sl], L::TILE_BYTES);
#pragma unroll
            for (int c = 0; c < L::CHUNKS; ++c)
              ptx::tma_load_3d(sR + sl * L::TILE_BYTES + c * L::CHUNK, tm, &bars->r_full[sl],
                               c * 64, b * BK, h, pol);
          }
        }
        ++gr;
      };
      load(&tm_k, kl.block(0));
      for (int j = 0; j < n; ++j) {
        if (j + 1 < n) load(&tm_k, kl.block(j + 1));
        load(&tm_v, kl.block(j));
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ============================
    constexpr uint32_t IDESC_S = tc::make_idesc(BM, BK, 0, tc::Elem<E>::kBf16);
    constexpr uint32_t IDESC_H = tc::make_idesc(BM, HN, 0, tc::Elem<E>::kBf16);
    constexpr uint32_t IDESC_O = tc::make_idesc(BM, D, 1, tc::Elem<E>::kBf16);
    const uint32_t aQ = ptx::smem_u32(sQ), aR = ptx::smem_u32(sR);
    const uint32_t s_col = tmem, o_col = tmem + 128;
    uint32_t it = 0, gr = 0, gs = 0, qloads = 0;
    auto take = [&]() {
      const int sl = gr % RING;
      ptx::mbar_wait(&bars->r_full[sl], (gr / RING) & 1);
      ++gr;
      return sl;
    };
    // S columns [c0, c0 + N) = Q K^T over key rows [r0, r0 + N) of the K tile in slot kt
    auto qk = [&](int kt, int r0, uint32_t c0, uint32_t idesc) {
      const uint32_t kb = aR + kt * L::TILE_BYTES + r0 * 128;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const uint32_t off = (kk >> 2) * L::CHUNK + (kk & 3) * 32;
        ptx::mma_ss(s_col + c0, tc::make_sdesc(aQ + off, 16, 1024),
                    tc::make_sdesc(kb + off, 16, 1024), idesc, kk > 0 ? 1u : 0u);
      }
    };
    // O (+)= P[keys 64h .. 64h+63] V[same keys]
    auto pv = [&](int vt, int half, bool first) {
#pragma unroll
      for (int kk = 4 * half; kk < 4 * half + 4; ++kk) {
        const uint32_t vb = aR + vt * L::TILE_BYTES + kk * 16 * 128;
        ptx::mma_ts(o_col, s_col + kk * 8, tc::make_sdesc(vb, L::CHUNK, 1024), IDESC_O,
                    (!first || kk > 0) ? 1u : 0u);
      }
    };
    for (;; ++it) {
      const int slot = it & 1;
      ptx::mbar_wait(&bars->sched_full[slot], (it >> 1) & 1);
      const int item = __shfl_sync(0xffffffffu, bars->sched_item[slot], 0);
      if (lane == 0) ptx::mbar_arrive(&bars->sched_empty[slot]);
      if (item < 0) break;
      int h, qb;
      decode_item(item, s, h, qb);
      const bool vis = qb < s.M_v;
      const int n = __shfl_sync(0xffffffffu, vis ? kv_cnt[(int64_t)h * s.M_v + qb] : s.M_total, 0);
      if (n == 0) {  // cannot come from build_block_mask; keep the epilogue in step
        if (it > 0) ptx::mbar_wait(&bars->o_empty, (it - 1) & 1);
        if (ptx::elect_one()) ptx::mma_commit(&bars->o_full);
        __syncwarp();
        continue;
      }
      ptx::mbar_wait(&bars->q_full, qloads & 1);
      ++qloads;
      int kt = take();
      ptx::tc_fence_after();
      if (ptx::elect_one()) {
        qk(kt, 0, 0, IDESC_S);
        ptx::mma_commit(&bars->r_empty[kt]);
        ptx::mma_commit(&bars->s_full);
        if (n == 1) ptx::mma_commit(&bars->q_empty);
      }
      __syncwarp();
      for (int j = 0; j < n; ++j, ++gs) {
        const bool more = j + 1 < n;
        ptx::mbar_wait(&bars->s_read, gs & 1);  // S(j) is in the softmax registers
        if (more) {
          kt = take();
          ptx::tc_fence_after();
          if (ptx::elect_one()) qk(kt, HN, HN, IDESC_H);  // keys 64..127 of S(j+1)
          __syncwarp();
        }
        ptx::mbar_wait(&bars->p_half[0], gs & 1);
        if (j == 0 && it > 0) ptx::mbar_wait(&bars->o_empty, (it - 1) & 1);  // epilogue read O
        const int vt = take();
        ptx::tc_fence_after();
        if (ptx::elect_one()) pv(vt, 0, j == 0);
        __syncwarp();
        ptx::mbar_wait(&bars->p_half[1], gs & 1);
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
          pv(vt, 1, false);
          ptx::mma_commit(&bars->r_empty[vt]);
          if (more) {
            qk(kt, 0, 0, IDESC_H);  // keys 0..63 of S(j+1), over P(j)'s columns
            ptx::mma_commit(&bars->r_empty[kt]);
            ptx::mma_commit(&bars->s_full);
            if (j + 2 == n) ptx::mma_commit(&bars->q_empty);
          } else {
            ptx::mma_commit(&bars->o_full);
          }
        }
        __syncwarp();
      }
    }
  } else {
    // ============================ softmax / correction / epilogue ============================
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t t_row = tmem + ((uint32_t)(quarter * 32) << 16);
    constexpr uint32_t s_col = 0, o_col = 128;
    uint32_t it = 0, g = 0;
    for (;; ++it) {
      const int slot = it & 1;
      ptx::mbar_wait(&bars->sched_full[slot], (it >> 1) & 1);
      const int item = bars->sched_item[slot];
      ptx::named_bar_sync(1, 128);
      if (threadIdx.x == 64) ptx::mbar_arrive(&bars->sched_empty[slot]);
      if (item < 0) break;
      int h, qb;
      decode_item(item, s, h, qb);
      const bool vis = qb < s.M_v;
      const int n = vis ? kv_cnt[(int64_t)h * s.M_v + qb] : s.M_total;
      tc::KvList kl(vis ? kv_idx + ((int64_t)h * s.M_v + qb) * s.M_total : nullptr, n, lane);
      float m_run = -INFINITY, l_run = 0.f;
      for (int j = 0; j < n; ++j, ++g) {
        const int b = kl.block(j);
        const int kvalid = block_valid(b, BK, s.M_v, s.n_valid, s.n_cond);
        const float bias = (vis && b >= s.M_v) ? beta_log2 : 0.f;
        ptx::mbar_wait(&bars->s_full, g & 1);
        ptx::tc_fence_after();
        uint32_t sr[128];
#pragma unroll
        for (int c = 0; c < 4; ++c)
          ptx::tmem_ld32(t_row + s_col + 32 * c, *reinterpret_cast<uint32_t(*)[32]>(&sr[32 * c]));
        ptx::tmem_wait_ld();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&bars->s_read);
        if (dbg & 2) {  // timing experiment: no softmax work
          l_run = 1.f;
          ptx::mbar_arrive(&bars->p_half[0]);
          ptx::mbar_arrive(&bars->p_half[1]);
          continue;
        }
        if (kvalid < BK) {  // padding keys of a partial block -> -inf (attention.py:193)
#pragma unroll
          for (int e = 0; e < 128; ++e)
            if (e >= kvalid) sr[e] = __float_as_uint(-INFINITY);
        }
        float mx8[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) mx8[e] = __uint_as_float(sr[e]);
#pragma unroll
        for (int e = 8; e < 120; e += 16)
#pragma unroll
          for (int q = 0; q < 8; ++q)
            mx8[q] = tc::fmax3(mx8[q], __uint_as_float(sr[e + q]), __uint_as_float(sr[e + 8 + q]));
#pragma unroll
        for (int q = 0; q < 8; ++q) mx8[q] = fmaxf(mx8[q], __uint_as_float(sr[120 + q]));
        const float mraw = tc::fmax3(tc::fmax3(mx8[0], mx8[1], mx8[2]),
                                     tc::fmax3(mx8[3], mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]));
        const float m_blk = (mraw == -INFINITY) ? -INFINITY : fmaf(mraw, scale_log2, bias);
        const float m_new = fmaxf(m_run, m_blk);
        const bool first = (j == 0);
        const bool need = !first && (m_new > m_run + RESCALE_THRESHOLD);
        const float m_use = (first || need) ? m_new : m_run;
        const float alpha = need ? ptx::ex2(m_run - m_new) : 1.f;
        if (__any_sync(0xffffffffu, need)) {
          // PV(j-1) retired before S(j) was committed; PV(j) waits for p_half[0] below
#pragma unroll 1
          for (int c = 0; c < D / 32; ++c) {
            uint32_t ov[32];
            ptx::tmem_ld32(t_row + o_col + c * 32, ov);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * alpha);
            ptx::tmem_st32(t_row + o_col + c * 32, ov);
          }
        }
        const float c0 = bias - m_use;
        const uint64_t sc2 = tc::f2_pack(scale_log2, scale_log2), c02 = tc::f2_pack(c0, c0);
        uint64_t acc2[4] = {0, 0, 0, 0};
#pragma unroll
        for (int c = 0; c < 4; ++c) {  // 32 keys -> 16 packed columns per store
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const int k = 32 * c + 2 * e;
            const uint64_t x = tc::ffma2(
                tc::f2_pack(__uint_as_float(sr[k]), __uint_as_float(sr[k + 1])), sc2, c02);
            const float p0 = ptx::ex2(tc::f2_lo(x)), p1 = ptx::ex2(tc::f2_hi(x));
            acc2[e & 3] = tc::fadd2(acc2[e & 3], tc::f2_pack(p0, p1));
            pk[e] = tc::Elem<E>::pack(p0, p1);
          }
          ptx::tmem_st16(t_row + s_col + 16 * c, pk);
          if (c & 1) {  // keys [0,64) then [64,128) published for PV
            ptx::tmem_wait_st();
            ptx::tc_fence_before();
            ptx::mbar_arrive(&bars->p_half[c >> 1]);
          }
        }
        const uint64_t sum2 = tc::fadd2(tc::fadd2(acc2[0], acc2[1]), tc::fadd2(acc2[2], acc2[3]));
        l_run = l_run * alpha + (tc::f2_lo(sum2) + tc::f2_hi(sum2));
        m_run = m_use;
      }
      // ---- epilogue: O / l -> row, padding rows zero (attention.py:203-206)
      ptx::mbar_wait(&bars->o_full, it & 1);
      ptx::tc_fence_after();
      const int qvalid = block_valid(qb, BM, s.M_v, s.n_valid, s.n_cond);
      const float inv_l = (row < qvalid && n > 0) ? 1.f / l_run : 0.f;
      E* orow = o + (int64_t)h * s.sh + ((int64_t)qb * BM + row) * s.sn;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        uint32_t ov[32];
        ptx::tmem_ld32(t_row + o_col + c * 32, ov);
        ptx::tmem_wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e)
          pk[e] = n > 0 ? tc::Elem<E>::pack(__uint_as_float(ov[2 * e]) * inv_l,
                                            __uint_as_float(ov[2 * e + 1]) * inv_l)
                        : 0u;
        int4* dst = reinterpret_cast<int4*>(orow + c * 32);
#pragma unroll
        for (int e = 0; e < 4; ++e)
          __stcs(dst + e, make_int4((int)pk[4 * e], (int)pk[4 * e + 1], (int)pk[4 * e + 2],
                                    (int)pk[4 * e + 3]));
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&bars->o_empty);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<TMEM_COLS>(tmem);
  }
}

}  // namespace tc3

// =====================================================================================
// tcgen05 kernel, two independent tile pipelines per CTA (TCB_CARVE_V2=4 while under test).
// One CTA per SM; tile a in {0,1} owns producer warp a, MMA warp 2+a, softmax warps
// 4+4a .. 7+4a, Q slot a, a 2-slot K/V ring and TMEM columns [256a, 256a+256): S [0,128)
// (a full 128-key block -> QK^T at N = 128, full tensor rate) and O [128,256).  Two MMA
// issuers keep the tensor pipe fed (a single issuer stalls on its own waits).  PV(j) is
// split in key halves so PV over keys 0..63 runs while the softmax finishes keys 64..127.
// Optional (TCB_CARVE_DEBUG bit 4): the two tiles' exp2 phases strictly alternate (MUFU
// token), so one tile's softmax overlaps the other tile's MMAs instead of its softmax.
// =====================================================================================
namespace tc4 {

using tc::BM;
using tc::BK;
using tc::HN;
constexpr int NUM_THREADS = 384;
constexpr int TMEM_COLS = 512;
constexpr int MAX_SMEM = 232448;
constexpr float RESCALE_THRESHOLD = 8.0f;

template <int D>
struct Smem {
  static constexpr int Q_BYTES = BM * D * 2;
  static constexpr int TILE_BYTES = BK * D * 2;
  static constexpr int CHUNKS = D / 64;
  static constexpr int CHUNK = BM * 128;
  static constexpr int BAR_BYTES = 1024;
  static constexpr int R0 = (MAX_SMEM - BAR_BYTES - 2 * Q_BYTES) / (2 * TILE_BYTES);
  static constexpr int RING = R0 > 8 ? 8 : R0;  // K/V tiles in flight per tile (2 at d = 128)
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_RING = 2 * Q_BYTES;
  static constexpr int OFF_BAR = OFF_RING + 2 * RING * TILE_BYTES;
  static constexpr int BYTES = OFF_BAR + BAR_BYTES;
};

struct TileBars {
  uint64_t q_full, q_empty, s_full, o_full, o_empty, exp_done;
  uint64_t p_half[2];
  uint64_t sched_full[2], sched_empty[2];
  uint64_t r_full[8], r_empty[8];
  int sched_item[2];
  volatile int finished;
  uint32_t pad;
};
struct Bars {
  TileBars t[2];
  uint32_t tmem_base;
};
static_assert(sizeof(Bars) <= 1024, "barrier block must fit the reserved smem");

template <int D, typename E = __nv_bfloat16>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    k_carve_tc4(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                const __grid_constant__ CUtensorMap tm_v, E* __restrict__ o, CarveShape s,
                const int32_t* __restrict__ kv_idx, const int32_t* __restrict__ kv_cnt,
                int* __restrict__ counter, int total_items, float scale_log2, float beta_log2,
                int dbg) {
  using L = Smem<D>;
  constexpr int RING = L::RING;
  extern __shared__ __align__(1024) uint8_t smem[];
  Bars* bars = reinterpret_cast<Bars*>(smem + L::OFF_BAR);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int a = warp < 4 ? (warp & 1) : (warp - 4) >> 2;  // tile of this warp
  TileBars* tb = &bars->t[a];
  uint8_t* sQ = smem + L::OFF_Q + a * L::Q_BYTES;
  uint8_t* sR = smem + L::OFF_RING + a * RING * L::TILE_BYTES;

  if (threadIdx.x == 0) {
    if (ptx::smem_u32(smem) & 1023u) __trap();
    for (int i = 0; i < 2; ++i) {
      TileBars* b = &bars->t[i];
      ptx::mbar_init(&b->q_full, 1);
      ptx::mbar_init(&b->q_empty, 1);
      ptx::mbar_init(&b->s_full, 1);
      ptx::mbar_init(&b->o_full, 1);
      ptx::mbar_init(&b->o_empty, 128);
      ptx::mbar_init(&b->exp_done, 128);
      ptx::mbar_init(&b->p_half[0], 128);
      ptx::mbar_init(&b->p_half[1], 128);
      for (int k = 0; k < 2; ++k) {
        ptx::mbar_init(&b->sched_full[k], 1);
        ptx::mbar_init(&b->sched_empty[k], 2);
      }
      for (int k = 0; k < RING; ++k) {
        ptx::mbar_init(&b->r_full[k], 1);
        ptx::mbar_init(&b->r_empty[k], 1);
      }
      b->finished = 0;
    }
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&tm_q);
    ptx::tma_prefetch_desc(&tm_k);
    ptx::tma_prefetch_desc(&tm_v);
  }
  if (warp == 2) ptx::tmem_alloc<TMEM_COLS>(&bars->tmem_base);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = bars->tmem_base + a * 256;

  if (warp < 2) {
    // ============================ TMA producer + scheduler (tile a) ============================
    const uint64_t pol_kv = ptx::policy_evict_last();
    const uint64_t pol_q = ptx::policy_evict_first();
    uint32_t it = 0, gr = 0, qloads = 0;
    for (;; ++it) {
      const int slot = it & 1;
      int item = 0;
      if (lane == 0) {
        ptx::mbar_wait(&tb->sched_empty[slot], ((it >> 1) & 1) ^ 1);
        item = atomicAdd(counter, 1);
        if (item >= total_items) item = -1;
        tb->sched_item[slot] = item;
        ptx::mbar_arrive(&tb->sched_full[slot]);
      }
      item = __shfl_sync(0xffffffffu, item, 0);
      if (item < 0) break;
      int h, qb;
      decode_item(item, s, h, qb);
      const bool vis = qb < s.M_v;
      const int n = vis ? __ldg(kv_cnt + (int64_t)h * s.M_v + qb) : s.M_total;
      if (n == 0) continue;
      tc::KvList kl(vis ? kv_idx + ((int64_t)h * s.M_v + qb) * s.M_total : nullptr, n, lane);
      const uint64_t pol = vis ? pol_kv : pol_q;
      if (lane == 0) {
        ptx::mbar_wait(&tb->q_empty, (qloads & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&tb->q_full, L::Q_BYTES);
#pragma unroll
        for (int c = 0; c < L::CHUNKS; ++c)
          ptx::tma_load_3d(sQ + c * L::CHUNK, &tm_q, &tb->q_full, c * 64, qb * BM, h, pol_q);
      }
      ++qloads;
      for (int j = 0; j < n; ++j) {  // ring order = consumption order: K(j), V(j)
        const int b = kl.block(j);
#pragma unroll
        for (int kv = 0; kv < 2; ++kv) {
          if (lane == 0) {
            const int sl = gr % RING;
            ptx::mbar_wait(&tb->r_empty[sl], ((gr / RING) & 1) ^ 1);
            if ((dbg & 1) && gr >= (uint32_t)RING) {  // timing experiment: no operand traffic
              ptx::mbar_arrive(&tb->r_full[sl]);
            } else {
              ptx::mbar_arrive_expect_tx(&tb->r_full[sl], L::TILE_BYTES);
#pragma unroll
              for (int c = 0; c < L::CHUNKS; ++c)
                ptx::tma_load_3d(sR + sl * L::TILE_BYTES + c * L::CHUNK, kv ? &tm_v : &tm_k,
                                 &tb->r_full[sl], c * 64, b * BK, h, pol);
            }
          }
          ++gr;
        }
      }
    }
  } else if (warp < 4) {
    // ============================ MMA issuer (tile a) ============================
    constexpr uint32_t IDESC_S = tc::make_idesc(BM, BK, 0, tc::Elem<E>::kBf16);
    constexpr uint32_t IDESC_O = tc::make_idesc(BM, D, 1, tc::Elem<E>::kBf16);
    const uint32_t aQ = ptx::smem_u32(sQ), aR = ptx::smem_u32(sR);
    const uint32_t s_col = tmem, o_col = tmem + 128;
    uint32_t it = 0, gr = 0, gs = 0, qloads = 0;
    auto take = [&]() {
      const int sl = gr % RING;
      ptx::mbar_wait(&tb->r_full[sl], (gr / RING) & 1);
      ++gr;
      return sl;
    };
    for (;; ++it) {
      const int slot = it & 1;
      ptx::mbar_wait(&tb->sched_full[slot], (it >> 1) & 1);
      const int item = __shfl_sync(0xffffffffu, tb->sched_item[slot], 0);
      if (lane == 0) ptx::mbar_arrive(&tb->sched_empty[slot]);
      if (item < 0) break;
      int h, qb;
      decode_item(item, s, h, qb);
      const bool vis = qb < s.M_v;
      const int n = __shfl_sync(0xffffffffu, vis ? kv_cnt[(int64_t)h * s.M_v + qb] : s.M_total, 0);
      if (n == 0) {  // cannot come from build_block_mask; keep the epilogue in step
        if (it > 0) ptx::mbar_wait(&tb->o_empty, (it - 1) & 1);
        if (ptx::elect_one()) ptx::mma_commit(&tb->o_full);
        __syncwarp();
        continue;
      }
      ptx::mbar_wait(&tb->q_full, qloads & 1);
      ++qloads;
      for (int j = 0; j < n; ++j, ++gs) {
        const int kt = take();
        ptx::tc_fence_after();
        if (ptx::elect_one()) {  // S = Q K(j)^T, M = N = 128 (after PV(j-1): in order)
          const uint32_t kb = aR + kt * L::TILE_BYTES;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk >> 2) * L::CHUNK + (kk & 3) * 32;
            ptx::mma_ss(s_col, tc::make_sdesc(aQ + off, 16, 1024), tc::make_sdesc(kb + off, 16, 1024),
                        IDESC_S, kk > 0 ? 1u : 0u);
          }
          ptx::mma_commit(&tb->r_empty[kt]);
          ptx::mma_commit(&tb->s_full);
          if (j + 1 == n) ptx::mma_commit(&tb->q_empty);
        }
        __syncwarp();
        const int vt = take();
#pragma unroll
        for (int half = 0; half < 2; ++half) {  // O (+)= P V over keys [64 half, 64 half + 64)
          ptx::mbar_wait(&tb->p_half[half], gs & 1);
          if (half == 0 && j == 0 && it > 0) ptx::mbar_wait(&tb->o_empty, (it - 1) & 1);
          ptx::tc_fence_after();
          if (ptx::elect_one()) {
#pragma unroll
            for (int kk = 4 * half; kk < 4 * half + 4; ++kk) {
              const uint32_t vb = aR + vt * L::TILE_BYTES + kk * 16 * 128;
              ptx::mma_ts(o_col, s_col + kk * 8, tc::make_sdesc(vb, L::CHUNK, 1024), IDESC_O,
                          (j > 0 || kk > 0) ? 1u : 0u);
            }
            if (half == 1) {
              ptx::mma_commit(&tb->r_empty[vt]);
              if (j + 1 == n) ptx::mma_commit(&tb->o_full);
            }
          }
          __syncwarp();
        }
      }
    }
  } else {
    // ============================ softmax / correction / epilogue (tile a) ============================
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t t_row = tmem + ((uint32_t)(quarter * 32) << 16);
    constexpr uint32_t s_col = 0, o_col = 128;
    const bool token = (dbg & 16) != 0;
    TileBars* other = &bars->t[a ^ 1];
    uint32_t it = 0, g = 0;
    for (;; ++it) {
      const int slot = it & 1;
      ptx::mbar_wait(&tb->sched_full[slot], (it >> 1) & 1);
      const int item = tb->sched_item[slot];
      ptx::named_bar_sync(1 + a, 128);
      if (threadIdx.x == 128 + 128 * a) ptx::mbar_arrive(&tb->sched_empty[slot]);
      if (item < 0) break;
      int h, qb;
      decode_item(item, s, h, qb);
      const bool vis = qb < s.M_v;
      const int n = vis ? kv_cnt[(int64_t)h * s.M_v + qb] : s.M_total;
      tc::KvList kl(vis ? kv_idx + ((int64_t)h * s.M_v + qb) * s.M_total : nullptr, n, lane);
      float m_run = -INFINITY, l_run = 0.f;
      for (int j = 0; j < n; ++j, ++g) {
        const int b = kl.block(j);
        const int kvalid = block_valid(b, BK, s.M_v, s.n_valid, s.n_cond);
        const float bias = (vis && b >= s.M_v) ? beta_log2 : 0.f;
        ptx::mbar_wait(&tb->s_full, g & 1);
        ptx::tc_fence_after();
        uint32_t sr[128];
#pragma unroll
        for (int c = 0; c < 4; ++c)
          ptx::tmem_ld32(t_row + s_col + 32 * c, *reinterpret_cast<uint32_t(*)[32]>(&sr[32 * c]));
        ptx::tmem_wait_ld();
        if (dbg & 2) {  // timing experiment: no softmax work
          l_run = 1.f;
          ptx::tc_fence_before();
          ptx::mbar_arrive(&tb->p_half[0]);
          ptx::mbar_arrive(&tb->p_half[1]);
          continue;
        }
        if (kvalid < BK) {  // padding keys of a partial block -> -inf (attention.py:193)
#pragma unroll
          for (int e = 0; e < 128; ++e)
            if (e >= kvalid) sr[e] = __float_as_uint(-INFINITY);
        }
        float mx8[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) mx8[e] = __uint_as_float(sr[e]);
#pragma unroll
        for (int e = 8; e < 120; e += 16)
#pragma unroll
          for (int q = 0; q < 8; ++q)
            mx8[q] = tc::fmax3(mx8[q], __uint_as_float(sr[e + q]), __uint_as_float(sr[e + 8 + q]));
#pragma unroll
        for (int q = 0; q < 8; ++q) mx8[q] = fmaxf(mx8[q], __uint_as_float(sr[120 + q]));
        const float mraw = tc::fmax3(tc::fmax3(mx8[0], mx8[1], mx8[2]),
                                     tc::fmax3(mx8[3], mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]));
        const float m_blk = (mraw == -INFINITY) ? -INFINITY : fmaf(mraw, scale_log2, bias);
        const float m_new = fmaxf(m_run, m_blk);
        const bool first = (j == 0);
        const bool need = !first && (m_new > m_run + RESCALE_THRESHOLD);
        const float m_use = (first || need) ? m_new : m_run;
        const float alpha = need ? ptx::ex2(m_run - m_new) : 1.f;
        if (__any_sync(0xffffffffu, need)) {
          // PV(j-1) retired before S(j) was committed; PV(j) waits for p_half[0] below
#pragma unroll 1
          for (int c = 0; c < D / 32; ++c) {
            uint32_t ov[32];
            ptx::tmem_ld32(t_row + o_col + c * 32, ov);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * alpha);
            ptx::tmem_st32(t_row + o_col + c * 32, ov);
          }
        }
        if (token && !(a == 0 && g == 0)) {  // MUFU token: tiles' exp2 phases alternate
          const uint32_t k = a == 0 ? g - 1 : g;
          while (!ptx::mbar_try_wait(&other->exp_done, k & 1))
            if (other->finished) break;
        }
        const float c0 = bias - m_use;
        const uint64_t sc2 = tc::f2_pack(scale_log2, scale_log2), c02 = tc::f2_pack(c0, c0);
        uint64_t acc2[4] = {0, 0, 0, 0};
#pragma unroll
        for (int c = 0; c < 4; ++c) {  // 32 keys -> 16 packed columns per store
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const int k = 32 * c + 2 * e;
            const uint64_t x = tc::ffma2(
                tc::f2_pack(__uint_as_float(sr[k]), __uint_as_float(sr[k + 1])), sc2, c02);
            const float p0 = ptx::ex2(tc::f2_lo(x)), p1 = ptx::ex2(tc::f2_hi(x));
            acc2[e & 3] = tc::fadd2(acc2[e & 3], tc::f2_pack(p0, p1));
            pk[e] = tc::Elem<E>::pack(p0, p1);
          }
          ptx::tmem_st16(t_row + s_col + 16 * c, pk);
          if (c & 1) {  // keys [0,64) then [64,128) published for PV
            ptx::tmem_wait_st();
            ptx::tc_fence_before();
            ptx::mbar_arrive(&tb->p_half[c >> 1]);
          }
        }
        if (token) ptx::mbar_arrive(&tb->exp_done);
        const uint64_t sum2 = tc::fadd2(tc::fadd2(acc2[0], acc2[1]), tc::fadd2(acc2[2], acc2[3]));
        l_run = l_run * alpha + (tc::f2_lo(sum2) + tc::f2_hi(sum2));
        m_run = m_use;
      }
      // ---- epilogue: O / l -> row, padding rows zero (attention.py:203-206)
      ptx::mbar_wait(&tb->o_full, it & 1);
      ptx::tc_fence_after();
      const int qvalid = block_valid(qb, BM, s.M_v, s.n_valid, s.n_cond);
      const float inv_l = (row < qvalid && n > 0) ? 1.f / l_run : 0.f;
      E* orow = o + (int64_t)h * s.sh + ((int64_t)qb * BM + row) * s.sn;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        uint32_t ov[32];
        ptx::tmem_ld32(t_row + o_col + c * 32, ov);
        ptx::tmem_wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e)
          pk[e] = n > 0 ? tc::Elem<E>::pack(__uint_as_float(ov[2 * e]) * inv_l,
                                            __uint_as_float(ov[2 * e + 1]) * inv_l)
                        : 0u;
        int4* dst = reinterpret_cast<int4*>(orow + c * 32);
#pragma unroll
        for (int e = 0; e < 4; ++e)
          __stcs(dst + e, make_int4((int)pk[4 * e], (int)pk[4 * e + 1], (int)pk[4 * e + 2],
                                    (int)pk[4 * e + 3]));
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tb->o_empty);
    }
    if (token) {  // release the other tile for good
      ptx::named_bar_sync(1 + a, 128);
      if (threadIdx.x == 128 + 128 * a) tb->finished = 1;
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<TMEM_COLS>(bars->tmem_base);
  }
}

}  // namespace tc4

// =====================================================================================
// tcgen05 kernel, full-block steps with a triple-buffered S (TCB_CARVE_V2=5 while under test).
// One CTA per SM, one query tile at a time.  TMEM (512 columns): S0 S1 S2 (fp32 128 x 128,
// P(j) written as bf16 over the first 64 columns of its S buffer) and O [384, 512).  Every
// QK^T is M = N = 128 (full tensor rate).  Two MMA warps issue independently: the QK warp
// runs up to two blocks ahead of the softmax (S(j+2) while P(j) is being computed), the PV
// warp follows the softmax -- so the tensor pipe always has a queued stream while the
// softmax warps (one per SMSP, alone on its MUFU) run back to back.  Q is double-buffered so
// the next item's QK^T starts while the current item's PV drains.
// =====================================================================================
namespace tc5 {

using tc::BM;
using tc::BK;
constexpr int NUM_THREADS = 224;  // w0 TMA, w1 QK MMA + TMEM owner, w2 PV MMA, w3..6 softmax
constexpr int TMEM_COLS = 512;
constexpr int O_COL = 384;
constexpr int NS = 3;             // S buffers
constexpr int QS = 2;             // Q buffers
constexpr int SCHED = 4;          // scheduler ring entries
constexpr int MAX_SMEM = 232448;
constexpr float RESCALE_THRESHOLD = 8.0f;

template <int D>
struct Smem {
  static constexpr int Q_BYTES = BM * D * 2;
  static constexpr int TILE_BYTES = BK * D * 2;
  static constexpr int CHUNKS = D / 64;
  static constexpr int CHUNK = BM * 128;
  static constexpr int BAR_BYTES = 1024;
  static constexpr int TILES = (MAX_SMEM - BAR_BYTES - QS * Q_BYTES) / TILE_BYTES;
  static constexpr int KS = TILES >= 6 ? 4 : (TILES + 1) / 2;  // K ring (5 tiles at d = 128: 3 + 2)
  static constexpr int VS0 = TILES - KS;
  static constexpr int VS = VS0 > 4 ? 4 : VS0;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = QS * Q_BYTES;
  static constexpr int OFF_V = OFF_K + KS * TILE_BYTES;
  static constexpr int OFF_BAR = OFF_V + VS * TILE_BYTES;
  static constexpr int BYTES = OFF_BAR + BAR_BYTES;
};

struct Bars {
  uint64_t q_full[QS], q_empty[QS];
  uint64_t s_full[NS], p_full[NS], s_free[NS];
  uint64_t o_done, o_full, o_empty;
  uint64_t k_full[4], k_empty[4], v_full[4], v_empty[4];
  uint64_t sched_full[SCHED], sched_empty[SCHED];
  int sched_item[SCHED];
  uint32_t tmem_base;
};
static_assert(sizeof(Bars) <= 1024, "barrier block must fit the reserved smem");

template <int D, typename E = __nv_bfloat16>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    k_carve_tc5(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                const __grid_constant__ CUtensorMap tm_v, E* __restrict__ o, CarveShape s,
                const int32_t* __restrict__ kv_idx, const int32_t* __restrict__ kv_cnt,
                int* __restrict__ counter, int total_items, float scale_log2, float beta_log2,
                int dbg) {
  using L = Smem<D>;
  constexpr int KS = L::KS, VS = L::VS;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sQ = smem + L::OFF_Q;
  uint8_t* sK = smem + L::OFF_K;
  uint8_t* sV = smem + L::OFF_V;
  Bars* bars = reinterpret_cast<Bars*>(smem + L::OFF_BAR);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    if (ptx::smem_u32(smem) & 1023u) __trap();
    for (int i = 0; i < QS; ++i) {
      ptx::mbar_init(&bars->q_full[i], 1);
      ptx::mbar_init(&bars->q_empty[i], 1);
    }
    for (int i = 0; i < NS; ++i) {
      ptx::mbar_init(&bars->s_full[i], 1);
      ptx::mbar_init(&bars->p_full[i], 128);
      ptx::mbar_init(&bars->s_free[i], 1);
    }
    ptx::mbar_init(&bars->o_done, 1);
    ptx::mbar_init(&bars->o_full, 1);
    ptx::mbar_init(&bars->o_empty, 128);
    for (int i = 0; i < KS; ++i) {
      ptx::mbar_init(&bars->k_full[i], 1);
      ptx::mbar_init(&bars->k_empty[i], 1);
    }
    for (int i = 0; i < VS; ++i) {
      ptx::mbar_init(&bars->v_full[i], 1);
      ptx::mbar_init(&bars->v_empty[i], 1);
    }
    for (int i = 0; i < SCHED; ++i) {
      ptx::mbar_init(&bars->sched_full[i], 1);
      ptx::mbar_init(&bars->sched_empty[i], 3);  // QK warp, PV warp, softmax group
    }
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&tm_q);
    ptx::tma_prefetch_desc(&tm_k);
    ptx::tma_prefetch_desc(&tm_v);
  }
  if (warp == 1) ptx::tmem_alloc<TMEM_COLS>(&bars->tmem_base);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  // every role walks the same item sequence from the scheduler ring
  auto next_item = [&](uint32_t it, int& h, int& qb, bool& vis, int& n) -> bool {
    const int slot = it % SCHED;
    ptx::mbar_wait(&bars->sched_full[slot], (it / SCHED) & 1);
    const int item = __shfl_sync(0xffffffffu, bars->sched_item[slot], 0);
    if (item < 0) return false;
    decode_item(item, s, h, qb);
    vis = qb < s.M_v;
    n = __shfl_sync(0xffffffffu, vis ? __ldg(kv_cnt + (int64_t)h * s.M_v + qb) : s.M_total, 0);
    return true;
  };

  if (warp == 0) {
    // ============================ TMA producer + scheduler ============================
    // Issue order K(0) K(1) [V(0) K(2)] [V(1) K(3)] ...: the QK warp runs ahead of the PV warp.
    const uint64_t pol_kv = ptx::policy_evict_last();
    const uint64_t pol_q = ptx::policy_evict_first();
    uint32_t gk = 0, gv = 0, qn = 0;
    for (uint32_t it = 0;; ++it) {
      const int slot = it % SCHED;
      int item = 0;
      if (lane == 0) {
        ptx::mbar_wait(&bars->sched_empty[slot], ((it / SCHED) & 1) ^ 1);
        item = atomicAdd(counter, 1);
        if (item >= total_items) item = -1;
        bars->sched_item[slot] = item;
        ptx::mbar_arrive(&bars->sched_full[slot]);
      }
      item = __shfl_sync(0xffffffffu, item, 0);
      if (item < 0) break;
      int h, qb;
      decode_item(item, s, h, qb);
      const bool vis = qb < s.M_v;
      const int n = vis ? __ldg(kv_cnt + (int64_t)h * s.M_v + qb) : s.M_total;
      if (n == 0) continue;
      tc::KvList kl(vis ? kv_idx + ((int64_t)h * s.M_v + qb) * s.M_total : nullptr, n, lane);
      const uint64_t pol = vis ? pol_kv : pol_q;
      if (lane == 0) {
        const int qs = qn % QS;
        ptx::mbar_wait(&bars->q_empty[qs], ((qn / QS) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&bars->q_full[qs], L::Q_BYTES);
#pragma unroll
        for (int c = 0; c < L::CHUNKS; ++c)
          ptx::tma_load_3d(sQ + qs * L::Q_BYTES + c * L::CHUNK, &tm_q, &bars->q_full[qs], c * 64,
                           qb * BM, h, pol_q);
      }
      ++qn;
      auto load = [&](bool is_v, int b) {
        uint32_t& cnt = is_v ? gv : gk;
        const int slots = is_v ? VS : KS;
        if (lane == 0) {
          const int sl = cnt % slots;
          uint64_t* full = is_v ? bars->v_full : bars->k_full;
          uint64_t* empty = is_v ? bars->v_empty : bars->k_empty;
          ptx::mbar_wait(&empty[sl], ((cnt / slots) & 1) ^ 1);
          if ((dbg & 1) && cnt >= (uint32_t)slots) {  // timing experiment: no operand traffic
            ptx::mbar_arrive(&full[sl]);
          } else {
            ptx::mbar_arrive_expect_tx(&full[sl], L::TILE_BYTES);
            uint8_t* base = (is_v ? sV : sK) + sl * L::TILE_BYTES;
#pragma unroll
            for (int c = 0; c < L::CHUNKS; ++c)
              ptx::tma_load_3d(base + c * L::CHUNK, is_v ? &tm_v : &tm_k, &full[sl], c * 64, b * BK,
                               h, pol);
          }
        }
        ++cnt;
      };
      load(false, kl.block(0));
      if (n > 1) load(false, kl.block(1));
      for (int j = 0; j < n; ++j) {
        load(true, kl.block(j));
        if (j + 2 < n) load(false, kl.block(j + 2));
      }
    }
  } else if (warp == 1) {
    // ============================ QK^T issuer ============================
    constexpr uint32_t IDESC_S = tc::make_idesc(BM, BK, 0, tc::Elem<E>::kBf16);
    const uint32_t aQ = ptx::smem_u32(sQ), aK = ptx::smem_u32(sK);
    uint32_t gk = 0, gs = 0, qn = 0;
    for (uint32_t it = 0;; ++it) {
      int h, qb, n;
      bool vis;
      const bool ok = next_item(it, h, qb, vis, n);
      if (lane == 0) ptx::mbar_arrive(&bars->sched_empty[it % SCHED]);
      if (!ok) break;
      if (n == 0) continue;
      const int qs = qn % QS;
      ptx::mbar_wait(&bars->q_full[qs], (qn / QS) & 1);
      ++qn;
      const uint32_t qa = aQ + qs * L::Q_BYTES;
      for (int j = 0; j < n; ++j, ++gs, ++gk) {
        const int b = gs % NS;
        if (gs >= (uint32_t)NS) ptx::mbar_wait(&bars->s_free[b], ((gs / NS) - 1) & 1);
        const int sl = gk % KS;
        ptx::mbar_wait(&bars->k_full[sl], (gk / KS) & 1);
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
          const uint32_t kb = aK + sl * L::TILE_BYTES;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk >> 2) * L::CHUNK + (kk & 3) * 32;
            ptx::mma_ss(tmem + b * 128, tc::make_sdesc(qa + off, 16, 1024),
                        tc::make_sdesc(kb + off, 16, 1024), IDESC_S, kk > 0 ? 1u : 0u);
          }
          ptx::mma_commit(&bars->k_empty[sl]);
          ptx::mma_commit(&bars->s_full[b]);
          if (j + 1 == n) ptx::mma_commit(&bars->q_empty[qs]);
        }
        __syncwarp();
      }
    }
  } else if (warp == 2) {
    // ============================ PV issuer ============================
    constexpr uint32_t IDESC_O = tc::make_idesc(BM, D, 1, tc::Elem<E>::kBf16);
    const uint32_t aV = ptx::smem_u32(sV);
    uint32_t gv = 0, gs = 0, items = 0;
    for (uint32_t it = 0;; ++it) {
      int h, qb, n;
      bool vis;
      const bool ok = next_item(it, h, qb, vis, n);
      if (lane == 0) ptx::mbar_arrive(&bars->sched_empty[it % SCHED]);
      if (!ok) break;
      // O still holds the previous item until its epilogue has read it
      if (items > 0) ptx::mbar_wait(&bars->o_empty, (items - 1) & 1);
      ++items;
      if (n == 0) {  // cannot come from build_block_mask; keep the epilogue in step
        if (ptx::elect_one()) ptx::mma_commit(&bars->o_full);
        __syncwarp();
        continue;
      }
      for (int j = 0; j < n; ++j, ++gs, ++gv) {
        const int b = gs % NS;
        ptx::mbar_wait(&bars->p_full[b], (gs / NS) & 1);
        const int sl = gv % VS;
        ptx::mbar_wait(&bars->v_full[sl], (gv / VS) & 1);
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
          const uint32_t vb = aV + sl * L::TILE_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            ptx::mma_ts(tmem + O_COL, tmem + b * 128 + kk * 8,
                        tc::make_sdesc(vb + kk * 16 * 128, L::CHUNK, 1024),
                        IDESC_O, (j > 0 || kk > 0) ? 1u : 0u);
          ptx::mma_commit(&bars->v_empty[sl]);
          ptx::mma_commit(&bars->s_free[b]);
          ptx::mma_commit(&bars->o_done);
          if (j + 1 == n) ptx::mma_commit(&bars->o_full);
        }
        __syncwarp();
      }
    }
  } else {
    // ============================ softmax / correction / epilogue ============================
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t t_row = tmem + ((uint32_t)(quarter * 32) << 16);
    uint32_t g = 0;
    for (uint32_t it = 0;; ++it) {
      int h, qb, n;
      bool vis;
      const bool ok = next_item(it, h, qb, vis, n);
      ptx::named_bar_sync(1, 128);
      if (threadIdx.x == 96) ptx::mbar_arrive(&bars->sched_empty[it % SCHED]);
      if (!ok) break;
      tc::KvList kl(vis ? kv_idx + ((int64_t)h * s.M_v + qb) * s.M_total : nullptr, n, lane);
      float m_run = -INFINITY, l_run = 0.f;
      for (int j = 0; j < n; ++j, ++g) {
        const int bb = g % NS;
        const uint32_t scol = t_row + bb * 128;
        const int blk = kl.block(j);
        const int kvalid = block_valid(blk, BK, s.M_v, s.n_valid, s.n_cond);
        const float bias = (vis && blk >= s.M_v) ? beta_log2 : 0.f;
        ptx::mbar_wait(&bars->s_full[bb], (g / NS) & 1);
        ptx::tc_fence_after();
        uint32_t sr[128];
#pragma unroll
        for (int c = 0; c < 4; ++c)
          ptx::tmem_ld32(scol + 32 * c, *reinterpret_cast<uint32_t(*)[32]>(&sr[32 * c]));
        ptx::tmem_wait_ld();
        if (dbg & 2) {  // timing experiment: no softmax work
          l_run = 1.f;
          ptx::tc_fence_before();
          ptx::mbar_arrive(&bars->p_full[bb]);
          continue;
        }
        if (kvalid < BK) {  // padding keys of a partial block -> -inf (attention.py:193)
#pragma unroll
          for (int e = 0; e < 128; ++e)
            if (e >= kvalid) sr[e] = __float_as_uint(-INFINITY);
        }
        float mx8[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) mx8[e] = __uint_as_float(sr[e]);
#pragma unroll
        for (int e = 8; e < 120; e += 16)
#pragma unroll
          for (int q = 0; q < 8; ++q)
            mx8[q] = tc::fmax3(mx8[q], __uint_as_float(sr[e + q]), __uint_as_float(sr[e + 8 + q]));
#pragma unroll
        for (int q = 0; q < 8; ++q) mx8[q] = fmaxf(mx8[q], __uint_as_float(sr[120 + q]));
        const float mraw = tc::fmax3(tc::fmax3(mx8[0], mx8[1], mx8[2]),
                                     tc::fmax3(mx8[3], mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]));
        const float m_blk = (mraw == -INFINITY) ? -INFINITY : fmaf(mraw, scale_log2, bias);
        const float m_new = fmaxf(m_run, m_blk);
        const bool first = (j == 0);
        const bool need = !first && (m_new > m_run + RESCALE_THRESHOLD);
        const float m_use = (first || need) ? m_new : m_run;
        const float alpha = need ? ptx::ex2(m_run - m_new) : 1.f;
        if (__any_sync(0xffffffffu, need)) {
          // O is final only once PV(j-1) retired: o_done completes once per PV
          ptx::mbar_wait(&bars->o_done, (g - 1) & 1);
          ptx::tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < D / 32; ++c) {
            uint32_t ov[32];
            ptx::tmem_ld32(t_row + O_COL + c * 32, ov);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * alpha);
            ptx::tmem_st32(t_row + O_COL + c * 32, ov);
          }
        }
        const float c0 = bias - m_use;
        const uint64_t sc2 = tc::f2_pack(scale_log2, scale_log2), c02 = tc::f2_pack(c0, c0);
        uint64_t acc2[4] = {0, 0, 0, 0};
#pragma unroll
        for (int c = 0; c < 2; ++c) {  // 64 keys -> 32 packed columns per store
          uint32_t pk[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const int k = 64 * c + 2 * e;
            const uint64_t x = tc::ffma2(
                tc::f2_pack(__uint_as_float(sr[k]), __uint_as_float(sr[k + 1])), sc2, c02);
            const float p0 = ptx::ex2(tc::f2_lo(x)), p1 = ptx::ex2(tc::f2_hi(x));
            acc2[e & 3] = tc::fadd2(acc2[e & 3], tc::f2_pack(p0, p1));
            pk[e] = tc::Elem<E>::pack(p0, p1);
          }
          ptx::tmem_st32(scol + 32 * c, pk);
        }
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&bars->p_full[bb]);
        const uint64_t sum2 = tc::fadd2(tc::fadd2(acc2[0], acc2[1]), tc::fadd2(acc2[2], acc2[3]));
        l_run = l_run * alpha + (tc::f2_lo(sum2) + tc::f2_hi(sum2));
        m_run = m_use;
      }
      // ---- epilogue: O / l -> row, padding rows zero (attention.py:203-206)
      ptx::mbar_wait(&bars->o_full, it & 1);
      ptx::tc_fence_after();
      const int qvalid = block_valid(qb, BM, s.M_v, s.n_valid, s.n_cond);
      const float inv_l = (row < qvalid && n > 0) ? 1.f / l_run : 0.f;
      E* orow = o + (int64_t)h * s.sh + ((int64_t)qb * BM + row) * s.sn;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        uint32_t ov[32];
        ptx::tmem_ld32(t_row + O_COL + c * 32, ov);
        ptx::tmem_wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e)
          pk[e] = n > 0 ? tc::Elem<E>::pack(__uint_as_float(ov[2 * e]) * inv_l,
                                            __uint_as_float(ov[2 * e + 1]) * inv_l)
                        : 0u;
        int4* dst = reinterpret_cast<int4*>(orow + c * 32);
#pragma unroll
        for (int e = 0; e < 4; ++e)
          __stcs(dst + e, make_int4((int)pk[4 * e], (int)pk[4 * e + 1], (int)pk[4 * e + 2],
                                    (int)pk[4 * e + 3]));
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&bars->o_empty);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<TMEM_COLS>(tmem);
  }
}

}  // namespace tc5





// ---------------------------------------------------------------- host helpers
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

// (d, N_pad, H) bf16 view with box (64, 128, 1), 128-byte swizzle
static int make_tmap(CUtensorMap* tm, const void* base, int d, int64_t n_pad, int H, int64_t sh,
                     int64_t sn, int box_rows, bool f16 = false) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return set_error(TCB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)n_pad, (cuuint64_t)H};
  cuuint64_t strides[2] = {(cuuint64_t)sn * 2, (cuuint64_t)sh * 2};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(tm, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                   const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(TCB_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return TCB_OK;
}

static int validate(const void* q, const void* k, const void* v, void* o, int dtype,
                    const int32_t* kv_idx, const int32_t* kv_cnt, const CarveShape& s) {
  TCB_CHECK_ARG(q && k && v && o, TCB_ESHAPE, "null q/k/v/o");
  TCB_CHECK_ARG(dtype == TCB_F32 || dtype == TCB_BF16 || dtype == TCB_F16, TCB_EDOMAIN,
                "unsupported dtype %d", dtype);
  TCB_CHECK_ARG(s.H >= 1 && s.d >= 1 && s.m >= 1 && s.M_v >= 0 && s.M_total >= s.M_v &&
                    s.M_total >= 1,
                TCB_ESHAPE, "bad carve shape");
  TCB_CHECK_ARG(s.M_v == 0 || (kv_idx && kv_cnt), TCB_ESHAPE, "null kv list");
  TCB_CHECK_ARG((int64_t)s.H * s.M_total < (int64_t)1 << 31, TCB_ESIZE, "too many work items");
  return TCB_OK;
}

}  // namespace tcb

using namespace tcb;

template <typename T, int MT, int DT>
static int launch_f32t(const void* q, const void* k, const void* v, void* o, const CarveShape& s,
                       const int32_t* kv_idx, const int32_t* kv_cnt, float beta, cudaStream_t st) {
  constexpr int M = 16 * MT, D = 16 * DT;
  size_t smem = (size_t)3 * M * (D + 1) * sizeof(float);
  if (M * (M + 1) > M * (D + 1)) smem += (size_t)M * (M + 1) * sizeof(float);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_carve_f32t<T, MT, DT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return set_error(TCB_ECUDA, "f32t smem: %s", cudaGetErrorString(e));
    attr = true;
  }
  const float scale = (float)(1.0 / sqrt((double)s.d));
  k_carve_f32t<T, MT, DT><<<(unsigned)((int64_t)s.H * s.M_total), 256, smem, st>>>(
      (const T*)q, (const T*)k, (const T*)v, (T*)o, s, kv_idx, kv_cnt, beta, scale);
  return check_launch("k_carve_f32t");
}

template <typename T>
static int try_f32t(const void* q, const void* k, const void* v, void* o, const CarveShape& s,
                    const int32_t* kv_idx, const int32_t* kv_cnt, float beta, cudaStream_t st) {
  const int key = (s.m << 16) | s.d;
  switch (key) {
    case (128 << 16) | 128: return launch_f32t<T, 8, 8>(q, k, v, o, s, kv_idx, kv_cnt, beta, st);
    case (128 << 16) | 64: return launch_f32t<T, 8, 4>(q, k, v, o, s, kv_idx, kv_cnt, beta, st);
    case (64 << 16) | 128: return launch_f32t<T, 4, 8>(q, k, v, o, s, kv_idx, kv_cnt, beta, st);
    case (64 << 16) | 64: return launch_f32t<T, 4, 4>(q, k, v, o, s, kv_idx, kv_cnt, beta, st);
    case (64 << 16) | 32: return launch_f32t<T, 4, 2>(q, k, v, o, s, kv_idx, kv_cnt, beta, st);
    case (32 << 16) | 64: return launch_f32t<T, 2, 4>(q, k, v, o, s, kv_idx, kv_cnt, beta, st);
    case (32 << 16) | 32: return launch_f32t<T, 2, 2>(q, k, v, o, s, kv_idx, kv_cnt, beta, st);
    case (128 << 16) | 32: return launch_f32t<T, 8, 2>(q, k, v, o, s, kv_idx, kv_cnt, beta, st);
    case (128 << 16) | 16: return launch_f32t<T, 8, 1>(q, k, v, o, s, kv_idx, kv_cnt, beta, st);
    case (64 << 16) | 16: return launch_f32t<T, 4, 1>(q, k, v, o, s, kv_idx, kv_cnt, beta, st);
    case (16 << 16) | 16: return launch_f32t<T, 1, 1>(q, k, v, o, s, kv_idx, kv_cnt, beta, st);
    default: return -1;  // not tiled: the per-row kernel takes it
  }
}

template <typename T>
static int launch_simt_t(const void* q, const void* k, const void* v, void* o, const CarveShape& s,
                         const int32_t* kv_idx, const int32_t* kv_cnt, float beta, cudaStream_t st) {
  {  // tiled fp32-math kernel for the common block / head sizes
    const int rc = try_f32t<T>(q, k, v, o, s, kv_idx, kv_cnt, beta, st);
    if (rc != -1) return rc;
  }
  TCB_CHECK_ARG(s.d <= 32 * SIMT_MAXC, TCB_ESIZE, "SIMT carve supports d <= %d", 32 * SIMT_MAXC);
  const size_t smem = (size_t)4 * (s.m + s.d) * sizeof(float);
  const float scale = (float)(1.0 / sqrt((double)s.d));
  const unsigned grid = (unsigned)((int64_t)s.H * s.M_total);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_carve_simt<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return set_error(TCB_ECUDA, "simt smem: %s", cudaGetErrorString(e));
  }
  k_carve_simt<T><<<grid, 128, smem, st>>>((const T*)q, (const T*)k, (const T*)v, (T*)o, s, kv_idx,
                                           kv_cnt, beta, scale);
  return check_launch("k_carve_simt");
}

static int launch_simt(const void* q, const void* k, const void* v, void* o, int dtype,
                       const CarveShape& s, const int32_t* kv_idx, const int32_t* kv_cnt,
                       float beta, cudaStream_t st) {
  if (dtype == TCB_F32) return launch_simt_t<float>(q, k, v, o, s, kv_idx, kv_cnt, beta, st);
  if (dtype == TCB_BF16) return launch_simt_t<__nv_bfloat16>(q, k, v, o, s, kv_idx, kv_cnt, beta, st);
  return launch_simt_t<__half>(q, k, v, o, s, kv_idx, kv_cnt, beta, st);
}

// TCB_CARVE_DEBUG bit 0: stream no K/V after the first ring fill; bit 1: skip the softmax
// (wrong results; only to measure the pipeline ceilings)
static int dbg_flags() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TCB_CARVE_DEBUG");
    v = e ? atoi(e) : 0;
  }
  return v;
}

template <int D, int EMU, typename E = __nv_bfloat16>
static int launch_tc(const void* q, const void* k, const void* v, void* o, const CarveShape& s,
                     const int32_t* kv_idx, const int32_t* kv_cnt, float beta, int32_t* work,
                     cudaStream_t st) {
  CUtensorMap tq, tk, tv;
  const int64_t n_pad = (int64_t)s.M_total * s.m;
  int rc;
  if ((rc = make_tmap(&tq, q, D, n_pad, s.H, s.sh, s.sn, tc::BM, !tc::Elem<E>::kBf16))) return rc;
  if ((rc = make_tmap(&tk, k, D, n_pad, s.H, s.sh, s.sn, tc::HN, !tc::Elem<E>::kBf16))) return rc;
  if ((rc = make_tmap(&tv, v, D, n_pad, s.H, s.sh, s.sn, tc::HN, !tc::Elem<E>::kBf16))) return rc;
  const int smem = tc::Smem<D>::BYTES;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(tc::k_carve_tc<D, EMU, E>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return set_error(TCB_ECUDA, "carve smem attr: %s", cudaGetErrorString(e));
    attr_set = true;
  }
  cudaError_t e = cudaMemsetAsync(work, 0, sizeof(int32_t), st);
  if (e != cudaSuccess) return set_error(TCB_ECUDA, "memset counter: %s", cudaGetErrorString(e));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int total = s.H * s.M_total;
  int grid = 2 * sms;
  if (grid > total) grid = total;
  const float LOG2E = 1.4426950408889634f;
  const float scale_log2 = (float)(1.0 / sqrt((double)s.d)) * LOG2E;
  tc::k_carve_tc<D, EMU, E><<<grid, tc::NUM_THREADS, smem, st>>>(tq, tk, tv, (E*)o, s, kv_idx,
                                                         kv_cnt, work, total, scale_log2,
                                                         beta * LOG2E, dbg_flags());
  return check_launch("k_carve_tc");
}




template <int D, int NT, typename E = __nv_bfloat16>
static int launch_tc2(const void* q, const void* k, const void* v, void* o, const CarveShape& s,
                      const int32_t* kv_idx, const int32_t* kv_cnt, float beta, int32_t* work,
                      cudaStream_t st) {
  CUtensorMap tq, tk, tv;
  const int64_t n_pad = (int64_t)s.M_total * s.m;
  constexpr bool f16 = !tc::Elem<E>::kBf16;
  int rc;
  if ((rc = make_tmap(&tq, q, D, n_pad, s.H, s.sh, s.sn, tc::BM, f16))) return rc;
  if ((rc = make_tmap(&tk, k, D, n_pad, s.H, s.sh, s.sn, tc::BK, f16))) return rc;
  if ((rc = make_tmap(&tv, v, D, n_pad, s.H, s.sh, s.sn, tc::BK, f16))) return rc;
  const int smem = tc2::Smem<D, NT>::BYTES;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(tc2::k_carve_tc2<D, NT, E>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return set_error(TCB_ECUDA, "carve smem attr: %s", cudaGetErrorString(e));
    attr_set = true;
  }
  cudaError_t e = cudaMemsetAsync(work, 0, sizeof(int32_t), st);
  if (e != cudaSuccess) return set_error(TCB_ECUDA, "memset counter: %s", cudaGetErrorString(e));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int total = s.H * s.M_total;
  int grid = (3 - NT) * sms;  // NT = 1: two CTAs per SM
  if (grid > (total + NT - 1) / NT) grid = (total + NT - 1) / NT;
  const float LOG2E = 1.4426950408889634f;
  const float scale_log2 = (float)(1.0 / sqrt((double)s.d)) * LOG2E;
  tc2::k_carve_tc2<D, NT, E><<<grid, tc2::Cfg<NT>::NUM_THREADS, smem, st>>>(tq, tk, tv, (E*)o, s, kv_idx, kv_cnt,
                                                              work, total, scale_log2, beta * LOG2E,
                                                              dbg_flags());
  return check_launch("k_carve_tc2");
}

template <int D, typename E = __nv_bfloat16>
static int launch_tc3(const void* q, const void* k, const void* v, void* o, const CarveShape& s,
                      const int32_t* kv_idx, const int32_t* kv_cnt, float beta, int32_t* work,
                      cudaStream_t st) {
  CUtensorMap tq, tk, tv;
  const int64_t n_pad = (int64_t)s.M_total * s.m;
  constexpr bool f16 = !tc::Elem<E>::kBf16;
  int rc;
  if ((rc = make_tmap(&tq, q, D, n_pad, s.H, s.sh, s.sn, tc::BM, f16))) return rc;
  if ((rc = make_tmap(&tk, k, D, n_pad, s.H, s.sh, s.sn, tc::BK, f16))) return rc;
  if ((rc = make_tmap(&tv, v, D, n_pad, s.H, s.sh, s.sn, tc::BK, f16))) return rc;
  const int smem = tc3::Smem<D>::BYTES;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(tc3::k_carve_tc3<D, E>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return set_error(TCB_ECUDA, "carve smem attr: %s", cudaGetErrorString(e));
    attr_set = true;
  }
  cudaError_t e = cudaMemsetAsync(work, 0, sizeof(int32_t), st);
  if (e != cudaSuccess) return set_error(TCB_ECUDA, "memset counter: %s", cudaGetErrorString(e));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int total = s.H * s.M_total;
  int grid = 2 * sms;
  if (grid > total) grid = total;
  const float LOG2E = 1.4426950408889634f;
  const float scale_log2 = (float)(1.0 / sqrt((double)s.d)) * LOG2E;
  tc3::k_carve_tc3<D, E><<<grid, tc3::NUM_THREADS, smem, st>>>(tq, tk, tv, (E*)o, s, kv_idx, kv_cnt,
                                                              work, total, scale_log2, beta * LOG2E,
                                                              dbg_flags());
  return check_launch("k_carve_tc3");
}

template <int D, typename E = __nv_bfloat16>
static int launch_tc4(const void* q, const void* k, const void* v, void* o, const CarveShape& s,
                      const int32_t* kv_idx, const int32_t* kv_cnt, float beta, int32_t* work,
                      cudaStream_t st) {
  CUtensorMap tq, tk, tv;
  const int64_t n_pad = (int64_t)s.M_total * s.m;
  constexpr bool f16 = !tc::Elem<E>::kBf16;
  int rc;
  if ((rc = make_tmap(&tq, q, D, n_pad, s.H, s.sh, s.sn, tc::BM, f16))) return rc;
  if ((rc = make_tmap(&tk, k, D, n_pad, s.H, s.sh, s.sn, tc::BK, f16))) return rc;
  if ((rc = make_tmap(&tv, v, D, n_pad, s.H, s.sh, s.sn, tc::BK, f16))) return rc;
  const int smem = tc4::Smem<D>::BYTES;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(tc4::k_carve_tc4<D, E>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return set_error(TCB_ECUDA, "carve smem attr: %s", cudaGetErrorString(e));
    attr_set = true;
  }
  cudaError_t e = cudaMemsetAsync(work, 0, sizeof(int32_t), st);
  if (e != cudaSuccess) return set_error(TCB_ECUDA, "memset counter: %s", cudaGetErrorString(e));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int total = s.H * s.M_total;
  int grid = sms;
  if (grid > (total + 1) / 2) grid = (total + 1) / 2;
  const float LOG2E = 1.4426950408889634f;
  const float scale_log2 = (float)(1.0 / sqrt((double)s.d)) * LOG2E;
  tc4::k_carve_tc4<D, E><<<grid, tc4::NUM_THREADS, smem, st>>>(tq, tk, tv, (E*)o, s, kv_idx, kv_cnt,
                                                              work, total, scale_log2, beta * LOG2E,
                                                              dbg_flags());
  return check_launch("k_carve_tc4");
}

template <int D, typename E = __nv_bfloat16>
static int launch_tc5(const void* q, const void* k, const void* v, void* o, const CarveShape& s,
                      const int32_t* kv_idx, const int32_t* kv_cnt, float beta, int32_t* work,
                      cudaStream_t st) {
  CUtensorMap tq, tk, tv;
  const int64_t n_pad = (int64_t)s.M_total * s.m;
  constexpr bool f16 = !tc::Elem<E>::kBf16;
  int rc;
  if ((rc = make_tmap(&tq, q, D, n_pad, s.H, s.sh, s.sn, tc::BM, f16))) return rc;
  if ((rc = make_tmap(&tk, k, D, n_pad, s.H, s.sh, s.sn, tc::BK, f16))) return rc;
  if ((rc = make_tmap(&tv, v, D, n_pad, s.H, s.sh, s.sn, tc::BK, f16))) return rc;
  const int smem = tc5::Smem<D>::BYTES;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(tc5::k_carve_tc5<D, E>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return set_error(TCB_ECUDA, "carve smem attr: %s", cudaGetErrorString(e));
    attr_set = true;
  }
  cudaError_t e = cudaMemsetAsync(work, 0, sizeof(int32_t), st);
  if (e != cudaSuccess) return set_error(TCB_ECUDA, "memset counter: %s", cudaGetErrorString(e));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int total = s.H * s.M_total;
  int grid = sms;
  if (grid > total) grid = total;
  const float LOG2E = 1.4426950408889634f;
  const float scale_log2 = (float)(1.0 / sqrt((double)s.d)) * LOG2E;
  tc5::k_carve_tc5<D, E><<<grid, tc5::NUM_THREADS, smem, st>>>(tq, tk, tv, (E*)o, s, kv_idx, kv_cnt,
                                                              work, total, scale_log2, beta * LOG2E,
                                                              dbg_flags());
  return check_launch("k_carve_tc5");
}

extern "C" int tcb_carve_fwd_simt(const void* q, const void* k, const void* v, void* o, int dtype,
                                  int64_t stride_h, int64_t stride_n, const int32_t* kv_idx,
                                  const int32_t* kv_cnt, int H, int d, int m, int M_v, int M_total,
                                  int64_t n_valid, int64_t n_cond, float beta, void* stream) {
  CarveShape s{H, d, m, M_v, M_total, n_valid, n_cond, stride_h, stride_n};
  int rc = validate(q, k, v, o, dtype, kv_idx, kv_cnt, s);
  if (rc) return rc;
  return launch_simt(q, k, v, o, dtype, s, kv_idx, kv_cnt, beta, as_stream(stream));
}

extern "C" int tcb_carve_fwd(const void* q, const void* k, const void* v, void* o, int dtype,
                             int64_t stride_h, int64_t stride_n, const int32_t* kv_idx,
                             const int32_t* kv_cnt, int H, int d, int m, int M_v, int M_total,
                             int64_t n_valid, int64_t n_cond, float beta, int32_t* work,
                             void* stream) {
  CarveShape s{H, d, m, M_v, M_total, n_valid, n_cond, stride_h, stride_n};
  int rc = validate(q, k, v, o, dtype, kv_idx, kv_cnt, s);
  if (rc) return rc;
  const bool aligned = ((uintptr_t)q % 16 == 0) && ((uintptr_t)k % 16 == 0) &&
                       ((uintptr_t)v % 16 == 0) && ((uintptr_t)o % 16 == 0) &&
                       (stride_n * 2) % 16 == 0 && (stride_h * 2) % 16 == 0;
  const bool tc_ok = (dtype == TCB_BF16 || dtype == TCB_F16) && m == 128 && (d == 128 || d == 64) &&
                     aligned && work && M_v > 0;
  if (!tc_ok) return launch_simt(q, k, v, o, dtype, s, kv_idx, kv_cnt, beta, as_stream(stream));
  // pairs (of 8) whose exp2 runs on the FMA pipe instead of MUFU; TCB_CARVE_EMU overrides
  static int emu = -1;
  if (emu < 0) {
    const char* env = getenv("TCB_CARVE_EMU");
    emu = env ? atoi(env) : 0;
    if (emu != 0 && emu != 2 && emu != 3 && emu != 4) emu = 0;
  }
  cudaStream_t st = as_stream(stream);
  static int v2 = -1;
  if (v2 < 0) {
    const char* env = getenv("TCB_CARVE_V2");
    v2 = env ? atoi(env) : 0;
  }
  if (v2 == 1) {
    if (dtype == TCB_F16)
      return d == 128 ? launch_tc2<128, 1, __half>(q, k, v, o, s, kv_idx, kv_cnt, beta, work, st)
                      : launch_tc2<64, 1, __half>(q, k, v, o, s, kv_idx, kv_cnt, beta, work, st);
    return d == 128 ? launch_tc2<128, 1>(q, k, v, o, s, kv_idx, kv_cnt, beta, work, st)
                    : launch_tc2<64, 1>(q, k, v, o, s, kv_idx, kv_cnt, beta, work, st);
  }
  if (v2 == 3) {
    if (dtype == TCB_F16)
      return d == 128 ? launch_tc3<128, __half>(q, k, v, o, s, kv_idx, kv_cnt, beta, work, st)
                      : launch_tc3<64, __half>(q, k, v, o, s, kv_idx, kv_cnt, beta, work, st);
    return d == 128 ? launch_tc3<128>(q, k, v, o, s, kv_idx, kv_cnt, beta, work, st)
                    : launch_tc3<64>(q, k, v, o, s, kv_idx, kv_cnt, beta, work, st);
  }
  if (v2 == 4) {
    if (dtype == TCB_F16)
      return d == 128 ? launch_tc4<128, __half>(q, k, v, o, s, kv_idx, kv_cnt, beta, work, st)
                      : launch_tc4<64, __half>(q, k, v, o, s, kv_idx, kv_cnt, beta, work, st);
    return d == 128 ? launch_tc4<128>(q, k, v, o, s, kv_idx, kv_cnt, beta, work, st)
                    : launch_tc4<64>(q, k, v, o, s, kv_idx, kv_cnt, beta, work, st);
  }
  if (v2 == 5) {
    if (dtype == TCB_F16)
      return d == 128 ? launch_tc5<128, __half>(q, k, v, o, s, kv_idx, kv_cnt, beta, work, st)
                      : launch_tc5<64, __half>(q, k, v, o, s, kv_idx, kv_cnt, beta, work, st);
    return d == 128 ? launch_tc5<128>(q, k, v, o, s, kv_idx, kv_cnt, beta, work, st)
                    : launch_tc5<64>(q, k, v, o, s, kv_idx, kv_cnt, beta, work, st);
  }
  if (v2 == 2) {
    return d == 128 ? launch_tc2<128, 2>(q, k, v, o, s, kv_idx, kv_cnt, beta, work, st)
                    : launch_tc2<64, 2>(q, k, v, o, s, kv_idx, kv_cnt, beta, work, st);
  }
  if (dtype == TCB_F16)  // fp16 operands and P (kind::f16 with f16 inputs), f32 accumulation
    return d == 128 ? launch_tc<128, 0, __half>(q, k, v, o, s, kv_idx, kv_cnt, beta, work, st)
                    : launch_tc<64, 0, __half>(q, k, v, o, s, kv_idx, kv_cnt, beta, work, st);
  if (d == 128) {
    switch (emu) {
      case 3: return launch_tc<128, 3>(q, k, v, o, s, kv_idx, kv_cnt, beta, work, st);
      case 4: return launch_tc<128, 4>(q, k, v, o, s, kv_idx, kv_cnt, beta, work, st);
      case 2: return launch_tc<128, 2>(q, k, v, o, s, kv_idx, kv_cnt, beta, work, st);
      default: return launch_tc<128, 0>(q, k, v, o, s, kv_idx, kv_cnt, beta, work, st);
    }
  }
  return launch_tc<64, 0>(q, k, v, o, s, kv_idx, kv_cnt, beta, work, st);
}

// Debug only (not part of include/tokencarve_b200.h): copy out and clear the CTA-0 timeline
// (TRACE_EV x TRACE_STEPS clocks, 0 = not reached).
extern "C" int tcb_debug_trace_read(unsigned long long* host, int cap) {
  const int n = tcb::tc2::TRACE_EV * tcb::tc2::TRACE_STEPS;
  if (cap < n) return -1;
  cudaMemcpyFromSymbol(host, tcb::tc2::g_trace, sizeof(unsigned long long) * n);
  static unsigned long long zero[tcb::tc2::TRACE_EV * tcb::tc2::TRACE_STEPS];
  cudaMemcpyToSymbol(tcb::tc2::g_trace, zero, sizeof(zero));
  return n;
}
