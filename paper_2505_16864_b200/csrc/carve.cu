// K7/K8 block-sparse flash-attention forward (carve_attention, attention.py:162-243).
//
//  * k_carve_tc   -- bf16, m == 128, d in {64,128}: persistent warp-specialised
//                    tcgen05 kernel.  TMA loads Q/K/V tiles (128B swizzle) into smem
//                    under mbarriers, one thread issues tcgen05.mma for S = Q K^T
//                    into TMEM, four softmax warps read S with tcgen05.ld, do the
//                    online softmax in registers (exp2, lazy rescale), write P as
//                    bf16 back into TMEM over S, and the MMA thread issues
//                    O += P V with A read from TMEM.  Two CTAs per SM interleave so
//                    one CTA's softmax overlaps the other's MMAs.  Work items
//                    (head, q-block) come from a global atomic counter, condition
//                    q-blocks (full rows, ~10x longer) first, then vision q-blocks
//                    head-major so concurrently running items share a head's K/V
//                    in L2.
//  * k_carve_simt -- fp32 math for any (m, d, dtype): the parity path that mirrors
//                    the reference's per-block streaming softmax order.
#include "common.cuh"
#include "ptx.cuh"

#include <cuda.h>
#include <cuda_bf16.h>
#include <math.h>

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
template <typename T>
__device__ __forceinline__ T stf(float v);
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
// tcgen05 kernel
// =====================================================================================
namespace tc {

constexpr int BM = 128;          // query rows per tile (== m)
constexpr int BN = 128;          // key rows per kv block (== m)
constexpr int NUM_THREADS = 192;  // w0 TMA+scheduler, w1 MMA+TMEM owner, w2..w5 softmax
constexpr int TMEM_COLS = 256;   // S/P [0,128) + O [128, 128+D)
constexpr int S_COL = 0;
constexpr int P_COL = 0;         // bf16 P packed 2/col over the first 64 S columns
constexpr int O_COL = 128;
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 units: P <= 2^8 before a forced rescale

template <int D>
struct Smem {
  static constexpr int TILE_BYTES = BM * D * 2;  // one 128 x D bf16 tile
  static constexpr int CHUNKS = D / 64;          // 64-element (128 B) swizzle columns
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + TILE_BYTES;
  static constexpr int OFF_V = OFF_K + TILE_BYTES;
  static constexpr int OFF_BAR = OFF_V + TILE_BYTES;
  static constexpr int BYTES = OFF_BAR + 256 + 1024;  // + barriers + alignment slack
};

struct Bars {
  uint64_t q_full, q_empty, k_full, k_empty, v_full, v_empty, s_full, p_full, o_full;
  uint64_t sched_full[2], sched_empty[2];
  int sched_item[2];
  uint32_t tmem_base;
};

// instruction descriptor, kind::f16: bf16 x bf16 -> f32, K-major A, B major per arg
__host__ __device__ constexpr uint32_t make_idesc(int M, int N, int b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)b_mn_major << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// smem matrix descriptor, SWIZZLE_128B, sm_100 version bits
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}

template <int D>
__global__ void __launch_bounds__(NUM_THREADS, 2)
    k_carve_tc(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
               const __grid_constant__ CUtensorMap tm_v, __nv_bfloat16* __restrict__ o,
               CarveShape s, const int32_t* __restrict__ kv_idx,
               const int32_t* __restrict__ kv_cnt, int* __restrict__ counter, int total_items,
               float scale_log2, float beta_log2) {
  using L = Smem<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem + L::OFF_Q;
  uint8_t* sK = smem + L::OFF_K;
  uint8_t* sV = smem + L::OFF_V;
  Bars* bars = reinterpret_cast<Bars*>(smem + L::OFF_BAR);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    ptx::mbar_init(&bars->q_full, 1);
    ptx::mbar_init(&bars->q_empty, 1);
    ptx::mbar_init(&bars->k_full, 1);
    ptx::mbar_init(&bars->k_empty, 1);
    ptx::mbar_init(&bars->v_full, 1);
    ptx::mbar_init(&bars->v_empty, 1);
    ptx::mbar_init(&bars->s_full, 1);
    ptx::mbar_init(&bars->p_full, 128);
    ptx::mbar_init(&bars->o_full, 1);
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
    if (lane == 0) {
      const uint64_t pol_kv = ptx::policy_evict_last();
      const uint64_t pol_q = ptx::policy_evict_first();
      uint32_t it = 0, gk = 0, gv = 0;
      for (;; ++it) {
        const int slot = it & 1;
        ptx::mbar_wait(&bars->sched_empty[slot], ((it >> 1) & 1) ^ 1);
        int item = atomicAdd(counter, 1);
        if (item >= total_items) item = -1;
        bars->sched_item[slot] = item;
        ptx::mbar_arrive(&bars->sched_full[slot]);
        if (item < 0) break;
        int h, qb;
        decode_item(item, s, h, qb);
        const bool vis = qb < s.M_v;
        const int n = vis ? kv_cnt[(int64_t)h * s.M_v + qb] : s.M_total;
        const int32_t* list = vis ? kv_idx + ((int64_t)h * s.M_v + qb) * s.M_total : nullptr;
        ptx::mbar_wait(&bars->q_empty, (it & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&bars->q_full, L::TILE_BYTES);
#pragma unroll
        for (int c = 0; c < L::CHUNKS; ++c)
          ptx::tma_load_3d(sQ + c * BM * 128, &tm_q, &bars->q_full, c * 64, qb * BM, h, pol_q);
        for (int j = 0; j < n; ++j) {
          const int b = vis ? __ldg(list + j) : j;
          ptx::mbar_wait(&bars->k_empty, (gk & 1) ^ 1);
          ptx::mbar_arrive_expect_tx(&bars->k_full, L::TILE_BYTES);
#pragma unroll
          for (int c = 0; c < L::CHUNKS; ++c)
            ptx::tma_load_3d(sK + c * BN * 128, &tm_k, &bars->k_full, c * 64, b * BN, h, pol_kv);
          ++gk;
          ptx::mbar_wait(&bars->v_empty, (gv & 1) ^ 1);
          ptx::mbar_arrive_expect_tx(&bars->v_full, L::TILE_BYTES);
#pragma unroll
          for (int c = 0; c < L::CHUNKS; ++c)
            ptx::tma_load_3d(sV + c * BN * 128, &tm_v, &bars->v_full, c * 64, b * BN, h, pol_kv);
          ++gv;
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ============================ MMA issuer ============================
    if (lane == 0) {
      constexpr uint32_t IDESC_S = make_idesc(BM, BN, 0);  // Q (K-major) x K (K-major)
      constexpr uint32_t IDESC_O = make_idesc(BM, D, 1);   // P (TMEM)   x V (MN-major)
      const uint32_t aQ = ptx::smem_u32(sQ), aK = ptx::smem_u32(sK), aV = ptx::smem_u32(sV);
      uint32_t it = 0, g = 0;
      for (;; ++it) {
        const int slot = it & 1;
        ptx::mbar_wait(&bars->sched_full[slot], (it >> 1) & 1);
        const int item = bars->sched_item[slot];
        ptx::mbar_arrive(&bars->sched_empty[slot]);
        if (item < 0) break;
        int h, qb;
        decode_item(item, s, h, qb);
        const bool vis = qb < s.M_v;
        const int n = vis ? kv_cnt[(int64_t)h * s.M_v + qb] : s.M_total;
        ptx::mbar_wait(&bars->q_full, it & 1);
        for (int j = 0; j < n; ++j, ++g) {
          // ---- S = Q K^T  (K = D in steps of 16; 128B swizzle rows hold 64 elements)
          ptx::mbar_wait(&bars->k_full, g & 1);
          ptx::tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk >> 2) * (BM * 128) + (kk & 3) * 32;
            const uint64_t da = make_sdesc(aQ + off, 16, 1024);
            const uint64_t db = make_sdesc(aK + off, 16, 1024);
            ptx::mma_ss(tmem + S_COL, da, db, IDESC_S, kk > 0 ? 1u : 0u);
          }
          ptx::mma_commit(&bars->k_empty);
          ptx::mma_commit(&bars->s_full);
          if (j == n - 1) ptx::mma_commit(&bars->q_empty);
          // ---- O += P V   (K = kv rows in steps of 16 -> 2 KB of V per step)
          ptx::mbar_wait(&bars->p_full, g & 1);
          ptx::mbar_wait(&bars->v_full, g & 1);
          ptx::tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < BN / 16; ++kk) {
            const uint64_t dv = make_sdesc(aV + kk * 16 * 128, BN * 128, 1024);
            ptx::mma_ts(tmem + O_COL, tmem + P_COL + kk * 8, dv, IDESC_O,
                        (j > 0 || kk > 0) ? 1u : 0u);
          }
          ptx::mma_commit(&bars->v_empty);
        }
        if (n == 0) ptx::mma_commit(&bars->q_empty);
        ptx::mma_commit(&bars->o_full);
      }
    }
    __syncwarp();
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
      const int32_t* list = vis ? kv_idx + ((int64_t)h * s.M_v + qb) * s.M_total : nullptr;
      float m_run = -INFINITY, l_run = 0.f;
      for (int j = 0; j < n; ++j, ++g) {
        const int b = vis ? __ldg(list + j) : j;
        const int kvalid = block_valid(b, BN, s.M_v, s.n_valid, s.n_cond);
        const float bias = (vis && b >= s.M_v) ? beta_log2 : 0.f;
        ptx::mbar_wait(&bars->s_full, g & 1);
        ptx::tc_fence_after();
        uint32_t sr[4][32];
#pragma unroll
        for (int c = 0; c < 4; ++c) ptx::tmem_ld32(t_row + S_COL + c * 32, sr[c]);
        ptx::tmem_wait_ld();
        float mx = -INFINITY;
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            float t = fmaf(__uint_as_float(sr[c][e]), scale_log2, bias);
            if (c * 32 + e >= kvalid) t = -INFINITY;
            sr[c][e] = __float_as_uint(t);
            mx = fmaxf(mx, t);
          }
        const float m_new = fmaxf(m_run, mx);
        float m_use = m_run, alpha = 1.f;
        const bool need = (j == 0) ? false : (m_new > m_run + RESCALE_THRESHOLD);
        if (j == 0 || need) m_use = m_new;
        if (need) alpha = ptx::ex2(m_run - m_new);
        float psum = 0.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const float p0 = ptx::ex2(__uint_as_float(sr[c][2 * e]) - m_use);
            const float p1 = ptx::ex2(__uint_as_float(sr[c][2 * e + 1]) - m_use);
            psum += p0 + p1;
            pk[e] = ptx::pack_bf16(p0, p1);
          }
          // 16 packed columns per 32 scores; store as half of a x32 store pair
#pragma unroll
          for (int e = 0; e < 16; ++e) sr[c][e] = pk[e];
        }
        {
          uint32_t a0[32], a1[32];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            a0[e] = sr[0][e];
            a0[16 + e] = sr[1][e];
            a1[e] = sr[2][e];
            a1[16 + e] = sr[3][e];
          }
          ptx::tmem_st32(t_row + P_COL, a0);
          ptx::tmem_st32(t_row + P_COL + 32, a1);
        }
        l_run = l_run * alpha + psum;
        m_run = m_use;
        // lazy O correction: S_j complete => PV_{j-1} complete (in-order tensor pipe)
        if (__any_sync(0xffffffffu, need)) {
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
        ptx::mbar_arrive(&bars->p_full);
      }
      // ---- epilogue: O / l -> bf16 row, padding rows zero (attention.py:203-206)
      ptx::mbar_wait(&bars->o_full, it & 1);
      ptx::tc_fence_after();
      const int qvalid = block_valid(qb, BM, s.M_v, s.n_valid, s.n_cond);
      const float inv_l = (row < qvalid) ? 1.f / l_run : 0.f;
      __nv_bfloat16* orow = o + (int64_t)h * s.sh + ((int64_t)qb * BM + row) * s.sn;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        uint32_t ov[32];
        ptx::tmem_ld32(t_row + O_COL + c * 32, ov);
        ptx::tmem_wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e)
          pk[e] = ptx::pack_bf16(__uint_as_float(ov[2 * e]) * inv_l,
                                 __uint_as_float(ov[2 * e + 1]) * inv_l);
        int4* dst = reinterpret_cast<int4*>(orow + c * 32);
#pragma unroll
        for (int e = 0; e < 4; ++e)
          dst[e] = make_int4((int)pk[4 * e], (int)pk[4 * e + 1], (int)pk[4 * e + 2],
                             (int)pk[4 * e + 3]);
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
                     int64_t sn) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return set_error(TCB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)n_pad, (cuuint64_t)H};
  cuuint64_t strides[2] = {(cuuint64_t)sn * 2, (cuuint64_t)sh * 2};
  cuuint32_t box[3] = {64, 128, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(TCB_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return TCB_OK;
}

static int validate(const void* q, const void* k, const void* v, void* o, int dtype,
                    const int32_t* kv_idx, const int32_t* kv_cnt, const CarveShape& s) {
  TCB_CHECK_ARG(q && k && v && o, TCB_ESHAPE, "null q/k/v/o");
  TCB_CHECK_ARG(dtype == TCB_F32 || dtype == TCB_BF16, TCB_EDOMAIN, "unsupported dtype %d", dtype);
  TCB_CHECK_ARG(s.H >= 1 && s.d >= 1 && s.m >= 1 && s.M_v >= 0 && s.M_total >= s.M_v &&
                    s.M_total >= 1,
                TCB_ESHAPE, "bad carve shape");
  TCB_CHECK_ARG(s.M_v == 0 || (kv_idx && kv_cnt), TCB_ESHAPE, "null kv list");
  TCB_CHECK_ARG((int64_t)s.H * s.M_total < (int64_t)1 << 31, TCB_ESIZE, "too many work items");
  return TCB_OK;
}

}  // namespace tcb

using namespace tcb;

static int launch_simt(const void* q, const void* k, const void* v, void* o, int dtype,
                       const CarveShape& s, const int32_t* kv_idx, const int32_t* kv_cnt,
                       float beta, cudaStream_t st) {
  TCB_CHECK_ARG(s.d <= 32 * SIMT_MAXC, TCB_ESIZE, "SIMT carve supports d <= %d", 32 * SIMT_MAXC);
  const size_t smem = (size_t)4 * (s.m + s.d) * sizeof(float);
  const float scale = (float)(1.0 / sqrt((double)s.d));
  const unsigned grid = (unsigned)((int64_t)s.H * s.M_total);
  if (smem > 48 * 1024) {
    cudaError_t e;
    if (dtype == TCB_F32)
      e = cudaFuncSetAttribute(k_carve_simt<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem);
    else
      e = cudaFuncSetAttribute(k_carve_simt<__nv_bfloat16>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return set_error(TCB_ECUDA, "simt smem: %s", cudaGetErrorString(e));
  }
  if (dtype == TCB_F32)
    k_carve_simt<float><<<grid, 128, smem, st>>>((const float*)q, (const float*)k, (const float*)v,
                                                 (float*)o, s, kv_idx, kv_cnt, beta, scale);
  else
    k_carve_simt<__nv_bfloat16><<<grid, 128, smem, st>>>(
        (const __nv_bfloat16*)q, (const __nv_bfloat16*)k, (const __nv_bfloat16*)v,
        (__nv_bfloat16*)o, s, kv_idx, kv_cnt, beta, scale);
  return check_launch("k_carve_simt");
}

template <int D>
static int launch_tc(const void* q, const void* k, const void* v, void* o, const CarveShape& s,
                     const int32_t* kv_idx, const int32_t* kv_cnt, float beta, int32_t* work,
                     cudaStream_t st) {
  CUtensorMap tq, tk, tv;
  const int64_t n_pad = (int64_t)s.M_total * s.m;
  int rc;
  if ((rc = make_tmap(&tq, q, D, n_pad, s.H, s.sh, s.sn))) return rc;
  if ((rc = make_tmap(&tk, k, D, n_pad, s.H, s.sh, s.sn))) return rc;
  if ((rc = make_tmap(&tv, v, D, n_pad, s.H, s.sh, s.sn))) return rc;
  const int smem = tc::Smem<D>::BYTES;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(tc::k_carve_tc<D>,
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
  tc::k_carve_tc<D><<<grid, tc::NUM_THREADS, smem, st>>>(tq, tk, tv, (__nv_bfloat16*)o, s, kv_idx,
                                                         kv_cnt, work, total, scale_log2,
                                                         beta * LOG2E);
  return check_launch("k_carve_tc");
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
  const bool tc_ok = dtype == TCB_BF16 && m == 128 && (d == 128 || d == 64) && aligned && work &&
                     M_v > 0;
  if (!tc_ok) return launch_simt(q, k, v, o, dtype, s, kv_idx, kv_cnt, beta, as_stream(stream));
  if (d == 128) return launch_tc<128>(q, k, v, o, s, kv_idx, kv_cnt, beta, work, as_stream(stream));
  return launch_tc<64>(q, k, v, o, s, kv_idx, kv_cnt, beta, work, as_stream(stream));
}
