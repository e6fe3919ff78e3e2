// K7/K8 block-sparse flash-attention forward (carve_attention, attention.py:162-243).
//
//  * k_carve_tc   -- bf16 / fp16, m == 128, d in {64,128}: persistent warp-specialised
//                    tcgen05 kernel.  TMA loads Q/K/V tiles (128B swizzle) into smem
//                    under mbarriers, one elected lane of the MMA warp issues
//                    tcgen05.mma for S = Q K^T into TMEM (64-key half-steps, S
//                    double-buffered), four softmax warps read S with tcgen05.ld, do
//                    the online softmax in registers (exp2; max-free half-steps that
//                    take a block max only on a row's first half or when the p-sum says
//                    the running max moved), write P as 16-bit back into TMEM over S, and
//                    the MMA warp issues O += P V with A read from TMEM.  Two CTAs per SM
//                    interleave so one CTA's softmax overlaps the other's MMAs.  Work
//                    items (head, q-block) come from a global atomic counter, vision
//                    q-blocks head-major so concurrently running items share a head's
//                    K/V in L2; condition q-blocks (full rows, ~10x longer) run as kv-range
//                    chunks in their head's slot, merged by the last chunk, when the
//                    workspace allows (else all of them first, unsplit).
//                    has the measured bounds and the rejected variants.
//  * k_carve_f32t -- fp32 math on shared-memory tiles with register-blocked S / O for
//                    the common (m, d): fp32 inputs and shapes the tcgen05 kernel does
//                    not take; mirrors the reference's per-block streaming order (1e-5).
//  * k_carve_simt -- fp32 math, one warp per query row, any (m, d): the fallback.
#include <atomic>
#include <mutex>
#include "common.cuh"
#include "ptx.cuh"
#include "tc_common.cuh"

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <math.h>
#include <stdlib.h>

namespace tcb {

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
                                                    CarveShape s, const uint32_t* __restrict__ bits,
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
  const uint32_t* brow = vis ? bits + ((int64_t)h * s.M_v + qb) * s.W : nullptr;
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
    BitWalk bw(brow);
    for (int t = 0; t < nkv; ++t) {
      const int b = vis ? bw.get(t) : t;
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
                                                       CarveShape s, const uint32_t* __restrict__ bits,
                                                       const int32_t* __restrict__ kv_cnt, float beta,
                                                       float scale) {
  constexpr int M = 16 * MT, D = 16 * DT;
  // Q and K stay row-major, V is stored transposed and P row-major, so both inner loops read
  // their operands as float4 along the reduction axis (4 LDS.128 per 64 FMAs per thread);
  // the FMA order (c, then key) is the scalar kernel's, so results are unchanged.
  constexpr int QP = D + 4;   // row pitch (floats) of Q / K: 16-byte rows
  constexpr int VP = M + 4;   // row pitch of V^T
  constexpr int PP = M + 4;   // row pitch of P
  extern __shared__ __align__(16) float sm_f32t[];
  float* sQ = sm_f32t;
  float* sK = sQ + M * QP;
  float* sVt = sK + M * QP;
  float* sP = (M * PP <= M * QP) ? sK : sVt + D * VP;  // P reuses K's tile when it fits
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const int h = blockIdx.x / s.M_total;
  const int qb = blockIdx.x - h * s.M_total;
  const bool vis = qb < s.M_v;
  const int nkv = vis ? kv_cnt[(int64_t)h * s.M_v + qb] : s.M_total;
  BitWalk bw(vis ? bits + ((int64_t)h * s.M_v + qb) * s.W : nullptr);
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
    const int b = vis ? bw.get(t) : t;
    const int kvalid = block_valid(b, M, s.M_v, s.n_valid, s.n_cond);
    const bool add_beta = vis && beta != 0.f && b >= s.M_v;
    __syncthreads();  // previous block's P / V reads done
    for (int e = tid; e < M * D; e += 256) {
      const int r = e / D, c = e - r * D;
      const int64_t g = ((int64_t)b * M + r) * s.sn + c;
      sK[r * QP + c] = ldf(kh + g);
      sVt[c * VP + r] = ldf(vh + g);
    }
    __syncthreads();
    float sc[MT][MT];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < MT; ++j) sc[i][j] = 0.f;
#pragma unroll 2
    for (int c = 0; c < D; c += 4) {
      float4 a[MT], bk[MT];
#pragma unroll
      for (int i = 0; i < MT; ++i) a[i] = *reinterpret_cast<const float4*>(sQ + (ty + 16 * i) * QP + c);
#pragma unroll
      for (int j = 0; j < MT; ++j) bk[j] = *reinterpret_cast<const float4*>(sK + (tx + 16 * j) * QP + c);
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < MT; ++j) {
          float x = fmaf(a[i].x, bk[j].x, sc[i][j]);
          x = fmaf(a[i].y, bk[j].y, x);
          x = fmaf(a[i].z, bk[j].z, x);
          sc[i][j] = fmaf(a[i].w, bk[j].w, x);
        }
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
#pragma unroll 2
    for (int jk = 0; jk < M; jk += 4) {
      float4 pr[MT], vv[DT];
#pragma unroll
      for (int i = 0; i < MT; ++i) pr[i] = *reinterpret_cast<const float4*>(sP + (ty + 16 * i) * PP + jk);
#pragma unroll
      for (int j = 0; j < DT; ++j) vv[j] = *reinterpret_cast<const float4*>(sVt + (tx + 16 * j) * VP + jk);
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < DT; ++j) {
          float x = fmaf(pr[i].x, vv[j].x, acc[i][j]);
          x = fmaf(pr[i].y, vv[j].y, x);
          x = fmaf(pr[i].z, vv[j].z, x);
          acc[i][j] = fmaf(pr[i].w, vv[j].w, x);
        }
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
// max-free steps: a half-step whose p-sum stays <= 2^12 keeps the running max (P <= 2^12)
constexpr float RESCALE_SUM_LIMIT = 4096.0f;

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
  uint64_t q_full, q_empty, o_full;
  uint64_t p_full[2];  // by half-step parity: softmax(t+1) may finish before PV(t) is issued
  uint64_t s_full[2];
  uint64_t k_full[K_SLOTS], k_empty[K_SLOTS];
  uint64_t v_full[V_SLOTS], v_empty[V_SLOTS];
  uint64_t sched_full[2], sched_empty[2];
  int sched_item[2];
  int last;  // condition-row split: the chunk count this CTA's chunk observed
  uint32_t tmem_base;
};
static_assert(sizeof(Bars) <= 256, "barrier block must fit the reserved smem");

// Condition q-blocks attend all M_total kv blocks (~10x a vision row).  With a workspace,
// each is split into C chunks of `len` kv blocks that run as ordinary work items next to
// their head's vision rows (per-head item order: the head's K/V is read from DRAM about
// once instead of once by a condition-row sweep ahead of everything and again by the vision
// rows); each chunk leaves its unnormalised O, running max and sum in `part`, and the
// chunk that completes a row (per-row counter `cnt`) merges the C partials in chunk order.
// C == 1: no split, all condition rows first (longest-first order).
struct CondSplit {
  int C, len;
  float* part;  // [H*M_c*C][BM][D] O partials, then [H*M_c*C][BM][2] (m, l)
  int* cnt;     // [H*M_c] chunks finished per condition row
};

__device__ __forceinline__ void decode_tc(int item, const CarveShape& s, const CondSplit& cs, int& h,
                                          int& qb, int& c0, int& c1) {
  c0 = 0;
  c1 = s.M_total;
  if (cs.C <= 1) {
    decode_item(item, s, h, qb);
    return;
  }
  const int n_cc = (s.M_total - s.M_v) * cs.C;
  const int per = n_cc + s.M_v;
  h = item / per;
  const int r = item - h * per;
  if (r < n_cc) {
    const int ci = r / cs.C;
    qb = s.M_v + ci;
    c0 = (r - ci * cs.C) * cs.len;
    c1 = min(s.M_total, c0 + cs.len);
  } else {
    qb = r - n_cc;
  }
}

// Timeline stamps for tools/carve_trace1.py: compiled only into trace builds
// (TCB_NVCC_EXTRA=-DTCB_CARVE_TRACE python -m paper_2505_16864_b200._build), enabled at run
// time by TCB_CARVE_DEBUG bit 3; CTA 0 writes clock64() per (event, half-step).
#ifdef TCB_CARVE_TRACE
constexpr int TRACE_EV = 24, TRACE_STEPS = 8192;
__device__ unsigned long long g_trace[TRACE_EV][TRACE_STEPS];
#define TRACE(ev, step)                                                                 \
  do {                                                                                  \
    if ((dbg & 8) && blockIdx.x == 0 && (step) < (uint32_t)TRACE_STEPS)                 \
      g_trace[(ev)][(step)] = clock64();                                                \
  } while (0)
#else
#define TRACE(ev, step) \
  do {                  \
  } while (0)
#endif

template <int D, int EMU, typename E = __nv_bfloat16, int MAXFREE = 0>
__global__ void __launch_bounds__(NUM_THREADS, 2)
    k_carve_tc(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
               const __grid_constant__ CUtensorMap tm_v, E* __restrict__ o,
               CarveShape s, const uint32_t* __restrict__ bits,
               const int32_t* __restrict__ kv_cnt, int* __restrict__ counter, int total_items,
               float scale_log2, float beta_log2, int dbg, CondSplit cs) {
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
      int h, qb, c0, c1;
      decode_tc(item, s, cs, h, qb, c0, c1);
      const bool vis = qb < s.M_v;
      const int n = vis ? __ldg(kv_cnt + (int64_t)h * s.M_v + qb) : c1 - c0;
      const uint64_t pol_cond = cs.C > 1 ? pol_kv : pol_q;  // split rows share the head's K/V
      const uint32_t* brow = bits + ((int64_t)h * s.M_v + (vis ? qb : 0)) * s.W;
      // K runs one half-step ahead of V: one walk per stream (cond rows never walk)
      WarpKvList wk(vis ? brow : nullptr, s.W, lane), wv(vis ? brow : nullptr, s.W, lane);
      const int T = 2 * n;
      if (lane == 0) {
        ptx::mbar_wait(&bars->q_empty, (it & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&bars->q_full, L::Q_BYTES);
        ptx::tma_load_4d(sQ, &tm_q, &bars->q_full, 0, qb * BM, 0, h, pol_q);
      }
      auto load = [&](const CUtensorMap* tm, uint8_t* base, uint64_t* full, uint64_t* empty,
                      int slots, uint32_t& cnt, int t, WarpKvList& walk) {
        const int b = vis ? walk.block(t >> 1) : c0 + (t >> 1);
        if (lane == 0) {
          const int sl = cnt % slots;
          ptx::mbar_wait(&empty[sl], ((cnt / slots) & 1) ^ 1);
          if ((dbg & 1) && cnt >= (uint32_t)slots) {  // timing experiment: no operand traffic
            ptx::mbar_arrive(&full[sl]);
          } else {
            ptx::mbar_arrive_expect_tx(&full[sl], L::HALF_BYTES);
            ptx::tma_load_4d(base + sl * L::HALF_BYTES, tm, &full[sl], 0, b * BK + (t & 1) * HN, 0, h,
                             vis ? pol_kv : pol_cond);
          }
        }
        ++cnt;
      };
      // same order the MMA warp consumes: K0, K1, V0, K2, V1, ..., V(T-1); an empty row
      // (T == 0, only reachable through a hand-built mask) loads nothing, like the MMA warp
      if (T > 0) load(&tm_k, sK, bars->k_full, bars->k_empty, K_SLOTS, gk, 0, wk);
      for (int t = 0; t < T; ++t) {
        if (t + 1 < T) load(&tm_k, sK, bars->k_full, bars->k_empty, K_SLOTS, gk, t + 1, wk);
        load(&tm_v, sV, bars->v_full, bars->v_empty, V_SLOTS, gv, t, wv);
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
      if (lane == 0) TRACE(7, gs);
      ptx::mbar_wait(&bars->k_full[sl], (gk / K_SLOTS) & 1);
      if (lane == 0) TRACE(8, gs);
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
      if (lane == 0) TRACE(9, gs);
      ++gk;
      ++gs;
    };
    for (;; ++it) {
      const int slot = it & 1;
      ptx::mbar_wait(&bars->sched_full[slot], (it >> 1) & 1);
      const int item = bars->sched_item[slot];
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&bars->sched_empty[slot]);
      if (item < 0) break;
      int h, qb, c0, c1;
      decode_tc(item, s, cs, h, qb, c0, c1);
      const bool vis = qb < s.M_v;
      const int n = vis ? kv_cnt[(int64_t)h * s.M_v + qb] : c1 - c0;
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
      issue_s();
      for (int t = 0; t < T; ++t) {
        if (t + 1 < T) {
          issue_s();
          if (t + 2 == T) {
            if (ptx::elect_one()) ptx::mma_commit(&bars->q_empty);
            __syncwarp();
          }
        }
        // ---- O += P(t) V(t): A = P from TMEM (32 packed columns), K = 64 keys
        if (lane == 0) TRACE(1, gp);
        ptx::mbar_wait(&bars->p_full[gp & 1], (gp >> 1) & 1);
        if (lane == 0) TRACE(3, gp);
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
        }
        __syncwarp();
        if (lane == 0) TRACE(5, gp);
        ++gv;
        ++gp;
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
      int h, qb, c0, c1;
      decode_tc(item, s, cs, h, qb, c0, c1);
      const bool vis = qb < s.M_v;
      const int n = vis ? kv_cnt[(int64_t)h * s.M_v + qb] : c1 - c0;
      // the block index itself is not needed here: only where condition keys start and
      // which entries can be partial blocks (RowShape); condition q-blocks visit c0..c1-1
      const RowShape rs = vis ? RowShape(bits + ((int64_t)h * s.M_v + qb) * s.W, s.W, lane, BK, s.M_v,
                                         s.M_total, s.n_valid, s.n_cond)
                              : RowShape();
      const int T = 2 * n;
      float m_run = -INFINITY, l_run = 0.f;
      int kvalid = BK;
      float bias = 0.f;
      // one iteration per kv block, its two 64-key half-steps unrolled (the half index and
      // the per-block bookkeeping are then compile-time / once per block)
      for (int j = 0; j < n; ++j) {
        if (vis) {
          kvalid = j == rs.n_vis - 1 ? rs.kv_last_vis : (j == n - 1 ? rs.kv_last : BK);
          bias = j >= rs.n_vis ? beta_log2 : 0.f;
        } else {
          kvalid = block_valid(c0 + j, BK, s.M_v, s.n_valid, s.n_cond);
        }
#pragma unroll
      for (int hf = 0; hf < 2; ++hf, ++g) {
        const int t = 2 * j + hf;
        const int hvalid = kvalid - hf * HN;  // valid keys in this half (may be <= 0)
        if (lane == 0 && (warp & 3) == 2) TRACE(14, g);
        ptx::mbar_wait(&bars->s_full[g & 1], (g >> 1) & 1);
        if (lane == 0 && (warp & 3) == 2) TRACE(10, g);
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
        // p = 2^(s * scale_log2 + bias - m): one FFMA2 per two keys; returns the half's sum
        uint32_t pk[32];
        auto exps = [&](float c0) -> float {
          const uint64_t sc2 = f2_pack(scale_log2, scale_log2), c02 = f2_pack(c0, c0);
          uint64_t acc2[4];
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const uint64_t x = ffma2(
                f2_pack(__uint_as_float(sr[2 * e]), __uint_as_float(sr[2 * e + 1])), sc2, c02);
            float p0, p1;
            if ((e & 7) >= 8 - EMU) {  // FMA-pipe exp2 for EMU of every 8 pairs
              const uint64_t pp = exp2_poly2(x);
              p0 = f2_lo(pp);
              p1 = f2_hi(pp);
            } else {
              p0 = ptx::ex2(f2_lo(x));
              p1 = ptx::ex2(f2_hi(x));
            }
            acc2[e & 3] = e < 4 ? f2_pack(p0, p1) : fadd2(acc2[e & 3], f2_pack(p0, p1));
            pk[e] = Elem<E>::pack(p0, p1);
          }
          const uint64_t sum2 = fadd2(fadd2(acc2[0], acc2[1]), fadd2(acc2[2], acc2[3]));
          return f2_lo(sum2) + f2_hi(sum2);
        };
        // block max in the scaled log2 domain (scale > 0 keeps the argmax)
        auto block_max = [&]() -> float {
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
          return (mraw == -INFINITY) ? -INFINITY : fmaf(mraw, scale_log2, bias);
        };
        const bool first = (t == 0);
        bool need = false;
        float alpha = 1.f, sum;
        if (MAXFREE && !first) {
          // Max-free step: exponentiate against the running max first.  Every p <= sum, so a
          // half whose sum stays <= RESCALE_SUM_LIMIT (2^12) has no p above it and needs no
          // max at all; otherwise (a new row maximum, or NaN/inf) redo it the classic way.
          sum = exps(bias - m_run);
          const bool over = !(sum <= RESCALE_SUM_LIMIT);
          if (__any_sync(0xffffffffu, over)) {
            if (over) {
              const float m_new = fmaxf(m_run, block_max());
              need = m_new > m_run;
              if (need) alpha = ptx::ex2(m_run - m_new);
              m_run = m_new;
              sum = exps(bias - m_new);
            }
          }
        } else {
          const float m_new = fmaxf(m_run, block_max());
          need = !first && (m_new > m_run + RESCALE_THRESHOLD);
          const float m_use = (first || need) ? m_new : m_run;
          if (need) alpha = ptx::ex2(m_run - m_new);
          sum = exps(bias - m_use);
          m_run = m_use;
        }
        ptx::tmem_st32(t_row + (g & 1) * HN, pk);
        l_run = l_run * alpha + sum;
        if (__any_sync(0xffffffffu, need)) {
          // O is final only once PV(t-1) retired: its commit to the V slot's empty barrier
          // (the k-th PV on a slot completes that barrier's phase k).  S(t) being ready means
          // PV(t-2), issued before QK(t), is complete, so the parity cannot alias.
          ptx::mbar_wait(&bars->v_empty[(g - 1) % V_SLOTS], ((g - 1) / V_SLOTS) & 1);
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
        if (lane == 0 && (warp & 3) == 2) TRACE(12, g);
      }
      }
      // ---- epilogue: O / l -> bf16 row, padding rows zero (attention.py:203-206)
      ptx::mbar_wait(&bars->o_full, it & 1);
      ptx::tc_fence_after();
      const int qvalid = block_valid(qb, BM, s.M_v, s.n_valid, s.n_cond);
      if (!vis && cs.C > 1) {
        // one chunk of a split condition row: leave (O unnormalised, m, l); the chunk that
        // completes the row merges all C in chunk order (run-to-run deterministic)
        const int64_t rid = (int64_t)h * (s.M_total - s.M_v) + (qb - s.M_v);
        const int64_t n_part = (int64_t)s.H * (s.M_total - s.M_v) * cs.C;
        const int64_t slot = rid * cs.C + c0 / cs.len;
        float4* po = reinterpret_cast<float4*>(cs.part + (slot * BM + row) * D);
#pragma unroll 1
        for (int c = 0; c < D / 32; ++c) {
          uint32_t ov[32];
          ptx::tmem_ld32(t_row + O_COL + c * 32, ov);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 8; ++e)
            __stcg(po + c * 8 + e, make_float4(__uint_as_float(ov[4 * e]), __uint_as_float(ov[4 * e + 1]),
                                               __uint_as_float(ov[4 * e + 2]), __uint_as_float(ov[4 * e + 3])));
        }
        ptx::tc_fence_before();
        __stcg(reinterpret_cast<float2*>(cs.part + n_part * BM * D) + slot * BM + row,
               make_float2(m_run, l_run));
        __threadfence();
        ptx::named_bar_sync(1, 128);
        if (warp == 2 && lane == 0) bars->last = atomicAdd(cs.cnt + rid, 1);
        ptx::named_bar_sync(1, 128);
        // (`last` is rewritten only after the next split item's first barrier, which every
        // softmax thread reaches after reading it here)
        if (bars->last == cs.C - 1) {
          __threadfence();
          const float2* ml = reinterpret_cast<const float2*>(cs.part + n_part * BM * D) + rid * cs.C * BM + row;
          float mx = -INFINITY;
          for (int c = 0; c < cs.C; ++c) mx = fmaxf(mx, __ldcg(ml + c * BM).x);
          float lsum = 0.f;
          for (int c = 0; c < cs.C; ++c) {
            const float2 v = __ldcg(ml + c * BM);
            lsum += ptx::ex2(v.x - mx) * v.y;
          }
          const float inv_l = row < qvalid ? 1.f / lsum : 0.f;
          const float4* pr = reinterpret_cast<const float4*>(cs.part + (rid * cs.C * BM + row) * D);
          E* orow = o + (int64_t)h * s.sh + ((int64_t)qb * BM + row) * s.sn;
#pragma unroll 1
          for (int cc = 0; cc < D / 32; ++cc) {
            float acc[32];
#pragma unroll
            for (int e = 0; e < 32; ++e) acc[e] = 0.f;
#pragma unroll 1
            for (int c = 0; c < cs.C; ++c) {
              const float w = ptx::ex2(__ldcg(ml + c * BM).x - mx);
              const float4* src = pr + (int64_t)c * BM * (D / 4) + cc * 8;
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const float4 v = __ldcg(src + e);
                acc[4 * e] = fmaf(w, v.x, acc[4 * e]);
                acc[4 * e + 1] = fmaf(w, v.y, acc[4 * e + 1]);
                acc[4 * e + 2] = fmaf(w, v.z, acc[4 * e + 2]);
                acc[4 * e + 3] = fmaf(w, v.w, acc[4 * e + 3]);
              }
            }
            uint32_t pk[16];
#pragma unroll
            for (int e = 0; e < 16; ++e)
              pk[e] = row < qvalid ? Elem<E>::pack(acc[2 * e] * inv_l, acc[2 * e + 1] * inv_l) : 0u;
            int4* dst = reinterpret_cast<int4*>(orow + cc * 32);
#pragma unroll
            for (int e = 0; e < 4; ++e)
              __stcs(dst + e, make_int4((int)pk[4 * e], (int)pk[4 * e + 1], (int)pk[4 * e + 2],
                                        (int)pk[4 * e + 3]));
          }
        }
        continue;
      }
      const float inv_l = (row < qvalid && T > 0) ? 1.f / l_run : 0.f;
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

#undef TRACE
}  // namespace tc





static int validate(const void* q, const void* k, const void* v, void* o, int dtype,
                    const uint32_t* bits, const int32_t* kv_cnt, const CarveShape& s) {
  TCB_CHECK_ARG(q && k && v && o, TCB_ESHAPE, "null q/k/v/o");
  TCB_CHECK_ARG(dtype == TCB_F32 || dtype == TCB_BF16 || dtype == TCB_F16, TCB_EDOMAIN,
                "unsupported dtype %d", dtype);
  TCB_CHECK_ARG(s.H >= 1 && s.d >= 1 && s.m >= 1 && s.M_v >= 0 && s.M_total >= s.M_v &&
                    s.M_total >= 1,
                TCB_ESHAPE, "bad carve shape");
  TCB_CHECK_ARG(s.M_v == 0 || (bits && kv_cnt), TCB_ESHAPE, "null mask");
  TCB_CHECK_ARG(s.W >= (s.M_total + 31) / 32, TCB_ESHAPE, "mask row has %d words < %d columns", s.W,
                s.M_total);
  TCB_CHECK_ARG((int64_t)s.H * s.M_total < (int64_t)1 << 31, TCB_ESIZE, "too many work items");
  return TCB_OK;
}

}  // namespace tcb

using namespace tcb;

template <typename T, int MT, int DT>
static int launch_f32t(const void* q, const void* k, const void* v, void* o, const CarveShape& s,
                       const uint32_t* bits, const int32_t* kv_cnt, float beta, cudaStream_t st) {
  constexpr int M = 16 * MT, D = 16 * DT;
  // Q, K (M x (D+4)), V^T (D x (M+4)), and P (M x (M+4)) unless it fits in K's tile
  size_t smem = ((size_t)2 * M * (D + 4) + (size_t)D * (M + 4)) * sizeof(float);
  if (M + 4 > D + 4) smem += (size_t)M * (M + 4) * sizeof(float);
  static std::atomic<uint64_t> attr{0};
  {
    const cudaError_t e = once_per_device(attr, [&] {
      return cudaFuncSetAttribute(k_carve_f32t<T, MT, DT>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    });
    if (e != cudaSuccess) return set_error(TCB_ECUDA, "f32t smem: %s", cudaGetErrorString(e));
  }
  const float scale = (float)(1.0 / sqrt((double)s.d));
  k_carve_f32t<T, MT, DT><<<(unsigned)((int64_t)s.H * s.M_total), 256, smem, st>>>(
      (const T*)q, (const T*)k, (const T*)v, (T*)o, s, bits, kv_cnt, beta, scale);
  return check_launch("k_carve_f32t");
}

template <typename T>
static int try_f32t(const void* q, const void* k, const void* v, void* o, const CarveShape& s,
                    const uint32_t* bits, const int32_t* kv_cnt, float beta, cudaStream_t st) {
  const int key = (s.m << 16) | s.d;
  switch (key) {
    case (128 << 16) | 128: return launch_f32t<T, 8, 8>(q, k, v, o, s, bits, kv_cnt, beta, st);
    case (128 << 16) | 64: return launch_f32t<T, 8, 4>(q, k, v, o, s, bits, kv_cnt, beta, st);
    case (64 << 16) | 128: return launch_f32t<T, 4, 8>(q, k, v, o, s, bits, kv_cnt, beta, st);
    case (64 << 16) | 64: return launch_f32t<T, 4, 4>(q, k, v, o, s, bits, kv_cnt, beta, st);
    case (64 << 16) | 32: return launch_f32t<T, 4, 2>(q, k, v, o, s, bits, kv_cnt, beta, st);
    case (32 << 16) | 64: return launch_f32t<T, 2, 4>(q, k, v, o, s, bits, kv_cnt, beta, st);
    case (32 << 16) | 32: return launch_f32t<T, 2, 2>(q, k, v, o, s, bits, kv_cnt, beta, st);
    case (128 << 16) | 32: return launch_f32t<T, 8, 2>(q, k, v, o, s, bits, kv_cnt, beta, st);
    case (128 << 16) | 16: return launch_f32t<T, 8, 1>(q, k, v, o, s, bits, kv_cnt, beta, st);
    case (64 << 16) | 16: return launch_f32t<T, 4, 1>(q, k, v, o, s, bits, kv_cnt, beta, st);
    case (16 << 16) | 16: return launch_f32t<T, 1, 1>(q, k, v, o, s, bits, kv_cnt, beta, st);
    default: return -1;  // not tiled: the per-row kernel takes it
  }
}

template <typename T>
static int launch_simt_t(const void* q, const void* k, const void* v, void* o, const CarveShape& s,
                         const uint32_t* bits, const int32_t* kv_cnt, float beta, cudaStream_t st) {
  {  // tiled fp32-math kernel for the common block / head sizes
    const int rc = try_f32t<T>(q, k, v, o, s, bits, kv_cnt, beta, st);
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
  k_carve_simt<T><<<grid, 128, smem, st>>>((const T*)q, (const T*)k, (const T*)v, (T*)o, s, bits,
                                           kv_cnt, beta, scale);
  return check_launch("k_carve_simt");
}

static int launch_simt(const void* q, const void* k, const void* v, void* o, int dtype,
                       const CarveShape& s, const uint32_t* bits, const int32_t* kv_cnt,
                       float beta, cudaStream_t st) {
  if (dtype == TCB_F32) return launch_simt_t<float>(q, k, v, o, s, bits, kv_cnt, beta, st);
  if (dtype == TCB_BF16) return launch_simt_t<__nv_bfloat16>(q, k, v, o, s, bits, kv_cnt, beta, st);
  return launch_simt_t<__half>(q, k, v, o, s, bits, kv_cnt, beta, st);
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

// Workspace of tcb_carve_fwd: [0, 256) scheduler counter; then, when condition rows are
// split, the per-row chunk counters (256-aligned) and the partials (O, then (m, l)).
constexpr int SPLIT_LEN = 128;  // target kv blocks per condition-row chunk (~a vision row)
static void cond_split_plan(int M_v, int M_total, int& C, int& len) {
  C = (M_total - M_v) > 0 ? (M_total + SPLIT_LEN - 1) / SPLIT_LEN : 1;
  if (C < 2) C = 1;
  len = (M_total + C - 1) / C;
}
static int64_t align256(int64_t x) { return (x + 255) & ~(int64_t)255; }
static int64_t split_cnt_bytes(int H, int M_c) { return align256((int64_t)H * M_c * 4); }
constexpr int64_t SPLIT_MAX_BYTES = 256ll << 20;  // beyond this, condition rows run unsplit
static int64_t carve_work_bytes(int H, int M_v, int M_total, int d) {
  int C, len;
  cond_split_plan(M_v, M_total, C, len);
  if (C == 1) return 256;
  const int64_t parts = (int64_t)H * (M_total - M_v) * C * tc::BM;
  const int64_t items = (int64_t)H * (M_v + (int64_t)(M_total - M_v) * C);
  const int64_t bytes = 256 + split_cnt_bytes(H, M_total - M_v) + parts * (d + 2) * 4;
  // many condition blocks already give plenty of parallel items: a bounded workspace
  if (bytes > SPLIT_MAX_BYTES || items >= ((int64_t)1 << 31)) return 256;
  return bytes;
}

static bool split_disabled() {  // TCB_CARVE_NOSPLIT=1: A/B of the unsplit order
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TCB_CARVE_NOSPLIT");
    v = (e && atoi(e) != 0) ? 1 : 0;
  }
  return v == 1;
}

template <int D, int EMU, typename E = __nv_bfloat16, int MAXFREE = 0>
static int launch_tc(const void* q, const void* k, const void* v, void* o, const CarveShape& s,
                     const uint32_t* bits, const int32_t* kv_cnt, float beta, int32_t* work,
                     int64_t work_bytes, cudaStream_t st) {
  CUtensorMap tq, tk, tv;
  const int64_t n_pad = (int64_t)s.M_total * s.m;
  int rc;
  if ((rc = make_tmap_rows(&tq, q, D, n_pad, s.H, s.sh, s.sn, tc::BM, !tc::Elem<E>::kBf16))) return rc;
  if ((rc = make_tmap_rows(&tk, k, D, n_pad, s.H, s.sh, s.sn, tc::HN, !tc::Elem<E>::kBf16))) return rc;
  if ((rc = make_tmap_rows(&tv, v, D, n_pad, s.H, s.sh, s.sn, tc::HN, !tc::Elem<E>::kBf16))) return rc;
  const int smem = tc::Smem<D>::BYTES;
  static std::atomic<uint64_t> attr{0};
  {
    const cudaError_t e = once_per_device(attr, [&] {
      return cudaFuncSetAttribute(tc::k_carve_tc<D, EMU, E, MAXFREE>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    });
    if (e != cudaSuccess) return set_error(TCB_ECUDA, "carve smem attr: %s", cudaGetErrorString(e));
  }
  // split condition rows when the caller's workspace holds the partials (else all condition
  // rows run first, unsplit)
  tc::CondSplit cs{1, s.M_total, nullptr, nullptr};
  int64_t zero_bytes = sizeof(int32_t);
  if (work_bytes >= carve_work_bytes(s.H, s.M_v, s.M_total, D) && carve_work_bytes(s.H, s.M_v, s.M_total, D) > 256 &&
      !split_disabled()) {
    cond_split_plan(s.M_v, s.M_total, cs.C, cs.len);
    uint8_t* base = reinterpret_cast<uint8_t*>(work);
    cs.cnt = reinterpret_cast<int*>(base + 256);
    cs.part = reinterpret_cast<float*>(base + 256 + split_cnt_bytes(s.H, s.M_total - s.M_v));
    zero_bytes = 256 + split_cnt_bytes(s.H, s.M_total - s.M_v);
  }
  cudaError_t e = cudaMemsetAsync(work, 0, zero_bytes, st);
  if (e != cudaSuccess) return set_error(TCB_ECUDA, "memset counter: %s", cudaGetErrorString(e));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int total = s.H * (s.M_v + (s.M_total - s.M_v) * cs.C);
  int grid = 2 * sms;
  if (grid > total) grid = total;
  const float LOG2E = 1.4426950408889634f;
  const float scale_log2 = (float)(1.0 / sqrt((double)s.d)) * LOG2E;
  tc::k_carve_tc<D, EMU, E, MAXFREE><<<grid, tc::NUM_THREADS, smem, st>>>(tq, tk, tv, (E*)o, s, bits,
                                                         kv_cnt, work, total, scale_log2,
                                                         beta * LOG2E, dbg_flags(), cs);
  return check_launch("k_carve_tc");
}




extern "C" int tcb_carve_fwd_simt(const void* q, const void* k, const void* v, void* o, int dtype,
                                  int64_t stride_h, int64_t stride_n, const uint32_t* bits,
                                  int words, const int32_t* kv_cnt, int H, int d, int m, int M_v,
                                  int M_total, int64_t n_valid, int64_t n_cond, float beta,
                                  void* stream) {
  CarveShape s{H, d, m, M_v, M_total, words, n_valid, n_cond, stride_h, stride_n};
  int rc = validate(q, k, v, o, dtype, bits, kv_cnt, s);
  if (rc) return rc;
  return launch_simt(q, k, v, o, dtype, s, bits, kv_cnt, beta, as_stream(stream));
}

extern "C" int64_t tcb_carve_workspace_bytes(int H, int M_v, int M_total, int m, int d) {
  if (H < 1 || M_v < 0 || M_total < M_v || M_total < 1) return 256;
  if (m != 128 || (d != 64 && d != 128)) return 256;  // SIMT kernels: only the counter
  return carve_work_bytes(H, M_v, M_total, d);
}

extern "C" int tcb_carve_fwd(const void* q, const void* k, const void* v, void* o, int dtype,
                             int64_t stride_h, int64_t stride_n, const uint32_t* bits, int words,
                             const int32_t* kv_cnt, int H, int d, int m, int M_v, int M_total,
                             int64_t n_valid, int64_t n_cond, float beta, int32_t* work,
                             int64_t work_bytes, void* stream) {
  CarveShape s{H, d, m, M_v, M_total, words, n_valid, n_cond, stride_h, stride_n};
  if ((uintptr_t)work % 256 != 0) work_bytes = 0;  // partials need 256-byte alignment
  int rc = validate(q, k, v, o, dtype, bits, kv_cnt, s);
  if (rc) return rc;
  const bool aligned = ((uintptr_t)q % 16 == 0) && ((uintptr_t)k % 16 == 0) &&
                       ((uintptr_t)v % 16 == 0) && ((uintptr_t)o % 16 == 0) &&
                       (stride_n * 2) % 16 == 0 && (stride_h * 2) % 16 == 0;
  const bool tc_ok = (dtype == TCB_BF16 || dtype == TCB_F16) && m == 128 && (d == 128 || d == 64) &&
                     aligned && work && M_v > 0;
  if (!tc_ok) return launch_simt(q, k, v, o, dtype, s, bits, kv_cnt, beta, as_stream(stream));
  // pairs (of 8) whose exp2 runs on the FMA pipe instead of MUFU; TCB_CARVE_EMU overrides.
  // TCB_CARVE_MAXFREE=0 selects the classic per-half-step block max (A/B experiments).
  static int emu = -1, maxfree = -1;
  if (emu < 0) {
    const char* env = getenv("TCB_CARVE_EMU");
    emu = env ? atoi(env) : 0;
    if (emu < 0 || emu > 2) emu = 0;
    env = getenv("TCB_CARVE_MAXFREE");
    maxfree = env ? atoi(env) != 0 : 1;
  }
  cudaStream_t st = as_stream(stream);
  if (dtype == TCB_F16)  // fp16 operands and P (kind::f16 with f16 inputs), f32 accumulation
    return d == 128 ? launch_tc<128, 0, __half, 1>(q, k, v, o, s, bits, kv_cnt, beta, work, work_bytes, st)
                    : launch_tc<64, 0, __half, 1>(q, k, v, o, s, bits, kv_cnt, beta, work, work_bytes, st);
  if (d == 128) {
    if (!maxfree) return launch_tc<128, 0, __nv_bfloat16, 0>(q, k, v, o, s, bits, kv_cnt, beta, work, work_bytes, st);
    switch (emu) {
      case 1: return launch_tc<128, 1, __nv_bfloat16, 1>(q, k, v, o, s, bits, kv_cnt, beta, work, work_bytes, st);
      case 2: return launch_tc<128, 2, __nv_bfloat16, 1>(q, k, v, o, s, bits, kv_cnt, beta, work, work_bytes, st);
      default: return launch_tc<128, 0, __nv_bfloat16, 1>(q, k, v, o, s, bits, kv_cnt, beta, work, work_bytes, st);
    }
  }
  return launch_tc<64, 0, __nv_bfloat16, 1>(q, k, v, o, s, bits, kv_cnt, beta, work, work_bytes, st);
}

#ifdef TCB_CARVE_TRACE
// Trace builds only (not part of include/tokencarve_b200.h): copy out and clear CTA 0's
// timeline, TRACE_EV x TRACE_STEPS clocks (0 = not reached).
extern "C" int tcb_debug_trace_read(unsigned long long* host, int cap) {
  const int n = tcb::tc::TRACE_EV * tcb::tc::TRACE_STEPS;
  if (cap < n) return -1;
  cudaMemcpyFromSymbol(host, tcb::tc::g_trace, sizeof(unsigned long long) * n);
  static unsigned long long zero[tcb::tc::TRACE_EV * tcb::tc::TRACE_STEPS];
  cudaMemcpyToSymbol(tcb::tc::g_trace, zero, sizeof(zero));
  return n;
}
#endif
