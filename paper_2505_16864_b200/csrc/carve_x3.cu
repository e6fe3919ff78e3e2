// fp32 inputs on the tensor cores: block-sparse attention (carve_attention, attention.py:162-243,
// the reference's own fp32 semantics) as three fp16 products per operand pair.
//
// Every fp32 operand x is carried as x * 2^e = hi + lo with hi = fp16(x * 2^e) and
// lo = fp16(x * 2^e - hi) (22 significant bits; 2^e puts the tensor's max magnitude in
// [2^14, 2^15) so neither half overflows and the subnormal floor of lo sits 2^-39 below the
// max).  A product a.b is taken as hi_a.hi_b + hi_a.lo_b + lo_a.hi_b on kind::f16 with fp32
// accumulation (the dropped lo.lo term is ~2^-22 relative), which keeps the layer within the
// north_star's 1e-5 of the fp32 reference at the full fp16 tensor rate: 3 MMAs per product
// vs 6 for 3xTF32 (kind::tf32 runs at half the f16 rate).
//
//   * Q: each softmax thread reads its own fp32 query row, picks the row's exponent, splits it
//     and stores hi / lo straight into TMEM (A operand of the TS QK^T) -- no pre-pass.
//   * K, V: k_kv_absmax (max |x| per tensor and head, padding rows skipped) and k_kv_split
//     (hi / lo fp16 planes, padding rows zeroed) write a (2H, N_pad, d) fp16 stack per tensor
//     into the caller's workspace, TMA-tiled by the main kernel exactly like the bf16 K / V.
//   * P: softmax computes p' = 2^6 p in fp32 (ex2), splits it into hi / lo fp16 over the
//     first / second 32 columns of its S buffer; O += Ph.Vh + Ph.Vl + Pl.Vh.
//   * Scales fold into the softmax: the score multiplier of row r is
//     log2(e)/sqrt(d) * 2^-(e_q[r] + e_k[h]); the epilogue multiplies O by 2^-e_v[h] / l.
//   * O is not accumulated across kv blocks in TMEM: the tensor core's fp32 accumulation
//     rounds toward zero (measured: |O| shrinks by ~4e-5 relative over a 95-block row when
//     every PV accumulates onto the running O), so O_mma collects one pair of PVs (one kv
//     block: fresh at even half-steps, accumulating at odd ones) and the softmax warps fold
//     each pair into O_tot with round-to-nearest fp32 (O_tot = (O_tot + O_mma) * alpha)
//     before releasing the next even P -- the same spot the lazy rescale used.  (A fold per
//     PV: 1.3e-6 max error on a C2 head and 52.0 ms; per pair: 1.5e-6 and 50.3 ms.)
//
// Structure follows k_carve_tc (carve.cu) with one CTA per SM (the split K / V tiles need
// 192 KB of shared memory): warp 0 TMA producer + scheduler, warp 1 MMA issuer, warps 2-5
// softmax / Q split / epilogue.  TMEM (512 columns): Qh [0, D/2), Ql [D/2, D), S0, S1 (64
// keys each), O_mma, O_tot.
#include "tc_common.cuh"

#include <math.h>

namespace tcb {
namespace x3 {

constexpr int BM = 128, BK = 128, HN = 64;
constexpr int NUM_THREADS = 192;
constexpr int K_SLOTS = 3, V_SLOTS = 3;
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 units, as k_carve_tc
constexpr float P_SHIFT = 6.0f;            // p' = 2^6 p <= 2^14 < fp16 max

template <int D>
struct Cfg {
  static constexpr int HALF_BYTES = HN * D * 2;       // one fp16 plane of a 64-key tile
  static constexpr int SLOT_BYTES = 2 * HALF_BYTES;   // hi + lo
  static constexpr int CHUNKS = D / 64;
  static constexpr int H_CHUNK = HN * 128;
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = OFF_K + K_SLOTS * SLOT_BYTES;
  static constexpr int OFF_BAR = OFF_V + V_SLOTS * SLOT_BYTES;
  static constexpr int BYTES = OFF_BAR + 256;
  static constexpr int QH = 0, QL = D / 2, S_COL = D, O_COL = D + 2 * HN, OT_COL = O_COL + D;
  static constexpr int TMEM_COLS = 512;
  static_assert(OT_COL + D <= TMEM_COLS, "TMEM budget");
};

struct Bars {
  uint64_t q_full, o_full;
  uint64_t p_full[2], s_full[2];
  uint64_t k_full[K_SLOTS], k_empty[K_SLOTS];
  uint64_t v_full[V_SLOTS], v_empty[V_SLOTS];
  uint64_t sched_full[2], sched_empty[2];
  int sched_item[2];
  uint32_t tmem_base;
};
static_assert(sizeof(Bars) <= 256, "barrier block must fit the reserved smem");

// exponent e with max * 2^e in [2^14, 2^15) (0 for an all-zero / non-finite tensor)
__device__ __forceinline__ int split_exp(float amax) {
  if (!(amax > 0.f) || !isfinite(amax)) return 0;
  const int E = ((__float_as_uint(amax) >> 23) & 255) - 127;
  int e = 14 - E;
  return e < -120 ? -120 : (e > 120 ? 120 : e);
}
__device__ __forceinline__ float pow2(int e) { return __uint_as_float((uint32_t)(127 + e) << 23); }

__device__ __forceinline__ uint32_t h2_bits(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }

// (x0, x1) -> packed fp16 hi pair and lo pair
__device__ __forceinline__ void split2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(x0, x1);
  const float2 hf = __half22float2(h);
  hi = h2_bits(h);
  lo = h2_bits(__floats2half2_rn(x0 - hf.x, x1 - hf.y));
}

__device__ __forceinline__ bool row_valid(int64_t t, const CarveShape& s) {
  const int b = (int)(t / s.m);
  return (int)(t - (int64_t)b * s.m) < block_valid(b, s.m, s.M_v, s.n_valid, s.n_cond);
}

// max |x| over the valid rows of K (z = 0) and V (z = 1) per head -> amax_bits[z * H + h]
template <int D>
__global__ void __launch_bounds__(256) k_kv_absmax(const float* __restrict__ k,
                                                   const float* __restrict__ v, CarveShape s,
                                                   int rows_per_cta, uint32_t* __restrict__ amax_bits) {
  constexpr int V4 = D / 4;
  const int h = blockIdx.y, z = blockIdx.z;
  const float* src = (z ? v : k) + (int64_t)h * s.sh;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t n_pad = (int64_t)s.M_total * s.m;
  float mx = 0.f;
  for (int i = threadIdx.x; i < rows_per_cta * V4; i += blockDim.x) {
    const int64_t t = r0 + i / V4;
    if (t >= n_pad || !row_valid(t, s)) continue;
    const float4 x = __ldg(reinterpret_cast<const float4*>(src + t * s.sn) + (i % V4));
    mx = fmaxf(mx, fmaxf(fmaxf(fabsf(x.x), fabsf(x.y)), fmaxf(fabsf(x.z), fabsf(x.w))));
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  __shared__ float red[8];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = fmaxf(mx, red[w]);
    atomicMax(amax_bits + z * s.H + h, __float_as_uint(mx));  // non-negative: bit order == value order
  }
}

// hi / lo fp16 planes of K and V: out_z[(p * H + h), t, c], padding rows zero
template <int D>
__global__ void __launch_bounds__(256) k_kv_split(const float* __restrict__ k, const float* __restrict__ v,
                                                  CarveShape s, int rows_per_cta,
                                                  const uint32_t* __restrict__ amax_bits,
                                                  __half* __restrict__ kst, __half* __restrict__ vst) {
  constexpr int V4 = D / 4;
  const int h = blockIdx.y, z = blockIdx.z;
  const float* src = (z ? v : k) + (int64_t)h * s.sh;
  __half* dst = z ? vst : kst;
  const int64_t n_pad = (int64_t)s.M_total * s.m;
  const float sc = pow2(split_exp(__uint_as_float(amax_bits[z * s.H + h])));
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  __half* hi = dst + (int64_t)h * n_pad * D;
  __half* lo = dst + (int64_t)(s.H + h) * n_pad * D;
  for (int i = threadIdx.x; i < rows_per_cta * V4; i += blockDim.x) {
    const int64_t t = r0 + i / V4;
    if (t >= n_pad) break;
    const int c4 = i % V4;
    uint2 ho = make_uint2(0u, 0u), lw = make_uint2(0u, 0u);
    if (row_valid(t, s)) {
      const float4 x = __ldg(reinterpret_cast<const float4*>(src + t * s.sn) + c4);
      split2(x.x * sc, x.y * sc, ho.x, lw.x);
      split2(x.z * sc, x.w * sc, ho.y, lw.y);
    }
    reinterpret_cast<uint2*>(hi + t * D)[c4] = ho;
    reinterpret_cast<uint2*>(lo + t * D)[c4] = lw;
  }
}

template <int D>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    k_carve_x3(const float* __restrict__ q, const __grid_constant__ CUtensorMap tm_k,
               const __grid_constant__ CUtensorMap tm_v, float* __restrict__ o, CarveShape s,
               const uint32_t* __restrict__ bits, const int32_t* __restrict__ kv_cnt,
               const uint32_t* __restrict__ amax_bits, int* __restrict__ counter, int total_items,
               float scale_log2, float beta_log2) {
  using C = Cfg<D>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sK = smem + C::OFF_K;
  uint8_t* sV = smem + C::OFF_V;
  Bars* bars = reinterpret_cast<Bars*>(smem + C::OFF_BAR);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    if (ptx::smem_u32(smem) & 1023u) __trap();
    ptx::mbar_init(&bars->q_full, 128);
    ptx::mbar_init(&bars->o_full, 1);
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&bars->p_full[i], 128);
      ptx::mbar_init(&bars->s_full[i], 1);
      ptx::mbar_init(&bars->sched_full[i], 1);
      ptx::mbar_init(&bars->sched_empty[i], 1 + 4);
    }
    for (int i = 0; i < K_SLOTS; ++i) {
      ptx::mbar_init(&bars->k_full[i], 1);
      ptx::mbar_init(&bars->k_empty[i], 1);
    }
    for (int i = 0; i < V_SLOTS; ++i) {
      ptx::mbar_init(&bars->v_full[i], 1);
      ptx::mbar_init(&bars->v_empty[i], 1);
    }
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&tm_k);
    ptx::tma_prefetch_desc(&tm_v);
  }
  if (warp == 1) ptx::tmem_alloc<C::TMEM_COLS>(&bars->tmem_base);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == 0) {
    // ============================ TMA producer + scheduler ============================
    const uint64_t pol_kv = ptx::policy_evict_last();
    const uint64_t pol_cond = ptx::policy_evict_first();
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
      const uint32_t* brow = bits + ((int64_t)h * s.M_v + (vis ? qb : 0)) * s.W;
      WarpKvList wk(vis ? brow : nullptr, s.W, lane), wv(vis ? brow : nullptr, s.W, lane);
      const int T = 2 * n;
      auto load = [&](const CUtensorMap* tm, uint8_t* base, uint64_t* full, uint64_t* empty,
                      int slots, uint32_t& cnt, int t, WarpKvList& walk) {
        const int b = vis ? walk.block(t >> 1) : (t >> 1);
        if (lane == 0) {
          const int sl = cnt % slots;
          ptx::mbar_wait(&empty[sl], ((cnt / slots) & 1) ^ 1);
          ptx::mbar_arrive_expect_tx(&full[sl], C::SLOT_BYTES);
#pragma unroll
          for (int p = 0; p < 2; ++p)
#pragma unroll
            for (int c = 0; c < C::CHUNKS; ++c)
              ptx::tma_load_3d(base + sl * C::SLOT_BYTES + p * C::HALF_BYTES + c * C::H_CHUNK, tm,
                               &full[sl], c * 64, b * BK + (t & 1) * HN, h + p * s.H,
                               vis ? pol_kv : pol_cond);
        }
        ++cnt;
      };
      if (T > 0) load(&tm_k, sK, bars->k_full, bars->k_empty, K_SLOTS, gk, 0, wk);
      for (int t = 0; t < T; ++t) {
        if (t + 1 < T) load(&tm_k, sK, bars->k_full, bars->k_empty, K_SLOTS, gk, t + 1, wk);
        load(&tm_v, sV, bars->v_full, bars->v_empty, V_SLOTS, gv, t, wv);
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ============================
    constexpr uint32_t IDESC_S = tc::make_idesc(BM, HN, 0, 0);  // Q (TMEM) x K (K-major), f16
    constexpr uint32_t IDESC_O = tc::make_idesc(BM, D, 1, 0);   // P (TMEM) x V (MN-major), f16
    const uint32_t aK = ptx::smem_u32(sK), aV = ptx::smem_u32(sV);
    uint32_t it = 0, gk = 0, gv = 0, gs = 0, gp = 0;
    // S(gs) = Qh Kl^T + Ql Kh^T + Qh Kh^T: the small cross terms go first, while the
    // accumulator is small, so the tensor core's truncating fp32 adds cost ~8 instead of ~24
    // half-ulps of S (measured: 3x smaller score error on peaked rows)
    auto issue_s = [&]() {
      const int sl = gk % K_SLOTS;
      ptx::mbar_wait(&bars->k_full[sl], (gk / K_SLOTS) & 1);
      ptx::tc_fence_after();
      const uint32_t kbase = aK + sl * C::SLOT_BYTES;
      const uint32_t sbuf = tmem + C::S_COL + (gs & 1) * HN;
      if (ptx::elect_one()) {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t kh = kbase + (kk >> 2) * C::H_CHUNK + (kk & 3) * 32;
          ptx::mma_ts(sbuf, tmem + C::QH + kk * 8, tc::make_sdesc(kh + C::HALF_BYTES, 16, 1024), IDESC_S,
                      kk > 0 ? 1u : 0u);
          ptx::mma_ts(sbuf, tmem + C::QL + kk * 8, tc::make_sdesc(kh, 16, 1024), IDESC_S, 1u);
        }
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t kh = kbase + (kk >> 2) * C::H_CHUNK + (kk & 3) * 32;
          ptx::mma_ts(sbuf, tmem + C::QH + kk * 8, tc::make_sdesc(kh, 16, 1024), IDESC_S, 1u);
        }
        ptx::mma_commit(&bars->k_empty[sl]);
        ptx::mma_commit(&bars->s_full[gs & 1]);
      }
      __syncwarp();
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
      int h, qb;
      decode_item(item, s, h, qb);
      const bool vis = qb < s.M_v;
      const int n = vis ? kv_cnt[(int64_t)h * s.M_v + qb] : s.M_total;
      const int T = 2 * n;
      ptx::mbar_wait(&bars->q_full, it & 1);  // this item's Q is in TMEM, the last O read out
      ptx::tc_fence_after();
      if (T == 0) {
        if (ptx::elect_one()) ptx::mma_commit(&bars->o_full);
        __syncwarp();
        continue;
      }
      issue_s();
      for (int t = 0; t < T; ++t) {
        if (t + 1 < T) issue_s();
        ptx::mbar_wait(&bars->p_full[gp & 1], (gp >> 1) & 1);
        const int vs = gv % V_SLOTS;
        ptx::mbar_wait(&bars->v_full[vs], (gv / V_SLOTS) & 1);
        ptx::tc_fence_after();
        const uint32_t vbase = aV + vs * C::SLOT_BYTES;
        const uint32_t pcol = tmem + C::S_COL + (gp & 1) * HN;
        if (ptx::elect_one()) {
          // O_mma fresh at even t, accumulating at odd t (the softmax warps fold each pair
          // into O_tot); cross terms first
#pragma unroll
          for (int kk = 0; kk < HN / 16; ++kk) {
            const uint32_t vh = vbase + kk * 16 * 128;
            ptx::mma_ts(tmem + C::O_COL, pcol + kk * 8, tc::make_sdesc(vh + C::HALF_BYTES, C::H_CHUNK, 1024),
                        IDESC_O, (kk > 0 || (t & 1)) ? 1u : 0u);
            ptx::mma_ts(tmem + C::O_COL, pcol + 32 + kk * 8, tc::make_sdesc(vh, C::H_CHUNK, 1024), IDESC_O, 1u);
          }
#pragma unroll
          for (int kk = 0; kk < HN / 16; ++kk)
            ptx::mma_ts(tmem + C::O_COL, pcol + kk * 8, tc::make_sdesc(vbase + kk * 16 * 128, C::H_CHUNK, 1024),
                        IDESC_O, 1u);
          ptx::mma_commit(&bars->v_empty[vs]);
        }
        __syncwarp();
        ++gv;
        ++gp;
      }
      if (ptx::elect_one()) ptx::mma_commit(&bars->o_full);
      __syncwarp();
    }
  } else {
    // ============================ Q split / softmax / epilogue ============================
    const int quarter = warp & 3;
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
      const RowShape rs = vis ? RowShape(bits + ((int64_t)h * s.M_v + qb) * s.W, s.W, lane, BK, s.M_v,
                                         s.M_total, s.n_valid, s.n_cond)
                              : RowShape();
      const int T = 2 * n;
      const int qvalid = block_valid(qb, BM, s.M_v, s.n_valid, s.n_cond);
      const bool live = row < qvalid;
      // ---- this thread's query row -> TMEM as fp16 hi / lo (the previous item's MMAs are
      // all complete: its epilogue waited on o_full)
      int eq = 0;
      {
        const float4* src = reinterpret_cast<const float4*>(q + (int64_t)h * s.sh +
                                                            ((int64_t)qb * BM + row) * s.sn);
        float amax = 0.f;
        if (live) {
#pragma unroll 8
          for (int c = 0; c < D / 4; ++c) {
            const float4 x = __ldg(src + c);
            amax = fmaxf(amax, fmaxf(fmaxf(fabsf(x.x), fabsf(x.y)), fmaxf(fabsf(x.z), fabsf(x.w))));
          }
        }
        eq = split_exp(amax);
        const float sc = pow2(eq);
#pragma unroll 1
        for (int c = 0; c < D / 64; ++c) {
          uint32_t wh[32], wl[32];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
            if (live) x = __ldg(src + c * 16 + e);
            split2(x.x * sc, x.y * sc, wh[2 * e], wl[2 * e]);
            split2(x.z * sc, x.w * sc, wh[2 * e + 1], wl[2 * e + 1]);
          }
          ptx::tmem_st32(t_row + C::QH + c * 32, wh);
          ptx::tmem_st32(t_row + C::QL + c * 32, wl);
        }
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&bars->q_full);
      }
      const int ek = split_exp(__uint_as_float(__ldg(amax_bits + h)));
      const int ev = split_exp(__uint_as_float(__ldg(amax_bits + s.H + h)));
      const float c_row = scale_log2 * pow2(-(eq + ek));  // S_acc -> log2-domain scaled score
      float m_run = -INFINITY, l_run = 0.f;
      int kvalid = BK;
      float bias = 0.f;
      for (int j = 0; j < n; ++j) {  // kv blocks; their two half-steps unrolled (see carve.cu)
        if (vis) {
          kvalid = j == rs.n_vis - 1 ? rs.kv_last_vis : (j == n - 1 ? rs.kv_last : BK);
          bias = j >= rs.n_vis ? beta_log2 : 0.f;
        } else {
          kvalid = block_valid(j, BK, s.M_v, s.n_valid, s.n_cond);
        }
#pragma unroll
      for (int hf = 0; hf < 2; ++hf, ++g) {
        const int t = 2 * j + hf;
        const int hvalid = kvalid - hf * HN;
        ptx::mbar_wait(&bars->s_full[g & 1], (g >> 1) & 1);
        ptx::tc_fence_after();
        const uint32_t sb = t_row + C::S_COL + (g & 1) * HN;
        uint32_t sr[64];
        ptx::tmem_ld32(sb, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
        ptx::tmem_ld32(sb + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
        ptx::tmem_wait_ld();
        if (hvalid < HN) {  // padding keys -> -inf (attention.py:193)
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
          for (int qq = 0; qq < 8; ++qq)
            mx8[qq] = tc::fmax3(mx8[qq], __uint_as_float(sr[e + qq]), __uint_as_float(sr[e + 8 + qq]));
        const float mraw = tc::fmax3(tc::fmax3(mx8[0], mx8[1], mx8[2]), tc::fmax3(mx8[3], mx8[4], mx8[5]),
                                     fmaxf(mx8[6], mx8[7]));
        const float m_blk = (mraw == -INFINITY) ? -INFINITY : fmaf(mraw, c_row, bias);
        const float m_new = fmaxf(m_run, m_blk);
        const bool first = (t == 0);
        const bool need = !first && (m_new > m_run + RESCALE_THRESHOLD);
        const float m_use = (first || need) ? m_new : m_run;
        const float alpha = need ? ptx::ex2(m_run - m_new) : 1.f;
        const float c0 = bias - m_use + P_SHIFT;
        const uint64_t sc2 = tc::f2_pack(c_row, c_row), c02 = tc::f2_pack(c0, c0);
        uint64_t acc2[4] = {0, 0, 0, 0};
        uint32_t ph[32], pl[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const uint64_t x = tc::ffma2(tc::f2_pack(__uint_as_float(sr[2 * e]), __uint_as_float(sr[2 * e + 1])),
                                       sc2, c02);
          const float p0 = ptx::ex2(tc::f2_lo(x)), p1 = ptx::ex2(tc::f2_hi(x));
          acc2[e & 3] = tc::fadd2(acc2[e & 3], tc::f2_pack(p0, p1));
          split2(p0, p1, ph[e], pl[e]);
        }
        ptx::tmem_st32(sb, ph);
        ptx::tmem_st32(sb + 32, pl);
        const uint64_t sum2 = tc::fadd2(tc::fadd2(acc2[0], acc2[1]), tc::fadd2(acc2[2], acc2[3]));
        l_run = l_run * alpha + (tc::f2_lo(sum2) + tc::f2_hi(sum2));
        m_run = m_use;
        // O_mma collects a pair of PVs (even t fresh, odd t accumulating); at even t >= 2 the
        // pair PV(t-2) + PV(t-1) is folded into O_tot (round-to-nearest), rescaled to this
        // step's max; an odd step that raises the max rescales O_mma (and O_tot) in place
        // before PV(t) adds onto it.  PV(t-1) is waited for on its V slot's empty barrier (the
        // k-th PV on a slot completes phase k); S(t) complete implies PV(t-2) -- and so the
        // slot's previous PV(t-4) -- complete (issued before QK(t)): the parity cannot alias.
        const bool fold = t >= 2 && !(t & 1);
        if (fold || ((t & 1) && __any_sync(0xffffffffu, need))) {
          ptx::mbar_wait(&bars->v_empty[(g - 1) % V_SLOTS], ((g - 1) / V_SLOTS) & 1);
          ptx::tc_fence_after();
          const uint64_t a2 = tc::f2_pack(alpha, alpha);
          const bool ot_valid = t > 2;
#pragma unroll 1
          for (int c = 0; c < D / 32; ++c) {
            uint32_t om[32], ot[32];
            ptx::tmem_ld32(t_row + C::O_COL + c * 32, om);
            if (ot_valid) ptx::tmem_ld32(t_row + C::OT_COL + c * 32, ot);
            ptx::tmem_wait_ld();
            if (fold) {
#pragma unroll
              for (int e = 0; e < 16; ++e) {
                uint64_t sum = tc::f2_pack(__uint_as_float(om[2 * e]), __uint_as_float(om[2 * e + 1]));
                if (ot_valid)
                  sum = tc::fadd2(sum, tc::f2_pack(__uint_as_float(ot[2 * e]), __uint_as_float(ot[2 * e + 1])));
                sum = tc::fmul2(sum, a2);
                ot[2 * e] = __float_as_uint(tc::f2_lo(sum));
                ot[2 * e + 1] = __float_as_uint(tc::f2_hi(sum));
              }
              ptx::tmem_st32(t_row + C::OT_COL + c * 32, ot);
            } else {
#pragma unroll
              for (int e = 0; e < 32; ++e) {
                om[e] = __float_as_uint(__uint_as_float(om[e]) * alpha);
                if (ot_valid) ot[e] = __float_as_uint(__uint_as_float(ot[e]) * alpha);
              }
              ptx::tmem_st32(t_row + C::O_COL + c * 32, om);
              if (ot_valid) ptx::tmem_st32(t_row + C::OT_COL + c * 32, ot);
            }
          }
        }
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&bars->p_full[g & 1]);
      }
      }
      // ---- epilogue: O * 2^-ev / l -> fp32 row, padding rows zero (attention.py:203-206)
      ptx::mbar_wait(&bars->o_full, it & 1);
      ptx::tc_fence_after();
      const float inv = (live && T > 0) ? pow2(-ev) / l_run : 0.f;
      float* orow = o + (int64_t)h * s.sh + ((int64_t)qb * BM + row) * s.sn;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        uint32_t ov[32], ot[32];
        ptx::tmem_ld32(t_row + C::O_COL + c * 32, ov);
        if (T > 2) ptx::tmem_ld32(t_row + C::OT_COL + c * 32, ot);
        ptx::tmem_wait_ld();
        if (T > 2) {
#pragma unroll
          for (int e = 0; e < 32; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) + __uint_as_float(ot[e]));
        }
        float4* dst = reinterpret_cast<float4*>(orow + c * 32);
#pragma unroll
        for (int e = 0; e < 8; ++e)
          __stcs(dst + e, live ? make_float4(__uint_as_float(ov[4 * e]) * inv, __uint_as_float(ov[4 * e + 1]) * inv,
                                             __uint_as_float(ov[4 * e + 2]) * inv, __uint_as_float(ov[4 * e + 3]) * inv)
                               : make_float4(0.f, 0.f, 0.f, 0.f));
      }
      ptx::tc_fence_before();
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<C::TMEM_COLS>(tmem);
  }
}

}  // namespace x3

// (2H, N_pad, D) fp16 stacks of K and V + the per-(tensor, head) max words
static int64_t x3_workspace_bytes(int H, int64_t n_pad, int d) {
  const int64_t plane = (int64_t)2 * H * n_pad * d * 2;
  return 2 * plane + 256 + (int64_t)2 * H * 4;
}

template <int D>
static int launch_x3(const float* q, const float* k, const float* v, float* o, const CarveShape& s,
                     const uint32_t* bits, const int32_t* kv_cnt, float beta, void* ws, int32_t* work,
                     cudaStream_t st) {
  using C = x3::Cfg<D>;
  const int64_t n_pad = (int64_t)s.M_total * s.m;
  const int64_t plane = (int64_t)2 * s.H * n_pad * D * 2;
  __half* kst = reinterpret_cast<__half*>(ws);
  __half* vst = reinterpret_cast<__half*>(reinterpret_cast<uint8_t*>(ws) + plane);
  uint32_t* amax = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(ws) + 2 * plane + 256);
  cudaError_t e = cudaMemsetAsync(amax, 0, (size_t)2 * s.H * 4, st);
  if (e != cudaSuccess) return set_error(TCB_ECUDA, "memset amax: %s", cudaGetErrorString(e));
  e = cudaMemsetAsync(work, 0, sizeof(int32_t), st);
  if (e != cudaSuccess) return set_error(TCB_ECUDA, "memset counter: %s", cudaGetErrorString(e));
  const int rows = 64;
  const dim3 pg((unsigned)((n_pad + rows - 1) / rows), (unsigned)s.H, 2);
  x3::k_kv_absmax<D><<<pg, 256, 0, st>>>(k, v, s, rows, amax);
  int rc = check_launch("k_kv_absmax");
  if (rc) return rc;
  x3::k_kv_split<D><<<pg, 256, 0, st>>>(k, v, s, rows, amax, kst, vst);
  if ((rc = check_launch("k_kv_split"))) return rc;
  CUtensorMap tk, tv;
  if ((rc = make_tmap(&tk, kst, D, n_pad, 2 * s.H, n_pad * D, D, x3::HN, true))) return rc;
  if ((rc = make_tmap(&tv, vst, D, n_pad, 2 * s.H, n_pad * D, D, x3::HN, true))) return rc;
  static std::atomic<uint64_t> attr{0};
  e = once_per_device(attr, [&] {
    return cudaFuncSetAttribute(x3::k_carve_x3<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                C::BYTES);
  });
  if (e != cudaSuccess) return set_error(TCB_ECUDA, "x3 smem attr: %s", cudaGetErrorString(e));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int total = s.H * s.M_total;
  const int grid = sms < total ? sms : total;
  const float LOG2E = 1.4426950408889634f;
  const float scale_log2 = (float)(1.0 / sqrt((double)s.d)) * LOG2E;
  x3::k_carve_x3<D><<<grid, x3::NUM_THREADS, C::BYTES, st>>>(q, tk, tv, o, s, bits, kv_cnt, amax, work,
                                                              total, scale_log2, beta * LOG2E);
  return check_launch("k_carve_x3");
}

}  // namespace tcb

using namespace tcb;

extern "C" int64_t tcb_carve_f32_workspace_bytes(int H, int M_total, int m, int d) {
  if (H < 1 || M_total < 1 || m != 128 || (d != 64 && d != 128)) return 0;
  return x3_workspace_bytes(H, (int64_t)M_total * m, d);
}

// defined in carve.cu: the fp32 SIMT / tiled path (any m, d)
extern "C" int tcb_carve_fwd_simt(const void* q, const void* k, const void* v, void* o, int dtype,
                                  int64_t stride_h, int64_t stride_n, const uint32_t* bits,
                                  int words, const int32_t* kv_cnt, int H, int d, int m, int M_v,
                                  int M_total, int64_t n_valid, int64_t n_cond, float beta,
                                  void* stream);

extern "C" int tcb_carve_fwd_f32(const float* q, const float* k, const float* v, float* o,
                                 int64_t stride_h, int64_t stride_n, const uint32_t* bits, int words,
                                 const int32_t* kv_cnt, int H, int d, int m, int M_v, int M_total,
                                 int64_t n_valid, int64_t n_cond, float beta, void* workspace,
                                 int64_t workspace_bytes, int32_t* work, void* stream) {
  const int64_t need = tcb_carve_f32_workspace_bytes(H, M_total, m, d);
  const bool aligned = ((uintptr_t)q % 16 == 0) && ((uintptr_t)k % 16 == 0) &&
                       ((uintptr_t)v % 16 == 0) && ((uintptr_t)o % 16 == 0) &&
                       (stride_n * 4) % 16 == 0 && (stride_h * 4) % 16 == 0 &&
                       ((uintptr_t)workspace % 256 == 0);
  if (need == 0 || !workspace || workspace_bytes < need || !work || M_v == 0 || !aligned)
    return tcb_carve_fwd_simt(q, k, v, o, TCB_F32, stride_h, stride_n, bits, words, kv_cnt, H, d, m,
                              M_v, M_total, n_valid, n_cond, beta, stream);
  CarveShape s{H, d, m, M_v, M_total, words, n_valid, n_cond, stride_h, stride_n};
  TCB_CHECK_ARG(q && k && v && o && bits && kv_cnt, TCB_ESHAPE, "null argument");
  TCB_CHECK_ARG(M_total >= M_v && words >= (M_total + 31) / 32, TCB_ESHAPE, "bad carve shape");
  TCB_CHECK_ARG((int64_t)H * M_total < (int64_t)1 << 31, TCB_ESIZE, "too many work items");
  cudaStream_t st = as_stream(stream);
  return d == 128 ? launch_x3<128>(q, k, v, o, s, bits, kv_cnt, beta, workspace, work, st)
                  : launch_x3<64>(q, k, v, o, s, bits, kv_cnt, beta, workspace, work, st);
}
