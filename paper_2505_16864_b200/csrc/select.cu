// K3 block pool, K4 pooled relevance, K5+K6 selection/union, mask pack/unpack.
//
// K3  tcb_block_pool       <- block_pool        masks.py:98-116   (HBM bound)
// K4  tcb_block_relevance  <- relevance         masks.py:119-134  (fp64 FMA bound)
// K5  tcb_block_select     <- importance_mask   masks.py:137-159
//     (+ union)            <- union_mask        masks.py:162-175
#include <algorithm>

#include "common.cuh"

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <math.h>
#include <stdlib.h>

namespace tcb {

// ---------------------------------------------------------------------------
// K3 block pool.  A group of G threads owns one (head, block); thread j of the
// group owns columns chunk j (VE elements = one 16-byte vector) and sums the
// block's valid rows sequentially in float64 -- the same ascending-row order
// numpy uses for the axis-2 reduction of masks.py:112, so the pooled means are
// bit-exact.  Rows of consecutive lanes are contiguous -> coalesced 16B loads.
// ---------------------------------------------------------------------------
template <typename T>
struct Vec16;
template <>
struct Vec16<float> {
  static constexpr int VE = 4;
  __device__ static void load(const float* p, double* o) {
    float4 v = __ldcs(reinterpret_cast<const float4*>(p));
    o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
  }
};
template <>
struct Vec16<double> {
  static constexpr int VE = 2;
  __device__ static void load(const double* p, double* o) {
    double2 v = __ldcs(reinterpret_cast<const double2*>(p));
    o[0] = v.x; o[1] = v.y;
  }
};
template <>
struct Vec16<__nv_bfloat16> {
  static constexpr int VE = 8;
  __device__ static void load(const __nv_bfloat16* p, double* o) {
    int4 v = __ldcs(reinterpret_cast<const int4*>(p));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 f = __bfloat1622float2(h[i]);
      o[2 * i] = f.x;
      o[2 * i + 1] = f.y;
    }
  }
};

template <>
struct Vec16<__half> {
  static constexpr int VE = 8;
  __device__ static void load(const __half* p, double* o) {
    int4 v = __ldcs(reinterpret_cast<const int4*>(p));
    const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 f = __half22float2(h[i]);
      o[2 * i] = f.x;
      o[2 * i + 1] = f.y;
    }
  }
};

template <typename T>
__device__ __forceinline__ double to_f64(T x) { return (double)(float)x; }
template <>
__device__ __forceinline__ double to_f64<double>(double x) { return x; }

template <typename T, bool VEC>
__global__ void __launch_bounds__(128) k_pool(const T* __restrict__ x0, const T* __restrict__ x1,
                                              int64_t sh, int64_t sn, int H, int d, int m, int M_v,
                                              int M_total, int64_t n_valid, int64_t n_cond,
                                              double* __restrict__ o0, double* __restrict__ o1,
                                              int G, int chunks) {
  constexpr int VE = VEC ? Vec16<T>::VE : 1;
  const T* x = blockIdx.y ? x1 : x0;
  double* o = blockIdx.y ? o1 : o0;
  const int per_cta = blockDim.x / G;
  const int g = threadIdx.x / G;
  const int j = threadIdx.x - g * G;
  const int64_t item = (int64_t)blockIdx.x * per_cta + g;
  if (g >= per_cta || item >= (int64_t)H * M_total) return;
  const int h = (int)(item / M_total);
  const int b = (int)(item - (int64_t)h * M_total);
  const int cnt = block_valid(b, m, M_v, n_valid, n_cond);
  const double inv = 1.0 / (double)(cnt > 0 ? cnt : 1);
  (void)inv;
  const T* base = x + (int64_t)h * sh + (int64_t)b * m * sn;
  double* out = o + ((int64_t)h * M_total + b) * d;
  for (int c = j; c < chunks; c += G) {
    double acc[VE];
#pragma unroll
    for (int e = 0; e < VE; ++e) acc[e] = 0.0;
    const T* p = base + (int64_t)c * VE;
    int r = 0;
    // 4 rows of loads in flight per thread; adds stay in ascending row order
    for (; r + 4 <= cnt; r += 4) {
      double v[4][VE];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if constexpr (VEC) {
          Vec16<T>::load(p + (int64_t)(r + u) * sn, v[u]);
        } else {
          v[u][0] = to_f64(p[(int64_t)(r + u) * sn]);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int e = 0; e < VE; ++e) acc[e] += v[u][e];
    }
    for (; r < cnt; ++r) {
      double v[VE];
      if constexpr (VEC) {
        Vec16<T>::load(p + (int64_t)r * sn, v);
      } else {
        v[0] = to_f64(p[(int64_t)r * sn]);
      }
#pragma unroll
      for (int e = 0; e < VE; ++e) acc[e] += v[e];
    }
    // masks.py:115 divides the float64 sums by max(count, 1)
    const double den = (double)(cnt > 0 ? cnt : 1);
#pragma unroll
    for (int e = 0; e < VE; ++e) out[c * VE + e] = acc[e] / den;
  }
}

// ---------------------------------------------------------------------------
// K4 relevance: R[h,i,:] = softmax(pq_i . pk_j / sqrt(d)) in float64, two launches:
//  * k_scores: 64x64 output tiles per CTA, 4x4 register tile per thread, 32-wide d
//    chunks of pq/pk staged transposed in smem; writes pq.pk / sqrt(d) (the
//    reference divides after the product, masks.py:130-131);
//  * k_row_softmax: one warp per row -- max, exp, numpy-pairwise sum, divide
//    (masks.py:132-134), coalesced over the row.
// ---------------------------------------------------------------------------
constexpr int ST_TILE = 64;
constexpr int ST_KC = 32;

// numpy's pairwise summation (PW_BLOCKSIZE 128, 8-way unrolled leaves): the
// recursion splits n > 128 at n2 = n/2 - (n/2)%8 and sums left + right.  The leaves
// (contiguous runs of <= 128) are independent, so a warp sums them in parallel and
// lane 0 folds the leaf sums in the recursion's order.
constexpr int PW_MAX_LEAVES = 256;  // enough for n <= 16384
constexpr int SEL_MAX_LEAVES = 128;  // k_select: M_total <= 8192 -> <= 128 leaves of >= 64

__device__ __forceinline__ double pw_leaf(const double* p, int len) {
  if (len < 8) {
    double res = 0.0;
    for (int i = 0; i < len; ++i) res += p[i];
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = p[j];
  int i = 8;
  for (; i < len - (len % 8); i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] += p[i + j];
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < len; ++i) res += p[i];
  return res;
}

// Leaves of the pairwise tree of n in left-to-right order; returns their count.
__host__ __device__ int pw_leaves(int n, int* off, int* len) {
  int st_off[32], st_len[32], sp = 0, nl = 0;
  st_off[sp] = 0; st_len[sp] = n; ++sp;
  while (sp) {
    --sp;
    const int o = st_off[sp], l = st_len[sp];
    if (l <= 128) {
      off[nl] = o; len[nl] = l; ++nl;
      continue;
    }
    int n2 = l / 2;
    n2 -= n2 % 8;
    st_off[sp] = o + n2; st_len[sp] = l - n2; ++sp;  // right pushed first, popped second
    st_off[sp] = o; st_len[sp] = n2; ++sp;
  }
  return nl;
}

// Fold leaf sums in the recursion order: value(node) = value(left) + value(right).
__device__ double pw_fold(int n, const double* leaf) {
  int st_len[32], st_state[32], sp = 0, next = 0;
  double st_val[32], ret = 0.0;
  st_len[0] = n; st_state[0] = 0; sp = 1;
  while (sp) {
    const int top = sp - 1;
    if (st_state[top] == 0 && st_len[top] > 128) {  // descend left
      int n2 = st_len[top] / 2;
      n2 -= n2 % 8;
      st_state[top] = 1;
      st_len[sp] = n2; st_state[sp] = 0; ++sp;
      continue;
    }
    if (st_state[top] == 0) {  // leaf
      ret = leaf[next++];
      --sp;
    } else if (st_state[top] == 1) {  // left done -> descend right
      int n2 = st_len[top] / 2;
      n2 -= n2 % 8;
      st_val[top] = ret;
      st_state[top] = 2;
      st_len[sp] = st_len[top] - n2; st_state[sp] = 0; ++sp;
      continue;
    } else {  // right done
      ret = st_val[top] + ret;
      --sp;
    }
    // propagate completed child values upward happens via the loop
  }
  return ret;
}

// Whole-row pairwise sum by one warp: lane 0 enumerates the leaves into the warp's
// scratch, lanes sum leaves in parallel, lane 0 folds.  scratch: PW_MAX_LEAVES doubles
// followed by 2*PW_MAX_LEAVES ints.
// The fold as a straight-line program over value slots: leaves occupy slots [0, nl),
// internal node i (post-order, the order pw_fold evaluates them) writes slot nl + i =
// slot a_i + slot b_i.  Built once per CTA (the tree depends only on n), executed per
// row by one lane with no stack -- bitwise the pw_fold result.
__host__ __device__ int pw_program(int n, int nl, int2* ops) {
  int st_len[32], st_state[32], st_left[32], sp = 1, ret = -1, leafc = 0, nops = 0;
  st_len[0] = n;
  st_state[0] = 0;
  while (sp) {
    const int top = sp - 1;
    int n2 = st_len[top] / 2;
    n2 -= n2 % 8;
    if (st_state[top] == 0 && st_len[top] > 128) {
      st_state[top] = 1;
      st_len[sp] = n2; st_state[sp] = 0; ++sp;
    } else if (st_state[top] == 0) {
      ret = leafc++;
      --sp;
    } else if (st_state[top] == 1) {
      st_left[top] = ret;
      st_state[top] = 2;
      st_len[sp] = st_len[top] - n2; st_state[sp] = 0; ++sp;
    } else {
      ops[nops] = make_int2(st_left[top], ret);
      ret = nl + nops++;
      --sp;
    }
  }
  return nops;
}

__device__ double warp_pairwise_sum(const double* row, int n, double* scratch) {
  const int lane = threadIdx.x & 31;
  double* leaf = scratch;
  int* off = reinterpret_cast<int*>(scratch + PW_MAX_LEAVES);
  int* len = off + PW_MAX_LEAVES;
  int nl = 0;
  if (lane == 0) nl = pw_leaves(n, off, len);
  nl = __shfl_sync(0xffffffffu, nl, 0);
  __syncwarp();
  for (int i = lane; i < nl; i += 32) leaf[i] = pw_leaf(row + off[i], len[i]);
  __syncwarp();
  double total = 0.0;
  if (lane == 0) total = pw_fold(n, leaf);
  total = __shfl_sync(0xffffffffu, total, 0);
  __syncwarp();
  return total;
}

__global__ void __launch_bounds__(256) k_scores(const double* __restrict__ pq, int pq_blocks,
                                                const double* __restrict__ pk, int rows,
                                                int M_total, int d, double sqrt_d,
                                                double* __restrict__ R) {
  __shared__ double sA[ST_KC][ST_TILE + 1];
  __shared__ double sB[ST_KC][ST_TILE + 1];
  const int h = blockIdx.z;
  const int r0 = blockIdx.y * ST_TILE, c0 = blockIdx.x * ST_TILE;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const double* A = pq + (int64_t)h * pq_blocks * d;
  const double* B = pk + (int64_t)h * M_total * d;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int k0 = 0; k0 < d; k0 += ST_KC) {
    // coalesced along d, stored transposed (k-major) for the inner product loop
    for (int e = tid; e < ST_TILE * ST_KC; e += 256) {
      const int rr = e / ST_KC, kk = e - rr * ST_KC;
      const int gk = k0 + kk;
      const int gr = r0 + rr, gc = c0 + rr;
      sA[kk][rr] = (gr < rows && gk < d) ? A[(int64_t)gr * d + gk] : 0.0;
      sB[kk][rr] = (gc < M_total && gk < d) ? B[(int64_t)gc * d + gk] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < ST_KC; ++kk) {
      double a[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sA[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = sB[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  double* Rh = R + (int64_t)h * rows * M_total;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gr = r0 + ty + 16 * i;
    if (gr >= rows) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gc = c0 + tx + 16 * j;
      if (gc < M_total) Rh[(int64_t)gr * M_total + gc] = acc[i][j] / sqrt_d;
    }
  }
}

// Same product on the FP64 tensor core (DMMA.8x8x4, mma.sync m8n8k4 f64): warp tile
// 32 x 32 (4 x 4 MMA tiles, 32 fp64 accumulators per thread), CTA = 2 x 2 warps, operand
// fragments read straight from L1/L2 (pq/pk are 11 MB each, L2-resident).
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(128) k_scores_dmma(const double* __restrict__ pq, int pq_blocks,
                                                     const double* __restrict__ pk, int rows,
                                                     int M_total, int d, double sqrt_d,
                                                     double* __restrict__ R) {
  const int h = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = blockIdx.y * 64 + (warp >> 1) * 32;
  const int c0 = blockIdx.x * 64 + (warp & 1) * 32;
  const double* A = pq + (int64_t)h * pq_blocks * d;
  const double* B = pk + (int64_t)h * M_total * d;
  const int fr = lane >> 2, fk = lane & 3;
  const double* ap[4];
  const double* bp[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    ap[i] = A + (int64_t)min(r0 + 8 * i + fr, pq_blocks - 1) * d + fk;
    bp[i] = B + (int64_t)min(c0 + 8 * i + fr, M_total - 1) * d + fk;
  }
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll 4
  for (int k = 0; k < d; k += 4) {
    double a[4], b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      a[i] = __ldg(ap[i] + k);
      b[i] = __ldg(bp[i] + k);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
  }
  double* Rh = R + (int64_t)h * rows * M_total;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gr = r0 + 8 * i + fr;
    if (gr >= rows) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int gc = c0 + 8 * j + 2 * fk + e;
        if (gc < M_total) Rh[(int64_t)gr * M_total + gc] = acc[i][j][e] / sqrt_d;
      }
    }
  }
}

__global__ void __launch_bounds__(256) k_row_softmax(double* __restrict__ R, int64_t n_rows,
                                                     int M_total) {
  __shared__ double sbuf[8 * 2 * PW_MAX_LEAVES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * 8 + warp;
  if (r >= n_rows) return;
  double* row = R + r * M_total;
  double mx = -INFINITY;
  for (int j = lane; j < M_total; j += 32) mx = fmax(mx, row[j]);
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  for (int j = lane; j < M_total; j += 32) row[j] = exp(row[j] - mx);
  __syncwarp();
  const double ssum = warp_pairwise_sum(row, M_total, sbuf + warp * 2 * PW_MAX_LEAVES);
  for (int j = lane; j < M_total; j += 32) row[j] = row[j] / ssum;
}

// ---------------------------------------------------------------------------
// K5 selection.  CTA per (head, vision row).  The reference sorts the whole row
// (stable descending argsort, masks.py:150), takes the sequential float64 prefix
// (np.cumsum, masks.py:152), counts prefix <= p and keeps the first
// n_keep = min(max(n_cut, n_floor), n_cols) sorted columns.  Only two things are
// really needed: the exact sorted prefix up to where it first exceeds p, and the
// top-n_keep set under the (value desc, column asc) order.  So:
//   * columns get an order-preserving 64-bit key (ascending key == descending value)
//     and the total order is (key, column);
//   * MSB-first radix select (8-bit digits, smem histograms) finds the top-K set of
//     that order for any K without sorting;
//   * for p > 0 the top min(512, n) columns are radix-selected, sorted in registers
//     (warp bitonic) and scanned with the exact sequential prefix; when the prefix
//     cannot cross p inside that window the whole row is sorted in shared memory;
//     p == 0 needs no sort at all (n_cut = 1 when the row max is > 0);
//   * rows with negative entries (never produced by relevance) use a full sort.
// The top-n_keep columns are ORed with the condition columns and the adjacency row
// (masks.py:173-174) and emitted packed and as an ascending CSR kv list.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t desc_key(double v) {
  if (v == 0.0) v = 0.0;  // -0.0 == 0.0 for argsort
  uint64_t b = (uint64_t)__double_as_longlong(v);
  uint64_t asc = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
  return ~asc;  // ascending key == descending value
}
__device__ __forceinline__ double key_value(uint64_t k) {
  uint64_t asc = ~k;
  uint64_t b = (asc >> 63) ? (asc & 0x7fffffffffffffffull) : ~asc;
  return __longlong_as_double((long long)b);
}

// The pairwise-sum tree of a row depends only on M_total: built once on the host per launch
// and passed by value (it used to be built by thread 0 of every CTA while the CTA waited).
struct PwProg {
  int nl, nops;
  int off[SEL_MAX_LEAVES], len[SEL_MAX_LEAVES];
  int2 ops[SEL_MAX_LEAVES];
};

// Sort-buffer entries per warp of the complete / exact passes: the shared-memory sort needs
// the row's power of two (>= the 544-slot register-window staging), and rows of <= 1024
// columns stage their register-sorted keys with one pad slot per 32 (33 x 32 entries).
__host__ __device__ constexpr int sel_full_sort(int np2, int M_total) {
  return (np2 > 544 ? np2 : 544) < 1056 && M_total <= 1024 ? 1056 : (np2 > 544 ? np2 : 544);
}

// ---- warp-per-row selection ------------------------------------------------------
constexpr int SW_WARPS = 4;  // rows (one warp each) per CTA
constexpr unsigned FULL = 0xffffffffu;

struct RadixState {
  uint64_t prefix, mask;
  int remaining;  // rank still needed inside the current bin
  int binc;       // elements in the chosen bin
};

// MSB-first radix select over the (key, column) order of keys[0, n) by one warp: the
// top-K set is {(key & mask) < prefix} U {first `remaining` columns with
// (key & mask) == prefix}.  Bytes on which every key agrees (the sign/exponent bytes of a
// row of probabilities) cannot split the candidates; they are folded into the prefix
// without a histogram pass (AND/OR of all keys finds them).
__device__ RadixState warp_radix(const uint64_t* keys, int n, int K, uint32_t* hist) {
  const int lane = threadIdx.x & 31;
  RadixState r{0ull, 0ull, K, 0};
  uint64_t kand = ~0ull, kor = 0ull;
  for (int j = lane; j < n; j += 32) {
    const uint64_t k = keys[j];
    kand &= k;
    kor |= k;
  }
  {
    const uint32_t al = __reduce_and_sync(FULL, (uint32_t)kand), ah = __reduce_and_sync(FULL, (uint32_t)(kand >> 32));
    const uint32_t ol = __reduce_or_sync(FULL, (uint32_t)kor), oh = __reduce_or_sync(FULL, (uint32_t)(kor >> 32));
    kand = ((uint64_t)ah << 32) | al;
    kor = ((uint64_t)oh << 32) | ol;
  }
  for (int byte = 7; byte >= 0; --byte) {
    const int sh = byte * 8;
    if ((((kand ^ kor) >> sh) & 0xFFull) == 0ull) {
      r.prefix |= kand & (0xFFull << sh);
      r.mask |= 0xFFull << sh;
      continue;
    }
    for (int i = lane; i < 256; i += 32) hist[i] = 0u;
    __syncwarp();
    for (int j = lane; j < n; j += 32) {
      const uint64_t k = keys[j];
      if ((k & r.mask) == r.prefix) atomicAdd(&hist[(int)((k >> sh) & 0xFF)], 1u);
    }
    __syncwarp();
    uint32_t c[8];
    uint32_t ct = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      c[i] = hist[lane * 8 + i];
      ct += c[i];
    }
    uint32_t cin = ct;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, cin, o);
      if (lane >= o) cin += y;
    }
    uint32_t cex = cin - ct;
    const bool hit = (cex < (uint32_t)r.remaining) && ((uint32_t)r.remaining <= cin);
    const unsigned bal = __ballot_sync(FULL, hit);
    const int src = __ffs(bal) - 1;
    int bin = 7;
    uint32_t binc = 0;
    if (lane == src) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {  // unrolled: c[] stays in registers
        if (bin == 7 && i < 7 && (uint32_t)r.remaining <= cex + c[i]) {
          bin = i;
          binc = c[i];
        } else if (bin == 7 && i < 7) {
          cex += c[i];
        }
      }
      if (bin == 7) binc = c[7];
    }
    const int dg = __shfl_sync(FULL, src * 8 + bin, src);
    const uint32_t before = __shfl_sync(FULL, cex, src);
    binc = __shfl_sync(FULL, binc, src);
    r.prefix |= (uint64_t)dg << sh;
    r.mask |= 0xFFull << sh;
    r.binc = (int)binc;
    r.remaining -= (int)before;
    if ((int)binc == r.remaining) return r;  // whole bin selected
    __syncwarp();
  }
  return r;
}

// Visit the top-K set of `r` in ascending column order: fn(j, slot).
template <typename F>
__device__ void warp_topk_visit(const uint64_t* keys, int n, const RadixState& r, F fn) {
  const int lane = threadIdx.x & 31;
  int eq_base = 0, slot_base = 0;
  for (int j0 = 0; j0 < n; j0 += 32) {
    const int j = j0 + lane;
    uint64_t km = ~0ull;
    if (j < n) km = keys[j] & r.mask;
    const bool eq = (j < n) && km == r.prefix;
    const unsigned eqb = __ballot_sync(FULL, eq);
    const int eq_rank = eq_base + __popc(eqb & ((1u << lane) - 1u));
    const bool sel = (j < n) && (km < r.prefix || (eq && eq_rank < r.remaining));
    const unsigned selb = __ballot_sync(FULL, sel);
    if (sel) fn(j, slot_base + __popc(selb & ((1u << lane) - 1u)));
    eq_base += __popc(eqb);
    slot_base += __popc(selb);
  }
}

__device__ void warp_bitonic(uint64_t* key, int* col, int np2) {
  const int lane = threadIdx.x & 31;
  for (int kk = 2; kk <= np2; kk <<= 1) {
    for (int jj = kk >> 1; jj > 0; jj >>= 1) {
      for (int t = lane; t < (np2 >> 1); t += 32) {
        const int a = ((t & ~(jj - 1)) << 1) | (t & (jj - 1));
        const int b = a + jj;
        const bool up = (a & kk) == 0;
        const uint64_t ka = key[a], kb = key[b];
        const int ca = col[a], cb = col[b];
        const bool a_gt_b = (ka > kb) || (ka == kb && ca > cb);
        if (a_gt_b == up) {
          key[a] = kb; key[b] = ka;
          col[a] = cb; col[b] = ca;
        }
      }
      __syncwarp();
    }
  }
}

// Register bitonic sort of up to 512 (key, col) pairs by one warp: element e = 16*lane + r
// lives in lane `lane`, register r.  Strides < 16 are in-register compare-exchanges,
// strides >= 16 pair lane with lane ^ (stride / 16) through shuffles -- no shared memory,
// no __syncwarp, full ILP.  Ascending (key, col) order == the reference's stable
// descending argsort.
struct KC {
  uint64_t k;
  int c;
};
__device__ __forceinline__ bool kc_less(const KC& a, const KC& b) {
  return a.k < b.k || (a.k == b.k && a.c < b.c);
}

template <int KK, int JJ>
__device__ __forceinline__ void reg_bitonic_stage(KC (&x)[16], int lane) {
  if constexpr (JJ >= 16) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const int e = lane * 16 + r;
      KC o;
      o.k = __shfl_xor_sync(FULL, x[r].k, JJ >> 4);
      o.c = __shfl_xor_sync(FULL, x[r].c, JJ >> 4);
      const bool up = (e & KK) == 0, lower = (e & JJ) == 0;
      const bool take_o = (up == lower) ? kc_less(o, x[r]) : kc_less(x[r], o);
      if (take_o) x[r] = o;
    }
  } else {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (r & JJ) continue;
      const bool up = ((lane * 16 + r) & KK) == 0;
      if (kc_less(x[r | JJ], x[r]) == up) {
        const KC t = x[r];
        x[r] = x[r | JJ];
        x[r | JJ] = t;
      }
    }
  }
  if constexpr (JJ > 1) reg_bitonic_stage<KK, JJ / 2>(x, lane);
}

template <int KK>
__device__ __forceinline__ void reg_bitonic_level(KC (&x)[16], int lane) {
  reg_bitonic_stage<KK, KK / 2>(x, lane);
  if constexpr (KK < 512) reg_bitonic_level<KK * 2>(x, lane);
}

__device__ __forceinline__ void reg_bitonic512(KC (&x)[16]) {
  reg_bitonic_level<2>(x, threadIdx.x & 31);
}

// The same network on packed 64-bit (key, col) words: when every key of the window shares
// its top `colbits` bits (one binade of probabilities does: sign + exponent), the column
// fits below the key's remaining bits and one unsigned compare orders (key, col) exactly.
template <int KK, int JJ>
__device__ __forceinline__ void reg_bitonic_stage_u(uint64_t (&y)[16], int lane) {
  if constexpr (JJ >= 16) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const int e = lane * 16 + r;
      const uint64_t o = __shfl_xor_sync(FULL, y[r], JJ >> 4);
      const bool up = (e & KK) == 0, lower = (e & JJ) == 0;
      const bool take_o = (up == lower) ? (o < y[r]) : (y[r] < o);
      if (take_o) y[r] = o;
    }
  } else {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (r & JJ) continue;
      const bool up = ((lane * 16 + r) & KK) == 0;
      if ((y[r | JJ] < y[r]) == up) {
        const uint64_t t = y[r];
        y[r] = y[r | JJ];
        y[r | JJ] = t;
      }
    }
  }
  if constexpr (JJ > 1) reg_bitonic_stage_u<KK, JJ / 2>(y, lane);
}

template <int KK>
__device__ __forceinline__ void reg_bitonic_level_u(uint64_t (&y)[16], int lane) {
  reg_bitonic_stage_u<KK, KK / 2>(y, lane);
  if constexpr (KK < 512) reg_bitonic_level_u<KK * 2>(y, lane);
}

// Keys only, R per lane (element e = R * lane + r): ascending 64-bit keys -- what the exact
// prefix scan needs (equal keys are equal values, so their order cannot change a sum).
template <int R, int KK, int JJ>
__device__ __forceinline__ void keys_bitonic_stage(uint64_t (&y)[R], int lane) {
  if constexpr (JJ >= R) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int e = lane * R + r;
      const uint64_t o = __shfl_xor_sync(FULL, y[r], JJ / R);
      const bool up = (e & KK) == 0, lower = (e & JJ) == 0;
      const bool take_o = (up == lower) ? (o < y[r]) : (y[r] < o);
      if (take_o) y[r] = o;
    }
  } else {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (r & JJ) continue;
      const bool up = ((lane * R + r) & KK) == 0;
      if ((y[r | JJ] < y[r]) == up) {
        const uint64_t t = y[r];
        y[r] = y[r | JJ];
        y[r | JJ] = t;
      }
    }
  }
  if constexpr (JJ > 1) keys_bitonic_stage<R, KK, JJ / 2>(y, lane);
}

template <int R, int KK>
__device__ __forceinline__ void keys_bitonic_level(uint64_t (&y)[R], int lane) {
  keys_bitonic_stage<R, KK, KK / 2>(y, lane);
  if constexpr (KK < 32 * R) keys_bitonic_level<R, KK * 2>(y, lane);
}

// Sort the window x[16] (cnt real entries, the rest padding ~0 / INT_MAX) by (key, col);
// packed single-word compares when the keys leave room for the column, KC compares otherwise.
__device__ __forceinline__ void reg_sort_window(KC (&x)[16], int cnt, int M_total) {
  const int lane = threadIdx.x & 31;
  uint64_t kand = ~0ull, kor = 0ull;
#pragma unroll
  for (int r = 0; r < 16; ++r)
    if (lane * 16 + r < cnt) {
      kand &= x[r].k;
      kor |= x[r].k;
    }
  const uint32_t al = __reduce_and_sync(FULL, (uint32_t)kand), ah = __reduce_and_sync(FULL, (uint32_t)(kand >> 32));
  const uint32_t ol = __reduce_or_sync(FULL, (uint32_t)kor), oh = __reduce_or_sync(FULL, (uint32_t)(kor >> 32));
  kand = ((uint64_t)ah << 32) | al;
  kor = ((uint64_t)oh << 32) | ol;
  const int colbits = M_total > 1 ? 32 - __clz(M_total - 1) : 0;
  const uint64_t diff = kand ^ kor;
  const int lead = diff ? __clzll((long long)diff) : 64;
  if (lead < colbits) {
    reg_bitonic512(x);
    return;
  }
  const uint64_t cmask = colbits ? (~0ull >> (64 - colbits)) : 0ull;
  const uint64_t top = colbits ? (kand & ~(~0ull >> colbits)) : 0ull;
  uint64_t y[16];
#pragma unroll
  for (int r = 0; r < 16; ++r)
    y[r] = (lane * 16 + r < cnt) ? ((x[r].k << colbits) | (uint64_t)x[r].c) : ~0ull;
  reg_bitonic_level_u<2>(y, lane);
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    x[r].k = top | (y[r] >> colbits);
    x[r].c = (int)(y[r] & cmask);
  }
}

// Exact np.cumsum scan of the sorted values: the sorted keys go back to the (padded)
// staging buffer and lane 0 runs the dependent float64 add chain over them (loads
// software-pipelined by the unrolled loop); returns 1 + #(prefix <= p), stopping at the
// first crossing (the prefix of non-negative values is monotone).
__device__ int reg_sorted_cut(const KC (&x)[16], uint64_t* stage, int cnt, double p,
                              bool* crossed) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int r = 0; r < 16; ++r) stage[lane * 17 + r] = x[r].k;
  __syncwarp();
  int c = 0;
  bool cr = false;
  if (lane == 0) {
    double pre = 0.0;
#pragma unroll 8
    for (int t = 0; t < cnt; ++t) {
      pre = __dadd_rn(pre, key_value(stage[t + (t >> 4)]));  // np.cumsum order (masks.py:152)
      if (pre > p) {
        cr = true;
        break;
      }
      ++c;
    }
  }
  *crossed = __shfl_sync(FULL, (int)cr, 0) != 0;
  return __shfl_sync(FULL, c, 0) + 1;
}

// The crossing rank of the exact sequential prefix (np.cumsum, masks.py:152) without the
// dependent fp64 chain when possible.  Sorted keys are held R per lane (element e = R lane + r);
// a warp-parallel prefix (in-lane sums + a shuffle scan) differs from the sequential one by
// at most ~(e + R + 5) u S_e for non-negative values (u = 2^-53), far below a 1e-12
// relative margin, so every prefix outside that margin around p compares exactly as the
// sequential one does.  Returns 1 + #(prefix <= p) (and *crossed), or -1 when some prefix
// lies inside the margin -- the caller then replays the sequential chain.
template <int R, typename KeyOf>
__device__ __forceinline__ int par_cut(KeyOf key_of, int cnt, double p, bool* crossed) {
  const int lane = threadIdx.x & 31;
  double tot = 0.0;
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (lane * R + r < cnt) tot += key_value(key_of(r));
  double inc = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(FULL, inc, o);
    if (lane >= o) inc += y;
  }
  double pre = __shfl_up_sync(FULL, inc, 1);
  if (lane == 0) pre = 0.0;
  int first = 0x7fffffff;
  bool amb = false;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int e = lane * R + r;
    if (e < cnt && first == 0x7fffffff) {
      pre += key_value(key_of(r));
      const double m = 1e-12 * pre;
      if (pre > p - m) {
        first = e;
        amb = !(pre - m > p);
      }
    }
  }
  int f = first;
#pragma unroll
  for (int o = 16; o; o >>= 1) f = min(f, __shfl_xor_sync(FULL, f, o));
  if (f == 0x7fffffff) {  // every prefix certainly <= p
    *crossed = false;
    return cnt + 1;
  }
  const int src = __ffs(__ballot_sync(FULL, first == f)) - 1;
  if (__shfl_sync(FULL, (int)amb, src)) return -1;
  *crossed = true;
  return f + 1;
}

// Sort (key, col) pairs [0, cnt) of skey/scol (padded to np2) and return
// 1 + #(sequential prefix <= p) over the sorted values; *crossed reports whether the
// monotone prefix exceeded p inside the sorted window.
__device__ int warp_sorted_cut(uint64_t* skey, int* scol, int cnt, int np2, double p, bool monotone,
                               bool* crossed) {
  const int lane = threadIdx.x & 31;
  for (int j = cnt + lane; j < np2; j += 32) { skey[j] = ~0ull; scol[j] = 0x7fffffff; }
  __syncwarp();
  warp_bitonic(skey, scol, np2);
  int cut = 0;
  bool cr = false;
  if (lane == 0) {
    double pre = 0.0;
    int c = 0;
    for (int s2 = 0; s2 < cnt; ++s2) {
      pre = __dadd_rn(pre, key_value(skey[s2]));  // np.cumsum order (masks.py:152)
      if (pre <= p) ++c;
      else if (monotone) { cr = true; break; }
    }
    cut = c + 1;
  }
  *crossed = __shfl_sync(FULL, (int)cr, 0) != 0;
  return __shfl_sync(FULL, cut, 0);
}

// ---- the row program ----------------------------------------------------------------
// One warp selects one (head, vision row).  `vals` holds the row in shared memory: float64
// probabilities (RAW = false), or scaled pooled scores (RAW = true) that are first turned
// into R in place (max, exp, numpy-pairwise sum, divide; masks.py:132-134) and written back
// to Rr when Rr != nullptr.  FASTS (RAW, p == 0 only): the selection is taken on the scores
// themselves -- R = exp(S - max) / sum is monotone in S, so the top-n_floor set of R is the
// top-n_floor set of S -- unless the set's boundary is a near tie (|S_in - S_out| within
// 1e-12 of the exp argument, where exp / divide rounding could merge or swap the two values)
// or lies in exp's underflow range; such rows are marked kv_cnt = -1 for the exact pass.
// MODE 0: complete program (shared memory for a full-row sort).  MODE 1: slim main pass of
// the cutoff path -- staging for the register sort only; a row whose cut cannot be decided
// in the top-512 window (p near the row total, or negative values) is marked kv_cnt = -1.
// MODE 2: the exact pass over the marked rows only.
// Output: the packed row (union with the condition columns and the adjacency row when
// with_union) and its popcount kv_cnt -- the carve kernels walk the packed bits, so no CSR.
struct RowScratch {
  uint32_t* hist;  // 256
  uint32_t* sbits; // words_pad
  double* leaf;    // nslots
  uint64_t* skey;  // SORT: max(np2, 544) (MODE 1: 544)
  int* scol;
};

template <bool RAW, bool SORT, int MODE, bool FASTS>
__device__ void select_row(double* vals, double* __restrict__ Rr, const RowScratch& sc,
                           int64_t row, int i, int M_v, int M_total, int words, int n_floor,
                           double p, int with_union, const uint32_t* __restrict__ adja,
                           uint32_t* __restrict__ bits, int32_t* __restrict__ kv_cnt, int nl,
                           int nops, const int* leaf_off, const int* leaf_len,
                           const int2* fold_ops) {
  const int lane = threadIdx.x & 31;
  uint64_t* keys = reinterpret_cast<uint64_t*>(vals);  // keys overwrite vals in place
  uint32_t* hist = sc.hist;
  uint32_t* sbits = sc.sbits;
  double* leaf = sc.leaf;
  uint64_t* skey = sc.skey;
  int* scol = sc.scol;
  double mx = -INFINITY;
  for (int j = lane; j < M_total; j += 32) mx = fmax(mx, vals[j]);
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
  if (RAW && !FASTS) {
    for (int j = lane; j < M_total; j += 32) vals[j] = exp(vals[j] - mx);
    __syncwarp();
    for (int l = lane; l < nl; l += 32) leaf[l] = pw_leaf(vals + leaf_off[l], leaf_len[l]);
    __syncwarp();
    double tot = 0.0;
    if (lane == 0) {
      for (int q = 0; q < nops; ++q) leaf[nl + q] = leaf[fold_ops[q].x] + leaf[fold_ops[q].y];
      tot = leaf[nops ? nl + nops - 1 : 0];
    }
    tot = __shfl_sync(FULL, tot, 0);
    for (int j = lane; j < M_total; j += 32) {
      const double v = vals[j] / tot;
      if (Rr) Rr[j] = v;
      vals[j] = v;
    }
  }
  __syncwarp();
  bool neg = false, pos = false;
  for (int j = lane; j < M_total; j += 32) {
    const double v = vals[j];
    neg |= v < 0.0;
    pos |= v > 0.0;
    keys[j] = desc_key(v);
  }
  neg = __any_sync(FULL, neg);
  pos = __any_sync(FULL, pos);
  for (int w = lane; w < words; w += 32) sbits[w] = 0u;
  __syncwarp();

  // ---- n_cut = 1 + #(sorted sequential prefix <= p)  (masks.py:150-153) ----
  int n_cut;
  bool reg_bits = false;  // the register path already wrote the top-keep set
  if (FASTS) {
    n_cut = 1;  // every softmax row has a positive maximum
  } else if (!neg && p == 0.0) {
    n_cut = pos ? 1 : M_total + 1;  // prefix_0 = row max
  } else if (SORT) {
    // The register path sorts the top min(512, M_total) (one radix select) and scans them
    // exactly; it decides n_cut whenever the prefix crosses p inside that window (or the
    // window is the whole row).  Otherwise (p close to the row total, or negative values
    // from an external R) the shared-memory paths below sort as much as needed.
    const int k_ub = min(512, M_total);
    bool done = false;
    if (MODE != 2 && !neg) {
      const RadixState t = warp_radix(keys, M_total, k_ub, hist);
      uint64_t* stage_k = skey;  // staging with one pad slot per 16 (conflict-free lane reads)
      int* stage_c = scol;
      for (int e = lane; e < 512 + 32; e += 32) { stage_k[e] = ~0ull; stage_c[e] = 0x7fffffff; }
      __syncwarp();
      double part = 0.0;
      warp_topk_visit(keys, M_total, t, [&](int j, int slot) {
        stage_k[slot + (slot >> 4)] = keys[j];
        stage_c[slot + (slot >> 4)] = j;
        part += key_value(keys[j]);
      });
#pragma unroll
      for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(FULL, part, o);
      __syncwarp();
      // the (any-order) window total must exceed p by more than any summation-order
      // rounding for the exact prefix to cross inside the window
      const bool window_ok = k_ub == M_total || part > p + 1e-12 * (1.0 + part);
      if (window_ok) {
        KC x[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          x[r].k = stage_k[lane * 17 + r];
          x[r].c = stage_c[lane * 17 + r];
        }
        reg_sort_window(x, k_ub, M_total);
        bool crossed;
        __syncwarp();
        n_cut = par_cut<16>([&](int r) { return x[r].k; }, k_ub, p, &crossed);
        if (n_cut < 0) n_cut = reg_sorted_cut(x, stage_k, k_ub, p, &crossed);
        if (crossed || k_ub == M_total) {
          done = true;
          const int reg_keep = max(n_cut, n_floor);
          if (reg_keep <= k_ub) {  // the top-keep set is the first keep sorted slots
#pragma unroll
            for (int r = 0; r < 16; ++r)
              if (lane * 16 + r < reg_keep) atomicOr(sbits + (x[r].c >> 5), 1u << (x[r].c & 31));
            reg_bits = true;
          }
        }
      }
      __syncwarp();
    }
    if (MODE == 1 && !done) {  // decided by the MODE 2 pass
      if (lane == 0) kv_cnt[row] = -1;
      return;
    }
    if (!done && !neg && M_total <= 1024) {
      // whole row in registers (32 keys per lane), keys only; then the exact sequential
      // scan by lane 0 over the sorted keys staged with one pad slot per 32
      uint64_t y[32];
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const int j = lane * 32 + r;
        y[r] = j < M_total ? keys[j] : ~0ull;
      }
      keys_bitonic_level<32, 2>(y, lane);
      bool crossed;
      n_cut = par_cut<32>([&](int r) { return y[r]; }, M_total, p, &crossed);
      if (n_cut < 0) {
#pragma unroll
        for (int r = 0; r < 32; ++r) skey[lane * 33 + r] = y[r];
        __syncwarp();
        int c = 0;
        if (lane == 0) {
          double pre = 0.0;
#pragma unroll 8
          for (int t = 0; t < M_total; ++t) {
            pre = __dadd_rn(pre, key_value(skey[t + (t >> 5)]));  // np.cumsum order (masks.py:152)
            if (pre > p) break;
            ++c;
          }
        }
        n_cut = __shfl_sync(FULL, c, 0) + 1;
      }
      done = true;
    }
    if (!done) {  // full sort of the row in shared memory, exact scan
      for (int j = lane; j < M_total; j += 32) { skey[j] = keys[j]; scol[j] = j; }
      int npf = 2;
      while (npf < M_total) npf <<= 1;
      bool crossed;
      n_cut = warp_sorted_cut(skey, scol, M_total, npf, p, !neg, &crossed);
    }
  } else {
    n_cut = M_total + 1;  // unreachable: the host enables SORT whenever p > 0 or R is external
  }
  int keep = max(n_cut, n_floor);
  keep = min(keep, M_total);

  // ---- top-n_keep set -> bits ----
  if (!reg_bits) {
    const RadixState t = warp_radix(keys, M_total, keep, hist);
    if (FASTS) {
      // boundary check: smallest selected vs largest unselected score
      double vin = INFINITY, vout = -INFINITY;
      int eq_base = 0;
      for (int j0 = 0; j0 < M_total; j0 += 32) {
        const int j = j0 + lane;
        uint64_t km = ~0ull;
        if (j < M_total) km = keys[j] & t.mask;
        const bool eq = (j < M_total) && km == t.prefix;
        const unsigned eqb = __ballot_sync(FULL, eq);
        const int eq_rank = eq_base + __popc(eqb & ((1u << lane) - 1u));
        const bool sel = (j < M_total) && (km < t.prefix || (eq && eq_rank < t.remaining));
        if (j < M_total) {
          const double v = key_value(keys[j]);
          if (sel) {
            vin = fmin(vin, v);
            atomicOr(sbits + (j >> 5), 1u << (j & 31));
          } else {
            vout = fmax(vout, v);
          }
        }
        eq_base += __popc(eqb);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        vin = fmin(vin, __shfl_xor_sync(FULL, vin, o));
        vout = fmax(vout, __shfl_xor_sync(FULL, vout, o));
      }
      const double scale = fmax(1.0, fmax(fabs(vin - mx), fabs(vout - mx)));
      const bool exact = vin - mx > -700.0 && (vout == -INFINITY || vin - vout > 1e-12 * scale);
      if (!exact) {  // leave the row to the exact pass (MODE 2, softmax on)
        if (lane == 0) kv_cnt[row] = -1;
        return;
      }
    } else {
      warp_topk_visit(keys, M_total, t,
                      [&](int j, int) { atomicOr(sbits + (j >> 5), 1u << (j & 31)); });
    }
  }
  __syncwarp();
  uint32_t* brow = bits + row * words;
  int run = 0;
  for (int w = lane; w < words; w += 32) {
    uint32_t x = sbits[w];
    if (with_union) {
      if (adja) x |= __ldg(adja + (int64_t)i * words + w);
      const int lo = w * 32;  // condition columns j >= M_v (masks.py:173)
      if (lo + 32 <= M_total && lo >= M_v) {
        x = ~0u;
      } else {
        for (int bb = 0; bb < 32; ++bb) {
          const int j = lo + bb;
          if (j >= M_v && j < M_total) x |= 1u << bb;
        }
      }
    }
    brow[w] = x;
    run += __popc(x);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) run += __shfl_xor_sync(FULL, run, o);
  if (lane == 0) kv_cnt[row] = run;
}

// Per-warp shared-memory carve-up shared by both select kernels.
__device__ __forceinline__ RowScratch carve_scratch(unsigned char* base, int words, int nslots,
                                                    int sortn) {
  RowScratch sc;
  sc.hist = reinterpret_cast<uint32_t*>(base);
  sc.sbits = sc.hist + 256;
  const int words_pad = (words + 1) & ~1;
  sc.leaf = reinterpret_cast<double*>(sc.sbits + words_pad);
  sc.skey = reinterpret_cast<uint64_t*>(sc.leaf + nslots);
  sc.scol = reinterpret_cast<int*>(sc.skey + sortn);
  return sc;
}

__device__ __forceinline__ void load_prog(const PwProg& prog, int* leaf_off, int* leaf_len,
                                          int2* fold_ops) {
  for (int i = threadIdx.x; i < prog.nl; i += blockDim.x) {
    leaf_off[i] = prog.off[i];
    leaf_len[i] = prog.len[i];
  }
  for (int i = threadIdx.x; i < prog.nops; i += blockDim.x) fold_ops[i] = prog.ops[i];
}

// One warp per (head, vision row) over a row-major R / score tensor in global memory.
// Per-warp smem: vals[M_pad] | scratch (hist, sbits, leaves, sort buffers).
template <bool RAW, bool SORT, int MODE = 0, bool FASTS = false>
__global__ void __launch_bounds__(SW_WARPS * 32) k_select(double* __restrict__ R, int64_t n_rows,
                                                          int M_v, int M_total, int np2,
                                                          const uint32_t* __restrict__ adja,
                                                          int words, int n_floor, double p,
                                                          int with_union,
                                                          uint32_t* __restrict__ bits,
                                                          int32_t* __restrict__ kv_cnt,
                                                          int per_warp_bytes, int nslots,
                                                          const __grid_constant__ PwProg prog) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int leaf_off[SEL_MAX_LEAVES], leaf_len[SEL_MAX_LEAVES];
  __shared__ int2 fold_ops[SEL_MAX_LEAVES];
  if (RAW && !FASTS) {
    load_prog(prog, leaf_off, leaf_len, fold_ops);
    __syncthreads();
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (row >= n_rows) return;
  if (MODE == 2 && kv_cnt[row] != -1) return;
  unsigned char* base = smem + (size_t)warp * per_warp_bytes;
  const int M_pad = (M_total + 1) & ~1;
  double* vals = reinterpret_cast<double*>(base);
  const RowScratch sc = carve_scratch(base + (size_t)M_pad * 8, words, nslots,
                                      MODE == 1 ? 544 : sel_full_sort(np2, M_total));
  double* Rr = R + row * M_total;
  for (int j = lane; j < M_total; j += 32) vals[j] = Rr[j];
  __syncwarp();
  // RAW: softmax first (a MODE 2 pass after a non-FASTS MODE 1 pass is launched RAW = false:
  // MODE 1 already turned the row into probabilities in place)
  select_row<RAW, SORT, MODE, FASTS>(
      vals, RAW ? Rr : nullptr, sc, row, (int)(row % M_v), M_v, M_total, words, n_floor, p,
      with_union, adja, bits, kv_cnt, prog.nl, prog.nops, leaf_off, leaf_len, fold_ops);
}

// ---- p == 0 on raw scores, rows of <= 32 * NPL columns: registers only ----------------
// The same decision as select_row<RAW, !SORT, MODE 1, FASTS> (top-n_floor set of the scores
// under (value desc, column asc), exact iff the boundary is no near tie and clear of exp's
// underflow range, else kv_cnt = -1 for the exact pass) without shared-memory radix passes:
// lane l holds columns l, l + 32, ... as fp32 images (double -> float is monotone), a
// bisection on those narrows the boundary to an interval (a, b] holding <= 32 columns (about
// log2(M_total / 32) counting rounds of one FSETP per element and a warp reduction), the
// candidates in it are ranked exactly by their float64 scores (ties: lower column first), and
// mask word i is the ballot of register i.  Only the boundary candidates and the extreme
// elements are ever compared in float64.  Rows with a non-finite or huge score, or whose
// boundary cannot be narrowed to 32 candidates (mass ties), go to the exact pass.
template <int NPL>
__global__ void __launch_bounds__(128, 4) k_select_p0(const double* __restrict__ S, int64_t n_rows,
                                                    int M_v, int M_total,
                                                    const uint32_t* __restrict__ adja, int words,
                                                    int n_floor, int with_union,
                                                    uint32_t* __restrict__ bits,
                                                    int32_t* __restrict__ kv_cnt) {
  __shared__ double c_val[4][32];
  __shared__ int c_col[4][32];
  __shared__ uint32_t c_bits[4][NPL];  // chosen candidates: word i, bit l = column l + 32 i
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * 4 + warp;
  if (row >= n_rows) return;
  const double* Sr = S + row * M_total;
  float f[NPL];
  bool bad = false;
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int j = lane + 32 * i;
    double x = j < M_total ? Sr[j] : 0.0;
    bad |= !(fabs(x) < 1e30);  // NaN / inf / out of float range: exact pass
    f[i] = j < M_total ? (float)x : -INFINITY;
  }
  auto redo = [&]() {
    if (lane == 0) kv_cnt[row] = -1;
  };
  if (__any_sync(FULL, bad)) return redo();
  float fmx = -INFINITY, fmn = INFINITY;
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    fmx = fmaxf(fmx, f[i]);
    if (lane + 32 * i < M_total) fmn = fminf(fmn, f[i]);
  }
  #pragma unroll
  for (int o = 16; o; o >>= 1) {
    fmx = fmaxf(fmx, __shfl_xor_sync(FULL, fmx, o));
    fmn = fminf(fmn, __shfl_xor_sync(FULL, fmn, o));
  }
  const int keep = min(max(n_floor, 1), M_total);
  auto count_gt = [&](float x) {
    int c = 0;
#pragma unroll
    for (int i = 0; i < NPL; ++i) c += f[i] > x ? 1 : 0;  // padding is -inf: never counted
    return (int)__reduce_add_sync(FULL, (unsigned)c);
  };
  // invariant: count_gt(b) < keep <= count_gt(a): the keep-th element's image lies in (a, b]
  float a = fmn, b = fmx;
  int ca = count_gt(a), cb = 0;
  if (ca >= keep) {
    for (int itn = 0; itn < 40 && ca - cb > 32; ++itn) {
      const float mid = a + 0.5f * (b - a);
      if (!(mid > a && mid < b)) break;
      const int c = count_gt(mid);
      if (c >= keep) { a = mid; ca = c; } else { b = mid; cb = c; }
    }
  } else {  // the boundary image is the row minimum: the candidates are its ties
    b = fmn;
    cb = ca;
    a = -INFINITY;
    ca = M_total;
  }
  const int ncand = ca - cb;
  if (ncand > 32) return redo();  // mass ties around the boundary: the exact pass sorts
  // gather the candidates (a, b] in column order, with their float64 scores
  for (int w = lane; w < NPL; w += 32) c_bits[warp][w] = 0u;
  int base = 0;
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int j = lane + 32 * i;
    const bool c = f[i] > a && f[i] <= b && j < M_total;
    const unsigned bal = __ballot_sync(FULL, c);
    if (c) {
      const int sl = base + __popc(bal & ((1u << lane) - 1u));
      c_val[warp][sl] = Sr[j];
      c_col[warp][sl] = j;
    }
    base += __popc(bal);
  }
  __syncwarp();
  const int need = keep - cb;  // candidates to take, best (value desc, column asc) first
  double cin = INFINITY, cout = -INFINITY;  // selected / unselected candidates' extremes
  if (lane < ncand) {
    const double mv = c_val[warp][lane];
    const int mc = c_col[warp][lane];
    int rank = 0;
    for (int u = 0; u < ncand; ++u) {
      const double uv = c_val[warp][u];
      rank += (uv > mv || (uv == mv && c_col[warp][u] < mc)) ? 1 : 0;
    }
    const bool sel = rank < need;
    if (sel) atomicOr(&c_bits[warp][mc >> 5], 1u << (mc & 31));
    if (sel) cin = mv; else cout = mv;
  }
  __syncwarp();
  // selected = {image > b} U chosen candidates; mask word i = ballot of register i
  float fin = INFINITY, fout = -INFINITY;  // min image above b, max image at or below a
  uint32_t mine = 0u;
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int j = lane + 32 * i;
    const bool sel = f[i] > b || ((c_bits[warp][i] >> lane) & 1u);
    if (f[i] > b) fin = fminf(fin, f[i]);
    if (f[i] <= a && j < M_total) fout = fmaxf(fout, f[i]);
    const unsigned w = __ballot_sync(FULL, sel);
    if (lane == i) mine = w;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    fin = fminf(fin, __shfl_xor_sync(FULL, fin, o));
    fout = fmaxf(fout, __shfl_xor_sync(FULL, fout, o));
    cin = fmin(cin, __shfl_xor_sync(FULL, cin, o));
    cout = fmax(cout, __shfl_xor_sync(FULL, cout, o));
  }
  // float64 extremes: the row max (image fmx), the smallest selected value (min of the
  // selected candidates and of the elements whose image is fin), the largest unselected
  // (max of the unselected candidates and of the elements whose image is fout)
  double mx = -INFINITY, vin = cin, vout = cout;
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int j = lane + 32 * i;
    if (j < M_total && (f[i] == fmx || (f[i] > b && f[i] == fin) || (f[i] <= a && f[i] == fout))) {
      const double x = Sr[j];
      if (f[i] == fmx) mx = fmax(mx, x);
      if (f[i] > b && f[i] == fin) vin = fmin(vin, x);
      if (f[i] <= a && f[i] == fout) vout = fmax(vout, x);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
    vin = fmin(vin, __shfl_xor_sync(FULL, vin, o));
    vout = fmax(vout, __shfl_xor_sync(FULL, vout, o));
  }
  const double scale = fmax(1.0, fmax(fabs(vin - mx), fabs(vout - mx)));
  const bool exact = vin - mx > -700.0 && (vout == -INFINITY || vin - vout > 1e-12 * scale);
  if (!exact) return redo();
  const int i_adj = (int)(row % M_v);
  uint32_t* brow = bits + row * words;
  int run = 0;
  for (int w = lane; w < words; w += 32) {
    uint32_t x = w == lane ? mine : 0u;
    if (with_union) {
      if (adja) x |= __ldg(adja + (int64_t)i_adj * words + w);
      const int lo = w * 32;  // condition columns j >= M_v (masks.py:173)
      if (lo + 32 <= M_total && lo >= M_v) {
        x = ~0u;
      } else {
        for (int bb = 0; bb < 32; ++bb) {
          const int j = lo + bb;
          if (j >= M_v && j < M_total) x |= 1u << bb;
        }
      }
    }
    brow[w] = x;
    run += __popc(x);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) run += __shfl_xor_sync(FULL, run, o);
  if (lane == 0) kv_cnt[row] = run;
}

// ---- p > 0 on raw scores, rows of <= 32 * NPL columns: the cutoff without sorting -------
// Same decision as select_row<RAW, SORT, MODE 1> (R = exp(S - max) / numpy-pairwise sum, in
// the same operations, so R is bitwise the shared-memory path's; n_cut = 1 + #(sorted
// sequential prefix <= p); keep = min(max(n_cut, n_floor), M_total) top columns under
// (R desc, column asc)), but instead of a radix-selected 512-wide window sorted in
// registers: a bisection on fp32 images of R brackets the prefix crossing to <= 32 candidate
// columns (a, b] with the tree-summed mass above b <= p < the mass above a; the candidates are
// ranked exactly and their prefixes formed from that mass.  Every prefix within 1e-12 of p
// (where the tree and np.cumsum's sequential order could round to different sides), a
// boundary that cannot be narrowed to 32 candidates (mass ties), or a non-finite score sends
// the row to the exact pass (kv_cnt = -1, R written back for it; with write_r every row's R
// is written, as tcb_block_select_scores returns it).
template <int NPL>
__global__ void __launch_bounds__(128) k_select_cut(double* __restrict__ S, int64_t n_rows, int M_v,
                                                     int M_total, const uint32_t* __restrict__ adja,
                                                     int words, int n_floor, double p, int with_union,
                                                     int write_r, uint32_t* __restrict__ bits,
                                                     int32_t* __restrict__ kv_cnt,
                                                     const __grid_constant__ PwProg prog) {
  __shared__ int leaf_off[SEL_MAX_LEAVES], leaf_len[SEL_MAX_LEAVES];
  __shared__ int2 fold_ops[SEL_MAX_LEAVES];
  __shared__ double vals[4][NPL * 32];
  __shared__ double leafv[4][64];
  __shared__ double c_val[4][32];
  __shared__ int c_col[4][32];
  __shared__ uint32_t c_bits[4][NPL];
  load_prog(prog, leaf_off, leaf_len, fold_ops);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * 4 + warp;
  if (row >= n_rows) return;
  double* Sr = S + row * M_total;
  double* vs = vals[warp];
  // ---- R, exactly as select_row<RAW>: max, exp, pairwise sum, divide (R kept in shared
  // memory, only its fp32 images in registers: occupancy for the fp64 exp / divide latency)
  bool bad = false;
  double mx = -INFINITY;
  for (int j = lane; j < M_total; j += 32) {
    const double x = Sr[j];
    vs[j] = x;
    bad |= !isfinite(x);
    mx = fmax(mx, x);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
  for (int j = lane; j < M_total; j += 32) vs[j] = exp(vs[j] - mx);
  __syncwarp();
  for (int l = lane; l < prog.nl; l += 32) leafv[warp][l] = pw_leaf(vs + leaf_off[l], leaf_len[l]);
  __syncwarp();
  double tot = 0.0;
  if (lane == 0) {
    for (int q = 0; q < prog.nops; ++q)
      leafv[warp][prog.nl + q] = leafv[warp][fold_ops[q].x] + leafv[warp][fold_ops[q].y];
    tot = leafv[warp][prog.nops ? prog.nl + prog.nops - 1 : 0];
  }
  tot = __shfl_sync(FULL, tot, 0);
  float f[NPL];
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int j = lane + 32 * i;
    double rv = 0.0;
    if (j < M_total) {
      rv = vs[j] / tot;
      vs[j] = rv;
      if (write_r) Sr[j] = rv;
    }
    f[i] = j < M_total ? (float)rv : -INFINITY;
  }
  auto redo = [&]() {
    if (!write_r)
      for (int j = lane; j < M_total; j += 32) Sr[j] = vs[j];
    if (lane == 0) kv_cnt[row] = -1;
  };
  if (__any_sync(FULL, bad)) return redo();
  // mass and count of the columns whose image exceeds x (tree order: bracketing only)
  auto mass_gt = [&](float x, int& cnt) {
    double m = 0.0;
    int c = 0;
#pragma unroll
    for (int i = 0; i < NPL; ++i)
      if (f[i] > x) {
        m += vs[lane + 32 * i];
        ++c;
      }
#pragma unroll
    for (int o = 16; o; o >>= 1) m += __shfl_xor_sync(FULL, m, o);
    cnt = (int)__reduce_add_sync(FULL, (unsigned)c);
    return m;
  };
  // ---- n_cut: bracket the prefix crossing, mass(b) <= p < mass(a); p == 0: n_cut = 1
  // (masks.py:152-153 with prefix_0 = the row max > 0, as select_row's p == 0 branch)
  float a = -1.0f, b = 2.0f;  // R in [0, 1]
  int na = M_total, nb = 0;
  double ma = 0.0, mb = 0.0;
  ma = mass_gt(a, na);
  if (p > 0.0 && !(ma > p + 1e-12)) return redo();  // the row total does not clear p
  {
    float fmx = -INFINITY;
#pragma unroll
    for (int i = 0; i < NPL; ++i) fmx = fmaxf(fmx, f[i]);
#pragma unroll
    for (int o = 16; o; o >>= 1) fmx = fmaxf(fmx, __shfl_xor_sync(FULL, fmx, o));
    b = fmx;  // nothing exceeds the maximum image
  }
  for (int itn = 0; p > 0.0 && itn < 48 && na - nb > 32; ++itn) {
    const float mid = a + 0.5f * (b - a);
    if (!(mid > a && mid < b)) break;
    int c;
    const double m = mass_gt(mid, c);
    if (m <= p) { b = mid; mb = m; nb = c; } else { a = mid; ma = m; na = c; }
  }
  auto gather = [&](float lo, float hi) -> int {  // candidates (lo, hi] in column order
    int base = 0;
#pragma unroll
    for (int i = 0; i < NPL; ++i) {
      const bool c = f[i] > lo && f[i] <= hi;
      const unsigned bal = __ballot_sync(FULL, c);
      if (c) {
        const int sl = base + __popc(bal & ((1u << lane) - 1u));
        c_val[warp][sl] = vs[lane + 32 * i];
        c_col[warp][sl] = lane + 32 * i;
      }
      base += __popc(bal);
    }
    __syncwarp();
    return base;
  };
  int ncand = na - nb;
  int cut_count = 0;
  bool ambiguous = false;
  if (p > 0.0) {
  if (ncand > 32 || p - mb <= 1e-12) return redo();
  gather(a, b);
  // candidate t's rank under (R desc, column asc) and the prefix through it
  {
    int rank = 1 << 30;
    double pre = 0.0;
    if (lane < ncand) {
      const double mv = c_val[warp][lane];
      const int mc = c_col[warp][lane];
      rank = 0;
      for (int u = 0; u < ncand; ++u) {
        const double uv = c_val[warp][u];
        rank += (uv > mv || (uv == mv && c_col[warp][u] < mc)) ? 1 : 0;
      }
      double ssum = 0.0;  // candidates up to and including this one, in rank order
      for (int u = 0; u < ncand; ++u) {
        const double uv = c_val[warp][u];
        const bool before = uv > mv || (uv == mv && c_col[warp][u] <= mc);
        if (before) ssum += uv;
      }
      pre = mb + ssum;
      ambiguous = fabs(pre - p) <= 1e-12;
    }
    cut_count = (int)__reduce_add_sync(FULL, (unsigned)(lane < ncand && pre <= p));
    ambiguous = __any_sync(FULL, ambiguous);
  }
  if (ambiguous) return redo();
  } else {
    na = nb = 0;  // no cutoff bracket: the top-keep set is count-bracketed below
  }
  const int n_cut = p > 0.0 ? nb + cut_count + 1 : 1;
  const int keep = min(max(n_cut, n_floor), M_total);
  // ---- the top-keep set: count-bracket its boundary (a2, b2] to <= 32 candidates
  float a2 = a, b2 = b;
  int na2 = na, nb2 = nb;
  if (!(nb2 < keep && keep <= na2)) {  // keep outside the cutoff bracket: re-bracket by count
    a2 = -1.0f;
    na2 = M_total;
    {
      float fmx = -INFINITY;
#pragma unroll
      for (int i = 0; i < NPL; ++i) fmx = fmaxf(fmx, f[i]);
#pragma unroll
      for (int o = 16; o; o >>= 1) fmx = fmaxf(fmx, __shfl_xor_sync(FULL, fmx, o));
      b2 = fmx;
      nb2 = 0;
    }
    for (int itn = 0; itn < 48 && na2 - nb2 > 32; ++itn) {
      const float mid = a2 + 0.5f * (b2 - a2);
      if (!(mid > a2 && mid < b2)) break;
      int c;
      mass_gt(mid, c);
      if (c >= keep) { a2 = mid; na2 = c; } else { b2 = mid; nb2 = c; }
    }
    if (na2 - nb2 > 32) return redo();
    __syncwarp();
    gather(a2, b2);
  }
  const int ncand2 = na2 - nb2;
  const int need = keep - nb2;
  for (int w = lane; w < NPL; w += 32) c_bits[warp][w] = 0u;
  __syncwarp();
  if (lane < ncand2) {
    const double mv = c_val[warp][lane];
    const int mc = c_col[warp][lane];
    int rank = 0;
    for (int u = 0; u < ncand2; ++u) {
      const double uv = c_val[warp][u];
      rank += (uv > mv || (uv == mv && c_col[warp][u] < mc)) ? 1 : 0;
    }
    if (rank < need) atomicOr(&c_bits[warp][mc >> 5], 1u << (mc & 31));
  }
  __syncwarp();
  uint32_t mine = 0u;
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const bool sel = f[i] > b2 || ((c_bits[warp][i] >> lane) & 1u);
    const unsigned w = __ballot_sync(FULL, sel);
    if (lane == i) mine = w;
  }
  const int i_adj = (int)(row % M_v);
  uint32_t* brow = bits + row * words;
  int run = 0;
  for (int w = lane; w < words; w += 32) {
    uint32_t x = w == lane ? mine : 0u;
    if (with_union) {
      if (adja) x |= __ldg(adja + (int64_t)i_adj * words + w);
      const int lo = w * 32;  // condition columns j >= M_v (masks.py:173)
      if (lo + 32 <= M_total && lo >= M_v) {
        x = ~0u;
      } else {
        for (int bb = 0; bb < 32; ++bb) {
          const int j = lo + bb;
          if (j >= M_v && j < M_total) x |= 1u << bb;
        }
      }
    }
    brow[w] = x;
    run += __popc(x);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) run += __shfl_xor_sync(FULL, run, o);
  if (lane == 0) kv_cnt[row] = run;
}

__global__ void __launch_bounds__(128) k_mask_pack(const uint8_t* __restrict__ dense, int M_total,
                                                   int words, uint32_t* __restrict__ bits,
                                                   int32_t* __restrict__ kv_cnt) {
  __shared__ int s_cnt;
  const int64_t row = blockIdx.x;
  const uint8_t* d = dense + row * M_total;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  int cnt = 0;
  for (int w = threadIdx.x; w < words; w += blockDim.x) {
    uint32_t x = 0;
    for (int bb = 0; bb < 32; ++bb) {
      const int j = w * 32 + bb;
      if (j < M_total && d[j]) x |= 1u << bb;
    }
    bits[row * words + w] = x;
    cnt += __popc(x);
  }
  atomicAdd(&s_cnt, cnt);
  __syncthreads();
  if (threadIdx.x == 0) kv_cnt[row] = s_cnt;
}

__global__ void k_mask_unpack(const uint32_t* __restrict__ bits, int64_t rows, int M_total,
                              int words, uint8_t* __restrict__ dense) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * M_total) return;
  const int64_t r = e / M_total;
  const int j = (int)(e - r * M_total);
  dense[e] = (uint8_t)((bits[r * words + (j >> 5)] >> (j & 31)) & 1u);
}

}  // namespace tcb

using namespace tcb;

// K4a launcher: DMMA (FP64 tensor core) by default, the SIMT-DFMA tile kernel with
// TCB_SCORES_SIMT=1 (kept for A/B).
static int launch_scores(const double* pq, int pq_blocks, const double* pk, int H, int rows,
                         int M_total, int d, double* R, cudaStream_t st) {
  static int simt = -1;
  if (simt < 0) {
    const char* e = getenv("TCB_SCORES_SIMT");
    simt = e ? atoi(e) : 0;
  }
  if (simt || d % 4 != 0) {
    dim3 grid((unsigned)ceil_div(M_total, ST_TILE), (unsigned)ceil_div(rows, ST_TILE), H);
    k_scores<<<grid, 256, 0, st>>>(pq, pq_blocks, pk, rows, M_total, d, sqrt((double)d), R);
    return check_launch("k_scores");
  }
  dim3 grid((unsigned)ceil_div(M_total, 64), (unsigned)ceil_div(rows, 64), H);
  k_scores_dmma<<<grid, 128, 0, st>>>(pq, pq_blocks, pk, rows, M_total, d, sqrt((double)d), R);
  return check_launch("k_scores_dmma");
}

template <typename T>
static void launch_pool(bool vec, dim3 grid, cudaStream_t s, const void* x0, const void* x1,
                        int64_t sh, int64_t sn, int H, int d, int m, int M_v, int M_total,
                        int64_t n_valid, int64_t n_cond, double* o0, double* o1, int G, int chunks) {
  if (vec)
    k_pool<T, true><<<grid, 128, 0, s>>>((const T*)x0, (const T*)x1, sh, sn, H, d, m, M_v, M_total,
                                         n_valid, n_cond, o0, o1, G, chunks);
  else
    k_pool<T, false><<<grid, 128, 0, s>>>((const T*)x0, (const T*)x1, sh, sn, H, d, m, M_v,
                                          M_total, n_valid, n_cond, o0, o1, G, chunks);
}

extern "C" int tcb_block_pool(const void* x0, const void* x1, int dtype, int64_t stride_h,
                              int64_t stride_n, int H, int d, int m, int M_v, int M_total,
                              int64_t n_valid, int64_t n_cond, double* out0, double* out1,
                              void* stream) {
  TCB_CHECK_ARG(x0 && out0, TCB_ESHAPE, "null tensor");
  TCB_CHECK_ARG((x1 == nullptr) == (out1 == nullptr), TCB_ESHAPE, "x1/out1 must both be set");
  TCB_CHECK_ARG(H >= 1 && d >= 1 && m >= 1 && M_total >= M_v && M_v >= 0, TCB_ESHAPE,
                "bad pool shape");
  TCB_CHECK_ARG(dtype == TCB_F32 || dtype == TCB_BF16 || dtype == TCB_F16 || dtype == TCB_F64,
                TCB_EDOMAIN, "unsupported dtype %d", dtype);
  if ((int64_t)H * M_total == 0) return TCB_OK;
  const int esz = dtype == TCB_F64 ? 8 : dtype == TCB_F32 ? 4 : 2;
  const int VE = 16 / esz;
  const bool vec = (d % VE == 0) && (stride_n % VE == 0) && (stride_h % VE == 0) &&
                   ((uintptr_t)x0 % 16 == 0) && ((uintptr_t)x1 % 16 == 0);
  const int chunks = vec ? d / VE : d;
  int G = 1;
  while (G < chunks && G < 128) G <<= 1;
  const int per_cta = 128 / G;
  const int64_t items = (int64_t)H * M_total;
  dim3 grid((unsigned)ceil_div(items, per_cta), x1 ? 2 : 1);
  cudaStream_t s = as_stream(stream);
  if (dtype == TCB_F32)
    launch_pool<float>(vec, grid, s, x0, x1, stride_h, stride_n, H, d, m, M_v, M_total, n_valid,
                       n_cond, out0, out1, G, chunks);
  else if (dtype == TCB_BF16)
    launch_pool<__nv_bfloat16>(vec, grid, s, x0, x1, stride_h, stride_n, H, d, m, M_v, M_total,
                               n_valid, n_cond, out0, out1, G, chunks);
  else if (dtype == TCB_F16)
    launch_pool<__half>(vec, grid, s, x0, x1, stride_h, stride_n, H, d, m, M_v, M_total, n_valid,
                        n_cond, out0, out1, G, chunks);
  else
    launch_pool<double>(vec, grid, s, x0, x1, stride_h, stride_n, H, d, m, M_v, M_total, n_valid,
                        n_cond, out0, out1, G, chunks);
  return check_launch("k_pool");
}

extern "C" int tcb_block_relevance(const double* pq, int pq_blocks, const double* pk, int H,
                                   int rows, int M_total, int d, double* R, void* stream) {
  TCB_CHECK_ARG(pq && pk && R, TCB_ESHAPE, "null tensor");
  TCB_CHECK_ARG(H >= 1 && rows >= 0 && rows <= pq_blocks && M_total >= 1 && d >= 1, TCB_ESHAPE,
                "bad relevance shape");
  TCB_CHECK_ARG(M_total <= 16384, TCB_ESIZE, "M_total %d > 16384 unsupported", M_total);
  if (rows == 0) return TCB_OK;
  cudaStream_t st = as_stream(stream);
  int rc = launch_scores(pq, pq_blocks, pk, H, rows, M_total, d, R, st);
  if (rc) return rc;
  const int64_t n_rows = (int64_t)H * rows;
  k_row_softmax<<<(unsigned)ceil_div(n_rows, 8), 256, 0, st>>>(R, n_rows, M_total);
  return check_launch("k_row_softmax");
}

struct SelPlan {
  int nslots, np2, words_pad, M_pad;
  PwProg prog;
};

static SelPlan plan_select(int M_total, int words) {
  SelPlan pl;
  // per-warp leaf slots: nl leaves + (nl - 1) folds, nl <= 8192 / 64 = SEL_MAX_LEAVES
  pl.prog.nl = pw_leaves(M_total, pl.prog.off, pl.prog.len);
  pl.prog.nops = pw_program(M_total, pl.prog.nl, pl.prog.ops);
  pl.nslots = (2 * pl.prog.nl + 1) & ~1;
  pl.np2 = 2;
  while (pl.np2 < M_total) pl.np2 <<= 1;
  pl.M_pad = (M_total + 1) & ~1;
  pl.words_pad = (words + 1) & ~1;
  return pl;
}

// scratch bytes per warp (without the row values): hist | sbits | leaves | sort buffers
static size_t scratch_bytes(const SelPlan& pl, int sortn) {
  const size_t b = 256 * 4 + (size_t)pl.words_pad * 4 + (size_t)pl.nslots * 8 + (size_t)sortn * 12;
  return (b + 15) & ~size_t(15);
}

constexpr size_t SMEM_CAP = 232448 - 8192;  // opt-in limit minus the static leaf tables

// n_rows rows of R (row r uses adjacency row r % M_v; chunk callers offset the pointers)
// write_r: the raw scores must come back as R for every row (tcb_block_select_scores returns
// them); tcb_block_mask's scratch only needs R for the rows left to the exact pass.
static int launch_select(double* R, bool raw, int64_t n_rows, int M_v, int M_total,
                         const uint32_t* adja, int words, int n_floor, double p, int with_union,
                         uint32_t* bits, int32_t* kv_cnt, cudaStream_t s, bool fasts = false,
                         bool write_r = true) {
  TCB_CHECK_ARG(R && bits && kv_cnt, TCB_ESHAPE, "null tensor");
  TCB_CHECK_ARG(n_rows >= 0 && M_v >= 0 && M_total >= 1, TCB_ESHAPE, "bad select shape");
  TCB_CHECK_ARG(words >= ceil_div(M_total, 32), TCB_ESHAPE, "words too small");
  TCB_CHECK_ARG(M_total <= 8192, TCB_ESIZE, "M_total %d > 8192 unsupported", M_total);
  TCB_CHECK_ARG(n_floor >= 1, TCB_EDOMAIN, "n_floor must be >= 1");
  const SelPlan pl = plan_select(M_total, words);
  if (n_rows == 0) return TCB_OK;
  const bool sort = !raw || p > 0.0;
  const int full_sort = sel_full_sort(pl.np2, M_total);
  // rows (warps) per CTA: SW_WARPS while their shared memory fits, fewer for long rows
  // (M_total = 8192 with the sort buffers needs 163 KB for one warp)
  auto go = [&](auto kern, int sortn) -> int {
    const size_t pw = (size_t)pl.M_pad * 8 + scratch_bytes(pl, sortn);
    const int wpc = (int)std::min<size_t>(SW_WARPS, SMEM_CAP / pw);
    if (wpc < 1) return set_error(TCB_ESIZE, "k_select: %zu B of shared memory per row", pw);
    const size_t sm = pw * wpc;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return set_error(TCB_ECUDA, "k_select smem: %s", cudaGetErrorString(e));
    kern<<<(unsigned)ceil_div(n_rows, wpc), wpc * 32, sm, s>>>(
        R, n_rows, M_v, M_total, pl.np2, adja, words, n_floor, p, with_union, bits, kv_cnt,
        (int)pw, pl.nslots, pl.prog);
    return check_launch("k_select");
  };
  if (raw && !sort && fasts) {
    // p == 0 on scores nobody reads back as R: select on the scores (FASTS), then the exact
    // softmax program on the rows whose top-k boundary was a near tie (grid-stride, usually
    // nothing to do).  Rows of <= 1024 columns take the register kernel (k_select_p0).
    int rc;
    static int legacy = -1;
    if (legacy < 0) {
      const char* e = getenv("TCB_SELECT_LEGACY");
      legacy = (e && atoi(e) != 0) ? 1 : 0;
    }
    if (M_total <= 1024 && !legacy) {
      const unsigned grid = (unsigned)ceil_div(n_rows, 4);
      if (M_total <= 256)
        k_select_p0<8><<<grid, 128, 0, s>>>(R, n_rows, M_v, M_total, adja, words, n_floor, with_union, bits, kv_cnt);
      else if (M_total <= 512)
        k_select_p0<16><<<grid, 128, 0, s>>>(R, n_rows, M_v, M_total, adja, words, n_floor, with_union, bits, kv_cnt);
      else
        k_select_p0<32><<<grid, 128, 0, s>>>(R, n_rows, M_v, M_total, adja, words, n_floor, with_union, bits, kv_cnt);
      rc = check_launch("k_select_p0");
    } else {
      rc = go(k_select<true, false, 1, true>, 0);
    }
    if (rc) return rc;
    return go(k_select<true, false, 2, false>, 0);
  }
  static int legacy_cut = -1;
  if (legacy_cut < 0) {
    const char* e = getenv("TCB_SELECT_LEGACY");
    legacy_cut = (e && atoi(e) != 0) ? 1 : 0;
  }
  if (raw && M_total <= 1024 && !legacy_cut && p > 0.0) {
    // the cutoff on raw scores of <= 1024 columns: the register kernel (k_select_cut, no
    // sort) decides almost every row; the exact pass takes the rest.  (Its p = 0 branch is
    // correct but slower than k_select<RAW, !SORT> there: 0.78 vs 0.71 ms at C2.)
    const unsigned grid = (unsigned)ceil_div(n_rows, 4);
    const int wr = write_r ? 1 : 0;
    if (M_total <= 256)
      k_select_cut<8><<<grid, 128, 0, s>>>(R, n_rows, M_v, M_total, adja, words, n_floor, p, with_union, wr, bits, kv_cnt, pl.prog);
    else if (M_total <= 512)
      k_select_cut<16><<<grid, 128, 0, s>>>(R, n_rows, M_v, M_total, adja, words, n_floor, p, with_union, wr, bits, kv_cnt, pl.prog);
    else
      k_select_cut<32><<<grid, 128, 0, s>>>(R, n_rows, M_v, M_total, adja, words, n_floor, p, with_union, wr, bits, kv_cnt, pl.prog);
    int rc = check_launch("k_select_cut");
    if (rc) return rc;
    return go(k_select<false, true, 2>, full_sort);
  }
  if (raw && !sort) return go(k_select<true, false>, 0);
  // cutoff path: slim pass (register sort of the top-512 window, ~35 % less shared memory
  // per warp -> 1.5x the resident warps), then the full-sort pass over the rows it left
  int rc = raw ? go(k_select<true, true, 1>, 544) : go(k_select<false, true, 1>, 544);
  if (rc) return rc;
  return go(k_select<false, true, 2>, full_sort);
}

extern "C" int tcb_block_select(const double* R, int H, int M_v, int M_total,
                                const uint32_t* adja, int words, int n_floor, double p,
                                int with_union, uint32_t* bits, int32_t* kv_cnt, void* stream) {
  // R is only read on this path (RAW=false never writes it)
  TCB_CHECK_ARG(H >= 1, TCB_ESHAPE, "bad select shape");
  return launch_select(const_cast<double*>(R), false, (int64_t)H * M_v, M_v, M_total, adja, words,
                       n_floor, p, with_union, bits, kv_cnt, as_stream(stream));
}

extern "C" int tcb_block_select_scores(double* S, int H, int M_v, int M_total,
                                       const uint32_t* adja, int words, int n_floor, double p,
                                       int with_union, uint32_t* bits, int32_t* kv_cnt,
                                       void* stream) {
  TCB_CHECK_ARG(H >= 1, TCB_ESHAPE, "bad select shape");
  return launch_select(S, true, (int64_t)H * M_v, M_v, M_total, adja, words, n_floor, p, with_union,
                       bits, kv_cnt, as_stream(stream));
}

// Scratch doubles tcb_block_mask uses: all heads' scores when they fit 256 MB, else one
// bounded chunk (whole heads, or a row range of one head).
extern "C" int64_t tcb_block_mask_scratch(int H, int M_v, int M_total) {
  const int64_t cap = (int64_t)32 << 20;  // 256 MB of float64 scores
  const int64_t all = (int64_t)H * M_v * M_total;
  if (all <= cap) return std::max<int64_t>(all, 1);
  const int64_t rows = std::max<int64_t>(1, std::min<int64_t>(M_v, cap / std::max(1, M_total)));
  const int64_t per_head = (int64_t)M_v * M_total;
  if (rows == M_v) return (cap / per_head) * per_head;  // whole heads per chunk
  return rows * M_total;
}

extern "C" int tcb_block_mask(const double* pq, int pq_blocks, const double* pk, int H, int M_v,
                              int M_total, int d, const uint32_t* adja, int words, int n_floor,
                              double p, uint32_t* bits, int32_t* kv_cnt, double* scratch,
                              int64_t scratch_elems, void* stream) {
  TCB_CHECK_ARG(pq && pk && bits && kv_cnt, TCB_ESHAPE, "null tensor");
  TCB_CHECK_ARG(H >= 1 && M_v >= 0 && M_total >= M_v && M_total >= 1 && d >= 1 &&
                    M_v <= pq_blocks,
                TCB_ESHAPE, "bad mask shape");
  TCB_CHECK_ARG(words >= ceil_div(M_total, 32), TCB_ESHAPE, "words too small");
  TCB_CHECK_ARG(M_total <= 8192, TCB_ESIZE, "M_total %d > 8192 unsupported", M_total);
  TCB_CHECK_ARG(n_floor >= 1, TCB_EDOMAIN, "n_floor must be >= 1");
  TCB_CHECK_ARG(p >= 0.0 && p < 1.0, TCB_EDOMAIN, "p %g outside [0, 1)", p);
  if ((int64_t)H * M_v == 0) return TCB_OK;
  TCB_CHECK_ARG(scratch && scratch_elems >= M_total, TCB_ESIZE,
                "scratch of %lld doubles < one row of %d", (long long)scratch_elems, M_total);
  cudaStream_t s = as_stream(stream);
  const int64_t per_head = (int64_t)M_v * M_total;
  const bool fasts = p == 0.0;
  int rc;
  if (scratch_elems >= per_head) {  // whole heads per chunk
    const int hc = (int)std::min<int64_t>(H, scratch_elems / per_head);
    for (int h0 = 0; h0 < H; h0 += hc) {
      const int nh = std::min(hc, H - h0);
      rc = launch_scores(pq + (int64_t)h0 * pq_blocks * d, pq_blocks, pk + (int64_t)h0 * M_total * d,
                         nh, M_v, M_total, d, scratch, s);
      if (rc) return rc;
      rc = launch_select(scratch, true, (int64_t)nh * M_v, M_v, M_total, adja, words, n_floor, p, 1,
                         bits + (int64_t)h0 * M_v * words, kv_cnt + (int64_t)h0 * M_v, s, fasts, false);
      if (rc) return rc;
    }
    return TCB_OK;
  }
  // a row range of one head per chunk (the adjacency rows of the range start at r0)
  const int rows_chunk = (int)(scratch_elems / M_total);
  for (int h = 0; h < H; ++h) {
    for (int r0 = 0; r0 < M_v; r0 += rows_chunk) {
      const int nr = std::min(rows_chunk, M_v - r0);
      rc = launch_scores(pq + ((int64_t)h * pq_blocks + r0) * d, nr, pk + (int64_t)h * M_total * d,
                         1, nr, M_total, d, scratch, s);
      if (rc) return rc;
      rc = launch_select(scratch, true, nr, M_v, M_total, adja ? adja + (int64_t)r0 * words : nullptr,
                         words, n_floor, p, 1, bits + ((int64_t)h * M_v + r0) * words,
                         kv_cnt + (int64_t)h * M_v + r0, s, fasts, false);
      if (rc) return rc;
    }
  }
  return TCB_OK;
}

extern "C" int tcb_block_scores(const double* pq, int pq_blocks, const double* pk, int H, int rows,
                                int M_total, int d, double* S, void* stream) {
  TCB_CHECK_ARG(pq && pk && S, TCB_ESHAPE, "null tensor");
  TCB_CHECK_ARG(H >= 1 && rows >= 0 && rows <= pq_blocks && M_total >= 1 && d >= 1, TCB_ESHAPE,
                "bad scores shape");
  if (rows == 0) return TCB_OK;
  return launch_scores(pq, pq_blocks, pk, H, rows, M_total, d, S, as_stream(stream));
}

extern "C" int tcb_mask_pack(const uint8_t* dense, int64_t rows, int M_total, int words,
                             uint32_t* bits, int32_t* kv_cnt, void* stream) {
  TCB_CHECK_ARG(dense && bits && kv_cnt, TCB_ESHAPE, "null tensor");
  TCB_CHECK_ARG(words >= ceil_div(M_total, 32), TCB_ESHAPE, "words too small");
  if (rows == 0) return TCB_OK;
  k_mask_pack<<<(unsigned)rows, 128, 0, as_stream(stream)>>>(dense, M_total, words, bits, kv_cnt);
  return check_launch("k_mask_pack");
}

extern "C" int tcb_mask_unpack(const uint32_t* bits, int64_t rows, int M_total, int words,
                               uint8_t* dense, void* stream) {
  TCB_CHECK_ARG(dense && bits, TCB_ESHAPE, "null tensor");
  const int64_t n = rows * M_total;
  if (n == 0) return TCB_OK;
  k_mask_unpack<<<(unsigned)ceil_div(n, 256), 256, 0, as_stream(stream)>>>(bits, rows, M_total,
                                                                           words, dense);
  return check_launch("k_mask_unpack");
}
