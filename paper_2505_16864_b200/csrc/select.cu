// K3 block pool, K4 pooled relevance, K5+K6 selection/union, mask pack/unpack.
//
// K3  tcb_block_pool       <- block_pool        masks.py:98-116   (HBM bound)
// K4  tcb_block_relevance  <- relevance         masks.py:119-134  (fp64 FMA bound)
// K5  tcb_block_select     <- importance_mask   masks.py:137-159
//     (+ union)            <- union_mask        masks.py:162-175
#include "common.cuh"

#include <cuda_bf16.h>
#include <math.h>

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
          v[u][0] = (double)(float)p[(int64_t)(r + u) * sn];
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
        v[0] = (double)(float)p[(int64_t)r * sn];
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
// K4 relevance: R[h,i,:] = softmax(pq_i . pk_j / sqrt(d)).  CTA = (head, 32 rows);
// float64 register-tiled product (2 rows x 4 cols per thread) over 64-column
// chunks of pk staged in smem; raw scaled scores go to R, then one thread per row
// does max / exp / numpy-pairwise sum / divide in place (masks.py:130-134).
// ---------------------------------------------------------------------------
constexpr int RT_ROWS = 32;
constexpr int RT_COLS = 64;
constexpr int RT_KC = 32;  // d-chunk staged per step

// numpy's pairwise summation (PW_BLOCKSIZE 128, 8-way unrolled leaves): the
// recursion splits n > 128 at n2 = n/2 - (n/2)%8 and sums left + right.  The leaves
// (contiguous runs of <= 128) are independent, so a warp sums them in parallel and
// lane 0 folds the leaf sums in the recursion's order.
constexpr int PW_MAX_LEAVES = 256;  // enough for n <= 16384

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
__device__ int pw_leaves(int n, int* off, int* len) {
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

__global__ void __launch_bounds__(256) k_relevance(const double* __restrict__ pq, int pq_blocks,
                                                   const double* __restrict__ pk, int rows,
                                                   int M_total, int d, double inv_sqrt_unused,
                                                   double sqrt_d, double* __restrict__ R) {
  // phase 1 tiles and phase 2 per-warp scratch share one buffer
  __shared__ double sbuf[8 * 2 * PW_MAX_LEAVES];
  static_assert(RT_ROWS * (RT_KC + 1) + RT_KC * (RT_COLS + 1) <= 8 * 2 * PW_MAX_LEAVES, "smem");
  double(*sA)[RT_KC + 1] = reinterpret_cast<double(*)[RT_KC + 1]>(sbuf);
  double(*sB)[RT_COLS + 1] = reinterpret_cast<double(*)[RT_COLS + 1]>(sbuf + RT_ROWS * (RT_KC + 1));
  const int h = blockIdx.y;
  const int r0 = blockIdx.x * RT_ROWS;
  const int tid = threadIdx.x;
  const int rg = tid >> 4;  // 16 row groups x 2 rows
  const int cg = tid & 15;  // 16 col groups x 4 cols (cg, cg+16, cg+32, cg+48)
  const double* A = pq + (int64_t)h * pq_blocks * d;
  const double* B = pk + (int64_t)h * M_total * d;
  double* Rh = R + (int64_t)h * rows * M_total;
  for (int c0 = 0; c0 < M_total; c0 += RT_COLS) {
    double acc[2][4];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    for (int k0 = 0; k0 < d; k0 += RT_KC) {
      __syncthreads();
      for (int e = tid; e < RT_ROWS * RT_KC; e += 256) {
        int rr = e / RT_KC, kk = e % RT_KC;
        int gr = r0 + rr, gk = k0 + kk;
        sA[rr][kk] = (gr < rows && gk < d) ? A[(int64_t)gr * d + gk] : 0.0;
      }
      for (int e = tid; e < RT_COLS * RT_KC; e += 256) {
        int cc = e / RT_KC, kk = e % RT_KC;
        int gc = c0 + cc, gk = k0 + kk;
        sB[kk][cc] = (gc < M_total && gk < d) ? B[(int64_t)gc * d + gk] : 0.0;
      }
      __syncthreads();
#pragma unroll 8
      for (int kk = 0; kk < RT_KC; ++kk) {
        double a0 = sA[2 * rg][kk], a1 = sA[2 * rg + 1][kk];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          double bv = sB[kk][cg + 16 * b];
          acc[0][b] = fma(a0, bv, acc[0][b]);
          acc[1][b] = fma(a1, bv, acc[1][b]);
        }
      }
    }
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      int gr = r0 + 2 * rg + a;
      if (gr >= rows) continue;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        int gc = c0 + cg + 16 * b;
        if (gc < M_total) Rh[(int64_t)gr * M_total + gc] = acc[a][b] / sqrt_d;  // masks.py:131
      }
    }
  }
  __syncthreads();
  // per-row softmax (masks.py:132-134): one warp per row, lanes stride the row
  // (coalesced); the row sum is numpy's pairwise order (bit-faithful).
  const int warp = tid >> 5, lane = tid & 31;
  double* scratch = sbuf + warp * 2 * PW_MAX_LEAVES;
  for (int rr = warp; rr < RT_ROWS; rr += 8) {
    if (r0 + rr >= rows) break;
    double* row = Rh + (int64_t)(r0 + rr) * M_total;
    double mx = -INFINITY;
    for (int j = lane; j < M_total; j += 32) mx = fmax(mx, row[j]);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    for (int j = lane; j < M_total; j += 32) row[j] = exp(row[j] - mx);
    __syncwarp();
    const double ssum = warp_pairwise_sum(row, M_total, scratch);
    for (int j = lane; j < M_total; j += 32) row[j] = row[j] / ssum;
    __syncwarp();
  }
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
//   * for p > 0 a value-weighted radix pass bounds n_cut, only that many top columns
//     are sorted (bitonic, smem) and scanned with the exact sequential prefix;
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

__device__ void emit_row(uint32_t* sbits, int words, int M_total, uint32_t* __restrict__ bits_row,
                         int32_t* __restrict__ kv_row, int32_t* __restrict__ cnt_out,
                         int* s_scan) {
  const int tid = threadIdx.x;
  for (int w = tid; w < words; w += blockDim.x) bits_row[w] = sbits[w];
  __syncthreads();
  if (tid < 32) {  // warp-level exclusive scan of popcounts over the row's words
    int run = 0;
    for (int w0 = 0; w0 < words; w0 += 32) {
      const int w = w0 + tid;
      const int c = (w < words) ? __popc(sbits[w]) : 0;
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (tid >= o) incl += y;
      }
      if (w < words) s_scan[w] = run + incl - c;
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (tid == 0) *cnt_out = run;
  }
  __syncthreads();
  for (int w = tid; w < words; w += blockDim.x) {
    uint32_t x = sbits[w];
    int pos = s_scan[w];
    while (x) {
      const int b = __ffs(x) - 1;
      x &= x - 1;
      kv_row[pos++] = w * 32 + b;
    }
  }
}

constexpr int SEL_THREADS = 256;

struct SelSmem {
  uint32_t hist[256];
  double hsum[256];
  int warp_tot[SEL_THREADS / 32];
  uint64_t prefix, mask;
  int remaining, n_cut, n_keep, k_ub, flag;
  double cum;
};

// Block-wide inclusive-exclusive scan helper: returns the exclusive prefix of v over
// threads in tid order; *total gets the block sum.
__device__ int block_excl_scan(int v, SelSmem& S, int* total) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) S.warp_tot[w] = incl;
  __syncthreads();
  int base = 0, tot = 0;
  for (int i = 0; i < SEL_THREADS / 32; ++i) {
    if (i < w) base += S.warp_tot[i];
    tot += S.warp_tot[i];
  }
  __syncthreads();
  *total = tot;
  return base + incl - v;
}

// MSB-first radix select of the K-th element (1-based) of the (key, column) order over
// keys[0, n).  On return S.prefix/S.mask/S.remaining describe the top-K set:
// {(key & mask) < prefix}  U  {first `remaining` columns (ascending) with (key & mask) == prefix}.
// weighted: digit choice by cumulative value sum crossing `p` (K ignored) -> bound on n_cut.
__device__ void radix_select(const uint64_t* keys, int n, int K, bool weighted, double p,
                             SelSmem& S) {
  const int tid = threadIdx.x;
  if (tid == 0) {
    S.prefix = 0; S.mask = 0; S.remaining = K; S.cum = 0.0; S.flag = 0;
  }
  __syncthreads();
  for (int byte = 7; byte >= 0; --byte) {
    for (int i = tid; i < 256; i += SEL_THREADS) {
      S.hist[i] = 0u;
      S.hsum[i] = 0.0;
    }
    __syncthreads();
    const uint64_t pre = S.prefix, msk = S.mask;
    const int sh = byte * 8;
    for (int j = tid; j < n; j += SEL_THREADS) {
      const uint64_t k = keys[j];
      if ((k & msk) != pre) continue;
      const int dg = (int)((k >> sh) & 0xFF);
      atomicAdd(&S.hist[dg], 1u);
      if (weighted) atomicAdd(&S.hsum[dg], key_value(k));
    }
    __syncthreads();
    if (tid < 32) {
      // lane owns bins [8*lane, 8*lane+8): local totals, then warp scan over lanes
      uint32_t c[8];
      double sm[8];
      uint32_t ct = 0;
      double st = 0.0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        c[i] = S.hist[tid * 8 + i];
        sm[i] = S.hsum[tid * 8 + i];
        ct += c[i];
        st += sm[i];
      }
      uint32_t cin = ct;
      double sin_ = st;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, cin, o);
        const double z = __shfl_up_sync(0xffffffffu, sin_, o);
        if (tid >= o) { cin += y; sin_ += z; }
      }
      uint32_t cex = cin - ct;
      double sex = sin_ - st;
      const int rem = S.remaining;
      const double base = S.cum;
      // find the lane whose bins contain the target, then the bin
      bool hit;
      if (weighted) hit = (base + sin_ > p) && !(base + sex > p);
      else hit = (cex < (uint32_t)rem) && ((uint32_t)rem <= cin);
      const unsigned bal = __ballot_sync(0xffffffffu, hit);
      if (bal == 0u) {
        // weighted: the total never exceeds p -> no cutoff inside this candidate set
        if (tid == 0) S.flag = 1;
      } else if (tid == __ffs(bal) - 1) {
        int bin = 7;
        for (int i = 0; i < 8; ++i) {
          const bool in = weighted ? (base + sex + sm[i] > p) : ((uint32_t)rem <= cex + c[i]);
          if (in) { bin = i; break; }
          cex += c[i];
          sex += sm[i];
        }
        const int dg = tid * 8 + bin;
        S.prefix = pre | ((uint64_t)dg << sh);
        S.mask = msk | (0xFFull << sh);
        if (weighted) {
          S.cum = base + sex;
          S.remaining = rem + (int)cex;  // elements ranked before the candidate bin
          S.hist[0] = c[bin];      // stash candidates-in-bin for the early-exit test
        } else {
          S.remaining = rem - (int)cex;
          S.hist[0] = c[bin];
        }
      }
    }
    __syncthreads();
    if (S.flag) return;
    if (!weighted && (int)S.hist[0] == S.remaining) return;  // whole bin selected
    if (weighted && S.hist[0] == 1u) return;                 // unique crossing element
    __syncthreads();
  }
}

// selected(j) for the top-K set described by S (see radix_select); also the rank of
// equal-prefix columns in ascending column order via a block scan.
__device__ void mark_selected(const uint64_t* keys, int n, SelSmem& S, uint32_t* sbits) {
  const int tid = threadIdx.x;
  const uint64_t pre = S.prefix, msk = S.mask;
  const int rem = S.remaining;
  // contiguous chunk per thread keeps ascending column order across the scan
  const int per = (n + SEL_THREADS - 1) / SEL_THREADS;
  const int j0 = tid * per, j1 = min(n, j0 + per);
  int eq = 0;
  for (int j = j0; j < j1; ++j) eq += ((keys[j] & msk) == pre);
  int total;
  int rank = block_excl_scan(eq, S, &total);
  for (int j = j0; j < j1; ++j) {
    const uint64_t km = keys[j] & msk;
    bool sel = km < pre;
    if (km == pre) sel = (rank++ < rem);
    if (sel) atomicOr(sbits + (j >> 5), 1u << (j & 31));
  }
}

// Bitonic sort (ascending (key, col)) of cnt <= n_pow2 entries in smem.
__device__ void bitonic_sort(uint64_t* key, int* col, int n_pow2) {
  const int tid = threadIdx.x;
  for (int kk = 2; kk <= n_pow2; kk <<= 1) {
    for (int jj = kk >> 1; jj > 0; jj >>= 1) {
      for (int t = tid; t < (n_pow2 >> 1); t += SEL_THREADS) {
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
      __syncthreads();
    }
  }
}

// smem layout: keys[M_total] | skey[n_pow2] | scol[n_pow2] | sbits[words] | scan[words+1]
__global__ void __launch_bounds__(SEL_THREADS) k_select(const double* __restrict__ R, int M_v,
                                                        int M_total, int n_pow2,
                                                        const uint32_t* __restrict__ adja,
                                                        int words, int n_floor, double p,
                                                        int with_union,
                                                        uint32_t* __restrict__ bits,
                                                        int32_t* __restrict__ kv_idx,
                                                        int32_t* __restrict__ kv_cnt) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem);
  uint64_t* skey = keys + M_total;
  int* scol = reinterpret_cast<int*>(skey + n_pow2);
  uint32_t* sbits = reinterpret_cast<uint32_t*>(scol + n_pow2);
  int* s_scan = reinterpret_cast<int*>(sbits + words);
  __shared__ SelSmem S;
  __shared__ int s_neg;
  const int64_t row = blockIdx.x;  // h * M_v + i
  const int i = (int)(row % M_v);
  const double* Rr = R + row * M_total;
  const int tid = threadIdx.x;
  if (tid == 0) s_neg = 0;
  for (int w = tid; w < words; w += SEL_THREADS) sbits[w] = 0u;
  __syncthreads();
  int neg = 0;
  for (int j = tid; j < M_total; j += SEL_THREADS) {
    const double v = Rr[j];
    keys[j] = desc_key(v);
    neg |= (v < 0.0);
  }
  if (__syncthreads_or(neg) && tid == 0) s_neg = 1;
  __syncthreads();

  // ---- n_cut: 1 + #(sequential sorted prefix <= p)
  if (tid == 0) { S.n_cut = -1; S.k_ub = M_total; }
  __syncthreads();
  if (!s_neg) {
    if (p == 0.0) {
      // prefix_0 = row max > 0 ends the count at once; an all-zero row never exceeds 0
      double mx = 0.0;
      for (int j = tid; j < M_total; j += SEL_THREADS) mx = fmax(mx, key_value(keys[j]));
      const int pos = __syncthreads_or(mx > 0.0);
      if (tid == 0) S.n_cut = pos ? 1 : M_total + 1;
    } else {
      radix_select(keys, M_total, 0, true, p, S);
      if (tid == 0) {
        if (S.flag) {
          S.k_ub = M_total;  // approximate total <= p: scan the whole row exactly
        } else {
          // rank of the crossing element <= (#elements with smaller key) + bin size
          const int est = S.remaining + (int)S.hist[0];
          int ub = est + 16 + est / 64;
          S.k_ub = ub < M_total ? ub : M_total;
        }
      }
      __syncthreads();
    }
  }
  __syncthreads();
  if (S.n_cut < 0) {
    // sort the top-k_ub (all columns for rows with negative entries) and scan exactly
    const int K = S.k_ub;
    int np2 = 2;
    while (np2 < K) np2 <<= 1;
    if (K < M_total) {
      radix_select(keys, M_total, K, false, 0.0, S);
      // gather the top-K set (any order) into skey/scol
      const uint64_t pre = S.prefix, msk = S.mask;
      const int rem = S.remaining;
      const int per = (M_total + SEL_THREADS - 1) / SEL_THREADS;
      const int j0 = tid * per, j1 = min(M_total, j0 + per);
      int eq = 0, cnt = 0;
      for (int j = j0; j < j1; ++j) eq += ((keys[j] & msk) == pre);
      int tot;
      int rank = block_excl_scan(eq, S, &tot);
      for (int j = j0; j < j1; ++j) {
        const uint64_t km = keys[j] & msk;
        cnt += (km < pre) || (km == pre && rank++ < rem);
      }
      int slot = block_excl_scan(cnt, S, &tot);
      rank -= eq;  // restart the equal-rank walk
      for (int j = j0; j < j1; ++j) {
        const uint64_t km = keys[j] & msk;
        bool sel = km < pre;
        if (km == pre) sel = (rank++ < rem);
        if (sel) { skey[slot] = keys[j]; scol[slot] = j; ++slot; }
      }
    } else {
      for (int j = tid; j < M_total; j += SEL_THREADS) { skey[j] = keys[j]; scol[j] = j; }
    }
    for (int j = K + tid; j < np2; j += SEL_THREADS) { skey[j] = ~0ull; scol[j] = 0x7fffffff; }
    __syncthreads();
    bitonic_sort(skey, scol, np2);
    if (tid == 0) {
      double pre = 0.0;
      int cnt = 0;
      bool crossed = false;
      for (int s2 = 0; s2 < K; ++s2) {
        pre = __dadd_rn(pre, key_value(skey[s2]));
        if (pre <= p) ++cnt;
        else if (!s_neg) { crossed = true; break; }
      }
      // non-monotone rows: every prefix counted (full row sorted); monotone rows that did
      // not cross within the bound (should not happen) -> mark for the full scan fallback
      S.n_cut = (crossed || s_neg || K == M_total) ? cnt + 1 : -2;
    }
    __syncthreads();
    if (S.n_cut == -2) {
      // exact fallback: sort everything
      int np = 2;
      while (np < M_total) np <<= 1;
      for (int j = tid; j < np; j += SEL_THREADS) {
        skey[j] = j < M_total ? keys[j] : ~0ull;
        scol[j] = j < M_total ? j : 0x7fffffff;
      }
      __syncthreads();
      bitonic_sort(skey, scol, np);
      if (tid == 0) {
        double pre = 0.0;
        int cnt = 0;
        for (int s2 = 0; s2 < M_total; ++s2) {
          pre = __dadd_rn(pre, key_value(skey[s2]));
          if (pre <= p) ++cnt; else break;
        }
        S.n_cut = cnt + 1;
      }
      __syncthreads();
    }
  }
  // ---- n_keep and the top-n_keep set
  if (tid == 0) {
    int keep = S.n_cut;
    if (keep < n_floor) keep = n_floor;
    if (keep > M_total) keep = M_total;
    S.n_keep = keep;
  }
  __syncthreads();
  radix_select(keys, M_total, S.n_keep, false, 0.0, S);
  mark_selected(keys, M_total, S, sbits);
  __syncthreads();
  if (with_union) {
    for (int w = tid; w < words; w += SEL_THREADS) {
      uint32_t x = sbits[w];
      if (adja) x |= adja[(int64_t)i * words + w];
      const int lo = w * 32;  // condition columns j >= M_v (masks.py:173)
      for (int bb = 0; bb < 32; ++bb) {
        const int j = lo + bb;
        if (j >= M_v && j < M_total) x |= 1u << bb;
      }
      sbits[w] = x;
    }
    __syncthreads();
  }
  emit_row(sbits, words, M_total, bits + row * words, kv_idx + row * M_total, kv_cnt + row, s_scan);
}

__global__ void __launch_bounds__(128) k_mask_pack(const uint8_t* __restrict__ dense, int M_total,
                                                   int words, uint32_t* __restrict__ bits,
                                                   int32_t* __restrict__ kv_idx,
                                                   int32_t* __restrict__ kv_cnt) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* sbits = reinterpret_cast<uint32_t*>(smem);
  int* s_scan = reinterpret_cast<int*>(sbits + words);
  const int64_t row = blockIdx.x;
  const uint8_t* d = dense + row * M_total;
  for (int w = threadIdx.x; w < words; w += blockDim.x) {
    uint32_t x = 0;
    for (int bb = 0; bb < 32; ++bb) {
      int j = w * 32 + bb;
      if (j < M_total && d[j]) x |= 1u << bb;
    }
    sbits[w] = x;
  }
  __syncthreads();
  emit_row(sbits, words, M_total, bits + row * words, kv_idx + row * M_total, kv_cnt + row, s_scan);
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

extern "C" int tcb_block_pool(const void* x0, const void* x1, int dtype, int64_t stride_h,
                              int64_t stride_n, int H, int d, int m, int M_v, int M_total,
                              int64_t n_valid, int64_t n_cond, double* out0, double* out1,
                              void* stream) {
  TCB_CHECK_ARG(x0 && out0, TCB_ESHAPE, "null tensor");
  TCB_CHECK_ARG((x1 == nullptr) == (out1 == nullptr), TCB_ESHAPE, "x1/out1 must both be set");
  TCB_CHECK_ARG(H >= 1 && d >= 1 && m >= 1 && M_total >= M_v && M_v >= 0, TCB_ESHAPE,
                "bad pool shape");
  TCB_CHECK_ARG(dtype == TCB_F32 || dtype == TCB_BF16, TCB_EDOMAIN, "unsupported dtype %d", dtype);
  if ((int64_t)H * M_total == 0) return TCB_OK;
  const int esz = dtype == TCB_F32 ? 4 : 2;
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
  if (dtype == TCB_F32) {
    if (vec)
      k_pool<float, true><<<grid, 128, 0, s>>>((const float*)x0, (const float*)x1, stride_h,
                                               stride_n, H, d, m, M_v, M_total, n_valid, n_cond,
                                               out0, out1, G, chunks);
    else
      k_pool<float, false><<<grid, 128, 0, s>>>((const float*)x0, (const float*)x1, stride_h,
                                                stride_n, H, d, m, M_v, M_total, n_valid, n_cond,
                                                out0, out1, G, chunks);
  } else {
    using B = __nv_bfloat16;
    if (vec)
      k_pool<B, true><<<grid, 128, 0, s>>>((const B*)x0, (const B*)x1, stride_h, stride_n, H, d,
                                           m, M_v, M_total, n_valid, n_cond, out0, out1, G,
                                           chunks);
    else
      k_pool<B, false><<<grid, 128, 0, s>>>((const B*)x0, (const B*)x1, stride_h, stride_n, H, d,
                                            m, M_v, M_total, n_valid, n_cond, out0, out1, G,
                                            chunks);
  }
  return check_launch("k_pool");
}

extern "C" int tcb_block_relevance(const double* pq, int pq_blocks, const double* pk, int H,
                                   int rows, int M_total, int d, double* R, void* stream) {
  TCB_CHECK_ARG(pq && pk && R, TCB_ESHAPE, "null tensor");
  TCB_CHECK_ARG(H >= 1 && rows >= 0 && rows <= pq_blocks && M_total >= 1 && d >= 1, TCB_ESHAPE,
                "bad relevance shape");
  TCB_CHECK_ARG(M_total <= 16384, TCB_ESIZE, "M_total %d > 16384 unsupported", M_total);
  if (rows == 0) return TCB_OK;
  dim3 grid((unsigned)ceil_div(rows, RT_ROWS), H);
  k_relevance<<<grid, 256, 0, as_stream(stream)>>>(pq, pq_blocks, pk, rows, M_total, d, 0.0,
                                                   sqrt((double)d), R);
  return check_launch("k_relevance");
}

extern "C" int tcb_block_select(const double* R, int H, int M_v, int M_total,
                                const uint32_t* adja, int words, int n_floor, double p,
                                int with_union, uint32_t* bits, int32_t* kv_idx, int32_t* kv_cnt,
                                void* stream) {
  TCB_CHECK_ARG(R && bits && kv_idx && kv_cnt, TCB_ESHAPE, "null tensor");
  TCB_CHECK_ARG(H >= 1 && M_v >= 0 && M_total >= 1, TCB_ESHAPE, "bad select shape");
  TCB_CHECK_ARG(words >= ceil_div(M_total, 32), TCB_ESHAPE, "words too small");
  TCB_CHECK_ARG(M_total <= 16384, TCB_ESIZE, "M_total %d > 16384 unsupported", M_total);
  if ((int64_t)H * M_v == 0) return TCB_OK;
  int n_pow2 = 1;
  while (n_pow2 < M_total) n_pow2 <<= 1;
  if (n_pow2 < 2) n_pow2 = 2;
  const size_t smem = (size_t)M_total * 8 + (size_t)n_pow2 * (8 + 4) + (size_t)words * 4 +
                      (size_t)(words + 1) * 4;
  cudaStream_t s = as_stream(stream);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return set_error(TCB_ECUDA, "k_select smem: %s", cudaGetErrorString(e));
  }
  k_select<<<(unsigned)((int64_t)H * M_v), SEL_THREADS, smem, s>>>(
      R, M_v, M_total, n_pow2, adja, words, n_floor, p, with_union, bits, kv_idx, kv_cnt);
  return check_launch("k_select");
}

extern "C" int tcb_mask_pack(const uint8_t* dense, int64_t rows, int M_total, int words,
                             uint32_t* bits, int32_t* kv_idx, int32_t* kv_cnt, void* stream) {
  TCB_CHECK_ARG(dense && bits && kv_idx && kv_cnt, TCB_ESHAPE, "null tensor");
  TCB_CHECK_ARG(words >= ceil_div(M_total, 32), TCB_ESHAPE, "words too small");
  if (rows == 0) return TCB_OK;
  const size_t smem = (size_t)words * 4 + (size_t)(words + 1) * 4;
  k_mask_pack<<<(unsigned)rows, 128, smem, as_stream(stream)>>>(dense, M_total, words, bits,
                                                                kv_idx, kv_cnt);
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
