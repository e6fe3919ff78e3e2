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

// numpy's pairwise summation (PW_BLOCKSIZE 128, 8-way unrolled leaves)
__device__ double pairwise_sum(const double* a, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res += a[i];
    return res;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  // iterative form of the recursive split: explicit stack of (offset, length)
  int st_off[32], st_len[32];
  double st_val[32];
  int st_state[32];
  int sp = 0;
  st_off[0] = 0; st_len[0] = n; st_state[0] = 0; sp = 1;
  double ret = 0.0;
  while (sp > 0) {
    int top = sp - 1;
    int off = st_off[top], len = st_len[top];
    if (len <= 128) {
      // leaf
      const double* p = a + off;
      double res;
      if (len < 8) {
        res = 0.0;
        for (int i = 0; i < len; ++i) res += p[i];
      } else {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = p[j];
        int i = 8;
        for (; i < len - (len % 8); i += 8)
          for (int j = 0; j < 8; ++j) r[j] += p[i + j];
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < len; ++i) res += p[i];
      }
      --sp;
      ret = res;
      // propagate to parent
      while (sp > 0) {
        int pt = sp - 1;
        if (st_state[pt] == 0) {  // left child finished -> push right child
          st_val[pt] = ret;
          st_state[pt] = 1;
          int n2 = st_len[pt] / 2;
          n2 -= n2 % 8;
          st_off[sp] = st_off[pt] + n2;
          st_len[sp] = st_len[pt] - n2;
          st_state[sp] = 0;
          ++sp;
          break;
        } else {  // right child finished
          ret = st_val[pt] + ret;
          --sp;
        }
      }
    } else {
      int n2 = len / 2;
      n2 -= n2 % 8;
      st_off[sp] = off;
      st_len[sp] = n2;
      st_state[sp] = 0;
      ++sp;
    }
  }
  return ret;
}

__global__ void __launch_bounds__(256) k_relevance(const double* __restrict__ pq, int pq_blocks,
                                                   const double* __restrict__ pk, int rows,
                                                   int M_total, int d, double inv_sqrt_unused,
                                                   double sqrt_d, double* __restrict__ R) {
  __shared__ double sA[RT_ROWS][RT_KC + 1];
  __shared__ double sB[RT_KC][RT_COLS + 1];
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
  // per-row softmax (masks.py:132-134); 32 rows -> 32 threads, row-sequential
  if (tid < RT_ROWS && r0 + tid < rows) {
    double* row = Rh + (int64_t)(r0 + tid) * M_total;
    double mx = -INFINITY;
    for (int j = 0; j < M_total; ++j) mx = fmax(mx, row[j]);
    for (int j = 0; j < M_total; ++j) row[j] = exp(row[j] - mx);
    const double s = pairwise_sum(row, M_total);
    for (int j = 0; j < M_total; ++j) row[j] = row[j] / s;
  }
}

// ---------------------------------------------------------------------------
// K5 selection.  CTA per (head, vision row).  Bitonic sort in smem of
// (order-preserving key of -R, column) pairs == stable descending argsort
// (masks.py:150); thread 0 walks the sorted probabilities with the sequential
// float64 prefix of np.cumsum (masks.py:152-153); the first n_keep columns are
// set, ORed with the condition columns and the adjacency row (masks.py:173-174),
// and the row is emitted packed plus as an ascending CSR kv list.
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
  // exclusive prefix of popcounts over words (words <= 4 * blockDim), simple 2-level scan
  for (int w = tid; w < words; w += blockDim.x) bits_row[w] = sbits[w];
  __syncthreads();
  if (tid == 0) {
    int run = 0;
    for (int w = 0; w < words; ++w) {
      s_scan[w] = run;
      run += __popc(sbits[w]);
    }
    s_scan[words] = run;
    *cnt_out = run;
  }
  __syncthreads();
  for (int w = tid; w < words; w += blockDim.x) {
    uint32_t x = sbits[w];
    int pos = s_scan[w];
    while (x) {
      int b = __ffs(x) - 1;
      x &= x - 1;
      kv_row[pos++] = w * 32 + b;
    }
  }
}

__global__ void __launch_bounds__(256) k_select(const double* __restrict__ R, int M_v, int M_total,
                                                int n_pow2, const uint32_t* __restrict__ adja,
                                                int words, int n_floor, double p, int with_union,
                                                uint32_t* __restrict__ bits,
                                                int32_t* __restrict__ kv_idx,
                                                int32_t* __restrict__ kv_cnt) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* key = reinterpret_cast<uint64_t*>(smem);
  int* col = reinterpret_cast<int*>(key + n_pow2);
  uint32_t* sbits = reinterpret_cast<uint32_t*>(col + n_pow2);
  int* s_scan = reinterpret_cast<int*>(sbits + words);
  __shared__ int s_keep;
  const int64_t row = blockIdx.x;  // h * M_v + i
  const int i = (int)(row % M_v);
  const double* Rr = R + row * M_total;
  const int tid = threadIdx.x;
  for (int j = tid; j < n_pow2; j += blockDim.x) {
    if (j < M_total) {
      key[j] = desc_key(Rr[j]);
      col[j] = j;
    } else {
      key[j] = ~0ull;
      col[j] = 0x7fffffff;
    }
  }
  for (int w = tid; w < words; w += blockDim.x) sbits[w] = 0u;
  __syncthreads();
  for (int kk = 2; kk <= n_pow2; kk <<= 1) {
    for (int jj = kk >> 1; jj > 0; jj >>= 1) {
      for (int t = tid; t < (n_pow2 >> 1); t += blockDim.x) {
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
  if (tid == 0) {
    // np.cumsum is sequential; count prefix <= p (masks.py:152-153).  With all
    // values >= 0 the prefix is monotone and the walk can stop at the first miss.
    const bool nonneg = key_value(key[M_total - 1]) >= 0.0;
    double pre = 0.0;
    int cnt = 0;
    for (int s = 0; s < M_total; ++s) {
      pre = __dadd_rn(pre, key_value(key[s]));
      if (pre <= p) ++cnt;
      else if (nonneg) break;
    }
    int keep = cnt + 1;
    if (keep < n_floor) keep = n_floor;
    if (keep > M_total) keep = M_total;
    s_keep = keep;
  }
  __syncthreads();
  const int keep = s_keep;
  for (int s = tid; s < keep; s += blockDim.x) {
    const int c = col[s];
    atomicOr(sbits + (c >> 5), 1u << (c & 31));
  }
  __syncthreads();
  if (with_union) {
    for (int w = tid; w < words; w += blockDim.x) {
      uint32_t x = sbits[w];
      if (adja) x |= adja[(int64_t)i * words + w];
      // condition columns j >= M_v (masks.py:173)
      const int lo = w * 32;
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
  const size_t smem = (size_t)n_pow2 * (8 + 4) + (size_t)words * 4 + (size_t)(words + 1) * 4;
  cudaStream_t s = as_stream(stream);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return set_error(TCB_ECUDA, "k_select smem: %s", cudaGetErrorString(e));
  }
  k_select<<<(unsigned)((int64_t)H * M_v), 256, smem, s>>>(
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
