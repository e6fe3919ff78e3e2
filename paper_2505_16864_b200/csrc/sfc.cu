// K1 curve index builder, K2 row gather, K6 block adjacency (HBM / latency bound).
//
// K1  tcb_curve_build      <- build_curve        sfc.py:198-210
// K2  tcb_gather_rows      <- _permute           sfc.py:213-237
// K6  tcb_adjacency_build  <- adjacency_mask     partition.py:107-136
#include "common.cuh"
#include "gilbert.cuh"

namespace tcb {

// One thread per row-major cell: descend the plane split tree, compose the slab
// position, scatter both directions.  inv[] stores are coalesced, fwd[] scattered.
__global__ void __launch_bounds__(256) k_curve(CurveGeom g, int64_t n, int32_t* __restrict__ fwd,
                                               int32_t* __restrict__ inv) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  int64_t pos = curve_position(g, c);
  inv[c] = (int32_t)pos;
  fwd[pos] = (int32_t)c;
}

// Row gather with 2^LOG_V-byte vectors; a group of `lanes` threads copies one row,
// every thread keeps UNROLL independent vector loads in flight before storing.
template <typename V, int UNROLL>
__global__ void __launch_bounds__(256) k_gather(const V* __restrict__ src, V* __restrict__ dst,
                                                const int32_t* __restrict__ idx, int64_t rows,
                                                int64_t vpr, int lanes) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t groups = ((int64_t)gridDim.x * blockDim.x) / lanes;
  const int lane = (int)(tid % lanes);
  for (int64_t r = tid / lanes; r < rows; r += groups) {
    const int64_t s = __ldg(idx + r);
    const V* sp = src + s * vpr;
    V* dp = dst + r * vpr;
    int64_t c = lane;
    for (; c + (UNROLL - 1) * lanes < vpr; c += UNROLL * lanes) {
      V buf[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) buf[u] = __ldcs(sp + c + u * lanes);
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) __stcs(dp + c + u * lanes, buf[u]);
    }
    for (; c < vpr; c += lanes) __stcs(dp + c, __ldcs(sp + c));
  }
}

__device__ __forceinline__ void set_bit(uint32_t* rowp, int j) {
  atomicOr(rowp + (j >> 5), 1u << (j & 31));
}

// One thread per cell; the 13 lexicographically positive offsets cover every
// unordered neighbour pair once (partition.py:29-35); both directions are set so
// the result is already symmetric; the diagonal is set by the first M_v threads.
__global__ void __launch_bounds__(256) k_adjacency(const int32_t* __restrict__ inv, int t, int h,
                                                   int w, int m, int M_v, int words,
                                                   uint32_t* __restrict__ adja) {
  const int64_t n = (int64_t)t * h * w;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < M_v) set_bit(adja + c * words, (int)c);
  if (c >= n) return;
  const int64_t hw = (int64_t)h * w;
  const int ct = (int)(c / hw);
  const int ch = (int)((c - (int64_t)ct * hw) / w);
  const int cw = (int)(c - (int64_t)ct * hw - (int64_t)ch * w);
  const int b0 = __ldg(inv + c) / m;
#pragma unroll
  for (int o = 0; o < 13; ++o) {
    // offsets (dt,dh,dw) > (0,0,0): dt=1 -> 9 offsets, dt=0,dh=1 -> 3, dt=0,dh=0,dw=1 -> 1
    int dt, dh, dw;
    if (o < 9) { dt = 1; dh = o / 3 - 1; dw = o % 3 - 1; }
    else if (o < 12) { dt = 0; dh = 1; dw = o - 10; }
    else { dt = 0; dh = 0; dw = 1; }
    const int nt = ct + dt, nh = ch + dh, nw = cw + dw;
    if (nt >= t || nh < 0 || nh >= h || nw < 0 || nw >= w) continue;
    const int b1 = __ldg(inv + (int64_t)nt * hw + (int64_t)nh * w + nw) / m;
    if (b1 == b0) continue;
    set_bit(adja + (int64_t)b0 * words, b1);
    set_bit(adja + (int64_t)b1 * words, b0);
  }
}

}  // namespace tcb

using namespace tcb;

extern "C" int tcb_curve_build(int t, int h, int w, int32_t* fwd, int32_t* inv, void* stream) {
  TCB_CHECK_ARG(t >= 1 && h >= 1 && w >= 1, TCB_ESHAPE, "grid axes must be >= 1, got %d,%d,%d", t,
                h, w);
  const int64_t n = (int64_t)t * h * w;
  TCB_CHECK_ARG(n < (int64_t(1) << 31), TCB_ESIZE,
                "%lld cells exceed the int32 device index range", (long long)n);
  TCB_CHECK_ARG(fwd && inv, TCB_ESHAPE, "null output");
  CurveGeom g = curve_geom(t, h, w);
  k_curve<<<(unsigned)ceil_div(n, 256), 256, 0, as_stream(stream)>>>(g, n, fwd, inv);
  return check_launch("k_curve");
}

extern "C" int tcb_gather_rows(const void* src, void* dst, const int32_t* idx, int64_t rows,
                               int64_t row_bytes, int64_t src_rows, void* stream) {
  TCB_CHECK_ARG(rows >= 0 && row_bytes >= 0 && src_rows >= 0, TCB_ESHAPE, "negative size");
  if (rows == 0 || row_bytes == 0) return TCB_OK;
  TCB_CHECK_ARG(src && dst && idx, TCB_ESHAPE, "null pointer");
  const uintptr_t align = (uintptr_t)src | (uintptr_t)dst | (uintptr_t)row_bytes;
  const cudaStream_t s = as_stream(stream);
  auto launch = [&](auto tag, int vbytes) {
    using V = decltype(tag);
    const int64_t vpr = row_bytes / vbytes;
    int lanes = 1;
    while (lanes < 32 && lanes < vpr) lanes <<= 1;
    const int64_t groups_needed = rows;
    int64_t blocks = ceil_div(groups_needed * lanes, 256);
    const int64_t cap = 148 * 16;  // enough resident warps to saturate HBM, grid-stride after
    if (blocks > cap) blocks = cap;
    k_gather<V, 4><<<(unsigned)blocks, 256, 0, s>>>((const V*)src, (V*)dst, idx, rows, vpr, lanes);
  };
  if (align % 16 == 0) launch(int4{}, 16);
  else if (align % 8 == 0) launch(int2{}, 8);
  else if (align % 4 == 0) launch(int{}, 4);
  else if (align % 2 == 0) launch(short{}, 2);
  else launch(char{}, 1);
  return check_launch("k_gather");
}

extern "C" int tcb_adjacency_build(const int32_t* inv, int t, int h, int w, int m, int M_v,
                                   int words, uint32_t* adja, void* stream) {
  TCB_CHECK_ARG(t >= 1 && h >= 1 && w >= 1 && m >= 1, TCB_ESHAPE, "bad dims/block size");
  const int64_t n = (int64_t)t * h * w;
  TCB_CHECK_ARG(M_v == ceil_div(n, m), TCB_ESHAPE, "M_v %d inconsistent with %lld cells / m=%d",
                M_v, (long long)n, m);
  TCB_CHECK_ARG(words >= ceil_div(M_v, 32), TCB_ESHAPE, "words %d < ceil(M_v/32)", words);
  cudaStream_t s = as_stream(stream);
  cudaError_t e = cudaMemsetAsync(adja, 0, sizeof(uint32_t) * (size_t)M_v * words, s);
  if (e != cudaSuccess) return set_error(TCB_ECUDA, "memset adjacency: %s", cudaGetErrorString(e));
  const int64_t threads = n > M_v ? n : M_v;
  k_adjacency<<<(unsigned)ceil_div(threads, 256), 256, 0, s>>>(inv, t, h, w, m, M_v, words, adja);
  return check_launch("k_adjacency");
}
