// Shared helpers for the sm_100a kernels: status/error plumbing and launch checks.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>

#include "../../include/tokencarve_b200.h"

namespace tcb {

int set_error(int code, const char* fmt, ...);

// After a launch: map a launch/runtime error to TCB_ECUDA.
int check_launch(const char* what);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Valid tokens in block b of the layout [vision | pad | cond | pad]
// (partition.py:3-13, 83-88): valid tokens always form a prefix of the block.
__host__ __device__ __forceinline__ int block_valid(int b, int m, int M_v, int64_t n_valid,
                                                    int64_t n_cond) {
  int64_t start, cnt;
  if (b < M_v) {
    start = (int64_t)b * m;
    cnt = n_valid - start;
  } else {
    start = (int64_t)(b - M_v) * m;
    cnt = n_cond - start;
  }
  if (cnt < 0) cnt = 0;
  if (cnt > m) cnt = m;
  return (int)cnt;
}

// Ascending walk over the set bits of one packed mask row (32 columns per uint32 word,
// column j = bit j % 32 of word j / 32): the mask's kv list without a materialised CSR.
// Every calling thread runs it identically (uniform, L1-resident loads); get(j) returns the
// j-th set column for non-decreasing j -- kv_idx[j] of the reference's ascending
// flatnonzero(bits[h, qb]) (attention.py:179).  The caller bounds j by the row's count.
struct BitWalk {
  const uint32_t* row;
  int w, j, b;
  uint32_t cur;
  __device__ explicit BitWalk(const uint32_t* r) : row(r), w(-1), j(-1), b(0), cur(0u) {}
  __device__ __forceinline__ int get(int jj) {
    while (j < jj) {
      while (cur == 0u) cur = __ldg(row + ++w);
      b = w * 32 + __ffs((int)cur) - 1;
      cur &= cur - 1u;
      ++j;
    }
    return b;
  }
};

// Warp-cooperative kv list for the carve kernel's producer and softmax warps (all 32 lanes
// call block() with the same j, j ascending): the row's words are loaded once per item (one
// coalesced load, lane i holds word i) with an exclusive popc prefix across lanes; then every
// 32 list entries each lane decodes one of them (5-step shuffle search for its word + fns)
// and block(j) is a single shuffle -- the kv_idx CSR's cost profile without storing it.
// Rows of more than 32 words (M_total > 1024) walk the bits per block instead.
struct WarpKvList {
  const uint32_t* row;
  int words, lane, chunk, cache, pre;
  uint32_t mine;
  BitWalk slow;
  __device__ WarpKvList(const uint32_t* r, int words_, int lane_)
      : row(r), words(words_), lane(lane_), chunk(-1), cache(0), pre(0), mine(0u), slow(r) {
    if (!r || words > 32) return;
    mine = lane < words ? __ldg(r + lane) : 0u;
    int c = __popc(mine), inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    pre = inc - c;  // set bits in words before mine
  }
  __device__ __forceinline__ int block(int j) {
    if (words > 32) return slow.get(j);
    const int c = j >> 5;
    if (c != chunk) {
      chunk = c;
      const int r = c * 32 + lane;  // this lane decodes list entry r
      int i = 0;                    // last word with pre <= r (pre is non-decreasing)
#pragma unroll
      for (int step = 16; step; step >>= 1) {
        const int p = __shfl_sync(0xffffffffu, pre, i + step);
        if (p <= r) i += step;
      }
      const uint32_t wd = __shfl_sync(0xffffffffu, mine, i);
      const int k = r - __shfl_sync(0xffffffffu, pre, i);
      cache = (k < __popc(wd)) ? i * 32 + (int)__fns(wd, 0, k + 1) : 0;
    }
    return __shfl_sync(0xffffffffu, cache, j & 31);
  }
};

// What the softmax warps need from a vision row's kv list without decoding it: the list is
// ascending, so its vision blocks (< M_v) come first and its condition blocks last.  Only
// the last vision block (M_v - 1) and the last condition block (M_total - 1) can be partial,
// and they can only sit at list positions n_vis - 1 and n - 1.  Warp-uniform; one coalesced
// load per 32 words.
struct RowShape {
  int n_vis;        // kv entries < M_v (condition keys start at position n_vis)
  int kv_last_vis;  // valid keys of entry n_vis - 1 (m unless it is the partial block M_v - 1)
  int kv_last;      // valid keys of entry n - 1 when it is the partial block M_total - 1, else m
  __device__ RowShape() : n_vis(0), kv_last_vis(0), kv_last(0) {}
  __device__ RowShape(const uint32_t* row, int words, int lane, int m, int M_v, int M_total,
                      int64_t n_valid, int64_t n_cond) {
    int cnt = 0;
    for (int w0 = 0; w0 < words; w0 += 32) {
      const int w = w0 + lane;
      uint32_t x = w < words ? __ldg(row + w) : 0u;
      const int lo = w * 32;  // keep columns < M_v
      x = lo >= M_v ? 0u : (lo + 32 <= M_v ? x : (x & ((1u << (M_v - lo)) - 1u)));
      cnt += __popc(x);
    }
    n_vis = __reduce_add_sync(0xffffffffu, cnt);
    const bool has_lv = (__ldg(row + (M_v - 1) / 32) >> ((M_v - 1) & 31)) & 1u;
    const bool has_lc = M_total > M_v && ((__ldg(row + (M_total - 1) / 32) >> ((M_total - 1) & 31)) & 1u);
    kv_last_vis = has_lv ? block_valid(M_v - 1, m, M_v, n_valid, n_cond) : m;
    kv_last = has_lc ? block_valid(M_total - 1, m, M_v, n_valid, n_cond) : m;
  }
};

}  // namespace tcb

#define TCB_CHECK_ARG(cond, code, ...)                  \
  do {                                                  \
    if (!(cond)) return ::tcb::set_error(code, __VA_ARGS__); \
  } while (0)
