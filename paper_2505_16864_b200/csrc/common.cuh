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

}  // namespace tcb

#define TCB_CHECK_ARG(cond, code, ...)                  \
  do {                                                  \
    if (!(cond)) return ::tcb::set_error(code, __VA_ARGS__); \
  } while (0)
