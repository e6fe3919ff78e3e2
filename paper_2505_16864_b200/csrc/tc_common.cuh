// tcgen05 helpers shared by the carve kernels (carve.cu: bf16/fp16 k_carve_tc; carve_x3.cu:
// fp32 inputs as fp16 hi/lo splits): instruction / shared-memory descriptors, packed-fp32
// arithmetic, 16-bit element traits, TMA tensor maps and per-device kernel attributes.
#pragma once
#include <atomic>
#include <mutex>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include "common.cuh"
#include "ptx.cuh"

namespace tcb {

struct CarveShape {
  int H, d, m, M_v, M_total, W;  // W = uint32 words per packed mask row
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

namespace tc {

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
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
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
// x is clamped to [-126, 126] so the exponent never wraps into the sign bit (the max-free
// carve step feeds x > 0 before it knows the block max; 2^126 still trips its redo check).
__device__ __forceinline__ uint64_t exp2_poly2(uint64_t x) {
  const float x0 = fmaxf(fminf(f2_lo(x), 126.f), -126.f);
  const float x1 = fmaxf(fminf(f2_hi(x), 126.f), -126.f);
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

}  // namespace tc

// ---------------------------------------------------------------- host helpers
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static inline PFN_encodeTiled get_encode() {
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
static inline int make_tmap(CUtensorMap* tm, const void* base, int d, int64_t n_pad, int H, int64_t sh,
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

// (64, N_pad, d/64, H) view of a (H, N_pad, d) 16-bit tensor with box (64, box_rows, d/64, 1):
// one TMA request brings all 64-column chunks of a row range, landing chunk-major -- the
// same shared-memory layout as d/64 separate 3D boxes (128-byte swizzle per chunk).
static inline int make_tmap_rows(CUtensorMap* tm, const void* base, int d, int64_t n_pad, int H,
                                 int64_t sh, int64_t sn, int box_rows, bool f16 = false) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return set_error(TCB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[4] = {64, (cuuint64_t)n_pad, (cuuint64_t)(d / 64), (cuuint64_t)H};
  cuuint64_t strides[3] = {(cuuint64_t)sn * 2, 128, (cuuint64_t)sh * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)box_rows, (cuuint32_t)(d / 64), 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(tm, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(TCB_ECUDA, "cuTensorMapEncodeTiled (rows) failed (%d)", (int)r);
  return TCB_OK;
}

// Kernel attributes are per device: set one once per device under a lock, and remember the
// device only after cudaFuncSetAttribute succeeded (a failure is retried on the next launch).
template <typename F>
static inline cudaError_t once_per_device(std::atomic<uint64_t>& seen, F&& set_attr) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (seen.load(std::memory_order_acquire) & bit) return cudaSuccess;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (seen.load(std::memory_order_relaxed) & bit) return cudaSuccess;
  const cudaError_t e = set_attr();
  if (e == cudaSuccess) seen.fetch_or(bit, std::memory_order_release);
  return e;
}

}  // namespace tcb
