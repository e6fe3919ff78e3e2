// K9/K10 progressive-resolution stage switch: predict_clean -> area upsample ->
// re-noise in one pass over the target latent, plus the Euler step.
//
//   predict_clean      pipeline.py:124-128   x0 = x - sigma * v          (float32)
//   upsample_area_3d   pipeline.py:140-173   separable area weights, float64 taps
//   stage_transition   pipeline.py:176-194   (1 - s) * up + s * eps     (float32)
//   denoise_step       pipeline.py:131-137   x + (s_next - s) * v       (float32)
//
// Upsampling (dst >= src per axis) gives every output at most two source taps per
// axis; the float64 weights are recomputed per output exactly like _axis_weights
// (overlap / step).  The reference applies the axes in order 0 -> 1 -> 2 with a
// float64 intermediate; the kernel accumulates the same products in the same
// axis order, so results agree to float64 rounding before the float32 cast.
#include "common.cuh"

#include <math.h>

namespace tcb {

struct Taps {
  int i0, n;
  double w0, w1;
};

// overlap weights of output o along one axis (pipeline.py:140-150)
__device__ __forceinline__ Taps axis_taps(int o, int src, int dst) {
  Taps t;
  if (src == dst) {
    t.i0 = o; t.n = 1; t.w0 = 1.0; t.w1 = 0.0;
    return t;
  }
  const double step = (double)src / (double)dst;
  const double lo = o * step, hi = (o + 1) * step;
  const int i0 = (int)floor(lo);
  int i1 = (int)ceil(hi);
  if (i1 > src) i1 = src;
  t.i0 = i0; t.n = 0; t.w0 = 0.0; t.w1 = 0.0;
  for (int i = i0; i < i1 && t.n < 2; ++i) {
    const double a = fmax(0.0, fmin(hi, (double)(i + 1)) - fmax(lo, (double)i));
    if (t.n == 0) t.w0 = a / step; else t.w1 = a / step;
    ++t.n;
  }
  return t;
}

// Philox4x32-10 (counter-based) + Box-Muller, for production noise.
__device__ __forceinline__ void philox(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
    c[0] = n0; c[1] = (uint32_t)p1; c[2] = n2; c[3] = (uint32_t)p0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}
__device__ __forceinline__ float philox_normal(uint64_t seed, uint64_t idx) {
  uint32_t c[4] = {(uint32_t)(idx >> 1), (uint32_t)(idx >> 33), 0u, 0u};
  philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  const float u1 = ((float)(c[0] >> 8) + 0.5f) * (1.0f / 16777216.0f);
  const float u2 = ((float)(c[1] >> 8) + 0.5f) * (1.0f / 16777216.0f);
  const float r = sqrtf(-2.0f * logf(u1));
  return (idx & 1) ? r * sinf(6.283185307179586f * u2) : r * cosf(6.283185307179586f * u2);
}

__global__ void __launch_bounds__(256) k_upsample_renoise(
    const float* __restrict__ x, const float* __restrict__ vel, const int32_t* __restrict__ inv,
    const float* __restrict__ eps, float* __restrict__ out, int st, int sh, int sw, int dt, int dh,
    int dw, int C, float sigma_f, int mode, uint64_t seed, uint64_t offset) {
  const int64_t n = (int64_t)dt * dh * dw * C;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const int c = (int)(e % C);
  int64_t cell = e / C;
  const int ow = (int)(cell % dw);
  cell /= dw;
  const int oh = (int)(cell % dh);
  const int ot = (int)(cell / dh);
  const Taps tt = axis_taps(ot, st, dt), th = axis_taps(oh, sh, dh), tw = axis_taps(ow, sw, dw);
  // same axis order as the reference's separable tensordots: t, then h, then w
  double acc_w = 0.0;
  for (int b = 0; b < tw.n; ++b) {
    double acc_h = 0.0;
    for (int a = 0; a < th.n; ++a) {
      double acc_t = 0.0;
      for (int z = 0; z < tt.n; ++z) {
        const int64_t cell = ((int64_t)(tt.i0 + z) * sh + (th.i0 + a)) * sw + (tw.i0 + b);
        const int64_t src = cell * C + c;
        float x0 = x[src];
        if (vel) {  // predict_clean in fp32; a curve-order velocity is read through inv
          const float v = vel[(inv ? (int64_t)inv[cell] : cell) * C + c];
          x0 = __fsub_rn(x0, __fmul_rn(sigma_f, v));
        }
        acc_t += (z == 0 ? tt.w0 : tt.w1) * (double)x0;
      }
      acc_h += (a == 0 ? th.w0 : th.w1) * acc_t;
    }
    acc_w += (b == 0 ? tw.w0 : tw.w1) * acc_h;
  }
  const float up = (float)acc_w;
  if (mode == 0) {
    out[e] = up;
    return;
  }
  const float nz = (mode == 1) ? eps[e] : philox_normal(seed, offset + (uint64_t)e);
  // (1 - s) * up + s * noise, each op rounded like numpy's float32 arrays
  out[e] = __fadd_rn(__fmul_rn(__fsub_rn(1.0f, sigma_f), up), __fmul_rn(sigma_f, nz));
}

__global__ void k_euler(const float* __restrict__ x, const float* __restrict__ v,
                        float* __restrict__ out, int64_t n, float ds) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) out[e] = __fadd_rn(x[e], __fmul_rn(ds, v[e]));
}

}  // namespace tcb

using namespace tcb;

extern "C" int tcb_upsample_renoise(const float* x, const float* vel, const float* eps, float* out,
                                    int st, int sh, int sw, int dt, int dh, int dw, int C,
                                    double sigma, int mode, uint64_t seed, uint64_t offset,
                                    void* stream) {
  TCB_CHECK_ARG(x && out, TCB_ESHAPE, "null tensor");
  TCB_CHECK_ARG(st >= 1 && sh >= 1 && sw >= 1 && C >= 1, TCB_ESHAPE, "bad source dims");
  TCB_CHECK_ARG(dt >= st && dh >= sh && dw >= sw, TCB_EDOMAIN, "target shrinks source");
  TCB_CHECK_ARG(mode >= 0 && mode <= 2, TCB_EDOMAIN, "bad mode %d", mode);
  TCB_CHECK_ARG(mode != 1 || eps, TCB_ESHAPE, "mode 1 needs eps");
  TCB_CHECK_ARG(sigma >= 0.0 && sigma <= 1.0, TCB_EDOMAIN, "sigma %g outside [0, 1]", sigma);
  const int64_t n = (int64_t)dt * dh * dw * C;
  k_upsample_renoise<<<(unsigned)ceil_div(n, 256), 256, 0, as_stream(stream)>>>(
      x, vel, nullptr, eps, out, st, sh, sw, dt, dh, dw, C, (float)sigma, mode, seed, offset);
  return check_launch("k_upsample_renoise");
}

extern "C" int tcb_upsample_renoise_curve(const float* x, const float* vel_curve,
                                          const int32_t* inv, const float* eps, float* out, int st,
                                          int sh, int sw, int dt, int dh, int dw, int C,
                                          double sigma, int mode, uint64_t seed, uint64_t offset,
                                          void* stream) {
  TCB_CHECK_ARG(x && out && vel_curve && inv, TCB_ESHAPE, "null tensor");
  TCB_CHECK_ARG(st >= 1 && sh >= 1 && sw >= 1 && C >= 1, TCB_ESHAPE, "bad source dims");
  TCB_CHECK_ARG(dt >= st && dh >= sh && dw >= sw, TCB_EDOMAIN, "target shrinks source");
  TCB_CHECK_ARG(mode >= 0 && mode <= 2, TCB_EDOMAIN, "bad mode %d", mode);
  TCB_CHECK_ARG(mode != 1 || eps, TCB_ESHAPE, "mode 1 needs eps");
  TCB_CHECK_ARG(sigma >= 0.0 && sigma <= 1.0, TCB_EDOMAIN, "sigma %g outside [0, 1]", sigma);
  const int64_t n = (int64_t)dt * dh * dw * C;
  k_upsample_renoise<<<(unsigned)ceil_div(n, 256), 256, 0, as_stream(stream)>>>(
      x, vel_curve, inv, eps, out, st, sh, sw, dt, dh, dw, C, (float)sigma, mode, seed, offset);
  return check_launch("k_upsample_renoise");
}

extern "C" int tcb_euler_step(const float* x, const float* v, float* out, int64_t n, float dsigma,
                              void* stream) {
  TCB_CHECK_ARG(x && v && out, TCB_ESHAPE, "null tensor");
  if (n == 0) return TCB_OK;
  k_euler<<<(unsigned)ceil_div(n, 256), 256, 0, as_stream(stream)>>>(x, v, out, n, dsigma);
  return check_launch("k_euler");
}
