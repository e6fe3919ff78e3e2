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

// Output cell -> source taps, computed once per (cell, 4-channel group) thread and reused
// for every channel of the group.  VEC = channels per thread (4: float4 / 2x double2 loads and
// stores along C; 1: any C).  Index math is int32 (the host guarantees n_cells * C < 2^31).
template <typename TI, typename TO, int VEC>
__global__ void __launch_bounds__(256, 4) k_upsample_renoise(
    const TI* __restrict__ x, const float* __restrict__ vel, const int32_t* __restrict__ inv,
    const float* __restrict__ eps, TO* __restrict__ out, int st, int sh, int sw, int dt, int dh,
    int dw, int C, float sigma_f, int mode, uint64_t seed, uint64_t offset) {
  // grid (x: (ow, channel group) of one output row, y: oh, z: ot) -- no per-element index
  // division beyond the group split, and the t / h taps are uniform across the CTA
  const int groups = C / VEC;
  const int x_ = blockIdx.x * blockDim.x + threadIdx.x;
  const int oh = blockIdx.y, ot = blockIdx.z;
  // the float64 tap weights (divisions, floor / ceil) are computed once per CTA: t / h taps
  // are uniform over the CTA's output row, w taps once per distinct output column (the
  // per-thread version spent ~80 % of its instructions here)
  __shared__ Taps s_th[2];
  __shared__ Taps s_tw[256];
  const int ow_lo = (blockIdx.x * blockDim.x) / groups;
  const int ow_hi = min(dw - 1, (int)((blockIdx.x * blockDim.x + blockDim.x - 1) / groups));
  for (int i = threadIdx.x; i <= ow_hi - ow_lo; i += blockDim.x) s_tw[i] = axis_taps(ow_lo + i, sw, dw);
  if (threadIdx.x == 0) s_th[0] = axis_taps(ot, st, dt);
  if (threadIdx.x == min(32, (int)blockDim.x - 1)) s_th[1] = axis_taps(oh, sh, dh);
  __syncthreads();
  if (x_ >= dw * groups) return;
  const int ow = x_ / groups;
  const int c0 = (x_ - ow * groups) * VEC;
  const int cell = (ot * dh + oh) * dw + ow;
  const Taps tt = s_th[0], th = s_th[1], tw = s_tw[ow - ow_lo];
  // Always two taps per axis: a missing second tap repeats the first index with weight 0,
  // and 0 * x adds an exact zero -- as the reference's dense tensordot rows do.
  const int ti[2] = {tt.i0, tt.n > 1 ? tt.i0 + 1 : tt.i0};
  const int hi[2] = {th.i0, th.n > 1 ? th.i0 + 1 : th.i0};
  const int wi[2] = {tw.i0, tw.n > 1 ? tw.i0 + 1 : tw.i0};
  const double tw_[2] = {tt.w0, tt.w1}, hw_[2] = {th.w0, th.w1}, ww_[2] = {tw.w0, tw.w1};
  // same axis order as the reference's separable tensordots: t, then h, then w
  double acc_w[VEC];
#pragma unroll
  for (int u = 0; u < VEC; ++u) acc_w[u] = 0.0;
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    double acc_h[VEC];
#pragma unroll
    for (int u = 0; u < VEC; ++u) acc_h[u] = 0.0;
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      double acc_t[VEC];
#pragma unroll
      for (int u = 0; u < VEC; ++u) acc_t[u] = 0.0;
#pragma unroll
      for (int z = 0; z < 2; ++z) {
        const int scell = (ti[z] * sh + hi[a]) * sw + wi[b];
        double x0[VEC];
        const TI* xp = x + (int64_t)scell * C + c0;
        if constexpr (VEC == 4 && sizeof(TI) == 4) {
          const float4 f = __ldg(reinterpret_cast<const float4*>(xp));
          x0[0] = f.x; x0[1] = f.y; x0[2] = f.z; x0[3] = f.w;
        } else {
#pragma unroll
          for (int u = 0; u < VEC; ++u) x0[u] = (double)__ldg(xp + u);
        }
        if (vel) {  // predict_clean in fp32; a curve-order velocity is read through inv
          const float* vp = vel + (int64_t)(inv ? inv[scell] : scell) * C + c0;
#pragma unroll
          for (int u = 0; u < VEC; ++u)
            x0[u] = (double)__fsub_rn((float)x0[u], __fmul_rn(sigma_f, __ldg(vp + u)));
        }
#pragma unroll
        for (int u = 0; u < VEC; ++u) acc_t[u] = fma(tw_[z], x0[u], acc_t[u]);
      }
#pragma unroll
      for (int u = 0; u < VEC; ++u) acc_h[u] = fma(hw_[a], acc_t[u], acc_h[u]);
    }
#pragma unroll
    for (int u = 0; u < VEC; ++u) acc_w[u] = fma(ww_[b], acc_h[u], acc_w[u]);
  }
  const int64_t o = (int64_t)cell * C + c0;
  TO r[VEC];
  if (mode == 0) {
#pragma unroll
    for (int u = 0; u < VEC; ++u) r[u] = (TO)acc_w[u];
  } else {
    float nz[VEC];
    if (mode == 1) {
#pragma unroll
      for (int u = 0; u < VEC; ++u) nz[u] = __ldcs(eps + o + u);
    } else {
#pragma unroll
      for (int u = 0; u < VEC; ++u) nz[u] = philox_normal(seed, offset + (uint64_t)(o + u));
    }
    // (1 - s) * up + s * noise on the float32-cast upsample, each op rounded like numpy's
    // float32 arrays (pipeline.py:190-192)
#pragma unroll
    for (int u = 0; u < VEC; ++u)
      r[u] = (TO)__fadd_rn(__fmul_rn(__fsub_rn(1.0f, sigma_f), (float)acc_w[u]),
                           __fmul_rn(sigma_f, nz[u]));
  }
  if constexpr (VEC == 4 && sizeof(TO) == 4) {
    __stcs(reinterpret_cast<float4*>(out + o), make_float4(r[0], r[1], r[2], r[3]));
  } else {
#pragma unroll
    for (int u = 0; u < VEC; ++u) out[o + u] = r[u];
  }
}

template <typename T>
__global__ void k_euler(const T* __restrict__ x, const T* __restrict__ v, T* __restrict__ out,
                        int64_t n, T ds) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) {
    if constexpr (sizeof(T) == 4)
      out[e] = __fadd_rn(x[e], __fmul_rn(ds, v[e]));
    else
      out[e] = __dadd_rn(x[e], __dmul_rn(ds, v[e]));
  }
}

template <typename TI, typename TO>
static int launch_switch(const TI* x, const float* vel, const int32_t* inv, const float* eps, TO* out,
                         int st, int sh, int sw, int dt, int dh, int dw, int C, double sigma,
                         int mode, uint64_t seed, uint64_t offset, cudaStream_t stream) {
  TCB_CHECK_ARG((int64_t)dt * dh * dw * C < ((int64_t)1 << 31) &&
                    (int64_t)st * sh * sw * C < ((int64_t)1 << 31),
                TCB_ESIZE, "latent too large");
  const bool vec = (C % 4 == 0) && ((uintptr_t)x % 16 == 0) && ((uintptr_t)out % 16 == 0) &&
                   (!eps || (uintptr_t)eps % 16 == 0) && (!vel || (uintptr_t)vel % 16 == 0);
  TCB_CHECK_ARG(dh <= 65535 && dt <= 65535, TCB_ESIZE, "target t/h above 65535");
  const int64_t row = (int64_t)dw * (vec ? C / 4 : C);
  const int64_t nblk = ceil_div(row, 256);
  const int threads = (int)ceil_div(ceil_div(row, nblk), 32) * 32;  // balanced, warp multiple
  const dim3 grid((unsigned)nblk, (unsigned)dh, (unsigned)dt);
  if (vec)
    k_upsample_renoise<TI, TO, 4><<<grid, threads, 0, stream>>>(x, vel, inv, eps, out, st, sh, sw, dt,
                                                               dh, dw, C, (float)sigma, mode, seed,
                                                               offset);
  else
    k_upsample_renoise<TI, TO, 1><<<grid, threads, 0, stream>>>(x, vel, inv, eps, out, st, sh, sw, dt,
                                                               dh, dw, C, (float)sigma, mode, seed,
                                                               offset);
  return check_launch("k_upsample_renoise");
}

}  // namespace tcb

using namespace tcb;

#define TCB_SWITCH_CHECKS()                                                                 \
  TCB_CHECK_ARG(st >= 1 && sh >= 1 && sw >= 1 && C >= 1, TCB_ESHAPE, "bad source dims");    \
  TCB_CHECK_ARG(dt >= st && dh >= sh && dw >= sw, TCB_EDOMAIN, "target shrinks source");    \
  TCB_CHECK_ARG(mode >= 0 && mode <= 2, TCB_EDOMAIN, "bad mode %d", mode);                  \
  TCB_CHECK_ARG(mode != 1 || eps, TCB_ESHAPE, "mode 1 needs eps");                          \
  TCB_CHECK_ARG(sigma >= 0.0 && sigma <= 1.0, TCB_EDOMAIN, "sigma %g outside [0, 1]", sigma)

extern "C" int tcb_upsample_renoise(const float* x, const float* vel, const float* eps, float* out,
                                    int st, int sh, int sw, int dt, int dh, int dw, int C,
                                    double sigma, int mode, uint64_t seed, uint64_t offset,
                                    void* stream) {
  TCB_CHECK_ARG(x && out, TCB_ESHAPE, "null tensor");
  TCB_SWITCH_CHECKS();
  return launch_switch<float, float>(x, vel, nullptr, eps, out, st, sh, sw, dt, dh, dw, C, sigma,
                                     mode, seed, offset, as_stream(stream));
}

extern "C" int tcb_upsample_renoise_f64(const double* x, const float* eps, void* out, int st,
                                        int sh, int sw, int dt, int dh, int dw, int C,
                                        double sigma, int mode, uint64_t seed, uint64_t offset,
                                        void* stream) {
  TCB_CHECK_ARG(x && out, TCB_ESHAPE, "null tensor");
  TCB_SWITCH_CHECKS();
  cudaStream_t s = as_stream(stream);
  if (mode == 0)  // upsample_area_3d keeps the float64 dtype (pipeline.py:173)
    return launch_switch<double, double>(x, nullptr, nullptr, nullptr, (double*)out, st, sh, sw, dt,
                                         dh, dw, C, 0.0, 0, seed, offset, s);
  // stage_transition casts the float64 upsample to float32 before mixing (pipeline.py:190)
  return launch_switch<double, float>(x, nullptr, nullptr, eps, (float*)out, st, sh, sw, dt, dh, dw,
                                      C, sigma, mode, seed, offset, s);
}

extern "C" int tcb_upsample_renoise_curve(const float* x, const float* vel_curve,
                                          const int32_t* inv, const float* eps, float* out, int st,
                                          int sh, int sw, int dt, int dh, int dw, int C,
                                          double sigma, int mode, uint64_t seed, uint64_t offset,
                                          void* stream) {
  TCB_CHECK_ARG(x && out && vel_curve && inv, TCB_ESHAPE, "null tensor");
  TCB_SWITCH_CHECKS();
  return launch_switch<float, float>(x, vel_curve, inv, eps, out, st, sh, sw, dt, dh, dw, C, sigma,
                                     mode, seed, offset, as_stream(stream));
}

extern "C" int tcb_euler_step(const float* x, const float* v, float* out, int64_t n, float dsigma,
                              void* stream) {
  TCB_CHECK_ARG(x && v && out, TCB_ESHAPE, "null tensor");
  if (n == 0) return TCB_OK;
  k_euler<float><<<(unsigned)ceil_div(n, 256), 256, 0, as_stream(stream)>>>(x, v, out, n, dsigma);
  return check_launch("k_euler");
}

extern "C" int tcb_euler_step_f64(const double* x, const double* v, double* out, int64_t n,
                                  double dsigma, void* stream) {
  TCB_CHECK_ARG(x && v && out, TCB_ESHAPE, "null tensor");
  if (n == 0) return TCB_OK;
  k_euler<double><<<(unsigned)ceil_div(n, 256), 256, 0, as_stream(stream)>>>(x, v, out, n, dsigma);
  return check_launch("k_euler");
}
