// Fused kernels on either side of the carved-attention path:
//
//  * k_curve_positions  -- positions = apply_permutation(unravel(arange(n)), perm)
//                          (pipeline.py:334-337) computed straight from fwd, one pass;
//  * k_patchify_permute -- patchify (pt, ph, pw) of a (T, Hl, Wl, C) latent gathered
//                          directly in curve order (pipeline.py:345 with patch 1x1x1 is
//                          apply_permutation(x.reshape(n, C), perm)); and its inverse
//                          fused with the Euler update (pipeline.py:363-371):
//                          x + dsigma * unpatchify(unpermute(vel_curve));
//  * k_rope_permute     -- raster-order token-major Q/K/V (n, H, d) -> curve-order
//                          head-major (H, N_pad, d) with 3D rotary embedding on Q and K,
//                          one read and one write per element instead of permute +
//                          rotate + transpose passes.
// All are HBM-bound index/byte kernels: 16-byte vector accesses, grid-stride over SMs.
#include "common.cuh"

#include <cuda_bf16.h>

namespace tcb {

__global__ void __launch_bounds__(256) k_curve_positions(const int32_t* __restrict__ fwd, int64_t n,
                                                         int h, int w, int64_t* __restrict__ pos) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t f = fwd[i];
  const int64_t hw = (int64_t)h * w;
  pos[3 * i] = f / hw;
  pos[3 * i + 1] = (f / w) % h;
  pos[3 * i + 2] = f % w;
}

// Patch geometry: the latent is (T, Hl, Wl, C) float32 row-major; the token grid is
// (t, h, w) = (T/pt, Hl/ph, Wl/pw); token features are ordered (pt, ph, pw, C).
struct PatchGeom {
  int t, h, w, pt, ph, pw, C;
};

__device__ __forceinline__ int64_t patch_src(const PatchGeom& g, int64_t cell, int f) {
  const int c = f % g.C;
  int r = f / g.C;
  const int dw = r % g.pw;
  r /= g.pw;
  const int dh = r % g.ph;
  const int dt = r / g.ph;
  const int64_t cw = cell % g.w;
  const int64_t ch = (cell / g.w) % g.h;
  const int64_t ct = cell / ((int64_t)g.w * g.h);
  const int64_t T = ct * g.pt + dt, Hh = ch * g.ph + dh, Ww = cw * g.pw + dw;
  return ((T * ((int64_t)g.h * g.ph) + Hh) * ((int64_t)g.w * g.pw) + Ww) * g.C + c;
}

// tokens[i, f] = latent[patch(fwd[i]), f]
__global__ void __launch_bounds__(256) k_patchify_permute(const float* __restrict__ x,
                                                          const int32_t* __restrict__ fwd,
                                                          PatchGeom g, int64_t n,
                                                          float* __restrict__ tok) {
  const int F = g.pt * g.ph * g.pw * g.C;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * F) return;
  const int64_t i = e / F;
  const int f = (int)(e - i * F);
  tok[e] = x[patch_src(g, fwd[i], f)];
}

// out[latent elem] = x[elem] + ds * vel_curve[inv[cell], f]   (unpatchify + unpermute +
// Euler, each op rounded like numpy's float32 arrays: pipeline.py:137)
__global__ void __launch_bounds__(256) k_unpermute_euler(const float* __restrict__ x,
                                                         const float* __restrict__ vel,
                                                         const int32_t* __restrict__ inv,
                                                         PatchGeom g, float ds,
                                                         float* __restrict__ out) {
  const int64_t Wl = (int64_t)g.w * g.pw, Hl = (int64_t)g.h * g.ph;
  const int64_t total = (int64_t)g.t * g.pt * Hl * Wl * g.C;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= total) return;
  const int c = (int)(e % g.C);
  int64_t r = e / g.C;
  const int64_t Ww = r % Wl;
  r /= Wl;
  const int64_t Hh = r % Hl;
  const int64_t T = r / Hl;
  const int64_t cell = ((T / g.pt) * g.h + Hh / g.ph) * g.w + Ww / g.pw;
  const int f = (((int)(T % g.pt) * g.ph + (int)(Hh % g.ph)) * g.pw + (int)(Ww % g.pw)) * g.C + c;
  const int F = g.pt * g.ph * g.pw * g.C;
  const float v = vel[(int64_t)inv[cell] * F + f];
  out[e] = __fadd_rn(x[e], __fmul_rn(ds, v));
}

// ---- 3D RoPE permute.  Table: float2 (cos, sin) rows, [t positions x d_t/2 pairs] then
// [h x d_h/2] then [w x d_w/2]; head-dim sections [0, d_t) t, [d_t, d_t+d_h) h, rest w;
// pair j of a section rotates elements (2j, 2j+1):
//   out0 = x0*cos - x1*sin, out1 = x0*sin + x1*cos  (fp32, each product and sum rounded)
struct RopeGeom {
  int t, h, w, d_t, d_h, d_w;
};

__device__ __forceinline__ float2 bf2_unpack(uint32_t u) {  // (lo, hi) bf16 -> fp32
  return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xffff0000u));
}
__device__ __forceinline__ uint32_t bf2_pack(float lo, float hi) {  // RNE, like __floats2bfloat162_rn
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

struct RopeIO {
  const __nv_bfloat16* src[3];
  __nv_bfloat16* dst[3];
  int rotate[3];
};

// A CTA walks groups of TOK tokens (grid-stride); its threads cover a token's H x d/8
// 16-byte chunks, so each token's source row block (H*d contiguous elements of a (n, H, d)
// tensor) is read coalesced, and every thread keeps TOK independent 16-byte loads in
// flight (latency hiding: one token per thread left the kernel at ~45 % of HBM).
// dst[hh, i, :] = rope(src[fwd[i], hh, :]); blockIdx.y selects Q / K / V.
constexpr int ROPE_TOK = 4;

__global__ void __launch_bounds__(1024) k_rope_permute(RopeIO io, int64_t src_sn, int64_t src_sh,
                                                       int64_t dst_sh, int64_t dst_sn,
                                                       const int32_t* __restrict__ fwd, int n,
                                                       int H, int d, const float2* __restrict__ tab,
                                                       RopeGeom r) {
  const int which = blockIdx.y;
  const int chunks = d >> 3;
  const int per_tok = H * chunks;
  const __nv_bfloat16* src = io.src[which];
  __nv_bfloat16* dst = io.dst[which];
  const bool rot = io.rotate[which] != 0;
  const int hw = r.h * r.w;
  // The launch gives every thread exactly one (head, chunk) slot of a token (blockDim ==
  // H * d/8 <= 1024), so the chunk's 4 rotation pairs -- their axis, table base and
  // per-position stride -- are resolved once, outside the token loop.
  const int j = threadIdx.x;
  if (j >= per_tok) return;
  const int hh = j / chunks, c = j - hh * chunks;
  const int64_t so = (int64_t)hh * src_sh + c * 8, dof = (int64_t)hh * dst_sh + c * 8;
  int axis[4], tb[4], ts[4];
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    int e = c * 8 + 2 * p;
    if (e < r.d_t) {
      axis[p] = 0; tb[p] = e / 2; ts[p] = r.d_t / 2;
    } else if ((e -= r.d_t) < r.d_h) {
      axis[p] = 1; tb[p] = r.t * (r.d_t / 2) + e / 2; ts[p] = r.d_h / 2;
    } else {
      e -= r.d_h;
      axis[p] = 2; tb[p] = r.t * (r.d_t / 2) + r.h * (r.d_h / 2) + e / 2; ts[p] = r.d_w / 2;
    }
  }
  for (int i0 = blockIdx.x * ROPE_TOK; i0 < n; i0 += gridDim.x * ROPE_TOK) {
    int cell[ROPE_TOK];  // tail tokens re-read the last valid one (store skipped)
#pragma unroll
    for (int u = 0; u < ROPE_TOK; ++u) cell[u] = __ldg(fwd + min(i0 + u, n - 1));
    int4 raw[ROPE_TOK];
#pragma unroll
    for (int u = 0; u < ROPE_TOK; ++u)
      raw[u] = __ldcs(reinterpret_cast<const int4*>(src + (int64_t)cell[u] * src_sn + so));
#pragma unroll
    for (int u = 0; u < ROPE_TOK; ++u) {
      int4 res = raw[u];
      if (rot) {
        const int ct = cell[u] / hw, rem = cell[u] - ct * hw;
        const int ch = rem / r.w, cw = rem - ch * r.w;
        uint32_t w4[4] = {(uint32_t)res.x, (uint32_t)res.y, (uint32_t)res.z, (uint32_t)res.w};
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const int pos = axis[p] == 0 ? ct : (axis[p] == 1 ? ch : cw);
          const float2 cs = __ldg(tab + tb[p] + pos * ts[p]);
          const float2 x = bf2_unpack(w4[p]);
          const float o0 = __fsub_rn(__fmul_rn(x.x, cs.x), __fmul_rn(x.y, cs.y));
          const float o1 = __fadd_rn(__fmul_rn(x.x, cs.y), __fmul_rn(x.y, cs.x));
          w4[p] = bf2_pack(o0, o1);
        }
        res = make_int4((int)w4[0], (int)w4[1], (int)w4[2], (int)w4[3]);
      }
      if (i0 + u < n) __stcs(reinterpret_cast<int4*>(dst + (int64_t)(i0 + u) * dst_sn + dof), res);
    }
  }
}

}  // namespace tcb

using namespace tcb;

extern "C" int tcb_curve_positions(const int32_t* fwd, int64_t n, int t, int h, int w,
                                   int64_t* pos, void* stream) {
  TCB_CHECK_ARG(fwd && pos, TCB_ESHAPE, "null tensor");
  TCB_CHECK_ARG(t >= 1 && h >= 1 && w >= 1 && n == (int64_t)t * h * w, TCB_ESHAPE,
                "n %lld != t*h*w", (long long)n);
  k_curve_positions<<<(unsigned)ceil_div(n, 256), 256, 0, as_stream(stream)>>>(fwd, n, h, w, pos);
  return check_launch("k_curve_positions");
}

static int check_patch(int t, int h, int w, int pt, int ph, int pw, int C) {
  TCB_CHECK_ARG(t >= 1 && h >= 1 && w >= 1 && C >= 1, TCB_ESHAPE, "bad token grid");
  TCB_CHECK_ARG(pt >= 1 && ph >= 1 && pw >= 1, TCB_EDOMAIN, "patch sizes must be >= 1");
  TCB_CHECK_ARG((int64_t)pt * ph * pw * C < (1 << 30), TCB_ESIZE, "patch too large");
  return TCB_OK;
}

extern "C" int tcb_patchify_permute(const float* x, const int32_t* fwd, int t, int h, int w,
                                    int pt, int ph, int pw, int C, float* tokens, void* stream) {
  TCB_CHECK_ARG(x && fwd && tokens, TCB_ESHAPE, "null tensor");
  int rc = check_patch(t, h, w, pt, ph, pw, C);
  if (rc) return rc;
  const PatchGeom g{t, h, w, pt, ph, pw, C};
  const int64_t n = (int64_t)t * h * w;
  const int64_t total = n * pt * ph * pw * C;
  if (total == 0) return TCB_OK;
  k_patchify_permute<<<(unsigned)ceil_div(total, 256), 256, 0, as_stream(stream)>>>(x, fwd, g, n,
                                                                                    tokens);
  return check_launch("k_patchify_permute");
}

extern "C" int tcb_unpermute_euler(const float* x, const float* vel_curve, const int32_t* inv,
                                   int t, int h, int w, int pt, int ph, int pw, int C,
                                   float dsigma, float* out, void* stream) {
  TCB_CHECK_ARG(x && vel_curve && inv && out, TCB_ESHAPE, "null tensor");
  int rc = check_patch(t, h, w, pt, ph, pw, C);
  if (rc) return rc;
  const PatchGeom g{t, h, w, pt, ph, pw, C};
  const int64_t total = (int64_t)t * h * w * pt * ph * pw * C;
  if (total == 0) return TCB_OK;
  k_unpermute_euler<<<(unsigned)ceil_div(total, 256), 256, 0, as_stream(stream)>>>(
      x, vel_curve, inv, g, dsigma, out);
  return check_launch("k_unpermute_euler");
}

extern "C" int tcb_rope_permute(const void* const* src, int64_t src_sn, int64_t src_sh,
                                void* const* dst, int64_t dst_sh, int64_t dst_sn,
                                const int* rotate, int n_tensors, const int32_t* fwd, int t,
                                int h, int w, int H, int d, const float* cos_sin, int d_t, int d_h,
                                int d_w, void* stream) {
  TCB_CHECK_ARG(src && dst && fwd && rotate, TCB_ESHAPE, "null argument");
  TCB_CHECK_ARG(n_tensors >= 1 && n_tensors <= 3, TCB_ESHAPE, "1..3 tensors");
  TCB_CHECK_ARG(t >= 1 && h >= 1 && w >= 1 && H >= 1, TCB_ESHAPE, "bad grid");
  TCB_CHECK_ARG(d % 8 == 0, TCB_ESHAPE, "d must be a multiple of 8");
  TCB_CHECK_ARG(src_sn % 8 == 0 && src_sh % 8 == 0 && dst_sh % 8 == 0 && dst_sn % 8 == 0,
                TCB_ESHAPE, "strides must be multiples of 8 elements (16 bytes)");
  RopeIO io{};
  bool any_rot = false;
  for (int k = 0; k < n_tensors; ++k) {
    TCB_CHECK_ARG(src[k] && dst[k], TCB_ESHAPE, "null tensor %d", k);
    TCB_CHECK_ARG((uintptr_t)src[k] % 16 == 0 && (uintptr_t)dst[k] % 16 == 0, TCB_ESHAPE,
                  "tensors must be 16-byte aligned");
    io.src[k] = (const __nv_bfloat16*)src[k];
    io.dst[k] = (__nv_bfloat16*)dst[k];
    io.rotate[k] = rotate[k];
    any_rot |= rotate[k] != 0;
  }
  if (any_rot) {
    TCB_CHECK_ARG(cos_sin, TCB_ESHAPE, "rotation needs the cos/sin table");
    TCB_CHECK_ARG(d_t >= 0 && d_h >= 0 && d_w >= 0 && d_t % 2 == 0 && d_h % 2 == 0 &&
                      d_w % 2 == 0 && d_t + d_h + d_w == d,
                  TCB_EDOMAIN, "rope sections (%d, %d, %d) must be even and sum to d=%d", d_t,
                  d_h, d_w, d);
  }
  const int64_t n = (int64_t)t * h * w;
  TCB_CHECK_ARG(n < ((int64_t)1 << 31), TCB_ESIZE, "too many tokens");
  if (n == 0) return TCB_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t groups = ceil_div(n, ROPE_TOK);
  int64_t blocks = groups < (int64_t)sms * 16 ? groups : (int64_t)sms * 16;  // grid-stride
  dim3 grid((unsigned)blocks, (unsigned)n_tensors);
  // one thread per 16-byte chunk of a token's H*d row block (384 at H=24, d=128)
  TCB_CHECK_ARG((int64_t)H * (d / 8) <= 1024, TCB_ESIZE, "H * d / 8 = %d > 1024 chunks per token",
                H * (d / 8));
  const int threads = (int)ceil_div((int64_t)H * (d / 8), 32) * 32;
  k_rope_permute<<<grid, threads, 0, as_stream(stream)>>>(io, src_sn, src_sh, dst_sh, dst_sn, fwd,
                                                      (int)n, H, d, (const float2*)cos_sin,
                                                      RopeGeom{t, h, w, d_t, d_h, d_w});
  return check_launch("k_rope_permute");
}
