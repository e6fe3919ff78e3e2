/*
 * tokencarve_b200.h -- C ABI of the B200-native (sm_100a) Jenga attention-carving
 * hot path.  Plain pointers, sizes and a cudaStream_t passed as void*; no torch
 * types.  All device pointers are caller-owned (the library never allocates
 * persistent device memory and never frees caller memory).  Every entry point
 * is stream-ordered and asynchronous (no host synchronisation), returns 0 on
 * success or one of the TCB_E* codes, with a human-readable message from
 * tcb_last_error() (thread-local).
 *
 * The reference (tokencarve 0.1.0, /root/reference/pkg/src/tokencarve) is a
 * pure-numpy package with no FFI; each entry point names the reference
 * function whose semantics it implements (file:line).  The Python host package
 * paper_2505_16864_b200 binds these with ctypes behind the reference's own
 * function signatures.
 *
 * Error codes map 1:1 to the reference exception taxonomy (errors.py:4-29).
 */
#ifndef TOKENCARVE_B200_H
#define TOKENCARVE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TCB_OK 0
#define TCB_ESHAPE 1    /* ShapeError    errors.py:4   */
#define TCB_EDOMAIN 2   /* DomainError   errors.py:8   */
#define TCB_ESIZE 3     /* SizeError     errors.py:12  */
#define TCB_ECONTRACT 4 /* ContractError errors.py:16  */
#define TCB_ECUDA 5     /* CUDA launch / runtime failure (RuntimeError) */

/* element types for tensors whose dtype is not fixed */
#define TCB_F32 0
#define TCB_BF16 1
#define TCB_F16 2
#define TCB_F64 3 /* tcb_block_pool and the stage point ops only (reference float64 callers) */

const char* tcb_last_error(void);
int tcb_abi_version(void); /* 2 since the packed-bit mask ABI (no kv_idx) */

/* K1 -- space-filling-curve index builder.
 * Replaces build_curve (sfc.py:198-210) = _gilbert2d/_gen2d (sfc.py:98-157)
 * + _curve_coords (sfc.py:160-195).  fwd[i] = row-major cell at curve position
 * i; inv[fwd[i]] = i.  int32 (n_cells < 2^31, else TCB_ESIZE). */
int tcb_curve_build(int t, int h, int w, int32_t* fwd, int32_t* inv, void* stream);

/* K2 -- row gather dst[i,:] = src[idx[i],:] for rows of row_bytes bytes.
 * Replaces apply_permutation / invert_permutation -> _permute (sfc.py:213-237).
 * idx must lie in [0, src_rows). */
int tcb_gather_rows(const void* src, void* dst, const int32_t* idx, int64_t rows,
                    int64_t row_bytes, int64_t src_rows, void* stream);

/* K6 -- 26-neighbour block adjacency, packed.  Replaces adjacency_mask
 * (partition.py:107-136).  adja is (M_v, words) uint32, bit j of row i set
 * iff blocks i, j touch; symmetric, diagonal set.  Zeroed by the call. */
int tcb_adjacency_build(const int32_t* inv, int t, int h, int w, int m, int M_v, int words,
                        uint32_t* adja, void* stream);

/* K3 -- block mean-pool of Q and K over valid tokens, float64 accumulation.
 * Replaces block_pool (masks.py:98-116).  x{0,1}: (H, N_pad, d) with strides
 * (stride_h, stride_n, 1) in elements; out{0,1}: (H, M_total, d) float64
 * contiguous.  x1/out1 may be NULL (pool one tensor). */
int tcb_block_pool(const void* x0, const void* x1, int dtype, int64_t stride_h, int64_t stride_n,
                   int H, int d, int m, int M_v, int M_total, int64_t n_valid, int64_t n_cond,
                   double* out0, double* out1, void* stream);

/* K4 -- row-stochastic pooled relevance in float64.  Replaces relevance
 * (masks.py:119-134) on the vision rows (masks.py:194-197):
 * R[h,i,:] = softmax_j(pq[h,i].pk[h,j] / sqrt(d)), i < rows, j < M_total.
 * pq: (H, pq_blocks, d), pk: (H, M_total, d) contiguous float64. */
int tcb_block_relevance(const double* pq, int pq_blocks, const double* pk, int H, int rows,
                        int M_total, int d, double* R, void* stream);

/* Mask representation (every select entry point writes it, every carve entry point reads
 * it): bits (rows, words) uint32 -- column j of a row is bit j % 32 of word j / 32 -- plus
 * the row popcounts kv_cnt (rows) int32.  The carve kernels walk the set bits of a row in
 * ascending order, i.e. the reference's flatnonzero(bits[h, qb]) (attention.py:179); no
 * CSR index array exists.  (H, M_v, words) at C2 is 2.7 MB; at the 8,192-block maximum
 * 24 heads take 201 MB. */

/* K5 + K6 union -- importance selection + union with condition and adjacency.
 * Replaces importance_mask (masks.py:137-159) and union_mask (masks.py:162-175).
 * R: (H, M_v, M_total) float64; adja: (M_v, words) or NULL (no adjacency term);
 * outputs: bits (H, M_v, words), kv_cnt (H, M_v).  n_floor = max(1, ceil(k*M_v)) computed
 * by the host in float64 (masks.py:154).  with_union=0 returns the bare importance mask
 * (no cond / adjacency OR).  Bit-exact given R. */
int tcb_block_select(const double* R, int H, int M_v, int M_total, const uint32_t* adja, int words,
                     int n_floor, double p, int with_union, uint32_t* bits, int32_t* kv_cnt,
                     void* stream);

/* K4a -- scaled pooled scores S[h,i,j] = pq[h,i].pk[h,j] / sqrt(d) (masks.py:130-131),
 * float64, i < rows, j < M_total.  First half of tcb_block_relevance. */
int tcb_block_scores(const double* pq, int pq_blocks, const double* pk, int H, int rows,
                     int M_total, int d, double* S, void* stream);

/* K4b+K5 -- S (from tcb_block_scores) is turned into R in place (row softmax,
 * masks.py:132-134, numpy pairwise row sums) and selected like tcb_block_select:
 * build_block_mask (masks.py:178-199) when the caller wants R back. */
int tcb_block_select_scores(double* S, int H, int M_v, int M_total, const uint32_t* adja,
                            int words, int n_floor, double p, int with_union, uint32_t* bits,
                            int32_t* kv_cnt, void* stream);

/* K4+K5 without R -- the mask of build_block_mask (masks.py:178-199) from the pooled means,
 * for callers that do not read R back (the layer path): the float64 scores of a chunk of
 * heads (all of them at C2) go into the caller's bounded `scratch` (never an (H, M_v,
 * M_total) R tensor beyond 256 MB), then the select kernel works on them; at p == 0 it
 * selects on the scores directly (the row softmax is monotone) and re-runs the rows whose
 * top-k boundary is a near tie through the exact softmax program.  pq: (H, pq_blocks, d),
 * pk: (H, M_total, d) float64; scratch_elems >= tcb_block_mask_scratch(H, M_v, M_total)
 * is best (any value >= M_total works, in more chunks).  Union with the condition columns
 * and adja is always applied.  Bitwise the mask of tcb_block_select_scores. */
int tcb_block_mask(const double* pq, int pq_blocks, const double* pk, int H, int M_v, int M_total,
                   int d, const uint32_t* adja, int words, int n_floor, double p, uint32_t* bits,
                   int32_t* kv_cnt, double* scratch, int64_t scratch_elems, void* stream);

/* Scratch doubles tcb_block_mask uses for a shape (all heads' scores up to 256 MB, else one
 * bounded chunk). */
int64_t tcb_block_mask_scratch(int H, int M_v, int M_total);

/* Mask conversions for user-built BlockMask(bits=bool array) (masks.py:78-95). */
int tcb_mask_pack(const uint8_t* dense, int64_t rows, int M_total, int words, uint32_t* bits,
                  int32_t* kv_cnt, void* stream);
int tcb_mask_unpack(const uint32_t* bits, int64_t rows, int M_total, int words, uint8_t* dense,
                    void* stream);

/* K7/K8 -- block-sparse flash-attention forward.  Replaces carve_attention /
 * _carve_rows (attention.py:162-243).  q,k,v,o: (H, N_pad, d) with element
 * strides (stride_h, stride_n, 1), N_pad = M_total*m.  Vision q-block i of
 * head h streams the kv blocks set in bits[h,i,:] (words per row), ascending, kv_cnt[h,i]
 * of them; condition q-blocks attend all M_total blocks; padding keys get -inf, beta is
 * added on condition keys of vision rows, padding rows of o are zeroed.
 * dtype TCB_BF16 or TCB_F16 with m == 128 and d in {64,128} runs the tcgen05/TMEM/TMA
 * kernel; everything else runs the fp32 SIMT kernel (parity path).
 * work: caller-provided device scratch, 256-byte aligned, work_bytes long: >= 16 bytes
 * (scheduler counter); with tcb_carve_workspace_bytes() bytes the tcgen05 kernel also splits
 * each condition q-block into kv-range chunks that run beside their head's vision rows and
 * merges their partials (less DRAM traffic; results within the same tolerance). */
int64_t tcb_carve_workspace_bytes(int H, int M_v, int M_total, int m, int d);
int tcb_carve_fwd(const void* q, const void* k, const void* v, void* o, int dtype,
                  int64_t stride_h, int64_t stride_n, const uint32_t* bits, int words,
                  const int32_t* kv_cnt, int H, int d, int m, int M_v, int M_total,
                  int64_t n_valid, int64_t n_cond, float beta, int32_t* work, int64_t work_bytes,
                  void* stream);

/* Like tcb_carve_fwd but forces the fp32-math SIMT kernel for any shape. */
int tcb_carve_fwd_simt(const void* q, const void* k, const void* v, void* o, int dtype,
                       int64_t stride_h, int64_t stride_n, const uint32_t* bits, int words,
                       const int32_t* kv_cnt, int H, int d, int m, int M_v, int M_total,
                       int64_t n_valid, int64_t n_cond, float beta, void* stream);

/* K7/K8 for fp32 inputs on the tensor cores (the reference's own dtype, attention.py:184-201).
 * Every fp32 operand is split into fp16 hi + lo (scaled by a power of two per tensor/head or
 * per query row) and each product is taken as hi.hi + hi.lo + lo.hi on tcgen05 kind::f16 with
 * fp32 accumulation: within 1e-5 of the reference.  workspace: device scratch of
 * tcb_carve_f32_workspace_bytes() bytes, 256-byte aligned (split K / V planes).  Shapes the
 * tensor-core kernel does not take (m != 128, d not in {64,128}, no workspace, misaligned)
 * run the fp32 SIMT kernel instead.  work: as tcb_carve_fwd. */
int64_t tcb_carve_f32_workspace_bytes(int H, int M_total, int m, int d);  /* 0: not applicable */
int tcb_carve_fwd_f32(const float* q, const float* k, const float* v, float* o, int64_t stride_h,
                      int64_t stride_n, const uint32_t* bits, int words, const int32_t* kv_cnt,
                      int H, int d, int m, int M_v, int M_total, int64_t n_valid, int64_t n_cond,
                      float beta, void* workspace, int64_t workspace_bytes, int32_t* work,
                      void* stream);

/* K9/K10 -- fused predict_clean -> area upsample -> re-noise.
 * Replaces predict_clean (pipeline.py:124-128), upsample_area_3d
 * (pipeline.py:153-173) and stage_transition (pipeline.py:176-194).
 * x: (st,sh,sw,C) float32; vel: same or NULL (then x is already x0);
 * out = (1-sigma)*U(x - sigma*vel) + sigma*eps at (dt,dh,dw,C).
 * mode 0: out = U(x0) (sigma = 0 path, float64 taps, cast to float32)
 * mode 1: eps read from eps (host-drawn noise, bitwise reference parity)
 * mode 2: eps drawn in-kernel (Philox4x32-10 + Box-Muller, seed/offset). */
int tcb_upsample_renoise(const float* x, const float* vel, const float* eps, float* out, int st,
                         int sh, int sw, int dt, int dh, int dw, int C, double sigma, int mode,
                         uint64_t seed, uint64_t offset, void* stream);

/* float64 source latent (a numpy float64 caller of upsample_area_3d / stage_transition):
 * mode 0 writes float64 U(x) (pipeline.py:173 keeps x.dtype), modes 1/2 write float32
 * (1-sigma)*float32(U(x)) + sigma*eps (pipeline.py:190-192).  No velocity term. */
int tcb_upsample_renoise_f64(const double* x, const float* eps, void* out, int st, int sh, int sw,
                             int dt, int dh, int dw, int C, double sigma, int mode, uint64_t seed,
                             uint64_t offset, void* stream);

/* Euler step x + (sigma_next - sigma) * v (pipeline.py:131-137), float32; predict_clean
 * (pipeline.py:124-128) is the same op with dsigma = -sigma. */
int tcb_euler_step(const float* x, const float* v, float* out, int64_t n, float dsigma,
                   void* stream);
/* The same in float64 (numpy float64 callers). */
int tcb_euler_step_f64(const double* x, const double* v, double* out, int64_t n, double dsigma,
                       void* stream);

/* ---- fused neighbours of the path ---- */

/* K9 variant reading a curve-order velocity through inv: vel(cell) = vel_curve[inv[cell]].
 * Fuses invert_permutation (pipeline.py:363) into the stage switch. */
int tcb_upsample_renoise_curve(const float* x, const float* vel_curve, const int32_t* inv,
                               const float* eps, float* out, int st, int sh, int sw, int dt,
                               int dh, int dw, int C, double sigma, int mode, uint64_t seed,
                               uint64_t offset, void* stream);

/* positions = apply_permutation(unravel_index(arange(n), (t,h,w)), perm)
 * (pipeline.py:334-337) straight from fwd: pos (n, 3) int64. */
int tcb_curve_positions(const int32_t* fwd, int64_t n, int t, int h, int w, int64_t* pos,
                        void* stream);

/* Patchify + permute: latent (t*pt, h*ph, w*pw, C) float32 -> tokens (n, pt*ph*pw*C) in
 * curve order, tokens[i] = patch(fwd[i]).  With pt=ph=pw=1 this is
 * apply_permutation(x.reshape(n, C), perm) (pipeline.py:345). */
int tcb_patchify_permute(const float* x, const int32_t* fwd, int t, int h, int w, int pt, int ph,
                         int pw, int C, float* tokens, void* stream);

/* Unpatchify + invert_permutation + Euler (pipeline.py:363-371) in one pass:
 * out = x + dsigma * unpatchify(vel_curve[inv]). */
int tcb_unpermute_euler(const float* x, const float* vel_curve, const int32_t* inv, int t, int h,
                        int w, int pt, int ph, int pw, int C, float dsigma, float* out,
                        void* stream);

/* Raster-order token-major bf16 (n, H, d) tensors (element strides src_sn, src_sh; d
 * contiguous) -> curve-order head-major (dst_sh, dst_sn): dst[hh, i] = f(src[fwd[i], hh]),
 * f = 3D rotary embedding where rotate[k] != 0 (Q, K), plain copy otherwise (V).
 * cos_sin: float (cos, sin) pairs, [t x d_t/2][h x d_h/2][w x d_w/2]; head-dim sections
 * [0,d_t) t, [d_t,d_t+d_h) h, rest w; pair j rotates elements (2j, 2j+1).  Rows >= n of
 * dst are not touched (padding / condition tokens belong to the caller). */
int tcb_rope_permute(const void* const* src, int64_t src_sn, int64_t src_sh, void* const* dst,
                     int64_t dst_sh, int64_t dst_sn, const int* rotate, int n_tensors,
                     const int32_t* fwd, int t, int h, int w, int H, int d,
                     const float* cos_sin, int d_t, int d_h, int d_w, void* stream);

/* ---- mask file format (§8f-3): tensorio.py write_mask / read_mask (tensorio.py:80-100) ----
 * words (rows, words_per_row) uint32, little-endian bit order -> packed (rows,
 * ceil(M_total/8)) bytes in np.packbits order (column 8b = MSB of byte b). */
int tcb_mask_words_to_packbits(const uint32_t* words, int64_t rows, int M_total,
                               int words_per_row, uint8_t* packed, void* stream);
/* packed bytes (np.packbits order) -> dense (rows, M_total) 0/1 bytes. */
int tcb_packbits_to_dense(const uint8_t* packed, int64_t rows, int M_total, uint8_t* dense,
                          void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TOKENCARVE_B200_H */
