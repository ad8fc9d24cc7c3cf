/*
 * acdc_b200.h — C ABI of the B200-native ACDC structured-linear-layer kernels.
 *
 * Drop-in boundary for the reference package's forward / backward /
 * parameter-gradient hot path (reference: /root/reference/pkg/src/acdc).
 * Every entry point takes plain device pointers, sizes and a CUDA stream
 * handle; no torch or numpy types cross this boundary.  The library never
 * allocates or frees caller memory (the only library-owned device memory is
 * a per-device, per-N cache of fp32 twiddle tables, built from fp64 on first
 * use or by acdc_prepare).
 *
 * Conventions
 *   - fp32 row-major matrices: row r of x starts at x + r*ldx (ldx >= n).
 *   - n is a power of two, 1 <= n <= acdc_max_n() (32768).
 *   - Calls are stream-ordered and asynchronous; the library keeps no mutable
 *     per-call state, so calls on distinct streams from distinct host threads
 *     are safe.  Call acdc_prepare(n) before CUDA-graph capture.
 *   - Return 0 on success or a negative ACDC_E_* code; acdc_strerror(code)
 *     gives the message (for ACDC_E_SIZE it is the reference's ValueError text,
 *     transforms.py:96-97).
 *
 * Reference interface each entry point replaces (file:line under pkg/src/acdc):
 *   acdc_fwd_f32   AcdcLayer.forward                 layers.py:141-146
 *   acdc_bwd_f32   AcdcLayer.backward (accumulates)  layers.py:148-156
 *   acdc_dct2_f32  dct(plan, x)  / kernels.dct2_batch transforms.py:137-145, _kernels.pyx:60-73
 *   acdc_dct3_f32  idct(plan, y) / kernels.dct3_batch transforms.py:148-156, _kernels.pyx:76-91
 *   acdc_prepare   DctPlan(n, mode="fast") table build transforms.py:86-122
 *   afdf_fwd_c64   AfdfLayer.forward                 layers.py:199-204
 *   afdf_bwd_c64   AfdfLayer.backward (accumulates)  layers.py:206-215
 *   acdc_fft_c64   fft(plan, z) / ifft(plan, z) / kernels.fft_inplace
 *                                                    transforms.py:166-179, _kernels.pyx:18-57
 *   acdc_bwd_sgd_f32  AcdcLayer.backward + Sgd.step  layers.py:148-156, training.py:58-98
 */
#ifndef ACDC_B200_H
#define ACDC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ACDC_ABI_VERSION 1

#define ACDC_OK 0
#define ACDC_E_SIZE (-1)  /* n not a power of two, or n > acdc_max_n()  (ValueError) */
#define ACDC_E_SHAPE (-2) /* rows < 0 or ld < n                          (ValueError) */
#define ACDC_E_ALIGN (-3) /* misaligned pointer                          (ValueError) */
#define ACDC_E_WS (-4)    /* workspace missing or too small              (ValueError) */
#define ACDC_E_CUDA (-5)  /* CUDA launch / runtime failure               (RuntimeError) */
#define ACDC_E_NULL (-6)  /* required pointer is NULL                    (ValueError) */

/* cudaStream_t without requiring cuda_runtime.h (0 = legacy default stream). */
typedef struct CUstream_st* acdc_stream_t;

int acdc_abi_version(void);
const char* acdc_strerror(int code);
const char* acdc_last_error(void);
int acdc_max_n(void);

/* Build the twiddle tables and launch configuration for size n on the current
 * device (the DctPlan constructor, transforms.py:86-122).  Synchronous. */
int acdc_prepare(int32_t n);

/* y = C3(d * C2(a * x) + bias) row-wise; C2 = orthonormal DCT-II, C3 its
 * inverse (layers.py:141-146).  x, y: [rows, n]; a, d, bias: [n]. */
int acdc_fwd_f32(const float* x, float* y, const float* a, const float* d, const float* bias, int64_t rows,
                 int32_t n, int64_t ldx, int64_t ldy, acdc_stream_t stream);

/* Bytes of scratch acdc_bwd_f32 needs for (rows, n) on the current device
 * (per-group gradient partials; 0 on error). */
size_t acdc_bwd_workspace_bytes(int64_t rows, int32_t n);
/* Kernels one backward call launches for this shape (the backward plus its one-
 * or two-stage gradient reduction); cached != 0 for the h2-cache backward.
 * -1 on invalid arguments. */
int acdc_bwd_launch_count(int64_t rows, int32_t n, int cached);

/* Backward of acdc_fwd_f32 (layers.py:148-156), h2 recomputed:
 *   g3 = C2(dy); g1 = C3(d * g3); dx = a * g1
 *   grad_bias (+)= sum_rows g3; grad_d (+)= sum_rows C2(a*x) * g3; grad_a (+)= sum_rows x * g1
 * accumulate != 0 adds into the existing grads (the reference's "+="),
 * accumulate == 0 overwrites them.  The batch reduction is deterministic
 * (fixed-order, fp64 second pass): identical inputs give bitwise-identical
 * gradients on the same device. */
int acdc_bwd_f32(const float* x, const float* dy, float* dx, const float* a, const float* d, float* grad_a,
                 float* grad_d, float* grad_bias, int accumulate, void* ws, size_t ws_bytes, int64_t rows,
                 int32_t n, int64_t ldx, int64_t ldy, int64_t lddx, acdc_stream_t stream);

/* h2-cache variant (the reference caches h2 = C2(a*x) in forward, layers.py:145).
 * acdc_fwd_cache_f32 also writes h2 into `h2cache` (acdc_h2cache_bytes(rows, n)
 * bytes, opaque layout); acdc_bwd_cached_f32 reads it instead of recomputing
 * C2(a*x), trading 8n bytes/row of HBM traffic for one of the backward's three
 * transforms.  Same results as the pair above.  256 <= n <= 32768 (bytes() == 0
 * otherwise).  For n >= 1024 the kernels run the half-length plan (one
 * n/2-point complex FFT per row) and need 16-byte aligned rows with ld a
 * multiple of 4 (ACDC_E_ALIGN otherwise); the cache layout follows the plan,
 * so a cache is only valid for the backward of the same size. */
size_t acdc_h2cache_bytes(int64_t rows, int32_t n);
int acdc_fwd_cache_f32(const float* x, float* y, const float* a, const float* d, const float* bias, float* h2cache,
                       int64_t rows, int32_t n, int64_t ldx, int64_t ldy, acdc_stream_t stream);
int acdc_bwd_cached_f32(const float* x, const float* dy, float* dx, const float* a, const float* d,
                        const float* h2cache, float* grad_a, float* grad_d, float* grad_bias, int accumulate, void* ws,
                        size_t ws_bytes, int64_t rows, int32_t n, int64_t ldx, int64_t ldy, int64_t lddx,
                        acdc_stream_t stream);

/* Fused single-layer step for small batches: the forward of acdc_fwd_f32 and
 * the backward of acdc_bwd_f32 for an upstream gradient dy that does not depend
 * on y (AcdcLayer.forward then AcdcLayer.backward, layers.py:141-156), in ONE
 * kernel launch of one CTA, gradients written directly (no reduction launch).
 * For batches whose step is launch-latency bound (BASELINE configs[0]: n = 256,
 * 128 rows).  256 <= n <= 2048 and rows <= acdc_step_max_rows(n) (0 where the
 * size has no fused step; ACDC_E_SIZE otherwise).  Same results as the pair of
 * calls (bitwise while the separate backward runs one CTA); y, dx must not
 * alias x, dy or each other. */
int64_t acdc_step_max_rows(int32_t n);
int acdc_step_f32(const float* x, const float* dy, float* y, float* dx, const float* a, const float* d,
                  const float* bias, float* grad_a, float* grad_d, float* grad_bias, int accumulate, int64_t rows,
                  int32_t n, int64_t ldx, int64_t ldy, int64_t ldo_y, int64_t ldo_dx, acdc_stream_t stream);

/* Row-wise orthonormal DCT-II / DCT-III (the reference dct / idct). */
/* ---- backward fused with the momentum-SGD step of the reference optimizer
 * (Sgd.step, training.py:58-98) applied to the layer's a, d, bias_d ----
 * The backward of acdc_bwd_f32 (h2cache NULL: h2 recomputed) or of
 * acdc_bwd_cached_f32 / cascade_bwd_block_f32 (h2cache set; prev_perm and
 * prev_relu as for the block backward), whose deterministic gradient
 * reduction feeds the update instead of storing the gradient:
 *   g = sum_rows(...) (+ grad_k if accumulate);  v_k <- momentum*v_k - lr_k*(g + weight_decay_k*p_k);
 *   p_k <- p_k + v_k                                  for k = a, d, bias_d
 * lr_k = lr_t * lr_mult_k; weight_decay_k = 0 for parameters whose decay flag is
 * off (the reference's diagonals).  grad_* may be NULL unless accumulate; if
 * given they are zeroed, like the reference's p.grad[...] = 0.  value[0] and
 * value[1] are the a and d the backward reads (before the update: stream
 * order).  The update is computed in fp64 from the fp32 state.
 * prev_relu: bit 0 = the previous block's ReLU epilogue; bit 1 = h2cache was
 * written by cascade_fwd_f32 (the cascade's row-pair layout) rather than by
 * acdc_fwd_cache_f32. */
typedef struct acdc_sgd_step {
  float* value[3];        /* a, d, bias_d: [n] fp32, updated in place */
  float* velocity[3];     /* momentum buffers: [n] fp32 */
  float lr[3];            /* lr_t * lr_mult per parameter */
  float weight_decay[3];  /* weight decay, or 0 where decay is off */
  float momentum;
} acdc_sgd_step_t;
int acdc_bwd_sgd_f32(const float* x, const float* dy, float* dx, const float* h2cache, const int32_t* prev_perm,
                     int prev_relu, float* grad_a, float* grad_d, float* grad_bias, int accumulate,
                     const acdc_sgd_step_t* step, void* ws, size_t ws_bytes, int64_t rows, int32_t n, int64_t ldx,
                     int64_t ldy, int64_t lddx, acdc_stream_t stream);

int acdc_dct2_f32(const float* x, float* y, int64_t rows, int32_t n, int64_t ldx, int64_t ldy, acdc_stream_t stream);
int acdc_dct3_f32(const float* x, float* y, int64_t rows, int32_t n, int64_t ldx, int64_t ldy, acdc_stream_t stream);

/* ---- Fused ACDC cascade (Cascade over AcdcLayer / ReluLayer / PermutationLayer,
 * layers.py:309-357, 218-265); 256 <= n <= 16384 ----
 * Block l (l < depth): u = ACDC_l(x_l) with a/d/bias rows l of [depth][n]
 * arrays; then ReLU if flags[l] & 1; then x_{l+1}[j] = r[perm_l[j]] if
 * flags[l] & 2 (perm: [depth][n] int32).  y = output of the last block.
 * cascade_fwd_f32 runs all blocks in one kernel with activations on chip and
 * writes checkpoints into ckpt (cascade_ckpt_bytes): x_{l+1} ([depth-1][rows][n],
 * natural layout, at ckpt) followed by the h2 caches of every block.
 * The backward is one cascade_bwd_block_f32 per block, last to first: a
 * cached-h2 ACDC backward of block l (x = x_l, h2cache = block l's cache)
 * whose epilogue applies block l-1's ReLU (prev_relu) and permutation
 * (prev_perm, scatter) so dx is already the gradient of block l-1's output. */
size_t cascade_ckpt_bytes(int64_t rows, int32_t n, int32_t depth);
int cascade_fwd_f32(const float* x, float* y, int32_t depth, int32_t n, const float* a, const float* d,
                    const float* bias, const int32_t* perm, const uint8_t* flags, float* ckpt, int64_t rows,
                    int64_t ldx, int64_t ldy, acdc_stream_t stream);
int cascade_bwd_block_f32(const float* x, const float* dy, float* dx, const float* a, const float* d,
                          const float* h2cache, const int32_t* prev_perm, int prev_relu, float* grad_a, float* grad_d,
                          float* grad_bias, int accumulate, void* ws, size_t ws_bytes, int64_t rows, int32_t n,
                          int64_t ldx, int64_t ldy, int64_t lddx, acdc_stream_t stream);

/* ---- AFDF: complex diagonals around the FFT pair (layers.py:159-215) ----
 * Rows are complex64, interleaved (re, im); ld in complex elements; a, d, grads
 * are n complex values.  2 <= n <= 16384, 8-byte aligned pointers.
 *   afdf_fwd_c64:  y = IFFT(d * FFT(a * x))        (FFT unnormalised, IFFT 1/n;
 *                                                    transforms.py:166-179)
 *   afdf_bwd_c64:  g3 = FFT(dy)/n; grad_d (+)= sum g3 * conj(FFT(a*x));
 *                  g1 = n * IFFT(g3 * conj(d)); grad_a (+)= sum g1 * conj(x);
 *                  dx = g1 * conj(a)             (gradient = dL/dRe + i dL/dIm) */
int afdf_fwd_c64(const float* x, float* y, const float* a, const float* d, int64_t rows, int32_t n, int64_t ldx,
                 int64_t ldy, acdc_stream_t stream);
size_t afdf_bwd_workspace_bytes(int64_t rows, int32_t n);
int afdf_bwd_c64(const float* x, const float* dy, float* dx, const float* a, const float* d, float* grad_a,
                 float* grad_d, int accumulate, void* ws, size_t ws_bytes, int64_t rows, int32_t n, int64_t ldx,
                 int64_t ldy, int64_t lddx, acdc_stream_t stream);

/* Row-wise complex DFT of interleaved complex64 rows (transforms.py:166-179,
 * _kernels.pyx:18-57): inverse == 0: out = FFT(z) (unnormalised);
 * inverse != 0: out = IFFT(z) = conj(FFT(conj z)) / n.  z == out (in place)
 * is allowed; ldz, ldo in complex elements.  Non-power-of-two n gives
 * ACDC_E_SIZE with FftPlan's message (transforms.py:77-78). */
int acdc_fft_c64(const float* z, float* out, int64_t rows, int32_t n, int inverse, int64_t ldz, int64_t ldo,
                 acdc_stream_t stream);

/* Fused-cascade block backward with the permutation moved from the next
 * block's epilogue (a scattered store) to this block's dy load (a gather):
 * dy[:, i] = dy_in[:, dy_gather[i]] with dy_gather = argsort(perm) of the
 * permutation that follows this block; prev_relu masks this block's dx by
 * x > 0 (the previous block's ReLU), which is then written unpermuted.  Only
 * where the TMEM backward runs (cascade_gather_supported(n) != 0, 512 <= n <=
 * 8192); ACDC_E_SIZE otherwise (use cascade_bwd_block_f32). */
int cascade_gather_supported(int32_t n);
int cascade_bwd_block_gather_f32(const float* x, const float* dy, float* dx, const float* a, const float* d,
                                 const float* h2cache, const int32_t* dy_gather, int prev_relu, float* grad_a,
                                 float* grad_d, float* grad_bias, int accumulate, void* ws, size_t ws_bytes,
                                 int64_t rows, int32_t n, int64_t ldx, int64_t ldy, int64_t lddx,
                                 acdc_stream_t stream);

/* Fused-cascade block backward with the gradient reduction deferred: writes
 * only the per-CTA gradient partials of block l into ws (a block-private
 * region of cascade_defer_ws_bytes(rows, n) bytes), so the block-to-block
 * backward chain does not wait for each block's reduction.  prev_perm
 * (scatter, as cascade_bwd_block_f32) and dy_gather (gather, as
 * cascade_bwd_block_gather_f32) are exclusive; prev_relu as for both.
 * cascade_grad_reduce_f32 then reduces `blocks` such regions (region l at
 * ws + l * ws_stride_bytes) in one launch, in the same fixed fp64 order as
 * the per-block reduction: grads is a DEVICE array of 3*blocks float*
 * ((grad_a, grad_d, grad_bias) of region 0, then region 1, ...), each
 * stored (=) or accumulated (+=, accumulate != 0).  cascade_defer_ws_bytes
 * returns 0 where the deferred form does not apply (n outside the fused
 * cascade's sizes, or more row groups than one reduction pass takes); use the
 * per-block entry points there. */
size_t cascade_defer_ws_bytes(int64_t rows, int32_t n);
int cascade_bwd_block_defer_f32(const float* x, const float* dy, float* dx, const float* a, const float* d,
                                const float* h2cache, const int32_t* prev_perm, const int32_t* dy_gather,
                                int prev_relu, void* ws, size_t ws_bytes, int64_t rows, int32_t n, int64_t ldx,
                                int64_t ldy, int64_t lddx, acdc_stream_t stream);
int cascade_grad_reduce_f32(const void* ws, size_t ws_stride_bytes, int32_t blocks, int64_t rows, int32_t n,
                            float* const* grads, int accumulate, acdc_stream_t stream);

/* Two consecutive fused-cascade blocks in one launch, deferred reduction:
 * block hi = l+1 (x_hi = x_{l+1}, h2_hi, a_hi, d_hi; dy gathered through
 * dy_gather_hi as in cascade_bwd_block_gather_f32; dx masked by relu_hi = the
 * ReLU after block l) then block lo = l on the same rows, whose dy is block
 * hi's dx kept on chip (gathered through dy_gather_lo = argsort of the
 * permutation after block l, or NULL) and whose dx is masked by relu_lo and
 * written to dx.  Partials go to ws_hi / ws_lo (block-private regions of
 * cascade_defer_ws_bytes bytes each) for cascade_grad_reduce_f32.  Only where
 * cascade_pair_supported(rows, n) != 0 (the TMEM backward sizes whose two-block
 * form fits on chip with both blocks' parameter stashes, 512 <= n <= 2048). */
int cascade_pair_supported(int64_t rows, int32_t n);
int cascade_bwd_pair_defer_f32(const float* x_hi, const float* x_lo, const float* dy, float* dx, const float* a_hi,
                               const float* d_hi, const float* a_lo, const float* d_lo, const float* h2_hi,
                               const float* h2_lo, const int32_t* dy_gather_hi, const int32_t* dy_gather_lo,
                               int relu_hi, int relu_lo, void* ws_hi, void* ws_lo, size_t ws_bytes, int64_t rows,
                               int32_t n, int64_t ldx_hi, int64_t ldx_lo, int64_t ldy, int64_t lddx,
                               acdc_stream_t stream);

/* Fused cascade of ACDC-only blocks (the reference's acdc_cascade) on the
 * half-length plan, 1024 <= n <= 16384 (cascade_hl_supported(n) != 0):
 * cascade_fwd_hl_f32 runs every block on chip like cascade_fwd_f32 and writes
 * the same checkpoint buffer (cascade_ckpt_bytes), with the h2 caches in this
 * plan's layout; 16-byte aligned rows and parameters.  Block l's backward is
 * the single-layer cached backward (acdc_bwd_cached_f32 with h2cache = block
 * l's cache), or, deferred, cascade_bwd_hl_defer_f32 into a block-private
 * workspace of cascade_hl_defer_ws_bytes bytes and one
 * cascade_grad_reduce_hl_f32 for all blocks (arguments as
 * cascade_grad_reduce_f32). */
int cascade_hl_supported(int32_t n);
int cascade_fwd_hl_f32(const float* x, float* y, int32_t depth, int32_t n, const float* a, const float* d,
                       const float* bias, float* ckpt, int64_t rows, int64_t ldx, int64_t ldy, acdc_stream_t stream);
size_t cascade_hl_defer_ws_bytes(int64_t rows, int32_t n);
int cascade_bwd_hl_defer_f32(const float* x, const float* dy, float* dx, const float* a, const float* d,
                             const float* h2cache, void* ws, size_t ws_bytes, int64_t rows, int32_t n, int64_t ldx,
                             int64_t ldy, int64_t lddx, acdc_stream_t stream);
int cascade_grad_reduce_hl_f32(const void* ws, size_t ws_stride_bytes, int32_t blocks, int64_t rows, int32_t n,
                               float* const* grads, int accumulate, acdc_stream_t stream);

/* ---- ReLU and Permutation layers outside the fused cascade (layers.py:218-265) ----
 * acdc_relu_fwd_f32: y = x > 0 ? x : 0 (strict mask, layers.py:227).
 * acdc_relu_bwd_f32: dx = y > 0 ? dy : 0, with y the forward's OUTPUT
 *   (y > 0 exactly where x > 0, layers.py:231-233).
 * acdc_gather_cols: y[r, j] = x[r, idx[j]] for elem_bytes 4 (fp32) or 8
 *   (complex64): the permutation forward with idx = perm and its backward
 *   with idx = argsort(perm) (layers.py:254-265).  Not in place. */
int acdc_relu_fwd_f32(const float* x, float* y, int64_t rows, int32_t n, int64_t ldx, int64_t ldy,
                      acdc_stream_t stream);
int acdc_relu_bwd_f32(const float* y, const float* dy, float* dx, int64_t rows, int32_t n, int64_t ldy, int64_t lddy,
                      int64_t lddx, acdc_stream_t stream);
int acdc_gather_cols(const void* x, void* y, const int32_t* idx, int64_t rows, int32_t n, int32_t elem_bytes,
                     int64_t ldx, int64_t ldy, acdc_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* ACDC_B200_H */
