// Launch parameters of the single-layer ACDC kernels (acdc_kernels.cu, and
// the half-length large-N kernels in hl_kernels.cu).
#pragma once
#include <cstdint>

#include <cuda_runtime.h>

namespace acdc {

struct KParams {
  const float* x;
  const float* dy;
  float* y;  // y (fwd) or dx (bwd)
  const float* a;
  const float* d;
  const float* bias;
  float* ws;          // bwd partials [groups][3][N]
  float* scratch;     // bwd stash when it does not fit in smem [groups][STASH*T]
  float* h2c;         // h2 cache [row pairs][2N] in thread-native layout (H2C kernels)
  const int* epi_perm;  // bwd epilogue (fused cascade): scatter dx through this permutation
  int epi_relu;         // bwd epilogue: zero dx where x <= 0 (the previous block's ReLU)
  int stage;            // bwd (TMEM kernel): dy rows are 16-byte aligned -> bulk-copy them into smem ahead
  const int* dy_gather;  // bwd (TMEM kernel, fused cascade): dy[:, i] = dy_in[:, dy_gather[i]] (inverse perm)
  const float2* tab;  // [pass twiddles | c'_k]
  // two-block cascade backward (acdc_bwd_tm2_kernel): the second (lower) block's operands
  const float* x2;
  const float* a2;
  const float* d2;
  const float* h2c2;
  const int* dy_gather2;
  float* ws2;
  int epi_relu2;
  int64_t ldx2;
  // fused single-layer step (acdc_step_kernel): the forward's y and the final gradients (written directly)
  float* yf;
  float* gout_a;
  float* gout_d;
  float* gout_b;
  int accumulate;
  int64_t ldyf;
  int64_t rows;
  int64_t ldx, ldy, ldo;
};

}  // namespace acdc
