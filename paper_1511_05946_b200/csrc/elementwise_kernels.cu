// ReLU and column-permutation layers for stacks the fused cascade does not
// cover (reference layers.py:218-265): one HBM pass each, rows of any length.
//
//   acdc_relu_fwd_f32   y = x > 0 ? x : 0                      (layers.py:225-229, strict mask)
//   acdc_relu_bwd_f32   dx = y > 0 ? dy : 0  (y > 0 <=> x > 0)  (layers.py:231-233)
//   acdc_gather_cols    y[:, j] = x[:, idx[j]] for 4- or 8-byte elements
//                       (Permutation forward with perm, backward with argsort(perm),
//                       layers.py:254-265; complex64 rows are 8-byte elements)
//
// A row is staged in shared memory with coalesced 128-bit loads when it fits
// (n * elem <= 96 KB), so the gather's random reads hit shared memory and the
// global traffic is one coalesced read and one coalesced write per element.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/acdc_b200.h"
#include "runtime.h"

namespace acdc {

__global__ void relu_fwd_kernel(const float* __restrict__ x, float* __restrict__ y, int64_t rows, int n, int64_t ldx,
                                int64_t ldy) {
  const int64_t total = rows * (int64_t)n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / n, c = i - r * n;
    const float v = x[r * ldx + c];
    y[r * ldy + c] = v > 0.f ? v : 0.f;
  }
}

__global__ void relu_bwd_kernel(const float* __restrict__ y, const float* __restrict__ dy, float* __restrict__ dx,
                                int64_t rows, int n, int64_t ldy, int64_t ldg, int64_t ldo) {
  const int64_t total = rows * (int64_t)n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / n, c = i - r * n;
    dx[r * ldo + c] = y[r * ldy + c] > 0.f ? dy[r * ldg + c] : 0.f;
  }
}

// One CTA per row (grid-stride over rows): stage the row in smem, gather.
template <class E>
__global__ void gather_cols_smem_kernel(const E* __restrict__ x, E* __restrict__ y, const int32_t* __restrict__ idx,
                                        int64_t rows, int n, int64_t ldx, int64_t ldy) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  E* row = reinterpret_cast<E*>(sm_raw);
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const E* xr = x + r * ldx;
    for (int c = threadIdx.x; c < n; c += blockDim.x) row[c] = xr[c];
    __syncthreads();
    E* yr = y + r * ldy;
    for (int c = threadIdx.x; c < n; c += blockDim.x) yr[c] = row[__ldg(idx + c)];
    __syncthreads();
  }
}

template <class E>
__global__ void gather_cols_kernel(const E* __restrict__ x, E* __restrict__ y, const int32_t* __restrict__ idx,
                                   int64_t rows, int n, int64_t ldx, int64_t ldy) {
  const int64_t total = rows * (int64_t)n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / n, c = i - r * n;
    y[r * ldy + c] = x[r * ldx + __ldg(idx + c)];
  }
}

static int ew_grid(int64_t total) {
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t need = (total + 255) / 256;
  const int64_t cap = (int64_t)sms * 8;
  return (int)(need < cap ? (need > 0 ? need : 1) : cap);
}

static int ew_check(const void* a, const void* b, int64_t rows, int32_t n, int64_t lda, int64_t ldb) {
  if (rows < 0 || n < 1 || lda < n || ldb < n) return ACDC_E_SHAPE;
  if (rows > 0 && (!a || !b)) return ACDC_E_NULL;
  return ACDC_OK;
}

static int ew_done() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ACDC_OK : set_cuda_error(e);
}

}  // namespace acdc

using namespace acdc;

extern "C" {

int acdc_relu_fwd_f32(const float* x, float* y, int64_t rows, int32_t n, int64_t ldx, int64_t ldy,
                      acdc_stream_t stream) {
  int rc = ew_check(x, y, rows, n, ldx, ldy);
  if (rc || rows == 0) return rc;
  relu_fwd_kernel<<<ew_grid(rows * (int64_t)n), 256, 0, (cudaStream_t)stream>>>(x, y, rows, n, ldx, ldy);
  return ew_done();
}

int acdc_relu_bwd_f32(const float* y, const float* dy, float* dx, int64_t rows, int32_t n, int64_t ldy, int64_t lddy,
                      int64_t lddx, acdc_stream_t stream) {
  int rc = ew_check(y, dx, rows, n, ldy, lddx);
  if (rc || rows == 0) return rc;
  if (!dy) return ACDC_E_NULL;
  if (lddy < n) return ACDC_E_SHAPE;
  relu_bwd_kernel<<<ew_grid(rows * (int64_t)n), 256, 0, (cudaStream_t)stream>>>(y, dy, dx, rows, n, ldy, lddy,
                                                                                  lddx);
  return ew_done();
}

int acdc_gather_cols(const void* x, void* y, const int32_t* idx, int64_t rows, int32_t n, int32_t elem_bytes,
                     int64_t ldx, int64_t ldy, acdc_stream_t stream) {
  int rc = ew_check(x, y, rows, n, ldx, ldy);
  if (rc || rows == 0) return rc;
  if (!idx) return ACDC_E_NULL;
  if (elem_bytes != 4 && elem_bytes != 8) return set_error(ACDC_E_SHAPE, "elements must be 4 or 8 bytes");
  if (x == y) return set_error(ACDC_E_SHAPE, "the column gather cannot run in place");
  cudaStream_t st = (cudaStream_t)stream;
  const size_t row_bytes = (size_t)n * elem_bytes;
  if (row_bytes <= 96 * 1024) {
    int sms = 148, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t cap = (int64_t)sms * (row_bytes <= 24 * 1024 ? 8 : 2);
    const int grid = (int)(rows < cap ? rows : cap);
    if (elem_bytes == 4) {
      if (row_bytes > 48 * 1024)
        cudaFuncSetAttribute(gather_cols_smem_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
      gather_cols_smem_kernel<float><<<grid, 256, row_bytes, st>>>((const float*)x, (float*)y, idx, rows, n, ldx,
                                                                   ldy);
    } else {
      if (row_bytes > 48 * 1024)
        cudaFuncSetAttribute(gather_cols_smem_kernel<float2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             96 * 1024);
      gather_cols_smem_kernel<float2><<<grid, 256, row_bytes, st>>>((const float2*)x, (float2*)y, idx, rows, n, ldx,
                                                                    ldy);
    }
  } else if (elem_bytes == 4) {
    gather_cols_kernel<float><<<ew_grid(rows * (int64_t)n), 256, 0, st>>>((const float*)x, (float*)y, idx, rows, n,
                                                                          ldx, ldy);
  } else {
    gather_cols_kernel<float2><<<ew_grid(rows * (int64_t)n), 256, 0, st>>>((const float2*)x, (float2*)y, idx, rows,
                                                                           n, ldx, ldy);
  }
  return ew_done();
}

}  // extern "C"
