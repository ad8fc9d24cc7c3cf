// Probe: a two-pass 64 x 64 four-step complex FFT for N = 4096 (64 values per
// thread, 64 threads per transform, ONE shared-memory exchange), against the
// engine's three-pass radix-16 plan (two exchanges).  Experimental, not part
// of the product library: scripts/r64_probe.py builds it into
// gpurun_variants/r64_probe.so and times it on batched complex64 rows.
//
//   n = n1 + 64 n2, k = 64 k1 + k2:
//   X[64 k1 + k2] = sum_n1 W64^(n1 k1) W4096^(n1 k2) [sum_n2 x[n1 + 64 n2] W64^(n2 k2)]
// pass 1: thread n1 runs DFT64 over n2, twiddles by W4096^(n1 k2);
// exchange [k2][n1]; pass 2: thread k2 runs DFT64 over n1 -> X[64 k1 + k2].
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "../paper_1511_05946_b200/csrc/fft_engine.cuh"

using namespace acdc;

#ifndef R64_GPC
#define R64_GPC 4  // transforms (64-thread groups) per CTA
#endif
#ifndef R64_K  // transforms per row (> 1: compute-throughput probe; output = FFT^K / 4096^(K-1))
#define R64_K 1
#endif
#ifndef R64_MINB
#define R64_MINB 1
#endif
constexpr int PADW = 65;  // float2 slots per exchange row

// W64^m, m = 0..63 (forward)
__device__ __forceinline__ float2 w64(int m) {
  const double a = -2.0 * 3.14159265358979323846 * (m & 63) / 64.0;
  return make_float2((float)cos(a), (float)sin(a));
}

// W64^m = exp(-2 pi i m / 64): compile-time constants (nvcc does not fold device cos/sin)
__device__ constexpr float W64C[64] = {1.000000000e+00f, 9.951847267e-01f, 9.807852804e-01f, 9.569403357e-01f, 9.238795325e-01f, 8.819212643e-01f, 8.314696123e-01f, 7.730104534e-01f, 7.071067812e-01f, 6.343932842e-01f, 5.555702330e-01f, 4.713967368e-01f, 3.826834324e-01f, 2.902846773e-01f, 1.950903220e-01f, 9.801714033e-02f, 6.123233996e-17f, -9.801714033e-02f, -1.950903220e-01f, -2.902846773e-01f, -3.826834324e-01f, -4.713967368e-01f, -5.555702330e-01f, -6.343932842e-01f, -7.071067812e-01f, -7.730104534e-01f, -8.314696123e-01f, -8.819212643e-01f, -9.238795325e-01f, -9.569403357e-01f, -9.807852804e-01f, -9.951847267e-01f, -1.000000000e+00f, -9.951847267e-01f, -9.807852804e-01f, -9.569403357e-01f, -9.238795325e-01f, -8.819212643e-01f, -8.314696123e-01f, -7.730104534e-01f, -7.071067812e-01f, -6.343932842e-01f, -5.555702330e-01f, -4.713967368e-01f, -3.826834324e-01f, -2.902846773e-01f, -1.950903220e-01f, -9.801714033e-02f, -1.836970199e-16f, 9.801714033e-02f, 1.950903220e-01f, 2.902846773e-01f, 3.826834324e-01f, 4.713967368e-01f, 5.555702330e-01f, 6.343932842e-01f, 7.071067812e-01f, 7.730104534e-01f, 8.314696123e-01f, 8.819212643e-01f, 9.238795325e-01f, 9.569403357e-01f, 9.807852804e-01f, 9.951847267e-01f};
__device__ constexpr float W64S[64] = {-0.000000000e+00f, -9.801714033e-02f, -1.950903220e-01f, -2.902846773e-01f, -3.826834324e-01f, -4.713967368e-01f, -5.555702330e-01f, -6.343932842e-01f, -7.071067812e-01f, -7.730104534e-01f, -8.314696123e-01f, -8.819212643e-01f, -9.238795325e-01f, -9.569403357e-01f, -9.807852804e-01f, -9.951847267e-01f, -1.000000000e+00f, -9.951847267e-01f, -9.807852804e-01f, -9.569403357e-01f, -9.238795325e-01f, -8.819212643e-01f, -8.314696123e-01f, -7.730104534e-01f, -7.071067812e-01f, -6.343932842e-01f, -5.555702330e-01f, -4.713967368e-01f, -3.826834324e-01f, -2.902846773e-01f, -1.950903220e-01f, -9.801714033e-02f, -1.224646799e-16f, 9.801714033e-02f, 1.950903220e-01f, 2.902846773e-01f, 3.826834324e-01f, 4.713967368e-01f, 5.555702330e-01f, 6.343932842e-01f, 7.071067812e-01f, 7.730104534e-01f, 8.314696123e-01f, 8.819212643e-01f, 9.238795325e-01f, 9.569403357e-01f, 9.807852804e-01f, 9.951847267e-01f, 1.000000000e+00f, 9.951847267e-01f, 9.807852804e-01f, 9.569403357e-01f, 9.238795325e-01f, 8.819212643e-01f, 8.314696123e-01f, 7.730104534e-01f, 7.071067812e-01f, 6.343932842e-01f, 5.555702330e-01f, 4.713967368e-01f, 3.826834324e-01f, 2.902846773e-01f, 1.950903220e-01f, 9.801714033e-02f};
// In-place DFT64 of v[0..63] (natural-order input); output X[8c + d] at v[c + 8d].
__device__ __forceinline__ void dft64_t(float2 (&v)[64]) {
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    float2 t[8];
#pragma unroll
    for (int b = 0; b < 8; ++b) t[b] = v[a + 8 * b];
    dft8(t);
#pragma unroll
    for (int d = 0; d < 8; ++d) v[a + 8 * d] = t[d];
  }
#pragma unroll
  for (int a = 1; a < 8; ++a)
#pragma unroll
    for (int d = 1; d < 8; ++d) {
      const int m = a * d;
      float2& z = v[a + 8 * d];
      if (m % 16 == 0) {
        // W64^16 = -i, W64^32 = -1, W64^48 = i
        const int q = (m / 16) & 3;
        z = q == 1 ? mul_ni(z) : (q == 2 ? make_float2(-z.x, -z.y) : (q == 3 ? make_float2(-z.y, z.x) : z));
      } else if (m % 8 == 0) {
        const int q = (m / 8) & 7;  // W8^q
        z = q == 1 ? mul_w8_1(z) : (q == 3 ? mul_w8_3(z) : (q == 5 ? make_float2(-mul_w8_1(z).x, -mul_w8_1(z).y)
                                                                       : make_float2(-mul_w8_3(z).x, -mul_w8_3(z).y)));
      } else {
        z = cmulc(z, W64C[m], W64S[m]);
      }
    }
#pragma unroll
  for (int d = 0; d < 8; ++d) {
    float2 t[8];
#pragma unroll
    for (int a = 0; a < 8; ++a) t[a] = v[a + 8 * d];
    dft8(t);
#pragma unroll
    for (int c = 0; c < 8; ++c) v[c + 8 * d] = t[c];
  }
}

struct R64Params {
  const float2* in;
  float2* out;
  const float2* tw;  // [16][64]: W4096^(n1 m), m = 0..7, then W4096^(8 n1 m), m = 0..7
  int64_t rows;
};

__global__ void __launch_bounds__(64 * R64_GPC, R64_MINB) r64_fft_kernel(R64Params p) {
  extern __shared__ __align__(16) float2 smem2[];
  float2* tws = smem2;                 // [64][16]
  float2* xbuf = smem2 + 64 * 16;      // [GPC][64 * PADW]
  for (int i = threadIdx.x; i < 64 * 16; i += blockDim.x) tws[i] = p.tw[i];
  __syncthreads();
  const int grp = threadIdx.x >> 6, t = threadIdx.x & 63;
  float2* xb = xbuf + grp * 64 * PADW;
  const int64_t gstride = (int64_t)gridDim.x * R64_GPC;
  for (int64_t r = (int64_t)blockIdx.x * R64_GPC + grp; r < p.rows; r += gstride) {
    float2 v[64];
    const float2* src = p.in + r * 4096 + t;
#pragma unroll
    for (int n2 = 0; n2 < 64; ++n2) v[n2] = __ldg(src + 64 * n2);
#pragma unroll 1
    for (int rep = 0; rep < R64_K; ++rep) {
    if (rep > 0) {  // compute-throughput mode: thread t holds X[t + 64 k1] at v[c + 8d], k1 = 8c + d, which
                    // is the next transform's input layout (n1 = t, n2 = k1): a register renaming, no exchange
      float2 w[64];
#pragma unroll
      for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int d = 0; d < 8; ++d) w[8 * c + d] = vmul(v[c + 8 * d], bc(1.f / 4096.f));
#pragma unroll
      for (int i = 0; i < 64; ++i) v[i] = w[i];
    }
    dft64_t(v);  // X1[8c + d] at v[c + 8d], k2 = 8c + d
    // twiddle W4096^(n1 k2), k2 = 8c + d = 8 m1 + m0
    {
      float2 lo[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) lo[m] = tws[64 * m + t];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float2 hi = tws[64 * (8 + c) + t];
#pragma unroll
        for (int d = 0; d < 8; ++d) {
          if (c == 0 && d == 0) continue;
          const float2 w = c == 0 ? lo[d] : (d == 0 ? hi : cmul(hi, lo[d]));
          v[c + 8 * d] = cmul(v[c + 8 * d], w);
        }
      }
    }
    // exchange: [k2][n1]
    asm volatile("bar.sync %0, 64;" ::"r"(grp + 1));
#pragma unroll
    for (int c = 0; c < 8; ++c)
#pragma unroll
      for (int d = 0; d < 8; ++d) xb[(8 * c + d) * PADW + t] = v[c + 8 * d];
    asm volatile("bar.sync %0, 64;" ::"r"(grp + 1));
#pragma unroll
    for (int n1 = 0; n1 < 64; ++n1) v[n1] = xb[t * PADW + n1];
    dft64_t(v);  // X[64 k1 + k2], k1 = 8c + d at v[c + 8d]
    }
    float2* dst = p.out + r * 4096 + t;
#pragma unroll
    for (int c = 0; c < 8; ++c)
#pragma unroll
      for (int d = 0; d < 8; ++d) dst[64 * (8 * c + d)] = v[c + 8 * d];
  }
}

extern "C" {
int r64_fft(const float2* in, float2* out, const float2* tw, int64_t rows, int grid, cudaStream_t st) {
  R64Params p{in, out, tw, rows};
  const int smem = (64 * 16 + R64_GPC * 64 * PADW) * 8;
  cudaFuncSetAttribute(r64_fft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  r64_fft_kernel<<<grid, 64 * R64_GPC, smem, st>>>(p);
  return (int)cudaGetLastError();
}
int r64_gpc() { return R64_GPC; }
int r64_k() { return R64_K; }
}
