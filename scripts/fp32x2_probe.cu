// Throughput probe: scalar FFMA/FADD vs sm_100 packed FFMA2/FADD2 (fp32x2).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp32x2_probe fp32x2_probe.cu
// Prints fp32 lane-ops per second for each form (an FFMA2 counts as 2 FMAs).
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 8;       // independent chains per thread
constexpr int IT = 4096;    // iterations

__global__ void k_ffma(float* out, const float* p) {
  float b = p[0], c = p[1];
  float acc[2 * CH];
#pragma unroll
  for (int i = 0; i < 2 * CH; ++i) acc[i] = p[2 + i] + threadIdx.x;
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int i = 0; i < 2 * CH; ++i) acc[i] = fmaf(acc[i], b, c);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 2 * CH; ++i) s += acc[i];
  if (s == 12345.f) out[0] = s;
}

__global__ void k_ffma2(float* out, const float* p) {
  float2 b = make_float2(p[0], p[1]), c = make_float2(p[1], p[0]);
  float2 acc[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) acc[i] = make_float2(p[2 + i] + threadIdx.x, p[3 + i]);
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) acc[i] = __ffma2_rn(acc[i], b, c);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i].x + acc[i].y;
  if (s == 12345.f) out[0] = s;
}

__global__ void k_fadd(float* out, const float* p) {
  float b = p[0];
  float acc[2 * CH];
#pragma unroll
  for (int i = 0; i < 2 * CH; ++i) acc[i] = p[2 + i] + threadIdx.x;
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int i = 0; i < 2 * CH; ++i) acc[i] = acc[i] + b;
    b = -b;
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 2 * CH; ++i) s += acc[i];
  if (s == 12345.f) out[0] = s;
}

__global__ void k_fadd2(float* out, const float* p) {
  float2 b = make_float2(p[0], p[1]);
  float2 acc[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) acc[i] = make_float2(p[2 + i] + threadIdx.x, p[3 + i]);
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) acc[i] = __fadd2_rn(acc[i], b);
    b = make_float2(-b.x, -b.y);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i].x + acc[i].y;
  if (s == 12345.f) out[0] = s;
}

// Mixed: one FFMA2 + one scalar ALU-pipe op (to see whether they co-issue).
__global__ void k_ffma2_mix(float* out, const float* p) {
  float2 b = make_float2(p[0], p[1]), c = make_float2(p[1], p[0]);
  float2 acc[CH];
  unsigned u[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) { acc[i] = make_float2(p[2 + i] + threadIdx.x, p[3 + i]); u[i] = threadIdx.x + i; }
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) { acc[i] = __ffma2_rn(acc[i], b, c); u[i] = (u[i] ^ (u[i] >> 3)) + 7u; }
  }
  float s = 0;
  unsigned us = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) { s += acc[i].x + acc[i].y; us += u[i]; }
  if (s == 12345.f || us == 77u) out[0] = s;
}

template <typename K>
float timeit(K k, float* out, const float* p, int blocks, int threads) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  k<<<blocks, threads>>>(out, p);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) k<<<blocks, threads>>>(out, p);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / 5;
}

int main() {
  float *out, *p;
  cudaMalloc(&out, 64); cudaMalloc(&p, 256);
  float h[64]; for (int i = 0; i < 64; ++i) h[i] = 1.0f + 1e-7f * i;
  cudaMemcpy(p, h, sizeof(h), cudaMemcpyHostToDevice);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 512, blocks = sms * 4;
  const double lane_ops = (double)blocks * threads * IT * 2 * CH;   // fp32 ops (FMA=1 op)
  struct { const char* n; float ms; } r[] = {
    {"ffma", timeit(k_ffma, out, p, blocks, threads)},
    {"ffma2", timeit(k_ffma2, out, p, blocks, threads)},
    {"fadd", timeit(k_fadd, out, p, blocks, threads)},
    {"fadd2", timeit(k_fadd2, out, p, blocks, threads)},
    {"ffma2+alu", timeit(k_ffma2_mix, out, p, blocks, threads)},
  };
  for (auto& e : r)
    printf("{\"op\": \"%s\", \"ms\": %.4f, \"Gops\": %.1f, \"ops_per_clk_per_sm_at_1965\": %.1f}\n", e.n, e.ms,
           lane_ops / e.ms * 1e-6, lane_ops / (e.ms * 1e-3) / 1.965e9 / sms);
  return 0;
}
