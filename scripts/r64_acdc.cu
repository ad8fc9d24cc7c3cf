// Prototype: the ACDC forward (layers.py:141-146) at N = 4096 on a two-pass
// 64 x 64 four-step FFT (64 complex values per thread, 64 threads per row
// pair, ONE shared-memory exchange per transform instead of the engine's two).
// Built by scripts/build_r64.sh into gpurun_variants/r64_acdc.so; timed and
// checked against the library forward by scripts/r64_acdc.py.
//
// Index maps (group-local thread t, warp w = t / 32, lane l):
//   colA(t): FFT1 pass-1 column n1 and FFT2 pass-2 column k2'; partner lane
//            l ^ 31 holds column 63 - col (the spatial pairing m <-> N-1-m).
//   colB(t): FFT1 pass-2 column k2 (= FFT2 pass-1 column); partner lane l ^ 31
//            holds column 64 - col (frequency pairing k <-> N-k), except the
//            self-paired columns 0 and 32 (warp 0, lanes 0 and 31).
//   slot(k) = (k >> 3) + 8 (k & 7): where dft64_t leaves output k.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <vector>

#include "../paper_1511_05946_b200/csrc/dct_pair.cuh"

using namespace acdc;

#ifndef R64_GPC
#define R64_GPC 4
#endif
#ifndef R64_LDCHUNK
#define R64_LDCHUNK 8
#endif
namespace {
constexpr int N = 4096;
constexpr int PADW = 65;
constexpr int GPC = R64_GPC;
constexpr int CTA = 64 * GPC;
// smem layout (float2 units): tw [16][64] | cp [N/2 + 1] (+pad) | pst [32][64] float4 | xbuf [GPC][64*PADW]
constexpr int TW_F2 = 64 * 16;
constexpr int CP_F2 = N / 2 + 2;
constexpr int PST_F2 = 32 * 64 * 2;
constexpr int XB_F2 = 64 * PADW;
constexpr int SMEM = 8 * (TW_F2 + CP_F2 + PST_F2 + GPC * XB_F2);

__device__ __forceinline__ int colA(int w, int l) { return w ? l + 16 : (l < 16 ? l : l + 32); }
__device__ __forceinline__ int colB(int w, int l) {
  return w ? (l < 16 ? 16 + l : 17 + l) : (l == 0 ? 0 : (l < 16 ? l : (l < 31 ? l + 33 : 32)));
}
__host__ __device__ constexpr int slot(int k) { return (k >> 3) + 8 * (k & 7); }

// W64^m = exp(-2 pi i m / 64): compile-time constants (nvcc does not fold device cos/sin)
__device__ constexpr float W64C[64] = {1.000000000e+00f, 9.951847267e-01f, 9.807852804e-01f, 9.569403357e-01f, 9.238795325e-01f, 8.819212643e-01f, 8.314696123e-01f, 7.730104534e-01f, 7.071067812e-01f, 6.343932842e-01f, 5.555702330e-01f, 4.713967368e-01f, 3.826834324e-01f, 2.902846773e-01f, 1.950903220e-01f, 9.801714033e-02f, 6.123233996e-17f, -9.801714033e-02f, -1.950903220e-01f, -2.902846773e-01f, -3.826834324e-01f, -4.713967368e-01f, -5.555702330e-01f, -6.343932842e-01f, -7.071067812e-01f, -7.730104534e-01f, -8.314696123e-01f, -8.819212643e-01f, -9.238795325e-01f, -9.569403357e-01f, -9.807852804e-01f, -9.951847267e-01f, -1.000000000e+00f, -9.951847267e-01f, -9.807852804e-01f, -9.569403357e-01f, -9.238795325e-01f, -8.819212643e-01f, -8.314696123e-01f, -7.730104534e-01f, -7.071067812e-01f, -6.343932842e-01f, -5.555702330e-01f, -4.713967368e-01f, -3.826834324e-01f, -2.902846773e-01f, -1.950903220e-01f, -9.801714033e-02f, -1.836970199e-16f, 9.801714033e-02f, 1.950903220e-01f, 2.902846773e-01f, 3.826834324e-01f, 4.713967368e-01f, 5.555702330e-01f, 6.343932842e-01f, 7.071067812e-01f, 7.730104534e-01f, 8.314696123e-01f, 8.819212643e-01f, 9.238795325e-01f, 9.569403357e-01f, 9.807852804e-01f, 9.951847267e-01f};
__device__ constexpr float W64S[64] = {-0.000000000e+00f, -9.801714033e-02f, -1.950903220e-01f, -2.902846773e-01f, -3.826834324e-01f, -4.713967368e-01f, -5.555702330e-01f, -6.343932842e-01f, -7.071067812e-01f, -7.730104534e-01f, -8.314696123e-01f, -8.819212643e-01f, -9.238795325e-01f, -9.569403357e-01f, -9.807852804e-01f, -9.951847267e-01f, -1.000000000e+00f, -9.951847267e-01f, -9.807852804e-01f, -9.569403357e-01f, -9.238795325e-01f, -8.819212643e-01f, -8.314696123e-01f, -7.730104534e-01f, -7.071067812e-01f, -6.343932842e-01f, -5.555702330e-01f, -4.713967368e-01f, -3.826834324e-01f, -2.902846773e-01f, -1.950903220e-01f, -9.801714033e-02f, -1.224646799e-16f, 9.801714033e-02f, 1.950903220e-01f, 2.902846773e-01f, 3.826834324e-01f, 4.713967368e-01f, 5.555702330e-01f, 6.343932842e-01f, 7.071067812e-01f, 7.730104534e-01f, 8.314696123e-01f, 8.819212643e-01f, 9.238795325e-01f, 9.569403357e-01f, 9.807852804e-01f, 9.951847267e-01f, 1.000000000e+00f, 9.951847267e-01f, 9.807852804e-01f, 9.569403357e-01f, 9.238795325e-01f, 8.819212643e-01f, 8.314696123e-01f, 7.730104534e-01f, 7.071067812e-01f, 6.343932842e-01f, 5.555702330e-01f, 4.713967368e-01f, 3.826834324e-01f, 2.902846773e-01f, 1.950903220e-01f, 9.801714033e-02f};
// In-place DFT64 of v[0..63] (natural-order input); output X[k] at v[slot(k)].
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
        const int q = (m / 16) & 3;
        z = q == 1 ? mul_ni(z) : (q == 2 ? make_float2(-z.x, -z.y) : (q == 3 ? make_float2(-z.y, z.x) : z));
      } else if (m % 8 == 0) {
        const int q = (m / 8) & 7;
        const float2 u = (q == 1 || q == 5) ? mul_w8_1(z) : mul_w8_3(z);
        z = q < 4 ? u : make_float2(-u.x, -u.y);
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

// v[slot(k)] *= W4096^(col * k)  (tw table [16][64]: W^(col m), then W^(8 col m), m < 8; twr = tw + col)
__device__ __forceinline__ void twiddle64(float2 (&v)[64], const float2* twr) {
  float2 lo[8];
#pragma unroll
  for (int m = 0; m < 8; ++m) lo[m] = twr[64 * m];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const float2 hi = twr[64 * (8 + c)];
#pragma unroll
    for (int d = 0; d < 8; ++d) {
      if (c == 0 && d == 0) continue;
      const float2 w = c == 0 ? lo[d] : (d == 0 ? hi : cmul(hi, lo[d]));
      v[c + 8 * d] = cmul(v[c + 8 * d], w);  // k = 8c + d sits at slot(k) = c + 8d
    }
  }
}

// exchange: this thread's outputs v[slot(k2)] of column `cin` -> buf[k2][cin];
// then read column `cout`: v[n] = buf[cout][n] (natural order)
__device__ __forceinline__ void exchange64(float2 (&v)[64], float2* xb, int cin, int cout, int grp) {
  asm volatile("bar.sync %0, 64;" ::"r"(grp + 1));
#pragma unroll
  for (int k = 0; k < 64; ++k) xb[k * PADW + cin] = v[slot(k)];
  asm volatile("bar.sync %0, 64;" ::"r"(grp + 1));
#pragma unroll
  for (int n = 0; n < 64; ++n) v[n] = xb[cout * PADW + n];
}

struct P64 {
  const float* x;
  float* y;
  const float* a;
  const float* d;
  const float* bias;
  const float2* tab;  // tw [64][16] | cp [N/2 + 1]
  int64_t rows, ldx, ldy;
};

__global__ void __launch_bounds__(CTA, 1) acdc_fwd_r64_kernel(P64 p) {
  extern __shared__ __align__(16) float2 sm[];
  float2* tws = sm;
  float2* cps = sm + TW_F2;
  float4* pst = reinterpret_cast<float4*>(sm + TW_F2 + CP_F2);
  float2* xbuf = sm + TW_F2 + CP_F2 + PST_F2;
  const int grp = threadIdx.x >> 6, t = threadIdx.x & 63, w = t >> 5, l = t & 31;
  const int ca = colA(w, l), cb = colB(w, l);
  for (int i = threadIdx.x; i < TW_F2 + N / 2 + 1; i += CTA) sm[i] = p.tab[i];
  if (grp == 0) {  // pst[j][t] = (d[lo], d[hi], b[lo], b[hi]), lo = 64 j + cb, hi = N - lo (special: 0 / N/2)
#pragma unroll 4
    for (int j = 0; j < 32; ++j) {
      const int lo = 64 * j + cb;
      const int hi = (cb == 0 && j == 0) ? N / 2 : N - lo;
      pst[j * 64 + t] = make_float4(p.d[lo], p.d[hi], p.bias[lo], p.bias[hi]);
    }
  }
  __syncthreads();
  float2* xb = xbuf + grp * XB_F2;
  const bool self0 = (w == 0 && l == 0), self32 = (w == 0 && l == 31);
  const int pl = (self0 || self32) ? l : (l ^ 31);
  const float2 chi = cps[N / 2];
  const int64_t npairs = (p.rows + 1) >> 1;
  const int64_t gstride = (int64_t)gridDim.x * GPC;
  for (int64_t rp = (int64_t)blockIdx.x * GPC + grp; rp < npairs; rp += gstride) {
    asm volatile("" ::: "memory");  // keep the per-column tables (smem / L1) from being hoisted out of the loop
    const int64_t ra = 2 * rp;
    const bool hasb = ra + 1 < p.rows;
    const float* xa = p.x + ra * p.ldx;
    const float* xbr = p.x + (hasb ? ra + 1 : ra) * p.ldx;
    float2 v[64];
    // load: pairs (u[2m], u[2m+1]) = (v[m], v[N-1-m]), m = ca + 64 n2, n2 < 32; u = a * x
#pragma unroll
    for (int n2 = 0; n2 < 32; ++n2) {
      if (n2 % R64_LDCHUNK == 0) __syncwarp();  // bound the loads in flight (registers)
      const int m = ca + 64 * n2;
      const float2 av = ldg_f2_volatile(reinterpret_cast<const float2*>(p.a) + m);  // not hoisted out of the row loop
      const float2 ua = vmul(__ldg(reinterpret_cast<const float2*>(xa) + m), av);
      float2 ub = vmul(__ldg(reinterpret_cast<const float2*>(xbr) + m), av);
      if (!hasb) ub = make_float2(0.f, 0.f);
      v[n2] = make_float2(ua.x, ub.x);
      const float2 give = make_float2(ua.y, ub.y);  // v[N-1-m]: the partner column's element 63 - n2
      v[63 - n2] = make_float2(__shfl_xor_sync(0xffffffffu, give.x, 31), __shfl_xor_sync(0xffffffffu, give.y, 31));
    }
    // FFT1 (DCT-II core): pass 1 over n2, twiddle, exchange, pass 2 over n1
    dft64_t(v);
    twiddle64(v, tws + ca);
    exchange64(v, xb, ca, cb, grp);
    dft64_t(v);  // Z[64 k1 + cb] at v[slot(k1)]
    // pair k = 64 j + cb (j < 32) with N - k: the partner's slot 63 - j (self columns: own slots
    // 63 - j for column 32; 64 - j, and 32 for j = 0, for column 0).  G[hi] goes back the same way.
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int sh0 = j == 0 ? 32 : 64 - j;  // column 0's mirror slot
      const float2 s = self0 ? v[slot(sh0)] : v[slot(63 - j)];
      const float2 zq = make_float2(__shfl_sync(0xffffffffu, s.x, pl), __shfl_sync(0xffffffffu, s.y, pl));
      const float2 cs = cps[64 * j + cb];
      const bool spec = self0 && j == 0;
      float2 xl, xh;
      dct2_post(v[slot(j)], zq, cs, spec, chi, xl, xh);
      const float4 pv = pst[j * 64 + t];
      xl = vfma(xl, bc(pv.x), bc(pv.z));
      xh = vfma(xh, bc(pv.y), bc(pv.w));
      float2 gl, gh;
      dct3_pre(xl, xh, cs, spec, chi, gl, gh);
      v[slot(j)] = gl;
      const float2 r = make_float2(__shfl_sync(0xffffffffu, gh.x, pl), __shfl_sync(0xffffffffu, gh.y, pl));
      if (j == 0) {
        v[slot(63)] = self0 ? v[slot(63)] : r;
        v[slot(32)] = self0 ? gh : v[slot(32)];
      } else {
        v[slot(63 - j)] = self0 ? v[slot(63 - j)] : r;
        v[slot(64 - j)] = self0 ? gh : v[slot(64 - j)];
      }
    }
    // FFT2 (DCT-III core): input G[cb + 64 n2] at v[slot(n2)] -> natural order by renaming
    {
      float2 u[64];
#pragma unroll
      for (int n2 = 0; n2 < 64; ++n2) u[n2] = v[slot(n2)];
#pragma unroll
      for (int n2 = 0; n2 < 64; ++n2) v[n2] = u[n2];
    }
    dft64_t(v);
    twiddle64(v, tws + cb);
    exchange64(v, xb, cb, ca, grp);
    dft64_t(v);  // H[64 k1 + ca] at v[slot(k1)]; vA = Re H, vB = -Im H
    // store: y[2j], y[2j+1] = (v[j], v[N-1-j]), j = 64 k1 + ca, k1 < 32; v[N-1-j] is the partner's slot 63 - k1
    float* ya = p.y + ra * p.ldy;
    float* yb = p.y + (hasb ? ra + 1 : ra) * p.ldy;
#pragma unroll
    for (int k1 = 0; k1 < 32; ++k1) {
      const float2 s = v[slot(63 - k1)];
      const float2 r = make_float2(__shfl_xor_sync(0xffffffffu, s.x, 31), __shfl_xor_sync(0xffffffffu, s.y, 31));
      const float2 o = v[slot(k1)];
      const int j = 64 * k1 + ca;
      reinterpret_cast<float2*>(ya)[j] = make_float2(o.x, r.x);
      if (hasb) reinterpret_cast<float2*>(yb)[j] = make_float2(-o.y, -r.y);
    }
  }
}

float2* g_tab = nullptr;
}  // namespace

extern "C" {
int r64_fwd(const float* x, float* y, const float* a, const float* d, const float* bias, int64_t rows, int grid,
            cudaStream_t st) {
  if (!g_tab) {
    std::vector<float2> h;
    const double pi = 3.14159265358979323846264338327950288;
    for (int r = 0; r < 16; ++r)  // [16][64]: W^(c m) for r = m < 8, W^(8 c m) for r = 8 + m
      for (int c = 0; c < 64; ++c) {
        const double th = 2 * pi * (double)(c * (r < 8 ? r : 8 * (r - 8))) / N;
        h.push_back(make_float2((float)cos(th), (float)-sin(th)));
      }
    for (int k = 0; k <= N / 2; ++k) {
      const double s = (k == 0 ? std::sqrt(1.0 / N) : std::sqrt(2.0 / N)) * 0.5;
      const double th = pi * (double)k / (2.0 * N);
      h.push_back(make_float2((float)(s * std::cos(th)), (float)(-s * std::sin(th))));
    }
    cudaMalloc(&g_tab, h.size() * sizeof(float2));
    cudaMemcpy(g_tab, h.data(), h.size() * sizeof(float2), cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(acdc_fwd_r64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  }
  P64 p{x, y, a, d, bias, g_tab, rows, N, N};
  acdc_fwd_r64_kernel<<<grid, CTA, SMEM, st>>>(p);
  return (int)cudaGetLastError();
}
int r64_gpc() { return GPC; }
int r64_smem() { return SMEM; }
}
