// Register/shared-memory FFT engine for the ACDC kernels (sm_100a).
//
// One "row-pair group" of T threads transforms an N-point complex vector whose
// real and imaginary parts are two independent real rows (A and B).  Each
// thread holds E complex values in registers; passes are Stockham radix-R
// (R in {2,4,8,16}) with compile-time internal twiddles, one dynamic twiddle
// multiply per element between passes, and a padded shared-memory exchange
// between passes (1 barrier per exchange when double-buffered).
//
// The Stockham pass (input read at stride N/R, autosorted output) is:
//   j in [0, N/R), k = j mod Ns
//   a[q] = in[j + q*N/R] * W_{Ns*R}^{q*k}
//   a    = DFT_R(a)
//   out[(j-k)*R + k + q'*Ns] = a[q']
// which after the last pass leaves the DFT in natural order.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace acdc {

// ------------------------------------------------------------ complex helpers
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 w) {
  return make_float2(fmaf(a.x, w.x, -a.y * w.y), fmaf(a.x, w.y, a.y * w.x));
}
// -i * z
__device__ __forceinline__ float2 mul_ni(float2 z) { return make_float2(z.y, -z.x); }
// +i * z
__device__ __forceinline__ float2 mul_pi(float2 z) { return make_float2(-z.y, z.x); }

// Forward-DFT constants: W_R^m = exp(-2 pi i m / R)
#define ACDC_C1 0.92387953251128675613f  // cos(pi/8)
#define ACDC_S1 0.38268343236508977173f  // sin(pi/8)
#define ACDC_H 0.70710678118654752440f   // sqrt(2)/2

// ------------------------------------------------------------ DFT butterflies
// All take a[0..R) in natural order and return the forward DFT in natural order.
__device__ __forceinline__ void dft2(float2& a0, float2& a1) {
  float2 t = a0;
  a0 = cadd(t, a1);
  a1 = csub(t, a1);
}

__device__ __forceinline__ void dft4(float2& a0, float2& a1, float2& a2, float2& a3) {
  float2 t0 = cadd(a0, a2), t1 = csub(a0, a2);
  float2 t2 = cadd(a1, a3), t3 = csub(a1, a3);
  a0 = cadd(t0, t2);
  a2 = csub(t0, t2);
  a1 = cadd(t1, mul_ni(t3));
  a3 = csub(t1, mul_ni(t3));
}

// z * W8^1 = z * (h, -h)
__device__ __forceinline__ float2 mul_w8_1(float2 z) { return make_float2(ACDC_H * (z.x + z.y), ACDC_H * (z.y - z.x)); }
// z * W8^3 = z * (-h, -h)
__device__ __forceinline__ float2 mul_w8_3(float2 z) { return make_float2(ACDC_H * (z.y - z.x), -ACDC_H * (z.x + z.y)); }

__device__ __forceinline__ void dft8(float2* a) {
  // decimation in time: E = DFT4(even), O = DFT4(odd)
  dft4(a[0], a[2], a[4], a[6]);
  dft4(a[1], a[3], a[5], a[7]);
  float2 o1 = mul_w8_1(a[3]), o2 = mul_ni(a[5]), o3 = mul_w8_3(a[7]);
  float2 e0 = a[0], e1 = a[2], e2 = a[4], e3 = a[6];
  a[0] = cadd(e0, a[1]);
  a[4] = csub(e0, a[1]);
  a[1] = cadd(e1, o1);
  a[5] = csub(e1, o1);
  a[2] = cadd(e2, o2);
  a[6] = csub(e2, o2);
  a[3] = cadd(e3, o3);
  a[7] = csub(e3, o3);
}

__device__ __forceinline__ float2 cmulc(float2 z, float wr, float wi) {
  return make_float2(fmaf(z.x, wr, -z.y * wi), fmaf(z.x, wi, z.y * wr));
}

__device__ __forceinline__ void dft16(float2* a) {
  // 4 x 4: n = 4 n1 + n2, k = k1 + 4 k2
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) dft4(a[n2], a[n2 + 4], a[n2 + 8], a[n2 + 12]);
  // a[n2 + 4 k1] *= W16^(n2 k1)
  a[5] = cmulc(a[5], ACDC_C1, -ACDC_S1);   // n2=1,k1=1 : W^1
  a[9] = mul_w8_1(a[9]);                   // n2=1,k1=2 : W^2
  a[13] = cmulc(a[13], ACDC_S1, -ACDC_C1); // n2=1,k1=3 : W^3
  a[6] = mul_w8_1(a[6]);                   // n2=2,k1=1 : W^2
  a[10] = mul_ni(a[10]);                   // n2=2,k1=2 : W^4
  a[14] = mul_w8_3(a[14]);                 // n2=2,k1=3 : W^6
  a[7] = cmulc(a[7], ACDC_S1, -ACDC_C1);   // n2=3,k1=1 : W^3
  a[11] = mul_w8_3(a[11]);                 // n2=3,k1=2 : W^6
  a[15] = cmulc(a[15], -ACDC_C1, ACDC_S1); // n2=3,k1=3 : W^9
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) dft4(a[4 * k1], a[4 * k1 + 1], a[4 * k1 + 2], a[4 * k1 + 3]);
  // X[k1 + 4 k2] sits at a[4 k1 + k2]: transpose 4x4
  float2 t[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) t[i] = a[i];
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1)
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) a[k1 + 4 * k2] = t[4 * k1 + k2];
}

template <int R>
__device__ __forceinline__ void dft(float2* a) {
  if constexpr (R == 1) {
  } else if constexpr (R == 2) {
    dft2(a[0], a[1]);
  } else if constexpr (R == 4) {
    dft4(a[0], a[1], a[2], a[3]);
  } else if constexpr (R == 8) {
    dft8(a);
  } else {
    static_assert(R == 16, "radix");
    dft16(a);
  }
}

// ------------------------------------------------------------ geometry
__host__ __device__ constexpr int ilog2c(int n) { return n <= 1 ? 0 : 1 + ilog2c(n >> 1); }

// Per-N compile-time geometry.
template <int LOGN>
struct Geo {
  static constexpr int N = 1 << LOGN;
  static constexpr int E = LOGN >= 15 ? 32 : (N >= 16 ? 16 : N);  // complex values per thread
  static constexpr int T = N / E;                                 // threads per row-pair group
  static constexpr int CTA = T >= 128 ? T : 128;                  // threads per CTA
  static constexpr int GPC = CTA / T;                             // groups per CTA
  static constexpr int PADN = N + N / 16;                         // padded float2 slots per buffer
  static constexpr bool SPLIT = (N >= 32768);                     // exchange re / im separately
  static constexpr int NBUF = (N >= 8192) ? 1 : 2;                // double-buffered exchanges
  static constexpr int BUF_FLOATS = SPLIT ? PADN : 2 * PADN;      // floats per buffer
  static constexpr int SMEM_BYTES = GPC * NBUF * BUF_FLOATS * 4;
  // resident CTAs per SM requested from ptxas (caps registers at 64K / (CTA * MINB))
  static constexpr int MINB = CTA >= 512 ? 1 : 512 / CTA;
  // radix plan: 16 x small x 16 x 16 ...   (LOGN = 4a + r)
  static constexpr int A16 = LOGN / 4;
  static constexpr int REM = LOGN % 4;
  static constexpr int NPASS = LOGN < 4 ? 1 : A16 + (REM ? 1 : 0);
  __host__ __device__ static constexpr int radix(int p) {
    return LOGN < 4 ? N : ((REM && p == 1) ? (1 << REM) : 16);
  }
  __host__ __device__ static constexpr int span(int p) {  // Ns before pass p
    return p == 0 ? 1 : span(p - 1) * radix(p - 1);
  }
};

__device__ __forceinline__ int padi(int i) { return i + (i >> 4); }

// Group-local barrier: warp mask for T <= 32, named barrier otherwise.
template <class G>
struct GroupSync {
  unsigned mask;
  int bar_id;
  __device__ __forceinline__ GroupSync(int grp) {
    if constexpr (G::T < 32) {
      int lane = threadIdx.x & 31;
      mask = ((G::T == 32 ? 0xffffffffu : ((1u << G::T) - 1u)) << (lane & ~(G::T - 1)));
    } else {
      mask = 0xffffffffu;
    }
    bar_id = 1 + grp;
  }
  __device__ __forceinline__ void sync() const {
    if constexpr (G::T <= 32) {
      __syncwarp(mask);
    } else if constexpr (G::GPC == 1) {
      __syncthreads();
    } else {
      asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(G::T) : "memory");
    }
  }
};

// ------------------------------------------------------------ Stockham passes
// Compute pass P in registers (twiddle + DFT_R).  v[b*R + q] holds
// in[j_b + q*N/R] for butterfly j_b = t + b*T.
template <class G, int P>
__device__ __forceinline__ void pass_compute(float2 (&v)[G::E], const float2* __restrict__ tw, int t) {
  constexpr int R = G::radix(P);
  constexpr int NS = G::span(P);
  constexpr int NB = G::E / R;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    if constexpr (NS > 1) {
      const int j = t + b * G::T;
      const int k = j & (NS - 1);
      constexpr int S = G::N / (NS * R);
      const int base = k * S;
#pragma unroll
      for (int q = 1; q < R; ++q) v[b * R + q] = cmul(v[b * R + q], __ldg(&tw[q * base]));
    }
    dft<R>(&v[b * R]);
  }
}

// ------------------------------------------------------------ exchanges
// Element accessors for one exchange: full float2 slots, or one component
// (re or im) at a time when the buffer only holds N floats (SPLIT mode).
struct PutFull {
  float2* b;
  __device__ __forceinline__ void operator()(int i, float2 v) const { b[padi(i)] = v; }
};
struct GetFull {
  const float2* b;
  __device__ __forceinline__ void operator()(int i, float2& d) const { d = b[padi(i)]; }
};
struct PutComp {
  float* b;
  int c;
  __device__ __forceinline__ void operator()(int i, float2 v) const { b[padi(i)] = c ? v.y : v.x; }
};
struct GetComp {
  const float* b;
  int c;
  __device__ __forceinline__ void operator()(int i, float2& d) const {
    float f = b[padi(i)];
    if (c) d.y = f; else d.x = f;
  }
};

// Exchange-buffer state: which buffer the next exchange uses.
template <class G>
struct Xbuf {
  float* base;  // NBUF buffers of BUF_FLOATS floats
  int phase;
  __device__ __forceinline__ float* cur() const { return base + phase * G::BUF_FLOATS; }
  __device__ __forceinline__ void flip() {
    if constexpr (G::NBUF == 2) phase ^= 1;
  }
};

// One exchange through shared memory.  wf(put) writes every value this thread
// owns, rf(get) reads every value it needs.  Double-buffered exchanges need one
// barrier; single-buffered ones also need the write-after-read barrier.
template <class G, class WF, class RF>
__device__ __forceinline__ void xchg(Xbuf<G>& xb, const GroupSync<G>& gs, WF&& wf, RF&& rf) {
  if constexpr (G::SPLIT) {
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      gs.sync();
      wf(PutComp{xb.cur(), c});
      gs.sync();
      rf(GetComp{xb.cur(), c});
    }
  } else {
    if constexpr (G::NBUF == 1) gs.sync();
    float2* b = reinterpret_cast<float2*>(xb.cur());
    wf(PutFull{b});
    gs.sync();
    rf(GetFull{b});
    xb.flip();
  }
}

// Write the outputs of pass P at their autosorted positions.
template <class G, int P, class PUT>
__device__ __forceinline__ void pass_store(const float2 (&v)[G::E], const PUT& put, int t) {
  constexpr int R = G::radix(P);
  constexpr int NS = G::span(P);
  constexpr int NB = G::E / R;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int j = t + b * G::T;
    const int k = j & (NS - 1);
    const int d = (j - k) * R + k;
#pragma unroll
    for (int q = 0; q < R; ++q) put(d + q * NS, v[b * R + q]);
  }
}

// Read the inputs of pass P (stride N/R).
template <class G, int P, class GET>
__device__ __forceinline__ void pass_load(float2 (&v)[G::E], const GET& get, int t) {
  constexpr int R = G::radix(P);
  constexpr int NB = G::E / R;
  constexpr int STRIDE = G::N / R;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int j = t + b * G::T;
#pragma unroll
    for (int q = 0; q < R; ++q) get(j + q * STRIDE, v[b * R + q]);
  }
}

// All passes of the FFT; v holds pass-0 inputs on entry and the natural-order
// outputs of the last pass on exit (v[b*R_L + q] = X[j_b + q*N/R_L]).
template <class G, int P = 0>
__device__ __forceinline__ void fft_passes(float2 (&v)[G::E], Xbuf<G>& xb, const GroupSync<G>& gs,
                                           const float2* __restrict__ tw, int t) {
  pass_compute<G, P>(v, tw, t);
  if constexpr (P + 1 < G::NPASS) {
    xchg(
        xb, gs, [&](const auto& put) { pass_store<G, P>(v, put, t); },
        [&](const auto& get) { pass_load<G, P + 1>(v, get, t); });
    fft_passes<G, P + 1>(v, xb, gs, tw, t);
  }
}

// Position n of the last-pass output slot (b, q).
template <class G>
__device__ __forceinline__ int last_pos(int t, int b, int q) {
  constexpr int R = G::radix(G::NPASS - 1);
  return t + b * G::T + q * (G::N / R);
}
// Position m of the first-pass input slot (b, q).
template <class G>
__device__ __forceinline__ int first_pos(int t, int b, int q) {
  constexpr int R = G::radix(0);
  return t + b * G::T + q * (G::N / R);
}

// Makhoul reorder: packed index m -> signal index (transforms.py:109-113)
template <int N>
__device__ __forceinline__ int reorder_src(int m) {
  return m < N / 2 ? 2 * m : 2 * (N - 1 - m) + 1;
}

}  // namespace acdc
