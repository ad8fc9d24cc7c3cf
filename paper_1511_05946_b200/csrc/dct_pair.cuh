// Packed two-row orthonormal DCT-II / DCT-III on top of the FFT engine.
//
// Two real rows A, B of length N are transformed by ONE N-point complex FFT of
// z[n] = vA[n] + i vB[n], where v = x[reorder] is Makhoul's even-ascending /
// odd-descending reordering (reference: transforms.py:109-113, the reorder
// used by _kernels.pyx:69-70).
//
// DCT-II (reference _kernels.pyx:60-73: X_k = Re(w4s_k * FFT(v)_k)):
//   with Z = DFT_N(z), P = Z[k], Q = conj Z[N-k], c'_k = s_k e^{-i pi k/2N}/2:
//     WA = c'_k (P + Q)        XA[k] = Re WA,  XA[N-k] = -Im WA
//     WB = c'_k (-i)(P - Q)    XB[k] = Re WB,  XB[N-k] = -Im WB
//   k = 0 and k = N/2 are self-paired and handled by the "special" slot.
//
// DCT-III (reference _kernels.pyx:76-91: V_k = u1_k y_k - i u2_k y_{N-k},
// v = IFFT(V), out[reorder] = Re v), computed through a FORWARD FFT:
//   G[k] = conj(VA[k] + i VB[k]) / N,  H = DFT_N(G),  vA = Re H,  vB = -Im H
//   with u'_k = conj(c'_k) = u1_k / N for k >= 1 (1/N of the IFFT folded in).
//
// Pair slots: thread t of a group owns E/2 slots i, each a bin pair
//   lo = t + i*T,  hi = N - lo      (slot t=0,i=0 holds the special pair 0, N/2)
// so every bin of [0, N) is owned by exactly one thread of the group, and the
// pairing needed by both the DCT-II post-pass and the DCT-III pre-pass is
// thread-local.
#pragma once
#include "fft_engine.cuh"

namespace acdc {

template <class G>
__device__ __forceinline__ void slot_bins(int t, int i, int& lo, int& hi) {
  lo = t + i * G::T;
  hi = (lo == 0) ? (G::N / 2) : (G::N - lo);
}

// Store the last-pass outputs (natural order) through an exchange, read back
// the pair slots: zp[2i] = Z[lo_i], zp[2i+1] = Z[hi_i].
template <class G>
__device__ __forceinline__ void gather_pairs(const float2 (&v)[G::E], float2 (&zp)[G::E], Xbuf<G>& xb,
                                             const GroupSync<G>& gs, int t) {
  constexpr int P = G::NPASS - 1;
  constexpr int R = G::radix(P);
  constexpr int NB = G::E / R;
  constexpr int STRIDE = G::N / R;
  xchg(
      xb, gs,
      [&](const auto& put) {
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
          for (int q = 0; q < R; ++q) put(t + b * G::T + q * STRIDE, v[b * R + q]);
      },
      [&](const auto& get) {
#pragma unroll
        for (int i = 0; i < G::E / 2; ++i) {
          int lo, hi;
          slot_bins<G>(t, i, lo, hi);
          get(lo, zp[2 * i]);
          get(hi & (G::N - 1), zp[2 * i + 1]);
        }
      });
}

// DCT-II post-pass for one slot: (Z[lo], Z[hi]) -> X[lo] = (XA, XB), X[hi].
template <class G>
__device__ __forceinline__ void dct2_post(float2 zlo, float2 zhi, float2 c, bool special, float2 c_hi, float2& xlo,
                                          float2& xhi) {
  if (special) {
    const float f0 = 2.f * c.x, fh = 2.f * c_hi.x;
    xlo = make_float2(f0 * zlo.x, f0 * zlo.y);
    xhi = make_float2(fh * zhi.x, fh * zhi.y);
  } else {
    const float2 q = make_float2(zhi.x, -zhi.y);
    const float2 s = cadd(zlo, q);
    const float2 dn = mul_ni(csub(zlo, q));
    const float2 wa = cmul(s, c);
    const float2 wb = cmul(dn, c);
    xlo = make_float2(wa.x, wb.x);
    xhi = make_float2(-wa.y, -wb.y);
  }
}

// DCT-III pre-pass for one slot: Y[lo] = (YA, YB), Y[hi] -> G[lo], G[hi].
template <class G>
__device__ __forceinline__ void dct3_pre(float2 ylo, float2 yhi, float2 c, bool special, float2 c_hi, float2& glo,
                                         float2& ghi) {
  if (special) {
    const float f0 = 2.f * c.x, fh = 2.f * c_hi.x;
    glo = make_float2(f0 * ylo.x, -f0 * ylo.y);
    ghi = make_float2(fh * yhi.x, -fh * yhi.y);
  } else {
    const float2 u = make_float2(c.x, -c.y);
    const float2 ua = cmul(make_float2(ylo.x, -yhi.x), u);
    const float2 ub = cmul(make_float2(ylo.y, -yhi.y), u);
    glo = make_float2(ua.x - ub.y, -ua.y - ub.x);
    ghi = make_float2(ua.x + ub.y, ua.y - ub.x);
  }
}

// Write G (pair-slot layout) through an exchange and read the pass-0 inputs.
template <class G>
__device__ __forceinline__ void scatter_pairs_to_fft(const float2 (&gp)[G::E], float2 (&v)[G::E], Xbuf<G>& xb,
                                                     const GroupSync<G>& gs, int t) {
  xchg(
      xb, gs,
      [&](const auto& put) {
#pragma unroll
        for (int i = 0; i < G::E / 2; ++i) {
          int lo, hi;
          slot_bins<G>(t, i, lo, hi);
          put(lo, gp[2 * i]);
          if (hi != G::N) put(hi, gp[2 * i + 1]);
        }
      },
      [&](const auto& get) { pass_load<G, 0>(v, get, t); });
}

}  // namespace acdc
