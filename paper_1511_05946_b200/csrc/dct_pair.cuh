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

// Pair-slot addressing: bins lo = t + i*T and hi = N - lo.  Element pointers
// for the hi bins are (base + N - t) - i*T; padded exchange indices are
// padi(t) + padoff(iT) and padoff(N - iT) - hb(t) (T a multiple of 16).
template <class G>
struct Slots {
  static constexpr int N = G::N, T = G::T, NS = G::E / 2;
  int t;
  bool t0;
  __device__ __forceinline__ explicit Slots(int t_) : t(t_), t0(t_ == 0) {}
  __device__ __forceinline__ bool special(int i) const { return i == 0 && t0; }
  __device__ __forceinline__ int lo(int i) const { return t + i * T; }
  __device__ __forceinline__ int hi(int i) const { return special(i) ? N / 2 : N - t - i * T; }
  // element of an array indexed by bin: a[lo], a[hi]
  template <class P>
  __device__ __forceinline__ P* plo(P* a, int i) const { return a + t + i * T; }
  template <class P>
  __device__ __forceinline__ P* phi(P* a, int i) const {
    return (i == 0) ? (t0 ? a + N / 2 : a + (N - t)) : (a + (N - t)) - i * T;
  }
  // padded exchange indices
  __device__ __forceinline__ int xlo(int i) const { return padi(t) + padoff(i * T); }
  __device__ __forceinline__ int xhi(int i) const {
    if constexpr (T % 16 == 0) {
      const int hb = t + ACDC_PADS * ((t + 15) >> 4);
      return (i == 0 && t0) ? padoff(N / 2) : padoff(N - i * T) - hb;
    } else {
      return padi(hi(i));
    }
  }
};

// Store the last-pass outputs (natural order) through an exchange, read back
// the pair slots: zp[2i] = Z[lo_i], zp[2i+1] = Z[hi_i].
template <class G>
__device__ __forceinline__ void gather_pairs(const float2 (&v)[G::E], float2 (&zp)[G::E], Xbuf<G>& xb,
                                             const GroupSync<G>& gs, int t) {
  constexpr int P = G::NPASS - 1;
  constexpr int R = G::radix(P);
  constexpr int NB = G::E / R;
  constexpr int S = G::N / R;
  const Slots<G> sl(t);
  xchg(
      xb, gs,
      [&](const auto& put) {
        const int pt = padi(t);
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
          for (int q = 0; q < R; ++q) put(pt + padoff(b * G::T) + padoff(q * S), v[b * R + q]);
      },
      [&](const auto& get) {
#pragma unroll
        for (int i = 0; i < G::E / 2; ++i) {
          get(sl.xlo(i), zp[2 * i]);
          get(sl.xhi(i), zp[2 * i + 1]);
        }
      });
}

// DCT-II post-pass for one slot: (Z[lo], Z[hi]) -> X[lo] = (XA, XB), X[hi].
// With U = Z[lo] + Z[hi] and M = Z[lo] - Z[hi] the four outputs are
//   X[lo] = c.x U + c.y (i M),   X[hi] = c.x (i M) - c.y U
// (expanding XA = Re c(P+Q), XB = Re c(-i)(P-Q) etc.): 6 packed instructions.
__device__ __forceinline__ void dct2_post(float2 zlo, float2 zhi, float2 c, bool special, float2 c_hi, float2& xlo,
                                          float2& xhi) {
  if (special) {
    xlo = vmul(bc(2.f * c.x), zlo);
    xhi = vmul(bc(2.f * c_hi.x), zhi);
  } else {
    const float2 u = cadd(zlo, zhi), m = csub(zlo, zhi);
    const float2 im = make_float2(-m.y, m.x);
    xlo = vfma(bc(c.y), im, vmul(bc(c.x), u));
    xhi = vfma(bc(c.x), im, vmul(bc(-c.y), u));
  }
}

// DCT-III pre-pass for one slot: Y[lo] = (YA, YB), Y[hi] -> G[lo], G[hi].
// With K = Y[lo] - i Y[hi] and L = Y[lo] + i Y[hi] (u = conj c):
//   G[lo] = c.x conj(K) + c.y swap(K),   G[hi] = c.x conj(L) - c.y swap(L).
__device__ __forceinline__ void dct3_pre(float2 ylo, float2 yhi, float2 c, bool special, float2 c_hi, float2& glo,
                                         float2& ghi) {
  if (special) {
    glo = vmul(bc(2.f * c.x), make_float2(ylo.x, -ylo.y));
    ghi = vmul(bc(2.f * c_hi.x), make_float2(yhi.x, -yhi.y));
  } else {
    const float2 k = cadd_ni(ylo, yhi), l = cadd_pi(ylo, yhi);
    glo = vfma(bc(c.y), make_float2(k.y, k.x), vmul(bc(c.x), make_float2(k.x, -k.y)));
    ghi = vfma(bc(-c.y), make_float2(l.y, l.x), vmul(bc(c.x), make_float2(l.x, -l.y)));
  }
}

// Write G (pair-slot layout) through an exchange and read the pass-0 inputs.
template <class G>
__device__ __forceinline__ void scatter_pairs_to_fft(const float2 (&gp)[G::E], float2 (&v)[G::E], Xbuf<G>& xb,
                                                     const GroupSync<G>& gs, int t) {
  const Slots<G> sl(t);
  xchg(
      xb, gs,
      [&](const auto& put) {
#pragma unroll
        for (int i = 0; i < G::E / 2; ++i) {
          put(sl.xlo(i), gp[2 * i]);
          put(sl.xhi(i), gp[2 * i + 1]);
        }
      },
      [&](const auto& get) { pass_load<G, 0>(v, get, t); });
}

// =====================================================================
// Fast-pairing path (N >= 256, E = 16): the first and last pass have one
// radix-16 butterfly per thread (T = S = N/16).  Butterflies are remapped so
// that the two pairings the DCT needs sit in partner lanes (lane ^ H):
//   spatial  j <-> S-1-j : x[2m], x[2m+1] are z[m] and z[N-1-m]  (Makhoul)
//   frequency j <-> S-j  : Z[k] and Z[N-k]                       (real FFT)
// so the pair exchanges are register shuffles, the DCT-II post-pass feeds
// the DCT-III pre-pass without touching shared memory, and global rows are
// moved as 64-bit pairs.  Butterflies 0 and S/2 are self-paired.
#ifndef ACDC_FP_SELFSRC  // 1: frequency pairing shuffles from a per-lane source (no selects for the self-paired slots)
#define ACDC_FP_SELFSRC 0
#endif
template <class G>
struct FastMap {
  static constexpr int N = G::N;
  static constexpr int S = G::N / 16;      // == T
  static constexpr int B = G::T < 32 ? G::T : 32;
  static constexpr int H = B / 2;          // partner = lane ^ H
  int jsp, jfq;                            // spatial / frequency butterfly
  bool isz, ish;                           // jfq == 0 / jfq == S/2
  unsigned mask;
  int fsrc;                                // frequency partner lane (self for the two self-paired slots)
  __device__ __forceinline__ FastMap(int t, unsigned group_mask) {
    const int w = t / B, l = t % B;
    const int lo = H * w + l;
    isz = (w == 0 && l == 0);
    ish = (w == 0 && l == H);
    jsp = l < H ? lo : S - 1 - H * w - (l - H);
    jfq = l < H ? lo : (ish ? S / 2 : S - H * w - (l - H));
    mask = group_mask;
    const int lane = threadIdx.x & 31;
    fsrc = (isz || ish) ? lane : (lane ^ H);
  }
  __device__ __forceinline__ float2 freq_shfl(float2 v) const {
    return make_float2(__shfl_sync(mask, v.x, fsrc), __shfl_sync(mask, v.y, fsrc));
  }
  __device__ __forceinline__ float2 xor_shfl(float2 v) const {
    return make_float2(__shfl_xor_sync(mask, v.x, H), __shfl_xor_sync(mask, v.y, H));
  }
  // bins of frequency slot s: lo = jfq + s*S, hi = N - lo (special slot: 0, N/2)
  __device__ __forceinline__ bool special(int s) const { return s == 0 && isz; }
  template <class P>
  __device__ __forceinline__ P* plo(P* a, int s) const { return a + jfq + s * S; }
  template <class P>
  __device__ __forceinline__ P* phi(P* a, int s) const {
    return (s == 0 && isz) ? a + N / 2 : (a + (N - jfq)) - s * S;
  }
};

// Z[jfq + q*S] (q < 16, last-pass output) -> W[s] = Z[hi_s] for s < 8.
template <class G>
__device__ __forceinline__ void fp_partner(const float2 (&z)[16], float2 (&w)[8], const FastMap<G>& fm) {
#if ACDC_FP_SELFSRC
  // the self-paired slots shuffle from their own lane: slot 0 sends its own
  // mirror values, slot S/2 receives what it sends
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const float2 self0 = s == 0 ? z[8] : z[(16 - s) & 15];
    w[s] = fm.freq_shfl(fm.isz ? self0 : z[15 - s]);
  }
  return;
#endif
  float2 r[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) r[s] = fm.xor_shfl(z[15 - s]);
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const float2 self0 = s == 0 ? z[8] : z[(16 - s) & 15];
    w[s] = fm.isz ? self0 : (fm.ish ? z[15 - s] : r[s]);
  }
}

// G at (lo_s, hi_s) for s < 8 -> v[q] = G[jfq + q*S] (pass-0 inputs).
template <class G>
__device__ __forceinline__ void fp_scatter(const float2 (&gl)[8], const float2 (&gh)[8], float2 (&v)[16],
                                           const FastMap<G>& fm) {
#if ACDC_FP_SELFSRC
  {
    float2 r[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) r[s] = fm.freq_shfl(fm.isz ? gh[s == 7 ? 0 : s + 1] : gh[s]);
#pragma unroll
    for (int s = 0; s < 8; ++s) v[s] = gl[s];
#pragma unroll
    for (int q = 8; q < 16; ++q) v[q] = r[15 - q];
    return;
  }
#endif
  float2 r[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) r[s] = fm.xor_shfl(gh[s]);
#pragma unroll
  for (int s = 0; s < 8; ++s) v[s] = gl[s];
#pragma unroll
  for (int q = 8; q < 16; ++q) {
    const float2 self0 = q == 8 ? gh[0] : gh[16 - q];
    v[q] = fm.isz ? self0 : (fm.ish ? gh[15 - q] : r[15 - q]);
  }
}

__device__ __forceinline__ float2 ld_f2(const float* p) { return __ldg(reinterpret_cast<const float2*>(p)); }
// Activation rows are touched once per launch: optionally streamed (evict-first)
// so they do not push the L2-prefetched rows out.
__device__ __forceinline__ float2 ld_row_f2(const float* p) {
#ifdef ACDC_LD_CS
  return __ldcs(reinterpret_cast<const float2*>(p));
#else
  return __ldg(reinterpret_cast<const float2*>(p));
#endif
}
__device__ __forceinline__ void st_row_f2(float2* p, float2 v) {
#ifdef ACDC_ST_CS
  __stcs(p, v);
#else
  *p = v;
#endif
}

// Pass-0 inputs from two rows (and an optional scale row): the 64-bit pair
// x[2m], x[2m+1] at m = jsp + q*S (q < 8) holds z[m] (kept) and z[N-1-m]
// (the partner's slot 15-q, sent).
template <class G, bool SCALE>
__device__ __forceinline__ void fp_load(float2 (&v)[16], const float* xa, const float* xb, const float* sc,
                                        const FastMap<G>& fm) {
  constexpr int S = FastMap<G>::S;
  const float* pa = xa + 2 * fm.jsp;
  const float* pb = (xb ? xb : xa) + 2 * fm.jsp;
  const float* ps = (SCALE ? sc : xa) + 2 * fm.jsp;
  float2 snd[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    float2 a2 = ld_row_f2(pa + 2 * q * S);
    float2 b2 = xb ? ld_row_f2(pb + 2 * q * S) : make_float2(0.f, 0.f);
    if constexpr (SCALE) {
      const float2 s2 = ld_f2(ps + 2 * q * S);
      a2 = vmul(a2, s2);
      b2 = vmul(b2, s2);
    }
    v[q] = make_float2(a2.x, b2.x);
    snd[q] = make_float2(a2.y, b2.y);
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) v[15 - q] = fm.xor_shfl(snd[q]);
}

// Last-pass outputs h[q] = H[jsp + q*S] (rowA = H.x, rowB = -H.y) -> the
// thread's 64-bit output pairs at 2m, m = jsp + q*S (q < 8): (own, partner's
// slot 15-q).  Returns rowA/rowB pairs in oa/ob.
template <class G>
__device__ __forceinline__ void fp_out_pairs(const float2 (&h)[16], float2 (&oa)[8], float2 (&ob)[8],
                                             const FastMap<G>& fm) {
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float2 r = fm.xor_shfl(h[15 - q]);
    oa[q] = make_float2(h[q].x, r.x);
    ob[q] = make_float2(-h[q].y, -r.y);
  }
}

}  // namespace acdc
