// Register/shared-memory FFT engine for the ACDC kernels (sm_100a).
//
// One "row-pair group" of T threads transforms an N-point complex vector whose
// real and imaginary parts are two independent real rows (A and B).  Each
// thread holds E complex values in registers; passes are Stockham radix-R
// (R in {2,4,8,16}) with compile-time internal twiddles, one table twiddle
// multiply per element between passes, and a padded shared-memory exchange
// between passes.
//
// Stockham pass p (span Ns = product of earlier radices, input stride N/R):
//   butterfly j in [0, N/R), k = j mod Ns
//   a[q] = in[j + q*N/R] * W_{Ns*R}^{q*k}
//   a    = DFT_R(a)
//   out[(j-k)*R + k + q'*Ns] = a[q']
// which after the last pass leaves the DFT in natural order.
//
// Addressing discipline: every shared/global address is "per-thread base +
// compile-time immediate".  Otherwise ptxas CSEs the (thread-invariant)
// address arithmetic of the two FFTs of a row iteration and keeps dozens of
// addresses live across the whole iteration, which spills.  This is why the
// twiddles live in per-pass [q][k] tables and the padding function padi()
// is split into base and offset parts below.
#pragma once
#include <type_traits>
#include <cstdint>
#include <cuda_runtime.h>

#ifdef ACDC_NO_LB  // experiments: report the natural register demand
#define ACDC_LB(...)
#else
#define ACDC_LB(...) __launch_bounds__(__VA_ARGS__::CTA, __VA_ARGS__::MINB)
#endif

namespace acdc {

// ------------------------------------------------------------ complex helpers
// sm_100 executes fp32 pairs as ONE instruction (FADD2 / FMUL2 / FFMA2, PTX
// add/mul/fma.rn.f32x2), and the packed operands take a lane swap (.LO_HI),
// a hi-lane negation (.NP), a whole-operand negation and a scalar broadcast
// (.F32 / immediate) for free.  A complex value is one register pair, so
// every complex add is one FADD2, z * (-i) folds into the consumer's operand
// and a complex multiply is FMUL2 + FFMA2 (scalar: 4 FP instructions).  The
// probe (scripts/fp32x2_probe.cu) measures the same lane throughput for
// FFMA2 and FFMA, so the gain is issue slots: the FP instructions of the FFT
// halve.  -DACDC_SCALAR_FP builds the scalar forms for A/B comparisons.
#ifndef ACDC_SCALAR_FP
#define ACDC_PACKED 1
#endif
__device__ __forceinline__ float2 bc(float s) { return make_float2(s, s); }
#ifdef ACDC_PACKED
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
// a + (-i) b  and  a + i b
__device__ __forceinline__ float2 cadd_ni(float2 a, float2 b) { return __fadd2_rn(a, make_float2(b.y, -b.x)); }
__device__ __forceinline__ float2 cadd_pi(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.y, b.x)); }
// lane-wise a * b, a * b + c
__device__ __forceinline__ float2 vmul(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 vfma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
#else
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cadd_ni(float2 a, float2 b) { return make_float2(a.x + b.y, a.y - b.x); }
__device__ __forceinline__ float2 cadd_pi(float2 a, float2 b) { return make_float2(a.x - b.y, a.y + b.x); }
__device__ __forceinline__ float2 vmul(float2 a, float2 b) { return make_float2(a.x * b.x, a.y * b.y); }
__device__ __forceinline__ float2 vfma(float2 a, float2 b, float2 c) {
  return make_float2(fmaf(a.x, b.x, c.x), fmaf(a.y, b.y, c.y));
}
#endif
// a * w = w.x a + w.y (i a)
__device__ __forceinline__ float2 cmul(float2 a, float2 w) {
  return vfma(make_float2(-a.y, a.x), bc(w.y), vmul(bc(w.x), a));
}
__device__ __forceinline__ float2 cmulc(float2 z, float wr, float wi) { return cmul(z, make_float2(wr, wi)); }
// -i * z
__device__ __forceinline__ float2 mul_ni(float2 z) { return make_float2(z.y, -z.x); }

// Global load that ptxas may not hoist across barriers (large-N tables).
__device__ __forceinline__ float2 ldg_f2_volatile(const float2* p) {
  float2 r;
  asm volatile("ld.global.nc.v2.f32 {%0, %1}, [%2];" : "=f"(r.x), "=f"(r.y) : "l"(p));
  return r;
}

// Forward-DFT constants: W_R^m = exp(-2 pi i m / R)
#define ACDC_C1 0.92387953251128675613f  // cos(pi/8)
#define ACDC_S1 0.38268343236508977173f  // sin(pi/8)
#define ACDC_H 0.70710678118654752440f   // sqrt(2)/2

// ------------------------------------------------------------ DFT butterflies
// All take a[0..R) in natural order and return the forward DFT in natural order.
// Written so every step is one packed instruction (see the helpers above).
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
  a1 = cadd_ni(t1, t3);
  a3 = cadd_pi(t1, t3);
}

// z * W8^1 = H (x + y, y - x);  z * W8^3 = -H (x - y, x + y)
__device__ __forceinline__ float2 mul_w8_1(float2 z) { return vmul(bc(ACDC_H), cadd_ni(z, z)); }
__device__ __forceinline__ float2 mul_w8_3(float2 z) { return vmul(bc(-ACDC_H), cadd_pi(z, z)); }

__device__ __forceinline__ void dft8(float2* a) {
  // decimation in time: E = DFT4(even), O = DFT4(odd)
  dft4(a[0], a[2], a[4], a[6]);
  dft4(a[1], a[3], a[5], a[7]);
  float2 o1 = mul_w8_1(a[3]), o3 = mul_w8_3(a[7]);
  float2 e0 = a[0], e1 = a[2], e2 = a[4], e3 = a[6], o2 = a[5];
  a[0] = cadd(e0, a[1]);
  a[4] = csub(e0, a[1]);
  a[1] = cadd(e1, o1);
  a[5] = csub(e1, o1);
  a[2] = cadd_ni(e2, o2);
  a[6] = cadd_pi(e2, o2);
  a[3] = cadd(e3, o3);
  a[7] = csub(e3, o3);
}

#define ACDC_T1 0.41421356237309504880f  // tan(pi/8)
#ifndef ACDC_DFT16_PLAIN
#define ACDC_DFT16_FMA 1  // FMA-folded second stage (A/B: -1..2% step time at N=4096)
#endif

// Second-stage DFT4 outputs from t0 = u0 + u2, t1 = u0 - u2 and t2 = c*e,
// t3 = c*f (the common twiddle factor c folded into the final FMAs):
//   out0 = t0 + t2, out2 = t0 - t2, out1 = t1 - i t3, out3 = t1 + i t3.
__device__ __forceinline__ void dft4_tail(float2 t0, float2 t1, float2 e, float2 f, float c, float2& o0, float2& o1,
                                          float2& o2, float2& o3) {
  o0 = vfma(bc(c), e, t0);
  o2 = vfma(bc(-c), e, t0);
  o1 = vfma(bc(c), mul_ni(f), t1);
  o3 = vfma(bc(-c), mul_ni(f), t1);
}
// z W^1 = C1 (x + T1 y, y - T1 x);  z W^3 = C1 (T1 x + y, T1 y - x);  z W^9 = -(z W^1 form)
__device__ __forceinline__ float2 tw1_r(float2 z) { return vfma(bc(ACDC_T1), mul_ni(z), z); }
__device__ __forceinline__ float2 tw3_s(float2 z) { return vfma(bc(ACDC_T1), z, mul_ni(z)); }
// z W^2 = H (x + y, y - x);  z W^6 = H (y - x, -(x + y)) = -H (x - y, x + y)
__device__ __forceinline__ float2 tw2_p(float2 z) { return cadd_ni(z, z); }
__device__ __forceinline__ float2 tw6_qn(float2 z) { return cadd_pi(z, z); }  // = -(z W^6) / H

__device__ __forceinline__ void dft16(float2* a) {
  // 4 x 4: n = 4 n1 + n2, k = k1 + 4 k2
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) dft4(a[n2], a[n2 + 4], a[n2 + 8], a[n2 + 12]);
#ifdef ACDC_DFT16_FMA
  // a[n2 + 4 k1] * W16^(n2 k1), then DFT4 over n2, with every non-trivial
  // twiddle folded into FMAs.
  float2 o[16];
  dft4(a[0], a[1], a[2], a[3]);
  o[0] = a[0], o[4] = a[1], o[8] = a[2], o[12] = a[3];
  {  // k1 = 1: W^1, W^2, W^3 (common factor C1 for the odd pair)
    const float2 p = tw2_p(a[6]), r = tw1_r(a[5]), s = tw3_s(a[7]);
    const float2 t0 = vfma(bc(ACDC_H), p, a[4]);
    const float2 t1 = vfma(bc(-ACDC_H), p, a[4]);
    dft4_tail(t0, t1, cadd(r, s), csub(r, s), ACDC_C1, o[1], o[5], o[9], o[13]);
  }
  {  // k1 = 2: W^2, W^4 = -i, W^6 (common factor H)
    const float2 p = tw2_p(a[9]), qn = tw6_qn(a[11]);
    const float2 t0 = cadd_ni(a[8], a[10]);
    const float2 t1 = cadd_pi(a[8], a[10]);
    dft4_tail(t0, t1, csub(p, qn), cadd(p, qn), ACDC_H, o[2], o[6], o[10], o[14]);
  }
  {  // k1 = 3: W^3, W^6, W^9 = -(W^1 form)
    const float2 qn = tw6_qn(a[14]), s = tw3_s(a[13]), r = tw1_r(a[15]);
    const float2 t0 = vfma(bc(-ACDC_H), qn, a[12]);
    const float2 t1 = vfma(bc(ACDC_H), qn, a[12]);
    dft4_tail(t0, t1, csub(s, r), cadd(s, r), ACDC_C1, o[3], o[7], o[11], o[15]);
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = o[i];
  return;
#endif
  // a[n2 + 4 k1] *= W16^(n2 k1)
  a[5] = cmulc(a[5], ACDC_C1, -ACDC_S1);   // W^1
  a[9] = mul_w8_1(a[9]);                   // W^2
  a[13] = cmulc(a[13], ACDC_S1, -ACDC_C1); // W^3
  a[6] = mul_w8_1(a[6]);                   // W^2
  a[10] = mul_ni(a[10]);                   // W^4
  a[14] = mul_w8_3(a[14]);                 // W^6
  a[7] = cmulc(a[7], ACDC_S1, -ACDC_C1);   // W^3
  a[11] = mul_w8_3(a[11]);                 // W^6
  a[15] = cmulc(a[15], -ACDC_C1, ACDC_S1); // W^9
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) dft4(a[4 * k1], a[4 * k1 + 1], a[4 * k1 + 2], a[4 * k1 + 3]);
  // X[k1 + 4 k2] sits at a[4 k1 + k2]: transpose 4x4 (register renaming)
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
  if constexpr (R == 2) {
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
// Radix-16 pass twiddles from 4 loaded powers (W^k, W^2k, W^4k, W^8k) and 11
// packed complex products (2 instructions each) instead of 15 loads: the
// twiddle shared-memory traffic drops 4x (the forward is bound by the
// shared-memory pipe) and the table shrinks from 18 to 4 float2 per k.  The
// products add <= 3 roundings (|err| < 4e-7, far inside the parity bound).
#ifndef ACDC_NO_TWGEN
#define ACDC_TWGEN 1
#else
#define ACDC_TWGEN 0
#endif
// Radix plan and per-pass twiddle-table layout for N = 2^LOGN (16 x small x 16...).
template <int LOGN>
struct Plan {
  static constexpr int N = 1 << LOGN;
  static constexpr int A16 = LOGN / 4;
  static constexpr int REM = LOGN % 4;
  static constexpr int NPASS = LOGN < 4 ? 1 : A16 + (REM ? 1 : 0);
  __host__ __device__ static constexpr int radix(int p) {
    return LOGN < 4 ? N : ((REM && p == 1) ? (1 << REM) : 16);
  }
  __host__ __device__ static constexpr int span(int p) {  // Ns before pass p
    return p == 0 ? 1 : span(p - 1) * radix(p - 1);
  }
  // pass p >= 1 twiddles W_{Ns R}^{q k}, stored at tw_off(p) + k*tw_stride(R) + (q-1):
  // one row per butterfly k so consecutive q pairs load as one 128-bit LDS; the
  // row stride (R+2 float2, or 1 for R = 2) keeps 8 consecutive k on disjoint banks.
  // Radix-16 passes (ACDC_TWGEN) store only W^k, W^2k (float4 at tw_off + 2k) and
  // W^4k, W^8k (float4 at tw_off + 2 Ns + 2k); the other 11 are products.
  __host__ __device__ static constexpr int tw_stride(int r) { return r == 2 ? 1 : ((r == 16 && ACDC_TWGEN) ? 4 : r + 2); }
  __host__ __device__ static constexpr int tw_off(int p) {
    return p <= 1 ? 0 : tw_off(p - 1) + tw_stride(radix(p - 1)) * span(p - 1);
  }
  static constexpr int TW_ENTRIES = tw_off(NPASS);  // float2 entries (0 for one pass)
  static constexpr int CP_ENTRIES = N / 2 + 1;      // DCT post-twiddles c'_k
};

// Per-N compile-time geometry and shared-memory plan.
//
// STASH = floats per thread of per-group scratch the kernel needs besides the
// exchange buffers (the backward keeps g3 and grad_a partials there).  CTAs
// hold GPC row-pair groups (512 threads when T <= 512) sharing one copy of the
// tables; the plan prefers tables in smem and double-buffered exchanges and
// falls back (single buffer, tables in global) until the CTA fits in 227 KB.
#ifndef ACDC_PADS  // float2 padding slots per 16 in the exchange buffers
#define ACDC_PADS 1
#endif
#ifndef ACDC_E32_FROM  // log2 N from which each thread holds 32 values (T = N / 32)
#define ACDC_E32_FROM 15
#endif
template <int LOGN, int STASH = 0, int GPCX = 0, bool GTAB = false, int NBUFX = 0>
struct Geo : Plan<LOGN> {
  using P_ = Plan<LOGN>;
  static constexpr int N = 1 << LOGN;
  static constexpr int E = LOGN >= ACDC_E32_FROM ? 32 : (N >= 16 ? 16 : N);  // complex values per thread
  static constexpr int T = N / E;                                 // threads per row-pair group
  static constexpr int GPC = GPCX ? GPCX : (T <= 512 ? 512 / T : 1);  // groups per CTA
  static constexpr int CTA = T * GPC;                             // threads per CTA
  static constexpr int PADN = N + ACDC_PADS * (N / 16);          // padded float2 slots per buffer
  static constexpr bool SPLIT = (N >= 32768);                     // exchange re / im separately
  static constexpr int BUF_FLOATS = SPLIT ? PADN : 2 * PADN;      // floats per exchange buffer
  static constexpr int STASH_FLOATS = STASH * T;                  // per group
  static constexpr int SMEM_LIMIT = 227 * 1024;
  static constexpr int TAB_FULL = (2 * (P_::TW_ENTRIES + P_::CP_ENTRIES) + 3) & ~3;
  __host__ __device__ static constexpr int bytes(bool tab, int nbuf, bool stash) {
    return 4 * ((tab ? TAB_FULL : 0) + GPC * (nbuf * BUF_FLOATS + (stash ? STASH_FLOATS : 0)));
  }
  // the stash goes to global scratch only if it cannot fit beside one buffer
  static constexpr bool STASH_SMEM = bytes(false, 1, true) <= SMEM_LIMIT;
  static constexpr bool FIT_T2 = !SPLIT && bytes(true, 2, STASH_SMEM) <= SMEM_LIMIT;
  static constexpr bool FIT_T1 = bytes(true, 1, STASH_SMEM) <= SMEM_LIMIT;
  static constexpr bool FIT_G2 = !SPLIT && bytes(false, 2, STASH_SMEM) <= SMEM_LIMIT;
  static constexpr bool TW_SMEM = !GTAB && (FIT_T2 || FIT_T1);  // tables staged in smem?
  static constexpr int NBUF = NBUFX ? NBUFX : (FIT_T2 ? 2 : (FIT_T1 ? 1 : (FIT_G2 ? 2 : 1)));
  static constexpr int TAB_FLOATS = TW_SMEM ? TAB_FULL : 0;
  static constexpr int SMEM_BYTES = bytes(TW_SMEM, NBUF, STASH_SMEM);
  static constexpr int GROUP_FLOATS = NBUF * BUF_FLOATS + (STASH_SMEM ? STASH_FLOATS : 0);
  // fast-pairing path (dct_pair.cuh): one radix-16 butterfly per thread in
  // the first and last pass
  static constexpr bool FP = E == 16 && N >= 256 && P_::NPASS >= 2 && P_::radix(0) == 16 &&
                             P_::radix(P_::NPASS - 1) == 16 && T == N / 16;
  // global scratch floats per group when the stash does not fit in smem
  static constexpr int GSCRATCH_FLOATS = STASH_SMEM ? 0 : STASH_FLOATS;
#ifdef ACDC_MINB_OVERRIDE
  static constexpr int MINB = ACDC_MINB_OVERRIDE;
#else
  static constexpr int MINB = 1;  // 512-thread CTAs: 128 registers per thread
#endif
};

// Padded exchange index (ACDC_PADS float2 of padding per 16 slots).  For a
// power-of-two stride S and base j < S (or S, j multiples of 16):
//   padi(j + q*S) = padi(j) + padoff(q*S)
// which lets every exchange address be a base register plus an immediate.
// With an even pad every 16-slot run starts 16-byte aligned, so the first
// pass (contiguous outputs per thread) stores 128-bit pairs.
__host__ __device__ constexpr int padi(int i) { return i + ACDC_PADS * (i >> 4); }
__host__ __device__ constexpr int padoff(int off) { return off + ACDC_PADS * (off >> 4); }

// Group-local barrier: warp mask for T <= 32, named barrier otherwise.
template <class G>
struct GroupSync {
  unsigned mask;
  int bar_id;
  __device__ __forceinline__ GroupSync(int grp) {
    if constexpr (G::T < 32) {
      int lane = threadIdx.x & 31;
      mask = ((1u << G::T) - 1u) << (lane & ~(G::T - 1));
    } else {
      mask = 0xffffffffu;
    }
    bar_id = 1 + grp;
  }
  __device__ __forceinline__ void sync() const {
    if constexpr (G::T <= 32) {
      __syncwarp(mask);
    } else if constexpr (G::GPC == 1) {
      asm volatile("bar.sync 0;" ::: "memory");
    } else {
      asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(G::T) : "memory");
    }
  }
};

// Table read: shared memory (ordered by the group barriers) or, for large N,
// a non-hoistable global load.
template <class G>
__device__ __forceinline__ float2 tab_load(const float2* tab, int i) {
  if constexpr (G::TW_SMEM) {
    return tab[i];
  } else {
    return ldg_f2_volatile(tab + i);
  }
}

template <class G>
__device__ __forceinline__ float4 tab_load4(const float2* tab) {
  if constexpr (G::TW_SMEM) {
    return *reinterpret_cast<const float4*>(tab);
  } else {
    float4 r;
    asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(tab));
    return r;
  }
}

// ------------------------------------------------------------ exchanges
// Element accessors for one exchange, taking PADDED indices: full float2
// slots, or one component at a time when the buffer holds N floats (SPLIT).
struct PutFull {
  static constexpr bool kPair = true;
  float2* b;
  __device__ __forceinline__ void operator()(int pi, float2 v) const { b[pi] = v; }
  // slots pi, pi + 1 (pi even): one 128-bit store
  __device__ __forceinline__ void pair(int pi, float2 v0, float2 v1) const {
    *reinterpret_cast<float4*>(b + pi) = make_float4(v0.x, v0.y, v1.x, v1.y);
  }
};
struct GetFull {
  const float2* b;
  __device__ __forceinline__ void operator()(int pi, float2& d) const { d = b[pi]; }
};
struct PutComp {
  static constexpr bool kPair = false;
  float* b;
  int c;
  __device__ __forceinline__ void operator()(int pi, float2 v) const { b[pi] = c ? v.y : v.x; }
};
struct GetComp {
  const float* b;
  int c;
  __device__ __forceinline__ void operator()(int pi, float2& d) const {
    float f = b[pi];
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

// ------------------------------------------------------------ Stockham passes
// The thread's butterflies in pass P are j0 + b*T (b < E/R).  Normally j0 = t;
// the fast-pairing path (dct_pair.cuh) remaps j0 in the first and last pass.
// All inputs/outputs are addressed as padi(j0) + padoff(b*T) + padoff(q*S).

// Compute pass P in registers (table twiddle + DFT_R).
template <class G, int P>
__device__ __forceinline__ void pass_compute(float2 (&v)[G::E], const float2* tw, int j0) {
  constexpr int R = G::radix(P);
  constexpr int NS = G::span(P);
  constexpr int NB = G::E / R;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    if constexpr (NS > 1) {
      const int k = (j0 + b * G::T) & (NS - 1);
      const float2* row = tw + G::tw_off(P) + k * G::tw_stride(R);  // row[q-1] = W_{NS R}^{q k}
      if constexpr (R == 16 && ACDC_TWGEN) {
        const float4 w12 = tab_load4<G>(tw + G::tw_off(P) + 2 * k);
        const float4 w48 = tab_load4<G>(tw + G::tw_off(P) + 2 * NS + 2 * k);
        float2* a = &v[b * R];
        const float2 w1 = make_float2(w12.x, w12.y), w2 = make_float2(w12.z, w12.w);
        const float2 w4 = make_float2(w48.x, w48.y), w8 = make_float2(w48.z, w48.w);
        const float2 w3 = cmul(w1, w2), w5 = cmul(w1, w4), w6 = cmul(w2, w4), w7 = cmul(w3, w4);
        a[1] = cmul(a[1], w1);
        a[2] = cmul(a[2], w2);
        a[3] = cmul(a[3], w3);
        a[4] = cmul(a[4], w4);
        a[5] = cmul(a[5], w5);
        a[6] = cmul(a[6], w6);
        a[7] = cmul(a[7], w7);
        a[8] = cmul(a[8], w8);
        a[9] = cmul(a[9], cmul(w1, w8));
        a[10] = cmul(a[10], cmul(w2, w8));
        a[11] = cmul(a[11], cmul(w3, w8));
        a[12] = cmul(a[12], cmul(w4, w8));
        a[13] = cmul(a[13], cmul(w5, w8));
        a[14] = cmul(a[14], cmul(w6, w8));
        a[15] = cmul(a[15], cmul(w7, w8));
      } else if constexpr (R == 2) {
        v[b * R + 1] = cmul(v[b * R + 1], tab_load<G>(row, 0));
      } else {
#pragma unroll
        for (int q = 1; q < R; q += 2) {
          const float4 w2 = tab_load4<G>(row + (q - 1));
          v[b * R + q] = cmul(v[b * R + q], make_float2(w2.x, w2.y));
          if (q + 1 < R) v[b * R + q + 1] = cmul(v[b * R + q + 1], make_float2(w2.z, w2.w));
        }
      }
    }
    dft<R>(&v[b * R]);
  }
}

// Exchange index: padded (the exchange after pass 0, whose writers are 16
// slots apart) or plain (every later exchange: each half-warp writes and reads
// 16 consecutive slots, and the frequency-pairing reads S-16w-15 ... S-16w
// then stay on 16 distinct bank pairs).
template <bool PAD>
__device__ __forceinline__ constexpr int xi(int i) { return PAD ? padi(i) : i; }

// Write the outputs of pass P at their autosorted positions.
template <class G, int P, class PUT, bool PAD = true>
__device__ __forceinline__ void pass_store(const float2 (&v)[G::E], const PUT& put, int j0) {
  constexpr int R = G::radix(P);
  constexpr int NS = G::span(P);
  constexpr int NB = G::E / R;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int j = j0 + b * G::T;
    const int k = j & (NS - 1);
    const int pd = xi<PAD>((j - k) * R + k);
    if constexpr (NS == 1 && ACDC_PADS % 2 == 0 && PUT::kPair && R >= 2) {
#pragma unroll
      for (int q = 0; q < R; q += 2) put.pair(pd + q, v[b * R + q], v[b * R + q + 1]);
    } else {
#pragma unroll
      for (int q = 0; q < R; ++q) put(pd + xi<PAD>(q * NS), v[b * R + q]);
    }
  }
}

// Read the inputs of pass P (stride N/R).
template <class G, int P, class GET, bool PAD = true>
__device__ __forceinline__ void pass_load(float2 (&v)[G::E], const GET& get, int j0) {
  constexpr int R = G::radix(P);
  constexpr int NB = G::E / R;
  constexpr int S = G::N / R;
  const int pt = xi<PAD>(j0);
#pragma unroll
  for (int b = 0; b < NB; ++b)
#pragma unroll
    for (int q = 0; q < R; ++q) get(pt + xi<PAD>(b * G::T) + xi<PAD>(q * S), v[b * R + q]);
}

// All passes of the FFT; v holds pass-0 inputs on entry and the natural-order
// outputs of the last pass on exit (v[b*R_L + q] = X[j_b + q*N/R_L]).  Pass 0
// uses butterfly base jf, the last pass jl, the others t.  LATE_PAD = false:
// the exchanges after pass 1, 2, ... use plain indices (see xi).
template <class G, int P = 0, bool LATE_PAD = true>
__device__ __forceinline__ void fft_passes(float2 (&v)[G::E], Xbuf<G>& xb, const GroupSync<G>& gs,
                                           const float2* tw, int t, int jf, int jl) {
  constexpr int L = G::NPASS - 1;
  const int jp = P == 0 ? jf : (P == L ? jl : t);
  pass_compute<G, P>(v, tw, jp);
  if constexpr (P < L) {
    constexpr int PN = P + 1;
    const int jn = PN == L ? jl : t;
    constexpr bool PAD = LATE_PAD || P == 0 || G::T < 16;
    xchg(
        xb, gs, [&](const auto& put) { pass_store<G, P, std::decay_t<decltype(put)>, PAD>(v, put, jp); },
        [&](const auto& get) { pass_load<G, PN, std::decay_t<decltype(get)>, PAD>(v, get, jn); });
    fft_passes<G, PN, LATE_PAD>(v, xb, gs, tw, t, jf, jl);
  }
}
template <class G>
__device__ __forceinline__ void fft_passes(float2 (&v)[G::E], Xbuf<G>& xb, const GroupSync<G>& gs,
                                           const float2* tw, int t) {
  fft_passes<G, 0>(v, xb, gs, tw, t, t, t);
}

// Makhoul reorder (transforms.py:109-113): packed index m -> signal index
// src = 2m (m < N/2) or 2(N-1-m)+1.  For the first/last-pass slot (b, q) of
// thread t, m = t + b*T + q*N/R lies in the lower half iff q < R/2, so
//   q <  R/2:  src = 2t         + off(b, q)
//   q >= R/2:  src = (2N-1-2t)  - off(b, q),   off = 2(b*T + q*N/R)
template <class G, int P>
struct RowMap {
  static constexpr int R = G::radix(P);
  static constexpr int NB = G::E / R;
  __host__ __device__ static constexpr bool lower(int q) { return 2 * q < R; }
  __host__ __device__ static constexpr int off(int b, int q) { return 2 * (b * G::T + q * (G::N / R)); }
};

}  // namespace acdc
