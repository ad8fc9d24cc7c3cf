// Half-length (HL) plan for long rows: N = 2^13 ... 2^15 (sm_100a).
//
// The row-pair kernels (acdc_kernels.cu) put two rows into one N-point
// complex FFT; at N >= 16384 that group needs 1024 threads with 32 or 64
// registers each and spills.  Here ONE row is one N/2-point complex FFT of
//   z[m] = v[2m] + i v[2m+1],   v = x[reorder]   (Makhoul, transforms.py:109-113)
// so a group is half as large and the engine is the M = N/2 fast-pairing
// engine of fft_engine.cuh / dct_pair.cuh unchanged.  With the reorder,
//   z[m] = x[4m] + i x[4m+2],   z[M-1-m] = x[4m+3] + i x[4m+1]   (m < M/2)
// so one 128-bit load of x[4m..4m+3] feeds a thread's slot and its partner
// lane's mirror slot (the spatial pairing the engine already shuffles).
//
// DCT-II (reference _kernels.pyx:60-73, X_j = Re(w4s_j V_j), V = FFT_N(v)):
// with Z = FFT_M(z), the frequency pairing k <-> M-k of the engine gives
//   P = Z_k + conj Z_{M-k},  Q = -i (Z_k - conj Z_{M-k}),  U = W_N^k Q
//   2 V_k = P + U,   2 V_{M-k} = conj(P - U)
// and, w4s = 2 c' (c'_j = s_j e^{-i pi j/2N} / 2, the row-pair tables),
//   X_k = Re(c'_k 2V_k),        X_{N-k} = -Im(c'_k 2V_k)
//   X_{M-k} = Re(c'_{M-k} 2V_{M-k}),  X_{M+k} = -Im(c'_{M-k} 2V_{M-k}).
// Each slot owns the four bins {k, N-k, M-k, M+k}; the self-paired slot of
// thread 0 owns {0, M, M/2, 3M/2}.
//
// DCT-III (reference _kernels.pyx:76-91: V'_j = u1_j y_j - i u2_j y_{N-j},
// out[reorder] = Re IFFT_N(V')): with F_j = V'_j / N = conj(c'_j)(y_j - i y_{N-j}),
//   A = F_k + conj F_{M-k},  D = F_k - conj F_{M-k}
//   G_k = conj(A) - i W conj(D),   G_{M-k} = A - i conj(W) D     (W = W_N^k)
// H = FFT_M(G) (a FORWARD FFT: IFFT(Z') = conj FFT(conj Z') / M, the 1/M and
// the 1/N folded in), z' = conj H: out[4m] = Re H_m, out[4m+2] = -Im H_m,
// out[4m+3] = Re H_{M-1-m}, out[4m+1] = -Im H_{M-1-m}.
//
// Backward (layers.py:148-156): g3 = DCT-II(dy) per bin, grad_bias += g3,
// grad_d += h2 g3 (h2 from the forward's cache, same bin layout), g1 =
// DCT-III(d g3), grad_a += x g1, dx = a g1.  The 96 per-thread gradient
// accumulators (3 x 4 bins x 8 slots) live in tensor memory; at N = 32768
// (1024-thread groups, 64 TMEM columns per thread) grad_a goes to the CTA's
// partial row in global memory instead (read-modify-write, L2-resident).
#include <cuda_runtime.h>

#include "kernel_common.cuh"
#include "kparams.h"
#include "runtime.h"
#include "tma.cuh"
#include "tmem.cuh"

#ifndef ACDC_HL_FWD_LD16  // 1: the forward loads the d / bias of two slots per TMEM load
#define ACDC_HL_FWD_LD16 0
#endif
#ifndef ACDC_HL_BWD_LD1  // 1: the backward loads its accumulators and d with one completion wait
#define ACDC_HL_BWD_LD1 0
#endif
#ifndef ACDC_HL_H2_STREAM  // 1: the forward stores the h2 cache evict-first
#define ACDC_HL_H2_STREAM 1
#endif
#ifndef ACDC_HL_Y_STREAM  // 1: the forward stores y evict-first
#define ACDC_HL_Y_STREAM 0
#endif
#ifndef ACDC_HL_SLOT_DYN
#define ACDC_HL_SLOT_DYN 0
#endif

namespace acdc {

template <int LOGN, int GPCX = 0>
struct GeoHL : Geo<LOGN - 1, 0, GPCX> {
  using B = Geo<LOGN - 1, 0, GPCX>;
  static constexpr int NR = 1 << LOGN;  // row length
  static constexpr int M = B::N;        // complex FFT length
  static constexpr int CPH = M + 1;     // c'_j, j <= N/2
  static constexpr int WNH = M / 2 + 1; // W_N^k, k <= N/4
  static constexpr int TAB_HL = (2 * (B::TW_ENTRIES + CPH + WNH) + 3) & ~3;  // floats: all tables
  static constexpr int TAB_TW = (2 * B::TW_ENTRIES + 3) & ~3;                 // floats: pass twiddles only
  static constexpr int SMEM_LIMIT = 227 * 1024;
  __host__ __device__ static constexpr int by(int tab, int nbuf) { return 4 * (tab + B::GPC * nbuf * B::BUF_FLOATS); }
  // all tables in smem if they fit; else the pass twiddles (read by every
  // butterfly, 32-bit addressing) in smem and c' / W_N (once per slot) in global
#ifndef ACDC_HL_PREFER_NBUF2  // 1: double-buffered exchanges before c' / W_N in smem (16384: 157 vs 186 KB)
#define ACDC_HL_PREFER_NBUF2 1  // A/B at N=16384: -2.9% step (scripts/ab_bench.py, round 2)
#endif
  static constexpr bool CP_SMEM = ACDC_HL_PREFER_NBUF2 ? by(TAB_HL, 2) <= SMEM_LIMIT : by(TAB_HL, 1) <= SMEM_LIMIT;
  static constexpr bool TW_SMEM = CP_SMEM || by(TAB_TW, 1) <= SMEM_LIMIT;
  static constexpr int TAB_FLOATS = CP_SMEM ? TAB_HL : (TW_SMEM ? TAB_TW : 0);
  static constexpr int NBUF = by(TAB_FLOATS, 2) <= SMEM_LIMIT ? 2 : 1;
  static constexpr int GROUP_FLOATS = NBUF * B::BUF_FLOATS;
  static constexpr int SMEM_BYTES = by(TAB_FLOATS, NBUF);
  static_assert(B::FP && !B::SPLIT, "the half-length plan runs on the fast-pairing engine");
};

template <class G>
__device__ __forceinline__ void stage_tables_hl(const float2* tab, float* smem, const float2*& tw, const float2*& cp,
                                                const float2*& wn) {
  constexpr int TOT = G::CP_SMEM ? G::TW_ENTRIES + G::CPH + G::WNH : G::TW_ENTRIES;
  if constexpr (G::TW_SMEM) {
    float2* st = reinterpret_cast<float2*>(smem);
    for (int i = threadIdx.x; i < TOT; i += blockDim.x) st[i] = tab[i];
    __syncthreads();
    tw = st;
  } else {
    tw = tab;
  }
  cp = (G::CP_SMEM ? tw : tab) + G::TW_ENTRIES;
  wn = cp + G::CPH;
}

// c' / W_N table read: shared memory, or a non-hoistable global load.
template <class G>
__device__ __forceinline__ float2 cp_load(const float2* tab, int i) {
  if constexpr (G::CP_SMEM) {
    return tab[i];
  } else {
    return ldg_f2_volatile(tab + i);
  }
}

// Bins of frequency slot s (k = jfq + s*S): {k, N-k, M-k, M+k}; special {0, M, M/2, 3M/2}.
template <class G>
struct HlSlot {
  int b[4];
  bool sp;
  __device__ __forceinline__ HlSlot(const FastMap<G>& fm, int s) {
    sp = fm.special(s);
    const int k = fm.jfq + s * FastMap<G>::S;
    b[0] = sp ? 0 : k;
    b[1] = sp ? G::M : G::NR - k;
    b[2] = sp ? G::M / 2 : G::M - k;
    b[3] = sp ? 3 * G::M / 2 : G::M + k;
  }
};

// Per-slot table values: cA = c'_{b0}, cB = c'_{b2} (special: c'_M), W = W_N^k (special: c'_{M/2}).
template <class G>
__device__ __forceinline__ void hl_coefs(const float2* cp, const float2* wn, const FastMap<G>& fm, int s, float2& cA,
                                         float2& cB, float2& W) {
  const int k = fm.jfq + s * FastMap<G>::S;
  if (fm.special(s)) {
    cA = cp_load<G>(cp, 0);
    cB = cp_load<G>(cp, G::M);
    W = cp_load<G>(cp, G::M / 2);
  } else {
    cA = cp_load<G>(cp, k);
    cB = cp_load<G>(cp, G::M - k);
    W = cp_load<G>(wn, k);
  }
}

__device__ __forceinline__ float2 conj2(float2 z) { return make_float2(z.x, -z.y); }

// DCT-II post-pass of one slot: (Z_k, Z_{M-k}) -> X at the slot's four bins.
__device__ __forceinline__ float4 hl_post(float2 zl, float2 zh, float2 cA, float2 cB, float2 W, bool special) {
  if (special) {  // zl = Z_0, zh = Z_{M/2}; W carries c'_{M/2}
    const float v0 = zl.x + zl.y, vm = zl.x - zl.y;
    const float2 wz = cmul(conj2(zh), W);
    return make_float4(2.f * cA.x * v0, 2.f * cB.x * vm, 2.f * wz.x, -2.f * wz.y);
  }
  const float2 zc = conj2(zh);
  const float2 P = cadd(zl, zc);
  const float2 U = cmul(mul_ni(csub(zl, zc)), W);
  const float2 wA = cmul(cadd(P, U), cA);
  const float2 wB = cmul(conj2(csub(P, U)), cB);
  return make_float4(wA.x, -wA.y, wB.x, -wB.y);
}

// DCT-III pre-pass of one slot: Y at the four bins -> G_k (gl), G_{M-k} (gh).
__device__ __forceinline__ void hl_pre(float4 Y, float2 cA, float2 cB, float2 W, bool special, float2& gl,
                                       float2& gh) {
  if (special) {
    const float f0 = 2.f * cA.x * Y.x, fm = 2.f * cB.x * Y.y;
    gl = make_float2(f0 + fm, fm - f0);
    const float2 F = cmul(make_float2(Y.z, -Y.w), conj2(W));
    gh = make_float2(2.f * F.x, 2.f * F.y);
    return;
  }
  const float2 Fk = cmul(make_float2(Y.x, -Y.y), conj2(cA));
  const float2 Fmc = conj2(cmul(make_float2(Y.z, -Y.w), conj2(cB)));
  const float2 A = cadd(Fk, Fmc);
  const float2 D = csub(Fk, Fmc);
  gl = cadd(conj2(A), mul_ni(cmul(conj2(D), W)));
  gh = cadd(A, mul_ni(cmul(D, conj2(W))));
}

__device__ __forceinline__ float4 ld_row_f4(const float4* p) { return __ldg(p); }
__device__ __forceinline__ float4 f4mul(float4 a, float4 b) { return make_float4(a.x * b.x, a.y * b.y, a.z * b.z, a.w * b.w); }

// Pass-0 inputs from a row already in registers as the quads hl_out produces
// (o[q] = x[4m..4m+3], m = jsp + q*S), scaled by a: the fused cascade feeds a
// layer's output into the next layer without a round trip through memory.
template <class G>
__device__ __forceinline__ void hl_from_quads(float2 (&v)[16], const float4 (&o)[8], const float* sc,
                                              const FastMap<G>& fm) {
  constexpr int S = FastMap<G>::S;
  const float4* ps = reinterpret_cast<const float4*>(sc) + fm.jsp;
  float2 snd[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float4 f = f4mul(o[q], __ldg(ps + q * S));
    v[q] = make_float2(f.x, f.z);
    snd[q] = make_float2(f.w, f.y);
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) v[15 - q] = fm.xor_shfl(snd[q]);
}

// Pass-0 inputs of one row: z[m] = (x[4m], x[4m+2]) kept, (x[4m+3], x[4m+1]) sent to the partner's slot 15-q.
template <class G, bool SCALE>
__device__ __forceinline__ void hl_load(float2 (&v)[16], const float* x, const float* sc, const FastMap<G>& fm) {
  constexpr int S = FastMap<G>::S;
  const float4* px = reinterpret_cast<const float4*>(x) + fm.jsp;
  const float4* ps = reinterpret_cast<const float4*>(SCALE ? sc : x) + fm.jsp;
  float2 snd[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    float4 f = ld_row_f4(px + q * S);
    if constexpr (SCALE) f = f4mul(f, __ldg(ps + q * S));
    v[q] = make_float2(f.x, f.z);
    snd[q] = make_float2(f.w, f.y);
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) v[15 - q] = fm.xor_shfl(snd[q]);
}

// Last-pass outputs H[jsp + q*S] -> the row values at 4m..4m+3, m = jsp + q*S (q < 8).
template <class G>
__device__ __forceinline__ void hl_out(const float2 (&h)[16], float4 (&o)[8], const FastMap<G>& fm) {
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float2 r = fm.xor_shfl(h[15 - q]);
    o[q] = make_float4(h[q].x, -r.y, -h[q].y, r.x);
  }
}

__device__ __forceinline__ void tmem_ld16f(uint32_t a, float (&r)[16]) {
  float2 v[8];
  tmem_ld16(a, v);
#pragma unroll
  for (int i = 0; i < 8; ++i) r[2 * i] = v[i].x, r[2 * i + 1] = v[i].y;
}
__device__ __forceinline__ void tmem_st16f(uint32_t a, const float (&r)[16]) {
  float2 v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = make_float2(r[2 * i], r[2 * i + 1]);
  tmem_st16(a, v);
}

// ------------------------------------------------------------------ forward
#ifndef ACDC_HL_FWD_CTA  // forward CTA size where a group is 256 threads (N = 8192): 3 groups, 85 registers
#define ACDC_HL_FWD_CTA 768
#endif
#ifndef ACDC_HL_FWD_CTA128  // forward CTA size where a group is 128 threads (N = 4096)
#define ACDC_HL_FWD_CTA128 512
#endif
template <int LOGN>
constexpr int hl_fwd_gpc() {
  return (Geo<LOGN - 1>::T == 256 && ACDC_HL_FWD_CTA == 768)    ? 3
         : (Geo<LOGN - 1>::T == 128 && ACDC_HL_FWD_CTA128 != 512) ? ACDC_HL_FWD_CTA128 / 128
                                                                   : 0;
}
template <int LOGN>
using GeoHLF = GeoHL<LOGN, hl_fwd_gpc<LOGN>()>;
// d / bias of every thread's 8 spectral slots (32 bins) staged once per launch
// in tensor memory, [slot] x (d0..d3, b0..b3), one tcgen05.ld per slot.
#ifndef ACDC_HL_BWD_ASMEM  // 1: the backward stages its a quads in shared memory where they fit
#define ACDC_HL_BWD_ASMEM 1  // A/B at N=4096: bwd -3%, step -1.6%
#endif
#ifndef ACDC_HL_FWD_ATM  // 1: the forward also stages its 8 a quads (32 floats) in TMEM (columns 64..95)
#define ACDC_HL_FWD_ATM 1  // A/B at N=4096: fwd -3.8%, step -1.8%
#endif
template <int LOGN>
__host__ __device__ constexpr int hl_fwd_ncol() {
  return (ACDC_HL_FWD_ATM && (GeoHLF<LOGN>::CTA / 128) * 96 <= 512) ? 96 : 64;
}
template <int LOGN>
__host__ __device__ constexpr int hl_fwd_cols() {
  constexpr int need = (GeoHLF<LOGN>::CTA / 128) * hl_fwd_ncol<LOGN>();
  return need <= 32 ? 32 : need <= 64 ? 64 : need <= 128 ? 128 : need <= 256 ? 256 : 512;
}
// y = C3(d * C2(a * x) + bias) (layers.py:141-146), one row per group
// iteration; H2C also stores h2 = C2(a x) as [row][slot][t] float4 (bins b0..b3).
template <int LOGN, bool H2C>
__global__ void ACDC_LB(GeoHLF<LOGN>) acdc_fwd_hl_kernel(KParams p) {
  using G = GeoHLF<LOGN>;
  constexpr int T = G::T;
  constexpr int COLS = hl_fwd_cols<LOGN>();
  pdl_launch_dependents();  // the backward may stage its prologue while this grid drains
  extern __shared__ __align__(16) float smem_f[];
#if ACDC_HL_SLOT_DYN  // the TMEM address slot after the dynamic shared memory (not at shared address 0)
  uint32_t& tm_slot = *reinterpret_cast<uint32_t*>(smem_f + G::SMEM_BYTES / 4);
#else
  __shared__ uint32_t tm_slot;
#endif
  const auto c = group_ctx<G>();
  const int t = c.t;
  const int warp = threadIdx.x >> 5;
  GroupSync<G> gs(c.grp);
  Xbuf<G> xb{smem_f + G::TAB_FLOATS + c.grp * G::GROUP_FLOATS, 0};
  const FastMap<G> fm(t, gs.mask);
  if (warp == 0) tmem_alloc<COLS>(&tm_slot);
  tmem_fence_before();
  const float2 *tw, *cp, *wn;
  stage_tables_hl<G>(p.tab, smem_f, tw, cp, wn);
  if constexpr (!G::TW_SMEM) __syncthreads();
  tmem_fence_after();
  constexpr int NCOLF = hl_fwd_ncol<LOGN>();
  const uint32_t ta = tmem_addr(tm_slot, warp, (warp >> 2) * NCOLF);
  // programmatic dependent launch: the prologue above (constant tables, TMEM)
  // may overlap the previous kernel; d / bias, x, y and the h2 cache only after
  pdl_wait();
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const HlSlot<G> sl(fm, s);
    float db[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) db[i] = __ldg(p.d + sl.b[i]), db[4 + i] = __ldg(p.bias + sl.b[i]);
    tmem_st8(ta + 8 * s, db);
  }
  if constexpr (NCOLF == 96) {  // a at this thread's quads jsp + q*S
    const float4* pa = reinterpret_cast<const float4*>(p.a) + fm.jsp;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float av[16];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float4 q4 = __ldg(pa + (4 * h + j) * FastMap<G>::S);
        av[4 * j] = q4.x, av[4 * j + 1] = q4.y, av[4 * j + 2] = q4.z, av[4 * j + 3] = q4.w;
      }
      tmem_st16f(ta + 64 + 16 * h, av);
    }
  }
  for (int64_t r = c.gid; r < p.rows; r += c.gstride) {
    if (t == 0 && r + c.gstride < p.rows) prefetch_row_l2(p.x + (r + c.gstride) * p.ldx, G::NR);
    float2 v[16];
    if constexpr (NCOLF == 96) {
      float4 o[8];
      const float4* px = reinterpret_cast<const float4*>(p.x + r * p.ldx) + fm.jsp;
#pragma unroll
      for (int q = 0; q < 8; ++q) o[q] = ld_row_f4(px + q * FastMap<G>::S);
      float av[32];
      {
        float a0[16], a1[16];
        tmem_ld16f(ta + 64, a0);
        tmem_ld16f(ta + 80, a1);
#pragma unroll
        for (int i = 0; i < 16; ++i) av[i] = a0[i], av[16 + i] = a1[i];
      }
      float2 snd[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 f = make_float4(o[q].x * av[4 * q], o[q].y * av[4 * q + 1], o[q].z * av[4 * q + 2],
                                     o[q].w * av[4 * q + 3]);
        v[q] = make_float2(f.x, f.z);
        snd[q] = make_float2(f.w, f.y);
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) v[15 - q] = fm.xor_shfl(snd[q]);
    } else {
      hl_load<G, true>(v, p.x + r * p.ldx, p.a, fm);
    }
    fft_passes<G, 0, true>(v, xb, gs, tw, t, fm.jsp, fm.jfq);
    {
      float2 w[8], gl[8], gh[8];
      fp_partner<G>(v, w, fm);
#if ACDC_HL_FWD_LD16
      float db16[16];  // d / bias of slots 2k, 2k+1: one TMEM load (one completion wait) per slot pair
#endif
#pragma unroll
      for (int s = 0; s < 8; ++s) {
#if ACDC_HL_FWD_LD16
        if ((s & 1) == 0) tmem_ld16f(ta + 8 * s, db16);
#endif
        float2 cA, cB, W;
        hl_coefs<G>(cp, wn, fm, s, cA, cB, W);
        const HlSlot<G> sl(fm, s);
        float4 X = hl_post(v[s], w[s], cA, cB, W, sl.sp);
        if constexpr (H2C) {
          float4* hp = reinterpret_cast<float4*>(p.h2c + r * G::NR) + s * T + t;
#if ACDC_HL_H2_STREAM
          __stcs(hp, X);
#else
          *hp = X;  // normal caching: the last rows' h2 stays in L2 for the last-first backward
#endif
        }
        float db[8];
#if ACDC_HL_FWD_LD16
#pragma unroll
        for (int i = 0; i < 8; ++i) db[i] = db16[8 * (s & 1) + i];
#else
        tmem_ld8(ta + 8 * s, db);
#endif
        X.x = fmaf(X.x, db[0], db[4]);
        X.y = fmaf(X.y, db[1], db[5]);
        X.z = fmaf(X.z, db[2], db[6]);
        X.w = fmaf(X.w, db[3], db[7]);
        hl_pre(X, cA, cB, W, sl.sp, gl[s], gh[s]);
      }
      fp_scatter<G>(gl, gh, v, fm);
    }
    fft_passes<G, 0, true>(v, xb, gs, tw, t, fm.jfq, fm.jsp);
    float4 o[8];
    hl_out<G>(v, o, fm);
    float4* py = reinterpret_cast<float4*>(p.y + r * p.ldo) + fm.jsp;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
#if ACDC_HL_Y_STREAM
      __stcs(py + q * FastMap<G>::S, o[q]);
#else
      py[q * FastMap<G>::S] = o[q];
#endif
    }
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (warp == 0) tmem_dealloc<COLS>(tm_slot);
}

// Fused cascade of ACDC-only blocks on the half-length plan (the reference's
// acdc_cascade, layers.py:360-362, Cascade.forward 336-339): every row runs
// through all `depth` layers on chip, each layer's output feeding the next
// layer's first FFT in registers (hl_from_quads); checkpoints for the
// backward: x_{l+1} (natural rows, [depth-1][rows][N]) and h2_l (this plan's
// cache layout, [depth][rows][N]) so each block's backward is the single-layer
// cached backward (acdc_bwd_hl_kernel).  d / bias of every layer are read per
// slot from global memory (L1 / L2): too many layers to stage in TMEM.
struct CHParams {
  const float* x;
  float* y;
  const float* a;     // [depth][N]
  const float* d;     // [depth][N]
  const float* bias;  // [depth][N]
  float* xck;         // [depth-1][rows][N]
  float* h2c;         // [depth][h2_stride]: block l's rows at h2c + l * h2_stride + r * N
  const float4* pstash;  // [depth][8 slots][2][T]: d / bias at each thread's slot bins (cascade_hl_pstash_kernel)
  const float2* tab;
  int64_t rows, ldx, ldy, h2_stride;
  int depth;
};

// d / bias of every layer re-laid out per thread and slot, [layer][slot][2][t]
// float4 ((d at the slot's four bins), (bias at them)): the cascade forward
// then reads two coalesced 128-bit values per slot instead of eight scalars.
// The cascade forward keeps two layers' worth of state live: 512-thread CTAs (128 registers) at
// every size (the single-layer forward's 768-thread CTAs at N = 8192 spill 288 B here).
template <int LOGN>
using GeoHLC = GeoHL<LOGN>;

template <int LOGN>
__global__ void cascade_hl_pstash_kernel(const float* d, const float* bias, float4* out, int depth) {
  using G = GeoHLC<LOGN>;
  constexpr int T = G::T, N = G::NR;
  const int t = threadIdx.x;  // one group's threads (T <= 1024)
  const int l = blockIdx.x;
  const FastMap<G> fm(t, 0xffffffffu);
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const HlSlot<G> sl(fm, s);
    const float* dl = d + (int64_t)l * N;
    const float* bl = bias + (int64_t)l * N;
    float4* o = out + ((int64_t)l * 8 + s) * 2 * T + t;
    o[0] = make_float4(dl[sl.b[0]], dl[sl.b[1]], dl[sl.b[2]], dl[sl.b[3]]);
    o[T] = make_float4(bl[sl.b[0]], bl[sl.b[1]], bl[sl.b[2]], bl[sl.b[3]]);
  }
}

template <int LOGN>
__global__ void ACDC_LB(GeoHLC<LOGN>) cascade_fwd_hl_kernel(CHParams p) {
  using G = GeoHLC<LOGN>;
  constexpr int T = G::T, N = G::NR;
  pdl_launch_dependents();
  extern __shared__ __align__(16) float smem_f[];
  const auto c = group_ctx<G>();
  const int t = c.t;
  GroupSync<G> gs(c.grp);
  Xbuf<G> xb{smem_f + G::TAB_FLOATS + c.grp * G::GROUP_FLOATS, 0};
  const FastMap<G> fm(t, gs.mask);
  const float2 *tw, *cp, *wn;
  stage_tables_hl<G>(p.tab, smem_f, tw, cp, wn);
  if constexpr (!G::TW_SMEM) __syncthreads();
  pdl_wait();
  for (int64_t r = c.gid; r < p.rows; r += c.gstride) {
    if (t == 0 && r + c.gstride < p.rows) prefetch_row_l2(p.x + (r + c.gstride) * p.ldx, N);
    float2 v[16];
    hl_load<G, true>(v, p.x + r * p.ldx, p.a, fm);
#pragma unroll 1
    for (int l = 0; l < p.depth; ++l) {
      const float4* pst = p.pstash + (int64_t)l * 16 * T + t;  // [slot][2][t]
      fft_passes<G, 0, true>(v, xb, gs, tw, t, fm.jsp, fm.jfq);
      {
        float2 w[8], gl[8], gh[8];
        fp_partner<G>(v, w, fm);
        float4* hp = reinterpret_cast<float4*>(p.h2c + (int64_t)l * p.h2_stride + r * N) + t;
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          float2 cA, cB, W;
          hl_coefs<G>(cp, wn, fm, s, cA, cB, W);
          const HlSlot<G> sl(fm, s);
          float4 X = hl_post(v[s], w[s], cA, cB, W, sl.sp);
          __stcs(hp + s * T, X);
          const float4 dv = __ldg(pst + 2 * s * T), bv = __ldg(pst + (2 * s + 1) * T);
          X.x = fmaf(X.x, dv.x, bv.x);
          X.y = fmaf(X.y, dv.y, bv.y);
          X.z = fmaf(X.z, dv.z, bv.z);
          X.w = fmaf(X.w, dv.w, bv.w);
          hl_pre(X, cA, cB, W, sl.sp, gl[s], gh[s]);
        }
        fp_scatter<G>(gl, gh, v, fm);
      }
      fft_passes<G, 0, true>(v, xb, gs, tw, t, fm.jfq, fm.jsp);
      float4 o[8];
      hl_out<G>(v, o, fm);
      float4* po = reinterpret_cast<float4*>(l + 1 < p.depth ? p.xck + ((int64_t)l * p.rows + r) * N
                                                             : p.y + r * p.ldy) + fm.jsp;
#pragma unroll
      for (int q = 0; q < 8; ++q) po[q * FastMap<G>::S] = o[q];
      if (l + 1 < p.depth) hl_from_quads<G>(v, o, p.a + (int64_t)(l + 1) * N, fm);
    }
  }
}

// ----------------------------------------------------------------- backward
#ifndef ACDC_HL_BWD_CTA128  // backward CTA size where a group is 128 threads (N = 4096); 0: 512
#define ACDC_HL_BWD_CTA128 0
#endif
template <int LOGN>
constexpr int hl_bwd_gpc() {
  return (Geo<LOGN - 1>::T == 128 && ACDC_HL_BWD_CTA128 > 0) ? ACDC_HL_BWD_CTA128 / 128 : 0;
}
template <int LOGN>
using GeoHLB = GeoHL<LOGN, hl_bwd_gpc<LOGN>()>;
template <int LOGN>
__host__ __device__ constexpr bool hl_tm_a() {  // grad_a also in TMEM (else: the CTA's partial row in global memory)
  return (GeoHLB<LOGN>::CTA / 128) * 96 <= 512;
}
template <int LOGN>
__host__ __device__ constexpr bool hl_tm_d() {  // d of the 32 slot bins also in TMEM (cols 96..127)
  return (GeoHLB<LOGN>::CTA / 128) * 128 <= 512;
}
template <int LOGN>
__host__ __device__ constexpr bool hl_bwd_astash() {  // a quads staged in shared memory (where they fit)
  // N <= 4096 (A/B: N=4096 step -1.6%; N=8192 / 16384 +5% / +4%: the larger stash costs L1 there)
  return ACDC_HL_BWD_ASMEM && GeoHLB<LOGN>::T <= 128 &&
         GeoHLB<LOGN>::SMEM_BYTES + 8 * GeoHLB<LOGN>::T * 16 + 1024 <= GeoHLB<LOGN>::SMEM_LIMIT;
}
template <int LOGN>
__host__ __device__ constexpr bool hl_cta_red() {  // one gradient partial per CTA (all accumulators in TMEM)
#ifdef ACDC_HL_NO_CTA_RED
  return GeoHLB<LOGN>::GPC == 1;
#else
  // leader groups read their followers' columns at the same TMEM lanes (T a multiple or a divisor of 128)
  return (hl_tm_a<LOGN>() && (GeoHLB<LOGN>::T % 128 == 0 || 128 % GeoHLB<LOGN>::T == 0)) ||
         GeoHLB<LOGN>::GPC == 1;
#endif
}
template <int LOGN>
__host__ __device__ constexpr int hl_red_leaders() {  // partials per CTA with hl_cta_red
  constexpr int L = GeoHLB<LOGN>::T >= 128 ? 1 : 128 / GeoHLB<LOGN>::T;
  return L < GeoHLB<LOGN>::GPC ? L : GeoHLB<LOGN>::GPC;
}
template <int LOGN>
__host__ __device__ constexpr int hl_ncol() {
  return hl_tm_d<LOGN>() ? 128 : (hl_tm_a<LOGN>() ? 96 : 64);
}
template <int LOGN>
__host__ __device__ constexpr int hl_cols() {
  constexpr int need = (GeoHLB<LOGN>::CTA / 128) * hl_ncol<LOGN>();
  return need <= 32 ? 32 : need <= 64 ? 64 : need <= 128 ? 128 : need <= 256 ? 256 : 512;
}

// RECOMP: h2 = C2(a x) is recomputed instead of read from the cache.
template <int LOGN, bool RECOMP>
__global__ void ACDC_LB(GeoHLB<LOGN>) acdc_bwd_hl_kernel(KParams p) {
  using G = GeoHLB<LOGN>;
  constexpr int T = G::T;
  constexpr int S = FastMap<G>::S;
  constexpr bool TMA = hl_tm_a<LOGN>();
  constexpr int NCOL = hl_ncol<LOGN>();
  constexpr int COLS = hl_cols<LOGN>();
  constexpr bool PRE = T <= 512;  // h2 of the row loaded across the dy transform (register budget)
  pdl_launch_dependents();        // the reduction may launch early; it waits for this grid
  extern __shared__ __align__(16) float smem_f[];
#if ACDC_HL_SLOT_DYN  // the TMEM address slot after the dynamic shared memory (not at shared address 0)
  uint32_t& tm_slot = *reinterpret_cast<uint32_t*>(smem_f + G::SMEM_BYTES / 4);
#else
  __shared__ uint32_t tm_slot;
#endif
  __shared__ __align__(8) uint64_t dy_bar[G::GPC];
  const auto c = group_ctx<G>();
  const int t = c.t;
  const int warp = threadIdx.x >> 5;
  GroupSync<G> gs(c.grp);
  Xbuf<G> xb{smem_f + G::TAB_FLOATS + c.grp * G::GROUP_FLOATS, 0};
  const FastMap<G> fm(t, gs.mask);
  // dy staging (double-buffered exchanges, an even number of exchanges per
  // row): the next row's dy is bulk-copied into exchange buffer A once the
  // row's last exchange (buffer B) has passed, and read from there next row.
  // 2 (NPASS - 1) exchanges per row, the last one on buffer B; not with RECOMP
  // (its extra h2 transform would run through buffer A before dy is read)
  constexpr bool STAGE = G::NBUF == 2 && !RECOMP;
  static_assert(!STAGE || G::NR <= G::BUF_FLOATS, "a dy row fits in one exchange buffer");
  const bool staged = STAGE && p.stage != 0;
  float* stg = smem_f + G::TAB_FLOATS + c.grp * G::GROUP_FLOATS;
  uint64_t* bar = &dy_bar[c.grp];
  if (staged && t == 0) mbar_init(bar, 1);
  if (warp == 0) tmem_alloc<COLS>(&tm_slot);
  tmem_fence_before();
  const float2 *tw, *cp, *wn;
  stage_tables_hl<G>(p.tab, smem_f, tw, cp, wn);  // __syncthreads: the barrier init is published
  if constexpr (!G::TW_SMEM) __syncthreads();
  tmem_fence_after();
  // columns: [16 sp, 16 sp + 16) = (b, d) bins of slots 2sp, 2sp+1; [64, 96) grad_a positions (TMA)
  const uint32_t ta = tmem_addr(tm_slot, warp, (warp >> 2) * NCOL);
  float* wsg = p.ws + c.gid * 3 * (int64_t)G::NR;  // this group's partial [3][N]: grad_a, grad_d, grad_bias
  float4* gag = reinterpret_cast<float4*>(wsg) + fm.jsp;  // grad_a partial (global, !TMA)
  {
    float z[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) z[i] = 0.f;
#pragma unroll
    for (int k = 0; k < NCOL / 16; ++k) tmem_st16f(ta + 16 * k, z);
    if constexpr (!TMA) {
#pragma unroll
      for (int q = 0; q < 8; ++q) gag[q * S] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if constexpr (hl_tm_d<LOGN>()) {
#pragma unroll
      for (int sp = 0; sp < 4; ++sp) {
        float dd[8];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const HlSlot<G> sl(fm, 2 * sp + j);
#pragma unroll
          for (int i = 0; i < 4; ++i) dd[4 * j + i] = __ldg(p.d + sl.b[i]);
        }
        tmem_st8(ta + 96 + 8 * sp, dd);
      }
    }
  }
  pdl_wait();  // x, dy (maybe the forward's y) and the h2 cache are read from here on
  // a at this thread's quads, [q][t] float4 after the tables / exchange buffers (shared by the groups)
  constexpr bool AST = hl_bwd_astash<LOGN>();
  float4* ast = reinterpret_cast<float4*>(smem_f + G::SMEM_BYTES / 4) + t;
  if constexpr (AST) {
    if (c.grp == 0) {
      const float4* pa0 = reinterpret_cast<const float4*>(p.a) + fm.jsp;
#pragma unroll
      for (int q = 0; q < 8; ++q) ast[q * T] = __ldg(pa0 + q * S);
    }
    __syncthreads();
  }
  auto issue_dy = [&](int64_t row) {  // thread 0 of the group
    fence_proxy_async_smem();
    mbar_expect_tx(bar, (uint32_t)G::NR * 4u);
    bulk_g2s(stg, p.dy + row * p.ldy, (uint32_t)G::NR * 4u, bar);
  };
  uint32_t parity = 0;
  if (staged && t == 0 && c.gid < p.rows) issue_dy(p.rows - 1 - c.gid);
  for (int64_t it = c.gid; it < p.rows; it += c.gstride) {
    const int64_t r = p.rows - 1 - it;  // last-first: the forward's last rows are still in L2
    if (t == 0 && it + c.gstride < p.rows) {
      const int64_t nr = p.rows - 1 - (it + c.gstride);
      prefetch_row_l2(p.dy + nr * p.ldy, G::NR);
      prefetch_row_l2(p.x + nr * p.ldx, G::NR);
    }
    const float4* hc = reinterpret_cast<const float4*>(p.h2c + r * G::NR) + t;
    float4 h2v[8];
    float2 v[16];
    if constexpr (RECOMP) {
      hl_load<G, true>(v, p.x + r * p.ldx, p.a, fm);
      fft_passes<G, 0, true>(v, xb, gs, tw, t, fm.jsp, fm.jfq);
      float2 w[8];
      fp_partner<G>(v, w, fm);
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        float2 cA, cB, W;
        hl_coefs<G>(cp, wn, fm, s, cA, cB, W);
        h2v[s] = hl_post(v[s], w[s], cA, cB, W, fm.special(s));
      }
    } else if constexpr (PRE) {
#pragma unroll
      for (int s = 0; s < 8; ++s) h2v[s] = __ldcs(hc + s * T);
    }
    if (staged) {
      mbar_wait(bar, parity);
      parity ^= 1u;
      float2 snd[8];
      const float4* sq = reinterpret_cast<const float4*>(stg) + fm.jsp;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 f = sq[q * S];
        v[q] = make_float2(f.x, f.z);
        snd[q] = make_float2(f.w, f.y);
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) v[15 - q] = fm.xor_shfl(snd[q]);
      gs.sync();  // buffer A is read by every thread before the first exchange writes it
    } else {
      hl_load<G, false>(v, p.dy + r * p.ldy, nullptr, fm);
    }
    fft_passes<G, 0, true>(v, xb, gs, tw, t, fm.jsp, fm.jfq);
    {
      float2 w[8], gl[8], gh[8];
      fp_partner<G>(v, w, fm);
#pragma unroll
      for (int sp = 0; sp < 4; ++sp) {
        float acc[16], dd[8];
#if ACDC_HL_BWD_LD1
        if constexpr (hl_tm_d<LOGN>()) tmem_ld16_ld8(ta + 16 * sp, acc, ta + 96 + 8 * sp, dd);  // one wait
        else tmem_ld16f(ta + 16 * sp, acc);
#else
        tmem_ld16f(ta + 16 * sp, acc);
        if constexpr (hl_tm_d<LOGN>()) tmem_ld8(ta + 96 + 8 * sp, dd);
#endif
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int s = 2 * sp + j;
          float2 cA, cB, W;
          hl_coefs<G>(cp, wn, fm, s, cA, cB, W);
          const HlSlot<G> sl(fm, s);
          const float4 g3 = hl_post(v[s], w[s], cA, cB, W, sl.sp);
          const float4 h4 = (RECOMP || PRE) ? h2v[s] : __ldcs(hc + s * T);
          float* ab = acc + 8 * j;
          ab[0] += g3.x, ab[1] += g3.y, ab[2] += g3.z, ab[3] += g3.w;
          ab[4] = fmaf(h4.x, g3.x, ab[4]), ab[5] = fmaf(h4.y, g3.y, ab[5]);
          ab[6] = fmaf(h4.z, g3.z, ab[6]), ab[7] = fmaf(h4.w, g3.w, ab[7]);
          float4 y;
          if constexpr (hl_tm_d<LOGN>()) {
            y = make_float4(g3.x * dd[4 * j], g3.y * dd[4 * j + 1], g3.z * dd[4 * j + 2], g3.w * dd[4 * j + 3]);
          } else {
            y = make_float4(g3.x * ld_plain(p.d + sl.b[0]), g3.y * ld_plain(p.d + sl.b[1]),
                            g3.z * ld_plain(p.d + sl.b[2]), g3.w * ld_plain(p.d + sl.b[3]));
          }
          hl_pre(y, cA, cB, W, sl.sp, gl[s], gh[s]);
        }
        tmem_st16f(ta + 16 * sp, acc);
      }
      fp_scatter<G>(gl, gh, v, fm);
    }
    // x of this row: in flight across the g1 transform
    float4 xv[PRE ? 8 : 1];
    const float4* px = reinterpret_cast<const float4*>(p.x + r * p.ldx) + fm.jsp;
    if constexpr (PRE) {
#pragma unroll
      for (int q = 0; q < 8; ++q) xv[q] = ld_row_f4(px + q * S);
    }
    fft_passes<G, 0, true>(v, xb, gs, tw, t, fm.jfq, fm.jsp);
    // the row's last exchange (buffer B) has passed: buffer A takes the next dy
    if (staged && t == 0 && it + c.gstride < p.rows) issue_dy(p.rows - 1 - (it + c.gstride));
    float4 g1[8];
    hl_out<G>(v, g1, fm);
    const float4* pa = reinterpret_cast<const float4*>(p.a) + fm.jsp;
    float4* po = reinterpret_cast<float4*>(p.y + r * p.ldo) + fm.jsp;
    if constexpr (TMA) {
#pragma unroll
      for (int qp = 0; qp < 2; ++qp) {
        float acc[16];
        tmem_ld16f(ta + 64 + 16 * qp, acc);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int q = 4 * qp + j;
          acc[4 * j] = fmaf(xv[PRE ? q : 0].x, g1[q].x, acc[4 * j]);
          acc[4 * j + 1] = fmaf(xv[PRE ? q : 0].y, g1[q].y, acc[4 * j + 1]);
          acc[4 * j + 2] = fmaf(xv[PRE ? q : 0].z, g1[q].z, acc[4 * j + 2]);
          acc[4 * j + 3] = fmaf(xv[PRE ? q : 0].w, g1[q].w, acc[4 * j + 3]);
        }
        tmem_st16f(ta + 64 + 16 * qp, acc);
      }
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 xq = PRE ? xv[PRE ? q : 0] : ld_row_f4(px + q * S);  // (1024-thread groups: loaded at use)
        float4 gacc = gag[q * S];
        gacc.x = fmaf(xq.x, g1[q].x, gacc.x);
        gacc.y = fmaf(xq.y, g1[q].y, gacc.y);
        gacc.z = fmaf(xq.z, g1[q].z, gacc.z);
        gacc.w = fmaf(xq.w, g1[q].w, gacc.w);
        gag[q * S] = gacc;
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) po[q * S] = f4mul(AST ? ast[q * T] : __ldg(pa + q * S), g1[q]);
  }
  // Fewer partials where every accumulator is in TMEM: a "leader" group l < L
  // (L = max(1, 128 / T) groups cover the four TMEM lane quadrants) reads the
  // columns of groups l + L, l + 2L, ... at its own lanes (thread t of group
  // l + kL is warp + kLT/32: same quadrant) and adds them in group order, so the
  // reduction sees L partials per CTA (single stage) instead of one per group.
  constexpr bool CRED = hl_cta_red<LOGN>() && !RECOMP;  // (recompute: +11% from the extra registers, not used)
  constexpr int L = hl_red_leaders<LOGN>();
  if constexpr (CRED && G::GPC > L) {
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    // non-leaders skip the writes (their columns are read by the leaders) and meet
    // everyone at the final barrier (one barrier site for the whole CTA)
    wsg = p.ws + ((int64_t)blockIdx.x * L + c.grp) * 3 * G::NR;
    gag = reinterpret_cast<float4*>(wsg) + fm.jsp;
  }
  const bool writer = !(CRED && G::GPC > L) || c.grp < L;
  auto ld_sum16 = [&](uint32_t col, float (&acc)[16]) {  // this group's 16 columns (+ its followers' in order)
    tmem_ld16f(ta + col, acc);
    if constexpr (CRED && G::GPC > L) {
#pragma unroll
      for (int k = 1; k < G::GPC / L; ++k) {
        float o[16];
        // group l + kL's thread t: warp + k L T / 32 (a multiple of 4: same lane quadrant)
        tmem_ld16f(tmem_addr(tm_slot, warp, ((warp + k * L * (T / 32)) >> 2) * NCOL) + col, o);
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] += o[i];
      }
    }
  };
  // this group's (CTA's) partials: grad_d / grad_bias at the slot bins, grad_a at 4m..4m+3
  if (writer) {
#pragma unroll
  for (int sp = 0; sp < 4; ++sp) {
    float acc[16];
    ld_sum16(16 * sp, acc);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const HlSlot<G> sl(fm, 2 * sp + j);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        wsg[2 * G::NR + sl.b[i]] = acc[8 * j + i];
        wsg[G::NR + sl.b[i]] = acc[8 * j + 4 + i];
      }
    }
  }
  if constexpr (TMA) {
#pragma unroll
    for (int qp = 0; qp < 2; ++qp) {
      float acc[16];
      ld_sum16(64 + 16 * qp, acc);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        gag[(4 * qp + j) * S] = make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
    }
  }
  }  // writer
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (warp == 0) tmem_dealloc<COLS>(tm_slot);
}

// ------------------------------------------------------------------ host
#ifndef ACDC_HL_MIN_LOGN  // smallest size run on the half-length plan (the row-pair kernels below it)
#define ACDC_HL_MIN_LOGN 10  // A/B fwd+bwd (h2 cache): N=1024 -4.4%, 2048 -8.4%, 4096 -4.6%
#endif

template <class K>
static void geom_hl(LaunchInfo& li) {
  li.cta = K::CTA;
  li.gpc = K::GPC;
  li.smem = K::SMEM_BYTES + (ACDC_HL_SLOT_DYN ? 16 : 0);
  li.unit_rows = 1;
  li.hl = true;
}

template <int LOGN>
static void hl_info(int kind, LaunchInfo* li) {
  if (kind == 0 || kind == 4) {
    geom_hl<GeoHLF<LOGN>>(*li);
    li->fn = kind == 0 ? (const void*)acdc_fwd_hl_kernel<LOGN, false> : (const void*)acdc_fwd_hl_kernel<LOGN, true>;
    li->max_per_sm = 512 / hl_fwd_cols<LOGN>();
#if !defined(ACDC_NO_PDL) && (!defined(ACDC_FWD_PDL) || ACDC_FWD_PDL)
    li->pdl = true;  // the prologue overlaps the previous kernel (pdl_wait before any data access)
#endif
    return;
  }
  using G = GeoHLB<LOGN>;
  geom_hl<G>(*li);
  switch (kind) {
    case 1:
    case 5:
      li->fn = kind == 1 ? (const void*)acdc_bwd_hl_kernel<LOGN, true> : (const void*)acdc_bwd_hl_kernel<LOGN, false>;
#ifndef ACDC_NO_PDL
      li->pdl = true;
#endif
      li->max_per_sm = 512 / hl_cols<LOGN>();
      if (hl_bwd_astash<LOGN>()) li->smem += 8 * GeoHLB<LOGN>::T * 16;  // the a stash
      if (hl_cta_red<LOGN>() && kind == 5) li->red_per_cta = hl_red_leaders<LOGN>();  // (cached backward)
      break;
    default: li->fn = nullptr;
  }
}

// Launch description of the half-length kernel for (logn, kind), kinds as in
// acdc_kernels.cu (0 fwd, 1 bwd recompute, 4 fwd + h2 cache, 5 bwd cached);
// returns false when the size / kind is not on the half-length plan.  The
// environment variable ACDC_HL=0 turns the plan off (A/B runs).
bool hl_launch_info(int logn, int kind, LaunchInfo* li) {
  static const bool on = [] {
    const char* e = getenv("ACDC_HL");
    return !(e && e[0] == '0');
  }();
  if (!on || logn < ACDC_HL_MIN_LOGN || logn > 15) return false;
  if (kind != 0 && kind != 1 && kind != 4 && kind != 5) return false;
  switch (logn) {
#if ACDC_HL_MIN_LOGN <= 12
    case 12: hl_info<12>(kind, li); break;
#endif
#if ACDC_HL_MIN_LOGN <= 11
    case 11: hl_info<11>(kind, li); break;
#endif
#if ACDC_HL_MIN_LOGN <= 10
    case 10: hl_info<10>(kind, li); break;
#endif
    case 13: hl_info<13>(kind, li); break;
    case 14: hl_info<14>(kind, li); break;
    case 15: hl_info<15>(kind, li); break;
    default: return false;
  }
  return li->fn != nullptr;
}

// Fused ACDC-only cascade on the half-length plan: launch description, or
// fn == nullptr where the size is not on the plan.
template <int LOGN>
static void hl_cascade_info(LaunchInfo* li) {
  geom_hl<GeoHLC<LOGN>>(*li);
  li->fn = (const void*)cascade_fwd_hl_kernel<LOGN>;
}
template <int LOGN>
static void hl_cascade_pstash(const float* d, const float* bias, float4* out, int depth, cudaStream_t st) {
  cascade_hl_pstash_kernel<LOGN><<<depth, GeoHLC<LOGN>::T, 0, st>>>(d, bias, out, depth);
}
static void hl_cascade_pstash_launch(int logn, const float* d, const float* bias, float4* out, int depth,
                                     cudaStream_t st) {
  switch (logn) {
#if ACDC_HL_MIN_LOGN <= 10
    case 10: hl_cascade_pstash<10>(d, bias, out, depth, st); break;
#endif
#if ACDC_HL_MIN_LOGN <= 11
    case 11: hl_cascade_pstash<11>(d, bias, out, depth, st); break;
#endif
#if ACDC_HL_MIN_LOGN <= 12
    case 12: hl_cascade_pstash<12>(d, bias, out, depth, st); break;
#endif
    case 13: hl_cascade_pstash<13>(d, bias, out, depth, st); break;
    case 14: hl_cascade_pstash<14>(d, bias, out, depth, st); break;
    default: break;
  }
}
static bool hl_cascade_launch_info(int logn, LaunchInfo* li) {
  LaunchInfo probe;
  // N >= 4096: below it the row-pair cascade's two-block backward wins (A/B, 32 blocks at N = 2048:
  // +7.7% on this plan; N = 4096: -4.2%)
  if (logn < 12 || logn > 14 || !hl_launch_info(logn, 4, &probe)) return false;
  switch (logn) {
#if ACDC_HL_MIN_LOGN <= 10
    case 10: hl_cascade_info<10>(li); return true;
#endif
#if ACDC_HL_MIN_LOGN <= 11
    case 11: hl_cascade_info<11>(li); return true;
#endif
#if ACDC_HL_MIN_LOGN <= 12
    case 12: hl_cascade_info<12>(li); return true;
#endif
    case 13: hl_cascade_info<13>(li); return true;
    case 14: hl_cascade_info<14>(li); return true;
    default: return false;
  }
}

bool hl_enabled(int logn) {
  LaunchInfo li;
  return hl_launch_info(logn, 0, &li);
}

}  // namespace acdc

using namespace acdc;

extern "C" {

int cascade_hl_supported(int32_t n) {
  int logn;
  if (check_n(n, &logn)) return 0;
  LaunchInfo li;
  return hl_cascade_launch_info(logn, &li) ? 1 : 0;
}

int cascade_fwd_hl_f32(const float* x, float* y, int32_t depth, int32_t n, const float* a, const float* d,
                       const float* bias, float* ckpt, int64_t rows, int64_t ldx, int64_t ldy, acdc_stream_t stream) {
  int logn;
  int rc = check_n(n, &logn);
  if (rc) return rc;
  LaunchInfo li;
  if (!hl_cascade_launch_info(logn, &li) || depth < 1)
    return set_error(ACDC_E_SIZE, "the half-length fused cascade needs 1024 <= n <= 16384 and depth >= 1");
  if (rows == 0) return ACDC_OK;
  if (rows < 0 || ldx < n || ldy < n) return ACDC_E_SHAPE;
  if (!x || !y || !a || !d || !bias || !ckpt) return ACDC_E_NULL;
  const bool quads = (((uintptr_t)x | (uintptr_t)y | (uintptr_t)a | (uintptr_t)ckpt) & 15) == 0 &&
                     (rows == 1 || ((ldx & 3) == 0 && (ldy & 3) == 0));
  if (!quads) return set_error(ACDC_E_ALIGN, "the half-length fused cascade needs 16-byte aligned rows");
  Tables tb;
  if ((rc = get_tables_hl(logn, &tb))) return rc;
  int64_t grid;
  if ((rc = grid_for(li, rows, &grid))) return rc;
  CHParams p{};
  p.x = x;
  p.y = y;
  p.a = a;
  p.d = d;
  p.bias = bias;
  p.xck = ckpt;
  p.h2c = ckpt + (size_t)(depth - 1) * (size_t)rows * n;
  p.h2_stride = ((rows + 1) / 2) * 2 * (int64_t)n;  // the cascade checkpoint layout (cascade_ckpt_bytes)
  // parameter re-layout after the checkpoints (cascade_ckpt_bytes reserves depth x 2n floats there)
  float4* pst = reinterpret_cast<float4*>(p.h2c + (size_t)depth * p.h2_stride);
  hl_cascade_pstash_launch(logn, d, bias, pst, depth, (cudaStream_t)stream);
  p.pstash = pst;
  p.tab = tb.tab;
  p.rows = rows;
  p.ldx = ldx;
  p.ldy = ldy;
  p.depth = depth;
  return launch(li, grid, &p, (cudaStream_t)stream);
}

}  // extern "C"
