// AFDF layer (complex diagonals around the FFT pair) for sm_100a.
//
// Reference (paths under /root/reference/pkg/src/acdc):
//   AfdfLayer.forward   layers.py:199-204   y  = IFFT(d * FFT(a * x))   (FFT unnormalised, IFFT 1/N)
//   AfdfLayer.backward  layers.py:206-215   g3 = FFT(dy)/N
//                                           grad_d += sum g3 * conj(FFT(a*x))
//                                           g1 = N * IFFT(g3 * conj(d))
//                                           grad_a += sum g1 * conj(x);  dx = g1 * conj(a)
// Gradient convention dL/dRe + i dL/dIm (layers.py:162-164).  Complex64 rows
// are interleaved (re, im) float pairs.  One complex row per FFT (no packing);
// the inverse transform is conj(FFT(conj(.)))/N so only forward FFTs run.
// For R_first == R_last the last-pass output slots of one FFT are exactly the
// first-pass input slots of the next, so FFT -> (diagonal) -> FFT needs no
// shared-memory exchange in between.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "kernel_common.cuh"  // fft_engine.cuh, pdl_*
#include "runtime.h"
#include "tmem.cuh"

#ifndef ACDC_AFDF_LATE_PAD  // 0: AFDF / row-FFT exchanges after pass 0 unpadded (C5 forward: +0.4%, stays padded)
#define ACDC_AFDF_LATE_PAD 1
#endif
#ifndef ACDC_AFDF_BWD_LATE_PAD  // the TMEM AFDF backward: unpadded after pass 0 (C5 backward -1.6%)
#define ACDC_AFDF_BWD_LATE_PAD 0
#endif
namespace acdc {

struct FParams {
  const float2* x;
  const float2* dy;
  float2* y;  // y (fwd) or dx (bwd)
  const float2* a;
  const float2* d;
  float2* ws;       // bwd partials [groups][2][N]: grad_a, grad_d
  float2* scratch;  // bwd stash when it does not fit in smem
  const float2* tab;
  int64_t rows;
  int64_t ldx, ldy, ldo;  // in complex elements
};

// Loop-invariant parameter load that ptxas may not hoist out of the row loop
// (a hoisted a/d vector would pin 2E registers for the whole kernel).
__device__ __forceinline__ float2 ld_param(const float2* p) {
  float2 r;
  asm volatile("ld.global.v2.f32 {%0, %1}, [%2];" : "=f"(r.x), "=f"(r.y) : "l"(p) : "memory");
  return r;
}

__device__ __forceinline__ float2 conjf2(float2 z) { return make_float2(z.x, -z.y); }
__device__ __forceinline__ float2 cmul_conj(float2 a, float2 b) {  // a * conj(b)
  return vfma(bc(b.y), mul_ni(a), vmul(bc(b.x), a));
}

template <class G>
__device__ __forceinline__ void f_stage_tables(const FParams& p, float* smem, const float2*& tw) {
  if constexpr (G::TW_SMEM) {
    float2* st = reinterpret_cast<float2*>(smem);
    for (int i = threadIdx.x; i < G::TW_ENTRIES; i += blockDim.x) st[i] = p.tab[i];
    __syncthreads();
    tw = st;
  } else {
    tw = p.tab;
  }
}

// Slot (b, q) of pass P sits at position t + b*T + q*N/R_P.
template <class G, int P>
__device__ __forceinline__ int fpos(int b, int q) {
  return b * G::T + q * (G::N / G::radix(P));
}

// Move last-pass slots to first-pass slots (only needed when the radices differ).
template <class G>
__device__ __forceinline__ void last_to_first(float2 (&v)[G::E], Xbuf<G>& xb, const GroupSync<G>& gs, int t) {
  constexpr int PL = G::NPASS - 1;
  if constexpr (G::radix(0) != G::radix(PL)) {
    constexpr int RL = G::radix(PL), R0 = G::radix(0);
    xchg(
        xb, gs,
        [&](const auto& put) {
          const int pt = padi(t);
#pragma unroll
          for (int b = 0; b < G::E / RL; ++b)
#pragma unroll
            for (int q = 0; q < RL; ++q) put(pt + padoff(b * G::T) + padoff(q * (G::N / RL)), v[b * RL + q]);
        },
        [&](const auto& get) { pass_load<G, 0>(v, get, t); });
    (void)R0;
  }
}

template <int LOGN>
__global__ void ACDC_LB(Geo<LOGN>) afdf_fwd_kernel(FParams p) {
  using G = Geo<LOGN>;
  constexpr int E = G::E;
  constexpr int R0 = G::radix(0), PL = G::NPASS - 1, RL = G::radix(PL);
  extern __shared__ __align__(16) float smem_f[];
  const int grp = threadIdx.x / G::T, t = threadIdx.x % G::T;
  const int64_t gid = (int64_t)blockIdx.x * G::GPC + grp, gstride = (int64_t)gridDim.x * G::GPC;
  GroupSync<G> gs(grp);
  Xbuf<G> xb{smem_f + G::TAB_FLOATS + grp * G::GROUP_FLOATS, 0};
  const float2* tw;
  f_stage_tables<G>(p, smem_f, tw);
  const float scale = 1.0f / G::N;
  for (int64_t r = gid; r < p.rows; r += gstride) {
    const float2* xr = p.x + r * p.ldx + t;
    const float2* ar = p.a + t;
    float2 v[E];
#pragma unroll
    for (int b = 0; b < E / R0; ++b)
#pragma unroll
      for (int q = 0; q < R0; ++q) v[b * R0 + q] = cmul(__ldg(xr + fpos<G, 0>(b, q)), ld_param(ar + fpos<G, 0>(b, q)));
    fft_passes<G, 0, ACDC_AFDF_LATE_PAD>(v, xb, gs, tw, t, t, t);
    // V = conj(d * X) at the last-pass slots
    const float2* dr = p.d + t;
#pragma unroll
    for (int b = 0; b < E / RL; ++b)
#pragma unroll
      for (int q = 0; q < RL; ++q) v[b * RL + q] = conjf2(cmul(v[b * RL + q], ld_param(dr + fpos<G, PL>(b, q))));
    last_to_first<G>(v, xb, gs, t);
    fft_passes<G, 0, ACDC_AFDF_LATE_PAD>(v, xb, gs, tw, t, t, t);
    float2* yr = p.y + r * p.ldo + t;
#pragma unroll
    for (int b = 0; b < E / RL; ++b)
#pragma unroll
      for (int q = 0; q < RL; ++q) {
        const float2 h = v[b * RL + q];
        yr[fpos<G, PL>(b, q)] = make_float2(h.x * scale, -h.y * scale);
      }
  }
}

template <int LOGN>
using GeoFT = Geo<LOGN>;
// smem: pass twiddles (no DCT table), two exchange buffers per group, a stash
template <int LOGN>
__host__ __device__ constexpr int afdf_tm_tab_floats() {
  return (2 * GeoFT<LOGN>::TW_ENTRIES + 3) & ~3;
}
template <int LOGN>
__host__ __device__ constexpr int afdf_tm_smem() {
  using G = GeoFT<LOGN>;
  return 4 * (afdf_tm_tab_floats<LOGN>() + G::GPC * 2 * G::BUF_FLOATS) + 16 * G::T * 8;
}
template <int LOGN>
__host__ __device__ constexpr bool afdf_tm_ok() {
  using G = GeoFT<LOGN>;
  return G::E == 16 && G::T >= 32 && G::NPASS >= 2 && G::radix(0) == 16 && G::radix(G::NPASS - 1) == 16 &&
         G::TW_SMEM && G::NBUF == 2 && !G::SPLIT && afdf_tm_smem<LOGN>() <= G::SMEM_LIMIT &&
         (G::CTA / 32 / 4) * 128 <= 512;
}

// Forward with a and d held in TMEM (64 columns per thread, loaded once per
// launch) instead of 32 global loads per row, and the next row's x loaded
// into registers across the second transform.  Same plan conditions as the
// TMEM backward.
template <int LOGN>
__host__ __device__ constexpr int afdf_tmf_smem() {
  using G = GeoFT<LOGN>;
  return 4 * (afdf_tm_tab_floats<LOGN>() + G::GPC * 2 * G::BUF_FLOATS);
}

template <int LOGN>
__global__ void ACDC_LB(GeoFT<LOGN>) afdf_fwd_tm_kernel(FParams p) {
  using G = GeoFT<LOGN>;
  pdl_launch_dependents();  // the backward may stage its prologue while this grid drains
  constexpr int T = G::T;
  static_assert(afdf_tm_ok<LOGN>(), "TMEM AFDF plan");
  extern __shared__ __align__(16) float smem_f[];
  __shared__ uint32_t tm_slot;
  const int grp = threadIdx.x / T, t = threadIdx.x % T;
  const int warp = threadIdx.x >> 5;
  const int64_t gid = (int64_t)blockIdx.x * G::GPC + grp, gstride = (int64_t)gridDim.x * G::GPC;
  GroupSync<G> gs(grp);
  constexpr int TABF = afdf_tm_tab_floats<LOGN>();
  Xbuf<G> xb{smem_f + TABF + grp * 2 * G::BUF_FLOATS, 0};
  if (warp == 0) tmem_alloc<256>(&tm_slot);
  tmem_fence_before();
  const float2* tw;
  f_stage_tables<G>(p, smem_f, tw);
  tmem_fence_after();
  // columns [0,32) a, [32,64) d at positions t + q T
  const uint32_t ta = tmem_addr(tm_slot, warp, (warp >> 2) * 64);
  {
    float2 h[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2* src = (k < 2 ? p.a : p.d) + t + (k & 1) * 8 * T;
#pragma unroll
      for (int j = 0; j < 8; ++j) h[j] = __ldg(src + j * T);
      tmem_st16(ta + 16 * k, h);
    }
  }
  const float scale = 1.0f / G::N;
  float2 xn[16];
  if (gid < p.rows) {
#pragma unroll
    for (int q = 0; q < 16; ++q) xn[q] = __ldg(p.x + gid * p.ldx + t + q * T);
  }
  for (int64_t r = gid; r < p.rows; r += gstride) {
    float2 v[16];
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      float2 av[8];
      tmem_ld16(ta + 16 * half, av);
#pragma unroll
      for (int j = 0; j < 8; ++j) v[8 * half + j] = cmul(xn[8 * half + j], av[j]);
    }
    fft_passes<G, 0, ACDC_AFDF_LATE_PAD>(v, xb, gs, tw, t, t, t);
    // V = conj(d * X)
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      float2 dv[8];
      tmem_ld16(ta + 32 + 16 * half, dv);
#pragma unroll
      for (int j = 0; j < 8; ++j) v[8 * half + j] = conjf2(cmul(v[8 * half + j], dv[j]));
    }
    if (r + gstride < p.rows) {  // next row: in flight across the inverse transform
#pragma unroll
      for (int q = 0; q < 16; ++q) xn[q] = __ldg(p.x + (r + gstride) * p.ldx + t + q * T);
    }
    fft_passes<G, 0, ACDC_AFDF_LATE_PAD>(v, xb, gs, tw, t, t, t);
    float2* yr = p.y + r * p.ldo + t;
#pragma unroll
    for (int q = 0; q < 16; ++q) yr[q * T] = make_float2(v[q].x * scale, -v[q].y * scale);
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (warp == 0) tmem_dealloc<256>(tm_slot);
}

// Row-wise complex DFT (transforms.py:166-179, _kernels.pyx:18-57): forward
// unnormalised, inverse = conj(FFT(conj z)) / N.  Reads a whole row into
// registers before writing, so z == out (in place) is allowed.
template <int LOGN, bool INV>
__global__ void ACDC_LB(Geo<LOGN>) fft_rows_kernel(FParams p) {
  using G = Geo<LOGN>;
  constexpr int E = G::E;
  constexpr int R0 = G::radix(0), PL = G::NPASS - 1, RL = G::radix(PL);
  extern __shared__ __align__(16) float smem_f[];
  const int grp = threadIdx.x / G::T, t = threadIdx.x % G::T;
  const int64_t gid = (int64_t)blockIdx.x * G::GPC + grp, gstride = (int64_t)gridDim.x * G::GPC;
  GroupSync<G> gs(grp);
  Xbuf<G> xb{smem_f + G::TAB_FLOATS + grp * G::GROUP_FLOATS, 0};
  const float2* tw;
  f_stage_tables<G>(p, smem_f, tw);
  const float scale = 1.0f / G::N;
  for (int64_t r = gid; r < p.rows; r += gstride) {
    const float2* xr = p.x + r * p.ldx + t;
    float2 v[E];
#pragma unroll
    for (int b = 0; b < E / R0; ++b)
#pragma unroll
      for (int q = 0; q < R0; ++q) {
        const float2 z = ld_param(xr + fpos<G, 0>(b, q));
        v[b * R0 + q] = INV ? conjf2(z) : z;
      }
    fft_passes<G, 0, ACDC_AFDF_LATE_PAD>(v, xb, gs, tw, t, t, t);
    float2* yr = p.y + r * p.ldo + t;
#pragma unroll
    for (int b = 0; b < E / RL; ++b)
#pragma unroll
      for (int q = 0; q < RL; ++q) {
        const float2 h = v[b * RL + q];
        yr[fpos<G, PL>(b, q)] = INV ? make_float2(h.x * scale, -h.y * scale) : h;
      }
  }
}

// Stash per thread: conj(h2) (E float2) and grad_a partials (E float2).
template <int LOGN>
using GeoF = Geo<LOGN, 4 * Geo<LOGN>::E>;

template <int LOGN>
__global__ void ACDC_LB(GeoF<LOGN>) afdf_bwd_kernel(FParams p) {
  using G = GeoF<LOGN>;
  constexpr int E = G::E, T = G::T;
  constexpr int R0 = G::radix(0), PL = G::NPASS - 1, RL = G::radix(PL);
  extern __shared__ __align__(16) float smem_f[];
  const int grp = threadIdx.x / T, t = threadIdx.x % T;
  const int64_t gid = (int64_t)blockIdx.x * G::GPC + grp, gstride = (int64_t)gridDim.x * G::GPC;
  GroupSync<G> gs(grp);
  float* gbase = smem_f + G::TAB_FLOATS + grp * G::GROUP_FLOATS;
  Xbuf<G> xb{gbase, 0};
  float2* sb = G::STASH_SMEM ? reinterpret_cast<float2*>(gbase + G::NBUF * G::BUF_FLOATS)
                             : p.scratch + gid * (G::GSCRATCH_FLOATS / 2);
  float2* st_h = sb + t;          // [E][T] conj(h2) at the last-pass slots
  float2* st_ga = sb + E * T + t;  // [E][T] grad_a partials at the inverse's output slots
  const float2* tw;
  f_stage_tables<G>(p, smem_f, tw);
  float2 acc_d[E];
#pragma unroll
  for (int i = 0; i < E; ++i) {
    acc_d[i] = make_float2(0.f, 0.f);
    st_ga[i * T] = make_float2(0.f, 0.f);
  }
  for (int64_t r = gid; r < p.rows; r += gstride) {
    const float2* xr = p.x + r * p.ldx + t;
    float2 v[E];
    // h2 = FFT(a * x) -> stash conj(h2)
#pragma unroll
    for (int b = 0; b < E / R0; ++b)
#pragma unroll
      for (int q = 0; q < R0; ++q) v[b * R0 + q] = cmul(__ldg(xr + fpos<G, 0>(b, q)), ld_param(p.a + t + fpos<G, 0>(b, q)));
    fft_passes<G, 0, ACDC_AFDF_LATE_PAD>(v, xb, gs, tw, t, t, t);
#pragma unroll
    for (int i = 0; i < E; ++i) st_h[i * T] = conjf2(v[i]);
    // g = FFT(dy): grad_d partial += g * conj(h2) (1/N applied at the end)
    const float2* dyr = p.dy + r * p.ldy + t;
#pragma unroll
    for (int b = 0; b < E / R0; ++b)
#pragma unroll
      for (int q = 0; q < R0; ++q) v[b * R0 + q] = __ldg(dyr + fpos<G, 0>(b, q));
    fft_passes<G, 0, ACDC_AFDF_LATE_PAD>(v, xb, gs, tw, t, t, t);
#pragma unroll
    for (int b = 0; b < E / RL; ++b)
#pragma unroll
      for (int q = 0; q < RL; ++q) {
        const int i = b * RL + q;
        const float2 h = st_h[i * T];
        acc_d[i] = cadd(acc_d[i], cmul(v[i], h));
        // V = conj(g) * d   (g1 = conj(FFT(V)) / N)
        v[i] = cmul(conjf2(v[i]), ld_param(p.d + t + fpos<G, PL>(b, q)));
      }
    last_to_first<G>(v, xb, gs, t);
    fft_passes<G, 0, ACDC_AFDF_LATE_PAD>(v, xb, gs, tw, t, t, t);
    const float scale = 1.0f / G::N;
    float2* oxr = p.y + r * p.ldo + t;
#pragma unroll
    for (int b = 0; b < E / RL; ++b)
#pragma unroll
      for (int q = 0; q < RL; ++q) {
        const int i = b * RL + q;
        const int pos = fpos<G, PL>(b, q);
        const float2 g1 = make_float2(v[i].x * scale, -v[i].y * scale);
        st_ga[i * T] = cadd(st_ga[i * T], cmul_conj(g1, ld_param(xr + pos)));
        oxr[pos] = cmul_conj(g1, ld_param(p.a + t + pos));
      }
  }
  // partials: ws[gid][0] = grad_a, [1] = grad_d (times 1/N)
  float2* w = p.ws + gid * 2 * G::N + t;
  const float scale = 1.0f / G::N;
#pragma unroll
  for (int b = 0; b < E / RL; ++b)
#pragma unroll
    for (int q = 0; q < RL; ++q) {
      const int i = b * RL + q;
      const int pos = fpos<G, PL>(b, q);
      w[pos] = st_ga[i * T];
      w[G::N + pos] = make_float2(acc_d[i].x * scale, acc_d[i].y * scale);
    }
}

// Backward with its per-thread state in TMEM (tmem.cuh): conj(h2), the x row
// (read once instead of twice), and the grad_a / grad_d partials, 128 columns
// per thread.  a is staged in shared memory once per launch; dy is loaded
// before the h2 transform and consumed after it.  Needs R_first == R_last
// (each thread owns positions t + q T in every stage), E = 16 and whole-warp
// groups.  Same partials and fixed-order reduction as afdf_bwd_kernel.
template <int LOGN>
__global__ void ACDC_LB(GeoFT<LOGN>) afdf_bwd_tm_kernel(FParams p) {
  using G = GeoFT<LOGN>;
  constexpr int T = G::T;
  static_assert(afdf_tm_ok<LOGN>(), "TMEM AFDF backward plan");
  extern __shared__ __align__(16) float smem_f[];
  __shared__ uint32_t tm_slot;
  const int grp = threadIdx.x / T, t = threadIdx.x % T;
  const int warp = threadIdx.x >> 5;
  const int64_t gid = (int64_t)blockIdx.x * G::GPC + grp, gstride = (int64_t)gridDim.x * G::GPC;
  GroupSync<G> gs(grp);
  constexpr int TABF = afdf_tm_tab_floats<LOGN>();
  Xbuf<G> xb{smem_f + TABF + grp * 2 * G::BUF_FLOATS, 0};
  float2* ast = reinterpret_cast<float2*>(smem_f + TABF + G::GPC * 2 * G::BUF_FLOATS) + t;  // [q][t] a at t + q T
  if (grp == 0) {
#pragma unroll
    for (int q = 0; q < 16; ++q) ast[q * T] = __ldg(p.a + t + q * T);
  }
  if (warp == 0) tmem_alloc<512>(&tm_slot);
  tmem_fence_before();
  const float2* tw;
  f_stage_tables<G>(p, smem_f, tw);  // __syncthreads: the a stash and the TMEM base are published
  tmem_fence_after();
  // columns: [0,32) conj(h2), [32,64) x, [64,96) grad_a partials, [96,128) grad_d partials
  const uint32_t ta = tmem_addr(tm_slot, warp, (warp >> 2) * 128);
  {
    float2 z[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) z[i] = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 4; k < 8; ++k) tmem_st16(ta + 16 * k, z);
  }
  pdl_wait();  // x and dy (which may be the forward's y) are read from here on
  const float scale = 1.0f / G::N;
  float2 xn[16];  // this row's x, loaded during the previous row's last transform
  if (gid < p.rows) {
#pragma unroll
    for (int q = 0; q < 16; ++q) xn[q] = __ldg(p.x + gid * p.ldx + t + q * T);
  }
  for (int64_t r = gid; r < p.rows; r += gstride) {
    const float2* dyr = p.dy + r * p.ldy + t;
    float2 v[16], g[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = xn[q];
#pragma unroll
    for (int q = 0; q < 16; ++q) g[q] = __ldg(dyr + q * T);  // in flight across the h2 transform
    {
      float2 h[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) h[q] = v[q];
      tmem_st16(ta + 32, h);
#pragma unroll
      for (int q = 0; q < 8; ++q) h[q] = v[8 + q];
      tmem_st16(ta + 48, h);
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = cmul(v[q], ast[q * T]);
    fft_passes<G, 0, ACDC_AFDF_BWD_LATE_PAD>(v, xb, gs, tw, t, t, t);  // h2 = FFT(a x)
    {
      float2 h[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) h[q] = conjf2(v[q]);
      tmem_st16(ta + 0, h);
#pragma unroll
      for (int q = 0; q < 8; ++q) h[q] = conjf2(v[8 + q]);
      tmem_st16(ta + 16, h);
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = g[q];
    fft_passes<G, 0, ACDC_AFDF_BWD_LATE_PAD>(v, xb, gs, tw, t, t, t);  // g = FFT(dy)
    // grad_d partial += g * conj(h2);  V = conj(g) * d
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      float2 h[8], ad[8];
      tmem_ld16(ta + 16 * half, h);
      tmem_ld16(ta + 96 + 16 * half, ad);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int q = 8 * half + j;
        ad[j] = cadd(ad[j], cmul(v[q], h[j]));
        v[q] = cmul(conjf2(v[q]), ld_param(p.d + t + q * T));
      }
      tmem_st16(ta + 96 + 16 * half, ad);
    }
    if (r + gstride < p.rows) {  // the next row's x: in flight across the last transform
#pragma unroll
      for (int q = 0; q < 16; ++q) xn[q] = __ldg(p.x + (r + gstride) * p.ldx + t + q * T);
    }
    fft_passes<G, 0, ACDC_AFDF_BWD_LATE_PAD>(v, xb, gs, tw, t, t, t);  // g1 = conj(FFT(V)) / N  (times N: the 1/N cancels, see header)
    float2* oxr = p.y + r * p.ldo + t;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      float2 xv[8], ga[8];
      tmem_ld16(ta + 32 + 16 * half, xv);
      tmem_ld16(ta + 64 + 16 * half, ga);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int q = 8 * half + j;
        const float2 g1 = make_float2(v[q].x * scale, -v[q].y * scale);
        ga[j] = cadd(ga[j], cmul_conj(g1, xv[j]));
        oxr[q * T] = cmul_conj(g1, ast[q * T]);
      }
      tmem_st16(ta + 64 + 16 * half, ga);
    }
  }
  // partials: ws[gid][0] = grad_a, [1] = grad_d (times 1/N)
  float2* w = p.ws + gid * 2 * G::N + t;
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    float2 ga[8], ad[8];
    tmem_ld16(ta + 64 + 16 * half, ga);
    tmem_ld16(ta + 96 + 16 * half, ad);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int q = 8 * half + j;
      w[q * T] = ga[j];
      w[G::N + q * T] = make_float2(ad[j].x * scale, ad[j].y * scale);
    }
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (warp == 0) tmem_dealloc<512>(tm_slot);
}

// out_k[i] (+)= sum_g ws[g][k][i] (k < 2 complex outputs of length n), in double,
// fixed order (same scheme as acdc_grad_reduce_kernel).
__global__ void __launch_bounds__(256) afdf_grad_reduce_kernel(const float* __restrict__ ws, int64_t groups, int n,
                                                               float* ga, float* gd, int accumulate) {
  __shared__ double part[8][33];
  const int o = threadIdx.x & 31, s = threadIdx.x >> 5;
  const int64_t len = 2LL * n;  // floats per component
  const int64_t total = 2 * len;
  const int64_t idx = blockIdx.x * 32LL + o;
  double acc = 0.0;
  int comp = 0;
  int64_t i = 0;
  if (idx < total) {
    comp = (int)(idx / len);
    i = idx - comp * len;
    const float* base = ws + comp * len + i;
    double a0 = 0.0, a1 = 0.0;
    int64_t g = s;
#pragma unroll 4
    for (; g + 8 < groups; g += 16) {
      a0 += (double)base[g * total];
      a1 += (double)base[(g + 8) * total];
    }
    for (; g < groups; g += 8) a0 += (double)base[g * total];
    acc = a0 + a1;
  }
  part[s][o] = acc;
  __syncthreads();
  if (s == 0 && idx < total) {
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += part[k][o];
    float* out = comp == 0 ? ga : gd;
    if (accumulate) t += (double)out[i];
    out[i] = (float)t;
  }
}

// kind: 0 = AFDF forward, 1 = AFDF backward, 2 = FFT rows, 3 = inverse FFT rows
template <int LOGN>
static LaunchInfo finfo(int kind) {
  using G = Geo<LOGN>;
  using GB = GeoF<LOGN>;
  const bool bwd = kind == 1;
  LaunchInfo li;
  li.fn = kind == 0   ? (const void*)afdf_fwd_kernel<LOGN>
          : kind == 1 ? (const void*)afdf_bwd_kernel<LOGN>
          : kind == 2 ? (const void*)fft_rows_kernel<LOGN, false>
                      : (const void*)fft_rows_kernel<LOGN, true>;
  li.cta = G::CTA;
  li.gpc = G::GPC;
  li.scratch = bwd ? GB::GSCRATCH_FLOATS : 0;
  li.smem = bwd ? GB::SMEM_BYTES : G::SMEM_BYTES;
#ifndef ACDC_NO_AFDF_TM
  if constexpr (afdf_tm_ok<LOGN>()) {
#ifndef ACDC_NO_AFDF_TMF
    if (kind == 0) {
      li.fn = (const void*)afdf_fwd_tm_kernel<LOGN>;
      li.smem = afdf_tmf_smem<LOGN>();
      li.max_per_sm = 2;  // 256 TMEM columns per CTA
    }
#endif
    if (bwd) {
      li.fn = (const void*)afdf_bwd_tm_kernel<LOGN>;
      li.scratch = 0;
      li.smem = afdf_tm_smem<LOGN>();
      li.max_per_sm = 1;  // 512 TMEM columns per CTA
#ifndef ACDC_NO_PDL
      li.pdl = true;  // prologue overlaps the forward's tail
#endif
    }
  }
#endif
  return li;
}

template <int LOGN>
static LaunchInfo finfo_fft(bool inverse) {
  return finfo<LOGN>(inverse ? 3 : 2);
}

static int fft_info_for(int logn, bool inverse, LaunchInfo* li) {
  switch (logn) {
#define ACDC_TCASE(L)               \
  case L:                           \
    *li = finfo_fft<L>(inverse);    \
    return ACDC_OK;
#ifndef ACDC_ONLY_LOGN
    ACDC_TCASE(1)
    ACDC_TCASE(2)
    ACDC_TCASE(3)
    ACDC_TCASE(4)
    ACDC_TCASE(5)
    ACDC_TCASE(6)
    ACDC_TCASE(7)
    ACDC_TCASE(8)
    ACDC_TCASE(9)
    ACDC_TCASE(10)
    ACDC_TCASE(11)
    ACDC_TCASE(12)
    ACDC_TCASE(13)
    ACDC_TCASE(14)
    ACDC_TCASE(15)
#else
    ACDC_TCASE(ACDC_ONLY_LOGN)
#endif
#undef ACDC_TCASE
    default:
      return set_error(ACDC_E_SIZE, "FFT rows support power-of-two sizes 1..32768");
  }
}

static int finfo_for(int logn, bool bwd, LaunchInfo* li) {
  switch (logn) {
#define ACDC_FCASE(L)       \
  case L:                   \
    *li = finfo<L>(bwd ? 1 : 0);    \
    return ACDC_OK;
#ifndef ACDC_ONLY_LOGN
    ACDC_FCASE(1)
    ACDC_FCASE(2)
    ACDC_FCASE(3)
    ACDC_FCASE(4)
    ACDC_FCASE(5)
    ACDC_FCASE(6)
    ACDC_FCASE(7)
    ACDC_FCASE(8)
    ACDC_FCASE(9)
    ACDC_FCASE(10)
    ACDC_FCASE(11)
    ACDC_FCASE(12)
    ACDC_FCASE(13)
    ACDC_FCASE(14)
#else
    ACDC_FCASE(ACDC_ONLY_LOGN)
#endif
#undef ACDC_FCASE
    default:
      return set_error(ACDC_E_SIZE, "AFDF supports power-of-two sizes 2..16384");
  }
}

static int fsized(int logn, bool bwd, int64_t rows, LaunchInfo* li, int64_t* grid) {
  int rc = finfo_for(logn, bwd, li);
  if (rc) return rc;
  return grid_for(*li, rows, grid);  // one row per group iteration
}

}  // namespace acdc

using namespace acdc;

extern "C" {

int afdf_fwd_c64(const float* x, float* y, const float* a, const float* d, int64_t rows, int32_t n, int64_t ldx,
                 int64_t ldy, acdc_stream_t stream) {
  int logn;
  int rc = check_n(n, &logn);
  if (rc) return rc;
  if (rows < 0 || ldx < n || ldy < n) return ACDC_E_SHAPE;
  if (rows > 0 && (!x || !y || !a || !d)) return ACDC_E_NULL;
  if (((uintptr_t)x | (uintptr_t)y | (uintptr_t)a | (uintptr_t)d) & 7) return ACDC_E_ALIGN;
  if (rows == 0) return ACDC_OK;
  Tables tb;
  if ((rc = get_tables(logn, &tb))) return rc;
  FParams p{};
  p.x = (const float2*)x;
  p.y = (float2*)y;
  p.a = (const float2*)a;
  p.d = (const float2*)d;
  p.tab = tb.tab;
  p.rows = rows;
  p.ldx = ldx;
  p.ldo = ldy;
  LaunchInfo li;
  int64_t grid;
  if ((rc = fsized(logn, false, rows, &li, &grid))) return rc;
  return launch(li, grid, &p, (cudaStream_t)stream);
}

size_t afdf_bwd_workspace_bytes(int64_t rows, int32_t n) {
  int logn;
  if (check_n(n, &logn)) return 0;
  LaunchInfo li;
  int64_t grid;
  if (fsized(logn, true, rows > 0 ? rows : 1, &li, &grid)) return 0;
  return (size_t)grid * li.gpc * (4 * (size_t)n + (size_t)li.scratch) * sizeof(float);
}

int afdf_bwd_c64(const float* x, const float* dy, float* dx, const float* a, const float* d, float* grad_a,
                 float* grad_d, int accumulate, void* ws, size_t ws_bytes, int64_t rows, int32_t n, int64_t ldx,
                 int64_t ldy, int64_t lddx, acdc_stream_t stream) {
  int logn;
  int rc = check_n(n, &logn);
  if (rc) return rc;
  if (rows < 0 || ldx < n || ldy < n || lddx < n) return ACDC_E_SHAPE;
  if (!a || !d || !grad_a || !grad_d || (rows > 0 && (!x || !dy || !dx))) return ACDC_E_NULL;
  if (((uintptr_t)x | (uintptr_t)dy | (uintptr_t)dx | (uintptr_t)a | (uintptr_t)d) & 7) return ACDC_E_ALIGN;
  cudaStream_t st = (cudaStream_t)stream;
  if (rows == 0) {
    if (!accumulate) {
      cudaMemsetAsync(grad_a, 0, 8 * (size_t)n, st);
      cudaMemsetAsync(grad_d, 0, 8 * (size_t)n, st);
    }
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? ACDC_OK : set_cuda_error(e);
  }
  const size_t need = afdf_bwd_workspace_bytes(rows, n);
  if (need == 0) return ACDC_E_CUDA;
  if (!ws || ws_bytes < need) return ACDC_E_WS;
  Tables tb;
  if ((rc = get_tables(logn, &tb))) return rc;
  LaunchInfo li;
  int64_t grid;
  if ((rc = fsized(logn, true, rows, &li, &grid))) return rc;
  const int64_t groups = grid * li.gpc;
  FParams p{};
  p.x = (const float2*)x;
  p.dy = (const float2*)dy;
  p.y = (float2*)dx;
  p.a = (const float2*)a;
  p.d = (const float2*)d;
  p.ws = (float2*)ws;
  p.scratch = p.ws + groups * 2 * (int64_t)n;
  p.tab = tb.tab;
  p.rows = rows;
  p.ldx = ldx;
  p.ldy = ldy;
  p.ldo = lddx;
  if ((rc = launch(li, grid, &p, st))) return rc;
  const int64_t total = 4LL * n;
  afdf_grad_reduce_kernel<<<(int)((total + 31) / 32), 256, 0, st>>>((const float*)ws, groups, n, grad_a, grad_d,
                                                                     accumulate);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ACDC_OK : set_cuda_error(e);
}

int acdc_fft_c64(const float* z, float* out, int64_t rows, int32_t n, int inverse, int64_t ldz, int64_t ldo,
                 acdc_stream_t stream) {
  if (n < 1 || (n & (n - 1)) != 0) {  // FftPlan's message (transforms.py:77-78)
    char msg[96];
    snprintf(msg, sizeof(msg), "FFT size must be a power of two, got %d", n);
    return set_error(ACDC_E_SIZE, msg);
  }
  int logn;
  int rc = check_n(n, &logn);
  if (rc) return rc;
  if (rows < 0 || ldz < n || ldo < n) return ACDC_E_SHAPE;
  if (rows > 0 && (!z || !out)) return ACDC_E_NULL;
  if (((uintptr_t)z | (uintptr_t)out) & 7) return ACDC_E_ALIGN;
  if (rows == 0) return ACDC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (logn == 0) {  // the 1-point DFT (and its inverse) is the identity
    if (z == out) return ACDC_OK;
    cudaError_t e = cudaMemcpy2DAsync(out, 8 * (size_t)ldo, z, 8 * (size_t)ldz, 8, (size_t)rows,
                                      cudaMemcpyDeviceToDevice, st);
    return e == cudaSuccess ? ACDC_OK : set_cuda_error(e);
  }
  Tables tb;
  if ((rc = get_tables(logn, &tb))) return rc;
  LaunchInfo li;
  if ((rc = fft_info_for(logn, inverse != 0, &li))) return rc;
  int64_t grid;
  if ((rc = grid_for(li, rows, &grid))) return rc;
  FParams p{};
  p.x = (const float2*)z;
  p.y = (float2*)out;
  p.tab = tb.tab;
  p.rows = rows;
  p.ldx = ldz;
  p.ldo = ldo;
  return launch(li, grid, &p, st);
}

}  // extern "C"
