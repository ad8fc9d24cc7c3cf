// Fused ACDC cascade forward for sm_100a (reference Cascade.forward,
// layers.py:336-339, over AcdcLayer / ReluLayer / PermutationLayer,
// layers.py:141-146, 225-228, 257-261).
//
// One kernel runs K blocks  x_{l+1} = perm_l( relu_l( ACDC_l(x_l) ) )  per row
// pair with every intermediate on chip: the ACDC output stays in registers,
// ReLU is applied in registers and the permutation is one shared-memory
// gather; x is read once and y written once.  For the backward it writes
// checkpoints: x_{l+1} (natural layout, needed for grad_a and the ReLU mask)
// and h2_l = C2(a_l x_l) (thread-native cache layout), so each block's backward
// is one cached-h2 ACDC backward whose epilogue applies the previous block's
// ReLU mask and inverse permutation (acdc_kernels.cu, KParams::epi_*).
// Fast-pairing sizes only (256 <= N <= 16384).
#include <cuda_runtime.h>

#include <cstdint>

#include "kernel_common.cuh"
#include "runtime.h"

#ifndef ACDC_CASCADE_LATE_PAD  // 0: the fused cascade forward's exchanges after pass 0 are unpadded
#define ACDC_CASCADE_LATE_PAD 1
#endif
namespace acdc {

#ifndef ACDC_CASCADE_CTA  // threads per CTA of the fused cascade forward (0: the plan's 512)
#define ACDC_CASCADE_CTA 0
#endif
template <int LOGN>
using GeoC = Geo<LOGN, 0, (ACDC_CASCADE_CTA && ACDC_CASCADE_CTA / Geo<LOGN>::T > 1) ? ACDC_CASCADE_CTA / Geo<LOGN>::T : 0>;

// d / bias of every block re-laid out per thread and slot, [block][slot][t]
// float4 (d_lo, d_hi, b_lo, b_hi): the forward reads one coalesced 128-bit
// value per slot and block instead of four scalar loads.
template <int LOGN>
__global__ void cascade_pstash_kernel(const float* d, const float* bias, float4* out) {
  using G = Geo<LOGN>;
  constexpr int T = G::T, N = G::N;
  const int t = threadIdx.x;  // one group's threads
  const int l = blockIdx.x;
  const FastMap<G> fm(t, 0xffffffffu);
  const float* dl = d + (int64_t)l * N;
  const float* bl = bias + (int64_t)l * N;
#pragma unroll
  for (int s = 0; s < 8; ++s)
    out[((int64_t)l * 8 + s) * T + t] = make_float4(*fm.plo(dl, s), *fm.phi(dl, s), *fm.plo(bl, s), *fm.phi(bl, s));
}

struct CParams {
  const float* x;
  float* y;
  const float* a;        // [K][N]
  const float* d;        // [K][N]
  const float* bias;     // [K][N]
  const int* perm;       // [K][N]; block l uses perm + l*N when flags[l] & 2
  const uint8_t* flags;  // [K]: bit0 ReLU after block l, bit1 permutation after it
  float* xck;            // [K-1][rows][N]: x_{l+1}
  float* h2c;            // [K][npairs][2N]: h2_l cache
  const float4* pstash;  // [K][8 slots][T]: (d_lo, d_hi, b_lo, b_hi) per thread (cascade_pstash_kernel)
  const float2* tab;
  int64_t rows, ldx, ldy;
  int depth;
};

template <int LOGN>
__global__ void ACDC_LB(GeoC<LOGN>) cascade_fwd_kernel(CParams p) {
  using G = GeoC<LOGN>;
  static_assert(G::FP, "cascade fusion needs the fast-pairing path");
  pdl_launch_dependents();  // the last block's backward may stage its prologue while this grid drains
  constexpr int N = G::N, T = G::T, S = FastMap<G>::S;
  extern __shared__ __align__(16) float smem_f[];
  const auto c = group_ctx<G>();
  const int t = c.t;
  GroupSync<G> gs(c.grp);
  Xbuf<G> xb{smem_f + G::TAB_FLOATS + c.grp * G::GROUP_FLOATS, 0};
  const float2 *tw, *cp;
  stage_tables<G>(p.tab, smem_f, tw, cp);
  const FastMap<G> fm(t, gs.mask);
  const int64_t npairs = (p.rows + 1) >> 1;
  const float2 chi = tab_load<G>(cp, N / 2);
  for (int64_t rp = c.gid; rp < npairs; rp += c.gstride) {
    const int64_t ra = 2 * rp;
    const bool hasb = ra + 1 < p.rows;
    const int64_t rb = hasb ? ra + 1 : ra;
    if (t == 0 && rp + c.gstride < npairs) {
      const int64_t nr = 2 * (rp + c.gstride);
      prefetch_row_l2(p.x + nr * p.ldx, N);
      if (nr + 1 < p.rows) prefetch_row_l2(p.x + (nr + 1) * p.ldx, N);
    }
    // block-0 input pairs (rows A, B) at 2m, 2m+1, m = jsp + q*S
    float2 pa[8], pb[8];
    {
      const float* xa = p.x + ra * p.ldx + 2 * fm.jsp;
      const float* xbr = p.x + rb * p.ldx + 2 * fm.jsp;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        pa[q] = ld_f2(xa + 2 * q * S);
        pb[q] = hasb ? ld_f2(xbr + 2 * q * S) : make_float2(0.f, 0.f);
      }
    }
    float2 an[8];  // a_l at this thread's position pairs (issued one block ahead)
    {
      const float* pav = p.a + 2 * fm.jsp;
#pragma unroll
      for (int q = 0; q < 8; ++q) an[q] = ld_f2(pav + 2 * q * S);
    }
    for (int l = 0; l < p.depth; ++l) {
      // d_l / bias_l of this thread's spectral slots: in flight across the first transform
      float4 dbv[8];
#pragma unroll
      for (int s = 0; s < 8; ++s) dbv[s] = __ldg(p.pstash + ((int64_t)l * 8 + s) * T + t);
      float2 v[16];
      {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          pa[q] = vmul(pa[q], an[q]);
          pb[q] = vmul(pb[q], an[q]);
        }
        fp_from_pairs<G>(v, pa, pb, fm);
      }
      fft_passes<G, 0, ACDC_CASCADE_LATE_PAD>(v, xb, gs, tw, t, fm.jsp, fm.jfq);
      {
        float2 w[8], gl[8], gh[8];
        fp_partner<G>(v, w, fm);
        float4* hc = reinterpret_cast<float4*>(p.h2c + ((int64_t)l * npairs + rp) * 2 * N) + t;
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          const float2 cs = tab_load<G>(fm.plo(cp, s), 0);
          float2 xl, xh;
          dct2_post(v[s], w[s], cs, fm.special(s), chi, xl, xh);
          __stcs(hc + s * T, make_float4(xl.x, xl.y, xh.x, xh.y));
          xl = vfma(xl, bc(dbv[s].x), bc(dbv[s].z));
          xh = vfma(xh, bc(dbv[s].y), bc(dbv[s].w));
          dct3_pre(xl, xh, cs, fm.special(s), chi, gl[s], gh[s]);
        }
        fp_scatter<G>(gl, gh, v, fm);
      }
      if (l + 1 < p.depth) {  // a_{l+1}: in flight across the second transform
        const float* pav = p.a + (int64_t)(l + 1) * N + 2 * fm.jsp;
#pragma unroll
        for (int q = 0; q < 8; ++q) an[q] = ld_f2(pav + 2 * q * S);
      }
      fft_passes<G, 0, ACDC_CASCADE_LATE_PAD>(v, xb, gs, tw, t, fm.jfq, fm.jsp);
      fp_out_pairs<G>(v, pa, pb, fm);  // ACDC_l output pairs
      const int fl = p.flags ? p.flags[l] : 0;
      if (fl & 1) {  // ReLU, strict x > 0 (layers.py:227)
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          pa[q] = make_float2(fmaxf(pa[q].x, 0.f), fmaxf(pa[q].y, 0.f));
          pb[q] = make_float2(fmaxf(pb[q].x, 0.f), fmaxf(pb[q].y, 0.f));
        }
      }
      if (l == p.depth - 1) break;
      if (fl & 2) {  // x_{l+1}[j] = r_l[perm[j]]  (layers.py:261) through shared memory
        const int* pl = p.perm + (int64_t)l * N + 2 * fm.jsp;
        xchg(
            xb, gs,
            [&](const auto& put) {
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                const int m2 = 2 * (fm.jsp + q * S);
                put(padi(m2), make_float2(pa[q].x, pb[q].x));
                put(padi(m2 + 1), make_float2(pa[q].y, pb[q].y));
              }
            },
            [&](const auto& get) {
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                const int s0 = ld_plain_i(pl + 2 * q * S), s1 = ld_plain_i(pl + 2 * q * S + 1);
                float2 e0, e1;
                get(padi(s0), e0);
                get(padi(s1), e1);
                pa[q] = make_float2(e0.x, e1.x);
                pb[q] = make_float2(e0.y, e1.y);
              }
            });
      }
      // checkpoint x_{l+1}
      float* xa = p.xck + ((int64_t)l * p.rows + ra) * N + 2 * fm.jsp;
      float* xbw = p.xck + ((int64_t)l * p.rows + rb) * N + 2 * fm.jsp;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        *reinterpret_cast<float2*>(xa + 2 * q * S) = pa[q];
        if (hasb) *reinterpret_cast<float2*>(xbw + 2 * q * S) = pb[q];
      }
    }
    float* ya = p.y + ra * p.ldy + 2 * fm.jsp;
    float* yb = p.y + rb * p.ldy + 2 * fm.jsp;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      *reinterpret_cast<float2*>(ya + 2 * q * S) = pa[q];
      if (hasb) *reinterpret_cast<float2*>(yb + 2 * q * S) = pb[q];
    }
  }
}

template <int LOGN>
static LaunchInfo cinfo() {
  using G = GeoC<LOGN>;
  LaunchInfo li;
  li.fn = (const void*)cascade_fwd_kernel<LOGN>;
  li.cta = G::CTA;
  li.gpc = G::GPC;
  li.smem = G::SMEM_BYTES;
  return li;
}

template <int LOGN>
static void pstash_launch(const float* d, const float* bias, float4* out, int depth, cudaStream_t st) {
  cascade_pstash_kernel<LOGN><<<depth, Geo<LOGN>::T, 0, st>>>(d, bias, out);
}
static void pstash_for(int logn, const float* d, const float* bias, float4* out, int depth, cudaStream_t st) {
  switch (logn) {
#ifndef ACDC_ONLY_LOGN
    case 8: pstash_launch<8>(d, bias, out, depth, st); break;
    case 9: pstash_launch<9>(d, bias, out, depth, st); break;
    case 10: pstash_launch<10>(d, bias, out, depth, st); break;
    case 11: pstash_launch<11>(d, bias, out, depth, st); break;
    case 12: pstash_launch<12>(d, bias, out, depth, st); break;
    case 13: pstash_launch<13>(d, bias, out, depth, st); break;
    case 14: pstash_launch<14>(d, bias, out, depth, st); break;
#elif ACDC_ONLY_LOGN >= 8 && ACDC_ONLY_LOGN <= 14
    case ACDC_ONLY_LOGN: pstash_launch<ACDC_ONLY_LOGN>(d, bias, out, depth, st); break;
#endif
    default: break;
  }
}

static int cinfo_for(int logn, LaunchInfo* li) {
  switch (logn) {
#ifndef ACDC_ONLY_LOGN
    case 8: *li = cinfo<8>(); return ACDC_OK;
    case 9: *li = cinfo<9>(); return ACDC_OK;
    case 10: *li = cinfo<10>(); return ACDC_OK;
    case 11: *li = cinfo<11>(); return ACDC_OK;
    case 12: *li = cinfo<12>(); return ACDC_OK;
    case 13: *li = cinfo<13>(); return ACDC_OK;
    case 14: *li = cinfo<14>(); return ACDC_OK;
#elif ACDC_ONLY_LOGN >= 8 && ACDC_ONLY_LOGN <= 14
    case ACDC_ONLY_LOGN: *li = cinfo<ACDC_ONLY_LOGN>(); return ACDC_OK;
#endif
    default:
      return set_error(ACDC_E_SIZE, "the fused cascade needs 256 <= n <= 16384");
  }
}

}  // namespace acdc

using namespace acdc;

extern "C" {

size_t cascade_ckpt_bytes(int64_t rows, int32_t n, int32_t depth) {
  if (n < 256 || n > 16384 || (n & (n - 1)) != 0 || rows < 0 || depth < 1) return 0;
  const size_t xck = (size_t)(depth - 1) * (size_t)rows * n;
  const size_t h2 = (size_t)depth * (size_t)((rows + 1) / 2) * 2 * n;
  const size_t pst = (size_t)depth * 2 * n;  // the half-length cascade's parameter re-layout (cascade_fwd_hl_f32)
  return (xck + h2 + pst) * sizeof(float);
}

int cascade_fwd_f32(const float* x, float* y, int32_t depth, int32_t n, const float* a, const float* d,
                    const float* bias, const int32_t* perm, const uint8_t* flags, float* ckpt, int64_t rows,
                    int64_t ldx, int64_t ldy, acdc_stream_t stream) {
  int logn;
  int rc = check_n(n, &logn);
  if (rc) return rc;
  if (cascade_ckpt_bytes(rows > 0 ? rows : 1, n, depth) == 0)
    return set_error(ACDC_E_SIZE, "the fused cascade needs 256 <= n <= 16384 and depth >= 1");
  if (rows == 0) return ACDC_OK;  // empty batch: nothing to read or write
  if (ldx < n || ldy < n) return ACDC_E_SHAPE;
  if (!x || !y || !a || !d || !bias || !ckpt) return ACDC_E_NULL;
  if ((((uintptr_t)x | (uintptr_t)y | (uintptr_t)a) & 7) || (ldx & 1) || (ldy & 1)) return ACDC_E_ALIGN;
  Tables tb;
  if ((rc = get_tables(logn, &tb))) return rc;
  LaunchInfo li;
  if ((rc = cinfo_for(logn, &li))) return rc;
  int64_t grid;
  if ((rc = grid_for(li, (rows + 1) / 2, &grid))) return rc;
  CParams p{};
  p.x = x;
  p.y = y;
  p.a = a;
  p.d = d;
  p.bias = bias;
  p.perm = perm;
  p.flags = flags;
  p.xck = ckpt;
  p.h2c = ckpt + (size_t)(depth - 1) * (size_t)rows * n;
  p.tab = tb.tab;
  // parameter re-layout after the checkpoints (cascade_ckpt_bytes reserves depth x 2n floats: 8 T float4 per block)
  float4* pst = reinterpret_cast<float4*>(p.h2c + (size_t)depth * (size_t)((rows + 1) / 2) * 2 * n);
  pstash_for(logn, d, bias, pst, depth, (cudaStream_t)stream);
  p.pstash = pst;
  p.rows = rows;
  p.ldx = ldx;
  p.ldy = ldy;
  p.depth = depth;
  return launch(li, grid, &p, (cudaStream_t)stream);
}

}  // extern "C"
