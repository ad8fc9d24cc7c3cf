// Helpers shared by the layer kernels (ACDC, cascade): L2 prefetch, loads the
// scheduler may not hoist, group bookkeeping, table staging.
#pragma once
#include <cstdint>

#include "dct_pair.cuh"

namespace acdc {

// Bulk prefetch of one row into L2 (TMA engine; no registers, no smem).
__device__ __forceinline__ void prefetch_row_l2(const float* row, int n) {
  uintptr_t a = reinterpret_cast<uintptr_t>(row);
  uintptr_t lo = a & ~uintptr_t(15);
  uintptr_t hi = (a + uintptr_t(n) * 4 + 15) & ~uintptr_t(15);
  for (uintptr_t p = lo; p < hi; p += 32768) {
    uint32_t bytes = (uint32_t)((hi - p) < 32768 ? (hi - p) : 32768);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
  }
}

// Plain (coherent) global load: unlike ld.global.nc it is ordered by the group
// barriers, so ptxas cannot hoist it to the top of the row iteration where it
// would pin a register across every FFT pass.
__device__ __forceinline__ float ld_plain(const float* p) {
  float r;
  asm volatile("ld.global.f32 %0, [%1];" : "=f"(r) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ int ld_plain_i(const int* p) {
  int r;
  asm volatile("ld.global.s32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ float2 ld_plain_f2(const float* p) {
  float2 r;
  asm volatile("ld.global.v2.f32 {%0, %1}, [%2];" : "=f"(r.x), "=f"(r.y) : "l"(p) : "memory");
  return r;
}

// Programmatic dependent launch: let the next kernel in the stream start its
// prologue now / wait here until the previous kernel's results are visible.
// Both are no-ops without a programmatic dependency.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <class G>
struct GroupCtx {
  int grp, t;
  int64_t gid, gstride;
};

template <class G>
__device__ __forceinline__ GroupCtx<G> group_ctx() {
  GroupCtx<G> c;
  c.grp = threadIdx.x / G::T;
  c.t = threadIdx.x % G::T;
  c.gid = (int64_t)blockIdx.x * G::GPC + c.grp;
  c.gstride = (int64_t)gridDim.x * G::GPC;
  return c;
}

// Stage the pass-twiddle / post-twiddle tables in shared memory (whole CTA)
// when the plan has room; return the table pointers the kernel should use.
template <class G>
__device__ __forceinline__ void stage_tables(const float2* tab, float* smem, const float2*& tw, const float2*& cp) {
  constexpr int TOT = G::TW_ENTRIES + G::CP_ENTRIES;
  if constexpr (G::TW_SMEM) {
    float2* st = reinterpret_cast<float2*>(smem);
    for (int i = threadIdx.x; i < TOT; i += blockDim.x) st[i] = tab[i];
    __syncthreads();
    tw = st;
  } else {
    tw = tab;
  }
  cp = tw + G::TW_ENTRIES;
}

// Fast-pairing pass-0 inputs from register pairs: pa[q] / pb[q] are rows A / B
// at (2m, 2m+1), m = jsp + q*S (q < 8); the odd element belongs to the partner.
template <class G>
__device__ __forceinline__ void fp_from_pairs(float2 (&v)[16], const float2 (&pa)[8], const float2 (&pb)[8],
                                              const FastMap<G>& fm) {
  float2 snd[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    v[q] = make_float2(pa[q].x, pb[q].x);
    snd[q] = make_float2(pa[q].y, pb[q].y);
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) v[15 - q] = fm.xor_shfl(snd[q]);
}

}  // namespace acdc
