// Host runtime shared by the kernel translation units: per-device twiddle
// tables, persistent-grid sizing, error state.  Defined in runtime.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/acdc_b200.h"

namespace acdc {

// Device table for size 2^logn: [pass twiddles W_{Ns R}^{q k} in the
// Plan<LOGN>::tw_off layout | c'_k = s_k e^{-i pi k/2N}/2, k <= N/2].
struct Tables {
  float2* tab = nullptr;
};

// Build (once per device and size) and return the tables.
int get_tables(int logn, Tables* out);
// Half-length plan tables (hl_kernels.cu): [pass twiddles of Plan<logn-1> |
// c'_j, j <= N/2 | W_N^k = e^{-2 pi i k/N}, k <= N/4].
int get_tables_hl(int logn, Tables* out);

// n must be a power of two in [1, 32768]; sets logn.
int check_n(int32_t n, int* logn);

// Record a CUDA error for acdc_strerror / acdc_last_error.
int set_cuda_error(cudaError_t e);
int set_error(int code, const char* msg);

// Launch description of one kernel instantiation.
struct LaunchInfo {
  const void* fn = nullptr;
  int cta = 0;      // threads per CTA
  int gpc = 1;      // row groups per CTA
  int scratch = 0;  // global scratch floats per group
  int smem = 0;     // dynamic shared memory bytes
  int max_per_sm = 0;  // cap on resident CTAs per SM (TMEM columns), 0 = occupancy only
  int red_per_cta = 0;  // gradient partials one CTA writes (0: one per group)
  bool pdl = false;     // programmatic dependent launch: may start while the previous kernel drains
  int unit_rows = 2;    // rows one group handles per iteration (2: a row pair; 1: the half-length plan)
  bool hl = false;      // half-length plan (hl_kernels.cu): its own tables
};

// Persistent grid: min(CTAs needed for `units` row groups, resident CTAs).
// Sets the dynamic-smem attribute on first use.
int grid_for(const LaunchInfo& li, int64_t units, int64_t* grid);
// Preferred shared-memory carveout percent for every kernel (ACDC_CARVEOUT; -1: driver default).
int carveout_pref();

// Half-length plan (hl_kernels.cu): launch description for (logn, kind) if
// that size / kind runs on it; hl_enabled(logn): the size runs on it.
bool hl_launch_info(int logn, int kind, LaunchInfo* li);
bool hl_enabled(int logn);

// Launch li.fn with one KParams-like argument struct.
int launch(const LaunchInfo& li, int64_t grid, void* params, cudaStream_t st);

}  // namespace acdc
