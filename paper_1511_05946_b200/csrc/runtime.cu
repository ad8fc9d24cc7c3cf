// Host runtime: twiddle tables, persistent-grid sizing, error state, and the
// size-independent C-ABI entry points (acdc_abi_version, acdc_strerror, ...).
#include "runtime.h"

#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

namespace acdc {

static std::mutex g_mu;
static std::map<std::pair<int, int>, Tables> g_tables;
static std::map<std::pair<int, const void*>, std::pair<int, int>> g_occ;  // (dev, fn) -> (blocks/SM, SMs)
static thread_local char g_errbuf[256];
static thread_local const char* g_last_error = "";

int set_cuda_error(cudaError_t e) {
  snprintf(g_errbuf, sizeof(g_errbuf), "CUDA error: %s", cudaGetErrorString(e));
  g_last_error = g_errbuf;
  return ACDC_E_CUDA;
}

int set_error(int code, const char* msg) {
  snprintf(g_errbuf, sizeof(g_errbuf), "%s", msg);
  g_last_error = g_errbuf;
  return code;
}

int check_n(int32_t n, int* logn) {
  if (n < 1 || (n & (n - 1)) != 0) {
    snprintf(g_errbuf, sizeof(g_errbuf), "fast DCT requires a power-of-two size, got %d", n);
    g_last_error = g_errbuf;
    return ACDC_E_SIZE;
  }
  int l = 0;
  while ((1 << l) < n) ++l;
  if (l > 15) {
    snprintf(g_errbuf, sizeof(g_errbuf), "size %d exceeds the on-chip limit 32768", n);
    g_last_error = g_errbuf;
    return ACDC_E_SIZE;
  }
  *logn = l;
  return ACDC_OK;
}

// exp(-2 pi i m / M) in double, rounded once to fp32
static float2 twiddle(long m, long M) {
  const double pi = 3.14159265358979323846264338327950288;
  m %= M;
  const double th = 2.0 * pi * (double)m / (double)M;
  return make_float2((float)std::cos(th), (float)-std::sin(th));
}

// fft_engine.cuh ACDC_TWGEN: radix-16 passes keep only W^k, W^2k, W^4k, W^8k.
#ifndef ACDC_NO_TWGEN
#define ACDC_TWGEN_HOST 1
#else
#define ACDC_TWGEN_HOST 0
#endif

// Host mirror of Plan<LOGN> (radix 16 x small x 16 ...), fft_engine.cuh.
static void host_plan(int logn, std::vector<int>& radix) {
  radix.clear();
  const int n = 1 << logn;
  if (logn < 4) {
    radix.push_back(n);
    return;
  }
  const int a16 = logn / 4, rem = logn % 4;
  const int np = a16 + (rem ? 1 : 0);
  for (int p = 0; p < np; ++p) radix.push_back((rem && p == 1) ? (1 << rem) : 16);
}

// hl: the half-length tables of a length-2^logn row (hl_kernels.cu): pass
// twiddles of the 2^(logn-1)-point engine, c'_j for j <= N/2, then W_N^k for
// k <= N/4.
static int build_tables(int logn, bool hl, Tables* out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return set_cuda_error(e);
  std::lock_guard<std::mutex> lk(g_mu);
  auto key = std::make_pair(dev, hl ? 100 + logn : logn);
  auto it = g_tables.find(key);
  if (it != g_tables.end()) {
    *out = it->second;
    return ACDC_OK;
  }
  const int n = 1 << logn;
  std::vector<int> radix;
  host_plan(hl ? logn - 1 : logn, radix);
  // per-pass [k][q] twiddle rows, stride Plan::tw_stride(R) (fft_engine.cuh)
  std::vector<float2> h;
  long ns = radix[0];
  for (size_t p = 1; p < radix.size(); ++p) {
    const int r = radix[p];
    if (r == 16 && ACDC_TWGEN_HOST) {  // [k](W^k, W^2k) then [k](W^4k, W^8k)
      for (int half = 0; half < 2; ++half)
        for (long k = 0; k < ns; ++k)
          for (int e = 0; e < 2; ++e) h.push_back(twiddle((long)(1 << (2 * half + e)) * k, ns * r));
      ns *= r;
      continue;
    }
    const int stride = r == 2 ? 1 : r + 2;
    for (long k = 0; k < ns; ++k)
      for (int slot = 0; slot < stride; ++slot)
        h.push_back(slot < r - 1 ? twiddle((long)(slot + 1) * k, ns * r) : make_float2(0.f, 0.f));
    ns *= r;
  }
  const double pi = 3.14159265358979323846264338327950288;
  for (int k = 0; k <= n / 2; ++k) {
    const double s = (k == 0 ? std::sqrt(1.0 / n) : std::sqrt(2.0 / n)) * 0.5;
    const double th = pi * (double)k / (2.0 * n);
    h.push_back(make_float2((float)(s * std::cos(th)), (float)(-s * std::sin(th))));
  }
  if (hl)
    for (int k = 0; k <= n / 4; ++k) h.push_back(twiddle(k, n));
  Tables tb;
  if ((e = cudaMalloc(&tb.tab, sizeof(float2) * h.size())) != cudaSuccess) return set_cuda_error(e);
  if ((e = cudaMemcpy(tb.tab, h.data(), sizeof(float2) * h.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
    return set_cuda_error(e);
  g_tables[key] = tb;
  *out = tb;
  return ACDC_OK;
}

int get_tables(int logn, Tables* out) { return build_tables(logn, false, out); }
int get_tables_hl(int logn, Tables* out) { return build_tables(logn, true, out); }

// Preferred shared-memory carveout for every kernel, in percent (ACDC_CARVEOUT
// overrides; -1: driver default).  50%: kernels that need more still get it
// (N = 4096's 196 KB), the smaller ones keep a large L1 instead of the
// driver's shared-memory-heavy choice.  Measured fwd+bwd at B = 16384
// (profiles/round2/probes/carveout_ab.txt): N = 512 / 1024 / 2048 / 8192
// -6% / -6% / -4% / -4%, N = 4096, C3, C4, C5 unchanged; 0% (smallest) costs
// C4 +4% (the reduction kernels lose occupancy).
int carveout_pref() {
  static const int v = [] {
    const char* e = std::getenv("ACDC_CARVEOUT");
    return e ? std::atoi(e) : 50;
  }();
  return v;
}

int grid_for(const LaunchInfo& li, int64_t units, int64_t* grid) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return set_cuda_error(e);
  std::pair<int, int> occ;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto key = std::make_pair(dev, li.fn);
    auto it = g_occ.find(key);
    if (it == g_occ.end()) {
      if (li.smem > 48 * 1024) {
        e = cudaFuncSetAttribute(li.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, li.smem);
        if (e != cudaSuccess) return set_cuda_error(e);
      }
      if (const int co = carveout_pref(); co >= 0)
        cudaFuncSetAttribute(li.fn, cudaFuncAttributePreferredSharedMemoryCarveout, co);
      int bps = 0, sms = 0;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, li.fn, li.cta, li.smem);
      if (e != cudaSuccess) return set_cuda_error(e);
      e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (e != cudaSuccess) return set_cuda_error(e);
      if (bps < 1) return set_error(ACDC_E_CUDA, "kernel does not fit on an SM (registers / shared memory)");
      if (li.max_per_sm > 0 && bps > li.max_per_sm) bps = li.max_per_sm;
      occ = std::make_pair(bps, sms);
      g_occ[key] = occ;
    } else {
      occ = it->second;
    }
  }
  const int64_t need = (units + li.gpc - 1) / li.gpc;
  const int64_t cap = (int64_t)occ.first * occ.second;
  *grid = need < cap ? need : cap;
  if (*grid < 1) *grid = 1;
  return ACDC_OK;
}

int launch(const LaunchInfo& li, int64_t grid, void* params, cudaStream_t st) {
  void* args[] = {params};
  cudaError_t e;
  if (li.pdl) {  // the kernel waits (griddepcontrol.wait) before reading the previous kernel's results
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr.val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(li.cta);
    cfg.dynamicSmemBytes = li.smem;
    cfg.stream = st;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelExC(&cfg, li.fn, args);
  } else {
    e = cudaLaunchKernel(li.fn, dim3((unsigned)grid), dim3(li.cta), args, li.smem, st);
  }
  if (e != cudaSuccess) return set_cuda_error(e);
  return ACDC_OK;
}

const char* last_error() { return g_last_error; }

}  // namespace acdc

using namespace acdc;

extern "C" {

int acdc_abi_version(void) { return ACDC_ABI_VERSION; }

const char* acdc_strerror(int code) {
  const char* le = last_error();
  switch (code) {
    case ACDC_OK:
      return "ok";
    case ACDC_E_SIZE:
      return le[0] ? le : "unsupported size";
    case ACDC_E_CUDA:
      return le[0] ? le : "CUDA error";
    case ACDC_E_SHAPE:
      return "invalid shape or leading dimension";
    case ACDC_E_ALIGN:
      return "misaligned pointer or leading dimension (n >= 256 needs 8-byte aligned rows)";
    case ACDC_E_WS:
      return "workspace too small";
    case ACDC_E_NULL:
      return "null pointer argument";
    default:
      return "unknown error";
  }
}

const char* acdc_last_error(void) { return last_error(); }

int acdc_max_n(void) { return 32768; }

}  // extern "C"
