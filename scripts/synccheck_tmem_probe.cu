// compute-sanitizer synccheck probe: does TMEM allocation alone (tcgen05.alloc
// writing the base address to shared memory) trigger "Barrier error detected.
// Missing init" reports?  Kernels: (a) alloc + dealloc, (b) the same after an
// mbarrier.init, (c) (a) with griddepcontrol.launch_dependents first (as the
// HL forward).  Build: nvcc -gencode arch=compute_100a,code=sm_100a
//   scripts/synccheck_tmem_probe.cu -o sc_probe;  compute-sanitizer --tool synccheck ./sc_probe MODE
#include <cstdint>
#include <cstdio>

#include "../paper_1511_05946_b200/csrc/tmem.cuh"

using namespace acdc;

template <int MODE>
__global__ void k(float* out) {
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  if (MODE == 2) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (MODE == 1 && threadIdx.x == 0)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<32>(&slot);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  float z[8] = {1, 2, 3, 4, 5, 6, 7, 8};
  const uint32_t ta = tmem_addr(slot, warp, 0);
  tmem_st8(ta, z);
  float r[8];
  tmem_ld8(ta, r);
  out[threadIdx.x] = r[threadIdx.x & 7];
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (warp == 0) tmem_dealloc<32>(slot);
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? argv[1][0] - '0' : 0;  // one kernel per process: synccheck kills the context
  float* d;
  cudaMalloc(&d, 128 * sizeof(float));
  if (mode == 0) k<0><<<1, 128>>>(d);
  if (mode == 1) k<1><<<1, 128>>>(d);
  if (mode == 2) k<2><<<1, 128>>>(d);
  printf("mode %d: %s\n", mode, cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
