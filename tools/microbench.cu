// microbench.cu — throughput probes for the epilogue's arithmetic options on sm_100a.
// Built by tools/microbench.py into tools/libmicro.so (not part of the product).
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2508_00441_b200/csrc/oz_common.cuh"

// kind 0: DADD chains, 1: emu_add chains, 2: IADD64 chains, 3: FFMA chains.
template <int kKind>
__global__ void __launch_bounds__(256) chains(uint64_t* out, int iters, uint64_t seed) {
  constexpr int kChains = 16;
  uint64_t a[kChains];
  uint32_t flags = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) a[c] = 0x3FF0000000000000ull + (seed ^ (threadIdx.x * 977u + c * 131u)) % 4096;
  const uint64_t t = 0x3E80000000000000ull | (seed & 0xFFFF);  // ~1e-7
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      if constexpr (kKind == 0) a[c] = oz::d2u(__dadd_rn(oz::u2d(a[c]), oz::u2d(t)));
      else if constexpr (kKind == 1) a[c] = oz::emu_add(a[c], t, flags);
      else if constexpr (kKind == 2) a[c] = a[c] + t;
      else a[c] = (uint64_t)__float_as_uint(__fmaf_rn(__uint_as_float((uint32_t)a[c]), 1.0001f, 1e-7f));
    }
  }
  uint64_t r = flags;
#pragma unroll
  for (int c = 0; c < kChains; ++c) r ^= a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

extern "C" float micro_run(int kind, int blocks, int iters) {
  uint64_t* out;
  cudaMalloc(&out, sizeof(uint64_t) * blocks * 256);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto launch = [&]() {
    switch (kind) {
      case 0: chains<0><<<blocks, 256>>>(out, iters, 12345); break;
      case 1: chains<1><<<blocks, 256>>>(out, iters, 12345); break;
      case 2: chains<2><<<blocks, 256>>>(out, iters, 12345); break;
      default: chains<3><<<blocks, 256>>>(out, iters, 12345); break;
    }
  };
  launch();
  cudaEventRecord(e0);
  launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(out);
  return ms;
}
