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

// ───────── tcgen05 MMA throughput vs shape (operands resident in smem, SS mode) ─────────
#include "../paper_2508_00441_b200/csrc/oz_pair_gemm.cu"

template <int kCta, int kN>
__global__ void __launch_bounds__(128, 1) mma_rate(int iters, unsigned long long* cycles) {
  extern __shared__ uint8_t raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* a = base;                       // 128 rows x 128 B
  uint8_t* b = base + 128 * 128;           // kN/kCta rows x 128 B
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < (128 + kN / kCta) * 128 / 4; i += blockDim.x) {
    // random E4M3 slice-like bytes (|v| <= 1, no NaN): sign | exp 1..7 | mantissa
    uint32_t h = (uint32_t)i * 2654435761u ^ (blockIdx.x * 97u);
    uint32_t w = 0;
    for (int b = 0; b < 4; ++b) { h = h * 1664525u + 1013904223u; w |= ((h >> 24) & 0xBFu) << (8 * b); }
    reinterpret_cast<uint32_t*>(base)[i] = w;
  }
  if (threadIdx.x == 0) { oz::mbar_init(&bar[0], 1); oz::mbar_init(&bar[1], 1); oz::fence_barrier_init(); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) oz::tmem_alloc_g<kCta>(&tbase);
  oz::tc_fence_before();
  if constexpr (kCta == 2) oz::cluster_sync(); else __syncthreads();
  oz::tc_fence_after();
  const bool leader = kCta == 1 || oz::cluster_rank() == 0;
  if (warp == 0 && leader && oz::elect_one()) {
    const uint32_t idesc = oz::make_idesc(0, 0, 128 * kCta, kN);
    const uint64_t ad = oz::smem_desc_sw128(a), bd = oz::smem_desc_sw128(b);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        oz::mma_issue<kCta, 1>(tbase, ad + ((kk * 32) >> 4), bd + ((kk * 32) >> 4), idesc, 1u);
      oz::mma_commit_g<kCta>(&bar[it & 1]);
      if (it >= 1) oz::mbar_wait(&bar[(it - 1) & 1], ((it - 1) >> 1) & 1);
    }
    oz::mbar_wait(&bar[(iters - 1) & 1], ((iters - 1) >> 1) & 1);
    cycles[blockIdx.x] = (unsigned long long)(clock64() - t0);
  }
  oz::tc_fence_before();
  if constexpr (kCta == 2) oz::cluster_sync(); else __syncthreads();
  if (warp == 0) oz::tmem_dealloc_g<kCta>(tbase);
}

template <int kCta, int kN>
static double run_mma_rate(int iters) {
  const int grid = 148;
  unsigned long long* cyc;
  cudaMalloc(&cyc, sizeof(unsigned long long) * grid);
  cudaMemset(cyc, 0, sizeof(unsigned long long) * grid);
  const size_t smem = (128 + kN) * 128 + 2048;
  auto k = mma_rate<kCta, kN>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kCta; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr; cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, iters, cyc);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(cyc);
  double mx = 0;
  for (int i = 0; i < grid; ++i) mx = h[i] > mx ? (double)h[i] : mx;
  // MACs per SM per cycle: each leader issues iters*4 MMAs of (128*kCta) x kN x 32 spread over kCta SMs
  return (double)iters * 4 * 128 * kCta * kN * 32 / kCta / mx;
}

extern "C" double micro_mma_rate(int cta, int n, int iters) {
  if (cta == 1 && n == 128) return run_mma_rate<1, 128>(iters);
  if (cta == 1 && n == 256) return run_mma_rate<1, 256>(iters);
  if (cta == 2 && n == 128) return run_mma_rate<2, 128>(iters);
  if (cta == 2 && n == 192) return run_mma_rate<2, 192>(iters);
  if (cta == 2 && n == 256) return run_mma_rate<2, 256>(iters);
  return -1;
}

// ───────── contention probe: MMA issue (warp 0) concurrent with ALU/FP64 side work (warps 4-11) ─────────
// side kind: 0 none, 1 DADD, 2 IADD64, 3 FFMA, 4 integer fast_add, 5 IMAD32
template <int kSide, int kN = 256>
__global__ void __launch_bounds__(384, 1) mma_side(int mma_iters, int side_iters, unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* a = base;
  uint8_t* b = base + 128 * 128;
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < (128 + 256) * 128 / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ (blockIdx.x * 97u);
    uint32_t w = 0;
    for (int q = 0; q < 4; ++q) { h = h * 1664525u + 1013904223u; w |= ((h >> 24) & 0xBFu) << (8 * q); }
    reinterpret_cast<uint32_t*>(base)[i] = w;
  }
  if (threadIdx.x == 0) { oz::mbar_init(&bar[0], 1); oz::mbar_init(&bar[1], 1); oz::fence_barrier_init(); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) oz::tmem_alloc<512>(&tbase);
  oz::tc_fence_before();
  __syncthreads();
  oz::tc_fence_after();
  if (warp == 0) {
    if (oz::elect_one() && mma_iters > 0) {
      const uint32_t idesc = oz::make_idesc(0, 0, 128, kN);
      const uint64_t ad = oz::smem_desc_sw128(a), bd = oz::smem_desc_sw128(b);
      long long t0 = clock64();
      for (int it = 0; it < mma_iters; ++it) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) oz::mma_issue<1, 1>(tbase, ad + ((kk * 32) >> 4), bd + ((kk * 32) >> 4), idesc, 1u);
        oz::mma_commit_g<1>(&bar[it & 1]);
        if (it >= 1) oz::mbar_wait(&bar[(it - 1) & 1], ((it - 1) >> 1) & 1);
      }
      oz::mbar_wait(&bar[(mma_iters - 1) & 1], ((mma_iters - 1) >> 1) & 1);
      out[blockIdx.x * 2] = (unsigned long long)(clock64() - t0);
    }
  } else if (warp >= 4 && kSide != 0) {
    constexpr int kC = 16;
    uint64_t v[kC];
    uint32_t flags = 0;
#pragma unroll
    for (int c = 0; c < kC; ++c) v[c] = 0x3FF0000000000000ull + (threadIdx.x * 977u + c * 131u) % 4096;
    const uint64_t t = 0x3E80000000000000ull | (clock64() & 0xFF);
    long long t0 = clock64();
    for (int i = 0; i < side_iters; ++i) {
#pragma unroll
      for (int c = 0; c < kC; ++c) {
        if constexpr (kSide == 1) v[c] = oz::d2u(__dadd_rn(oz::u2d(v[c]), oz::u2d(t)));
        else if constexpr (kSide == 2) v[c] = v[c] + t;
        else if constexpr (kSide == 3) v[c] = (uint64_t)__float_as_uint(__fmaf_rn(__uint_as_float((uint32_t)v[c]), 1.0001f, 1e-7f));
        else if constexpr (kSide == 4) v[c] = oz::fast_add<false>(v[c], t, flags);
        else v[c] = (uint64_t)((uint32_t)v[c] * 2654435761u + (uint32_t)t);
      }
    }
    uint64_t r = flags;
#pragma unroll
    for (int c = 0; c < kC; ++c) r ^= v[c];
    if (threadIdx.x == 128) out[blockIdx.x * 2 + 1] = (unsigned long long)(clock64() - t0) + (r == 42 ? 1 : 0);
  }
  oz::tc_fence_before();
  __syncthreads();
  if (warp == 0) oz::tmem_dealloc<512>(tbase);
}

template <int kSide, int kN = 256>
static void run_side(int mma_iters, int side_iters, double* mma_cyc, double* side_cyc) {
  const int grid = 148;
  unsigned long long* o;
  cudaMalloc(&o, sizeof(unsigned long long) * grid * 2);
  cudaMemset(o, 0, sizeof(unsigned long long) * grid * 2);
  const size_t smem = (128 + 256) * 128 + 2048;
  cudaFuncSetAttribute(mma_side<kSide, kN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mma_side<kSide, kN><<<grid, 384, smem>>>(mma_iters, side_iters, o);
  cudaDeviceSynchronize();
  unsigned long long h[296];
  cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(o);
  double m = 0, s = 0;
  for (int i = 0; i < grid; ++i) { m += (double)h[2 * i]; s += (double)h[2 * i + 1]; }
  *mma_cyc = m / grid;
  *side_cyc = s / grid;
}

// Returns MMA MAC/clk/SM and side ops/clk/SM (per SM: 8 warps x 32 lanes x 16 chains x iters).
extern "C" void micro_side(int side, int mma_iters, int side_iters, double* mma_rate, double* side_rate) {
  double mc = 0, sc = 0;
  switch (side) {
    case 0: run_side<0>(mma_iters, side_iters, &mc, &sc); break;
    case 1: run_side<1>(mma_iters, side_iters, &mc, &sc); break;
    case 2: run_side<2>(mma_iters, side_iters, &mc, &sc); break;
    case 3: run_side<3>(mma_iters, side_iters, &mc, &sc); break;
    case 4: run_side<4>(mma_iters, side_iters, &mc, &sc); break;
    default: run_side<5>(mma_iters, side_iters, &mc, &sc); break;
  }
  *mma_rate = mc > 0 ? (double)mma_iters * 4 * 128 * 256 * 32 / mc : 0;
  *side_rate = sc > 0 ? 256.0 * 16 * side_iters / sc : 0;
}

// DADD side load against MMAs of width n (128 / 192 / 256; M = 128, cta_group::1).
extern "C" void micro_side_n(int n, int mma_iters, int side_iters, double* mma_rate, double* side_rate) {
  double mc = 0, sc = 0;
  if (n == 128) run_side<1, 128>(mma_iters, side_iters, &mc, &sc);
  else if (n == 192) run_side<1, 192>(mma_iters, side_iters, &mc, &sc);
  else run_side<1, 256>(mma_iters, side_iters, &mc, &sc);
  *mma_rate = mc > 0 ? (double)mma_iters * 4 * 128 * n * 32 / mc : 0;
  *side_rate = sc > 0 ? 256.0 * 16 * side_iters / sc : 0;
}
