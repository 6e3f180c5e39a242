// oz_tile_gemm.cu — single-pass tcgen05 tile GEMM  D[m x n] (fp32) = A[m x k] . B[n x k]^T.
//
// Operands are K-major low-precision slice planes (E4M3 / E5M2 bytes, or
// FP16 / BF16 halves), exactly the layout the split kernel emits.  One CTA
// owns a 128 x 128 output tile; one thread drives TMA + tcgen05.mma with a
// two-stage ring, four warps drain TMEM.  This is deliberately the simplest
// correct tcgen05 path: it backs
//   * K4, the accumulator-width probe (north star: "the actual accumulator
//     width of the FP8 MMA is measured on the device"), and
//   * the `lp_gemm` seam of the reference (lpgemm.py:93-120), i.e. one
//     slice-pair product returned to the host.
// The production path is the fused persistent kernel in oz_pair_gemm.cu.
#include "oz_common.cuh"

namespace oz {

constexpr int kTileM = 128;
constexpr int kTileN = 128;
constexpr int kRowBytes = 128;                       // one SW128 row = one k-block
constexpr int kTileBytes = kTileM * kRowBytes;       // 16 KiB per operand tile
constexpr int kTileStages = 2;

struct TileSmem {
  alignas(1024) uint8_t a[kTileStages][kTileBytes];
  alignas(1024) uint8_t b[kTileStages][kTileBytes];
  uint64_t full[kTileStages];
  uint64_t empty[kTileStages];
  uint64_t done;
  uint32_t tmem_base;
};

// elem_bytes = 1 (kind::f8f6f4) or 2 (kind::f16).  fmt = the idesc format code.
__global__ void __launch_bounds__(128, 1)
    tile_gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                     float* __restrict__ D, int64_t ldd, int m, int n, int k, int plane_a, int plane_b,
                     int elem_bytes, uint32_t fmt, int fp6) {
  extern __shared__ uint8_t smem_raw[];
  TileSmem& s = *reinterpret_cast<TileSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x / 32;
  const int m0 = blockIdx.x * kTileM, n0 = blockIdx.y * kTileN;
  const int kb_elems = kRowBytes / elem_bytes;
  const int num_kb = (k + kb_elems - 1) / kb_elems;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    for (int i = 0; i < kTileStages; ++i) {
      mbar_init(&s.full[i], 1);
      mbar_init(&s.empty[i], 1);
    }
    mbar_init(&s.done, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<kTileN>(&s.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s.tmem_base;

  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc(fmt, fmt, kTileM, kTileN);
    for (int kb = 0; kb < num_kb; ++kb) {
      const int st = kb % kTileStages;
      if (kb >= kTileStages) mbar_wait(&s.empty[st], ((kb / kTileStages) - 1) & 1);
      mbar_arrive_expect_tx(&s.full[st], fp6 ? 2 * kTileBytes / 4 * 3 : 2 * kTileBytes);  // FP6: packed bytes
      tma_load_3d(s.a[st], &map_a, &s.full[st], kb * kb_elems, m0, plane_a, kEvictNormal);
      tma_load_3d(s.b[st], &map_b, &s.full[st], kb * kb_elems, n0, plane_b, kEvictNormal);
      mbar_wait(&s.full[st], (kb / kTileStages) & 1);
      tc_fence_after();
      const uint64_t ad = smem_desc_sw128(s.a[st]), bd = smem_desc_sw128(s.b[st]);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {  // 4 x 32 bytes of K per 128-byte row
        const uint64_t off = (uint64_t)((kk * 32) >> 4);
        if (elem_bytes == 1)
          mma_f8f6f4(tmem, ad + off, bd + off, idesc, (kb | kk) != 0);
        else
          mma_f16(tmem, ad + off, bd + off, idesc, (kb | kk) != 0);
      }
      mma_commit(&s.empty[st]);
    }
    mma_commit(&s.done);
  }
  __syncwarp();
  mbar_wait(&s.done, 0);
  tc_fence_after();

  // Epilogue: warp w reads TMEM lanes [32w, 32w+32), 32 columns at a time.
  const int row = m0 + warp * 32 + (int)lane_id();
#pragma unroll 1
  for (int c = 0; c < kTileN; c += 32) {
    uint32_t r[32];
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c, r);
    tmem_ld_wait();
    if (row < m) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int col = n0 + c + j;
        if (col < n) D[(int64_t)row * ldd + col] = __uint_as_float(r[j]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<kTileN>(tmem);
}

size_t tile_gemm_smem_bytes() { return sizeof(TileSmem) + 1024; }

}  // namespace oz
