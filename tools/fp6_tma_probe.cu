// fp6_tma_probe.cu — what does a TMA load with CU_TENSOR_MAP_DATA_TYPE_16U6_ALIGN16B
// put in shared memory, and how many transaction bytes does it signal?  One CTA,
// one 128 x 8 box, no swizzle; waits with a timeout (no hang).  Diagnostics only.
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

#include "../paper_2508_00441_b200/csrc/oz_common.cuh"

__global__ void probe(const __grid_constant__ CUtensorMap map, uint32_t expect, uint8_t* out, int* status) {
  __shared__ alignas(1024) uint8_t buf[4096];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4096; ++i) buf[i] = 0xEE;
    oz::mbar_init(&bar, 1);
    oz::fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    oz::mbar_arrive_expect_tx(&bar, expect);
    oz::tma_load_3d(buf, &map, &bar, 0, 0, 0, oz::kEvictNormal);
    long long t0 = clock64();
    uint32_t done = 0;
    while (!done && clock64() - t0 < (1ll << 28)) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done) : "r"(oz::smem_u32(&bar)) : "memory");
    }
    *status = done ? 1 : 0;
    for (int i = 0; i < 4096; ++i) out[i] = buf[i];
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)p;
  const int rows = 8, K = 128;
  uint8_t host[rows * K];  // packed: per 16 codes, 12 bytes + 4 zero
  for (int r = 0; r < rows; ++r)
    for (int g = 0; g < K / 16; ++g) {
      unsigned __int128 v = 0;
      for (int j = 0; j < 16; ++j) v |= (unsigned __int128)((r * 16 + g * 3 + j) & 63) << (6 * j);
      for (int b = 0; b < 16; ++b) host[r * K + g * 16 + b] = b < 12 ? (uint8_t)(v >> (8 * b)) : 0;
    }
  uint8_t *dg, *dout;
  int* dst;
  cudaMalloc(&dg, sizeof(host));
  cudaMalloc(&dout, 4096);
  cudaMalloc(&dst, 4);
  cudaMemcpy(dg, host, sizeof(host), cudaMemcpyHostToDevice);
  CUtensorMap map;
  const cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, 1};
  const cuuint64_t strides[2] = {(cuuint64_t)K, (cuuint64_t)K * rows};
  const cuuint32_t box[3] = {128, (cuuint32_t)rows, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  for (int sw = 0; sw < 2; ++sw) {
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_16U6_ALIGN16B, 3, dg, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, sw ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("swizzle %d encode %d\n", sw, (int)r);
    for (uint32_t expect : {128u * rows, 96u * rows, 64u * rows}) {
      probe<<<1, 32>>>(map, expect, dout, dst);
      cudaError_t e = cudaDeviceSynchronize();
      int st = -1;
      uint8_t out[4096];
      cudaMemcpy(&st, dst, 4, cudaMemcpyDeviceToHost);
      cudaMemcpy(out, dout, 4096, cudaMemcpyDeviceToHost);
      printf("  expect %u -> err %d done %d | row0:", expect, (int)e, st);
      for (int i = 0; i < 24; ++i) printf(" %02x", out[i]);
      printf(" | byte 128..136:");
      for (int i = 128; i < 136; ++i) printf(" %02x", out[i]);
      printf("\n");
      if (e != cudaSuccess) return 1;
    }
  }
  return 0;
}
