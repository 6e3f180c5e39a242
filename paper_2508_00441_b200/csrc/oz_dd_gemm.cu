// oz_dd_gemm.cu — K5: double-double reference GEMM (accuracy harness only).
//
// Stands in for the reference's exact oracle ref_gemm (oracle.py:150-174) at
// sizes where the exact limb product is unusable (n >= 4096): every product is
// split exactly with an FMA (TwoProd) and summed with TwoSum into a
// double-double accumulator, then rounded once to FP64.  Used by bench.py and
// tests to measure max relative error; never on the product path.
#include "oz_common.cuh"

namespace oz {

struct DD {
  double hi, lo;
};

// Explicit _rn intrinsics: no FMA contraction may touch the error-free transforms.
OZ_DEVICE DD dd_add_prod(DD s, double a, double b) {
  const double p = __dmul_rn(a, b);
  const double pe = __fma_rn(a, b, -p);  // exact product error (TwoProd)
  const double t = __dadd_rn(s.hi, p);   // TwoSum(s.hi, p)
  const double bb = __dsub_rn(t, s.hi);
  const double te = __dadd_rn(__dsub_rn(s.hi, __dsub_rn(t, bb)), __dsub_rn(p, bb));
  const double lo = __dadd_rn(__dadd_rn(s.lo, pe), te);
  const double hi = __dadd_rn(t, lo);    // renormalise (FastTwoSum)
  return DD{hi, __dsub_rn(lo, __dsub_rn(hi, t))};
}

// C[rows x n] for A rows r0..r0+rows (row-major A m x k, B k x n).  16x16 threads,
// each computing a 4x4 block; tiles of A/B staged through shared memory.
__global__ void __launch_bounds__(256) dd_gemm_kernel(const double* __restrict__ A, const double* __restrict__ B,
                                                      double* __restrict__ C, int m, int n, int k) {
  __shared__ double As[16][64 + 1];
  __shared__ double Bs[16][64 + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int r0 = blockIdx.y * 64, c0 = blockIdx.x * 64;
  DD acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = DD{0.0, 0.0};
  for (int k0 = 0; k0 < k; k0 += 16) {
    for (int idx = threadIdx.x; idx < 16 * 64; idx += 256) {
      const int kk = idx / 64, rr = idx % 64;
      const int ar = r0 + rr, ak = k0 + kk;
      As[kk][rr] = (ar < m && ak < k) ? A[(int64_t)ar * k + ak] : 0.0;
      const int bc = c0 + rr;
      Bs[kk][rr] = (ak < k && bc < n) ? B[(int64_t)ak * n + bc] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < 16; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = dd_add_prod(acc[i][j], a[i], b[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = r0 + ty * 4 + i, c = c0 + tx * 4 + j;
      if (r < m && c < n) C[(int64_t)r * n + c] = __dadd_rn(acc[i][j].hi, acc[i][j].lo);
    }
}

}  // namespace oz
