// oz_split.cu — K1/K2: error-free splitting of FP64 rows into power-of-two-scaled
// low-precision slices (restates slicing._slice_rows, slicing.py:128-177).
//
// One CTA owns one row of length kb; the row lives in registers (kEPT doubles
// per thread, 256 threads, kb <= 256*kEPT).  Every iteration of the reference
// loop (slicing.py:144-176) becomes:
//   * CTA max of |x| as an integer max over the sign-cleared bit patterns
//     (fp64emu.max_abs, fp64emu.py:315-319) — warp shuffles + one smem hop;
//   * c = ceil(log2 max) from the bit pattern (fp64emu.py:280-284);
//   * sigma = 1.5 * 2^(c+rho-1) assembled as bits (slicing.py:153-160);
//   * v = (x + sigma) - sigma ; x = x - v ; coeff = v * 2^-c (slicing.py:162-168)
//     with __dadd_rn/__dsub_rn (HW) or the integer emu_add (EMU);
//   * coeff encoded straight from its FP64 bit pattern into E4M3/E5M2/FP16/BF16
//     bits (integer only, exact; non-representable sets a flag — slicing.py:169-172).
// The split runs twice: a count pass (per-row slice count, global s via
// atomicMax, validation flags) and a write pass that emits exactly s planes
// (rows exhausted early get zero slices with exponent 0, slicing.py:149-152).
// Output layout: coeff[p][row][ld] (K-major, ld a multiple of 16 bytes),
// expo[p][row] int32.  Columns of B are sliced by transposing B first.
#include "oz_common.cuh"

namespace oz {

constexpr int kSplitThreads = 256;
constexpr int kV = 4;  // consecutive elements per thread chunk
constexpr int kHardSlices = 2100;  // slicing.py:38

struct LpFormat {
  int ebits, mbits, bias;
  int max_field;    // largest exponent field holding finite values
  int nan_top;      // 1: the all-ones mantissa in max_field is NaN (E4M3)
  int bytes;
};

struct SplitParams {
  const double* X;
  int64_t rows, kb, ldx;
  int rho;
  LpFormat fmt;
  int planes;        // write pass: number of planes to emit (= global s)
  uint8_t* coeff;    // [planes][rows][ld]
  int64_t ld;        // elements
  int32_t* expo;     // [planes][rows]
  int32_t* row_cnt;  // [rows]
  int32_t* s_max;    // count pass
  uint32_t* flags;
};

// FP64 bit pattern of a slice value v (a multiple of 2^(c+rho-53), |v| <= 2^c)
// -> low-precision code of coeff = v * 2^-c.  Integer only.
OZ_DEVICE uint32_t encode_coeff(uint64_t vb, int c, const LpFormat& f, uint32_t& flags) {
  if ((vb << 1) == 0) return 0u;
  const uint32_t sign = (uint32_t)(vb >> 63) << (f.ebits + f.mbits);
  const int E = (int)((vb >> 52) & 0x7FF) - 1023 - c;
  const uint64_t sig = (vb & kFracMask) | kHidden;  // 53-bit significand
  int field = E + f.bias;
  int drop = 52 - f.mbits;  // significand bits that must be zero
  uint32_t code;
  if (field >= 1) {
    if ((sig & ((1ull << drop) - 1)) != 0) flags |= FLAG_NOT_REPRESENTABLE;
    const uint32_t mant = (uint32_t)((sig >> drop) & ((1u << f.mbits) - 1));
    if (field > f.max_field || (f.nan_top && field == f.max_field && mant == (1u << f.mbits) - 1))
      flags |= FLAG_NOT_REPRESENTABLE;
    code = ((uint32_t)field << f.mbits) | mant;
  } else {
    drop += 1 - field;  // subnormal of the target format
    if (drop > 63 || (sig & ((1ull << drop) - 1)) != 0) {
      flags |= FLAG_NOT_REPRESENTABLE;
      code = 0;
    } else {
      code = (uint32_t)(sig >> drop);
    }
  }
  return sign | code;
}

OZ_DEVICE uint64_t warp_max_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t w = __shfl_xor_sync(0xFFFFFFFFu, v, o);
    v = w > v ? w : v;
  }
  return v;
}

template <int kEPT, bool kWrite, bool kEmu>
__global__ void __launch_bounds__(kSplitThreads) split_rows_kernel(const SplitParams P) {
  constexpr int kChunks = kEPT / kV;
  __shared__ uint64_t red[2][kSplitThreads / 32];
  const int64_t row = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const double* xr = P.X + row * P.ldx;
  const bool aligned = ((reinterpret_cast<uintptr_t>(xr) & 15) == 0);
  uint32_t flags = 0;

  uint64_t x[kEPT];  // residual as bit patterns
#pragma unroll
  for (int c = 0; c < kChunks; ++c) {
    const int64_t e0 = ((int64_t)c * kSplitThreads + t) * kV;
    // Loaded as raw 64-bit words: no double-typed value in the emulated kernels.
    const uint64_t* xw = reinterpret_cast<const uint64_t*>(xr);
    if (aligned && e0 + kV <= P.kb) {
      const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(xw + e0);
      const ulonglong2 b = *reinterpret_cast<const ulonglong2*>(xw + e0 + 2);
      x[c * kV + 0] = a.x;
      x[c * kV + 1] = a.y;
      x[c * kV + 2] = b.x;
      x[c * kV + 3] = b.y;
    } else {
#pragma unroll
      for (int u = 0; u < kV; ++u) x[c * kV + u] = (e0 + u < P.kb) ? xw[e0 + u] : 0ull;
    }
  }
  // _validate_input (slicing.py:119-125).
#pragma unroll
  for (int i = 0; i < kEPT; ++i) {
    const uint32_t ef = (uint32_t)((x[i] >> 52) & 0x7FF);
    if (ef == 2047) flags |= FLAG_NONFINITE_INPUT;
    else if (ef == 0 && (x[i] << 1) != 0) flags |= FLAG_SUBNORMAL_INPUT;
  }
  if (flags & FLAG_NONFINITE_INPUT) {
#pragma unroll
    for (int i = 0; i < kEPT; ++i) x[i] = 0;  // keep the loop finite; host raises
  }

  const int64_t plane_stride = P.rows * P.ld * P.fmt.bytes;  // bytes
  int cnt = 0;
  for (int it = 0;; ++it) {
    uint64_t m = 0;
#pragma unroll
    for (int i = 0; i < kEPT; ++i) {
      const uint64_t a = x[i] & ~kSign;
      m = a > m ? a : m;
    }
    m = warp_max_u64(m);
    if (lane == 0) red[it & 1][wid] = m;
    __syncthreads();
    m = 0;
#pragma unroll
    for (int w = 0; w < kSplitThreads / 32; ++w) m = red[it & 1][w] > m ? red[it & 1][w] : m;
    if (m == 0) break;
    if (it >= kHardSlices || (kWrite && it >= P.planes)) {
      flags |= FLAG_SLICE_CAP;
      break;
    }
    // c = ceil(log2 max|x|) from the bit pattern.
    const int e = (int)(m >> 52) - 1023;
    const int c = (m & kFracMask) == 0 ? e : e + 1;
    const int sig_exp = c + P.rho - 1 + 1023;
    if (sig_exp < 1 || sig_exp > 2046) {
      flags |= FLAG_SIGMA_RANGE;
      break;
    }
    const uint64_t sigma = ((uint64_t)sig_exp << 52) | (1ull << 51);
    uint32_t codes[kEPT];
#pragma unroll
    for (int i = 0; i < kEPT; ++i) {
      uint64_t v;
      if constexpr (kEmu) {
        v = emu_add(emu_add(x[i], sigma, flags), sigma ^ kSign, flags);
        x[i] = emu_add(x[i], v ^ kSign, flags);
      } else {
        const double xs = __dadd_rn(u2d(x[i]), u2d(sigma));
        v = d2u(__dsub_rn(xs, u2d(sigma)));
        x[i] = d2u(__dsub_rn(u2d(x[i]), u2d(v)));
      }
      const uint32_t ef = (uint32_t)((x[i] >> 52) & 0x7FF);
      if (ef == 0 && (x[i] << 1) != 0) flags |= FLAG_SUBNORMAL_RESID;
      if constexpr (kWrite) codes[i] = encode_coeff(v, c, P.fmt, flags);  // count pass: no codes
      else (void)codes;
    }
    if constexpr (kWrite) {
      uint8_t* plane = P.coeff + (int64_t)it * plane_stride + row * P.ld * P.fmt.bytes;
#pragma unroll
      for (int ch = 0; ch < kChunks; ++ch) {
        const int64_t e0 = ((int64_t)ch * kSplitThreads + t) * kV;
        if (e0 < P.ld) {
          if (P.fmt.bytes == 1) {
            const uint32_t w = codes[ch * kV] | (codes[ch * kV + 1] << 8) | (codes[ch * kV + 2] << 16) |
                               (codes[ch * kV + 3] << 24);
            *reinterpret_cast<uint32_t*>(plane + e0) = w;
          } else {
            uint2 w;
            w.x = codes[ch * kV] | (codes[ch * kV + 1] << 16);
            w.y = codes[ch * kV + 2] | (codes[ch * kV + 3] << 16);
            *reinterpret_cast<uint2*>(plane + e0 * 2) = w;
          }
        }
      }
      if (t == 0) P.expo[(int64_t)it * P.rows + row] = c;
    }
    ++cnt;
  }
  if constexpr (kWrite) {
    // Zero slices for a row exhausted before the global s (slicing.py:149-152).
    for (int p = cnt; p < P.planes; ++p) {
      uint8_t* plane = P.coeff + (int64_t)p * plane_stride + row * P.ld * P.fmt.bytes;
#pragma unroll
      for (int ch = 0; ch < kChunks; ++ch) {
        const int64_t e0 = ((int64_t)ch * kSplitThreads + t) * kV;
        if (e0 < P.ld) {
          if (P.fmt.bytes == 1)
            *reinterpret_cast<uint32_t*>(plane + e0) = 0u;
          else
            *reinterpret_cast<uint2*>(plane + e0 * 2) = make_uint2(0u, 0u);
        }
      }
      if (t == 0) P.expo[(int64_t)p * P.rows + row] = 0;
    }
  }
  if (t == 0) {
    P.row_cnt[row] = cnt;
    if constexpr (!kWrite) atomicMax(P.s_max, cnt);
  }
  // Combine flags across the CTA with one atomic per warp that saw something.
  flags = __reduce_or_sync(0xFFFFFFFFu, flags);
  if (lane == 0 && flags) atomicOr(P.flags, flags);
}

#define OZ_SPLIT_INST(EPT)                                                       \
  template __global__ void split_rows_kernel<EPT, false, false>(const SplitParams); \
  template __global__ void split_rows_kernel<EPT, true, false>(const SplitParams);  \
  template __global__ void split_rows_kernel<EPT, false, true>(const SplitParams);  \
  template __global__ void split_rows_kernel<EPT, true, true>(const SplitParams);
OZ_SPLIT_INST(4)
OZ_SPLIT_INST(8)
OZ_SPLIT_INST(16)
OZ_SPLIT_INST(32)
OZ_SPLIT_INST(64)

// dst[j][i] = src[i][j]  (rows x cols -> cols x rows), 32x32 smem tiles.
__global__ void __launch_bounds__(256) transpose_kernel(const double* __restrict__ src, int64_t rows, int64_t cols,
                                                        int64_t ld_src, double* __restrict__ dst, int64_t ld_dst) {
  __shared__ double tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const int64_t r = r0 + ty + k, c = c0 + tx;
    if (r < rows && c < cols) tile[ty + k][tx] = src[r * ld_src + c];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const int64_t c = c0 + ty + k, r = r0 + tx;
    if (r < rows && c < cols) dst[c * ld_dst + r] = tile[tx][ty + k];
  }
}

// tile_cnt[t] = max(row_cnt[t*128 .. t*128+127]).
__global__ void tile_counts_kernel(const int32_t* __restrict__ row_cnt, int64_t rows, int32_t* __restrict__ tile_cnt) {
  const int64_t r = (int64_t)blockIdx.x * 128 + threadIdx.x;
  int v = r < rows ? row_cnt[r] : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
  __shared__ int w[4];
  if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) tile_cnt[blockIdx.x] = max(max(w[0], w[1]), max(w[2], w[3]));
}

}  // namespace oz
