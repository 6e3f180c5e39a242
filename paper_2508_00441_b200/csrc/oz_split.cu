// oz_split.cu — K1/K2: error-free splitting of FP64 rows into power-of-two-scaled
// low-precision slices (restates slicing._slice_rows, slicing.py:128-177).
//
// One CTA (or a cluster of CTAs for kb > 16384) owns one row; the row lives in
// registers.  Every iteration of the reference loop (slicing.py:144-176) becomes:
//   * the row max of ceil_log2|x| (fp64emu.max_abs + ceil_log2_abs,
//     fp64emu.py:280-284, 315-319) as one u32 max per element + redux.sync;
//   * sigma = 1.5 * 2^(c+rho-1) assembled as bits (slicing.py:153-160);
//   * v = (x + sigma) - sigma ; x = x - v (slicing.py:162-168) with
//     __dadd_rn/__dsub_rn (HW) or the integer emu_add (EMU);
//   * coeff = v * 2^-c = k * 2^(rho-53) encoded by table lookup on k
//     (slicing.py:168-172; table built with the exact generic encoder).
// One pass writes the slices as they are produced (see split_fused_kernel);
// a count-only mode of the same kernel serves the exact two-pass fallback.
// Output layout: coeff[p][row][ld] (K-major, ld a multiple of 16 bytes),
// expo[p][row] int32.  Columns of B are sliced by transposing B first (K2).
#include "oz_common.cuh"

namespace oz {

constexpr int kHardSlices = 2100;  // slicing.py:38

struct LpFormat {
  int ebits, mbits, bias;
  int max_field;    // largest exponent field holding finite values
  int nan_top;      // 1: the all-ones mantissa in max_field is NaN (E4M3)
  int bytes;
  int shift;        // code position inside its container (FP6 in a byte)
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
  return (sign | code) << f.shift;
}

// ─────────────────────── K1 fused: one pass, table encode ───────────────────────
// The production split:
//   * ONE pass: slices are written as they are produced into a buffer of `cap`
//     planes; the global s is an atomicMax of the row counts, and rows that end
//     early are zero-padded afterwards by pad_planes_kernel (only the missing
//     planes are written).  A row needing more than `cap` planes raises
//     FLAG_PLANE_CAP and the host re-runs the exact two-pass split.
//   * The slice integer comes straight out of the shifted sum: xs = x + sigma
//     stays in sigma's binade (|x| <= 2^c << sigma = 1.5*2^(c+rho-1)) whose ulp is
//     q = 2^(c+rho-53), so bits(xs) = bits(sigma) + k with k*q = RN_q(x), and
//     sigma's low word is 0: k = (int)lo32(xs).  coeff = k*2^(rho-53), so the
//     type2 code is a lookup table over |k| <= 2^(53-rho) built once with the
//     generic encoder (it carries the representability bit, slicing.py:169-172).
//   * The next slice exponent needs only ceil_log2(max|x|) = max over elements
//     of ceil_log2|x|; the 32-bit key (hi32(x) << 1) | (lo32(x) != 0) orders
//     elements by exactly that, so each iteration is one u32 max (redux.sync).
//   * Residuals are multiples of ulp(x_original): when every input of a thread
//     has exponent >= -969 no residual can be subnormal, and the per-element
//     subnormal-residual check (max_abs, fp64emu.py:73-82) is skipped.
//   * kCL > 1: a cluster of kCL CTAs shares one row (kb up to kCL*kThreads*kEPT);
//     the per-iteration max goes through DSMEM and a cluster barrier.
// Each thread owns runs of kV = 16/kEB consecutive elements, so every plane
// store is one 16-byte vector.
constexpr uint32_t FLAG_PLANE_CAP_INTERNAL = 1u << 8;  // host falls back to the two-pass split

struct FusedSplitParams {
  const double* X;
  int64_t rows, kb, ldx;
  int rho;
  int cap;                 // planes allocated in coeff / expo
  uint8_t* coeff;          // [cap][rows][ld]
  int64_t ld;              // elements
  int32_t* expo;           // [cap][rows]
  int32_t* row_cnt;        // [rows]
  int32_t* s_max;          // atomicMax
  uint32_t* flags;
  const uint32_t* table;   // [2K+1] code | (not_representable << 16), index k + K
  int kmax;                // K = 2^(53-rho)
  int pack6;               // FP6: 16 codes -> 12 densely packed bytes (rows of ld*3/4 bytes),
                           // which TMA 16U6_ALIGN16B spreads to 16-byte groups in smem
  int table_clean;         // 1: no entry carries the not-representable bit
  // Fixed-step exponents (opt-in extension, GemmConfig.slice_exponents="fixed"):
  // fixed_w > 0 gives slice p the exponent c_p = c_0 - p * fixed_w (fixed_w = 54 - rho,
  // the step the reference's RN residual bound guarantees) instead of ceil_log2 of the
  // residual's max, so all pairs on an anti-diagonal p + q = l share one scale and
  // can be summed exactly on the tensor cores.  Exponents are written for every
  // allocated plane (padding planes keep the sequence).  max_planes > 0 stops after
  // that many slices (pairs beyond a cutoff are never used).
  int fixed_w;
  int max_planes;
};

// table[k + K] = code of k * 2^(rho-53) (| 1<<16 if not representable).
// Integer only (it also runs for the emulated-FP64 path, whose kernels must
// contain no FP64 instruction): the FP64 bits of k * 2^(rho-53) are assembled
// from the normalised |k| (|k| <= 2^11, so the value is exact and normal).
__global__ void build_code_table_kernel(uint32_t* table, int kmax, int rho, LpFormat f) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > 2 * kmax) return;
  const int k = i - kmax;
  uint32_t fl = 0;
  uint64_t vb = 0;
  if (k != 0) {
    const uint32_t a = (uint32_t)(k < 0 ? -k : k);
    const int pos = 31 - __clz((int)a);  // |k| = 1.f * 2^pos
    vb = ((uint64_t)(k < 0) << 63) | ((uint64_t)(pos + rho - 53 + 1023) << 52) |
         (((uint64_t)a << (52 - pos)) & kFracMask);
  }
  const uint32_t code = encode_coeff(vb, 0, f, fl);
  table[i] = code | (fl ? (1u << 16) : 0u);
}

OZ_DEVICE uint32_t elem_key(uint64_t x) {
  const uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
  return (hi << 1) + min(lo, 1u);  // IMNMX + LEA
}

OZ_DEVICE void st_cluster_u32(uint32_t* local_addr, uint32_t rank, uint32_t v) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(local_addr)), "r"(rank));
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(remote), "r"(v) : "memory");
}

OZ_DEVICE void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

OZ_DEVICE uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// Emulated mode, rows without tiny inputs: the reference's three emulated adds
// (xs = x + sigma, v = xs - sigma, x - v; slicing.py:161-164) have exact results
// that stay normal (see the residual argument above), so they reduce to the
// integer k = RNE(x / q), q = 2^g, and the exact residual x - k*q — computed here
// from x's significand with integer ops only (bit-identical to emu_add's results).
OZ_DEVICE uint64_t emu_slice_elem(uint64_t x, int g, int& k) {
  const int ef = (int)((x >> 52) & 0x7FF);
  if ((x << 1) == 0) {  // +-0: k = 0, residual unchanged
    k = 0;
    return x;
  }
  const uint64_t M = (x & kFracMask) | kHidden;
  const int sh = g - ef + 1075;  // right shift putting the q grid at bit 0
  const bool s = (x >> 63) != 0;
  if (sh <= 0) {                 // x is on the grid: exact cancellation -> +0
    const int k0 = (int)(M << -sh);
    k = s ? -k0 : k0;
    return 0ull;
  }
  if (sh >= 64) {                // |x| < q/2
    k = 0;
    return x;
  }
  const uint64_t k0 = M >> sh;
  const uint64_t rem = M & ((1ull << sh) - 1);
  const uint64_t half = 1ull << (sh - 1);
  const bool up = rem > half || (rem == half && (k0 & 1));  // ties to even
  const int kk = (int)(k0 + (up ? 1 : 0));
  k = s ? -kk : kk;
  const uint64_t rm = up ? (half * 2 - rem) : rem;  // |residual| in units of ulp(x)
  if (rm == 0) return 0ull;
  const uint64_t rs = (uint64_t)(up ? !s : s);
  const int pos = 63 - __clzll((long long)rm);      // <= 52
  return (rs << 63) | ((uint64_t)(ef + pos - 52) << 52) | ((rm << (52 - pos)) & kFracMask);
}

// Fixed-step emulated slicing in fixed point (no renormalisation per plane): an
// element's residual is kept as |r| in units of ulp(x) (53 bits), its sign, and
// sh0 = the right shift that puts plane 0's grid q_0 at bit 0 (clamped to 1023;
// sh0 >= rho - 1 > 0 since |x| <= 2^c0).  Plane p's shift is sh0 + dg with
// dg = g_p - g_0 = -p w.  k = RNE(r / q_p) and the exact residual are the values
// emu_slice_elem produces (the reference's three emulated adds), without the
// FP64 packing: state = rm | sign << 53 | sh0 << 54.
constexpr uint64_t kFxRm = (1ull << 53) - 1;

OZ_DEVICE uint64_t fx_state(uint64_t x, int g0) {
  if ((x << 1) == 0) return 0ull;  // +-0: residual 0 (k = 0 for every plane)
  const int ef = (int)((x >> 52) & 0x7FF);
  const int sh0 = min(g0 - ef + 1075, 1023);
  return ((x & kFracMask) | kHidden) | ((x >> 63) << 53) | ((uint64_t)sh0 << 54);
}

OZ_DEVICE uint64_t fx_slice(uint64_t st, int dg, int& k) {
  // (A branch-free form with one select was measured slower: 2.7 vs 2.0 ms per
  // 8192^2 operand; almost all elements take the general branch.)
  const uint64_t rm = st & kFxRm;
  const uint32_t sgn = (uint32_t)(st >> 53) & 1u;
  const int sh = (int)(st >> 54) + dg;
  uint64_t rm2;
  uint32_t kk, sg2 = sgn;
  if (sh <= 0) {          // the residual lies on the grid: it is the whole slice
    kk = (uint32_t)(rm << min(-sh, 63));
    rm2 = 0;
  } else if (sh >= 54) {  // |r| < q / 2 (rm < 2^53): k = 0
    kk = 0;
    rm2 = rm;
  } else {
    const uint64_t k0 = rm >> sh, rem = rm & ((1ull << sh) - 1), half = 1ull << (sh - 1);
    const bool up = rem > half || (rem == half && (k0 & 1ull));
    kk = (uint32_t)k0 + (up ? 1u : 0u);
    rm2 = up ? 2 * half - rem : rem;
    sg2 = up ? sgn ^ 1u : sgn;
  }
  k = sgn ? -(int)kk : (int)kk;
  return rm2 == 0 ? (st & ~((1ull << 54) - 1)) : (rm2 | ((uint64_t)sg2 << 53) | (st & ~((1ull << 54) - 1)));
}

// Row-max key of a fixed-point residual, ordered like elem_key for what col_c0
// reads (exponent field in bits 21+, non-zero low bits iff |r| is not a power of
// two): |r| = rm * 2^(g0 - sh0) (sh0 unclamped), normal for rows without tiny inputs.
OZ_DEVICE uint32_t fx_key(uint64_t st, int g0) {
  const uint64_t rm = st & kFxRm;
  if (rm == 0) return 0u;
  const int pos = 63 - __clzll((long long)rm);
  const int ef = pos + g0 - (int)(st >> 54) + 1023;
  return ((uint32_t)ef << 21) | ((rm & (rm - 1)) != 0 ? 1u : 0u);
}



// One reference iteration over this thread's elements (slicing.py:162-176):
// returns the next max key.  kWrite: emit the 16-byte plane vectors; kChecked:
// per-element subnormal-residual and representability checks (only needed for
// rows holding inputs below 2^-969, or code tables with unrepresentable entries).
// kKey = false (fixed-step fast path, kWrite only): return the OR of the codes
// instead of the max key (the row max is not needed there).
// kFx (emulated fixed-point paths): x[] holds fx_state() words and g is the
// plane's grid offset dg = g_p - g_0; with kKey the max key is fx_key(., g0).
template <int kThreads, int kEPT, int kEB, bool kEmu, bool kWrite, bool kChecked, bool kKey = true, bool kFx = false>
OZ_DEVICE uint32_t slice_iteration(uint64_t (&x)[kEPT], const uint64_t sigma, const int g, const uint32_t* __restrict__ tblc,
                                   int K, uint8_t* plane, int64_t base, int t, int64_t ld, uint32_t& flags,
                                   uint32_t& bad, const int pack6, const int g0 = 0) {
  constexpr int kV = 16 / kEB;
  constexpr int kChunks = kEPT / kV;
  uint32_t key = 0;
#pragma unroll
  for (int ch = 0; ch < kChunks; ++ch) {
    uint32_t codes[kV];
#pragma unroll
    for (int u = 0; u < kV; ++u) {
      const int i = ch * kV + u;
      uint64_t xn;
      int k;  // slice integer: coeff = k * 2^(rho-53)
      if constexpr (kFx) {
        xn = fx_slice(x[i], g, k);
      } else if constexpr (kEmu && !kChecked) {
        xn = emu_slice_elem(x[i], g, k);
      } else if constexpr (kEmu) {
        const uint64_t xs = emu_add(x[i], sigma, flags);
        const uint64_t v = emu_add(xs, sigma ^ kSign, flags);
        xn = emu_add(x[i], v ^ kSign, flags);
        k = (int)(uint32_t)xs;
      } else {
        const double xsd = __dadd_rn(u2d(x[i]), u2d(sigma));
        k = (int)(uint32_t)d2u(xsd);
        xn = d2u(__dsub_rn(u2d(x[i]), __dsub_rn(xsd, u2d(sigma))));
      }
      x[i] = xn;
      if constexpr (kWrite) {
        if constexpr (kEmu) k = min(max(k, -K), K);  // only reachable after a flagged range error
        const uint32_t ent = tblc[k];
        if constexpr (kChecked) bad |= ent;
        codes[u] = ent;
      }
      if constexpr (kKey && kFx) key = max(key, fx_key(xn, g0));
      else if constexpr (kKey) key = max(key, elem_key(xn));
      else key |= codes[u];
      if constexpr (kChecked) {
        const uint32_t ef = (uint32_t)((xn >> 52) & 0x7FF);
        if (ef == 0 && ((uint32_t)xn | ((uint32_t)(xn >> 32) << 1)) != 0u) flags |= FLAG_SUBNORMAL_RESID;
      }
    }
    if constexpr (kWrite) {
      const int64_t e0 = base + ((int64_t)ch * kThreads + t) * kV;
      if (e0 < ld) {
        uint4 w;
        if (kEB == 1 && pack6) {
          // 16 six-bit codes, little-endian bit order, into 96 bits; last word zero.
          uint32_t q[3] = {0u, 0u, 0u};
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const uint32_t c6 = codes[u & (kV - 1)] & 63u, bit = 6u * (uint32_t)u;
            q[bit >> 5] |= c6 << (bit & 31u);
            if ((bit & 31u) > 26u) q[(bit >> 5) + 1] |= c6 >> (32u - (bit & 31u));
          }
          // Dense: 12 bytes per 16 codes (the global side of TMA 16U6_ALIGN16B).
          uint32_t* dst = reinterpret_cast<uint32_t*>(plane + (e0 / 16) * 12);
          dst[0] = q[0];
          dst[1] = q[1];
          dst[2] = q[2];
          continue;
        } else if constexpr (kEB == 1) {
          w.x = __byte_perm(__byte_perm(codes[0], codes[1], 0x0040), __byte_perm(codes[2], codes[3], 0x0040), 0x5410);
          w.y = __byte_perm(__byte_perm(codes[4], codes[5], 0x0040), __byte_perm(codes[6], codes[7], 0x0040), 0x5410);
          w.z = __byte_perm(__byte_perm(codes[8], codes[9], 0x0040), __byte_perm(codes[10], codes[11], 0x0040), 0x5410);
          w.w = __byte_perm(__byte_perm(codes[12], codes[13], 0x0040), __byte_perm(codes[14], codes[15], 0x0040), 0x5410);
        } else {
          w.x = __byte_perm(codes[0], codes[1], 0x5410);
          w.y = __byte_perm(codes[2], codes[3], 0x5410);
          w.z = __byte_perm(codes[4], codes[5], 0x5410);
          w.w = __byte_perm(codes[6], codes[7], 0x5410);
        }
        *reinterpret_cast<uint4*>(plane + e0 * kEB) = w;
      }
    }
  }
  return key;
}

// Two CTAs per SM when a CTA holds <= 8192 elements (64 registers per thread at 512
// threads; one resident CTA with the full register file measured slower for the
// emulated kernels too: 4.7 vs 3.4 ms adaptive, 2.25 vs 2.03 ms fixed-step per
// 8192^2 operand, profiles/split_emu_r02.txt).
template <int kThreads, int kEPT, int kCL, int kEB, bool kEmu>
__global__ void __launch_bounds__(kThreads, kThreads * kEPT <= 8192 ? 2 : 1) split_fused_kernel(const FusedSplitParams P) {
  constexpr int kV = 16 / kEB;          // elements per 16-byte plane store
  constexpr int kChunks = kEPT / kV;
  constexpr int kWarps = kThreads / 32;
  static_assert(kEPT % kV == 0, "EPT must be a multiple of the store vector");
  __shared__ uint32_t red_w[2][kWarps];
  __shared__ uint32_t red_c[2][kCL];
  extern __shared__ uint32_t tbl[];      // 2K+1 entries

  const uint32_t rank = kCL > 1 ? cluster_ctarank() : 0u;
  const int64_t row = blockIdx.x / kCL;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int64_t base = (int64_t)rank * kThreads * kEPT;  // first element of this CTA's part
  const double* xr = P.X + row * P.ldx;
  const bool aligned = ((reinterpret_cast<uintptr_t>(xr) & 15) == 0);
  const int K = P.kmax;
  for (int i = t; i <= 2 * K; i += kThreads) tbl[i] = __ldg(P.table + i);
  uint32_t flags = 0, bad = 0;

  uint64_t x[kEPT];
  const uint64_t* xw = reinterpret_cast<const uint64_t*>(xr);
#pragma unroll
  for (int c = 0; c < kChunks; ++c) {
    const int64_t e0 = base + ((int64_t)c * kThreads + t) * kV;
    if (aligned && e0 + kV <= P.kb) {
#pragma unroll
      for (int u = 0; u < kV; u += 2) {
        const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(xw + e0 + u);
        x[c * kV + u] = a.x;
        x[c * kV + u + 1] = a.y;
      }
    } else {
#pragma unroll
      for (int u = 0; u < kV; ++u) x[c * kV + u] = (e0 + u < P.kb) ? xw[e0 + u] : 0ull;
    }
  }
  // _validate_input (slicing.py:119-125) + the first max key.
  bool tiny = false;
  uint32_t key = 0;
#pragma unroll
  for (int i = 0; i < kEPT; ++i) {
    const uint32_t ef = (uint32_t)((x[i] >> 52) & 0x7FF);
    if (ef == 2047) flags |= FLAG_NONFINITE_INPUT;
    else if (ef == 0 && (x[i] << 1) != 0) flags |= FLAG_SUBNORMAL_INPUT;
    if (ef < 1023 - 969 && (x[i] << 1) != 0) tiny = true;
  }
  if (flags & FLAG_NONFINITE_INPUT) {
#pragma unroll
    for (int i = 0; i < kEPT; ++i) x[i] = 0;  // keep the loop finite; host raises
  }
#pragma unroll
  for (int i = 0; i < kEPT; ++i) key = max(key, elem_key(x[i]));
  // Checked (slow) iterations only if some input of this CTA is tiny or the
  // table holds unrepresentable codes; the barrier also publishes the table.
  const bool checked = __syncthreads_or(tiny) || !P.table_clean;
  if constexpr (kCL > 1) cluster_barrier();  // peers running before any DSMEM store

  const int64_t row_bytes = P.pack6 ? P.ld * 3 / 4 : P.ld * kEB;  // packed FP6: 6 bits per code
  const int64_t plane_stride = P.rows * row_bytes;
  uint8_t* const row_plane0 = P.coeff + row * row_bytes;
  const uint32_t* tblc = tbl + K;
  const bool write = P.coeff != nullptr;  // count-only mode otherwise (no planes, no exponents)
  // Row max of a u32: warp redux -> smem -> (cluster DSMEM); slot alternates
  // between consecutive calls so one barrier per call suffices.
  auto row_max = [&](uint32_t v, int slot) -> uint32_t {
    uint32_t m = __reduce_max_sync(0xFFFFFFFFu, v);
    if (lane == 0) red_w[slot & 1][wid] = m;
    __syncthreads();
    m = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) m = max(m, red_w[slot & 1][w]);
    if constexpr (kCL > 1) {
      if (t < kCL) st_cluster_u32(&red_c[slot & 1][rank], (uint32_t)t, m);
      cluster_barrier();
      m = 0;
#pragma unroll
      for (int r = 0; r < kCL; ++r) m = max(m, red_c[slot & 1][r]);
    }
    return m;
  };
  int cnt = 0;
  int c_prev = 0;
  if (P.fixed_w > 0 && P.max_planes > 0) {
    // Fixed-step exponents with a plane limit: every exponent follows from the
    // first row max, so the iterations need no row reductions at all.  Each
    // thread slices its elements through L planes; the row count (the
    // reference loop's exit at the first all-zero residual, slicing.py:149-152)
    // is recovered afterwards from the per-thread count of leading non-zero
    // iterations (a zero residual stays zero and slices to code 0, so planes a
    // short row writes past its count are the zero padding it would get anyway).
    const uint32_t m0 = row_max(key, 0);
    if (m0 != 0) {
      const int e = (int)(m0 >> 21) - 1023;
      const int c0 = (m0 & 0x1FFFFFu) != 0 ? e + 1 : e;
      c_prev = c0;
      // L = planes the reference loop may produce before a limit check fires at
      // iteration L (same order as below: plane limit, allocation, sigma range).
      int L = 0;
      const int lim = write ? min(P.max_planes, P.cap) : P.max_planes;
      while (L < lim) {
        const int se = c0 - L * P.fixed_w + P.rho - 1 + 1023;
        if (se < 1 || se > 2046) break;
        ++L;
      }
      // Iterations this thread's elements need: with codes written, a residual
      // entering iteration it is non-zero exactly when a code of an iteration
      // >= it or the final residual is non-zero (count-only mode: the key).
      int z = 0;
      // Emulated mode, rows without tiny inputs: fixed-point residuals (fx_slice).
      const bool fx = kEmu && write && !checked && L * P.fixed_w <= 900;
      if (fx) {
        const int g0 = c0 + P.rho - 53;
#pragma unroll
        for (int i = 0; i < kEPT; ++i) x[i] = fx_state(x[i], g0);
      }
      for (int it = 0; it < L; ++it) {
        const int c = c0 - it * P.fixed_w;
        const uint64_t sigma = ((uint64_t)(c + P.rho - 1 + 1023) << 52) | (1ull << 51);
        uint8_t* plane = row_plane0 + (int64_t)it * plane_stride;
        if (kEmu && fx) {
          const uint32_t cor = slice_iteration<kThreads, kEPT, kEB, kEmu, true, false, false, true>(
              x, sigma, -it * P.fixed_w, tblc, K, plane, base, t, P.ld, flags, bad, P.pack6);
          if (cor & 0xFFFFu) z = it + 1;
          continue;
        }
        if (!write) {
          if (key != 0) z = it + 1;
          key = slice_iteration<kThreads, kEPT, kEB, kEmu, false, true>(x, sigma, c + P.rho - 53, tblc, K, plane, base,
                                                                        t, P.ld, flags, bad, P.pack6);
          continue;
        }
        const uint32_t cor =
            checked ? slice_iteration<kThreads, kEPT, kEB, kEmu, true, true, false>(x, sigma, c + P.rho - 53, tblc, K,
                                                                                   plane, base, t, P.ld, flags, bad,
                                                                                   P.pack6)
                    : slice_iteration<kThreads, kEPT, kEB, kEmu, true, false, false>(x, sigma, c + P.rho - 53, tblc, K,
                                                                                    plane, base, t, P.ld, flags, bad,
                                                                                    P.pack6);
        bad |= cor;
        if (cor & 0xFFFFu) z = it + 1;
      }
      uint32_t rest = 0;
#pragma unroll
      for (int i = 0; i < kEPT; ++i) {
        const uint64_t r = fx ? (x[i] & kFxRm) : x[i];
        rest |= (uint32_t)r | ((uint32_t)(r >> 32) << 1);
      }
      if (rest) z = L + 1;  // still non-zero where a limit check stops the loop
      const int need = (int)row_max((uint32_t)z, 1);
      cnt = min(need, L);
      if (need > L && L < P.max_planes) flags |= (write && L >= P.cap) ? FLAG_PLANE_CAP_INTERNAL : FLAG_SIGMA_RANGE;
      if (write && t == 0 && rank == 0)
        for (int p = 0; p < cnt; ++p) P.expo[(int64_t)p * P.rows + row] = c0 - p * P.fixed_w;
    }
  } else {
  // Emulated mode, rows without tiny inputs: this thread's residuals in fixed point
  // (fx_state / fx_slice, as in the fixed-step path) once c_0 is known — the
  // grid offset of slice p is dg = c_p - c_0 — unless an element is so far below
  // the row max that its shift would exceed fx_state's 10-bit field.
  bool fxa = false;
  int c0 = 0;
  for (int it = 0;; ++it) {
    const uint32_t m = row_max(key, it);
    if (m == 0) break;
    if (it >= kHardSlices) {
      flags |= FLAG_SLICE_CAP;
      break;
    }
    if (P.max_planes > 0 && it >= P.max_planes) break;  // fixed mode: planes past the cutoff are unused
    if (write && it >= P.cap) {
      flags |= FLAG_PLANE_CAP_INTERNAL;
      break;
    }
    // c = ceil(log2 max|x|): exponent field = key >> 21, fraction non-zero = low 21 key bits.
    const int e = (int)(m >> 21) - 1023;
    const int c = (P.fixed_w > 0 && it > 0) ? c_prev - P.fixed_w : ((m & 0x1FFFFFu) != 0 ? e + 1 : e);
    c_prev = c;
    const int sig_exp = c + P.rho - 1 + 1023;
    if (sig_exp < 1 || sig_exp > 2046) {
      flags |= FLAG_SIGMA_RANGE;
      break;
    }
    const uint64_t sigma = ((uint64_t)sig_exp << 52) | (1ull << 51);
    uint8_t* plane = row_plane0 + (int64_t)it * plane_stride;
    if constexpr (kEmu) {
      if (it == 0 && write && !checked) {
        c0 = c;
        const int g0 = c + P.rho - 53;
        fxa = true;
#pragma unroll
        for (int i = 0; i < kEPT; ++i)
          if ((x[i] << 1) != 0 && g0 - (int)((x[i] >> 52) & 0x7FF) + 1075 > 1000) fxa = false;
        if (fxa) {
#pragma unroll
          for (int i = 0; i < kEPT; ++i) x[i] = fx_state(x[i], g0);
        }
      }
      if (fxa) {
        // sh0 is held exactly (<= 1000 < 2^10); dg = c_p - c_0 <= 0 only lowers the
        // shift, and a shift <= 0 means the residual already lies on the grid
        // (k is the residual itself, |k| <= 2^(53-rho) by the choice of c_p).
        key = slice_iteration<kThreads, kEPT, kEB, kEmu, true, false, true, true>(
            x, sigma, c - c0, tblc, K, plane, base, t, P.ld, flags, bad, P.pack6, c0 + P.rho - 53);
        if (write && t == 0 && rank == 0) P.expo[(int64_t)it * P.rows + row] = c;
        ++cnt;
        continue;
      }
    }
    if (!write)
      key = slice_iteration<kThreads, kEPT, kEB, kEmu, false, true>(x, sigma, c + P.rho - 53, tblc, K, plane, base, t, P.ld,
                                                                    flags, bad, P.pack6);
    else if (checked)
      key = slice_iteration<kThreads, kEPT, kEB, kEmu, true, true>(x, sigma, c + P.rho - 53, tblc, K, plane, base, t, P.ld, flags,
                                                                   bad, P.pack6);
    else
      key = slice_iteration<kThreads, kEPT, kEB, kEmu, true, false>(x, sigma, c + P.rho - 53, tblc, K, plane, base, t, P.ld,
                                                                    flags, bad, P.pack6);
    if (write && t == 0 && rank == 0) P.expo[(int64_t)it * P.rows + row] = c;
    ++cnt;
  }
  }
  if (bad & (1u << 16)) flags |= FLAG_NOT_REPRESENTABLE;
  if (t == 0 && rank == 0) {
    P.row_cnt[row] = cnt;
    atomicMax(P.s_max, cnt);
    if (P.fixed_w > 0 && write) {  // the exponent sequence continues through the padding planes
      const int c0 = cnt > 0 ? P.expo[row] : 0;
      for (int p = cnt; p < P.cap; ++p) P.expo[(int64_t)p * P.rows + row] = c0 - p * P.fixed_w;
    }
  }
  flags = __reduce_or_sync(0xFFFFFFFFu, flags);
  if (lane == 0 && flags) atomicOr(P.flags, flags);
}

// ─────────── K1c: fixed-step split of COLUMNS, read in place (no transpose) ───────────
// Opt-in extension (GemmConfig.slice_exponents = "fixed" with a plane limit):
// slices column j of a row-major X[kb][cols] exactly as split_fused_kernel's
// fixed-step fast path slices row j of X^T, writing the same K-major planes
// coeff[p][j][ld] — so B needs no transposed FP64 copy (1 GB of traffic at
// n = 8192).  Three launches: per-column max key (atomics over k tiles), the
// slicing of 256 x 16 tiles staged through XOR-swizzled shared memory (each
// thread owns 16 consecutive k of one column, i.e. one 16-byte plane vector),
// and a per-column finish (counts, exponents, s).
struct ColSplitParams {
  const double* X;
  int64_t kb, cols, ldx;
  int rho, w, max_planes, cap;
  uint8_t* coeff;          // [cap][cols][ld] (nullptr: count only)
  int64_t ld;              // elements per plane row
  int32_t* expo;           // [cap][cols]
  int32_t* col_cnt;        // [cols]
  int32_t* s_max;
  uint32_t* flags;
  const uint32_t* table;   // as FusedSplitParams
  int kmax, pack6, table_clean;
  uint32_t* key;           // [cols] max element key (zeroed by the host)
  uint32_t* need;          // [cols] iterations the column needs (max over tiles; zeroed)
  uint32_t* tiny;          // [cols] 1: holds an input below 2^-969 (checked slicing)
};

constexpr int kColTK = 256, kColTJ = 16;  // tile: 256 k x 16 columns

OZ_DEVICE int col_c0(uint32_t m) {
  const int e = (int)(m >> 21) - 1023;
  return (m & 0x1FFFFFu) != 0 ? e + 1 : e;
}

// Planes column j may produce (same limit order as the row kernel).
OZ_DEVICE int col_limit(const ColSplitParams& P, int c0) {
  const int lim = P.coeff ? min(P.max_planes, P.cap) : P.max_planes;
  int L = 0;
  while (L < lim) {
    const int se = c0 - L * P.w + P.rho - 1 + 1023;
    if (se < 1 || se > 2046) break;
    ++L;
  }
  return L;
}

__global__ void __launch_bounds__(256) col_stats_kernel(const ColSplitParams P) {
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t j = (int64_t)blockIdx.x * kColTJ + tx;
  const int64_t k0 = (int64_t)blockIdx.y * kColTK;
  uint32_t key = 0, flags = 0;
  bool tiny = false;
  if (j < P.cols) {
#pragma unroll 4
    for (int i = ty; i < kColTK; i += 16) {
      const int64_t k = k0 + i;
      if (k >= P.kb) break;
      const uint64_t x = reinterpret_cast<const uint64_t*>(P.X)[k * P.ldx + j];
      const uint32_t ef = (uint32_t)((x >> 52) & 0x7FF);
      if (ef == 2047) {
        flags |= FLAG_NONFINITE_INPUT;  // sliced as zero; the host raises (slicing.py:119-122)
        continue;
      }
      if (ef == 0 && (x << 1) != 0) flags |= FLAG_SUBNORMAL_INPUT;
      if (ef < 1023 - 969 && (x << 1) != 0) tiny = true;
      key = max(key, elem_key(x));
    }
  }
  __shared__ uint32_t sk[16][17], st[16][17];
  sk[ty][tx] = key;
  st[ty][tx] = tiny ? 1u : 0u;
  __syncthreads();
  if (ty == 0 && j < P.cols) {
    uint32_t m = 0, ti = 0;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      m = max(m, sk[r][tx]);
      ti |= st[r][tx];
    }
    if (m) atomicMax(P.key + j, m);
    if (ti) atomicOr(P.tiny + j, 1u);
  }
  flags = __reduce_or_sync(0xFFFFFFFFu, flags);
  if ((threadIdx.x & 31) == 0 && flags) atomicOr(P.flags, flags);
}

// The plane loop of one thread (16 consecutive k of one column): returns the
// iterations its elements need (L + 1 if a residual is still non-zero after L).
// A residual entering iteration `it` is non-zero exactly when some code of an
// iteration >= it or the final residual is non-zero, so the count comes from
// the codes (no per-element zero test).
template <int kEB, bool kEmu, bool kChecked, bool kPack6>
OZ_DEVICE int col_slice_planes(const ColSplitParams& P, uint64_t (&x)[16], int c0, int L, const uint32_t* tblc,
                               int K, uint8_t* dst0, int64_t plane_stride, int nvec, uint32_t& flags) {
  constexpr int kV = 16 / kEB;
  uint32_t bad = 0;
  int z = 0;
  // Emulated mode without tiny inputs: fixed-point residuals (fx_slice).
  const bool fx = kEmu && !kChecked && L * P.w <= 900;
  if (fx) {
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = fx_state(x[u], c0 + P.rho - 53);
  }
  for (int it = 0; it < L; ++it) {
    const int c = c0 - it * P.w;
    const int g = c + P.rho - 53;
    const uint64_t sigma = ((uint64_t)(c + P.rho - 1 + 1023) << 52) | (1ull << 51);
    uint32_t codes[16];
    uint32_t cor = 0;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      uint64_t xn;
      int k;
      if constexpr (kEmu && !kChecked) {
        xn = fx ? fx_slice(x[u], -it * P.w, k) : emu_slice_elem(x[u], g, k);
      } else if constexpr (kEmu) {
        const uint64_t xs = emu_add(x[u], sigma, flags);
        const uint64_t v = emu_add(xs, sigma ^ kSign, flags);
        xn = emu_add(x[u], v ^ kSign, flags);
        k = min(max((int)(uint32_t)xs, -K), K);
      } else {
        const double xsd = __dadd_rn(u2d(x[u]), u2d(sigma));
        k = (int)(uint32_t)d2u(xsd);
        xn = d2u(__dsub_rn(u2d(x[u]), __dsub_rn(xsd, u2d(sigma))));
      }
      x[u] = xn;
      codes[u] = tblc[k];
      cor |= codes[u];
      if constexpr (kChecked) {
        if (((uint32_t)(xn >> 52) & 0x7FFu) == 0u && ((uint32_t)xn | ((uint32_t)(xn >> 32) << 1)) != 0u)
          flags |= FLAG_SUBNORMAL_RESID;
      }
    }
    bad |= cor;
    if (cor & 0xFFFFu) z = it + 1;
    if (dst0) {
      uint8_t* dst = dst0 + (int64_t)it * plane_stride;
      if constexpr (kPack6) {
        uint32_t q[3] = {0u, 0u, 0u};
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const uint32_t c6 = codes[u] & 63u, bit = 6u * (uint32_t)u;
          q[bit >> 5] |= c6 << (bit & 31u);
          if ((bit & 31u) > 26u) q[(bit >> 5) + 1] |= c6 >> (32u - (bit & 31u));
        }
        uint32_t* d = reinterpret_cast<uint32_t*>(dst);
        d[0] = q[0];
        d[1] = q[1];
        d[2] = q[2];
      } else {
#pragma unroll
        for (int h = 0; h < 16 / kV; ++h) {
          uint4 v;
          const uint32_t* cc = codes + h * kV;
          if constexpr (kEB == 1) {
            v.x = __byte_perm(__byte_perm(cc[0], cc[1], 0x0040), __byte_perm(cc[2], cc[3], 0x0040), 0x5410);
            v.y = __byte_perm(__byte_perm(cc[4], cc[5], 0x0040), __byte_perm(cc[6], cc[7], 0x0040), 0x5410);
            v.z = __byte_perm(__byte_perm(cc[8], cc[9], 0x0040), __byte_perm(cc[10], cc[11], 0x0040), 0x5410);
            v.w = __byte_perm(__byte_perm(cc[12], cc[13], 0x0040), __byte_perm(cc[14], cc[15], 0x0040), 0x5410);
          } else {
            v.x = __byte_perm(cc[0], cc[1], 0x5410);
            v.y = __byte_perm(cc[2], cc[3], 0x5410);
            v.z = __byte_perm(cc[4], cc[5], 0x5410);
            v.w = __byte_perm(cc[6], cc[7], 0x5410);
          }
          if (h < nvec) reinterpret_cast<uint4*>(dst)[h] = v;
        }
      }
    }
  }
  uint32_t rest = 0;
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const uint64_t r = fx ? (x[u] & kFxRm) : x[u];
    rest |= (uint32_t)r | ((uint32_t)(r >> 32) << 1);
  }
  if (rest) z = L + 1;  // still non-zero where a limit check stops the loop
  if (bad & (1u << 16)) flags |= FLAG_NOT_REPRESENTABLE;
  return z;
}

template <int kEB, bool kEmu>
__global__ void __launch_bounds__(256, 3) col_slice_kernel(const ColSplitParams P) {  // >= 3 CTAs (24 warps) per SM
  __shared__ uint64_t tile[kColTK * kColTJ];  // element (k, j) at k*16 + (j ^ (k >> 4 & 15))
  extern __shared__ uint32_t tbl[];
  const int t = threadIdx.x;
  const int64_t j0 = (int64_t)blockIdx.x * kColTJ, k0 = (int64_t)blockIdx.y * kColTK;
  const int K = P.kmax;
  for (int i = t; i <= 2 * K; i += 256) tbl[i] = __ldg(P.table + i);
  // Coalesced tile load: a warp reads two 128-byte row segments per step.
  {
    const int tx = t & 15, ty = t >> 4;
    const int64_t j = j0 + tx;
#pragma unroll 4
    for (int i = ty; i < kColTK; i += 16) {
      const int64_t k = k0 + i;
      uint64_t x = (k < P.kb && j < P.cols) ? reinterpret_cast<const uint64_t*>(P.X)[k * P.ldx + j] : 0ull;
      if (((x >> 52) & 0x7FF) == 0x7FF) x = 0;  // non-finite: flagged by col_stats
      tile[i * 16 + (tx ^ ((i >> 4) & 15))] = x;
    }
  }
  __syncthreads();
  const int lane = t & 31, wid = t >> 5;
  const int jl = 2 * wid + (lane >> 4), kseg = lane & 15;
  const int64_t j = j0 + jl;
  if (j >= P.cols) return;
  const uint32_t m0 = __ldg(P.key + j);
  if (m0 == 0) return;  // zero column: count 0, its planes are zero-padded later
  uint64_t x[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) x[u] = tile[(16 * kseg + u) * 16 + (jl ^ kseg)];
  const int c0 = col_c0(m0);
  const int L = col_limit(P, c0);
  const bool checked = __ldg(P.tiny + j) != 0 || !P.table_clean;
  const uint32_t* tblc = tbl + K;
  const int64_t e0 = k0 + 16 * kseg;
  const int64_t row_bytes = P.pack6 ? P.ld * 3 / 4 : P.ld * kEB;
  uint8_t* dst0 = (P.coeff && e0 < P.ld) ? P.coeff + j * row_bytes + (P.pack6 ? e0 / 16 * 12 : e0 * kEB) : nullptr;
  const int64_t nv = (P.ld - e0) * kEB / 16;
  const int nvec = nv < kEB ? (int)nv : kEB;  // 16-byte vectors of this thread inside the plane row
  const int64_t plane_stride = P.cols * row_bytes;
  uint32_t flags = 0;
  int z;
  if (kEB == 1 && P.pack6)
    z = checked ? col_slice_planes<kEB, kEmu, true, true>(P, x, c0, L, tblc, K, dst0, plane_stride, nvec, flags)
                : col_slice_planes<kEB, kEmu, false, true>(P, x, c0, L, tblc, K, dst0, plane_stride, nvec, flags);
  else
    z = checked ? col_slice_planes<kEB, kEmu, true, false>(P, x, c0, L, tblc, K, dst0, plane_stride, nvec, flags)
                : col_slice_planes<kEB, kEmu, false, false>(P, x, c0, L, tblc, K, dst0, plane_stride, nvec, flags);
  if (z) atomicMax(P.need + j, (uint32_t)z);
  if (flags) atomicOr(P.flags, flags);
}

// Per column: count = min(needed iterations, L), limit flags, the exponent
// sequence c0 - p w for every allocated plane, s = max count.
__global__ void col_finish_kernel(const ColSplitParams P) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int cnt = 0;
  if (j < P.cols) {
    const uint32_t m0 = P.key[j];
    const int c0 = m0 ? col_c0(m0) : 0;
    if (m0) {
      const int L = col_limit(P, c0);
      const int need = (int)P.need[j];
      cnt = min(need, L);
      if (need > L && L < P.max_planes)
        atomicOr(P.flags, (P.coeff && L >= P.cap) ? FLAG_PLANE_CAP_INTERNAL : FLAG_SIGMA_RANGE);
    }
    P.col_cnt[j] = cnt;
    if (P.coeff)
      for (int p = 0; p < P.cap; ++p) P.expo[(int64_t)p * P.cols + j] = c0 - p * P.w;
  }
  const int m = __reduce_max_sync(0xFFFFFFFFu, cnt);
  if ((threadIdx.x & 31) == 0 && m) atomicMax(P.s_max, m);
}

// Zero slices for rows exhausted before the global s (slicing.py:149-152):
// planes [row_cnt[row], s) of each row and their exponents.  One warp per row.
__global__ void pad_planes_kernel(uint8_t* __restrict__ coeff, int64_t row_bytes, int64_t rows, int s_arg,
                                  int32_t* __restrict__ expo, const int32_t* __restrict__ row_cnt,
                                  const int32_t* __restrict__ s_dev) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (row >= rows) return;
  const int s = s_dev ? min(*s_dev, s_arg) : s_arg;  // s_arg caps (planes allocated)
  const int lane = threadIdx.x & 31;
  const int cnt = row_cnt[row];
  for (int p = cnt; p < s; ++p) {
    uint4* dst = reinterpret_cast<uint4*>(coeff + ((int64_t)p * rows + row) * row_bytes);
    for (int64_t i = lane; i < row_bytes / 16; i += 32) dst[i] = make_uint4(0u, 0u, 0u, 0u);
    if (lane == 0 && expo) expo[(int64_t)p * rows + row] = 0;  // expo == nullptr: keep (fixed-step mode)
  }
}

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
