// oz_common.cuh — sm_100a building blocks shared by the Ozaki-scheme kernels.
//
// Everything here is a thin inline-PTX wrapper: mbarriers, TMA tensor loads,
// tcgen05 (TMEM alloc / MMA / commit / ld) and the FP64 bit helpers that the
// split kernel and the GEMM epilogue share.  No CUTLASS types are used; the
// descriptor bit layouts follow the sm_100 UMMA encodings (smem descriptor:
// start>>4 @[0,14), LBO>>4 @[16,30), SBO>>4 @[32,46), version=1 @[46,48),
// layout @[61,64); instruction descriptor: c_fmt @[4,6), a_fmt @[7,10),
// b_fmt @[10,13), a/b major @15/16, N>>3 @[17,23), M>>4 @[24,29)).
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#define OZ_DEVICE __device__ __forceinline__

namespace oz {

// ───────────────────────────── error flags ─────────────────────────────
// One 32-bit device word per call; kernels OR bits in, the host decodes them
// into the reference's exception classes (see paper_2508_00441_b200/_lib.py).
enum : uint32_t {
  FLAG_NONFINITE_INPUT  = 1u << 0,  // slicing.py:120-121  ValueError
  FLAG_SUBNORMAL_INPUT  = 1u << 1,  // slicing.py:122-125  RangeError
  FLAG_SIGMA_RANGE      = 1u << 2,  // slicing.py:157-158  RangeError
  FLAG_SLICE_CAP        = 1u << 3,  // slice count above the allocated cap
  FLAG_NOT_REPRESENTABLE= 1u << 4,  // slicing.py:169-172  SlicingInfeasible
  FLAG_EMU_RANGE        = 1u << 5,  // fp64emu.py:240-241  RangeError (emulated add result)
  FLAG_TERM_RANGE       = 1u << 6,  // ozgemm.py:137-139   RangeError (scaled term)
  FLAG_SUBNORMAL_RESID  = 1u << 7,  // fp64emu.py:73-82 via max_abs: subnormal residual
};

// ───────────────────────────── smem / barriers ─────────────────────────
OZ_DEVICE uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

OZ_DEVICE void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

OZ_DEVICE void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

OZ_DEVICE void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

OZ_DEVICE void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

OZ_DEVICE void mbar_wait(uint64_t* bar, uint32_t phase) {
  const uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t"
      ".reg .pred P1;\n\t"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n\t"
      "DONE:\n\t"
      "}" ::"r"(addr),
      "r"(phase), "r"(0x989680)
      : "memory");
}

// ───────────────────────────── TMA ─────────────────────────────────────
OZ_DEVICE void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// 3-D tiled load (coordinates innermost first) completing on an mbarrier.
OZ_DEVICE void tma_load_3d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                           uint64_t cache_hint) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "l"(cache_hint)
      : "memory");
}

// L2 cache-policy constants (createpolicy.fractional encodings used by CUTLASS).
constexpr uint64_t kEvictNormal = 0x1000000000000000ull;
constexpr uint64_t kEvictFirst = 0x12F0000000000000ull;
constexpr uint64_t kEvictLast = 0x14F0000000000000ull;

// ───────────────────────────── tcgen05 ─────────────────────────────────
template <uint32_t kCols>
OZ_DEVICE void tmem_alloc(uint32_t* smem_result) {
  static_assert(kCols >= 32 && kCols <= 512 && (kCols & (kCols - 1)) == 0, "TMEM cols: power of 2 in [32,512]");
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_result)),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

template <uint32_t kCols>
OZ_DEVICE void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols) : "memory");
}

OZ_DEVICE void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
OZ_DEVICE void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major, 128-byte-swizzled operand tile: rows of 128 B, 8-row core groups 1024 B apart.
OZ_DEVICE uint64_t smem_desc_sw128(const void* smem_tile) {
  const uint64_t addr = smem_u32(smem_tile);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;          // start address
  d |= (uint64_t)1 << 16;                // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;      // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                // sm100 descriptor version
  d |= (uint64_t)2 << 61;                // SWIZZLE_128B
  return d;
}

// Instruction descriptor (upper 32 bits of the 64-bit idesc operand).
// kind::f8f6f4: fmt E4M3=0 E5M2=1 ; kind::f16: F16=0 BF16=1.  D = F32, both K-major.
__host__ __device__ constexpr uint32_t make_idesc(uint32_t a_fmt, uint32_t b_fmt, uint32_t M, uint32_t N) {
  return (1u << 4) | (a_fmt << 7) | (b_fmt << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

OZ_DEVICE void mma_f8f6f4(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

OZ_DEVICE void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Arrive on an mbarrier once every previously issued tcgen05 op of this thread completes.
OZ_DEVICE void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// 32 lanes x 32 consecutive 32-bit columns: thread t of the warp receives lane (base+t).
OZ_DEVICE void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

OZ_DEVICE void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

OZ_DEVICE void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

OZ_DEVICE uint32_t lane_id() {
  uint32_t l;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(l));
  return l;
}

OZ_DEVICE bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .b32 rx;\n\t.reg .pred px;\n\t"
      "elect.sync rx|px, %1;\n\t"
      "@px mov.s32 %0, 1;\n\t}"
      : "+r"(pred)
      : "r"(0xFFFFFFFFu));
  return pred != 0;
}

// ───────────────────────────── FP64 bit helpers ────────────────────────
constexpr uint64_t kSign = 0x8000000000000000ull;
constexpr uint64_t kExpMask = 0x7FF0000000000000ull;
constexpr uint64_t kFracMask = 0x000FFFFFFFFFFFFFull;
constexpr uint64_t kHidden = 1ull << 52;

OZ_DEVICE uint64_t d2u(double x) { return static_cast<uint64_t>(__double_as_longlong(x)); }
OZ_DEVICE double u2d(uint64_t b) { return __longlong_as_double(static_cast<long long>(b)); }

// Integer-only IEEE binary64 addition, round-to-nearest-even, for normal or zero
// operands.  Restates fp64emu._add_core (fp64emu.py:193-251): magnitude order,
// 10 guard bits with a sticky jam, normalise, RNE on the guard bits, exact
// cancellation -> +0, IEEE zero-sign rules.  A non-zero result outside the
// normal range sets FLAG_EMU_RANGE (the reference raises RangeError).
OZ_DEVICE uint64_t emu_add(uint64_t a, uint64_t b, uint32_t& flags) {
  const uint64_t ma = a & ~kSign, mb = b & ~kSign;
  // Operand check (fp64emu.py:73-82): zero is fine; subnormal / inf / nan are rejected.
  const uint32_t ea_ = (uint32_t)(ma >> 52), eb_ = (uint32_t)(mb >> 52);
  if ((ea_ == 0 && ma != 0) || ea_ == 2047 || (eb_ == 0 && mb != 0) || eb_ == 2047) flags |= FLAG_EMU_RANGE;
  if (ma == 0 || mb == 0) {
    if (ma == 0 && mb == 0) return a & b & kSign;  // -0 only if both -0
    return ma == 0 ? b : a;
  }
  const bool swap = mb > ma;
  const uint64_t big = swap ? b : a, small = swap ? a : b;
  const uint64_t sbig = big >> 63;
  const bool same = (a >> 63) == (b >> 63);
  const int ebig = (int)((big & kExpMask) >> 52), esml = (int)((small & kExpMask) >> 52);
  const uint64_t mbig = ((big & kFracMask) | kHidden) << 10;
  uint64_t msml = ((small & kFracMask) | kHidden) << 10;
  int d = ebig - esml;
  d = d > 63 ? 63 : d;
  {
    const uint64_t lost = (d == 0) ? 0 : (msml & ((1ull << d) - 1));
    msml = (msml >> d) | (lost != 0 ? 1ull : 0ull);
  }
  uint64_t mag = same ? mbig + msml : mbig - msml;
  if (mag == 0) return 0;  // exact cancellation -> +0
  int pos = 63 - __clzll((long long)mag);
  int eadj = 0;
  if (pos == 63) {
    mag = (mag >> 1) | (mag & 1ull);
    eadj = 1;
  } else if (pos < 62) {
    mag <<= (62 - pos);
    eadj = -(62 - pos);
  }
  uint64_t sig = mag >> 10;
  const uint64_t rem = mag & 1023ull;
  const bool up = (rem > 512) || (rem == 512 && (sig & 1ull));
  sig += up ? 1ull : 0ull;
  int carry = 0;
  if (sig == (1ull << 53)) {
    sig >>= 1;
    carry = 1;
  }
  int exp = ebig + eadj + carry;
  if (exp < 1 || exp > 2046) {
    flags |= FLAG_EMU_RANGE;
    exp = exp < 1 ? 1 : 2046;
  }
  return (sbig << 63) | ((uint64_t)exp << 52) | (sig & kFracMask);
}

// IEEE binary64 a + b, round-to-nearest-even, in integer arithmetic, fast path.
//
// Why: on sm_100a the FP64 DADD competes with the FP8 tensor-core MMAs of the
// same SM (measured: the fused pair-GEMM epilogue stalled on the FP64 pipe and
// the MMA warp waited ~27% of its time for TMEM accumulators to be released),
// so the epilogue accumulates with integer ALU ops instead.  Bit-identical to
// __dadd_rn for every input.  The common case — two normal operands whose sum
// rounds to a normal — is straight-line code; zeros, subnormals, Inf/NaN, exact
// cancellation and out-of-range results go to the slow path: emu_add (kEmu: the
// reference's integer emulation, flags on range errors, fp64emu.py:193-251) or
// __dadd_rn (hardware mode: full IEEE semantics, rare).
template <bool kEmu>
__device__ __noinline__ uint64_t slow_add(uint64_t a, uint64_t b, uint32_t* flags) {
  if constexpr (kEmu) return emu_add(a, b, *flags);
  else return d2u(__dadd_rn(u2d(a), u2d(b)));
}

// Branch-free core of fast_add: r = a + b (RNE) unless `slow` is set, in which
// case r is meaningless and the caller must use slow_add.  Zero operands are
// handled here (same results as emu_add, fp64emu.py:247-250).
OZ_DEVICE uint64_t add_nb(uint64_t a, uint64_t b, bool& slow) {
  const uint64_t ua = a & ~kSign, ub = b & ~kSign;
  const bool sw = ub > ua;
  const uint64_t x = sw ? b : a;          // larger magnitude
  const uint64_t ux = sw ? ub : ua, uy = sw ? ua : ub;
  const int ex = (int)(ux >> 52), ey = (int)(uy >> 52);
  const int d = min(ex - ey, 63);         // d > 54 degenerates to a sticky bit: x + y rounds to x
  const uint64_t mx = ((ux & kFracMask) | kHidden) << 10;  // [2^62, 2^63), 10 guard bits
  const uint64_t my0 = ((uy & kFracMask) | kHidden) << 10;
  const uint64_t myd = my0 >> d;
  const uint64_t my = myd | ((myd << d) != my0 ? 1ull : 0ull);  // aligned, sticky in bit 0
  uint64_t m = ((a ^ b) >> 63) == 0 ? mx + my : mx - my;
  const uint32_t c = (uint32_t)(m >> 63);  // carry out of an addition: one right shift, sticky kept
  m = (m >> c) | (m & c);
  const int lz = __clzll((long long)m) - 1;  // cancellation in a subtraction: left shift
  m <<= lz;
  const int e = ex + (int)c - lz;
  const uint64_t sig = m >> 10;  // 53 bits with the hidden bit
  const uint32_t rem = (uint32_t)m & 1023u;
  const uint32_t up = (rem + ((uint32_t)sig & 1u) + 511u) >> 10;  // RNE on 10 guard bits (sticky folded)
  const uint64_t r = (x & kSign) | (((uint64_t)(e - 1) << 52) + sig + up);
  const bool yzero = uy == 0;
  // Slow: Inf/NaN or subnormal operands; a non-zero result whose exponent may
  // leave [1, 2045] (under/overflow).  Exact cancellation gives +0 (RNE).
  slow = ex >= 2047 || (ex == 0 && ux != 0) || (!yzero && (ey == 0 || (m != 0 && (unsigned)(e - 1) >= 2045u)));
  return yzero ? (ux == 0 ? (a & b & kSign) : x) : (m == 0 ? 0ull : r);
}

// add_lean: r = RN(a + b), integer only, for a and b each normal or +-0 (the
// emulated epilogue's Cb + T: Cb is +0 or normal, T normal or a zero product);
// slow = the result may leave the normal range (the caller redoes it with the
// checked emulated add, fp64emu.py:240-241).  ~70 instructions vs ~95 for the
// general add_nb: no Inf/NaN/subnormal operand handling (the callers' exponent
// guards exclude them), one unified normalisation.  Frame: the larger magnitude's significand at bits
// 62..10 (10 guard bits), the smaller aligned with a sticky bit, the sum
// normalised to bit 63 by one left shift (a carry leaves it at 63: shift 0),
// RNE on the 11 bits below the 53-bit significand.
// kSubIn: also send subnormal operands to the slow path (hardware-mode callers,
// where an earlier DADD may have left Cb subnormal).
template <bool kSubIn = false>
OZ_DEVICE uint64_t add_lean(uint64_t a, uint64_t b, bool& slow) {
  const uint32_t ah = (uint32_t)(a >> 32), al = (uint32_t)a, bh = (uint32_t)(b >> 32), bl = (uint32_t)b;
  const uint32_t amh = ah & 0x7FFFFFFFu, bmh = bh & 0x7FFFFFFFu;
  const bool bbig = (bmh > amh) || (bmh == amh && bl > al);
  const uint32_t xh = bbig ? bmh : amh, xl = bbig ? bl : al;
  const uint32_t yh = bbig ? amh : bmh, yl = bbig ? al : bl;
  const uint32_t sgn = (bbig ? bh : ah) & 0x80000000u;
  const bool sub = (int32_t)(ah ^ bh) < 0;
  const int ex = (int)(xh >> 20), ey = (int)(yh >> 20);
  const int d = min(ex - ey, 63);
  // significands << 10 (hidden bit only for a non-zero y)
  const uint32_t mxh = __funnelshift_l(xl, (xh & 0xFFFFFu) | 0x100000u, 10), mxl = xl << 10;
  const uint32_t myh = __funnelshift_l(yl, (yh & 0xFFFFFu) | (ey ? 0x100000u : 0u), 10), myl = yl << 10;
  // y >> d with sticky
  const uint32_t s = (uint32_t)d & 31u;
  const bool big = d >= 32;
  const uint32_t r_lo = __funnelshift_r(myl, myh, s), r_hi = myh >> s;
  const uint32_t lo = big ? r_hi : r_lo, hi = big ? 0u : r_hi;
  const uint32_t lmask = (1u << s) - 1u;
  const uint32_t lost = big ? (myl | (myh & lmask)) : (myl & lmask);
  const uint32_t ylo = lo | (lost != 0u ? 1u : 0u), yhi = hi;
  // x +- y
  const uint64_t mx = ((uint64_t)mxh << 32) | mxl;
  const uint64_t neg = sub ? ~0ull : 0ull;       // x - y = x + ~y + 1
  const uint64_t m = mx + ((((uint64_t)yhi << 32) | ylo) ^ neg) + (uint64_t)sub;
  // normalise to bit 63
  const int lz = __clzll((long long)m);        // 64 for m == 0 (exact cancellation)
  const uint64_t mn = m << (lz & 63);
  const int e = ex + 1 - lz;                    // exponent field of the result
  const uint64_t sig = mn >> 11;                // 53 bits incl. the hidden bit
  const uint32_t rem = (uint32_t)mn & 2047u;
  const uint32_t up = (rem + ((uint32_t)sig & 1u) + 1023u) >> 11;
  const uint64_t r = ((uint64_t)sgn << 32) | ((((uint64_t)(uint32_t)(e - 1)) << 52) + sig + up);
  slow = (unsigned)(e - 1) >= 2045u && m != 0;
  if constexpr (kSubIn) slow |= (ex == 0 && (xh | xl) != 0u) || (ey == 0 && (yh | yl) != 0u);
  return m == 0 ? 0ull : r;
}

template <bool kEmu>
OZ_DEVICE uint64_t fast_add(uint64_t a, uint64_t b, uint32_t& flags) {
  bool slow;
  const uint64_t r = add_nb(a, b, slow);
  return slow ? slow_add<kEmu>(a, b, &flags) : r;
}

// Branchy variant of fast_add (early exits instead of selects).  Measured
// faster than the straight-line form inside the emulated epilogue, where the
// ~60-op integer add is issue-bound and the early exits skip work.
OZ_DEVICE uint64_t fast_add_br(uint64_t a, uint64_t b, uint32_t& flags) {
  const uint64_t ua = a & ~kSign, ub = b & ~kSign;
  const bool sw = ub > ua;
  const uint64_t x = sw ? b : a;
  const uint64_t ux = sw ? ub : ua, uy = sw ? ua : ub;
  const int ex = (int)(ux >> 52), ey = (int)(uy >> 52);
  const int d = ex - ey;
  if (ey == 0 || ex >= 2047) return slow_add<true>(a, b, &flags);
  if (d > 54) return x;  // |y| < ulp(x)/4: x + y rounds to x
  const uint64_t mx = ((ux & kFracMask) | kHidden) << 10;
  const uint64_t my0 = ((uy & kFracMask) | kHidden) << 10;
  const uint64_t my = (my0 >> d) | ((my0 >> d) << d != my0 ? 1ull : 0ull);
  uint64_t m = ((a ^ b) >> 63) == 0 ? mx + my : mx - my;
  int e;
  if (m >> 63) {
    m = (m >> 1) | (m & 1ull);
    e = ex + 1;
  } else {
    if (m == 0) return 0ull;  // exact cancellation -> +0
    const int lz = __clzll((long long)m) - 1;
    m <<= lz;
    e = ex - lz;
  }
  if ((unsigned)(e - 1) >= 2045u) return slow_add<true>(a, b, &flags);
  const uint64_t sig = m >> 10;
  const uint32_t rem = (uint32_t)m & 1023u;
  const uint32_t up = (rem + ((uint32_t)sig & 1u) + 511u) >> 10;
  return (x & kSign) | (((uint64_t)(e - 1) << 52) + sig + up);
}

}  // namespace oz
