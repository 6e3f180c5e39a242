// oz_pair_gemm.cu — K3: fused slice-pair GEMM + exact scaling + ordered FP64 accumulation.
//
// Replaces, for one inner-product block, the reference's pair loop
//   ozgemm.py:179-183   pair list sorted by (-(p+q), p, q)  (or (p+q, p, q))
//   ozgemm.py:188-190   G = lp_gemm(A_p, B_q)              (error-free product)
//   ozgemm.py:192-193   T = ldexp(G, cA_p[i] + cB_q[j])     (_scale_terms_exact :132-140)
//   ozgemm.py:194-197   Cb = Cb + T   (hardware FP64 or fp64emu.add_arrays)
//   ozgemm.py:204-207   C  = C + Cb   (ascending blocks)
// G never touches HBM.  Persistent, warp-specialised; the FP64 Cb of a tile stays
// on chip (registers and/or TMEM) for all of its pairs.  Variants:
//   kCta = 1: one CTA per 128 x 128 tile, tcgen05.mma.cta_group::1 (M = 128);
//   kCta = 2: a CTA pair (cluster of 2) per 256 x kN tile, cta_group::2 (M = 256)
//             issued by the leader; each CTA stages its 128 A rows and half of the
//             B tile;
//   kN = 192 (default for large problems): 2 TMEM accumulators, Cb columns
//             [0,128) in registers and [128,192) in TMEM; kN = 128: 4 accumulators,
//             Cb in registers (emulated mode: 2 accumulators, Cb all in TMEM).
// Roles (384 threads; setmaxnreg moves registers to the epilogue):
//   warp 0      TMA producer: A_p / B_q k-blocks (128 B rows, SWIZZLE_128B), paced
//               across CTAs (below);
//   warp 1      TMEM owner + tcgen05.mma issuer (kind::f8f6f4 or kind::f16, FP32
//               accumulate, compile-time kind);
//   warps 4-11  epilogue: tcgen05.ld the FP32 G, build T = G * 2^(eA+eB) as an FP64
//               bit pattern with integer ops (exact), and add it into Cb in the
//               reference pair order, with __dadd_rn (HW mode) or the integer-only
//               add (EMU mode — no DADD/DMUL/DFMA in that instantiation,
//               tests/test_capi.py checks the SASS).
// Producers of all resident CTAs are paced to within `pace_slack` steps (a pair's
// k-blocks in chunks of kPaceBlocks) of each other so concurrently used slice
// panels stay L2-resident.
// Performance note: DADDs only drain while the MMA warp waits for
// an accumulator, so the epilogue work after a pair's first DADD is exposed.
#ifndef OZ_TERM_FMA
#define OZ_TERM_FMA 1  // HW-mode safe terms: DFMA(double(G), 2^(eA+eB), Cb) instead of bit assembly + DADD
#endif
#ifndef OZ_DIAGNOSTICS
#define OZ_DIAGNOSTICS 0  // 1: per-pair clock trace + OZ_DEBUG_MODE hooks (tools/ only; never the product)
#endif
#include <climits>
#include <type_traits>

#include "oz_common.cuh"

namespace oz {

constexpr int kPM = 128;                   // per-CTA output rows
constexpr int kEpiWarps = 8;                // default epilogue warps (two threads per C row)
constexpr int kLeadWarps = 4;               // warpgroup 0 (setmaxnreg is warpgroup-wide): warp 0 TMA, warp 1 MMA
constexpr int kPThreads = 32 * kLeadWarps + 32 * kEpiWarps;
constexpr int kTmemCols = 512;             // whole TMEM: accumulators (+ part of Cb for N > 128)
constexpr int kPaceBlocks = 64;            // k-blocks per cross-CTA pacing step (8192 FP8 / 4096 FP16 K)

// kN = output columns per CTA (and MMA N).  Hardware-FP64 mode: N = 128 keeps Cb
// fully in registers with 4 TMEM accumulators; N = 192 (cta_group::2 only) has 2
// accumulators of 192 columns, Cb columns [0,128) in registers and [128,192) as
// FP64 in TMEM columns [384, 512) — the tensor core runs at 98% of peak vs 87%
// for N = 128 (profiles/microbench_r01.txt) and reads 25% fewer operand bytes per
// flop.  Emulated mode (N = 128): Cb entirely in TMEM (2 accumulators + 256
// columns of FP64), so the ~60-op integer add is instantiated once in a rolled
// chunk loop — fully unrolled over 64 register columns it overflowed the
// instruction cache (ncu: "no instruction" was the top stall).
//   kEpi = 12 (N = 192, hardware mode): three epilogue threads per C row, each
//   with 48 Cb columns in registers and 16 in TMEM (one chunk), so the work
//   left for the per-pair FP64 gap is a third smaller and its dependent TMEM
//   load/store chain one chunk long (512 threads: 128 registers each).
template <int kCta, int kN, bool kEmu, int kEpi = kEpiWarps>
struct PairCfg {
  static constexpr int kThreads = 32 * kLeadWarps + 32 * kEpi;
  static constexpr int kParts = kEpi / 4;                     // epilogue threads per C row
  static constexpr int kBRows = kN / kCta;                    // B rows staged per CTA
  static constexpr int kStageBytes = (kPM + kBRows) * 128;    // per CTA
  static constexpr int kRegCols =
      kEmu ? 0 : (kN == 256 ? 128 : (kEpi == 12 ? kN * 3 / 4 : (kN < 128 ? kN : 128)));  // Cb cols in registers
  static constexpr int kRegHalf = kRegCols / kParts;          // ... per epilogue thread
  static constexpr int kAccBufs = kN == 64 ? 4 : ((kEmu || kN != 128) ? 2 : 4);
  // N = 256 (fixed-step grouped mode, single k-block): both accumulators fill TMEM,
  // so the Cb columns beyond the register part live in C itself (global memory,
  // read-modify-written once per pair group — 16 times per tile at cutoff 11).
  static constexpr int kTmCols = kN == 256 ? 0 : kN - kRegCols;  // C columns whose Cb lives in TMEM
  static constexpr int kGlbCols = kN - kRegCols - kTmCols;    // C columns whose Cb lives in C (N = 256)
  static constexpr int kCbTmem = kAccBufs * kN;               // first TMEM column of that Cb
  static constexpr int kSmemBudget = 227 * 1024 - 2048;
  static constexpr int kStages = kSmemBudget / kStageBytes > 10 ? 10 : kSmemBudget / kStageBytes;
  static_assert(kCbTmem + 2 * kTmCols <= kTmemCols, "TMEM budget");
  static_assert(kN <= 128 || kCta == 2, "N > 128 needs the CTA pair");
  static_assert(kGlbCols == 0 || (kN == 256 && kEpi == 8), "C-resident Cb: N = 256 only");
  static_assert(kRegHalf % 16 == 0 && (kN - kRegCols) % (16 * kParts) == 0, "16-column TMEM chunks per thread");
  static_assert(kEpi == 8 || (kEpi == 12 && !kEmu), "12 epilogue warps: hardware FP64 mode only");
  static constexpr int kRegLo = 40;                           // setmaxnreg: producer / MMA warps
  static constexpr int kRegHi = kEpi == 8 ? 232 : 152;        // setmaxnreg: epilogue warps
  static_assert(kLeadWarps * kRegLo + kEpi * kRegHi <= 2048, "register file");
};

template <int kCta, int kN, bool kEmu>
struct PairSmem {
  using Cfg = PairCfg<kCta, kN, kEmu>;
  alignas(1024) uint8_t a[Cfg::kStages][kPM * 128];
  alignas(1024) uint8_t b[Cfg::kStages][Cfg::kBRows * 128];
  uint64_t full[Cfg::kStages], empty[Cfg::kStages];
  uint64_t acc_full[Cfg::kAccBufs], acc_empty[Cfg::kAccBufs];
  uint32_t tmem_base;
};

struct PairParams {
  const int32_t* expo_a;     // [sx_planes][m]
  const int32_t* expo_b;     // [sy_planes][n]
  const int32_t* ebsh;       // [sy][n_pad] B exponents pre-shifted << 20 (prep_eb_kernel)
  const int32_t* ebmm;       // [sy][tiles_n][2] their min / max over each tile's columns
  int n_pad;                 // tiles_n * kN
  const int32_t* tile_cnt_a; // [m/128] max slice count over the tile's rows (nullable = no skip)
  const int32_t* tile_cnt_b; // [n/128] (128-column groups, whatever kN is)
  double* C;
  int64_t ldc;
  int m, n, kb;
  int sx, sy;                // slice counts after max_slices (caps when s_dev != nullptr)
  const int32_t* s_dev;      // nullable: device {s_A, s_B} of the split (counts = min(caps, these))
  int order;                 // 0 = smallest-first, 1 = largest-first
  int cutoff;                // keep pairs with p+q <= cutoff  (< 0: keep all)
  int accumulate;            // 0: C = Cb (first block), 1: C = C + Cb
  int tiles_m, tiles_n;      // tiles of (128*kCta) x kN
  int elem_bytes;            // 1: kind::f8f6f4, 2: kind::f16
  uint32_t fmt;              // idesc a/b format code
  uint32_t* flags;
  // Cross-CTA pacing (L2 locality): producers of all resident CTAs stay within
  // `pace_slack` steps of each other (a step = kPaceBlocks k-blocks of one pair).
  // step_ctr has waves*pairs_per_tile*ceil(num_kb/kPaceBlocks) zeroed counters;
  // nullptr disables pacing (required when tiles skip pairs).
  uint32_t* step_ctr;
  int pace_slack;
  int pairs_per_tile;
  int group;                 // raster band height in row-tiles
  uint64_t hint_a, hint_b;   // L2 cache policies of the operand loads
  uint32_t* band_done;       // [tiles_m / group] finished-tile counters (nullable)
  int fp6;                   // operands are packed FP6 (TMA 16U6_ALIGN16B)
  // FP32 exponent-field range of a non-zero G: coefficients sit on the grid
  // 2^(rho-53) >= 2^-m2 with |c| <= 1, so 2^(-2 m2) <= |G| <= kb, i.e. the field is in
  // [127 - 2 m2, 127 + ceil(log2 kb)].  The epilogue's fast (unchecked) term path is
  // taken only when every term of a (row, pair) is then provably normal.
  int g_lo, g_hi;
  // Pairs summed in one TMEM accumulator before the epilogue (fixed-step slice
  // exponents only, GemmConfig.slice_exponents="fixed"): consecutive pairs of one
  // anti-diagonal p + q = l share the scale 2^(c0A + c0B - l w), so up to group_max
  // of them accumulate exactly in FP32 (group_max * kb * 2^(2(53-rho)) <= 2^24) and
  // the FP64 epilogue runs once per group.  1 = one pair per epilogue pass (reference).
  int group_max;
  // 1: exclusive epilogue windows — the MMA warp starts a pair only after the
  // epilogue has finished the previous one, so the FP64 adds never run while the
  // tensor pipe streams (where they are held back) and the MMAs never run while
  // the adds do.  0: overlapped (up to kAccBufs accumulators in flight).
  int serial;
  unsigned long long* trace; // diagnostics (OZ_DIAGNOSTICS builds only): per-pair timestamps of unit 0
  int trace_cap;             // entries (pairs) the trace holds
  // Diagnostics only (OZ_DIAGNOSTICS builds, OZ_DEBUG_MODE): bit 0 = epilogue skips the
  // accumulation (MMA-only timing), bit 3 = no C stores.  Results are wrong with either.
  int debug;
};

// Pacing counters order nothing (scheduling only), so relaxed accesses suffice:
// an acquire load costs a CCTL.IVALL (L1 invalidate) per spin and a release
// reduction a MEMBAR.GPU per pair-step (ncu, profiles/pair_gemm_r01_v4).
OZ_DEVICE uint32_t ld_relaxed_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

OZ_DEVICE void red_relaxed_gpu_add(uint32_t* p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ───────────── cluster / 2-CTA primitives ─────────────
OZ_DEVICE uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

OZ_DEVICE void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Arrive on the mbarrier at the same smem offset in CTA `rank` of the cluster.
OZ_DEVICE void mbar_arrive_cluster(uint64_t* bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}

// TMA load into this CTA's smem whose completion bytes land on the LEADER
// CTA's barrier (peer bit cleared), as cta_group::2 MMAs require.
OZ_DEVICE void tma_load_3d_pair(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                uint64_t cache_hint) {
  const uint32_t leader_bar = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1), "r"(c2), "l"(cache_hint)
      : "memory");
}

template <int kCta>
OZ_DEVICE void tmem_alloc_g(uint32_t* dst) {
  if constexpr (kCta == 1) {
    tmem_alloc<kTmemCols>(dst);
  } else {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
}

template <int kCta>
OZ_DEVICE void tmem_dealloc_g(uint32_t taddr) {
  if constexpr (kCta == 1)
    tmem_dealloc<kTmemCols>(taddr);
  else
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kTmemCols)
                 : "memory");
}

// Commit all prior MMAs of this thread to `bar` (both CTAs' copies for kCta = 2).
template <int kCta>
OZ_DEVICE void mma_commit_g(uint64_t* bar) {
  if constexpr (kCta == 1) {
    mma_commit(bar);
  } else {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)0x3)
        : "memory");
  }
}

// One tcgen05.mma; the kind is a template parameter so no predicated-off
// alternative instruction is emitted (those still occupy the tensor issue pipe).
template <int kCta, int kElemBytes>
OZ_DEVICE void mma_issue(uint32_t d_tmem, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  if constexpr (kCta == 1) {
    if constexpr (kElemBytes == 1)
      mma_f8f6f4(d_tmem, ad, bd, idesc, acc);
    else
      mma_f16(d_tmem, ad, bd, idesc, acc);
  } else {
    if constexpr (kElemBytes == 1)
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
          "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
          : "memory");
    else
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
          "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
          : "memory");
  }
}

// Pair enumeration in reference order restricted to p < lp, q < lq, p+q <= cut.
struct PairIter {
  int lp, lq, dmax, d, p, dir;
  OZ_DEVICE void init(int lp_, int lq_, int order, int cutoff) {
    lp = lp_;
    lq = lq_;
    dmax = lp + lq - 2;
    if (cutoff >= 0 && cutoff < dmax) dmax = cutoff;
    dir = order == 0 ? -1 : 1;
    d = order == 0 ? dmax : 0;
    p = 0;
    if (lp <= 0 || lq <= 0) {
      d = -1;
      dir = -1;
      return;
    }
    p = d - (lq - 1) > 0 ? d - (lq - 1) : 0;
  }
  OZ_DEVICE bool valid() const { return d >= 0 && d <= dmax; }
  OZ_DEVICE int q() const { return d - p; }
  OZ_DEVICE void next() {
    const int pend = d < lp - 1 ? d : lp - 1;
    if (p < pend) {
      ++p;
      return;
    }
    d += dir;
    if (valid()) p = d - (lq - 1) > 0 ? d - (lq - 1) : 0;
  }
};

OZ_DEVICE void tile_coords(int tile, int tiles_m, int tiles_n, int G, int& tm, int& tn) {
  // Grouped raster: bands of G row-tiles walk across the column tiles, so the
  // CTAs resident at one time share A and B k-panels in L2.
  const int band = tile / (G * tiles_n);
  const int first_m = band * G;
  const int gm = min(G, tiles_m - first_m);
  const int r = tile - band * G * tiles_n;
  tm = first_m + r % gm;
  tn = r / gm;
}

// T = ldexp(G, e) rebuilt from the FP32 bit pattern of G (a multiple of
// 2^(2(rho-53)) below 2^24, so never FP32-subnormal), branch-free.  Returns +0
// when G is zero or the term is not added: it underflowed to zero the
// reference's way (HW mode: np.ldexp, ozgemm.py:136-139) or left the normal
// range (bad = true; the host raises RangeError, ozgemm.py:137-139, or in
// emulated mode fp64emu scale2's error, fp64emu.py:269-277).  e1 = e + 1023 - 127.
template <bool kEmu>
OZ_DEVICE uint64_t make_term(uint32_t g, int e1, bool& bad) {
  const int ex = (int)((g >> 23) & 0xFFu) + e1;
  const bool nz = (g << 1) != 0u;
  const bool inr = (unsigned)(ex - 1) < 2046u;
  const uint32_t hi = (g & 0x80000000u) | ((uint32_t)ex << 20) | ((g >> 3) & 0xFFFFFu);
  const uint64_t t = ((uint64_t)hi << 32) | (uint64_t)(g << 29);
  // Out of range: overflow always errs; HW mode lets a total underflow round to
  // +-0 (lead exponent ex-1023 <= -1076, or -1075 with a zero fraction).
  const bool to_zero = !kEmu && (ex <= -53 || (ex == -52 && (g & 0x7FFFFFu) == 0u));
  bad |= nz && !inr && !to_zero;
  return (nz && inr) ? t : 0ull;
}

// Pair limits for this CTA's 128-row slab (row128) and the tile's kN columns.
template <int kN>
OZ_DEVICE void tile_limits(const PairParams& P, int sx, int sy, int row128, int tn, int& lp, int& lq) {
  lp = sx;
  lq = sy;
  if (P.tile_cnt_a) {
    lp = row128 * kPM < P.m ? min(lp, __ldg(P.tile_cnt_a + row128)) : 0;
    int cq = 0;
    const int c_lo = tn * kN, c_hi = min(tn * kN + kN, P.n);
    for (int g = c_lo / 128; g * 128 < c_hi; ++g) cq = max(cq, __ldg(P.tile_cnt_b + g));
    lq = min(lq, cq);
  }
}

// Limits of the pair sequence a tile-processing unit walks: for a CTA pair both
// halves walk the same pairs (the wider A limit); a half whose rows have an
// all-zero slice p simply adds nothing for it.
template <int kCta, int kN>
OZ_DEVICE void unit_limits(const PairParams& P, int sx, int sy, int tm, int tn, int& lp_walk, int& lq) {
  tile_limits<kN>(P, sx, sy, tm * kCta, tn, lp_walk, lq);
  if constexpr (kCta == 2) {
    int lp1, lq1;
    tile_limits<kN>(P, sx, sy, tm * kCta + 1, tn, lp1, lq1);
    lp_walk = max(lp_walk, lp1);
  }
}

OZ_DEVICE void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
      "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
      "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

OZ_DEVICE void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// tcgen05.wait::ld that also "defines" the loaded registers, so the compiler
// cannot schedule their uses above the wait.
OZ_DEVICE void tmem_ld_wait_regs(uint32_t (&r)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15])
               :
               : "memory");
}

// Add the terms of 16 consecutive G values (one tcgen05.ld chunk) into 16 Cb
// entries (Cb += T in the reference pair order, ozgemm.py:194-197).  Straight-
// line code so the 16 independent adds overlap: a branch per element would
// serialise them on the add latency, and on sm_100a a DADD waits ~10x longer
// while the tensor cores run (profiles/microbench_r01.txt).  A zero term adds
// +0, which leaves Cb unchanged (Cb is never -0: it starts at +0 and exact
// cancellation gives +0).
//   safe: every term of this (row, pair) and its scale 2^(eA+eB) are known to
//   be normal (per-pair exponent bounds): one DFMA per element (OZ_TERM_FMA;
//   =0 builds the bit-assembled T + DADD form: FP32 bits >> 3 put G's exponent
//   in the FP64 field, + (eA + eB + 896) << 20 rebiases it, the sign is or-ed
//   back, the low word is G << 29).  Otherwise the checked make_term handles
//   range errors.
//   kInt (always in emulated mode; the TMEM-resident part of Cb in hardware
//   mode): integer add_lean (bit-identical RNE), the rare operands it cannot take
//   going to emu_add (emulated) or DADD (hardware).
template <bool kEmu, bool kInt = kEmu>
OZ_DEVICE void accumulate16(const uint32_t (&g)[16], const int32_t* eb_sh, int ea_sh, bool safe, uint64_t* cb,
                            uint32_t& flags) {
  const int4* ebv = reinterpret_cast<const int4*>(eb_sh);
  if constexpr (kInt) {
    // Emulated mode: groups of 8 terms added with the branch-free integer core
    // (independent chains the scheduler can interleave); the rare operands it
    // cannot take (zero/subnormal/Inf, possible under/overflow) go through
    // emu_add after the group.
    bool bad = false;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint64_t t[8];
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int4 e4 = __ldg(ebv + 2 * h + v);
        const int e[4] = {e4.x, e4.y, e4.z, e4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t gv = g[8 * h + 4 * v + u];
          if (safe) {
            const uint32_t hi = (((gv >> 3) & 0x0FFFFFFFu) + (uint32_t)(ea_sh + e[u])) | (gv & 0x80000000u);
            t[4 * v + u] = ((gv << 1) != 0u) ? (((uint64_t)hi << 32) | (uint64_t)(gv << 29)) : 0ull;
          } else {
            t[4 * v + u] = make_term<kEmu>(gv, (ea_sh >> 20) + (e[u] >> 20), bad);
          }
        }
      }
      uint32_t slow = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        // Cb is +0 or normal and every term normal or zero: add_lean's domain
        // (a zero term returns Cb unchanged); a result that may leave the normal
        // range goes to the checked emu_add below.
        bool sl;
        const uint64_t r = add_lean<!kEmu>(cb[8 * h + j], t[j], sl);
        slow |= (uint32_t)sl << j;
        cb[8 * h + j] = sl ? cb[8 * h + j] : r;
      }
      if (slow) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if ((slow >> j) & 1u) cb[8 * h + j] = slow_add<kEmu>(cb[8 * h + j], t[j], &flags);
      }
    }
    if (bad) flags |= FLAG_TERM_RANGE;
    return;
  }
  uint64_t t[16];
  if (safe) {
#if OZ_TERM_FMA
    // Cb = fma(double(G), 2^(eA+eB), Cb): the product is exact (safe: normal
    // term and normal scale), so the one rounding is that of Cb + T.  G = +-0
    // gives a zero product, which leaves Cb (never -0) unchanged.
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int4 e4 = __ldg(ebv + v);
      const int e[4] = {e4.x, e4.y, e4.z, e4.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double gd = (double)__uint_as_float(g[v * 4 + u]);
        const double sc = __hiloint2double(ea_sh + e[u] + (127 << 20), 0);
        cb[v * 4 + u] = d2u(__fma_rn(gd, sc, u2d(cb[v * 4 + u])));
      }
    }
    return;
#else
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int4 e4 = __ldg(ebv + v);
      const int e[4] = {e4.x, e4.y, e4.z, e4.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t gv = g[v * 4 + u];
        const uint32_t hi = (((gv >> 3) & 0x0FFFFFFFu) + (uint32_t)(ea_sh + e[u])) | (gv & 0x80000000u);
        t[v * 4 + u] = ((gv << 1) != 0u) ? (((uint64_t)hi << 32) | (uint64_t)(gv << 29)) : 0ull;
      }
    }
#endif
  } else {
    bool bad = false;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int4 e4 = __ldg(ebv + v);
      const int e[4] = {e4.x, e4.y, e4.z, e4.w};
#pragma unroll
      for (int u = 0; u < 4; ++u)
        t[v * 4 + u] = make_term<kEmu>(g[v * 4 + u], (ea_sh >> 20) + (e[u] >> 20), bad);  // eA + eB + 896
    }
    if (bad) flags |= FLAG_TERM_RANGE;
  }
#pragma unroll
  for (int j = 0; j < 16; ++j) cb[j] = d2u(__dadd_rn(u2d(cb[j]), u2d(t[j])));
}

// Cb[16] = C[row, col0 : col0+16] when `init` (the tile's C-resident Cb columns
// hold its running sum), else +0; columns past n and rows past m read as +0.
OZ_DEVICE void glb_load16(const PairParams& P, int row, int col0, bool init, uint64_t (&c)[16]) {
#pragma unroll
  for (int j = 0; j < 16; ++j) c[j] = 0ull;
  if (!init || row >= P.m) return;
  const uint64_t* crow = reinterpret_cast<const uint64_t*>(P.C) + (int64_t)row * P.ldc + col0;
  if (((reinterpret_cast<uintptr_t>(crow) & 15) == 0) && col0 + 16 <= P.n) {
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
      const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(crow + j);
      c[j] = v.x;
      c[j + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (col0 + j < P.n) c[j] = crow[j];
  }
}

// C[row, col0 : col0+cnt] = Cb (first block) or C + Cb (ozgemm.py:204-207).
template <bool kEmu, typename Acc>
OZ_DEVICE void store_row(const PairParams& P, int row, int col0, const Acc* cb, int cnt, uint32_t& flags) {
  Acc* crow = reinterpret_cast<Acc*>(P.C) + (int64_t)row * P.ldc + col0;
  // 16-byte stores only where this row segment is 16-byte aligned (callers may
  // pass C views at odd column offsets or 8-byte-aligned pointers).
  const bool vec = ((reinterpret_cast<uintptr_t>(crow) & 15) == 0) && (col0 + cnt <= P.n);
  if (vec) {
    using Acc2 = ulonglong2;
#pragma unroll
    for (int j = 0; j < cnt; j += 2) {
      Acc2 v;
      if (P.accumulate) {
        const Acc2 c = *reinterpret_cast<const Acc2*>(crow + j);
        if constexpr (kEmu) {
          v.x = fast_add<true>(c.x, cb[j], flags);
          v.y = fast_add<true>(c.y, cb[j + 1], flags);
        } else {
          v.x = d2u(__dadd_rn(u2d(c.x), u2d(cb[j])));
          v.y = d2u(__dadd_rn(u2d(c.y), u2d(cb[j + 1])));
        }
      } else {
        v.x = cb[j];
        v.y = cb[j + 1];
      }
      *reinterpret_cast<Acc2*>(crow + j) = v;
    }
  } else {
#pragma unroll
    for (int j = 0; j < cnt; ++j) {
      if (col0 + j < P.n) {
        Acc v = cb[j];
        if (P.accumulate) {
          if constexpr (kEmu) v = fast_add<true>(crow[j], cb[j], flags);
          else v = d2u(__dadd_rn(u2d(crow[j]), u2d(cb[j])));
        }
        crow[j] = v;
      }
    }
  }
}

// B exponents for the epilogue, laid out per output tile: ebsh[q][c] = eB_q[c] << 20
// (0 past n) and ebmm[q][tile] = (min, max) of eB_q over the tile's columns.  One
// CTA of kN threads per (tile, q).  Read through L1 by the epilogue, so no smem
// is spent on exponents and any slice count works.
__global__ void prep_eb_kernel(const int32_t* __restrict__ expo_b, int n, int kn, int n_pad, int tiles_n,
                               int32_t* __restrict__ ebsh, int32_t* __restrict__ ebmm, const int32_t* s_dev) {
  const int tile = blockIdx.x, q = blockIdx.y, c = threadIdx.x, gc = tile * kn + c;
  if (s_dev && q >= s_dev[1]) return;  // plane beyond the split's s: never read
  const int e = gc < n ? expo_b[(int64_t)q * n + gc] : 0;
  ebsh[(int64_t)q * n_pad + gc] = e * (1 << 20);
  __shared__ int lo[32], hi[32];
  const int wlo = __reduce_min_sync(0xFFFFFFFFu, gc < n ? e : INT_MAX);
  const int whi = __reduce_max_sync(0xFFFFFFFFu, gc < n ? e : INT_MIN);
  if ((c & 31) == 0) {
    lo[c >> 5] = wlo;
    hi[c >> 5] = whi;
  }
  __syncthreads();
  if (c == 0) {
    int a = INT_MAX, b = INT_MIN;
    for (int w = 0; w < kn / 32; ++w) {
      a = min(a, lo[w]);
      b = max(b, hi[w]);
    }
    ebmm[((int64_t)q * tiles_n + tile) * 2 + 0] = a == INT_MAX ? 0 : a;
    ebmm[((int64_t)q * tiles_n + tile) * 2 + 1] = b == INT_MIN ? 0 : b;
  }
}

template <bool kEmu, int kCta, int kElemBytes, int kN, int kEpi = kEpiWarps>
__global__ void __launch_bounds__(32 * kLeadWarps + 32 * kEpi, 1)
    pair_gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                     const PairParams P) {
  using Cfg = PairCfg<kCta, kN, kEmu, kEpi>;
  constexpr int kStages = Cfg::kStages;
  constexpr int kAccBufs = Cfg::kAccBufs;
  extern __shared__ uint8_t smem_raw[];
  PairSmem<kCta, kN, kEmu>& s =
      *reinterpret_cast<PairSmem<kCta, kN, kEmu>*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x / 32;
  const int lane = (int)lane_id();
  const uint32_t crank = kCta == 2 ? cluster_rank() : 0;  // rank in the CTA pair
  const bool leader = crank == 0;
  const int num_tiles = P.tiles_m * P.tiles_n;
  // Slice counts: host values, or caps on the split's device-side counts (no
  // host round trip between the split and this kernel).
  int sx = P.sx, sy = P.sy, pairs_per_tile = P.pairs_per_tile;
  if (P.s_dev) {
    sx = min(sx, __ldg(P.s_dev));
    sy = min(sy, __ldg(P.s_dev + 1));
    pairs_per_tile = 0;
    for (int p = 0; p < sx; ++p)
      for (int q = 0; q < sy; ++q) pairs_per_tile += (P.cutoff < 0 || p + q <= P.cutoff) ? 1 : 0;
  }
  const int unit = blockIdx.x / kCta, num_units = gridDim.x / kCta;  // tile-processing unit (CTA or pair)
  constexpr int kb_elems = 128 / kElemBytes;
  const int num_kb = (P.kb + kb_elems - 1) / kb_elems;
  const int spp = (num_kb + kPaceBlocks - 1) / kPaceBlocks;  // pacing steps per pair
  const int steps_per_tile = pairs_per_tile * spp;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&s.full[i], 1);
      mbar_init(&s.empty[i], 1);
    }
    for (int i = 0; i < kAccBufs; ++i) {
      mbar_init(&s.acc_full[i], 1);
      mbar_init(&s.acc_empty[i], kEpi * kCta);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_g<kCta>(&s.tmem_base);
  tc_fence_before();
  if constexpr (kCta == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s.tmem_base;

  if (warp < kLeadWarps) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(Cfg::kRegLo));
    if (warp == 0) {
      // ───────── TMA producer (both CTAs of a pair load their own halves) ─────────
      if (elect_one()) {
        uint32_t it = 0;
        bool pacing = true;
        for (int tile = unit; tile < num_tiles; tile += num_units) {
          int tm, tn, lp, lq;
          tile_coords(tile, P.tiles_m, P.tiles_n, P.group, tm, tn);
          unit_limits<kCta, kN>(P, sx, sy, tm, tn, lp, lq);
          const int wave = tile / num_units;
          const int arow = (tm * kCta + (int)crank) * kPM;
          const int brow = tn * kN + (int)crank * Cfg::kBRows;
          PairIter pi;
          int t = 0;
          for (pi.init(lp, lq, P.order, P.cutoff); pi.valid(); pi.next(), ++t) {
            const int p = pi.p, q = pi.q();
            for (int kbi = 0; kbi < num_kb; ++kbi, ++it) {
              // Pacing steps: chunks of kPaceBlocks k-blocks of a pair (one step per pair
              // for kb <= 8192 FP8), so long inner dimensions stay L2-local too.
              const int u = t * spp + kbi / kPaceBlocks;  // this tile's step index
              if (P.step_ctr && pacing && kbi % kPaceBlocks == 0) {
                // Wait until every CTA of the wave `pace_slack` steps back has issued its loads.
                // Scheduling only: if that takes implausibly long (CTAs not co-resident),
                // stop pacing instead of risking a deadlock.
                const int g = wave * steps_per_tile + u - P.pace_slack;
                if (g >= 0) {
                  const int gw = g / steps_per_tile;
                  const uint32_t need = (uint32_t)(kCta * min(num_units, num_tiles - gw * num_units));
                  const long long t0 = clock64();
                  while (ld_relaxed_gpu(P.step_ctr + g) < need) {
                    __nanosleep(32);
                    if (clock64() - t0 > (1ll << 26)) {
                      pacing = false;
                      break;
                    }
                  }
                }
              }
              const uint32_t st = it % kStages;
              if (it >= (uint32_t)kStages) mbar_wait(&s.empty[st], ((it / kStages) - 1) & 1);
              if constexpr (kCta == 1) {
                mbar_arrive_expect_tx(&s.full[st], P.fp6 ? Cfg::kStageBytes / 4 * 3 : Cfg::kStageBytes);
                tma_load_3d(s.a[st], &map_a, &s.full[st], kbi * kb_elems, arow, p, P.hint_a);
                tma_load_3d(s.b[st], &map_b, &s.full[st], kbi * kb_elems, brow, q, P.hint_b);
              } else {
                if (leader)  // FP6: TMA signals the packed global bytes (96 per 128 codes)
                  mbar_arrive_expect_tx(&s.full[st], P.fp6 ? 2 * Cfg::kStageBytes / 4 * 3 : 2 * Cfg::kStageBytes);
                tma_load_3d_pair(s.a[st], &map_a, &s.full[st], kbi * kb_elems, arow, p, P.hint_a);
                tma_load_3d_pair(s.b[st], &map_b, &s.full[st], kbi * kb_elems, brow, q, P.hint_b);
              }
              if (P.step_ctr && (kbi % kPaceBlocks == kPaceBlocks - 1 || kbi == num_kb - 1))
                red_relaxed_gpu_add(P.step_ctr + wave * steps_per_tile + u, 1u);
            }
          }
        }
      }
    } else if (warp == 1 && leader) {
      // ───────── MMA issuer (leader CTA only) ─────────
      const uint32_t idesc = make_idesc(P.fmt, P.fmt, kPM * kCta, kN);
      uint32_t it = 0, acc_it = 0;
      for (int tile = unit; tile < num_tiles; tile += num_units) {
        int tm, tn, lp, lq;
        tile_coords(tile, P.tiles_m, P.tiles_n, P.group, tm, tn);
        unit_limits<kCta, kN>(P, sx, sy, tm, tn, lp, lq);
        PairIter pi;
        pi.init(lp, lq, P.order, P.cutoff);
        for (; pi.valid(); ++acc_it) {
          const uint32_t buf = acc_it % kAccBufs;
          const bool tr = OZ_DIAGNOSTICS && P.trace && unit == 0 && acc_it < (uint32_t)P.trace_cap;
          long long full_wait = 0;
          if (tr && lane == 0) P.trace[acc_it * 8 + 0] = clock64();
          if (acc_it >= (uint32_t)kAccBufs) mbar_wait(&s.acc_empty[buf], ((acc_it / kAccBufs) - 1) & 1);
          if (P.serial && acc_it >= 1 && kAccBufs > 1) {
            const uint32_t prev = (acc_it - 1) % kAccBufs;
            mbar_wait(&s.acc_empty[prev], ((acc_it - 1) / kAccBufs) & 1);
          }
          if (tr && lane == 0) P.trace[acc_it * 8 + 1] = clock64();
          tc_fence_after();
          const uint32_t d_tmem = tmem + buf * kN;
          // One accumulator per group of pairs (one pair unless group_max > 1).
          const int lvl = pi.d;
          int gcnt = 0;
          do {
            for (int kbi = 0; kbi < num_kb; ++kbi, ++it) {
              const uint32_t st = it % kStages;
              const long long tw0 = tr ? clock64() : 0;
              mbar_wait(&s.full[st], (it / kStages) & 1);
              if (tr) full_wait += clock64() - tw0;
              tc_fence_after();
              if (elect_one()) {
                const uint64_t ad = smem_desc_sw128(s.a[st]), bd = smem_desc_sw128(s.b[st]);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                  const uint64_t off = (uint64_t)((kk * 32) >> 4);
                  mma_issue<kCta, kElemBytes>(d_tmem, ad + off, bd + off, idesc, (gcnt | kbi | kk) != 0);
                }
                mma_commit_g<kCta>(&s.empty[st]);
              }
              __syncwarp();
            }
            ++gcnt;
            pi.next();
          } while (pi.valid() && pi.d == lvl && gcnt < P.group_max);
          if (elect_one()) mma_commit_g<kCta>(&s.acc_full[buf]);
          if (tr && lane == 0) {
            P.trace[acc_it * 8 + 2] = clock64();
            P.trace[acc_it * 8 + 6] = (unsigned long long)full_wait;
          }
          __syncwarp();
        }
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(Cfg::kRegHi));
    // ───────── epilogue: ordered FP64 accumulation ─────────
    constexpr int kRegCols = Cfg::kRegCols;
    constexpr int kTmHalf = Cfg::kTmCols / Cfg::kParts;  // TMEM-resident Cb columns per thread
    constexpr int kGlbHalf = Cfg::kGlbCols / Cfg::kParts;  // C-resident Cb columns per thread (N = 256)
    // Integer adds (add_lean; bit-identical to the DADD/DFMA path): everything in
    // emulated mode; in hardware mode the C-resident half of Cb of the 256-column
    // grouped kernel, issued before the register half's DFMAs (integer work is not
    // held back by the MMAs).  Measured and dropped (profiles/): integer adds for
    // hardware mode's TMEM third (hw_int_tmem_ab_r02.txt), for the register half
    // and all of Cb in C at N = 256 (wide_tiles_ab_r02.txt).
    constexpr bool kTmInt = kEmu;
    constexpr bool kGlbInt = true;
    constexpr bool kRegInt = kEmu;
    const int quad = warp & 3;               // TMEM lane quadrant this warp may access
    constexpr int kRegHalf = Cfg::kRegHalf;
    const int half = (warp - kLeadWarps) >> 2;        // part: register Cb cols [kRegHalf h, +kRegHalf); TMEM Cb: [kRegCols + kTmHalf*h, +kTmHalf)
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    const uint32_t cb_tmem = tmem + lane_base + Cfg::kCbTmem + half * 2 * kTmHalf;  // 2 words per FP64
    uint32_t flags = 0;
    uint32_t acc_it = 0;
    for (int tile = unit; tile < num_tiles; tile += num_units) {
      int tm, tn, lp, lq;
      tile_coords(tile, P.tiles_m, P.tiles_n, P.group, tm, tn);
      const int row128 = tm * kCta + (int)crank;
      tile_limits<kN>(P, sx, sy, row128, tn, lp, lq);
      int lp_walk;  // pairs the MMA issuer walks (unit_limits)
      unit_limits<kCta, kN>(P, sx, sy, tm, tn, lp_walk, lq);
      const int row = row128 * kPM + quad * 32 + lane;
      // Cb is kept as raw FP64 bit patterns; in emulated mode no double-typed
      // value may exist at all, or nvcc turns bit tricks into FP64 instructions.
      using Acc = uint64_t;
      Acc cb[kRegCols > 0 ? kRegHalf : 1];
#pragma unroll
      for (int j = 0; j < (kRegCols > 0 ? kRegHalf : 1); ++j) cb[j] = Acc(0);
      if constexpr (kTmHalf > 0) {
        uint32_t z[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) z[j] = 0u;
#pragma unroll
        for (int c = 0; c < 2 * kTmHalf; c += 32) tmem_st32(cb_tmem + c, z);
        tmem_st_wait();
      }

      bool glb_init = false;  // N = 256: this tile's C-resident Cb columns written yet
      PairIter pi;
      pi.init(lp_walk, lq, P.order, P.cutoff);
      for (; pi.valid(); ++acc_it) {
        // This accumulator holds the group starting at pair (p, q) (one pair unless
        // group_max > 1; then its exponents give the whole level's scale, and a row
        // whose slices p.. are all zero (p >= lp) contributes nothing).
        const int p = pi.p, q = pi.q();
        {
          const int lvl = pi.d;
          int gcnt = 0;
          do {
            ++gcnt;
            pi.next();
          } while (pi.valid() && pi.d == lvl && gcnt < P.group_max);
        }
        const uint32_t buf = acc_it % kAccBufs;
        const bool tr = OZ_DIAGNOSTICS && P.trace && unit == 0 && crank == 0 && warp == 4 && lane == 0 &&
                         acc_it < (uint32_t)P.trace_cap;
        if (tr) P.trace[acc_it * 8 + 3] = clock64();
        // This pair's exponents are loaded before waiting for its accumulator, so
        // their latency overlaps the MMAs (short pairs are epilogue-latency-bound).
        const int ea = (row < P.m && p < lp) ? __ldg(P.expo_a + (int64_t)p * P.m + row) : 0;
        // Non-zero G has its FP32 exponent field in [g_lo, g_hi] (PairParams).
        const int2 mm = __ldg(reinterpret_cast<const int2*>(P.ebmm) + (int64_t)q * P.tiles_n + tn);
        const int32_t* ebq = P.ebsh + (int64_t)q * P.n_pad + tn * kN;
        // Pull this pair's B-exponent lines into L1 now: the loads that use them
        // come after the first DADD, i.e. in the short window in which the
        // epilogue's DADDs can drain, where an L2 miss would stall.
        constexpr int kRegLines = (kRegHalf + 31) / 32;  // 128-byte lines of this thread's register-part exponents
        constexpr int kOtherLines = (kTmHalf * 4 + 127) / 128 + (kGlbHalf * 4 + 127) / 128;
        if (lane < kRegLines + kOtherLines) {
          const int32_t* pf = lane < kRegLines ? ebq + half * kRegHalf + lane * 32
                                               : ebq + kRegCols + half * (kTmHalf + kGlbHalf) + (lane - kRegLines) * 32;
          asm volatile("prefetch.global.L1 [%0];" ::"l"(pf));
        }
        mbar_wait(&s.acc_full[buf], (acc_it / kAccBufs) & 1);
        if (tr) P.trace[acc_it * 8 + 4] = clock64();
        tc_fence_after();
        // p >= lp: this CTA's rows have an all-zero A slice p (the partner needs it):
        // the term is +0, nothing to add.
        if (p < lp && !(OZ_DIAGNOSTICS && (P.debug & 1))) {
          const int ea_sh = (ea + 896) * (1 << 20);
          // (FMA terms also need the scale 2^(eA+eB) itself normal.)
          const bool safe = ea + 896 + mm.x + P.g_lo >= 1 && ea + 896 + mm.y + P.g_hi <= 2046 &&
                            (kEmu || !OZ_TERM_FMA || (ea + 1023 + mm.x >= 1 && ea + 1023 + mm.y <= 2046));
          const uint32_t gaddr = tmem + lane_base + buf * kN;
          auto tmem_part = [&]() {
            // Integer adds (emulated mode): rolled, so the code stays in the instruction cache.
#pragma unroll(kTmInt || kTmHalf < 16 ? 1 : kTmHalf / 16)
            for (int ch = 0; ch < kTmHalf / 16; ++ch) {
              uint32_t g[16], w[32];
              tmem_ld16(gaddr + kRegCols + half * kTmHalf + ch * 16, g);
              tmem_ld32(cb_tmem + ch * 32, w);
              tmem_ld_wait();
              Acc c16[16];
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const uint64_t b = (uint64_t)w[2 * j] | ((uint64_t)w[2 * j + 1] << 32);
                c16[j] = b;
              }
              accumulate16<kEmu, kTmInt>(g, ebq + kRegCols + half * kTmHalf + ch * 16, ea_sh, safe, c16, flags);
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const uint64_t b = c16[j];
                w[2 * j] = (uint32_t)b;
                w[2 * j + 1] = (uint32_t)(b >> 32);
              }
              tmem_st32(cb_tmem + ch * 32, w);
            }
            tmem_st_wait();
          };
          auto glb_part = [&]() {
            // C-resident part (N = 256, first k-block only): Cb = C[row, cols] (+0
            // before this tile's first group), Cb += T, C[row, cols] = Cb, with the
            // integer add_lean.
            const int col0 = tn * kN + kRegCols + half * kGlbHalf;
#pragma unroll(kGlbInt || kGlbHalf < 16 ? 1 : kGlbHalf / 16)
            for (int ch = 0; ch < kGlbHalf / 16; ++ch) {
              uint32_t g[16];
              tmem_ld16(gaddr + kRegCols + half * kGlbHalf + ch * 16, g);
              uint64_t c16[16];
              glb_load16(P, row, col0 + ch * 16, glb_init, c16);
              tmem_ld_wait_regs(g);
              accumulate16<kEmu, kGlbInt>(g, ebq + kRegCols + half * kGlbHalf + ch * 16, ea_sh, safe, c16,
                                                   flags);
              if (row < P.m) store_row<kEmu>(P, row, col0 + ch * 16, c16, 16, flags);
            }
            glb_init = true;
          };
          if constexpr (kGlbHalf > 0) glb_part();

          // Software-pipelined TMEM reads: chunk ch+1 loads while chunk ch is
          // accumulated (the wait names the registers so no use is hoisted above it).
          if constexpr (kRegCols > 0) {
            uint32_t g[2][16];
            tmem_ld16(gaddr + half * kRegHalf, g[0]);
            tmem_ld_wait_regs(g[0]);
#pragma unroll
            for (int ch = 0; ch < kRegHalf / 16; ++ch) {
              if (ch + 1 < kRegHalf / 16) tmem_ld16(gaddr + half * kRegHalf + (ch + 1) * 16, g[(ch + 1) & 1]);
              accumulate16<kEmu, kRegInt>(g[ch & 1], ebq + half * kRegHalf + ch * 16, ea_sh, safe, cb + ch * 16, flags);
              if (ch + 1 < kRegHalf / 16) tmem_ld_wait_regs(g[(ch + 1) & 1]);
            }
          }
          if (tr) P.trace[acc_it * 8 + 7] = clock64();
          if constexpr (kTmHalf > 0) tmem_part();
        }
        tc_fence_before();
        __syncwarp();
        if (tr) P.trace[acc_it * 8 + 5] = clock64();
        if (lane == 0) {
          if constexpr (kCta == 1) mbar_arrive(&s.acc_empty[buf]);
          else mbar_arrive_cluster(&s.acc_empty[buf], 0);
        }
      }

      // C = Cb (first block) or C = C + Cb (ozgemm.py:204-207).  The TMEM reads
      // are warp-collective (.sync.aligned): issue them outside the row guard.
      const bool store = !(OZ_DIAGNOSTICS && (P.debug & 8));  // diagnostics: bit 3 skips the C stores
      if constexpr (kGlbHalf > 0) {
        if (!glb_init && row < P.m && store) {  // every group skipped (all-zero A slices): Cb = +0
          uint64_t z[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) z[j] = 0ull;
#pragma unroll
          for (int ch = 0; ch < kGlbHalf / 16; ++ch)
            store_row<kEmu>(P, row, tn * kN + kRegCols + half * kGlbHalf + ch * 16, z, 16, flags);
        }
      }
      if constexpr (kRegCols > 0)
        if (row < P.m && store) store_row<kEmu>(P, row, tn * kN + half * kRegHalf, cb, kRegHalf, flags);
      if constexpr (kTmHalf > 0) {
#pragma unroll(kEmu ? 1 : kTmHalf / 16)
        for (int ch = 0; ch < kTmHalf / 16; ++ch) {
          uint32_t w[32];
          tmem_ld32(cb_tmem + ch * 32, w);
          tmem_ld_wait();
          Acc c16[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            c16[j] = (uint64_t)w[2 * j] | ((uint64_t)w[2 * j + 1] << 32);
          }
          if (row < P.m && store) store_row<kEmu>(P, row, tn * kN + kRegCols + half * kTmHalf + ch * 16, c16, 16, flags);
        }
      }
      // Publish "this tile of C is final" per row band, so a copy stream waiting
      // on the band counter (cuStreamWaitValue32) can move finished bands to the
      // host while later tiles compute.
      if (P.band_done) {
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpi) : "memory");
        if (threadIdx.x == 32 * kLeadWarps) {
          __threadfence_system();
          atomicAdd(P.band_done + tm / P.group, 1u);
        }
      }
    }
    if (flags) atomicOr(P.flags, flags);
  }

  tc_fence_before();
  if constexpr (kCta == 2) cluster_sync(); else __syncthreads();
  if (warp == 1) tmem_dealloc_g<kCta>(tmem);
}

template <int kCta, int kN, bool kEmu>
size_t pair_gemm_smem_bytes() {  // independent of the epilogue warp count
  return sizeof(PairSmem<kCta, kN, kEmu>) + 1024;
}

}  // namespace oz
