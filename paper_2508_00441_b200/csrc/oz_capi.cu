// oz_capi.cu — the C ABI of liboz_b200.so (declared in include/oz_b200.h).
// Unity build: the kernel translation units are included here so one nvcc
// invocation produces the whole library.
#include "oz_tile_gemm.cu"
#include "oz_pair_gemm.cu"
#include "oz_split.cu"
#include "oz_dd_gemm.cu"

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "../../include/oz_b200.h"

namespace {

using oz::LpFormat;

bool fmt_info(int type2, LpFormat& f, uint32_t& idesc_fmt) {
  switch (type2) {
    case OZ_FMT_E4M3: f = {4, 3, 7, 15, 1, 1, 0}; idesc_fmt = 0; return true;
    case OZ_FMT_E5M2: f = {5, 2, 15, 30, 0, 1, 0}; idesc_fmt = 1; return true;
    case OZ_FMT_FP16: f = {5, 10, 15, 30, 0, 2, 0}; idesc_fmt = 0; return true;
    case OZ_FMT_BF16: f = {8, 7, 127, 254, 0, 2, 0}; idesc_fmt = 1; return true;
    // FP6 (OCP, no inf/NaN), kind::f8f6f4 E3M2 = 4, E2M3 = 3.  Slice planes hold the
    // codes densely packed (6 bits each); TMA 16U6_ALIGN16B spreads every 16 codes
    // to a 16-byte group in shared memory, the layout the MMA reads.
    case OZ_FMT_E3M2: f = {3, 2, 3, 7, 0, 1, 0}; idesc_fmt = 4; return true;
    case OZ_FMT_E2M3: f = {2, 3, 1, 3, 0, 1, 0}; idesc_fmt = 3; return true;
    default: return false;
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// 3-D map over slice planes [planes][rows][ld] with a 128-byte x box_rows box, SWIZZLE_128B.
using StreamWaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

StreamWaitFn get_wait_value() {
  static StreamWaitFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<StreamWaitFn>(p);
  });
  return fn;
}

// fp6: planes hold packed FP6 groups (16 codes in 12 bytes + 4 zero bytes per 16
// bytes, written by the split); TMA's 16U6_ALIGN16B type unpacks them into the
// one-byte-per-element shared-memory layout kind::f8f6f4 reads for E3M2/E2M3.
// Its K extent must be the padded ld (a multiple of 128, zero-filled).
int make_plane_map(CUtensorMap* map, const void* base, int elem_bytes, int64_t k, int64_t rows, int64_t planes,
                   int64_t ld, int box_rows = 128, bool fp6 = false) {
  EncodeFn enc = get_encode();
  if (!enc) return OZ_ETMAP;
  if ((reinterpret_cast<uintptr_t>(base) & 15) || ((ld * elem_bytes) & 15)) return OZ_EINVAL;
  if (fp6 && ((reinterpret_cast<uintptr_t>(base) & 31) || (ld & 127))) return OZ_EINVAL;
  const cuuint64_t dims[3] = {(cuuint64_t)(fp6 ? ld : k), (cuuint64_t)rows, (cuuint64_t)planes};
  const int64_t row_bytes = fp6 ? ld * 3 / 4 : ld * elem_bytes;  // FP6 rows are densely packed
  const cuuint64_t strides[2] = {(cuuint64_t)row_bytes, (cuuint64_t)(row_bytes * rows)};
  const cuuint32_t box[3] = {(cuuint32_t)(128 / elem_bytes), (cuuint32_t)box_rows, 1u};
  const cuuint32_t estr[3] = {1u, 1u, 1u};
  const CUtensorMapDataType dt = fp6 ? CU_TENSOR_MAP_DATA_TYPE_16U6_ALIGN16B
                                     : (elem_bytes == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16);
  const CUresult r =
      enc(map, dt, 3,
          const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? OZ_OK : OZ_ETMAP;
}

int num_sms() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

int launch_status() {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "oz_b200: CUDA launch error: %s\n", cudaGetErrorString(e));
    return OZ_ECUDA;
  }
  return OZ_OK;
}

template <bool kEmu, int kCta, int kEB, int kN, int kEpi = oz::kEpiWarps>
int launch_pair(const CUtensorMap& ma, const CUtensorMap& mb, const oz::PairParams& P, int tiles, cudaStream_t st) {
  const size_t smem = oz::pair_gemm_smem_bytes<kCta, kN, kEmu>();
  auto kern = oz::pair_gemm_kernel<kEmu, kCta, kEB, kN, kEpi>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(oz::PairCfg<kCta, kN, kEmu, kEpi>::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kCta;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // Persistent grid: never more units than can be co-resident (the pacing
  // assumes every CTA of a wave runs concurrently).
  int units = num_sms() / kCta;
  cfg.gridDim = dim3((unsigned)(units * kCta));
  int active = 0;
  if (cudaOccupancyMaxActiveClusters(&active, kern, &cfg) == cudaSuccess && active > 0 && active < units)
    units = active;
  cudaGetLastError();
  if (tiles < units) units = tiles;
  cfg.gridDim = dim3((unsigned)(units * kCta));
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ma, mb, P);
  if (e != cudaSuccess) {
    fprintf(stderr, "oz_b200: pair_gemm launch failed: %s\n", cudaGetErrorString(e));
    return OZ_ECUDA;
  }
  return launch_status();
}

template <bool kEmu, int kCta, int kN, int kEpi = oz::kEpiWarps>
int launch_pair_fmt(const CUtensorMap& ma, const CUtensorMap& mb, const oz::PairParams& P, int tiles,
                    cudaStream_t st) {
  return P.elem_bytes == 1 ? launch_pair<kEmu, kCta, 1, kN, kEpi>(ma, mb, P, tiles, st)
                           : launch_pair<kEmu, kCta, 2, kN, kEpi>(ma, mb, P, tiles, st);
}

// Code tables for the fused split, one per (format, rho), built on first use
// per device and kept for the process lifetime (a few KB each).
struct TableKey {
  int dev, type2, rho;
};
std::mutex g_table_mu;
struct TableEntry {
  TableKey key;
  uint32_t* ptr;
  bool clean;
};
TableEntry g_tables[64];
int g_ntables = 0;

int code_table(int type2, const LpFormat& f, int rho, cudaStream_t st, const uint32_t** out, int* clean) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_table_mu);
  for (int i = 0; i < g_ntables; ++i)
    if (g_tables[i].key.dev == dev && g_tables[i].key.type2 == type2 && g_tables[i].key.rho == rho) {
      *out = g_tables[i].ptr;
      *clean = g_tables[i].clean;
      return OZ_OK;
    }
  if (g_ntables == 64) return OZ_EUNSUPPORTED;
  const int kmax = 1 << (53 - rho);
  uint32_t* p = nullptr;
  if (cudaMalloc(&p, sizeof(uint32_t) * (2 * kmax + 1)) != cudaSuccess) return OZ_ECUDA;
  oz::build_code_table_kernel<<<(2 * kmax + 1 + 255) / 256, 256, 0, st>>>(p, kmax, rho, f);
  uint32_t* h = static_cast<uint32_t*>(malloc(sizeof(uint32_t) * (2 * kmax + 1)));
  if (!h) return OZ_ECUDA;
  if (cudaMemcpyAsync(h, p, sizeof(uint32_t) * (2 * kmax + 1), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess) {
    free(h);
    return OZ_ECUDA;
  }
  bool ok = true;
  for (int i = 0; i <= 2 * kmax; ++i) ok = ok && !(h[i] >> 16);
  free(h);
  g_tables[g_ntables++] = {{dev, type2, rho}, p, ok};
  *out = p;
  *clean = ok;
  return OZ_OK;
}

template <int kThreads, int kEPT, int kCL, int kEB, bool kEmu>
int launch_fused(const oz::FusedSplitParams& P, cudaStream_t st) {
  auto kern = oz::split_fused_kernel<kThreads, kEPT, kCL, kEB, kEmu>;
  const size_t smem = sizeof(uint32_t) * (2 * P.kmax + 1);
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(P.rows * kCL));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kCL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = kCL > 1 ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, P);
  if (e != cudaSuccess) {
    fprintf(stderr, "oz_b200: split launch failed: %s\n", cudaGetErrorString(e));
    return OZ_ECUDA;
  }
  return launch_status();
}

template <int kEB, bool kEmu>
int launch_fused_cfg(const oz::FusedSplitParams& P, cudaStream_t st) {
  const int64_t need = P.ld > P.kb ? P.ld : P.kb;
  if (need <= 1024) return launch_fused<64, 16, 1, kEB, kEmu>(P, st);
  if (need <= 2048) return launch_fused<128, 16, 1, kEB, kEmu>(P, st);
  if (need <= 4096) return launch_fused<256, 16, 1, kEB, kEmu>(P, st);
  // Fixed-step fast path (no per-slice reductions): 16 elements per thread and
  // 2 x 16 warps per SM hide the FP64 latency better than 32 elements x 16 warps.
  // The emulated (integer) adaptive split gains from the 32 warps too (3.43 ->
  // 3.06 ms per 8192^2 operand); the hardware one does not (0.79 -> 0.84 ms,
  // profiles/split_emu_r02.txt).
  if (need <= 8192 && (kEmu || (P.fixed_w > 0 && P.max_planes > 0))) return launch_fused<512, 16, 1, kEB, kEmu>(P, st);
  if (need <= 8192) return launch_fused<256, 32, 1, kEB, kEmu>(P, st);
  if (need <= 16384) return launch_fused<512, 32, 1, kEB, kEmu>(P, st);
  if (need <= 32768) return launch_fused<256, 32, 4, kEB, kEmu>(P, st);
  if (need <= 65536) return launch_fused<256, 32, 8, kEB, kEmu>(P, st);
  if (need <= 131072) return launch_fused<512, 32, 8, kEB, kEmu>(P, st);
  return OZ_EUNSUPPORTED;
}

// Kernel variant and tiling of one fused pair-GEMM call (shared with the
// workspace query so both agree).
struct PairPlan {
  int cta, tn, tiles_m, tiles_n, pairs, group, bands;
  size_t eb_bytes, band_bytes, pace_bytes;
};

// Tuning overrides (oz_set_pair_variant; 0 = automatic).  Process-wide, set
// once by experiments and the variant tests — never read from the environment.
std::atomic<int> g_force_cta{0}, g_force_tn{0}, g_force_group{0};
// Epilogue warps of the CTA-pair N = 192 hardware-mode kernel (8 or 12).
std::atomic<int> g_epi_warps{8};
// Pair-GEMM schedule: 0 overlapped epilogue, 1 exclusive epilogue windows.
std::atomic<int> g_pair_sched{0};

PairPlan plan_pair(int64_t m, int64_t n, int64_t kb, int elem_bytes, int sx, int sy, int pair_cutoff, int emu,
                   bool wide_ok = false) {
  PairPlan pl{};
  // CTA pair (cta_group::2) unless the problem has a single 128-row slab; N = 192
  // columns per pair tile in hardware-FP64 mode (tensor-bound), N = 128 in the
  // emulated mode (ALU-bound epilogue: 4 accumulators absorb its jitter, and all
  // of Cb sits in registers; measured 144 -> 109 ms at n = 8192, pair_cutoff = 11).
  // oz_set_pair_variant(cta_group, tile_n, group) overrides (experiments, tests).
  // Variant by a wave-cost model: time ~ waves x columns per CTA / efficiency,
  // efficiencies per output column measured at n = 8192 (profiles/variant_sweep_r01.txt,
  // profiles/variant_kb_r02.txt): 256 x 192 CTA pair 1.00; 256 x 128 pair 0.92, 128 x 128
  // single CTA 0.935, except short FP8 pairs (kb <= 2048: the 4-accumulator 1-CTA kernel
  // absorbs the epilogue better, 1.10); 128 x 64 single CTA 0.795.  N = 192 exists in
  // hardware mode only; a single 128-row slab uses single-CTA tiles.
  const int force_cta = g_force_cta.load(std::memory_order_relaxed);
  const int force_tn = g_force_tn.load(std::memory_order_relaxed);
  {
    const int64_t sms = num_sms();
    const bool short_fp8 = elem_bytes == 1 && kb <= 2048 && !emu;
    struct Cand { int cta, tn; double eff; };
    // 256 x 256 CTA-pair tiles (Cb partly in C itself): fixed-step grouped mode,
    // first k-block, hardware FP64 only (wide_ok).
    const Cand cands[5] = {{2, 256, 1.04}, {2, 192, 1.0}, {2, 128, 0.92}, {1, 128, short_fp8 ? 1.10 : 0.935},
                           {1, 64, 0.795}};
    double best = 0.0;
    pl.cta = 0;
    for (const Cand& c : cands) {
      if (c.tn == 192 && emu) continue;
      if (c.tn == 256 && !wide_ok) continue;  // grouped mode, first k-block
      if (c.cta == 2 && m <= oz::kPM) continue;
      if (force_cta && c.cta != (force_cta == 1 ? 1 : 2)) continue;
      if (force_tn && c.tn != force_tn) continue;
      const int64_t units = sms / c.cta, rows = (int64_t)oz::kPM * c.cta;
      const int64_t tiles = ((m + rows - 1) / rows) * ((n + c.tn - 1) / c.tn);
      const double cost = (double)((tiles + units - 1) / units) * c.tn / c.eff;
      if (pl.cta == 0 || cost < best) {
        best = cost;
        pl.cta = c.cta;
        pl.tn = c.tn;
      }
    }
    if (pl.cta == 0) {  // forced combination that does not exist (e.g. N = 192 emulated): nearest valid
      pl.cta = force_cta == 1 || m <= oz::kPM ? 1 : 2;
      pl.tn = (force_tn == 64 && pl.cta == 1) ? 64 : 128;
    }
  }
  pl.tiles_m = (int)((m + oz::kPM * pl.cta - 1) / (oz::kPM * pl.cta));
  pl.tiles_n = (int)((n + pl.tn - 1) / pl.tn);
  pl.pairs = 0;
  for (int p = 0; p < sx; ++p)
    for (int q = 0; q < sy; ++q)
      if (pair_cutoff < 0 || p + q <= pair_cutoff) ++pl.pairs;
  const size_t n_pad = (size_t)pl.tiles_n * pl.tn;
  pl.eb_bytes = (sizeof(int32_t) * (size_t)sy * (n_pad + 2 * (size_t)pl.tiles_n) + 255) / 256 * 256;
  const int64_t num_kb = (kb * elem_bytes + 127) / 128, spp = (num_kb + oz::kPaceBlocks - 1) / oz::kPaceBlocks;
  pl.pace_bytes = sizeof(uint32_t) * (size_t)pl.tiles_m * pl.tiles_n * (size_t)pl.pairs * (size_t)spp;
  pl.group = 8;
  if (const int f = g_force_group.load(std::memory_order_relaxed)) pl.group = f;
  pl.bands = (pl.tiles_m + pl.group - 1) / pl.group;
  pl.band_bytes = (sizeof(uint32_t) * (size_t)pl.bands + 255) / 256 * 256;
  return pl;
}

// Integer-only FP64 multiply (restates fp64emu._mul_core, fp64emu.py:150-187): normal or
// zero operands (others, and results outside the normal range, set FLAG_EMU_RANGE as the
// reference raises RangeError); 53 x 53-bit significand product, RNE to 53 bits.
__device__ uint64_t emu_mul(uint64_t a, uint64_t b, uint32_t& f) {
  constexpr uint64_t kSgn = 1ull << 63, kFrac = (1ull << 52) - 1;
  const uint32_t ea = (uint32_t)(a >> 52) & 0x7FFu, eb = (uint32_t)(b >> 52) & 0x7FFu;
  if ((ea == 0 && (a & kFrac)) || ea == 0x7FFu || (eb == 0 && (b & kFrac)) || eb == 0x7FFu) f |= oz::FLAG_EMU_RANGE;
  const uint64_t sign = (a ^ b) & kSgn;
  if ((a & ~kSgn) == 0 || (b & ~kSgn) == 0) return sign;  // a zero factor: signed zero
  const uint64_t ma = (a & kFrac) | (1ull << 52), mb = (b & kFrac) | (1ull << 52);
  const uint64_t lo = ma * mb, hi = __umul64hi(ma, mb);  // product in [2^104, 2^106)
  const int t = (int)((hi >> 41) & 1u);
  const int sh = 52 + t;
  uint64_t sig = (hi << (64 - sh)) | (lo >> sh);
  const uint64_t rem = lo & ((1ull << sh) - 1), half = 1ull << (sh - 1);
  sig += (rem > half || (rem == half && (sig & 1u))) ? 1u : 0u;  // guard && (sticky || odd)
  const int carry = sig == (1ull << 53) ? 1 : 0;
  sig >>= carry;
  const int e = (int)ea + (int)eb - 1023 + t + carry;
  if (e < 1 || e > 2046) {
    f |= oz::FLAG_EMU_RANGE;
    return sign;
  }
  return sign | ((uint64_t)e << 52) | (sig & kFrac);
}

// fp64emu._lt_core (fp64emu.py:257-266): -0 == +0, sign-magnitude -> monotone key.
__device__ uint64_t emu_order_key(uint64_t x) {
  constexpr uint64_t kSgn = 1ull << 63;
  const uint64_t v = (x & ~kSgn) == 0 ? 0ull : x;
  return (v & kSgn) ? ~v : (v | kSgn);
}

__global__ void emu_add_batch_kernel(const uint64_t* __restrict__ a, const uint64_t* __restrict__ b,
                                     uint64_t* __restrict__ out, int64_t n, int mode, uint32_t* flags) {
  uint32_t f = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (mode == 3) {
      out[i] = emu_mul(a[i], b[i], f);
      continue;
    }
    if (mode == 4) {
      out[i] = emu_order_key(a[i]) < emu_order_key(b[i]) ? 1ull : 0ull;
      continue;
    }
    if (mode == 2) {  // add_lean on its domain (normal or zero operands), emu_add otherwise / when slow
      const uint32_t ea = (uint32_t)(a[i] >> 52) & 0x7FFu, eb = (uint32_t)(b[i] >> 52) & 0x7FFu;
      const bool dom = (ea != 0 || (a[i] << 1) == 0) && (eb != 0 || (b[i] << 1) == 0) && ea != 0x7FFu && eb != 0x7FFu;
      bool slow = true;
      const uint64_t r = dom ? oz::add_lean<false>(a[i], b[i], slow) : 0ull;
      out[i] = slow ? oz::emu_add(a[i], b[i], f) : r;
      continue;
    }
    out[i] = mode == 0 ? oz::emu_add(a[i], b[i], f) : oz::fast_add<true>(a[i], b[i], f);
  }
  if (f) atomicOr(flags, f);
}

int split_impl(const double* X, int64_t rows, int64_t kb, int64_t ldx, int type2, int rho, int emu, int cap,
               int fixed_w, int max_planes, void* coeff, int64_t ld_coeff, int32_t* expo, int32_t* row_cnt,
               int32_t* s_max, uint32_t* flags, void* stream);

}  // namespace

extern "C" {

int64_t oz_pair_gemm_workspace(int64_t m, int64_t n, int64_t kb, int type2, int sx, int sy, int pair_cutoff) {
  if (m <= 0 || n <= 0 || kb <= 0 || sx <= 0 || sy <= 0) return 0;
  LpFormat f;
  uint32_t idf;
  if (!fmt_info(type2, f, idf)) return 0;
  const PairPlan p0 = plan_pair(m, n, kb, f.bytes, sx, sy, pair_cutoff, 0),
                 p1 = plan_pair(m, n, kb, f.bytes, sx, sy, pair_cutoff, 1),
                 p2 = plan_pair(m, n, kb, f.bytes, sx, sy, pair_cutoff, 0, true);
  const size_t b0 = p0.eb_bytes + p0.band_bytes + p0.pace_bytes, b1 = p1.eb_bytes + p1.band_bytes + p1.pace_bytes,
               b2 = p2.eb_bytes + p2.band_bytes + p2.pace_bytes;
  const size_t b01 = b0 > b1 ? b0 : b1;
  return (int64_t)(b01 > b2 ? b01 : b2);
}

int oz_split_fused(const double* X, int64_t rows, int64_t kb, int64_t ldx, int type2, int rho, int emu, int cap,
                   void* coeff, int64_t ld_coeff, int32_t* expo, int32_t* row_cnt, int32_t* s_max, uint32_t* flags,
                   void* stream) {
  return split_impl(X, rows, kb, ldx, type2, rho, emu, cap, 0, 0, coeff, ld_coeff, expo, row_cnt, s_max, flags,
                    stream);
}

int oz_split_fixed(const double* X, int64_t rows, int64_t kb, int64_t ldx, int type2, int rho, int emu, int cap,
                   int max_planes, void* coeff, int64_t ld_coeff, int32_t* expo, int32_t* row_cnt, int32_t* s_max,
                   uint32_t* flags, void* stream) {
  if (rho < 42 || rho > 53 || max_planes < 0) return OZ_EINVAL;
  return split_impl(X, rows, kb, ldx, type2, rho, emu, cap, 54 - rho, max_planes, coeff, ld_coeff, expo, row_cnt,
                    s_max, flags, stream);
}

int64_t oz_split_fixed_cols_scratch(int64_t cols) { return cols > 0 ? 3 * 4 * cols : 0; }

int oz_split_fixed_cols(const double* X, int64_t kb, int64_t cols, int64_t ldx, int type2, int rho, int emu, int cap,
                        int max_planes, void* coeff, int64_t ld_coeff, int32_t* expo, int32_t* col_cnt,
                        int32_t* s_max, uint32_t* flags, void* scratch, void* stream) {
  LpFormat f;
  uint32_t idf;
  if (!fmt_info(type2, f, idf)) return OZ_EUNSUPPORTED;
  if (rho < 42 || rho > 53) return OZ_EUNSUPPORTED;
  if (kb < 1 || cols < 0 || ldx < cols || ld_coeff < kb || cap < 0 || max_planes < 1 || !X || !col_cnt ||
      !s_max || !flags)
    return OZ_EINVAL;
  if ((ld_coeff * f.bytes) % 16) return OZ_EINVAL;
  if (cols == 0) return OZ_OK;
  if (!scratch || (cap > 0 && (!coeff || !expo))) return OZ_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  oz::ColSplitParams P{};
  P.X = X; P.kb = kb; P.cols = cols; P.ldx = ldx; P.rho = rho; P.w = 54 - rho; P.max_planes = max_planes;
  P.cap = cap; P.coeff = cap > 0 ? static_cast<uint8_t*>(coeff) : nullptr; P.ld = ld_coeff; P.expo = expo;
  P.col_cnt = col_cnt; P.s_max = s_max; P.flags = flags; P.kmax = 1 << (53 - rho);
  P.pack6 = (type2 == OZ_FMT_E3M2 || type2 == OZ_FMT_E2M3) ? 1 : 0;
  if (P.pack6 && (ld_coeff & 127)) return OZ_EINVAL;
  int rc = code_table(type2, f, rho, st, &P.table, &P.table_clean);
  if (rc) return rc;
  P.key = static_cast<uint32_t*>(scratch);
  P.need = P.key + cols;
  P.tiny = P.need + cols;
  if (cudaMemsetAsync(scratch, 0, (size_t)oz_split_fixed_cols_scratch(cols), st) != cudaSuccess) return OZ_ECUDA;
  const dim3 grid((unsigned)((cols + oz::kColTJ - 1) / oz::kColTJ), (unsigned)((kb + oz::kColTK - 1) / oz::kColTK));
  oz::col_stats_kernel<<<grid, 256, 0, st>>>(P);
  const size_t smem = sizeof(uint32_t) * (2 * P.kmax + 1);
  auto kern = f.bytes == 1 ? (emu ? oz::col_slice_kernel<1, true> : oz::col_slice_kernel<1, false>)
                           : (emu ? oz::col_slice_kernel<2, true> : oz::col_slice_kernel<2, false>);
  if (smem > 8 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<grid, 256, smem, st>>>(P);
  oz::col_finish_kernel<<<(unsigned)((cols + 255) / 256), 256, 0, st>>>(P);
  return launch_status();
}

}  // extern "C"

namespace {
int split_impl(const double* X, int64_t rows, int64_t kb, int64_t ldx, int type2, int rho, int emu, int cap,
               int fixed_w, int max_planes, void* coeff, int64_t ld_coeff, int32_t* expo, int32_t* row_cnt,
               int32_t* s_max, uint32_t* flags, void* stream) {
  LpFormat f;
  uint32_t idf;
  if (!fmt_info(type2, f, idf)) return OZ_EUNSUPPORTED;
  if (rows < 0 || kb < 1 || ldx < kb || ld_coeff < kb || cap < 0 || !X || !row_cnt || !s_max || !flags)
    return OZ_EINVAL;
  if ((ld_coeff * f.bytes) % 16) return OZ_EINVAL;
  if (rho < 42 || rho > 53) return OZ_EUNSUPPORTED;  // |k| <= 2^(53-rho) table; rho >= xi >= 42 for our formats
  if (rows == 0) return OZ_OK;
  if (cap > 0 && (!coeff || !expo)) return OZ_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  oz::FusedSplitParams P{};
  P.X = X; P.rows = rows; P.kb = kb; P.ldx = ldx; P.rho = rho; P.cap = cap;
  P.coeff = static_cast<uint8_t*>(coeff); P.ld = ld_coeff; P.expo = expo; P.row_cnt = row_cnt;
  P.s_max = s_max; P.flags = flags; P.kmax = 1 << (53 - rho);
  P.fixed_w = fixed_w; P.max_planes = max_planes;
  P.pack6 = (type2 == OZ_FMT_E3M2 || type2 == OZ_FMT_E2M3) ? 1 : 0;
  if (P.pack6 && (ld_coeff & 127)) return OZ_EINVAL;  // packed FP6 rows: multiples of 128 codes
  int rc = code_table(type2, f, rho, st, &P.table, &P.table_clean);
  if (rc) return rc;
  if (f.bytes == 1) return emu ? launch_fused_cfg<1, true>(P, st) : launch_fused_cfg<1, false>(P, st);
  return emu ? launch_fused_cfg<2, true>(P, st) : launch_fused_cfg<2, false>(P, st);
}
}  // namespace

extern "C" {

int oz_split_pad(void* coeff, int64_t ld_coeff, int64_t rows, int type2, int s, int32_t* expo,
                 const int32_t* row_cnt, const int32_t* s_dev, void* stream) {
  LpFormat f;
  uint32_t idf;
  if (!fmt_info(type2, f, idf)) return OZ_EUNSUPPORTED;
  if (rows < 0 || s < 0 || (ld_coeff * f.bytes) % 16) return OZ_EINVAL;
  if (rows == 0 || s == 0) return OZ_OK;
  if (!coeff || !row_cnt) return OZ_EINVAL;  // expo == NULL: exponents left as they are (fixed-step planes)
  const unsigned blocks = (unsigned)((rows + 7) / 8);
  const int64_t row_bytes = (type2 == OZ_FMT_E3M2 || type2 == OZ_FMT_E2M3) ? ld_coeff * 3 / 4 : ld_coeff * f.bytes;
  oz::pad_planes_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(static_cast<uint8_t*>(coeff), row_bytes,
                                                                   rows, s, expo, row_cnt, s_dev);
  return launch_status();
}

int oz_set_pair_variant(int cta_group, int tile_n, int raster_group) {
  if (cta_group < 0 || cta_group > 2 || (tile_n != 0 && tile_n != 64 && tile_n != 128 && tile_n != 192 && tile_n != 256) ||
      raster_group < 0)
    return OZ_EINVAL;
  g_force_cta.store(cta_group, std::memory_order_relaxed);
  g_force_tn.store(tile_n, std::memory_order_relaxed);
  g_force_group.store(raster_group, std::memory_order_relaxed);
  return OZ_OK;
}

int oz_pair_plan(int64_t m, int64_t n, int64_t kb, int type2, int sx, int sy, int pair_cutoff, int emu, int group_max,
                 int accumulate, int* cta_group, int* tile_n) {
  LpFormat f;
  uint32_t idf;
  if (!fmt_info(type2, f, idf)) return OZ_EUNSUPPORTED;
  if (m <= 0 || n <= 0 || kb <= 0 || sx < 0 || sy < 0 || !cta_group || !tile_n) return OZ_EINVAL;
  const PairPlan pl = plan_pair(m, n, kb, f.bytes, sx, sy, pair_cutoff, emu, group_max > 1 && !accumulate);
  *cta_group = pl.cta;
  *tile_n = pl.tn;
  return OZ_OK;
}

int oz_set_pair_schedule(int mode) {
  if (mode != 0 && mode != 1) return OZ_EINVAL;
  g_pair_sched.store(mode, std::memory_order_relaxed);
  return OZ_OK;
}

int oz_set_epilogue_warps(int warps) {
  if (warps != 8 && warps != 12) return OZ_EINVAL;
  g_epi_warps.store(warps, std::memory_order_relaxed);
  return OZ_OK;
}

const char* oz_version(void) { return "oz_b200 0.1 (sm_100a tcgen05; reference ozdgemm 1.0.0 semantics)"; }

const char* oz_strerror(int status) {
  switch (status) {
    case OZ_OK: return "ok";
    case OZ_EINVAL: return "invalid argument";
    case OZ_EUNSUPPORTED: return "unsupported format or size on sm_100a";
    case OZ_ECUDA: return "CUDA launch error";
    case OZ_ETMAP: return "cuTensorMapEncodeTiled failed";
    case OZ_ESLICES: return "reserved (no slice-count limit in this version)";
    default: return "unknown status";
  }
}

int oz_split_count(const double* X, int64_t rows, int64_t kb, int64_t ldx, int type2, int rho, int emu,
                   int32_t* row_cnt, int32_t* s_max, uint32_t* flags, void* stream) {
  // Count-only mode of the fused split (no coefficient buffer).
  LpFormat f;
  uint32_t idf;
  if (!fmt_info(type2, f, idf)) return OZ_EUNSUPPORTED;
  if (rows < 0 || kb < 1 || ldx < kb || !X || !row_cnt || !s_max || !flags) return OZ_EINVAL;
  const int64_t ld = (type2 == OZ_FMT_E3M2 || type2 == OZ_FMT_E2M3) ? (kb + 127) / 128 * 128 : (kb + 15) / 16 * 16;
  return oz_split_fused(X, rows, kb, ldx, type2, rho, emu, 0, nullptr, ld, nullptr, row_cnt, s_max, flags, stream);
}

int oz_split_rows(const double* X, int64_t rows, int64_t kb, int64_t ldx, int type2, int rho, int emu, int planes,
                  void* coeff, int64_t ld_coeff, int32_t* expo, int32_t* row_cnt, uint32_t* flags, void* stream) {
  // Exactly `planes` planes: fused split with cap = planes, then zero padding.
  LpFormat f;
  uint32_t idf;
  if (!fmt_info(type2, f, idf)) return OZ_EUNSUPPORTED;
  if (rows < 0 || kb < 1 || ldx < kb || ld_coeff < kb || planes < 0 || !X || !row_cnt || !flags) return OZ_EINVAL;
  if ((ld_coeff * f.bytes) % 16) return OZ_EINVAL;
  if (rows == 0 || planes == 0) return OZ_OK;
  if (!coeff || !expo) return OZ_EINVAL;
  int32_t* s_scratch = nullptr;
  if (cudaMallocAsync(&s_scratch, sizeof(int32_t), (cudaStream_t)stream) != cudaSuccess) return OZ_ECUDA;
  cudaMemsetAsync(s_scratch, 0, sizeof(int32_t), (cudaStream_t)stream);
  int rc = oz_split_fused(X, rows, kb, ldx, type2, rho, emu, planes, coeff, ld_coeff, expo, row_cnt, s_scratch,
                          flags, stream);
  cudaFreeAsync(s_scratch, (cudaStream_t)stream);
  if (rc) return rc;
  return oz_split_pad(coeff, ld_coeff, rows, type2, planes, expo, row_cnt, nullptr, stream);
}

int oz_transpose(const double* src, int64_t rows, int64_t cols, int64_t ld_src, double* dst, int64_t ld_dst,
                 void* stream) {
  if (rows < 0 || cols < 0 || ld_src < cols || ld_dst < rows) return OZ_EINVAL;
  if (rows == 0 || cols == 0) return OZ_OK;
  if (!src || !dst) return OZ_EINVAL;
  const dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
  oz::transpose_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(src, rows, cols, ld_src, dst, ld_dst);
  return launch_status();
}

int oz_tile_counts(const int32_t* row_cnt, int64_t rows, int32_t* tile_cnt, void* stream) {
  if (rows < 0 || !row_cnt || !tile_cnt) return OZ_EINVAL;
  if (rows == 0) return OZ_OK;
  oz::tile_counts_kernel<<<(unsigned)((rows + 127) / 128), 128, 0, (cudaStream_t)stream>>>(row_cnt, rows, tile_cnt);
  return launch_status();
}

static int pair_gemm_impl(const void* a_planes, const void* b_planes, int64_t ld_a, int64_t ld_b, int planes_a,
                          int planes_b, const int32_t* expo_a, const int32_t* expo_b, const int32_t* tile_cnt_a,
                          const int32_t* tile_cnt_b, int64_t m, int64_t n, int64_t kb, int sx, int sy, int type2,
                          int order, int pair_cutoff, int emu, int accumulate, double* C, int64_t ldc,
                          uint32_t* flags, void* workspace, int64_t workspace_bytes, int pace_slack, double* C_host,
                          int64_t ldc_host, void* copy_stream, const int32_t* s_dev, int group_max, void* stream) {
  LpFormat f;
  uint32_t idf;
  if (!fmt_info(type2, f, idf)) return OZ_EUNSUPPORTED;
  // FP6 operands: packed planes, TMA 16U6_ALIGN16B (fp6e2m3 never gets here: the
  // split reports SlicingInfeasible like the reference).
  const bool fp6 = type2 == OZ_FMT_E3M2 || type2 == OZ_FMT_E2M3;
  if (m < 0 || n < 0 || kb < 1 || sx < 0 || sy < 0 || sx > planes_a || sy > planes_b || ldc < n || !C || !flags)
    return OZ_EINVAL;
  if ((tile_cnt_a == nullptr) != (tile_cnt_b == nullptr)) return OZ_EINVAL;
  if (m == 0 || n == 0) return OZ_OK;
  if (m > INT32_MAX || n > INT32_MAX || kb > INT32_MAX) return OZ_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  if (sx == 0 || sy == 0) {
    // No pairs at all: Cb = 0, so C = 0 (first block) or C unchanged.
    if (!accumulate) {
      if (ldc == n) cudaMemsetAsync(C, 0, sizeof(double) * m * n, st);
      else cudaMemset2DAsync(C, ldc * sizeof(double), 0, n * sizeof(double), m, st);
    }
    if (C_host && ldc_host >= n)
      cudaMemcpy2DAsync(C_host, ldc_host * sizeof(double), C, ldc * sizeof(double), n * sizeof(double), m,
                        cudaMemcpyDeviceToHost, st);
    return launch_status();
  }
  if (!a_planes || !b_planes || !expo_a || !expo_b) return OZ_EINVAL;
  oz::PairParams P{};
  P.expo_a = expo_a; P.expo_b = expo_b; P.tile_cnt_a = tile_cnt_a; P.tile_cnt_b = tile_cnt_b;
  P.C = C; P.ldc = ldc; P.m = (int)m; P.n = (int)n; P.kb = (int)kb; P.sx = sx; P.sy = sy;
  P.order = order; P.cutoff = pair_cutoff; P.accumulate = accumulate;
  P.elem_bytes = f.bytes; P.fmt = idf; P.flags = flags; P.s_dev = s_dev;
  P.fp6 = (type2 == OZ_FMT_E3M2 || type2 == OZ_FMT_E2M3) ? 1 : 0;
  const PairPlan pl = plan_pair(m, n, kb, f.bytes, sx, sy, pair_cutoff, emu, group_max > 1 && !accumulate);
  const int cta = pl.cta, tn = pl.tn;
  if (!workspace || (size_t)workspace_bytes < pl.eb_bytes) return OZ_EINVAL;  // see oz_pair_gemm_workspace
  P.group = pl.group;
  P.hint_a = P.hint_b = oz::kEvictNormal;
  // Non-zero G (a sum of up to group_max pair products): FP32 exponent field in
  // [127 - 2 m2, 127 + ceil(log2(group_max kb))] (PairParams).
  if (group_max < 1 || group_max > 64) return OZ_EINVAL;
  P.group_max = group_max;
  P.g_lo = 127 - 2 * (f.mbits + 1);
  {
    int lg = 0;
    while ((1ll << lg) < kb * group_max) ++lg;
    P.g_hi = 127 + lg;
  }
  P.trace = nullptr; P.trace_cap = 0; P.debug = 0;
  P.serial = g_pair_sched.load(std::memory_order_relaxed);
#if OZ_DIAGNOSTICS
  // Diagnostic builds only (tools/): OZ_DEBUG_MODE bits, L2 hints, and
  // OZ_TRACE=<device address hex>:<entries> (tools/k3_trace.py).
  if (const char* e = getenv("OZ_DEBUG_MODE")) P.debug = atoi(e);
  {
    const uint64_t hints[3] = {oz::kEvictNormal, oz::kEvictFirst, oz::kEvictLast};
    const char* ha = getenv("OZ_HINT_A");
    const char* hb = getenv("OZ_HINT_B");
    P.hint_a = hints[ha ? (atoi(ha) % 3 + 3) % 3 : 0];
    P.hint_b = hints[hb ? (atoi(hb) % 3 + 3) % 3 : 0];
  }
  if (const char* e = getenv("OZ_TRACE")) {
    unsigned long long addr = 0;
    int cap = 0;
    if (sscanf(e, "%llx:%d", &addr, &cap) == 2) {
      P.trace = reinterpret_cast<unsigned long long*>(addr);
      P.trace_cap = cap;
    }
  }
#endif
  CUtensorMap ma, mb;
  int rc = make_plane_map(&ma, a_planes, f.bytes, kb, m, planes_a, ld_a, oz::kPM, fp6);
  if (rc) return rc;
  rc = make_plane_map(&mb, b_planes, f.bytes, kb, n, planes_b, ld_b, tn / cta, fp6);
  if (rc) return rc;
  P.tiles_m = pl.tiles_m;
  P.tiles_n = pl.tiles_n;
  const int tiles = P.tiles_m * P.tiles_n;
  // Per-tile B exponents for the epilogue (first part of the workspace).
  P.n_pad = P.tiles_n * tn;
  int32_t* eb_ws = static_cast<int32_t*>(workspace);
  P.ebsh = eb_ws;
  P.ebmm = eb_ws + (size_t)sy * P.n_pad;
  oz::prep_eb_kernel<<<dim3((unsigned)P.tiles_n, (unsigned)sy), tn, 0, st>>>(expo_b, (int)n, tn, P.n_pad, P.tiles_n,
                                                                         eb_ws, eb_ws + (size_t)sy * P.n_pad, s_dev);
  // Pacing needs an identical pair sequence in every tile (no skipping) and
  // scratch counters (one per tile-wave and pair) after the exponents and the
  // band counters.
  P.step_ctr = nullptr; P.pace_slack = 0; P.pairs_per_tile = 0;
  if (!tile_cnt_a && pace_slack > 0 && pl.pairs > 0 &&
      (size_t)workspace_bytes >= pl.eb_bytes + pl.band_bytes + pl.pace_bytes) {
    uint8_t* pace = static_cast<uint8_t*>(workspace) + pl.eb_bytes + pl.band_bytes;
    cudaMemsetAsync(pace, 0, pl.pace_bytes, st);
    P.step_ctr = reinterpret_cast<uint32_t*>(pace);
    P.pace_slack = pace_slack;
    P.pairs_per_tile = pl.pairs;
  }
  // Overlapped device->host copy of C (optional): band counters zeroed on the
  // compute stream, the copy stream joins after that memset, and per row band
  // it waits (cuStreamWaitValue32) for all of the band's tiles, then copies it.
  P.band_done = nullptr;
  cudaStream_t cst = (cudaStream_t)copy_stream;
  StreamWaitFn wait_fn = C_host ? get_wait_value() : nullptr;
  const bool overlap = C_host && cst && wait_fn && ldc_host >= n &&
                       (size_t)workspace_bytes >= pl.eb_bytes + pl.band_bytes;
  if (overlap) {
    // Zero the counters on the compute stream (ordered after whatever used this
    // workspace memory before), then let the copy stream start waiting only
    // after that memset — not after the kernel.
    P.band_done = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(workspace) + pl.eb_bytes);
    cudaMemsetAsync(P.band_done, 0, pl.band_bytes, st);
    cudaEvent_t ev;
    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    cudaEventRecord(ev, st);
    cudaStreamWaitEvent(cst, ev, 0);
    cudaEventDestroy(ev);
  }
  if (cta == 1 && tn == 64)
    rc = emu ? launch_pair_fmt<true, 1, 64>(ma, mb, P, tiles, st) : launch_pair_fmt<false, 1, 64>(ma, mb, P, tiles, st);
  else if (cta == 1)
    rc = emu ? launch_pair_fmt<true, 1, 128>(ma, mb, P, tiles, st) : launch_pair_fmt<false, 1, 128>(ma, mb, P, tiles, st);
  else if (tn == 256)  // fixed-step grouped mode, first k-block (plan_pair); emulated: all of Cb in C, integer adds
    rc = emu ? launch_pair_fmt<true, 2, 256>(ma, mb, P, tiles, st) : launch_pair_fmt<false, 2, 256>(ma, mb, P, tiles, st);
  else if (tn == 192)  // hardware mode only (plan_pair)
    rc = g_epi_warps.load(std::memory_order_relaxed) == 12 ? launch_pair_fmt<false, 2, 192, 12>(ma, mb, P, tiles, st)
                                                           : launch_pair_fmt<false, 2, 192, 8>(ma, mb, P, tiles, st);
  else
    rc = emu ? launch_pair_fmt<true, 2, 128>(ma, mb, P, tiles, st) : launch_pair_fmt<false, 2, 128>(ma, mb, P, tiles, st);
  if (rc) return rc;
  if (C_host) {
    const int64_t band_rows = (int64_t)pl.group * oz::kPM * cta;
    for (int b = 0; b < pl.bands; ++b) {
      const int64_t r0 = b * band_rows, r1 = r0 + band_rows < m ? r0 + band_rows : m;
      if (overlap) {
        const int band_tm = (pl.tiles_m - b * pl.group) < pl.group ? pl.tiles_m - b * pl.group : pl.group;
        const uint32_t expect = (uint32_t)(band_tm * pl.tiles_n * cta);
        if (wait_fn(cst, reinterpret_cast<CUdeviceptr>(P.band_done + b), expect, 0x0 /* GEQ */) != CUDA_SUCCESS)
          return OZ_ECUDA;
      }
      cudaMemcpy2DAsync(C_host + r0 * ldc_host, ldc_host * sizeof(double), C + r0 * ldc, ldc * sizeof(double),
                        n * sizeof(double), r1 - r0, cudaMemcpyDeviceToHost, overlap ? cst : st);
    }
  }
  return launch_status();
}

int oz_pair_gemm(const void* a_planes, const void* b_planes, int64_t ld_a, int64_t ld_b, int planes_a,
                 int planes_b, const int32_t* expo_a, const int32_t* expo_b, const int32_t* tile_cnt_a,
                 const int32_t* tile_cnt_b, int64_t m, int64_t n, int64_t kb, int sx, int sy, int type2,
                 int order, int pair_cutoff, int emu, int accumulate, double* C, int64_t ldc, uint32_t* flags,
                 void* workspace, int64_t workspace_bytes, int pace_slack, double* C_host, int64_t ldc_host,
                 void* copy_stream, const int32_t* s_dev, void* stream) {
  return pair_gemm_impl(a_planes, b_planes, ld_a, ld_b, planes_a, planes_b, expo_a, expo_b, tile_cnt_a, tile_cnt_b,
                        m, n, kb, sx, sy, type2, order, pair_cutoff, emu, accumulate, C, ldc, flags, workspace,
                        workspace_bytes, pace_slack, C_host, ldc_host, copy_stream, s_dev, 1, stream);
}

int oz_pair_gemm_grouped(const void* a_planes, const void* b_planes, int64_t ld_a, int64_t ld_b, int planes_a,
                         int planes_b, const int32_t* expo_a, const int32_t* expo_b, int64_t m, int64_t n,
                         int64_t kb, int sx, int sy, int type2, int order, int pair_cutoff, int group_max, int emu,
                         int accumulate, double* C, int64_t ldc, uint32_t* flags, void* workspace,
                         int64_t workspace_bytes, int pace_slack, double* C_host, int64_t ldc_host,
                         void* copy_stream, const int32_t* s_dev, void* stream) {
  return pair_gemm_impl(a_planes, b_planes, ld_a, ld_b, planes_a, planes_b, expo_a, expo_b, nullptr, nullptr, m, n,
                        kb, sx, sy, type2, order, pair_cutoff, emu, accumulate, C, ldc, flags, workspace,
                        workspace_bytes, pace_slack, C_host, ldc_host, copy_stream, s_dev, group_max, stream);
}

int oz_emu_add_batch(const uint64_t* a, const uint64_t* b, uint64_t* out, int64_t n, int mode, uint32_t* flags,
                     void* stream) {
  if (n < 0 || mode < 0 || mode > 4) return OZ_EINVAL;
  if (n == 0) return OZ_OK;
  if (!a || !b || !out || !flags) return OZ_EINVAL;
  const int64_t blocks = (n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096;
  emu_add_batch_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(a, b, out, n, mode, flags);
  return launch_status();
}

int oz_dd_gemm(const double* A, const double* B, double* C, int64_t m, int64_t n, int64_t k, void* stream) {
  if (m < 0 || n < 0 || k < 0 || m > INT32_MAX || n > INT32_MAX || k > INT32_MAX) return OZ_EINVAL;
  if (m == 0 || n == 0) return OZ_OK;
  if (!A || !B || !C) return OZ_EINVAL;
  const dim3 grid((unsigned)((n + 63) / 64), (unsigned)((m + 63) / 64));
  oz::dd_gemm_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(A, B, C, (int)m, (int)n, (int)k);
  return launch_status();
}

int oz_lp_gemm(const void* a_plane, const void* b_plane, int64_t ld_a, int64_t ld_b, int64_t m, int64_t n,
               int64_t k, int type2, float* D, int64_t ldd, void* stream) {
  LpFormat f;
  uint32_t idf;
  if (!fmt_info(type2, f, idf)) return OZ_EUNSUPPORTED;
  const bool fp6 = type2 == OZ_FMT_E3M2 || type2 == OZ_FMT_E2M3;  // packed planes, ld a multiple of 128
  if (m < 0 || n < 0 || k < 0 || ldd < n || !D) return OZ_EINVAL;
  if (m == 0 || n == 0) return OZ_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (k == 0) {
    cudaMemset2DAsync(D, ldd * sizeof(float), 0, n * sizeof(float), m, st);
    return launch_status();
  }
  if (!a_plane || !b_plane || m > INT32_MAX || n > INT32_MAX || k > INT32_MAX) return OZ_EINVAL;
  CUtensorMap ma, mb;
  int rc = make_plane_map(&ma, a_plane, f.bytes, k, m, 1, ld_a, 128, fp6);
  if (rc) return rc;
  rc = make_plane_map(&mb, b_plane, f.bytes, k, n, 1, ld_b, 128, fp6);
  if (rc) return rc;
  const size_t smem = oz::tile_gemm_smem_bytes();
  cudaFuncSetAttribute(oz::tile_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const dim3 grid((unsigned)((m + oz::kTileM - 1) / oz::kTileM), (unsigned)((n + oz::kTileN - 1) / oz::kTileN));
  oz::tile_gemm_kernel<<<grid, 128, smem, st>>>(ma, mb, D, ldd, (int)m, (int)n, (int)k, 0, 0, f.bytes, idf,
                                                 fp6 ? 1 : 0);
  return launch_status();
}

}  // extern "C"
