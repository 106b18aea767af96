// seed_i8.cu — the fused two-sided fp64 seed contraction (both seed GEMMs of
// Algorithm 2 in one pass over Y) on the int8 tensor cores, exact-integer
// digit arithmetic with fp64 recombination.
//
// Reference: right seed  cache.right = Y_(1:p) * KR(p+1..N)  (mttkrp.cpp:149-163)
//            left seed   cache.left  = Y_(1:p)^T * KR(1..p)  (mttkrp.cpp:195-210)
//
// Why: on B200 the FP64 pipe (DMMA and DFMA alike) peaks at 37 TF/s, so the
// fused pass (4 R flops per 8-byte element) is FP64-bound well below HBM speed
// for every fp64 config.  The int8 tensor pipe is ~60x faster; fp64 values are
// split into six balanced base-256 digits and every digit product is exact.
//
// Encoding.  Y carries one power-of-two scale for the whole tensor (2^eY >= max
// |Y|, cached per tensor version).  The Khatri-Rao rows of each side carry one
// scale per rank column for all tiles (the product of the factor column maxima),
// and their digits are generated straight from the factors (kr_digits_kernel).  v = rint(x 2^(46-e)) (|v| <= 2^46) is
// v = sum_k d_k 256^k, d_k in [-128, 127], k = 0..5.  One DFMA produces it:
// fma(x, 2^(46-e), 2^52 + sum_k 128 256^k) has v + sum_k 128 256^k in the low 48
// mantissa bits, whose bytes are d_k + 128 (xor 0x80 gives the signed digit).
// Top-first plane a = 5 - k.  The digit-pair products kept are a + b <= 5 (21 of
// 36); the dropped ones sit 2^-48 below the leading term and random-signed, so
// the relative error is ~1e-13 (tests/test_gpu_i8.py holds it to 1e-10).
//
// Tile = 128 rows i x 128 columns j, digits in two half-tile buffers (columns
// 0-63, 64-127).  Digit plane a of a half is 64 rows j of 128 bytes (i
// contiguous, 128-byte swizzle) and serves both products:
//   right  D_R[i][r] += sum_j P_a[i][j] B_R[r][j]  A = P_a, M = 128 (i), MN-major
//   left   D_L[j][r]  = sum_i P_a[i][j] B_L[r][i]  A = P_a^T, M = 64 (j), K-major,
//          half h in TMEM lanes 16 h .. 16 h + 15 of each 32-lane quarter
// (layouts checked bit-exactly by tools/microbench/i8_mma.cu).  For plane a one
// MMA per 32-deep K step covers all its partners b = 0..5-a: the Khatri-Rao
// digit planes are stacked along N and the accumulator starts at diagonal a, so
// column block b lands on diagonal a + b (6 accumulators of N columns per
// product, exact int32).  The right accumulators run across a row block's tiles
// (segments of <= kSeg tiles); the left ones are drained per tile.
//
// Warp roles (448 threads, one CTA per SM, persistent over a contiguous tile
// range in row-block-major order, like seed_f64.cu):
//   warps 0-7   split: raw fp64 slots (one 16 KB TMA box, 16 rows i x 128
//               columns j, 128-byte swizzle; 8 KB boxes cap TMA near 4 TB/s,
//               tools/microbench/tma_order.cu) -> digit planes; all eight warps
//               share each slot
//   warps 8-11  drain: TMEM lane = output row; Horner over the 6 diagonals in
//               fp64 times the column weight 2^(eY + e_r - 52); right sums once
//               per segment (-> Rpart slot at the row block's end), left per tile
//               (-> Lpart): the partial layouts the fp64 tail reduces (TI = 128).
//   warp 12     producer: lane 0 TMA of the raw slots (no dependency wait), lane
//               1 bulk copies of the Khatri-Rao digit images (right per tile, left
//               per row block) after griddepcontrol.wait
//   warp 13     TMEM allocation and the MMA issue (one lane)
// The default for large fp64 gradients with 128 x 128 tiles that waste <= 10 %
// (c2, c3: 18-22 % faster seeds than the DMMA pass); CPDGPU_I8=1 / 0 forces it on /
// off (cpdgpu.cu, build_f64_geometry).  DESIGN.md section 5 has the numbers.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>
#include <cstring>

#include "kernels.h"

namespace cpdgpu {
namespace {

constexpr int kSplitW = 8, kDrainW = 4;
constexpr int kWProd = kSplitW + kDrainW;
constexpr int kWMma = kWProd + 1;
constexpr int kI8Threads = (kWMma + 1) * 32;
constexpr int kPl = 6;                       // digit planes
constexpr int kPlane = 128 * 128;            // bytes per digit plane of a tile (128 j x 128 i)
constexpr int kRawSlot = 16 * 128 * 8;       // 16 KB: one TMA box, 16 rows i x 128 columns j fp64
constexpr double kMagic = 4503599627370496.0 + 141289400074368.0;  // 2^52 + sum_{k<6} 128 256^k
// The right accumulators run over a row block's column tiles in TMEM (the right
// Khatri-Rao digits share one scale per column); a segment is drained at the end
// of the row block or after kSeg tiles (int32 headroom: |D| < 6 2^21 per tile).
constexpr int kSeg = 128;
__device__ __forceinline__ bool seg_end(int64_t tile, int k, int n, int64_t nCT, int pos) {
  return k == n - 1 || (tile + 1) / nCT != tile / nCT || pos == kSeg - 1;
}

// stacked N of Y plane a on a product with rank block n (M = 128 needs N % 16 == 0)
__host__ __device__ constexpr int stacked_n(int n, int a) { return ((n * (kPl - a)) + 15) / 16 * 16; }
// Digit image of an NP-row rank block: 6 planes of NP rows, zero rows up to the
// rounded-up stacked N the MMAs read (NP = 12: 80 rows)
__host__ __device__ constexpr int left_image_bytes(int NP) { return stacked_n(NP, 0) * 128; }
// accumulator columns of one product: diagonal d at d NP, plus the slack the
// rounded-up stacked N writes past diagonal 5 (never read)
__host__ __device__ constexpr int acc_cols(int NP) {
  int m = 0;
  for (int a = 0; a < kPl; ++a) m = (a * NP + stacked_n(NP, a)) > m ? (a * NP + stacked_n(NP, a)) : m;
  return m;
}

template <int N, int NL>
struct Cfg {
  static constexpr int kNR = NL < N ? NL : N;        // right rank block (the left one when smaller)
  static constexpr int kB = left_image_bytes(kNR);   // right Khatri-Rao digit image
  static constexpr int kBL = left_image_bytes(NL);   // left image
  static constexpr int kRaw = N == 32 ? 5 : 6;       // 16 KB TMA boxes (8 KB boxes cap TMA near 4 TB/s)
  // TMEM: right accumulators, then kLB left buffers
  static constexpr int kRS = acc_cols(kNR);
  static constexpr int kLS = acc_cols(NL);
  static constexpr int kLB = (kRS + 2 * kLS <= 512) ? 2 : 1;
  static constexpr int kCols = 512;
  static constexpr size_t kSmem = 1024 + static_cast<size_t>(kRaw) * kRawSlot + kPl * kPlane + kB + kBL + 256;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
// Barrier waits, two builds of the kernel (template WD).  WD = false (default): a
// plain spin on try_wait — any per-wait watchdog bookkeeping measured 5-30 % on
// this kernel (a spin counter 4.6 us at c2 / 40 us at c3, a globaltimer deadline
// or a try_wait suspend hint more), so the production path carries none.  WD =
// true (CPDGPU_WATCHDOG=1, and the forced-stall tests): every 1024th failed try
// reads the CTA's abort flag and a spin budget (~2^31 tries, seconds); past it the
// wait records the fault in the context's fault word (mapped host memory, reported
// by the next API return as CPDGPU_CUDA_ERROR), raises the abort flag, and every
// wait of the CTA returns at once: the kernel unwinds and exits normally instead of
// trapping (a trap poisons the caller's whole CUDA context).  With
// SeedI8Params::progress each warp posts its position (progress[cta][warp]) and the
// first stuck thread prints its CTA's table.
__shared__ int wd_abort;  // per CTA
__device__ __noinline__ void wd_fire(int code, int info, unsigned* progress, int* fault) {
  if (progress) {
    const volatile unsigned* t = progress + blockIdx.x * 16;
    printf("seed_i8 stuck: cta %d warp %d code %d info %d | warps: %u %u %u %u %u %u %u %u | %u %u %u %u | %u %u\n",
           blockIdx.x, threadIdx.x >> 5, code, info, t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[7], t[8], t[9], t[10],
           t[11], t[12], t[13]);
  }
  if (fault) atomicExch(fault, 1000 + code);
  *reinterpret_cast<volatile int*>(&wd_abort) = 1;
  __threadfence_block();
}
template <bool WD>
__device__ __forceinline__ void mbar_wait_wd(uint64_t* bar, uint32_t parity, int code, int info, unsigned* progress,
                                             int* fault, uint32_t limit) {
  if (WD && progress && (threadIdx.x & 31) == 0)
    *reinterpret_cast<volatile unsigned*>(progress + blockIdx.x * 16 + (threadIdx.x >> 5)) =
        static_cast<unsigned>(code * 100000 + info);
  uint32_t done = 0, spins = 0;
  while (true) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    if (!WD || ((++spins & 1023u) != 0u)) continue;
    if (*reinterpret_cast<volatile int*>(&wd_abort)) return;
    if (spins >= limit) {
      wd_fire(code, info, progress, fault);
      return;
    }
  }
}
template <bool WD>
__device__ __forceinline__ bool wd_aborted() {
  return WD && *reinterpret_cast<volatile int*>(&wd_abort) != 0;
}
// Unwinding after an abort: wait for async work that WAS issued (TMA / bulk copies,
// MMAs) to land before the CTA exits.  That work completes in bounded time, so this
// wait ignores the abort flag (and gives up after ~2^22 spins regardless).
__device__ __forceinline__ void mbar_drain_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0, spins = 0;
  while (!done && ++spins < (1u << 22))
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
}
#define WAIT(bar, par, code, info) mbar_wait_wd<WD>(bar, par, code, info, p.progress, p.fault, wd_limit)
#define TWAIT(idx, bar, par, code, info)                 \
  do {                                                   \
    const long long t0_ = p.trace ? clock64() : 0;       \
    WAIT(bar, par, code, info);                          \
    if (p.trace) tw[idx] += clock64() - t0_;             \
  } while (0)
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                       uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
// shared-memory matrix descriptor, 128-byte swizzle, sm_100 version bit
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFFu) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}
// instruction descriptor, kind::i8: s8 x s8 -> s32, M = m, N = n, A MN- or K-major
__device__ __forceinline__ uint32_t idesc_i8(bool a_mn, int n, int m) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile("{\n .reg .pred P;\n elect.sync _|P, 0xffffffff;\n selp.u32 %0, 1, 0, P;\n}\n" : "=r"(p));
  return p != 0;
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
// Diagonal sums (top first, weights 256^(5-d)) -> one fp64 value.  Adjacent
// diagonals combine in int32 where they cannot overflow (|D_0| < 2^20,
// |D_1| < 2^22, |D_2| < 2^23, |D_3| < 2^23 per tile), so four conversions
// replace six.
__device__ __forceinline__ double horner6(uint32_t d0, uint32_t d1, uint32_t d2, uint32_t d3, uint32_t d4,
                                          uint32_t d5) {
  const int c01 = static_cast<int>(d0) * 256 + static_cast<int>(d1);
  const int c23 = static_cast<int>(d2) * 256 + static_cast<int>(d3);
  double h = fma(static_cast<double>(c01), 65536.0, static_cast<double>(c23));
  h = fma(h, 256.0, static_cast<double>(static_cast<int>(d4)));
  return fma(h, 256.0, static_cast<double>(static_cast<int>(d5)));
}
// The same recombination for sums over many tiles (the right accumulators run
// over up to kSeg tiles, |D_0| < 2^27): every diagonal is converted on its own,
// since the int32 pairing D_0 * 256 + D_1 would overflow.
__device__ __forceinline__ double horner6_wide(uint32_t d0, uint32_t d1, uint32_t d2, uint32_t d3, uint32_t d4,
                                               uint32_t d5) {
  double h = static_cast<double>(static_cast<int>(d0));
  h = fma(h, 256.0, static_cast<double>(static_cast<int>(d1)));
  h = fma(h, 256.0, static_cast<double>(static_cast<int>(d2)));
  h = fma(h, 256.0, static_cast<double>(static_cast<int>(d3)));
  h = fma(h, 256.0, static_cast<double>(static_cast<int>(d4)));
  return fma(h, 256.0, static_cast<double>(static_cast<int>(d5)));
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;\n" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}
__device__ __forceinline__ void st_shared_v2(uint32_t addr, uint32_t a, uint32_t b) {
  asm volatile("st.shared.v2.b32 [%0], {%1, %2};\n" ::"r"(addr), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// Four values' digit bytes (u = fma(x, s, kMagic)) -> six words, word k = byte k
// of each value (value 0 in the low byte), as signed digits.
__device__ __forceinline__ void pack4(double x0, double x1, double x2, double x3, double s, uint32_t (&w)[6]) {
  const double u0 = fma(x0, s, kMagic), u1 = fma(x1, s, kMagic), u2 = fma(x2, s, kMagic), u3 = fma(x3, s, kMagic);
  const uint32_t l0 = __double2loint(u0), l1 = __double2loint(u1), l2 = __double2loint(u2), l3 = __double2loint(u3);
  const uint32_t h0 = __double2hiint(u0), h1 = __double2hiint(u1), h2 = __double2hiint(u2), h3 = __double2hiint(u3);
  const uint32_t t01 = prmt(l0, l1, 0x5140), t23 = prmt(l2, l3, 0x5140);
  const uint32_t s01 = prmt(l0, l1, 0x7362), s23 = prmt(l2, l3, 0x7362);
  const uint32_t g01 = prmt(h0, h1, 0x5140), g23 = prmt(h2, h3, 0x5140);
  w[0] = prmt(t01, t23, 0x5410) ^ 0x80808080u;
  w[1] = prmt(t01, t23, 0x7632) ^ 0x80808080u;
  w[2] = prmt(s01, s23, 0x5410) ^ 0x80808080u;
  w[3] = prmt(s01, s23, 0x7632) ^ 0x80808080u;
  w[4] = prmt(g01, g23, 0x5410) ^ 0x80808080u;
  w[5] = prmt(g01, g23, 0x7632) ^ 0x80808080u;
}

template <int N, int NL, bool WD>
__global__ void __launch_bounds__(kI8Threads, 1)
    seed_i8_kernel(const SeedI8Params p, const __grid_constant__ CUtensorMap ymap) {
  using C = Cfg<N, NL>;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cta = blockIdx.x;
  const int64_t a0 = static_cast<int64_t>(cta) * p.T / p.P;
  const int64_t a1 = static_cast<int64_t>(cta + 1) * p.T / p.P;
  const int n = static_cast<int>(a1 - a0);

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  unsigned char* raw = base;                               // [kRaw][16 KB]
  unsigned char* dig = raw + C::kRaw * kRawSlot;           // [6][128 j][128 B]
  unsigned char* rbuf = dig + kPl * kPlane;               // [kB] right Khatri-Rao digits (per tile)
  unsigned char* lbuf = rbuf + C::kB;                      // [kBL] left Khatri-Rao digits (per row block)
  uint64_t* bars = reinterpret_cast<uint64_t*>(lbuf + C::kBL);
  uint64_t* raw_full = bars;
  uint64_t* raw_empty = raw_full + C::kRaw;
  uint64_t* dig_full = raw_empty + C::kRaw;  // [4] row chunks 2 ks, 2 ks + 1 of the tile split
  uint64_t* dig_empty = dig_full + 4;        // [2] tile's digits consumed (rhalf: rows 0-63 / 64-127)
  uint64_t* rb_full = dig_empty + 2;
  uint64_t* rb_empty = rb_full + 1;
  uint64_t* lb_full = rb_empty + 1;
  uint64_t* lb_empty = lb_full + 1;
  uint64_t* accR_full = lb_empty + 1;
  uint64_t* accR_empty = accR_full + 1;
  uint64_t* accL_full = accR_empty + 1;  // [2]
  uint64_t* accL_empty = accL_full + 2;  // [2]
  uint64_t* fin = accL_empty + 2;        // every MMA of the CTA done (before TMEM is released)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(fin + 1);

  // spins before the watchdog fires: forced-stall tests and the debug table use short limits
  const uint32_t wd_limit = p.stall ? (1u << 16) : (p.progress ? (1u << 24) : (1u << 31));
  if (tid == 0) {
    wd_abort = 0;
    for (int s = 0; s < C::kRaw; ++s) {
      mbar_init(&raw_full[s], 1);
      mbar_init(&raw_empty[s], kSplitW);
    }
    for (int b = 0; b < 4; ++b) mbar_init(&dig_full[b], kSplitW);
    mbar_init(&dig_empty[0], 1);
    mbar_init(&dig_empty[1], 1);
    mbar_init(rb_full, 1);
    mbar_init(rb_empty, 1);
    mbar_init(lb_full, 1);
    mbar_init(lb_empty, 1);
    mbar_init(accR_full, 1);
    mbar_init(accR_empty, kDrainW);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accL_full[b], 1);
      mbar_init(&accL_empty[b], kDrainW);
    }
    mbar_init(fin, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == kWMma) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(C::kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (warp == kWProd && lane == 0)
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&ymap)));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t nCT = p.nCT;
  long long tw[4] = {0, 0, 0, 0};  // CPDGPU_SEED_TRACE: per-warp wait cycles
  const long long tstart = clock64();

  if (warp == kWProd) {
    // ------------------------------------------------------------------ producer
    // lane 0 streams Y (independent of the preceding kernels, no dependency wait);
    // lane 1 waits for the Khatri-Rao digit images (griddepcontrol.wait) and loads
    // them: right per tile, left per row block, each once the MMAs released the last.
    if (lane == 0) {
      const uint64_t pol_y = policy_evict_first();
      const int nslots = n * 8;
      // Slot q = (tile k, row chunk c): q = 8 k + c, one box of 16 rows i x 128
      // columns j (128-byte swizzle).  Boxes wholly outside Y are not requested
      // (the split reads them as zeros).
      const auto issued = [&](int q) {  // box q was requested from HBM
        const int64_t tile = a0 + (q >> 3), rb = tile / nCT, ct = tile - rb * nCT;
        return ct * 128 < p.K && rb * 128 + 16 * (q & 7) < p.J && !(p.stall && q == 0);
      };
      int qn = 0;  // boxes announced
      for (int q = 0; q < nslots; ++q) {
        const int k = q >> 3, c = q & 7, slot = q % C::kRaw;
        if (q >= C::kRaw) WAIT(&raw_empty[slot], ((q / C::kRaw) - 1) & 1, 3, q);
        if (wd_aborted<WD>()) break;  // watchdog: no new loads
        const int64_t tile = a0 + k, rb = tile / nCT, ct = tile - rb * nCT;
        const int j = static_cast<int>(ct * 128), i = static_cast<int>(rb * 128 + 16 * c);
        const bool live = j < p.K && i < p.J;
        mbar_arrive_tx(&raw_full[slot], live ? kRawSlot : 0);
        // p.stall (tests): the first box is announced but never requested, so its
        // consumers wait until the watchdog fires
        if (issued(q)) tma_2d(raw + slot * kRawSlot, &ymap, i, j, &raw_full[slot], pol_y);
        qn = q + 1;
      }
      if (wd_aborted<WD>())  // the last loads of each slot land before the CTA exits
        for (int q = qn > C::kRaw ? qn - C::kRaw : 0; q < qn; ++q)
          if (issued(q)) mbar_drain_wait(&raw_full[q % C::kRaw], (q / C::kRaw) & 1);
    } else if (lane == 1) {
      const uint64_t pol_k = policy_evict_last();
      pdl_wait();
      int m = 0, kn = 0;  // left / right image loads issued
      int64_t cur_rb = -1;
      for (int k = 0; k < n; ++k) {
        const int64_t tile = a0 + k, rb = tile / nCT, ct = tile - rb * nCT;
        if (k > 0) WAIT(rb_empty, (k - 1) & 1, 1, k);
        if (wd_aborted<WD>()) break;
        mbar_arrive_tx(rb_full, C::kB);
        bulk_load(rbuf, p.img_r + ct * C::kB, C::kB, rb_full, pol_k);
        kn = k + 1;
        if (rb != cur_rb) {
          if (m > 0) WAIT(lb_empty, (m - 1) & 1, 2, m);
          if (wd_aborted<WD>()) break;
          mbar_arrive_tx(lb_full, C::kBL);
          bulk_load(lbuf, p.img_l + rb * C::kBL, C::kBL, lb_full, pol_k);
          cur_rb = rb;
          ++m;
        }
      }
      if (wd_aborted<WD>()) {
        if (kn > 0) mbar_drain_wait(rb_full, (kn - 1) & 1);
        if (m > 0) mbar_drain_wait(lb_full, (m - 1) & 1);
      }
    }
  } else if (warp == kWMma) {
    // ------------------------------------------------------------------ MMA issue
    // The whole warp runs the loop (lane 0 waits, then the warp reconverges) and one
    // elected lane issues: descriptors and accumulator addresses are warp-uniform, so
    // each tcgen05.mma is one instruction on uniform registers.  Issued from inside an
    // `if (lane == 0)` the compiler wrapped every MMA in an elect / R2UR.BROADCAST
    // waterfall loop (~16 instructions), and the issuing thread, not the tensor pipe,
    // set the pace (115 cycles per MMA at c3, the MMA warp busy 72 % of the pass).
    {
      const uint32_t dg = smem_u32(dig), lb = smem_u32(lbuf), rbb = smem_u32(rbuf);
      // base descriptors; a byte offset d inside the buffers is added as d >> 4
      const uint64_t dAl = sdesc(dg, 16, 1024), dBl = sdesc(lb, 16, 1024);
      const uint64_t dAr = sdesc(dg, 16384, 1024), dBr = sdesc(rbb, 16, 1024);
      const bool run = !(p.knobs & 8);
      int64_t cur_rb = -1;
      int m = 0;
      int seg = 0, pos = 0;  // right-accumulator segment and position in it
      for (int k = 0; k < n; ++k) {
        if (WD && __shfl_sync(0xffffffffu, wd_aborted<WD>() ? 1 : 0, 0)) break;  // watchdog: no new MMAs (warp-uniform)
        const int64_t tile = a0 + k, rb = tile / nCT;
        const bool last_of_rb = (k == n - 1) || ((tile + 1) / nCT != rb);
        const bool send = seg_end(tile, k, n, nCT, pos);
        // left: M = 128 columns j, K = rows i, one 32-row step as soon as the split
        // has delivered its two 16-row chunks (overlaps this tile's split)
        const int lbk = k % C::kLB, lu = k / C::kLB;  // left buffer, its use
        if (lane == 0) {
          if (rb != cur_rb) TWAIT(3, lb_full, m & 1, 7, m);
          if (lu > 0) TWAIT(3, &accL_empty[lbk], (lu - 1) & 1, 8, k);
        }
        if (rb != cur_rb) {
          cur_rb = rb;
          ++m;
        }
        const uint32_t dL = tmem + C::kRS + lbk * C::kLS;
#pragma unroll 1
        for (int ks = 0; ks < 4; ++ks) {
          if (lane == 0) TWAIT(0, &dig_full[ks], k & 1, 4, k);
          __syncwarp();
          tc_fence_after();
          if (elect_one() && run) {
            const uint64_t a_ks = dAl + static_cast<uint64_t>((ks * 32) >> 4), b_ks = dBl + static_cast<uint64_t>((ks * 32) >> 4);
#pragma unroll
            for (int a = 0; a < kPl; ++a)
              mma_i8(dL + a * NL, a_ks + static_cast<uint64_t>((a * kPlane) >> 4), b_ks,
                     idesc_i8(false, stacked_n(NL, a), 128), (ks > 0 || a > 0) ? 1u : 0u);
          }
          __syncwarp();
          if (p.rhalf && ks == 1) {  // rows 0-63 are split: their right product, M = 64
            if (lane == 0) {
              TWAIT(1, rb_full, k & 1, 5, k);
              if (pos == 0 && seg > 0) TWAIT(2, accR_empty, (seg - 1) & 1, 6, seg);
            }
            __syncwarp();
            tc_fence_after();
            if (elect_one()) {
              if (run) {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
#pragma unroll
                  for (int a = 0; a < kPl; ++a)
                    mma_i8(tmem + a * C::kNR, dAr + static_cast<uint64_t>((a * kPlane + kk * 4096) >> 4),
                           dBr + static_cast<uint64_t>((kk * 32) >> 4), idesc_i8(true, stacked_n(C::kNR, a), 64),
                           (kk > 0 || a > 0 || pos > 0) ? 1u : 0u);
              }
              umma_commit(&dig_empty[0]);  // every MMA over rows 0-63 (left ks 0, 1 and this half) is issued
            }
            __syncwarp();
          }
        }
        // right: M = rows i, K = the tile's 128 columns (rows of the plane).  rhalf: as two
        // M = 64 row halves, rows 0-63 issued inside the loop above after ks = 1 and rows
        // 64-127 here, so only the second half runs after the split and the next tile's
        // split of rows 0-63 never waits for it.  Otherwise one M = 128 product here.
        if (!p.rhalf) {
          if (lane == 0) {
            TWAIT(1, rb_full, k & 1, 5, k);
            if (pos == 0 && seg > 0) TWAIT(2, accR_empty, (seg - 1) & 1, 6, seg);
          }
          __syncwarp();
          tc_fence_after();
        }
        if (elect_one()) {
          if (run) {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
#pragma unroll
              for (int a = 0; a < kPl; ++a) {
                if (p.rhalf)  // rows 64-127: the second 64 bytes of the plane rows, TMEM lanes 16-31 of each quarter
                  mma_i8(tmem + (16u << 16) + a * C::kNR, dAr + static_cast<uint64_t>((a * kPlane + ks * 4096 + 64) >> 4),
                         dBr + static_cast<uint64_t>((ks * 32) >> 4), idesc_i8(true, stacked_n(C::kNR, a), 64),
                         (ks > 0 || a > 0 || pos > 0) ? 1u : 0u);
                else
                  mma_i8(tmem + a * C::kNR, dAr + static_cast<uint64_t>((a * kPlane + ks * 4096) >> 4),
                         dBr + static_cast<uint64_t>((ks * 32) >> 4), idesc_i8(true, stacked_n(C::kNR, a), 128),
                         (ks > 0 || a > 0 || pos > 0) ? 1u : 0u);
              }
          }
          if (send) umma_commit(accR_full);
          umma_commit(rb_empty);
          umma_commit(&dig_empty[p.rhalf ? 1 : 0]);
          umma_commit(&accL_full[lbk]);
          if (last_of_rb) umma_commit(lb_empty);
        }
        __syncwarp();
        if (send) {
          ++seg;
          pos = 0;
        } else {
          ++pos;
        }
      }
      if (elect_one()) umma_commit(fin);  // TMEM is released only after every issued MMA completed
      __syncwarp();
      mbar_drain_wait(fin, 0);
    }
    __syncwarp();
  } else if (warp < kSplitW) {
    // ------------------------------------------------------------------ split
    // All eight warps share every raw slot (16 rows i x 128 columns j), so each
    // slot's fills are observed in order by all its waiters.  Thread = (column j,
    // half hh of the 16-row chunk): 8 values -> 8 bytes of each digit plane in the
    // half-tile buffer of column j; a half-warp stores 128 conflict-free bytes.
    const int j = 16 * warp + (lane & 7) + 8 * (lane >> 4), hh = (lane >> 3) & 1;
    // no griddepcontrol.wait: the split reads only Y and the tensor's scale record,
    // which is written before the gradient's launches (bind_i8), and shared memory
    if (p.progress && lane == 0) reinterpret_cast<volatile unsigned*>(p.progress)[cta * 16 + warp] = 2;
    const double sy = p.yscale[0];
    const uint32_t row0 = smem_u32(dig) + j * 128 + 8 * hh;
    for (int k = 0; k < n; ++k) {
      const int64_t tile = a0 + k, rb = tile / nCT, ct = tile - rb * nCT;
      const bool col_live = ct * 128 < p.K;
#pragma unroll 1
      for (int ks = 0; ks < 4; ++ks) {  // row chunks c = 2 ks, 2 ks + 1 together (two slots in flight)
        double2 v[2][4];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = 2 * ks + e, q = k * 8 + c, slot = q % C::kRaw;
          TWAIT(0, &raw_full[slot], (q / C::kRaw) & 1, 9, q);
          const unsigned char* box = raw + slot * kRawSlot + j * 128;
          const bool rd = col_live && rb * 128 + 16 * c < p.J && !(p.knobs & 2);  // the box was requested
#pragma unroll
          for (int t = 0; t < 4; ++t)
            v[e][t] = rd ? *reinterpret_cast<const double2*>(box + (((4 * hh + t) ^ (j & 7)) << 4))
                         : make_double2(0.0, 0.0);
        }
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&raw_empty[(k * 8 + 2 * ks) % C::kRaw]);
          mbar_arrive(&raw_empty[(k * 8 + 2 * ks + 1) % C::kRaw]);
        }
        uint32_t w[2][2][6];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          pack4(v[e][0].x, v[e][0].y, v[e][1].x, v[e][1].y, sy, w[e][0]);
          pack4(v[e][2].x, v[e][2].y, v[e][3].x, v[e][3].y, sy, w[e][1]);
        }
        // the planes' rows 0-63 (ks 0, 1) / 64-127 (ks 2, 3) are free once the last tile's MMAs over them are done
        if (k > 0 && (ks == 0 || (p.rhalf && ks == 2))) TWAIT(1, &dig_empty[ks >> 1], (k - 1) & 1, 10, k);
        if (!(p.knobs & 1)) {  // experiment knob: stream only
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const uint32_t row = row0 + (((2 * ks + e) ^ (j & 7)) << 4);
#pragma unroll
            for (int kk = 0; kk < kPl; ++kk)  // byte k -> top-first plane 5 - k
              st_shared_v2(row + (kPl - 1 - kk) * kPlane, w[e][0][kk], w[e][1][kk]);
          }
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // the left MMAs of step ks may go
        __syncwarp();
        if (lane == 0) mbar_arrive(&dig_full[ks]);
      }
    }
  } else {
    // ------------------------------------------------------------------ drain
    const int qd = warp & 3, row = 32 * qd + lane;
    // rhalf: the M = 64 right halves keep row i = 64 h + 16 q + l in TMEM lane 32 q + 16 h + l
    const int rrow = p.rhalf ? 64 * (lane >> 4) + 16 * qd + (lane & 15) : row;
    const uint32_t lanes = static_cast<uint32_t>(32 * qd) << 16;
    if (p.progress && lane == 0) reinterpret_cast<volatile unsigned*>(p.progress)[cta * 16 + warp] = 1;
    pdl_wait();
    if (p.progress && lane == 0) reinterpret_cast<volatile unsigned*>(p.progress)[cta * 16 + warp] = 2;
    double acc[N];
#pragma unroll
    for (int r = 0; r < N; ++r) acc[r] = 0.0;
    const int64_t rb0 = a0 / nCT;
    int seg = 0, pos = 0;
    for (int k = 0; k < n; ++k) {
      const int64_t tile = a0 + k, rb = tile / nCT, ct = tile - rb * nCT;
      const bool last_of_rb = (k == n - 1) || ((tile + 1) / nCT != rb);
      const bool send = seg_end(tile, k, n, nCT, pos);
      pos = send ? 0 : pos + 1;
      // right: the segment's integer sums, once at its end (one scale per column)
      if (send) {
      TWAIT(0, accR_full, seg & 1, 11, seg);
      ++seg;
      __syncwarp();  // tcgen05.ld is .sync.aligned: reconverge after the spin
      tc_fence_after();
      const double* wr = p.w_r + ct * N;
#pragma unroll
      for (int rc = 0; rc < (C::kNR + 7) / 8; ++rc) {
        if (rc * 8 >= p.R || (p.knobs & 4)) break;  // warp-uniform: columns past the rank are zero
        uint32_t d[kPl][8];
#pragma unroll
        for (int dd = 0; dd < kPl; ++dd) tmem_ld8(tmem + lanes + dd * C::kNR + rc * 8, d[dd]);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const double h = horner6_wide(d[0][e], d[1][e], d[2][e], d[3][e], d[4][e], d[5][e]);
          acc[rc * 8 + e] = fma(h, __ldg(wr + rc * 8 + e), acc[rc * 8 + e]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(accR_empty);
      }
      if (last_of_rb) {
        double* dst = p.Rpart + (static_cast<int64_t>(cta) * p.slots + (rb - rb0)) * p.RP * 128;
#pragma unroll
        for (int r = 0; r < N; ++r) {
          if (r < p.RP) dst[r * 128 + rrow] = acc[r];
          acc[r] = 0.0;
        }
      }
      // left: this tile's columns, complete over its 128 rows
      const int lbk = k % C::kLB, lu = k / C::kLB;
      TWAIT(1, &accL_full[lbk], lu & 1, 12, k);
      __syncwarp();  // tcgen05.ld is .sync.aligned: reconverge after the spin
      tc_fence_after();
      const double* wl = p.w_l + rb * N;
      const int64_t j = ct * 128 + row;  // M = 128: TMEM lane = column
      double* lout = p.Lpart + (p.lred ? 0 : rb) * static_cast<int64_t>(p.R) * p.K + j;
#pragma unroll
      for (int rc = 0; rc < (NL + 7) / 8; ++rc) {
        if (rc * 8 >= p.R || (p.knobs & 4)) break;
        uint32_t d[kPl][8];
#pragma unroll
        for (int dd = 0; dd < kPl; ++dd) tmem_ld8(tmem + lanes + C::kRS + lbk * C::kLS + dd * NL + rc * 8, d[dd]);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const double h = horner6(d[0][e], d[1][e], d[2][e], d[3][e], d[4][e], d[5][e]);
          const int r = rc * 8 + e;
          if (r < p.R && j < p.K) {
            if (p.lred)
              atomicAdd(lout + static_cast<int64_t>(r) * p.K, h * __ldg(wl + r));  // red.global.add.f64 (L2)
            else
              lout[static_cast<int64_t>(r) * p.K] = h * __ldg(wl + r);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&accL_empty[lbk]);
    }
  }
  if (p.trace && lane == 0) {
    unsigned long long* t = p.trace + (static_cast<int64_t>(cta) * 14 + warp) * 6;
    for (int i = 0; i < 4; ++i) t[i] = static_cast<unsigned long long>(tw[i]);
    t[4] = static_cast<unsigned long long>(clock64() - tstart);
    t[5] = static_cast<unsigned long long>(n);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kWMma) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(C::kCols));
  }
}

// Khatri-Rao digit images of both sides in one launch, straight from the sorted
// factors: CTA = 128-row tile (right tiles first, then left), thread = (row q, 8
// rank columns).  Every tile of a side shares one scale per column, from the
// product of the factor column maxima (max |KR(:, r)| = prod_m max_i |A_m(i, r)|:
// every index combination occurs), so no pass over the Khatri-Rao rows is needed.
// Output per tile: [6 planes][N rank rows][128 bytes of the tile's rows, 128-byte
// swizzle] and the column weights 2^(eY + e_r - 52) (0: all-zero column, NaN:
// non-finite factor entry).
template <int N, int NL>
__global__ void __launch_bounds__(N * 16) kr_digits_kernel(const KRSpec right, int64_t Lr, const KRSpec left,
                                                           int64_t Ll, int R, int64_t nCT, const double* yscale,
                                                           unsigned char* img_r, double* w_r, unsigned char* img_l,
                                                           double* w_l, int64_t numel, double budget, int* fault) {
  __shared__ double sc[N];
  __shared__ unsigned long long mbits[kMaxModes * N];
  __shared__ double ssq[kMaxModes * N];  // tile 0 of each side: column sums of squares (error-budget check)
  __shared__ __align__(16) unsigned char im[kPl * N * 128 + 1024];
  const bool is_right = blockIdx.x < nCT;
  constexpr int NR = NL < N ? NL : N;
  const int NP = is_right ? NR : NL;  // rank rows per digit plane of this side's image
  const int IB = left_image_bytes(NP);
  const KRSpec& spec = is_right ? right : left;
  const int64_t L = is_right ? Lr : Ll, tile = is_right ? blockIdx.x : blockIdx.x - nCT;
  unsigned char* img = is_right ? img_r : img_l;
  double* w = is_right ? w_r : w_l;
  for (int e = threadIdx.x; e < kMaxModes * N; e += blockDim.x) {
    mbits[e] = 0ull;
    ssq[e] = 0.0;
  }
  const bool check = tile == 0 && fault != nullptr;
  for (int e = kPl * NP * 128 + threadIdx.x; e < IB; e += blockDim.x) im[e] = 0;  // zero rows past the planes
  pdl_trigger();  // the seed may launch now: its Y stream does not depend on this kernel
  pdl_wait();     // the sorted factors come from the prologue
  __syncthreads();
  {  // factor column maxima, all threads: column r, rows i = part (mod parts)
    const int r = threadIdx.x % N, part = threadIdx.x / N, parts = blockDim.x / N;
    for (int m = 0; m < spec.n; ++m) {
      double cm = 0.0;
      const int64_t I = spec.dims[m];
      if (r < R)
        for (int64_t i0 = part; i0 < I; i0 += 8 * static_cast<int64_t>(parts)) {
          double a[8];  // eight independent loads in flight
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int64_t i = i0 + u * static_cast<int64_t>(parts);
            a[u] = i < I ? fabs(__ldg(spec.A[m] + i + I * r)) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) cm = (a[u] > cm || a[u] != a[u]) ? a[u] : cm;  // NaN sticks
          if (check) {
            double q2 = 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u) q2 += a[u] * a[u];
            atomicAdd(&ssq[m * N + r], q2);
          }
        }
      atomicMax(&mbits[m * N + r], static_cast<unsigned long long>(__double_as_longlong(cm)));
    }
  }
  __syncthreads();
  if (check && threadIdx.x < R && threadIdx.x < N) {
    // the call's error budget (cpdgpu.cu i8_factors_ok_*): prod_m max / rms of this
    // side's column against 2^11 mean|Y| / max|Y|; a device-form call whose factors
    // were not checked on the host fails loudly here instead of returning a result
    // outside the 1e-10 gate (the next call of the plan runs the DMMA pass)
    const int r = threadIdx.x;
    double ratio = 1.0;
    for (int m = 0; m < spec.n; ++m) {
      const double mxm = __longlong_as_double(static_cast<long long>(mbits[m * N + r]));
      if (!(mxm > 0.0)) {
        ratio = 0.0;
        break;
      }
      ratio *= mxm / sqrt(ssq[m * N + r] / static_cast<double>(spec.dims[m]));
    }
    const double limit = yscale[2] > 0.0 ? budget * (yscale[3] / static_cast<double>(numel)) / yscale[2] : budget;
    if (isfinite(ratio) && ratio > limit) atomicExch(fault, 3000);
  }
  if (threadIdx.x < N) {
    const int r = threadIdx.x;
    double mx = 1.0;
    for (int m = 0; m < spec.n; ++m) mx *= __longlong_as_double(static_cast<long long>(mbits[m * N + r]));
    if (r >= R || mx == 0.0) {
      sc[r] = 0.0;
      w[tile * N + r] = 0.0;
    } else if (!isfinite(mx)) {
      sc[r] = 0.0;
      w[tile * N + r] = __longlong_as_double(0x7ff8000000000000ll);
    } else {
      int e;
      frexp(mx, &e);
      sc[r] = ldexp(1.0, 46 - e);
      w[tile * N + r] = ldexp(1.0, e + static_cast<int>(yscale[1]) - 52);
    }
  }
  __syncthreads();
  const int q = threadIdx.x & 127, r0 = (threadIdx.x >> 7) * 8;
  const int64_t row = tile * 128 + q;
  // the row's mixed-radix digits (first mode fastest, kron.cpp:54-68), once for all columns
  int64_t off_m[kMaxModes];
  {
    int64_t rem = row;
#pragma unroll 1
    for (int m = 0; m < spec.n; ++m) {
      off_m[m] = rem % spec.dims[m];
      rem /= spec.dims[m];
    }
  }
  double xs[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) xs[e] = (row < L && r0 + e < R) ? 1.0 : 0.0;
#pragma unroll 1
  for (int m = 0; m < spec.n; ++m) {  // eight independent loads per mode
    const double* a = spec.A[m] + off_m[m];
    const int64_t I = spec.dims[m];
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (xs[e] != 0.0) xs[e] *= __ldg(a + I * (r0 + e));
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int r = r0 + e;
    const double x = xs[e];
    const double u = fma(isfinite(x) ? x : 0.0, sc[r], kMagic);
    const uint32_t lo = __double2loint(u), hi = __double2hiint(u);
    if (r < NP) {
#pragma unroll
      for (int k = 0; k < kPl; ++k) {
        const uint32_t b = (k < 4 ? (lo >> (8 * k)) : (hi >> (8 * (k - 4)))) & 0xFFu;
        const int g = (kPl - 1 - k) * NP + r;  // row in the image: the swizzle phase is g mod 8
        im[g * 128 + ((((q >> 4) ^ (g & 7))) << 4) + (q & 15)] = static_cast<unsigned char>(b ^ 0x80u);
      }
    }
  }
  __syncthreads();
  uint4* dst = reinterpret_cast<uint4*>(img + tile * IB);
  const uint4* src = reinterpret_cast<const uint4*>(im);
  for (int e = threadIdx.x; e < IB / 16; e += N * 16) dst[e] = src[e];
}

// max |Y| -> scale record: [0] 2^(46 - eY), [1] eY, [2] max |Y| (NaN when Y has
// one), [3] sum |Y| (range guard).  Per-block results land in fixed slots and
// one thread folds them in block order, so the record (and with it the seed
// path chosen from it) is bitwise reproducible.
__global__ void y_amax_kernel(const double* y, int64_t n, unsigned long long* bmax, double* bsum) {
  __shared__ unsigned long long wm[32];
  __shared__ double ws[32];
  unsigned long long m = 0;
  double a = 0.0;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double v = fabs(y[e]);
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
    m = b > m ? b : m;  // NaN bit patterns sort above +inf
    a += v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(0xffffffffu, m, o);
    m = t > m ? t : m;
    a += __shfl_xor_sync(0xffffffffu, a, o);
  }
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    wm[warp] = m;
    ws[warp] = a;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < nw; ++w) {
      m = wm[w] > m ? wm[w] : m;
      a += ws[w];
    }
    bmax[blockIdx.x] = m;
    bsum[blockIdx.x] = a;
  }
}
// Exponent from frexp for every finite max > 0; a max whose scale 2^(46 - eY)
// leaves the double range (or a non-finite max / sum) is recorded as is, and the
// host range guard then keeps the tensor on the fp64 DMMA pass.
// One warp, fixed order (lane l sums blocks l, l + 32, ..., then a fixed shuffle tree):
// the record is bitwise reproducible, and the block partials are read 32 at a time
// (one thread walking them serially took 78 us at c2, per tensor version).
__global__ void __launch_bounds__(32) y_scale_final_kernel(const unsigned long long* bmax, const double* bsum, int nb,
                                                           double* out) {
  unsigned long long mb = 0;
  double a = 0.0;
  for (int b = threadIdx.x; b < nb; b += 32) {
    mb = bmax[b] > mb ? bmax[b] : mb;
    a += bsum[b];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(0xffffffffu, mb, o);
    mb = t > mb ? t : mb;
    a += __shfl_xor_sync(0xffffffffu, a, o);
  }
  if (threadIdx.x != 0) return;
  const double m = __longlong_as_double(static_cast<long long>(mb));
  int e = 0;
  if (m > 0.0 && isfinite(m)) frexp(m, &e);
  out[0] = ldexp(1.0, 46 - e);
  out[1] = static_cast<double>(e);
  out[2] = m;
  out[3] = a;
}

}  // namespace

template <int N, int NL>
void launch_one_i8(const SeedI8Params& p, const CUtensorMap* ymap, cudaStream_t s) {
  using C = Cfg<N, NL>;
  if (p.watchdog) {
    static unsigned long long configured = 0;
    set_smem_attr(seed_i8_kernel<N, NL, true>, C::kSmem, configured);
    launch_k(seed_i8_kernel<N, NL, true>, dim3(p.P), dim3(kI8Threads), C::kSmem, s, pdl_enabled(), p, *ymap);
    return;
  }
  static unsigned long long configured = 0;
  set_smem_attr(seed_i8_kernel<N, NL, false>, C::kSmem, configured);
  launch_k(seed_i8_kernel<N, NL, false>, dim3(p.P), dim3(kI8Threads), C::kSmem, s, pdl_enabled(), p, *ymap);
}

int i8_left_block(int N, int R) { return (N == 32 && R <= 24) ? 24 : ((N == 16 && R <= 12) ? 12 : N); }
size_t i8_left_image_bytes(int NL) { return static_cast<size_t>(left_image_bytes(NL)); }
size_t i8_right_image_bytes(int N, int NL) { return static_cast<size_t>(left_image_bytes(NL < N ? NL : N)); }

int launch_seed_i8(const SeedI8Params& p, const CUtensorMap* ymap, cudaStream_t s) {
  if (p.N == 16 && p.NL == 12)
    launch_one_i8<16, 12>(p, ymap, s);
  else if (p.N == 16)
    launch_one_i8<16, 16>(p, ymap, s);
  else if (p.NL == 24)
    launch_one_i8<32, 24>(p, ymap, s);
  else
    launch_one_i8<32, 32>(p, ymap, s);
  return 1;
}

int launch_kr_digits(const KRSpec& right, int64_t Kp, const KRSpec& left, int64_t Jp, int R, int N, int NL,
                     const double* yscale, void* img_r, double* w_r, void* img_l, double* w_l, int64_t numel,
                     double budget, int* fault, cudaStream_t s) {
  const int64_t nCT = ceil_div(Kp, 128), nRB = ceil_div(Jp, 128);
  const dim3 grid(static_cast<unsigned>(nCT + nRB));
  auto* ir = static_cast<unsigned char*>(img_r);
  auto* il = static_cast<unsigned char*>(img_l);
  if (N == 16 && NL == 12)
    launch_k(kr_digits_kernel<16, 12>, grid, dim3(256), 0, s, pdl_enabled(), right, Kp, left, Jp, R, nCT, yscale, ir,
             w_r, il, w_l, numel, budget, fault);
  else if (N == 16)
    launch_k(kr_digits_kernel<16, 16>, grid, dim3(256), 0, s, pdl_enabled(), right, Kp, left, Jp, R, nCT, yscale, ir,
             w_r, il, w_l, numel, budget, fault);
  else if (NL == 24)
    launch_k(kr_digits_kernel<32, 24>, grid, dim3(512), 0, s, pdl_enabled(), right, Kp, left, Jp, R, nCT, yscale, ir,
             w_r, il, w_l, numel, budget, fault);
  else
    launch_k(kr_digits_kernel<32, 32>, grid, dim3(512), 0, s, pdl_enabled(), right, Kp, left, Jp, R, nCT, yscale, ir,
             w_r, il, w_l, numel, budget, fault);
  return 1;
}

int y_scale_f64_blocks(int64_t n, int num_sms) {
  int64_t blocks = ceil_div(n, 256);
  if (blocks > 8LL * num_sms) blocks = 8LL * num_sms;
  return blocks < 1 ? 1 : static_cast<int>(blocks);
}

int launch_y_scale_f64(const double* y, int64_t n, void* scratch, double* out, int num_sms, cudaStream_t s) {
  const int blocks = y_scale_f64_blocks(n, num_sms);
  unsigned long long* bmax = static_cast<unsigned long long*>(scratch);
  double* bsum = reinterpret_cast<double*>(bmax + blocks);
  y_amax_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(y, n, bmax, bsum);
  y_scale_final_kernel<<<1, 32, 0, s>>>(bmax, bsum, blocks, out);
  return 2;
}

// int8 factor-range guard on device factors: one block per (side, rank column);
// sets *flag when prod_m max_i |A_m[i, r]| / rms_i A_m[i, r] exceeds `limit` or a
// factor entry is not finite (the host then runs the DMMA pass).
__global__ void __launch_bounds__(128) i8_factor_guard_kernel(const KRSpec right, const KRSpec left, int R,
                                                              double limit, int* flag) {
  const int side = blockIdx.x / R, r = blockIdx.x % R;
  const KRSpec& sp = side == 0 ? right : left;
  __shared__ double rm[4], rs[4];
  double ratio = 1.0;
  bool bad = false;
  for (int m = 0; m < sp.n; ++m) {
    const int64_t I = sp.dims[m];
    double mx = 0.0, ss = 0.0;
    for (int64_t i = threadIdx.x; i < I; i += blockDim.x) {
      const double a = fabs(sp.A[m][i + I * r]);
      mx = a > mx || a != a ? a : mx;  // NaN wins
      ss += a * a;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double t = __shfl_xor_sync(0xffffffffu, mx, o);
      mx = t > mx || t != t ? t : mx;
      ss += __shfl_xor_sync(0xffffffffu, ss, o);
    }
    if ((threadIdx.x & 31) == 0) {
      rm[threadIdx.x >> 5] = mx;
      rs[threadIdx.x >> 5] = ss;
    }
    __syncthreads();
    mx = 0.0;
    ss = 0.0;
    for (int w = 0; w < 4; ++w) {
      mx = rm[w] > mx || rm[w] != rm[w] ? rm[w] : mx;
      ss += rs[w];
    }
    __syncthreads();
    if (!isfinite(mx) || !isfinite(ss)) bad = true;
    else if (mx == 0.0) ratio = 0.0;
    else ratio *= mx / sqrt(ss / static_cast<double>(I));
  }
  if (threadIdx.x == 0 && (bad || !(ratio <= limit))) atomicOr(flag, 1);
}

int launch_i8_factor_guard(const KRSpec& right, const KRSpec& left, int R, double limit, int* flag, cudaStream_t s) {
  i8_factor_guard_kernel<<<2 * R, 128, 0, s>>>(right, left, R, limit, flag);
  return 1;
}

// Column-padded copy of an fp64 view (J rows -> leading dimension LD, rows J..LD-1
// zero): 128-byte column starts for the int8 pass's 16-row boxes (c3's 2744-row
// columns start 64 bytes off a line every other column).  Two doubles per thread.
__global__ void pad_rows_f64_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t J, int64_t LD,
                                    int64_t K) {
  const int64_t half = LD / 2;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < half * K;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = e / half, i = 2 * (e - j * half);
    const double* col = src + j * J;
    double2 v;
    v.x = i < J ? __ldcs(col + i) : 0.0;
    v.y = i + 1 < J ? __ldcs(col + i + 1) : 0.0;
    __stcs(reinterpret_cast<double2*>(dst + j * LD + i), v);
  }
}

int launch_pad_rows_f64(const double* src, double* dst, int64_t J, int64_t LD, int64_t K, int num_sms,
                        cudaStream_t s) {
  pad_rows_f64_kernel<<<num_sms * 8, 256, 0, s>>>(src, dst, J, LD, K);
  return 1;
}

}  // namespace cpdgpu
