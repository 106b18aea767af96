// seed_f32f.cu — both split-point seeds of an fp32 tensor in ONE pass over Y on
// the 5th-generation tensor cores (tcgen05.mma kind::f16, accumulators in TMEM).
//
//   right  Rs[i, r] = sum_j Y[i + J j] KR(p+1..N)[j, r]   (mttkrp.cpp:149-163)
//   left   Ls[j, r] = sum_i Y[i + J j] KR(1..p)[i, r]     (mttkrp.cpp:195-210)
//
// Both reference products read the same J_p x K_p view of Y (mttkrp.cpp:160,
// 207); here every 128 i x 64 j tile of it is read from HBM once, split once
// into fp16 hi / lo planes in shared memory, and feeds both products:
//
//   right  D_R[i][r]  += Y[i][j]   KRr[j][r]   A = Y plane (smem, MN-major: i
//                                              contiguous), B = KRr tile (smem,
//                                              K-major), M = 128 i, N = 64 r
//   left   D_L[m][j]  += KRl^T[m][i] Y[i][j]   A = KRl^T (TMEM: lane m = 2 r
//                                              holds the hi part of rank r,
//                                              lane 2 r + 1 the lo part), B =
//                                              the same Y plane read K-major,
//                                              M = 128, N = 64 j
//
// fp32 accuracy from fp16 tensor cores: x = x_hi + x_lo (22 significant bits);
// right: Y_hi KR_hi + Y_hi KR_lo + Y_lo KR_hi into one accumulator; left: both
// Y planes against the interleaved [KR_hi; KR_lo] rows, the lane pairs added
// at the drain with one shuffle (the extra lo * lo term only adds accuracy).
// Y and every Khatri-Rao column are scaled by powers of two into [-1, 1] first
// (exact).
//
// Work: unit = (band of kA = 3 row tiles, one 64-column tile); a CTA walks a
// contiguous range of units band-major, so its three right accumulators (one
// per row tile) persist across a band's columns while the left accumulator
// covers 384 rows of one column tile per unit:
//   right: the fp32 TMEM accumulators are drained every `window` units (tensor-
//          core fp32 accumulation truncates: 256-column windows keep ~1e-6) into
//          fp32 registers of the drain warps, and written once per band segment
//          as an fp64 partial block (a few slots per row tile: tail reduction).
//   left:  one fp32 partial [64 r][64 j] per unit, summed over the bands in
//          fp64 by the tail (kOpReduceLeft32).
//
// Pipeline (one CTA per SM, persistent, 512 threads):
//   warp 12      producer: TMA of the fp32 Y tiles into a 4-slot landing ring,
//                bulk copy of the KRr tiles
//   warps 0-3    split: thread = row pair x column half; reads its 64 fp32
//                values, frees the landing slot, converts, and writes fp16 hi /
//                lo words into a 2-slot plane ring (128-byte-swizzled operand
//                layout).  The landing ring holds 128 KB of loads in flight and
//                is released right after the split reads it, not after the MMAs.
//   warp 13      MMAs: the whole warp waits, one elected lane issues (uniform
//                operands: no per-instruction waterfall), commits free slots
//   warps 4-11   drains: TMEM lane quarter w % 4 x rank / column half: the
//                right windows, the left partial per unit, the band's KRl^T image
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include "kernels.h"

namespace cpdgpu {
namespace {

constexpr int kTI = 128;                      // tile rows (i) = right MMA M
constexpr int kTJ = 64;                       // tile columns (j) = left MMA N
constexpr int kA = 3;                         // row tiles per band
constexpr int kRP = 64;                       // rank columns (right MMA N)
constexpr int kNL = 4;                        // fp32 landing slots (loads in flight)
constexpr int kNP = 2;                        // fp16 plane slots (split -> MMA)
constexpr int kYBytes = kTI * kTJ * 4;        // 32 KB fp32 tile
constexpr int kPlane = kTI * kTJ * 2;         // 16 KB fp16 plane: [i half][64 j][128 B]
constexpr int kKRBytes = 2 * kTJ * kRP * 2;   // 16 KB KRr tile: [hi | lo][64 r][64 j] (kr_split)
constexpr int kSplitWarps = 4, kDrainWarps = 8;  // drains: lane quarter x column half
constexpr int kWDrain0 = kSplitWarps, kWProd = kSplitWarps + kDrainWarps, kWMma = kWProd + 1;
constexpr int kThreads = (kWMma + 3) * 32;  // + 2 idle warps: 16 warps keep 128 registers per thread
constexpr uint32_t kColR = 0;                 // D_R[t]: columns [64 t, 64 t + 64)
constexpr uint32_t kColK = kA * kRP;          // KRl^T[t]: [192 + 64 t, +64)
constexpr uint32_t kColL = 2 * kA * kRP;      // D_L[lb]: [384 + 64 lb, +64)
constexpr int kTmemCols = 512;
constexpr int kOffPlanes = kNL * kYBytes;
constexpr int kOffKR = kOffPlanes + kNP * 2 * kPlane;
constexpr int kOffBars = kOffKR + 2 * kKRBytes;
constexpr int kSmem = 1024 + kOffBars + 512 + kRP * 8;

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
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(tx)
               : "memory");
}
// Barrier waits.  The plain spin (mbar_wait) everywhere by default; the image
// kernel also has a watchdog build (template WD, CPDGPU_WATCHDOG=1 and the
// forced-stall tests): every 1024th failed try of a bounded wait reads the CTA's
// abort flag and a spin budget (~2^31 tries); past it the wait records the fault
// in the context's fault word and raises the abort flag, after which every
// bounded wait returns at once, so a broken pipeline unwinds and exits instead
// of hanging the GPU or trapping.  Any per-wait bookkeeping measured 1.5-8 % at
// c5 (a spin counter, a globaltimer deadline, a try_wait suspend hint), so the
// production build carries none.
__shared__ int wd_abort;
__shared__ int* wd_fault;
__shared__ uint32_t wd_limit;
__device__ __forceinline__ void wd_init(int* fault, int stall) {
  wd_abort = 0;
  wd_fault = fault;
  wd_limit = stall ? (1u << 16) : (1u << 31);
}
__device__ __noinline__ void wd_fire() {
  if (wd_fault) atomicExch(wd_fault, 2000);
  *reinterpret_cast<volatile int*>(&wd_abort) = 1;
  __threadfence_block();
}
template <bool WD = false>
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
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
    if (spins >= wd_limit) {
      wd_fire();
      return;
    }
  }
}
template <bool WD>
__device__ __forceinline__ bool wd_aborted() {
  return WD && *reinterpret_cast<volatile int*>(&wd_abort) != 0;
}
// Unwinding after an abort: issued async work (bulk copies, MMAs) lands before the
// CTA exits; it completes in bounded time, so this wait ignores the abort flag.
__device__ __forceinline__ void mbar_drain_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0, spins = 0;
  while (!done && ++spins < (1u << 22))
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
}
// Unbounded wait for register-heavy warps (the drains, whose fp32 window sums fill
// the register file: the watchdog's loop state there cost spills and ~0.7 ms at
// c5).  Their waits are released after an abort by the MMA warp (see its tail).
__device__ __forceinline__ void mbar_wait_plain(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile("{\n .reg .pred P;\n elect.sync _|P, 0xffffffff;\n selp.u32 %0, 1, 0, P;\n}\n" : "=r"(p));
  return p != 0;
}
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
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                            uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
// tcgen05 shared-memory matrix descriptor (sm_100 version 1): start, leading / stride
// byte offsets, layout type 2 = 128-byte swizzle (atoms of 8 rows x 128 B).  The
// start field is addr >> 4 in the low 14 bits: a byte offset d (< 256 KB total)
// is added to a descriptor as d >> 4.
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFFu) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}
// Instruction descriptor kind::f16: fp16 A / B, fp32 D, M = 128, N = 64, A major.
__host__ __device__ constexpr uint32_t idesc_f16(bool a_mn_major, int M = 128) {
  return (1u << 4) | ((a_mn_major ? 1u : 0u) << 15) | (static_cast<uint32_t>(64 >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
// 32 lanes x 16 consecutive 32-bit columns (no wait: the caller waits once)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
// 32 lanes x 64 consecutive 32-bit columns (no wait)
__device__ __forceinline__ void tmem_ld64(uint32_t taddr, uint32_t (&r)[64]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32, %33, %34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, %48, %49, %50, %51, %52, %53, %54, %55, %56, %57, %58, %59, %60, %61, %62, %63}, [%64];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint4 (&q)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};\n" ::"r"(taddr),
      "r"(q[0].x), "r"(q[0].y), "r"(q[0].z), "r"(q[0].w), "r"(q[1].x), "r"(q[1].y), "r"(q[1].z), "r"(q[1].w),
      "r"(q[2].x), "r"(q[2].y), "r"(q[2].z), "r"(q[2].w), "r"(q[3].x), "r"(q[3].y), "r"(q[3].z), "r"(q[3].w),
      "r"(q[4].x), "r"(q[4].y), "r"(q[4].z), "r"(q[4].w), "r"(q[5].x), "r"(q[5].y), "r"(q[5].z), "r"(q[5].w),
      "r"(q[6].x), "r"(q[6].y), "r"(q[6].z), "r"(q[6].w), "r"(q[7].x), "r"(q[7].y), "r"(q[7].z), "r"(q[7].w)
      : "memory");
}
__device__ __forceinline__ uint32_t pack_half2(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// Unit walk of one CTA: units [a, b) of u = band * nC + column tile (32-bit: a
// tensor that fits in HBM has far fewer than 2^31 units of 32 KB).
struct FWalk {
  int a, b, nC, nRT;
  int window;
  int A = kA;  // row tiles per band
  __device__ int band(int u) const { return u / nC; }
  __device__ int tiles(int u) const {
    const int r = nRT - band(u) * A;
    return r < A ? r : A;
  }
  __device__ bool band_start(int u) const { return u == a || u % nC == 0; }
  __device__ bool seg_end(int u) const { return u + 1 == b || (u + 1) % nC == 0; }
  // position of u in its segment (the CTA's run of units inside one band)
  __device__ int seg_pos(int u) const {
    const int s0 = u - u % nC;
    return u - (s0 > a ? s0 : a);
  }
  __device__ bool win_end(int u) const { return seg_end(u) || seg_pos(u) % window == window - 1; }
  __device__ bool win_start(int u) const { return band_start(u) || seg_pos(u) % window == 0; }
};

// The same walk as an incremental iterator (no runtime-divisor division or
// modulo per unit: the MMA warp's bookkeeping sits between MMA issue bursts).
struct UnitIter {
  int u, end, b, c, nt, wpos, nC, nRT, window, A;
  bool first;
  __device__ void init(const FWalk& w) {
    A = w.A;
    u = w.a;
    end = w.b;
    nC = w.nC;
    nRT = w.nRT;
    window = w.window;
    b = u / nC;
    c = u - b * nC;
    nt = tiles_of(b);
    wpos = 0;
    first = true;
  }
  __device__ int tiles_of(int band) const {
    const int r = nRT - band * A;
    return r < A ? r : A;
  }
  __device__ bool more() const { return u < end; }
  __device__ bool band_start() const { return first || c == 0; }
  __device__ bool seg_end() const { return u + 1 == end || c + 1 == nC; }
  __device__ bool win_start() const { return first || c == 0 || wpos == 0; }
  __device__ bool win_end() const { return seg_end() || wpos == window - 1; }
  __device__ void next() {
    first = false;
    ++u;
    if (++c == nC) {
      c = 0;
      ++b;
      nt = tiles_of(b);
      wpos = 0;
    } else {
      wpos = wpos + 1 == window ? 0 : wpos + 1;
    }
  }
};

__global__ void __launch_bounds__(kThreads, 1)
    seed_f32f_kernel(const Seed32FParams p, const __grid_constant__ CUtensorMap ymap) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cta = blockIdx.x;
  FWalk w;
  w.a = static_cast<int>(static_cast<int64_t>(cta) * p.units / p.P);
  w.b = static_cast<int>(static_cast<int64_t>(cta + 1) * p.units / p.P);
  w.nC = static_cast<int>(p.nC);
  w.nRT = static_cast<int>(p.nRT);
  w.window = p.window;
  const int seg0 = w.a / w.nC;  // first band of this CTA (segment index = band - seg0)

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  const uint32_t land_u = smem_u32(base);                // [kNL][32 KB] fp32 tiles
  const uint32_t planes_u = smem_u32(base + kOffPlanes);  // [kNP][hi 16 KB | lo 16 KB]
  const uint32_t krt_u = smem_u32(base + kOffKR);         // [2][16 KB] KRr tiles
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + kOffBars);
  uint64_t* full = bars;                 // [kNL] Y tile landed            (1 + tx)
  uint64_t* lfree = full + kNL;          // [kNL] landing slot read        (4 split warps)
  uint64_t* pfull = lfree + kNL;         // [kNP] planes written           (4 split warps)
  uint64_t* pfree = pfull + kNP;         // [kNP] planes consumed          (MMA commit)
  uint64_t* kfull = pfree + kNP;         // [2] KRr tile landed            (1 + tx)
  uint64_t* kempty = kfull + 2;          // [2] KRr tile consumed          (MMA commit)
  uint64_t* lfull = kempty + 2;          // [2] left unit accumulated      (MMA commit)
  uint64_t* lempty = lfull + 2;          // [2] left accumulator drained   (8 drain warps)
  uint64_t* rfull = lempty + 2;          // [kA] right window accumulated  (MMA commit)
  uint64_t* rempty = rfull + kA;         // [kA] right window drained      (the row tile's 4 drain warps)
  uint64_t* kl_full = rempty + kA;       // band's KRl^T in TMEM           (8 drain warps)
  uint64_t* kl_free = kl_full + 1;       // band's MMAs done               (MMA commit)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(kl_free + 1);
  double* unscale = reinterpret_cast<double*>(base + kOffBars + 512);  // [64] 1 / (scale_y scale_r)

  if (tid == 0) {
    wd_init(p.fault, 0);
    for (int s = 0; s < kNL; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&lfree[s], kSplitWarps);
    }
    for (int s = 0; s < kNP; ++s) {
      mbar_init(&pfull[s], kSplitWarps);
      mbar_init(&pfree[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&kfull[s], 1);
      mbar_init(&kempty[s], 1);
      mbar_init(&lfull[s], 1);
      mbar_init(&lempty[s], kDrainWarps);
    }
    for (int t = 0; t < kA; ++t) {
      mbar_init(&rfull[t], 1);
      mbar_init(&rempty[t], kDrainWarps);
    }
    mbar_init(kl_full, kDrainWarps);
    mbar_init(kl_free, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp != kWProd) pdl_wait();  // scales, Khatri-Rao images: the preceding kernels
  if (tid < kRP) unscale[tid] = p.inv_scale_y[0] * p.inv_scale_kr[tid];
  if (warp == kWMma) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (warp == kWProd && lane == 0)
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&ymap)));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp == kWProd) {
    // ------------------------------------------------------------------ producer
    if (lane == 0) {
      const uint64_t pol_y = policy_evict_first(), pol_k = policy_evict_last();
      int k = 0;  // running tile index
      bool waited = false;
      for (int u = w.a; u < w.b; ++u) {
        const int b = w.band(u), c = u % w.nC;
        const int nt = w.tiles(u);
        const int ul = u - w.a;
        for (int t = 0; t < nt; ++t, ++k) {
          const int s = k % kNL;
          if (k >= kNL) mbar_wait(&lfree[s], static_cast<uint32_t>((k / kNL - 1) & 1));
          mbar_arrive_tx(&full[s], kYBytes);
          tma_load_2d(land_u + s * kYBytes, &ymap, static_cast<int>((b * kA + t) * kTI), static_cast<int>(c * kTJ),
                      &full[s], pol_y);
          if (t == 0) {  // the unit's KRr tile (Khatri-Rao images come from the preceding kernels)
            if (!waited) {
              pdl_wait();
              waited = true;
            }
            const int ks = static_cast<int>(ul & 1);
            if (ul >= 2) mbar_wait(&kempty[ks], static_cast<uint32_t>(((ul >> 1) - 1) & 1));
            mbar_arrive_tx(&kfull[ks], kKRBytes);
            bulk_load(krt_u + ks * kKRBytes, p.kr_tiles + static_cast<int64_t>(c) * kKRBytes, kKRBytes, &kfull[ks],
                      pol_k);
          }
        }
      }
    }
  } else if (warp == kWMma) {
    // ------------------------------------------------------------------ MMA issuer
    // The whole warp runs the loop and waits; one elected lane issues.  Every
    // operand below is warp-uniform, so the MMAs go out back to back.
    constexpr uint32_t id_r = idesc_f16(true), id_l = idesc_f16(false);
    const uint64_t dA0 = sdesc(planes_u, 8192, 1024);  // right A: Y plane, MN-major
    const uint64_t dB0 = sdesc(krt_u, 16, 1024);       // right B: KRr tile, K-major
    const uint64_t dL0 = sdesc(planes_u, 16, 1024);    // left B: Y plane, K-major
    const bool all_terms_r = !(p.knobs & 2), all_terms_l = !(p.knobs & 4);
    int k = 0, bc = 0;
    int wc[kA] = {0, 0, 0};  // right windows started per row tile
    for (int u = w.a; u < w.b; ++u) {
      const int nt = w.tiles(u);
      const int ul = u - w.a;
      const int ks = static_cast<int>(ul & 1), lb = static_cast<int>(ul & 1);
      if (w.band_start(u)) mbar_wait(kl_full, static_cast<uint32_t>(bc & 1));
      if (ul >= 2) mbar_wait(&lempty[lb], static_cast<uint32_t>(((ul >> 1) - 1) & 1));
      mbar_wait(&kfull[ks], static_cast<uint32_t>((ul >> 1) & 1));
      tc_fence_after();
      const bool wstart = w.win_start(u), wend = w.win_end(u);
      const uint64_t kb = dB0 + static_cast<uint64_t>((ks * kKRBytes) >> 4);
      const uint32_t dL = tmem + kColL + kRP * lb;
#pragma unroll
      for (int t = 0; t < kA; ++t) {
        if (t >= nt) break;
        const int ps = k % kNP;
        if (wstart && wc[t] > 0) mbar_wait(&rempty[t], static_cast<uint32_t>((wc[t] - 1) & 1));
        mbar_wait(&pfull[ps], static_cast<uint32_t>((k / kNP) & 1));
        tc_fence_after();
        const uint64_t pa = static_cast<uint64_t>((ps * 2 * kPlane) >> 4);
        const uint64_t aH = dA0 + pa, aL = aH + (kPlane >> 4), lH = dL0 + pa, lL = lH + (kPlane >> 4);
        const uint32_t dR = tmem + kColR + kRP * t, aK = tmem + kColK + kRP * t;
        if (elect_one()) {
          // right: K = 64 columns j in 4 steps of 16 (2 KB of plane rows each)
#pragma unroll
          for (int q = 0; q < kTJ / 16; ++q) {
            mma_ss(dR, aH + q * 128, kb + q * 2, id_r, (wstart && q == 0) ? 0u : 1u);
            if (all_terms_r) {
              mma_ss(dR, aH + q * 128, kb + 512 + q * 2, id_r, 1u);
              mma_ss(dR, aL + q * 128, kb + q * 2, id_r, 1u);
            }
          }
          // left: K = 128 rows i in 8 steps of 16 (i half q / 4, 32 B steps inside the 128 B rows)
#pragma unroll
          for (int q = 0; q < kTI / 16; ++q) {
            const uint32_t off = ((q >> 2) * 8192 + (q & 3) * 32) >> 4;
            mma_ts(dL, aK + 8 * q, lH + off, id_l, (t == 0 && q == 0) ? 0u : 1u);
            if (all_terms_l) mma_ts(dL, aK + 8 * q, lL + off, id_l, 1u);
          }
          umma_commit(&pfree[ps]);
          if (wend) umma_commit(&rfull[t]);
        }
        __syncwarp();
        if (wend) ++wc[t];
        ++k;
      }
      if (elect_one()) {
        umma_commit(&kempty[ks]);
        umma_commit(&lfull[lb]);
        if (w.seg_end(u)) umma_commit(kl_free);
      }
      __syncwarp();
      if (w.seg_end(u)) ++bc;
    }
  } else if (warp > kWMma) {
    // idle (warps 14, 15: 16 warps keep the 128-register budget)
  } else if (warp < kWDrain0) {
    // ------------------------------------------------------------------ split
    // thread = row pair (2 pr, 2 pr + 1) x column half jh: 32 float2 loads (one
    // 8-byte row pair per column, conflict-free), then per column one packed hi
    // and one packed lo word at the pair's position of the swizzled planes
    // (the 32 lanes of a warp cover one 128-byte plane row: no bank conflicts).
    const float sy = p.scale_y[0];
    const bool scale = sy != 1.0f, store = !(p.knobs & 1);
    const int st = warp * 32 + lane;
    const int pr = st & 63, jh = st >> 6;
    const int i0 = 2 * pr, c0 = (i0 & 63) >> 3;
    uint32_t base8[8];  // plane offset of column j (j % 8 == k) minus j * 128
#pragma unroll
    for (int k = 0; k < 8; ++k)
      base8[k] = (i0 >> 6) * 8192 + jh * 32 * 128 + (((c0 ^ k)) << 4) + (i0 & 7) * 2;
    const unsigned char* land = base;
    int k = 0;
    for (int u = w.a; u < w.b; ++u) {
      const int nt = w.tiles(u);
      for (int t = 0; t < nt; ++t, ++k) {
        const int ls = k % kNL, ps = k % kNP;
        mbar_wait(&full[ls], static_cast<uint32_t>((k / kNL) & 1));
        const float2* src = reinterpret_cast<const float2*>(land + ls * kYBytes) + jh * 32 * (kTI / 2) + pr;
        uint32_t hw[32], lw[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          float2 x = src[e * (kTI / 2)];
          if (scale) {
            x.x *= sy;
            x.y *= sy;
          }
          hw[e] = pack_half2(x.x, x.y);
          const float2 back = __half22float2(*reinterpret_cast<const __half2*>(&hw[e]));
          lw[e] = pack_half2(x.x - back.x, x.y - back.y);
        }
        __syncwarp();  // every lane's reads of the landing slot are done (their values are in use)
        if (lane == 0) mbar_arrive(&lfree[ls]);
        if (k >= kNP) mbar_wait(&pfree[ps], static_cast<uint32_t>((k / kNP - 1) & 1));
        if (store) {
          const uint32_t hi = planes_u + ps * 2 * kPlane, lo = hi + kPlane;
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const uint32_t off = base8[e & 7] + e * 128;
            asm volatile("st.shared.b32 [%0], %1;\n" ::"r"(hi + off), "r"(hw[e]) : "memory");
            asm volatile("st.shared.b32 [%0], %1;\n" ::"r"(lo + off), "r"(lw[e]) : "memory");
          }
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic writes -> MMA reads
        __syncwarp();
        if (lane == 0) mbar_arrive(&pfull[ps]);
      }
    }
  } else {
    // ------------------------------------------------------------------ drains
    // warp (q, h): TMEM lane quarter q (== warp % 4), column half h: ranks
    // [32 h, 32 h + 32) of the three right accumulators (fp32 second-level sums),
    // the KRl^T image words [32 h, 32 h + 32), left-partial columns [32 h, +32)
    const int d = warp - kWDrain0, q = d & 3, h = d >> 2;
    const uint32_t lanes = static_cast<uint32_t>(q * 32) << 16;
    const int odd = lane & 1;
    const bool lstore = !(p.knobs & 8);
    float acc[kA][32];
#pragma unroll
    for (int t = 0; t < kA; ++t)
#pragma unroll
      for (int e = 0; e < 32; ++e) acc[t][e] = 0.0f;
    int bc = 0, wc = 0;
    for (int u = w.a; u < w.b; ++u) {
      const int nt = w.tiles(u);
      const int b = w.band(u), ul = u - w.a, c = u % w.nC;
      const int lb = ul & 1;
      if (w.band_start(u)) {  // the band's KRl^T image into TMEM, once its previous band is done
        if (bc > 0) mbar_wait(kl_free, static_cast<uint32_t>((bc - 1) & 1));
        __syncwarp();
        tc_fence_after();
        for (int t = 0; t < nt; ++t) {
          const uint4* src = reinterpret_cast<const uint4*>(static_cast<const __half*>(p.krl_img) +
                                                            (static_cast<int64_t>(b * kA + t) * 128 + q * 32 + lane) *
                                                                kTI) +
                             h * 8;  // words [32 h, 32 h + 32) of the slot's 64
          uint4 x[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) x[e] = __ldg(src + e);
          tmem_st32(tmem + lanes + kColK + kRP * t + 32 * h, x);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(kl_full);
      }
      // right: drain the window into the fp32 second level (before the left drain:
      // the next window's first MMA into these accumulators waits for it)
      if (w.win_end(u)) {
#pragma unroll
        for (int t = 0; t < kA; ++t) {
          if (t >= nt) break;
          mbar_wait(&rfull[t], static_cast<uint32_t>(wc & 1));
          __syncwarp();  // tcgen05.ld is .sync.aligned: reconverge after the spin
          tc_fence_after();
#pragma unroll
          for (int c8 = 0; c8 < 4; ++c8) {
            uint32_t y[8];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                         : "=r"(y[0]), "=r"(y[1]), "=r"(y[2]), "=r"(y[3]), "=r"(y[4]), "=r"(y[5]), "=r"(y[6]),
                           "=r"(y[7])
                         : "r"(tmem + lanes + kColR + kRP * t + 32 * h + 8 * c8));
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[t][8 * c8 + e] += __uint_as_float(y[e]);
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&rempty[t]);
        }
        ++wc;
      }
      // left: lanes (2 r', 2 r' + 1) hold the hi / lo products of rank 16 q + r';
      // per 8-column chunk the pair sums with one shuffle and each lane stores 4
      mbar_wait(&lfull[lb], static_cast<uint32_t>((ul >> 1) & 1));
      __syncwarp();
      tc_fence_after();
      const int r = 16 * q + (lane >> 1);
      float* lrow = p.lpart + ((static_cast<int64_t>(b) * w.nC + c) * kRP + r) * kTJ + 32 * h + 4 * odd;
#pragma unroll
      for (int c8 = 0; c8 < 4; ++c8) {
        uint32_t v[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(tmem + lanes + kColL + kRP * lb + 32 * h + 8 * c8));
        tmem_wait_ld();
        if (c8 == 3) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&lempty[lb]);
        }
        float o[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float keep = __uint_as_float(odd ? v[4 + e] : v[e]);  // the columns this lane stores
          const float give = __uint_as_float(odd ? v[e] : v[4 + e]);  // the partner's columns
          o[e] = keep + __shfl_xor_sync(0xffffffffu, give, 1);
        }
        if (lstore) *reinterpret_cast<float4*>(lrow + 8 * c8) = make_float4(o[0], o[1], o[2], o[3]);
      }
      if (w.seg_end(u)) {
        const int64_t slot0 = (static_cast<int64_t>(cta) * p.slots + (b - seg0)) * kA;  // CSR slots
#pragma unroll
        for (int t = 0; t < kA; ++t) {
          if (t >= nt) break;
          double* out = p.rpart + ((slot0 + t) * kRP + 32 * h) * kTI + q * 32 + lane;
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            out[e * kTI] = static_cast<double>(acc[t][e]) * unscale[32 * h + e];
            acc[t][e] = 0.0f;
          }
        }
        ++bc;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kWMma) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(kTmemCols));
  }
}

// ==================================================================================
// timed wait (CPDGPU_SEED_TRACE): cycles spent waiting added to *acc
template <bool WD>
// acc == nullptr (no CPDGPU_SEED_TRACE): no clock reads on the pipeline's roles
__device__ __forceinline__ void mbar_wait_t(uint64_t* bar, uint32_t parity, unsigned long long* acc) {
  if (!acc) {
    mbar_wait<WD>(bar, parity);
    return;
  }
  const long long t0 = clock64();
  mbar_wait<WD>(bar, parity);
  *acc += static_cast<unsigned long long>(clock64() - t0);
}
__device__ __forceinline__ void mbar_wait_plain_t(uint64_t* bar, uint32_t parity, unsigned long long* acc) {
  if (!acc) {
    mbar_wait_plain(bar, parity);
    return;
  }
  const long long t0 = clock64();
  mbar_wait_plain(bar, parity);
  *acc += static_cast<unsigned long long>(clock64() - t0);
}

// Operand-image variant: the tensor's fp16 hi / lo planes are built once per tensor
// version (build_f16_image_kernel, same 4 bytes per entry as the fp32 tensor) and
// TMA-loaded straight into the 128-byte-swizzled operand layout, so the kernel
// has no split stage: per 32 KB tile the shared-memory port carries the TMA write
// and the MMA operand reads only (136 KB instead of 200 KB).
//
//   warps 0-11   drains (q, t): TMEM lane quarter q == warp % 4, row tile t of the
//                band: the right window drains (64 fp32 second-level sums per
//                lane), the KRl^T image of row tile t, left chunks t, t+3, t+6 of
//                the unit's accumulator, staged in shared memory and added in L2 by
//                one bulk reduce per unit (A = 2: warps 8-11 drain only the left
//                accumulator, one tcgen05.ld per unit, warps 0-7 only right windows)
//   warp 12      producer: 4 TMA boxes (64 i x 64 j, one plane: 8 KB of consecutive
//                bytes in the 64-row-chunked image) per tile into a 5-slot ring
//   warp 13      right-product MMAs (whole warp waits, one elected lane issues):
//                three N = 64 MMAs per K step, or (A = 2) one N = 128 against the
//                [KR_hi | KR_lo] tile and one N = 64
//   warp 14      Khatri-Rao producer: the unit's KRr tile into a 2-deep ring (its
//                own warp: the Y stream never waits on a Khatri-Rao slot)
//   warp 15      left-product MMAs: Y_hi against all 128 KRl^T lanes (M = 128),
//                Y_lo against the hi lanes only (M = 64: lanes 0-15 of each quarter)
// Two issuing warps, one per product: the tensor pipe's queue is shallow, so a
// single issuer's per-tile barrier waits, fences and commits left it idle ~1/3
// of the time (1660 cycles per tile against 1112 of MMA work); with the two
// products issued by two warps one warp's bookkeeping overlaps the other's
// MMAs (tools/microbench/mma_mix.cu: 1355 -> 1082 cycles per tile).
constexpr int kINS = 5;                        // image slots (160 KB of loads in flight)
constexpr int kINK = 2;                        // KRr slots (units of look-ahead)
constexpr int kStage = kRP * kTJ * 4;          // 16 KB left-partial staging buffer [16 column quads][64 r][4 j] fp32
constexpr int kIDrain = 12, kIWProd = kIDrain, kIWMma = kIDrain + 1, kIWKr = kIDrain + 2, kIWMmaL = kIDrain + 3;
constexpr int kIThreads = 16 * 32;
constexpr int kIOffKR = kINS * 2 * kPlane;
constexpr int kIOffStage = kIOffKR + kINK * kKRBytes;
constexpr int kIOffBars = kIOffStage + 2 * kStage;
constexpr int kISmem = 1024 + kIOffBars + 512 + kRP * 8;

template <bool WD, int A>
__global__ void __launch_bounds__(kIThreads, 1)
    seed_f32i_kernel(const Seed32FParams p, const __grid_constant__ CUtensorMap imap) {
  // A = 3: one 64-column right accumulator per row tile, three N = 64 MMAs per K step.
  // A = 2 (stacked): 128 columns per row tile, [Y_hi KR_hi | Y_hi KR_lo + Y_lo KR_hi]:
  // one N = 128 MMA against the [KR_hi | KR_lo] tile and one N = 64 MMA per K step, so
  // the Y plane is read from shared memory twice instead of three times.
  constexpr bool STK = A == 2;
  constexpr uint32_t cRw = STK ? 2 * kRP : kRP;  // right accumulator columns per row tile
  constexpr uint32_t cK = A * cRw;               // KRl^T[t]: [cK + 64 t, +64)
  constexpr uint32_t cL = cK + A * kRP;          // D_L[lb]: [cL + 64 lb, +64)
  static_assert(cL + 2 * kRP <= kTmemCols, "TMEM columns");
  // drain warps of the left accumulator: all 12 (A = 3), or the lane-quarter group
  // without a row tile (A = 2: warps 8-11 drain only the left accumulator, warps 0-7
  // only the right windows, so a late left product never delays a right drain)
  constexpr int kLW = STK ? 4 : kIDrain;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cta = blockIdx.x;
  const bool trc = p.trace != nullptr;  // per-role wait timers (CPDGPU_SEED_TRACE)
  FWalk w;
  w.a = static_cast<int>(static_cast<int64_t>(cta) * p.units / p.P);
  w.b = static_cast<int>(static_cast<int64_t>(cta + 1) * p.units / p.P);
  w.nC = static_cast<int>(p.nC);
  w.nRT = static_cast<int>(p.nRT);
  w.window = p.window;
  w.A = A;
  const int seg0 = w.a / w.nC;

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  const uint32_t ring_u = smem_u32(base);            // [kINS][hi 16 KB | lo 16 KB]
  const uint32_t krt_u = smem_u32(base + kIOffKR);   // [kINK][16 KB] KRr tiles
  const uint32_t stage_u = smem_u32(base + kIOffStage);  // [2][16 KB] left partial of a unit
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + kIOffBars);
  uint64_t* full = bars;                 // [kINS] planes landed            (1 + tx)
  uint64_t* empty = full + kINS;         // [kINS] planes consumed          (MMA commit)
  uint64_t* kfull = empty + kINS;        // [kINK] KRr tile landed          (1 + tx)
  uint64_t* kempty = kfull + kINK;       // [kINK] KRr tile consumed        (MMA commit)
  uint64_t* lfull = kempty + kINK;       // [2] left unit accumulated       (MMA commit)
  uint64_t* lempty = lfull + 2;          // [2] left accumulator drained    (12 drain warps)
  uint64_t* rfull = lempty + 2;          // [kA] right window accumulated   (MMA commit)
  uint64_t* rempty = rfull + kA;         // [kA] right window drained       (the row tile's 4 warps)
  uint64_t* kl_full = rempty + kA;       // band's KRl^T in TMEM            (12 drain warps)
  uint64_t* kl_free = kl_full + 1;       // band's MMAs done                (MMA commit)
  uint64_t* fin = kl_free + 1;           // every MMA of the CTA done       (MMA commit, before dealloc)
  uint64_t* sfull = fin + 1;             // [2] staging buffer written      (12 drain warps)
  uint64_t* sfree = sfull + 2;           // [2] staging buffer read by its bulk operation (the issuing lane)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sfree + 2);
  unsigned* drains_out = tmem_slot + 1;  // drain warps that left their loop
  double* unscale = reinterpret_cast<double*>(base + kIOffBars + 512);  // [64] 1 / (scale_y scale_r)

  if (tid == 0) {
    if (WD) wd_init(p.fault, p.stall);
    for (int s = 0; s < kINS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 2);  // both issuing warps' commits
    }
    for (int s = 0; s < kINK; ++s) {
      mbar_init(&kfull[s], 1);
      mbar_init(&kempty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&lfull[s], 1);
      mbar_init(&lempty[s], kLW);
      mbar_init(&sfull[s], kLW);
      mbar_init(&sfree[s], 1);
    }
    for (int t = 0; t < kA; ++t) {
      mbar_init(&rfull[t], 1);
      mbar_init(&rempty[t], 4);
    }
    mbar_init(kl_full, kIDrain - (STK ? kLW : 0));
    mbar_init(kl_free, 1);
    mbar_init(fin, 2);
    *drains_out = 0;
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp != kIWProd) pdl_wait();  // scales, Khatri-Rao images: the preceding kernels (Y: not)
  if (tid < kRP) unscale[tid] = p.inv_scale_y[0] * p.inv_scale_kr[tid];
  if (warp == kIWMma) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (warp == kIWProd && lane == 0)
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&imap)));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kIWProd) {
    // ------------------------------------------------------------------ producer
    if (lane == 0) {
      const uint64_t pol_y = policy_evict_first();
      int k = 0;
      unsigned long long tw = 0;
      const long long tstart = clock64();
      int s = 0;
      uint32_t ph = 0;  // ring slot s, its empty-phase parity for this lap
      UnitIter it;
      for (it.init(w); it.more() && !wd_aborted<WD>(); it.next()) {
        const int b = it.b, c = it.c, nt = it.nt;
        for (int t = 0; t < nt; ++t, ++k) {
          if (k >= kINS) mbar_wait_t<WD>(&empty[s], ph ^ 1u, trc ? &tw : nullptr);
          if (wd_aborted<WD>()) break;  // watchdog: no new loads
          if ((p.knobs & 16) && k >= kINS) {  // timing experiment: no refill (stale planes)
            mbar_arrive(&full[s]);
          } else {
          mbar_arrive_tx(&full[s], 2 * kPlane);
          // tests (p.stall): the first tile is announced but never requested (watchdog path)
          if (!(p.stall && k == 0)) {
            const int i0 = (b * A + t) * kTI, j0 = c * kTJ;
#pragma unroll
            for (int pl = 0; pl < 2; ++pl)
#pragma unroll
              for (int ih = 0; ih < 2; ++ih)
                asm volatile(
                    "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
                    " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;\n" ::"r"(ring_u + s * 2 * kPlane + pl * kPlane + ih * 8192),
                    "l"(reinterpret_cast<uint64_t>(&imap)), "r"(0), "r"((i0 >> 6) + ih), "r"(j0), "r"(pl),
                    "r"(smem_u32(&full[s])), "l"(pol_y)
                    : "memory");
          }
          }
          if (++s == kINS) {
            s = 0;
            ph ^= 1u;
          }
        }
      }
      if (wd_aborted<WD>())  // the last load of each ring slot lands before the CTA exits
        for (int q = k > kINS ? k - kINS : 0; q < k; ++q)
          if (!(p.stall && q == 0)) mbar_drain_wait(&full[q % kINS], static_cast<uint32_t>((q / kINS) & 1));
      if (p.trace) {
        p.trace[(static_cast<int64_t>(cta) * 16 + warp) * 8 + 0] = tw;
        p.trace[(static_cast<int64_t>(cta) * 16 + warp) * 8 + 6] = static_cast<unsigned long long>(clock64() - tstart);
      }
    }
  } else if (warp == kIWKr) {
    // ------------------------------------------------------------------ KRr producer
    if (lane == 0) {
      const uint64_t pol_k = policy_evict_last();
      int ul = 0;
      UnitIter it;
      for (it.init(w); it.more(); it.next(), ++ul) {
        const int ks = ul & (kINK - 1);
        if (ul >= kINK) mbar_wait<WD>(&kempty[ks], static_cast<uint32_t>(((ul / kINK) - 1) & 1));
        if (wd_aborted<WD>()) break;  // watchdog: no new loads
        mbar_arrive_tx(&kfull[ks], kKRBytes);
        bulk_load(krt_u + ks * kKRBytes, p.kr_tiles + static_cast<int64_t>(it.c) * kKRBytes, kKRBytes, &kfull[ks],
                  pol_k);
      }
      if (wd_aborted<WD>())
        for (int q = ul > kINK ? ul - kINK : 0; q < ul; ++q)
          mbar_drain_wait(&kfull[q & (kINK - 1)], static_cast<uint32_t>((q / kINK) & 1));
    }
  } else if (warp == kIWMma) {
    // ------------------------------------------------------------------ right MMAs
    constexpr uint32_t id_r = idesc_f16(true);
    constexpr uint32_t id_r2 = id_r + (static_cast<uint32_t>(64 >> 3) << 17);  // N = 128
    const uint64_t dA0 = sdesc(ring_u, 8192, 1024);  // right A: Y plane, MN-major
    const uint64_t dB0 = sdesc(krt_u, 16, 1024);     // right B: KRr tile, K-major
    const bool all_terms_r = !(p.knobs & 2);
    const bool run = !(p.knobs & (32 | 256));  // timing experiments: no MMAs / no right MMAs
    int k = 0;
    int wc[kA] = {0, 0, 0};
    unsigned long long tr[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const long long tstart = clock64();
    int s = 0;
    uint32_t ph = 0;  // ring slot and its full-phase parity
    int ul = 0;
    UnitIter it;
    for (it.init(w); it.more() && !wd_aborted<WD>(); it.next(), ++ul) {
      const int nt = it.nt;
      const int ks = ul & (kINK - 1);
      mbar_wait_t<WD>(&kfull[ks], static_cast<uint32_t>((ul / kINK) & 1), trc ? &tr[2] : nullptr);
      tc_fence_after();
      const bool wstart = it.win_start(), wend = it.win_end();
      const uint64_t kb = dB0 + static_cast<uint64_t>((ks * kKRBytes) >> 4);
#pragma unroll
      for (int t = 0; t < A; ++t) {
        if (t >= nt) break;
        if (wstart && wc[t] > 0)
          mbar_wait_t<WD>(&rempty[t], static_cast<uint32_t>((wc[t] - 1) & 1), trc ? &tr[3] : nullptr);
        mbar_wait_t<WD>(&full[s], ph, trc ? &tr[0] : nullptr);
        tc_fence_after();
        const long long ti = trc ? clock64() : 0;
        const uint64_t aH = dA0 + static_cast<uint64_t>((s * 2 * kPlane) >> 4), aL = aH + (kPlane >> 4);
        const uint32_t dR = tmem + cRw * t;
        if (elect_one()) {
          if (run) {
#pragma unroll
            for (int q = 0; q < kTJ / 16; ++q) {
              if (STK) {
                mma_ss(dR, aH + q * 128, kb + q * 2, id_r2, (wstart && q == 0) ? 0u : 1u);
                if (all_terms_r) mma_ss(dR + kRP, aL + q * 128, kb + q * 2, id_r, 1u);
                continue;
              }
              mma_ss(dR, aH + q * 128, kb + q * 2, id_r, (wstart && q == 0) ? 0u : 1u);
              if (all_terms_r) {
                mma_ss(dR, aH + q * 128, kb + 512 + q * 2, id_r, 1u);
                mma_ss(dR, aL + q * 128, kb + q * 2, id_r, 1u);
              }
            }
          }
          umma_commit(&empty[s]);
          if (wend) umma_commit(&rfull[t]);
        }
        __syncwarp();
        if (trc) tr[5] += static_cast<unsigned long long>(clock64() - ti);
        if (wend) ++wc[t];
        ++k;
        if (++s == kINS) {
          s = 0;
          ph ^= 1u;
        }
      }
      if (elect_one()) umma_commit(&kempty[ks]);
      __syncwarp();
    }
    // after a watchdog abort the drains may sit in unbounded waits on the MMA-side
    // barriers: keep flipping those phases until every drain warp has left its loop
    if (wd_aborted<WD>() && lane == 0)
      for (uint32_t i = 0; i < (1u << 22) && *reinterpret_cast<volatile unsigned*>(drains_out) < kIDrain; ++i) {
        mbar_arrive(&lfull[0]);
        mbar_arrive(&lfull[1]);
        for (int q = 0; q < A; ++q) mbar_arrive(&rfull[q]);
        mbar_arrive(kl_free);
        __nanosleep(256);
      }
    __syncwarp();
    // every issued MMA (both issuing warps) has completed before TMEM is released;
    // MMA completion is bounded, so this spin ignores the abort flag
    if (elect_one()) umma_commit(fin);
    __syncwarp();
    {
      uint32_t done = 0;
      while (!done)
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(fin)), "r"(0u)
            : "memory");
    }
    if (p.trace && lane == 0) {
      tr[6] = static_cast<unsigned long long>(clock64() - tstart);
      tr[7] = static_cast<unsigned long long>(k);
      for (int e = 0; e < 8; ++e) p.trace[(static_cast<int64_t>(cta) * 16 + warp) * 8 + e] = tr[e];
    }
  } else if (warp == kIWMmaL) {
    // ------------------------------------------------------------------ left MMAs
    constexpr uint32_t id_l = idesc_f16(false);
    // the Y_lo plane against the hi parts only (M = 64: TMEM lanes 0-15 of every lane
    // quarter, where the image kernel's KRl^T layout keeps them): no lo * lo product
    const uint32_t id_l2 = p.left_m64 ? idesc_f16(false, 64) : id_l;
    const uint64_t dL0 = sdesc(ring_u, 16, 1024);  // left B: Y plane, K-major
    const bool all_terms_l = !(p.knobs & 4);
    const bool run = !(p.knobs & (32 | 128));  // timing experiments: no MMAs / no left MMAs
    int bc = 0;
    unsigned long long tr[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const long long tstart = clock64();
    int s = 0;
    uint32_t ph = 0;
    int ul = 0;
    UnitIter it;
    for (it.init(w); it.more() && !wd_aborted<WD>(); it.next(), ++ul) {
      const int nt = it.nt;
      const int lb = ul & 1;
      const bool seg_end = it.seg_end();
      if (it.band_start()) mbar_wait_t<WD>(kl_full, static_cast<uint32_t>(bc & 1), trc ? &tr[4] : nullptr);
      if (ul >= 2) mbar_wait_t<WD>(&lempty[lb], static_cast<uint32_t>(((ul >> 1) - 1) & 1), trc ? &tr[1] : nullptr);
      const uint32_t dL = tmem + cL + kRP * lb;
#pragma unroll
      for (int t = 0; t < A; ++t) {
        if (t >= nt) break;
        mbar_wait_t<WD>(&full[s], ph, trc ? &tr[0] : nullptr);
        tc_fence_after();
        const long long ti = trc ? clock64() : 0;
        const uint64_t lH = dL0 + static_cast<uint64_t>((s * 2 * kPlane) >> 4), lL = lH + (kPlane >> 4);
        const uint32_t aK = tmem + cK + kRP * t;
        if (elect_one()) {
          if (run) {
#pragma unroll
            for (int q = 0; q < kTI / 16; ++q) {
              const uint32_t off = ((q >> 2) * 8192 + (q & 3) * 32) >> 4;
              mma_ts(dL, aK + 8 * q, lH + off, id_l, (t == 0 && q == 0) ? 0u : 1u);
              if (all_terms_l) mma_ts(dL, aK + 8 * q, lL + off, id_l2, 1u);
            }
          }
          umma_commit(&empty[s]);
        }
        __syncwarp();
        if (trc) tr[5] += static_cast<unsigned long long>(clock64() - ti);
        if (++s == kINS) {
          s = 0;
          ph ^= 1u;
        }
      }
      if (elect_one()) {
        umma_commit(&lfull[lb]);
        if (seg_end) umma_commit(kl_free);
      }
      __syncwarp();
      if (seg_end) ++bc;
    }
    if (elect_one()) umma_commit(fin);
    __syncwarp();
    if (p.trace && lane == 0) {
      tr[6] = static_cast<unsigned long long>(clock64() - tstart);
      for (int e = 0; e < 8; ++e) p.trace[(static_cast<int64_t>(cta) * 16 + warp) * 8 + e] = tr[e];
    }
  } else if (STK && warp >= kIDrain - kLW && warp < kIDrain) {
    // ------------------------------------------------------------------ left drains (A = 2)
    // One warp per TMEM lane quarter: the unit's whole 64-column accumulator in ONE
    // tcgen05.ld (the load's round trip under a busy tensor pipe is what a drain costs;
    // two chunks at a time kept these four warps busy 98 % of the pass).
    const int q = warp & 3;
    const uint32_t lanes = static_cast<uint32_t>(q * 32) << 16;
    const int odd = lane >> 4;  // hi / lo part of rank 16 q + lane % 16 (lanes l, l + 16)
    const bool lstore = !(p.knobs & 8);
    const bool lred = (p.knobs & 512) != 0;
    unsigned long long tr[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const long long tstart = clock64();
    const int r = 16 * q + (lane & 15);
    int ul = 0;
    UnitIter it;
    for (it.init(w); it.more() && !wd_aborted<WD>(); it.next(), ++ul) {
      const int b = it.b, c = it.c;
      const int lb = ul & 1;
      mbar_wait_plain_t(&lfull[lb], static_cast<uint32_t>((ul >> 1) & 1), trc ? &tr[1] : nullptr);
      __syncwarp();
      tc_fence_after();
      uint32_t v[64];
      if (!(p.knobs & 64)) {
        tmem_ld64(tmem + lanes + cL + kRP * lb, v);
        tmem_wait_ld();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&lempty[lb]);  // the accumulator is in registers
      if (ul >= 2) mbar_wait<WD>(&sfree[lb], static_cast<uint32_t>(((ul >> 1) - 1) & 1));
      const uint32_t st_u = stage_u + lb * kStage + odd * (kRP * 16) + r * 16;
      if (!(p.knobs & 64)) {
#pragma unroll
        for (int c8 = 0; c8 < kTJ / 8; ++c8) {
          float o[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float keep = __uint_as_float(odd ? v[8 * c8 + 4 + e] : v[8 * c8 + e]);
            const float give = __uint_as_float(odd ? v[8 * c8 + e] : v[8 * c8 + 4 + e]);
            o[e] = keep + __shfl_xor_sync(0xffffffffu, give, 16);
          }
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(st_u + c8 * (kRP * 32)), "f"(o[0]), "f"(o[1]),
                       "f"(o[2]), "f"(o[3])
                       : "memory");
        }
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&sfull[lb]);
      if (warp == kIDrain - kLW && lane == 0) {  // the issuing lane: one bulk operation per unit
        mbar_wait<WD>(&sfull[lb], static_cast<uint32_t>((ul >> 1) & 1));
        if (lstore && !(p.knobs & 64) && !wd_aborted<WD>()) {
          float* dst = p.lpart + (static_cast<int64_t>(lred ? 0 : b) * w.nC + c) * (kRP * kTJ);
          if (lred)
            asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;\n" ::"l"(dst),
                         "r"(stage_u + lb * kStage), "r"(kStage)
                         : "memory");
          else
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst),
                         "r"(stage_u + lb * kStage), "r"(kStage)
                         : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
        if (ul >= 1) mbar_arrive(&sfree[lb ^ 1]);
      }
      __syncwarp();
    }
    if (warp == kIDrain - kLW && lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    if (lane == 0) atomicAdd(drains_out, 1u);
    if (p.trace && lane == 0) {
      tr[6] = static_cast<unsigned long long>(clock64() - tstart);
      for (int e = 0; e < 8; ++e) p.trace[(static_cast<int64_t>(cta) * 16 + warp) * 8 + e] = tr[e];
    }
  } else if (warp < kIDrain) {
    // ------------------------------------------------------------------ drains
    const int q = warp & 3, t = warp >> 2;
    const uint32_t lanes = static_cast<uint32_t>(q * 32) << 16;
    const int odd = lane >> 4;  // hi / lo part of rank 16 q + lane % 16 (lanes l, l + 16)
    const bool lstore = !(p.knobs & 8);
    const bool lred = (p.knobs & 512) != 0;  // left partials summed in L2 (red.add) into band slot 0
    float acc[kRP];
#pragma unroll
    for (int e = 0; e < kRP; ++e) acc[e] = 0.0f;
    int bc = 0, wc = 0;
    unsigned long long tr[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const long long tstart = clock64();
    int ul = 0;
    UnitIter it;
    for (it.init(w); it.more() && !wd_aborted<WD>(); it.next(), ++ul) {
      const int nt = it.nt;
      const bool mine = t < nt;
      const int b = it.b, c = it.c;
      const int lb = ul & 1;
      if (it.band_start()) {  // row tile t's KRl^T image into TMEM, once the previous band is done
        if (bc > 0) mbar_wait_plain(kl_free, static_cast<uint32_t>((bc - 1) & 1));
        __syncwarp();
        tc_fence_after();
        if (mine) {
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const uint4* src = reinterpret_cast<const uint4*>(static_cast<const __half*>(p.krl_img) +
                                                              (static_cast<int64_t>(b * A + t) * 128 + q * 32 + lane) *
                                                                  kTI) +
                               hh * 8;
            uint4 x[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) x[e] = __ldg(src + e);
            tmem_st32(tmem + lanes + cK + kRP * t + 32 * hh, x);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(kl_full);
      }
      if (mine && it.win_end()) {  // right window -> fp32 second level
        mbar_wait_plain_t(&rfull[t], static_cast<uint32_t>(wc & 1), trc ? &tr[0] : nullptr);
        __syncwarp();
        tc_fence_after();
#pragma unroll
        for (int c16 = 0; c16 < kRP / 16; ++c16) {
          if (p.knobs & 64) break;  // timing experiment: no TMEM reads in the drains
          uint32_t y[16];
          tmem_ld16(tmem + lanes + cRw * t + 16 * c16, y);
          if (STK) {  // main and correction halves
            uint32_t z[16];
            tmem_ld16(tmem + lanes + cRw * t + kRP + 16 * c16, z);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 16; ++e) acc[16 * c16 + e] += __uint_as_float(y[e]) + __uint_as_float(z[e]);
            continue;
          }
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e) acc[16 * c16 + e] += __uint_as_float(y[e]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&rempty[t]);
        ++wc;
      }
      // left: lanes l, l + 16 (hi, lo) of rank 16 q + l; 8-column chunks of the unit's
      // accumulator per warp (A = 3: t, t + 3, t + 6; A = 2: all eight, on the four
      // left-only warps), two chunks in flight.  The partial goes
      // through a 16 KB staging buffer [chunk][column half][64 r][4 j] (256 consecutive
      // bytes per half-warp store) and ONE bulk operation per unit: an L2 reduce-add into the band
      // slot (cp.reduce.async.bulk), or a bulk store of the band's own partial in
      // deterministic mode.  Per-lane red.global.add cost the drains ~0.3 ms at
      // A = 3 and 1.7 ms at A = 2 (their LSU issue rate, profiles/r02_f32i_knobs.txt).
      if (!STK) {
      mbar_wait_plain_t(&lfull[lb], static_cast<uint32_t>((ul >> 1) & 1), trc ? &tr[1] : nullptr);
      __syncwarp();
      tc_fence_after();
      const int r = 16 * q + (lane & 15);
      const uint32_t st_u = stage_u + lb * kStage + odd * (kRP * 16) + r * 16;
      const int lc0 = t, lcs = 3;
      const int ln = t == 2 ? 2 : 3;
      bool freed = ul < 2;
      for (int i0 = 0; i0 < ln; i0 += 2) {
        if (p.knobs & 64) {
          if (i0 + 2 >= ln) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&lempty[lb]);
          }
          continue;
        }
        const bool two = i0 + 1 < ln;
        const int ca = lc0 + i0 * lcs, cb = ca + lcs;
        uint32_t va[8], vb[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                     : "=r"(va[0]), "=r"(va[1]), "=r"(va[2]), "=r"(va[3]), "=r"(va[4]), "=r"(va[5]), "=r"(va[6]),
                       "=r"(va[7])
                     : "r"(tmem + lanes + cL + kRP * lb + 8 * ca));
        if (two)
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                       : "=r"(vb[0]), "=r"(vb[1]), "=r"(vb[2]), "=r"(vb[3]), "=r"(vb[4]), "=r"(vb[5]), "=r"(vb[6]),
                         "=r"(vb[7])
                       : "r"(tmem + lanes + cL + kRP * lb + 8 * cb));
        tmem_wait_ld();
        if (i0 + 2 >= ln) {  // the accumulator is in registers: the next unit's MMAs may overwrite it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&lempty[lb]);
        }
        float oa[4], ob[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float keep = __uint_as_float(odd ? va[4 + e] : va[e]);
          const float give = __uint_as_float(odd ? va[e] : va[4 + e]);
          oa[e] = keep + __shfl_xor_sync(0xffffffffu, give, 16);
        }
        if (two) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float keep = __uint_as_float(odd ? vb[4 + e] : vb[e]);
            const float give = __uint_as_float(odd ? vb[e] : vb[4 + e]);
            ob[e] = keep + __shfl_xor_sync(0xffffffffu, give, 16);
          }
        }
        if (!freed) {  // the bulk operation that read this buffer two units ago is done with it
          mbar_wait<WD>(&sfree[lb], static_cast<uint32_t>(((ul >> 1) - 1) & 1));
          freed = true;
        }
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(st_u + ca * (kRP * 32)), "f"(oa[0]), "f"(oa[1]),
                     "f"(oa[2]), "f"(oa[3])
                     : "memory");
        if (two)
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(st_u + cb * (kRP * 32)), "f"(ob[0]),
                       "f"(ob[1]), "f"(ob[2]), "f"(ob[3])
                       : "memory");
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&sfull[lb]);
      if (warp == kIDrain - kLW && lane == 0) {  // the issuing lane: one bulk operation per unit
        mbar_wait<WD>(&sfull[lb], static_cast<uint32_t>((ul >> 1) & 1));
        if (lstore && !(p.knobs & 64) && !wd_aborted<WD>()) {
          float* dst = p.lpart + (static_cast<int64_t>(lred ? 0 : b) * w.nC + c) * (kRP * kTJ);
          if (lred)
            asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;\n" ::"l"(dst),
                         "r"(stage_u + lb * kStage), "r"(kStage)
                         : "memory");
          else
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst),
                         "r"(stage_u + lb * kStage), "r"(kStage)
                         : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
        if (ul >= 1) mbar_arrive(&sfree[lb ^ 1]);
      }
      __syncwarp();
      }
      if (it.seg_end()) {
        if (mine) {
          const int64_t slot = (static_cast<int64_t>(cta) * p.slots + (b - seg0)) * A + t;  // CSR slot
          double* out = p.rpart + slot * kRP * kTI + q * 32 + lane;
#pragma unroll
          for (int e = 0; e < kRP; ++e) {
            out[e * kTI] = static_cast<double>(acc[e]) * unscale[e];
            acc[e] = 0.0f;
          }
        }
        ++bc;
      }
    }
    if (warp == kIDrain - kLW && lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");  // the bulk operations have landed
    if (lane == 0) atomicAdd(drains_out, 1u);  // the MMA warp's abort path waits for all drains
    if (p.trace && lane == 0) {
      tr[6] = static_cast<unsigned long long>(clock64() - tstart);
      for (int e = 0; e < 8; ++e) p.trace[(static_cast<int64_t>(cta) * 16 + warp) * 8 + e] = tr[e];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kIWMma) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(kTmemCols));
  }
}

// Operand image of an fp32 tensor view (J rows, K columns, column-major, leading
// dimension ldy): planes [2][K][LD] fp16, hi = fp16(s y), lo = fp16(s y - hi), rows
// J..LD-1 zero; s = the tensor's power-of-two scale.  Two rows per thread.
// chunked = 0: [2][K][LD] (column j: LD consecutive i); chunked = 1: [2][LD / 64][K][64]
// (64-row chunks of every column side by side, so one 64 i x 64 j TMA box is 8 KB
// of consecutive bytes instead of 64 rows 2 LD bytes apart)
__global__ void build_f16_image_kernel(const float* __restrict__ y, int64_t J, int64_t ldy, int64_t K, int64_t LD,
                                       const float* __restrict__ scale, __half2* __restrict__ img, int chunked) {
  const float sy = scale[0];
  const int64_t half = LD / 2, n = half * K, plane = n;  // in half2 units
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = e / half, i = 2 * (e - j * half);
    const float* col = y + j * ldy;
    const float a = i < J ? __ldcs(col + i) * sy : 0.0f;
    const float b = i + 1 < J ? __ldcs(col + i + 1) * sy : 0.0f;
    const __half2 hi = __floats2half2_rn(a, b);
    const float2 back = __half22float2(hi);
    const int64_t o = chunked ? ((i >> 6) * K * 64 + j * 64 + (i & 63)) / 2 : e;
    __stcs(img + o, hi);
    __stcs(img + plane + o, __floats2half2_rn(a - back.x, b - back.y));
  }
}

// The same image, eight rows per thread (two 16-byte loads, one 16-byte store per plane):
// for views whose columns start 16-byte aligned (ldy % 4 == 0); ~1.4x the scalar kernel's rate.
__global__ void build_f16_image_vec_kernel(const float* __restrict__ y, int64_t J, int64_t ldy, int64_t K, int64_t LD,
                                           const float* __restrict__ scale, __half* __restrict__ img, int chunked) {
  const float sy = scale[0];
  const int64_t oct = LD / 8, n = oct * K, plane = LD * K;  // plane in halves
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = e / oct, i = 8 * (e - j * oct);
    const float* col = y + j * ldy + i;
    float v[8];
    if (i + 8 <= J) {
      const float4 a = __ldcs(reinterpret_cast<const float4*>(col));
      const float4 b = __ldcs(reinterpret_cast<const float4*>(col) + 1);
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
      v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = i + k < J ? __ldcs(col + k) : 0.0f;
    }
    __half2 hi[4], lo[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float p = v[2 * k] * sy, q = v[2 * k + 1] * sy;
      hi[k] = __floats2half2_rn(p, q);
      const float2 back = __half22float2(hi[k]);
      lo[k] = __floats2half2_rn(p - back.x, q - back.y);
    }
    const int64_t o = chunked ? (i >> 6) * K * 64 + j * 64 + (i & 63) : j * LD + i;
    __stcs(reinterpret_cast<uint4*>(img + o), *reinterpret_cast<const uint4*>(hi));
    __stcs(reinterpret_cast<uint4*>(img + plane + o), *reinterpret_cast<const uint4*>(lo));
  }
}

// ---- Khatri-Rao operands of the fused pass, straight from the sorted factors ----
// (the north star's "never materialised when it can be recomputed": no fp64
// Khatri-Rao rows in HBM; each operand entry prod_m A_m[d_m, r] (kron.cpp:54-68)
// is formed once, scaled and split to fp16 hi / lo where it is stored)

// Column scales: one block per (side, rank column); max_x |KR[x, r]| =
// prod_m max_i |A_m[i, r]| (every index combination occurs), as a power of two.
__global__ void __launch_bounds__(128) kr_scale_cols_kernel(const KRSpec right, const KRSpec left, int R,
                                                            double* scale, double* inv) {
  const int side = blockIdx.x / kRP, r = blockIdx.x % kRP;
  const KRSpec& sp = side == 0 ? right : left;
  __shared__ double red[4];
  double bound = r < R ? 1.0 : 0.0;
  for (int m = 0; m < sp.n && r < R; ++m) {
    const int64_t I = sp.dims[m];
    double mx = 0.0;
    for (int64_t i = threadIdx.x; i < I; i += blockDim.x) mx = fmax(mx, fabs(__ldg(sp.A[m] + i + I * r)));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    mx = fmax(fmax(red[0], red[1]), fmax(red[2], red[3]));
    __syncthreads();
    bound *= mx;
  }
  if (threadIdx.x == 0) {
    int e = 0;
    if (bound > 0.0 && isfinite(bound)) frexp(bound, &e);
    scale[side * kRP + r] = ldexp(1.0, -e);
    inv[side * kRP + r] = ldexp(1.0, e);
  }
}

// Both operands in one launch.  Items [0, nR): right B tiles, K-major 128-byte
// swizzled (tile t = rows j in [64 t, 64 t + 64): [hi | lo][64 r][64 j], 16-byte
// chunk j8 of row r at chunk j8 ^ (r % 8)), 8 consecutive j per item.  Items
// [nR, nR + nL): the left KRl^T image [row tile][128 slots][128 i] (slot 2 r: hi
// of rank r, 2 r + 1: its lo), 8 consecutive i per item.  Rows past the view are 0.
__global__ void __launch_bounds__(256) kr_images_kernel(const KRSpec right, int64_t Kp, const KRSpec left, int64_t Jp,
                                                        int R, const double* __restrict__ scale, __half* rtiles,
                                                        int64_t nR, __half* limg, int64_t nL, int lane_halves) {
  int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  __half hi[8], lo[8];
  if (e < nR) {  // (t, r, j8): 8 consecutive items fill one 128-byte row of the tile
    const int j8 = static_cast<int>(e & 7);
    const int r = static_cast<int>((e >> 3) % kRP);
    const int64_t t = (e >> 3) / kRP;
    const double sc = scale[r];
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const int64_t j = t * kTJ + j8 * 8 + jj;
      const double x = (j < Kp && r < R) ? (j < (1LL << 31) ? kr_entry32(right, static_cast<uint32_t>(j), r) : kr_entry(right, j, r)) * sc : 0.0;
      hi[jj] = __double2half(x);
      lo[jj] = __double2half(x - static_cast<double>(__half2float(hi[jj])));
    }
    __half* dst = rtiles + t * (kKRBytes / 2) + static_cast<int64_t>(r) * kTJ + ((j8 ^ (r & 7)) << 3);
    *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(hi);
    *reinterpret_cast<uint4*>(dst + kTJ * kRP) = *reinterpret_cast<const uint4*>(lo);
    return;
  }
  e -= nR;
  if (e >= nL) return;
  const int i8 = static_cast<int>(e & 15);  // (t, r, i8)
  const int r = static_cast<int>((e >> 4) % kRP);
  const int64_t t = (e >> 4) / kRP;
  const double sc = scale[kRP + r];
#pragma unroll
  for (int ii = 0; ii < 8; ++ii) {
    const int64_t i = t * kTI + i8 * 8 + ii;
    const double x = (i < Jp && r < R) ? (i < (1LL << 31) ? kr_entry32(left, static_cast<uint32_t>(i), r) : kr_entry(left, i, r)) * sc : 0.0;
    hi[ii] = __double2half(x);
    lo[ii] = __double2half(x - static_cast<double>(__half2float(hi[ii])));
  }
  // slot of (rank r, part): 2 r + part, or (lane_halves, the operand-image kernel) hi in
  // TMEM lanes 0-15 of lane quarter r / 16 and lo in lanes 16-31: an M = 64 MMA reads
  // exactly the hi parts
  const int slot = lane_halves ? 32 * (r >> 4) + (r & 15) : 2 * r, lo_off = lane_halves ? 16 : 1;
  __half* dst = limg + (t * 128 + slot) * kTI + i8 * 8;
  *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(hi);
  *reinterpret_cast<uint4*>(dst + lo_off * kTI) = *reinterpret_cast<const uint4*>(lo);
}

}  // namespace

int seed_f32f_band_tiles() { return kA; }

int launch_seed_f32f(const Seed32FParams& p, const CUtensorMap* ymap, cudaStream_t s) {
  static unsigned long long cfg = 0;
  set_smem_attr(seed_f32f_kernel, kSmem, cfg);
  launch_k(seed_f32f_kernel, dim3(p.P), dim3(kThreads), kSmem, s, pdl_enabled(), p, *ymap);
  return 1;
}

template <bool WD, int A>
static void launch_f32i(const Seed32FParams& p, const CUtensorMap* imap, cudaStream_t s) {
  static unsigned long long cfg = 0;
  set_smem_attr(seed_f32i_kernel<WD, A>, kISmem, cfg);
  launch_k(seed_f32i_kernel<WD, A>, dim3(p.P), dim3(kIThreads), kISmem, s, pdl_enabled(), p, *imap);
}

int launch_seed_f32i(const Seed32FParams& p, const CUtensorMap* imap, cudaStream_t s) {
  if (p.band_tiles == 2) {
    if (p.watchdog) launch_f32i<true, 2>(p, imap, s);
    else launch_f32i<false, 2>(p, imap, s);
  } else {
    if (p.watchdog) launch_f32i<true, 3>(p, imap, s);
    else launch_f32i<false, 3>(p, imap, s);
  }
  return 1;
}

int64_t f16_image_ld(int64_t J) { return ceil_div(J, 64) * 64; }

int launch_build_f16_image(const float* y, int64_t J, int64_t ldy, int64_t K, const float* scale, void* img,
                           int num_sms, int chunked, cudaStream_t s) {
  if (ldy % 4 == 0 && (reinterpret_cast<uintptr_t>(y) & 15) == 0 && (reinterpret_cast<uintptr_t>(img) & 15) == 0)
    build_f16_image_vec_kernel<<<num_sms * 16, 256, 0, s>>>(y, J, ldy, K, f16_image_ld(J), scale,
                                                            static_cast<__half*>(img), chunked);
  else
    build_f16_image_kernel<<<num_sms * 8, 256, 0, s>>>(y, J, ldy, K, f16_image_ld(J), scale,
                                                       static_cast<__half2*>(img), chunked);
  return 1;
}

bool make_tensor_map_f16_image(CUtensorMap* out, const void* img, int64_t J, int64_t K, int chunked) {
  static PFN_cuTensorMapEncodeTiled encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return false;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
  }
  const int64_t LD = f16_image_ld(J);
  if ((reinterpret_cast<uintptr_t>(img) & 127) || K >= (1ll << 31) || LD >= (1ll << 31)) return false;
  // 4-D view (64 i in a chunk, i chunk, j, plane) of either layout; box 64 i (128 B,
  // swizzled) x 1 chunk x 64 j x 1 plane, coordinates (0, i0 / 64, j0, plane)
  const int64_t nIC = LD / 64;
  const cuuint64_t gdim[4] = {64, static_cast<cuuint64_t>(nIC), static_cast<cuuint64_t>(K), 2};
  const cuuint64_t gstride[3] = {
      static_cast<cuuint64_t>(chunked ? K * 128 : 128),  // i chunk
      static_cast<cuuint64_t>(chunked ? 128 : LD * 2),   // j
      static_cast<cuuint64_t>(LD * K) * 2};              // plane
  const cuuint32_t box[4] = {64, 1, 64, 1};
  const cuuint32_t estride[4] = {1, 1, 1, 1};
  return encode(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<void*>(img), gdim, gstride, box, estride,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int launch_kr_fused_operands(const KRSpec& right, int64_t Kp, const KRSpec& left, int64_t Jp, int R, double* scale,
                             double* inv, void* rtiles, void* limg, int lane_halves, cudaStream_t s) {
  kr_scale_cols_kernel<<<2 * kRP, 128, 0, s>>>(right, left, R, scale, inv);
  const int64_t nR = ceil_div(Kp, kTJ) * 8 * kRP, nL = ceil_div(Jp, kTI) * kRP * 16;
  kr_images_kernel<<<static_cast<unsigned>((nR + nL + 255) / 256), 256, 0, s>>>(
      right, Kp, left, Jp, R, scale, static_cast<__half*>(rtiles), nR, static_cast<__half*>(limg), nL, lane_halves);
  return 2;
}


}  // namespace cpdgpu
