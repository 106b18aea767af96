// seed_f32.cu — the split-point seed contractions for fp32 tensors on the
// 5th-generation tensor cores (tcgen05.mma kind::f16, accumulators in TMEM).
//
//   right pass  Rs[i, r] = sum_j Y[i + J j] KR(p+1..N)[j, r]   (mttkrp.cpp:149-163)
//   left pass   Ls[j, r] = sum_i Y[i + J j] KR(1..p)[i, r]     (mttkrp.cpp:195-210)
//
// fp32 accuracy from fp16 tensor cores: every operand x is split into
// x_hi = fp16(x) and x_lo = fp16(x - x_hi) (22 significant bits together), and
// a product is the three MMAs hi*hi + lo*hi + hi*lo accumulated in fp32 in TMEM
// (the dropped lo*lo term is ~2^-22 relative).  Y and every Khatri-Rao column
// are scaled by powers of two into [-1, 1] first (exact), and the fp32 TMEM
// accumulator is drained into fp64 registers every `chunk` k-tiles, so the
// long K = 90000 sums of config 5 keep ~1e-7 relative accuracy.
//
// One CTA per SM (persistent), 320 threads:
//   warp 8      producer: 2-D TMA of the fp32 Y tile + one bulk copy of the
//               pre-split Khatri-Rao tile per stage
//   warps 0-7   split each Y tile into fp16 hi and lo A operands written straight
//               into tensor memory (tcgen05.st; thread = A row = TMEM lane), then
//               drain the TMEM accumulators into fp64 registers and write the
//               per-CTA partial rows.  Warp w serves TMEM lanes 32 (w % 4).. and
//               K half / rank-column half w / 4.
//   warp 9      allocates TMEM and issues the MMAs (one elected lane):
//               D[tmem] += A[tmem] * B[smem], kind::f16, M = 128, N = 64, K = 16
//
// Shared memory then carries only the fp32 tile (TMA in, split out) and the
// Khatri-Rao B operand; the right tile (128 i x 64 j) is read down its columns
// (one row i per thread, conflict-free), the left tile (64 i x 128 j, fetched as
// two 128B-swizzled 32 i halves) along its rows.
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include "kernels.h"

namespace cpdgpu {
namespace {

constexpr int kBK = 64;             // K extent of one stage (j for right, i for left)
constexpr int kBM = 128;            // output rows per block (MMA M)
constexpr int kRP = 64;             // rank columns per pass (MMA N)
constexpr int kYTile = kBK * kBM * 4;           // fp32 tile bytes (32 KB)
constexpr int kKTile = 2 * kBK * kRP * 2;       // fp16 hi + lo Khatri-Rao tile (16 KB)
constexpr int kStages = 5;          // raw Y ring (fp32), released as soon as it is split
constexpr int kKStages = 3;         // Khatri-Rao tile ring, released by the MMAs
constexpr int kConv = 4;            // A operand ring in TMEM (fp16 hi + lo, 64 columns each)
constexpr int kLag = 2;             // a finished accumulation chunk is drained kLag tiles later
constexpr int kSplitWarps = 8;
constexpr int kThreads = (kSplitWarps + 2) * 32;
constexpr int kTmemA = 0;                  // A buffers: columns [0, 256)
constexpr int kTmemAcc = kConv * kBK;      // accumulators: 2 x [hi-product 64 | hi*lo 64] = [256, 512)
constexpr int kAccStride = 2 * kRP;
constexpr int kTmemCols = 512;

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
// L2 policies: Y streams through once (evict first); the Khatri-Rao tiles are
// re-read by every CTA (evict last), so they stay resident while Y streams.
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
// wait with cycle accounting (trace builds only: acc == nullptr costs nothing)
__device__ __forceinline__ void mbar_wait_t(uint64_t* bar, uint32_t parity, unsigned long long* acc) {
  if (acc) {
    const unsigned long long t0 = clock64();
    mbar_wait(bar, parity);
    *acc += clock64() - t0;
  } else {
    mbar_wait(bar, parity);
  }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
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

// tcgen05 shared-memory matrix descriptor: start, leading- and stride-dimension
// byte offsets, descriptor version 1 (sm_100), layout type (0: interleaved core
// matrices of 8 rows x 16 B, 2: 128-byte swizzle atoms of 8 rows x 128 B).
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout = 0) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFFu) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (static_cast<uint64_t>(layout) << 61);
}
// Instruction descriptor, kind::f16: fp16 A and B, fp32 D, M = 128, N = n.
__host__ __device__ constexpr uint32_t umma_idesc(bool a_mn_major, int n = kRP) {
  return (1u << 4) | (0u << 7) | (0u << 10) | ((a_mn_major ? 1u : 0u) << 15) | (0u << 16) |
         (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(kBM >> 4) << 24);
}
__device__ __forceinline__ void umma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};\n" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int c = 0; c < 32; ++c) v[c] = __uint_as_float(r[c]);
}

__device__ __forceinline__ uint32_t pack_half2(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}
// x -> (fp16 hi, fp16 lo) of 2 values, packed
__device__ __forceinline__ void split2(float a, float b, uint32_t& hi, uint32_t& lo) {
  hi = pack_half2(a, b);
  const float2 back = __half22float2(*reinterpret_cast<const __half2*>(&hi));
  lo = pack_half2(a - back.x, b - back.y);
}

// Right pass: raw tile [64 j][128 i] fp32 (512 B rows).  Thread = row i
// (= TMEM lane 32 (w % 4) + lane), K half h = w / 4: j in [32 h, 32 h + 32).
template <bool SCALE>
__device__ __forceinline__ void split_right(const unsigned char* raw, uint32_t tA, float sy, int warp, int lane) {
  const int i = (warp & 3) * 32 + lane, h = warp >> 2;
  const float* col = reinterpret_cast<const float*>(raw) + i + (32 * h) * kBM;
  uint32_t hw[16], lw[16];
#pragma unroll
  for (int jj = 0; jj < 16; ++jj) {
    float x0 = col[(2 * jj) * kBM], x1 = col[(2 * jj + 1) * kBM];
    if (SCALE) {
      x0 *= sy;
      x1 *= sy;
    }
    split2(x0, x1, hw[jj], lw[jj]);
  }
  const uint32_t lanes = static_cast<uint32_t>((warp & 3) * 32) << 16;
  tmem_st16(tA + lanes + 16 * h, hw);
  tmem_st16(tA + lanes + 32 + 16 * h, lw);
}
// Left pass: raw tile = two 128B-swizzled halves [128 j][32 i] fp32 (128 B rows,
// 16-B chunk c of row j at c ^ (j % 8)).  Thread = row j, K half h = w / 4.
template <bool SCALE>
__device__ __forceinline__ void split_left(const unsigned char* raw, uint32_t tA, float sy, int warp, int lane) {
  const int j = (warp & 3) * 32 + lane, h = warp >> 2;
  const unsigned char* row = raw + h * (kYTile / 2) + j * 128;
  uint32_t hw[16], lw[16];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    float4 v = *reinterpret_cast<const float4*>(row + ((c ^ (j & 7)) << 4));
    if (SCALE) {
      v.x *= sy; v.y *= sy; v.z *= sy; v.w *= sy;
    }
    split2(v.x, v.y, hw[2 * c], lw[2 * c]);
    split2(v.z, v.w, hw[2 * c + 1], lw[2 * c + 1]);
  }
  const uint32_t lanes = static_cast<uint32_t>((warp & 3) * 32) << 16;
  tmem_st16(tA + lanes + 16 * h, hw);
  tmem_st16(tA + lanes + 32 + 16 * h, lw);
}

// Walk of one CTA's units [a, a + n) (unit = block * nK + k-tile): segment
// (one output block) and chunk (fp32 accumulation window) boundaries.
struct Walk {
  int64_t nK;
  int chunk;
  int64_t t;  // k-tile index of the current unit
  __device__ Walk(int64_t a, int64_t nk, int ch) : nK(nk), chunk(ch), t(a % nk) {}
  __device__ bool seg_start(int k) const { return k == 0 || t == 0; }
  __device__ bool next_starts() const { return t + 1 == nK; }
  __device__ void advance() { t = (t + 1 == nK) ? 0 : t + 1; }
};

template <int LEFT>
__global__ void __launch_bounds__(kThreads, 1)
    seed_f32_kernel(const Seed32Params p, const __grid_constant__ CUtensorMap ymap) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cta = blockIdx.x;
  const int64_t a = static_cast<int64_t>(cta) * p.units / p.P;
  const int64_t b = static_cast<int64_t>(cta + 1) * p.units / p.P;
  const int n = static_cast<int>(b - a);
  Walk w(a, p.nK, p.chunk);
  constexpr int kProducer = kSplitWarps, kMma = kSplitWarps + 1;

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  unsigned char* ytiles = base;                          // [kStages][32 KB] fp32
  unsigned char* ktiles = ytiles + kStages * kYTile;     // [kKStages][16 KB]
  uint64_t* bars = reinterpret_cast<uint64_t*>(ktiles + kKStages * kKTile);
  uint64_t* full = bars;                   // raw Y landed              (1 + tx)
  uint64_t* empty = full + kStages;        // raw Y split               (8 warps)
  uint64_t* kfull = empty + kStages;       // Khatri-Rao tile landed    (1 + tx)
  uint64_t* kempty = kfull + kKStages;     // Khatri-Rao tile consumed  (MMA commit)
  uint64_t* cfull = kempty + kKStages;     // A operands in TMEM        (8 warps)
  uint64_t* cempty = cfull + kConv;        // A operands consumed       (MMA commit)
  uint64_t* accfull = cempty + kConv;      // [2] chunk accumulated     (commit)
  uint64_t* accempty = accfull + 2;        // [2] chunk drained         (8 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accempty + 2);
  double* unscale = reinterpret_cast<double*>(tmem_slot + 2);  // [kRP]

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kSplitWarps);
    }
    for (int s = 0; s < kKStages; ++s) {
      mbar_init(&kfull[s], 1);
      mbar_init(&kempty[s], 1);
    }
    for (int c = 0; c < kConv; ++c) {
      mbar_init(&cfull[c], kSplitWarps);
      mbar_init(&cempty[c], 1);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&accfull[q], 1);
      mbar_init(&accempty[q], kSplitWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp != kProducer) pdl_wait();  // scales and partial buffers: preceding kernels
  if (tid < kRP) unscale[tid] = p.inv_scale_y[0] * p.inv_scale_kr[tid];
  if (warp == kMma) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (warp == kProducer && lane == 0)
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&ymap)));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // optional per-warp cycle trace: [cta][warp][wait0, wait1, wait2, total]
  unsigned long long* tr = p.trace ? p.trace + (static_cast<int64_t>(cta) * (kThreads / 32) + warp) * 8 : nullptr;
  unsigned long long tw[5] = {0, 0, 0, 0, 0};
  const unsigned long long tstart = clock64();

  if (warp == kProducer) {
    // ------------------------------------------------------------------ producer
    if (lane == 0) {
      // Y runs up to kStages tiles ahead, the Khatri-Rao tiles kKStages ahead.
      // Y does not depend on the preceding kernel (PDL): the first stages are
      // requested before the wait.
      const uint64_t pol_y = policy_evict_first(), pol_k = policy_evict_last();
      int kk = 0;
      const int early = n < kStages ? n : kStages;
      for (int k = 0; k < early; ++k) {
        const int64_t u = a + k, blk = u / p.nK, t = u - blk * p.nK;
        mbar_arrive_tx(&full[k], kYTile);
        if (LEFT) {
          tma_load_2d(ytiles + k * kYTile, &ymap, static_cast<int>(t * kBK), static_cast<int>(blk * kBM), &full[k],
                      pol_y);
          tma_load_2d(ytiles + k * kYTile + kYTile / 2, &ymap, static_cast<int>(t * kBK + 32),
                      static_cast<int>(blk * kBM), &full[k], pol_y);
        } else {
          tma_load_2d(ytiles + k * kYTile, &ymap, static_cast<int>(blk * kBM), static_cast<int>(t * kBK), &full[k],
                      pol_y);
        }
      }
      pdl_wait();
      for (int k = 0; k < n; ++k) {
        if (k < early) {  // Y already requested
          for (; kk < n && kk <= k - (kStages - kKStages); ++kk) {
            const int sk = kk % kKStages;
            if (kk >= kKStages) mbar_wait(&kempty[sk], ((kk / kKStages) - 1) & 1);
            const int64_t uk = a + kk, tk = uk - (uk / p.nK) * p.nK;
            mbar_arrive_tx(&kfull[sk], kKTile);
            bulk_load(ktiles + sk * kKTile, p.kr_tiles + tk * kKTile, kKTile, &kfull[sk], pol_k);
          }
          continue;
        }
        const int s = k % kStages;
        if (k >= kStages) mbar_wait_t(&empty[s], ((k / kStages) - 1) & 1, tr ? &tw[0] : nullptr);
        const int64_t u = a + k, blk = u / p.nK, t = u - blk * p.nK;
        mbar_arrive_tx(&full[s], kYTile);
        if (LEFT) {  // rows i in [64 t, +64) as two 32-row halves, columns j in [128 blk, +128)
          tma_load_2d(ytiles + s * kYTile, &ymap, static_cast<int>(t * kBK), static_cast<int>(blk * kBM), &full[s],
                      pol_y);
          tma_load_2d(ytiles + s * kYTile + kYTile / 2, &ymap, static_cast<int>(t * kBK + 32),
                      static_cast<int>(blk * kBM), &full[s], pol_y);
        } else {     // rows i in [128 blk, +128), columns j in [64 t, +64)
          tma_load_2d(ytiles + s * kYTile, &ymap, static_cast<int>(blk * kBM), static_cast<int>(t * kBK), &full[s],
                      pol_y);
        }
        for (; kk < n && kk <= k - (kStages - kKStages); ++kk) {
          const int sk = kk % kKStages;
          if (kk >= kKStages) mbar_wait(&kempty[sk], ((kk / kKStages) - 1) & 1);
          const int64_t uk = a + kk, tk = uk - (uk / p.nK) * p.nK;
          mbar_arrive_tx(&kfull[sk], kKTile);
          bulk_load(ktiles + sk * kKTile, p.kr_tiles + tk * kKTile, kKTile, &kfull[sk], pol_k);
        }
      }
      for (; kk < n; ++kk) {
        const int sk = kk % kKStages;
        if (kk >= kKStages) mbar_wait(&kempty[sk], ((kk / kKStages) - 1) & 1);
        const int64_t uk = a + kk, tk = uk - (uk / p.nK) * p.nK;
        mbar_arrive_tx(&kfull[sk], kKTile);
        bulk_load(ktiles + sk * kKTile, p.kr_tiles + tk * kKTile, kKTile, &kfull[sk], pol_k);
      }
    }
  } else if (warp == kMma) {
    // ------------------------------------------------------------------ MMA issuer
    // A from TMEM (K-major rows).  Per k-step: A_hi x [B_hi | B_lo] as one N = 128 MMA
    // (the hi and lo Khatri-Rao pieces are adjacent rows of one swizzled operand) into
    // accumulator columns [0, 128), then A_lo x B_hi (N = 64) into [0, 64); the drain
    // adds the two halves.  8 MMAs per tile instead of 12, and A_hi is read once.
    constexpr uint32_t idesc128 = umma_idesc(false, 2 * kRP), idesc64 = umma_idesc(false, kRP);
    // B (Khatri-Rao, K-major, 128B swizzle): SBO next 8 r = 1 KB, +32 B per 16 K inside the atom
    constexpr uint32_t b_lbo = 16, b_sbo = 1024, b_kstep = 32;
    constexpr uint32_t b_layout = 2;  // SWIZZLE_128B
    int q = -1, pos = 0;
    for (int k = 0; k < n; ++k) {
      const int sk = k % kKStages, c = k % kConv;
      if (w.seg_start(k) || pos == w.chunk) {  // new accumulation chunk
        ++q;
        pos = 0;
        if (q >= 2) {
          mbar_wait_t(&accempty[q & 1], ((q >> 1) - 1) & 1, tr ? &tw[0] : nullptr);
          tc_fence_after();
        }
      }
      mbar_wait_t(&cfull[c], (k / kConv) & 1, tr ? &tw[1] : nullptr);
      mbar_wait_t(&kfull[sk], (k / kKStages) & 1, tr ? &tw[2] : nullptr);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t d = tmem + static_cast<uint32_t>(kTmemAcc + (q & 1) * kAccStride);
        const uint32_t ahi = tmem + static_cast<uint32_t>(kTmemA + c * kBK), alo = ahi + kBK / 2;
        const uint32_t kb = smem_u32(ktiles + sk * kKTile);
#pragma unroll
        for (int ks = 0; ks < kBK / 16; ++ks) {  // K = 16 per MMA = 8 packed TMEM columns
          const uint64_t ball = umma_desc(kb + ks * b_kstep, b_lbo, b_sbo, b_layout);  // rows: hi 0..63, lo 64..127
          umma_f16_ts(d, ahi + 8 * ks, ball, idesc128, (pos > 0 || ks > 0) ? 1u : 0u);
          if (!(p.debug & 1)) umma_f16_ts(d, alo + 8 * ks, ball, idesc64, 1u);
        }
        umma_commit(&kempty[sk]);
        umma_commit(&cempty[c]);
      }
      __syncwarp();
      ++pos;
      const bool chunk_end = (k == n - 1) || w.next_starts() || pos == w.chunk;
      w.advance();
      if (chunk_end && lane == 0) umma_commit(&accfull[q & 1]);
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------------ split + drain
    double acc[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) acc[c] = 0.0;
    const float sy = p.scale_y[0];
    const bool scale = sy != 1.0f;
    const int sp = warp & 3, colh = warp >> 2;  // TMEM lane quarter, rank-column half
    const uint32_t lane_base = static_cast<uint32_t>(sp * 32) << 16;
    int q = -1, pos = 0, seg = -1;
    // finished chunks waiting to be drained (FIFO, drained in order kLag tiles later)
    int fq[4], fk[4], fseg[4];
    bool flast[4];
    int fh = 0, ft = 0;
    for (int k = 0; k <= n; ++k) {
      if (k < n) {
        const int s = k % kStages, c = k % kConv;
        if (w.seg_start(k)) ++seg;
        if (w.seg_start(k) || pos == w.chunk) {
          ++q;
          pos = 0;
        }
        mbar_wait_t(&full[s], (k / kStages) & 1, tr ? &tw[0] : nullptr);
        if (k >= kConv) {
          mbar_wait_t(&cempty[c], ((k / kConv) - 1) & 1, tr ? &tw[1] : nullptr);
          tc_fence_after();
        }
        const unsigned long long ts0 = tr ? clock64() : 0;
        const uint32_t tA = tmem + static_cast<uint32_t>(kTmemA + c * kBK);
        const unsigned char* raw = ytiles + s * kYTile;
        if (p.debug & 2) {
        } else if (LEFT) {
          if (scale) split_left<true>(raw, tA, sy, warp, lane);
          else split_left<false>(raw, tA, sy, warp, lane);
        } else {
          if (scale) split_right<true>(raw, tA, sy, warp, lane);
          else split_right<false>(raw, tA, sy, warp, lane);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (tr) tw[3] += clock64() - ts0;
        if (lane == 0) {
          mbar_arrive(&empty[s]);
          mbar_arrive(&cfull[c]);
        }
      }
      // drain finished chunks kLag tiles late, so the MMAs of the newer tiles overlap it
      while (fh < ft && (k == n || fk[fh & 3] + kLag <= k)) {
        const int e = fh & 3;
        const int dq = fq[e];
        mbar_wait_t(&accfull[dq & 1], (dq >> 1) & 1, tr ? &tw[2] : nullptr);
        __syncwarp();  // tcgen05.ld is .sync.aligned: reconverge after the spin
        tc_fence_after();
        const unsigned long long td0 = tr ? clock64() : 0;
        float v[32], u[32];
        tmem_ld32(tmem + lane_base + static_cast<uint32_t>(kTmemAcc + (dq & 1) * kAccStride + colh * 32), v);
        tmem_ld32(tmem + lane_base + static_cast<uint32_t>(kTmemAcc + (dq & 1) * kAccStride + kRP + colh * 32), u);
#pragma unroll
        for (int c = 0; c < 32; ++c) acc[c] += static_cast<double>(v[c]) + static_cast<double>(u[c]);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&accempty[dq & 1]);
        if (flast[e]) {  // block segment finished: unscaled fp64 partial rows
          double* out = p.part + (static_cast<int64_t>(cta) * p.slots + fseg[e]) * kRP * kBM +
                        static_cast<int64_t>(colh * 32) * kBM + sp * 32 + lane;
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            out[c * kBM] = acc[c] * unscale[colh * 32 + c];
            acc[c] = 0.0;
          }
        }
        ++fh;
        if (tr) tw[4] += clock64() - td0;
      }
      if (k < n) {
        ++pos;
        const bool seg_end = (k == n - 1) || w.next_starts();
        w.advance();
        if (seg_end || pos == w.chunk) {
          const int e = ft & 3;
          fq[e] = q;
          fk[e] = k;
          flast[e] = seg_end;
          fseg[e] = seg;
          ++ft;
        }
      }
    }
  }
  if (tr && lane == 0) {
    tr[0] = tw[0];
    tr[1] = tw[1];
    tr[2] = tw[2];
    tr[3] = clock64() - tstart;
    tr[4] = tw[3];
    tr[5] = tw[4];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMma) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(kTmemCols));
  }
}

// ---- Khatri-Rao operand preparation ----------------------------------------------

// Power-of-two column scales: max_x |KR[x, r]| = prod_m max_i |A_m[i, r]| (the
// Khatri-Rao product runs over every index combination), scaled into [0.5, 1).
__global__ void kr_scale_kernel(const KRSpec right, const KRSpec left, int R, double* scale, double* inv) {
  const int r = threadIdx.x;
  if (r >= kRP) return;
  for (int side = 0; side < 2; ++side) {
    const KRSpec& s = side == 0 ? right : left;
    double bound = r < R ? 1.0 : 0.0;
    for (int m = 0; m < s.n && r < R; ++m) {
      double mx = 0.0;
      for (int64_t i = 0; i < s.dims[m]; ++i) mx = fmax(mx, fabs(s.A[m][i + s.dims[m] * r]));
      bound *= mx;
    }
    int e = 0;
    if (bound > 0.0 && isfinite(bound)) frexp(bound, &e);
    scale[side * kRP + r] = ldexp(1.0, -e);
    inv[side * kRP + r] = ldexp(1.0, e);
  }
}

// fp64 Khatri-Rao rows [L][ld] -> scaled fp16 hi / lo tiles laid out as the
// K-major B operand with 128-byte swizzle: tile t = rows [64 t, 64 t + 64),
// [piece][r (64)][64 K values, 16-byte chunks XOR-swizzled by r % 8].
__global__ void kr_split_kernel(const double* __restrict__ rows, int64_t L, int ld, const double* __restrict__ scale,
                                __half* __restrict__ tiles, int64_t ntiles) {
  const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;  // (t, j8, r8, rr)
  if (e >= ntiles * 8 * (kRP / 8) * 8) return;
  const int rr = static_cast<int>(e & 7);
  const int r8 = static_cast<int>((e >> 3) % (kRP / 8));
  const int64_t rest = (e >> 3) / (kRP / 8);
  const int j8 = static_cast<int>(rest & 7);
  const int64_t t = rest >> 3;
  const int r = r8 * 8 + rr;
  const double sc = scale[r];
  __half hi[8], lo[8];
#pragma unroll
  for (int jj = 0; jj < 8; ++jj) {
    const int64_t j = t * kBK + j8 * 8 + jj;
    const double x = (j < L && r < ld) ? rows[j * ld + r] * sc : 0.0;
    hi[jj] = __double2half(x);
    lo[jj] = __double2half(x - static_cast<double>(__half2float(hi[jj])));
  }
  // K-major 128B-swizzled rows: row r holds its 64 K values (128 B); 16-byte chunk j8
  // of row r sits at chunk j8 ^ (r % 8) (atoms of 8 rows x 128 B)
  __half* dst = tiles + t * (kKTile / 2) + static_cast<int64_t>(r) * kBK + ((j8 ^ (r & 7)) << 3);
  *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(hi);
  *reinterpret_cast<uint4*>(dst + kBK * kRP) = *reinterpret_cast<const uint4*>(lo);
}

// Y scale: power of two taking max |Y| into [0.5, 1).
__global__ void absmax_f32_kernel(const float* __restrict__ y, int64_t n, unsigned int* out) {
  float m = 0.0f;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    m = fmaxf(m, fabsf(y[i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));
}
__global__ void y_scale_kernel(const unsigned int* amax, float* scale, double* inv) {
  const float m = __uint_as_float(*amax);
  int e = 0;
  if (m > 0.0f && isfinite(m)) frexpf(m, &e);
  scale[0] = ldexpf(1.0f, -e);
  inv[0] = ldexp(1.0, e);
}

// Rows [J, J8) of a padded copy stay zero; columns are copied as is.
__global__ void pad_rows_f32_kernel(const float* __restrict__ src, float* __restrict__ dst, int64_t J, int64_t J8,
                                    int64_t K) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < J8 * K;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = e / J8, i = e - j * J8;
    dst[e] = i < J ? src[i + J * j] : 0.0f;
  }
}

}  // namespace

size_t seed_f32_smem_bytes() {
  return 1024 + kStages * kYTile + kKStages * kKTile + 256 + kRP * sizeof(double);
}
int seed_f32_rank_cols() { return kRP; }
int64_t seed_f32_tile_bytes() { return kKTile; }

int launch_seed_f32(const Seed32Params& p, const CUtensorMap* ymap, int left, cudaStream_t s) {
  const size_t smem = seed_f32_smem_bytes();
  if (left) {
    static unsigned long long cfg = 0;
    set_smem_attr(seed_f32_kernel<1>, static_cast<int>(smem), cfg);
    launch_k(seed_f32_kernel<1>, dim3(p.P), dim3(kThreads), smem, s, pdl_enabled(), p, *ymap);
  } else {
    static unsigned long long cfg = 0;
    set_smem_attr(seed_f32_kernel<0>, static_cast<int>(smem), cfg);
    launch_k(seed_f32_kernel<0>, dim3(p.P), dim3(kThreads), smem, s, pdl_enabled(), p, *ymap);
  }
  return 1;
}

int launch_kr_scale(const KRSpec& right, const KRSpec& left, int R, double* scale, double* inv, cudaStream_t s) {
  kr_scale_kernel<<<1, kRP, 0, s>>>(right, left, R, scale, inv);
  return 1;
}

int launch_kr_split(const double* rows, int64_t L, int ld, const double* scale, void* tiles, cudaStream_t s) {
  const int64_t ntiles = (L + kBK - 1) / kBK;
  const int64_t work = ntiles * 8 * (kRP / 8) * 8;
  kr_split_kernel<<<static_cast<unsigned>((work + 255) / 256), 256, 0, s>>>(rows, L, ld, scale,
                                                                             static_cast<__half*>(tiles), ntiles);
  return 1;
}

int launch_y_scale(const float* y, int64_t n, unsigned int* amax_scratch, float* scale, double* inv,
                   int num_sms, cudaStream_t s) {
  cudaMemsetAsync(amax_scratch, 0, sizeof(unsigned int), s);
  absmax_f32_kernel<<<num_sms * 8, 256, 0, s>>>(y, n, amax_scratch);
  y_scale_kernel<<<1, 1, 0, s>>>(amax_scratch, scale, inv);
  return 2;
}

int launch_pad_rows_f32(const float* src, float* dst, int64_t J, int64_t J8, int64_t K, int num_sms,
                        cudaStream_t s) {
  pad_rows_f32_kernel<<<num_sms * 8, 256, 0, s>>>(src, dst, J, J8, K);
  return 1;
}

bool make_tensor_map_y32(CUtensorMap* out, const void* base, int64_t J8, int64_t K, int left) {
  static PFN_cuTensorMapEncodeTiled encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return false;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
  }
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (J8 & 7) || K >= (1ll << 32) || J8 >= (1ll << 32)) return false;
  // J8 x K column-major fp32; right tiles 128 i x 64 j, left tiles 64 i x 128 j
  const cuuint64_t gdim[2] = {static_cast<cuuint64_t>(J8), static_cast<cuuint64_t>(K)};
  const cuuint64_t gstride[1] = {static_cast<cuuint64_t>(J8) * 4};
  const cuuint32_t box[2] = {left ? 32u : 128u, left ? 128u : 64u};
  const cuuint32_t estride[2] = {1, 1};
  return encode(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), gdim, gstride, box, estride,
                CU_TENSOR_MAP_INTERLEAVE_NONE, left ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                // no 256 B promotion: column starts are only 64 B aligned in general (J * 4 bytes apart),
                // and a promoted line straddling the neighbouring row block is evicted before that block
                // (another CTA) reads it
                CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace cpdgpu
