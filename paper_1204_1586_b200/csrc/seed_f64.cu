// seed_f64.cu — fused two-sided split-point contraction (the two seed GEMMs
// of Algorithm 2) in fp64 on the B200 FP64 tensor pipe (DMMA).
//
// Reference: the right seed  cache.right = Y_(1:p) * KR(p+1..N)  (mttkrp.cpp:149-163)
// and the left seed          cache.left  = Y_(1:p)^T * KR(1..p)   (mttkrp.cpp:195-210).
// Both read the same J_p x K_p column-major view of Y, so in gradient mode one
// pass over HBM feeds both products ("fused", MODE 3).  In ALS mode the left
// seed must see factors the right phase already updated (mttkrp.cpp:143,203),
// so the two products run as separate passes (MODE 1, MODE 2).
//
// Design:
//  * Warp-specialised persistent CTA: warp 8 is the producer, warps 0-7 consume.
//    Per tile (TI rows x 32 columns of Y) the producer issues two 2-D TMA loads
//    onto one mbarrier: the Y tile and the tile's 32 Khatri-Rao rows
//    KR(p+1..N) (kron_range_column, kron.cpp:54-68, later modes outermost).
//    STAGES-deep ring; out-of-range rows/columns arrive zero-filled.
//  * The Khatri-Rao rows are built by a pre-pass kernel (kr_materialize) into a
//    small L2-resident buffer (K_p x R and J_p x R, <= 1% of Y) instead of inside
//    this kernel: on B200 fp64 multiplies issue to the same FP64 datapath as
//    DMMA, and generating them here made the producer warp the bottleneck
//    (measured 87% busy on config 3, profiles/r01_seed_trace.txt).
//  * Consumers run mma.sync.m8n8k4.f64 (DMMA): measured 37.1 TF/s on B200 vs
//    36.7 TF/s for DFMA, with a sixteenth of the issue slots.  Right product
//    Rs = Y * KR_r (M = rows, N = rank, K = columns); left product as
//    Ls^T = KR_l^T * Y (M = rank, N = columns, K = rows).
//  * MODE 3 splits the consumers by product (warps 0-3 right, 4-7 left); right
//    partials persist in registers over a row block and go out once per (CTA,
//    row block) slot; the left warps split each tile's rows four ways with their
//    KR_l slice held in registers and combine once per tile (left_reg_role),
//    left partials go out once per tile and row block.  tail.cu reduces both in a fixed order, so results are
//    bitwise reproducible.
#include <cstdint>
#include <cstring>

#include <cudaTypedefs.h>

#include "common.cuh"
#include "kernels.h"

namespace cpdgpu {
namespace {

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

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
// 2-D TMA load with an L2 policy: Y streams through once (evict first), the
// Khatri-Rao rows are re-read for every row block (evict last).
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                            bool stream = false) {
  uint64_t pol;
  if (stream)
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  else
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, 256;\n" ::: "memory"); }

__device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
  return v;
}

// tile -> (row block, column tile) without the 64-bit division helper call
__device__ __forceinline__ int64_t tile_rb(int64_t tile, int64_t nCT) {
  if ((static_cast<uint64_t>(tile) >> 32) == 0 && (static_cast<uint64_t>(nCT) >> 32) == 0)
    return static_cast<uint32_t>(tile) / static_cast<uint32_t>(nCT);
  return tile / nCT;
}

constexpr int kTJ = 32;          // columns per tile
constexpr int kConsumers = 8;    // consumer warps
constexpr int kThreads = 288;    // + 1 producer warp

// ---- consumer roles ------------------------------------------------------------
struct Ring {
  uint64_t* full;
  uint64_t* empty;
  double* Ys;   // [STAGES][32 * LDY]
  double* KRr;  // [STAGES][32 * LDK]
  double* KRl;  // [TI * LDK]
  double* red;  // MODE 2: [2][4 * 32 * NT * 2]; MODE 3: [2][4][3][NT][2][32]
  int stages, TI, LDY, LDK;
};

// KR(1..p) rows of row block rb from the pre-built buffer (all 256 consumers).
__device__ __forceinline__ void load_krl(const SeedParams& p, const Ring& q, int64_t rb, int tid,
                                         int nthreads = kConsumers * 32) {
  const int64_t row0 = rb * q.TI;
  const int rows = static_cast<int>(min64(q.TI, p.J - row0));
  // 16-byte pieces (LDK is even), eight independent loads in flight per thread
  const double2* src = reinterpret_cast<const double2*>(p.KRl_g + row0 * q.LDK);
  double2* dst = reinterpret_cast<double2*>(q.KRl);
  const int n2 = (q.TI * q.LDK) >> 1, valid = (rows * q.LDK) >> 1;
#pragma unroll 8
  for (int e = tid; e < n2; e += nthreads) dst[e] = e < valid ? __ldg(src + e) : make_double2(0.0, 0.0);
}

// Row-block bookkeeping shared by every role: all consumers meet at the named
// barrier, the right roles flush, KR_l is refreshed, and they meet again.
template <typename Flush>
__device__ __forceinline__ void row_block_change(const SeedParams& p, const Ring& q, int64_t rb, int64_t& cur_rb,
                                                 bool need_krl, int tid, Flush&& flush) {
  consumer_sync();
  if (cur_rb >= 0) flush(cur_rb);
  if (need_krl) load_krl(p, q, rb, tid);
  consumer_sync();
  cur_rb = rb;
}

// Right product on W warps; this warp owns MC row fragments mf = warp + W m.
// Rs[i, r] += sum_j Y[i, j] KR_r[j, r] over the CTA's tiles; operands double-buffered.
template <int NT, int MC, int W>
__device__ void right_role(const SeedParams& p, const Ring& q, int64_t t0, int ntiles, int cta, int warp, int lane,
                           int tid, bool need_krl, unsigned long long& cw) {
  constexpr int RP = NT * 8;
  const int g = lane >> 2, t = lane & 3;
  constexpr int LDK = seed_ldk(NT);
  const int LDY = q.LDY, TI = q.TI;
  double acc[MC > 0 ? MC : 1][NT][2];
#pragma unroll
  for (int m = 0; m < MC; ++m)
#pragma unroll
    for (int nb = 0; nb < NT; ++nb) acc[m][nb][0] = acc[m][nb][1] = 0.0;
  const int64_t slot_rb0 = t0 / p.nCT;
  auto flush = [&](int64_t rb) {
    double* dst = p.Rpart + (static_cast<int64_t>(cta) * p.slots + (rb - slot_rb0)) * RP * TI;
#pragma unroll
    for (int m = 0; m < MC; ++m) {
      const int i = (warp + W * m) * 8 + g;
#pragma unroll
      for (int nb = 0; nb < NT; ++nb) {
        const int r = nb * 8 + 2 * t;
        dst[r * TI + i] = acc[m][nb][0];
        dst[(r + 1) * TI + i] = acc[m][nb][1];
        acc[m][nb][0] = acc[m][nb][1] = 0.0;
      }
    }
  };
  int64_t cur_rb = -1;
  for (int k = 0; k < ntiles; ++k) {
    const int s = k % q.stages;
    const int64_t tile = t0 + k;
    const int64_t rb = tile_rb(tile, p.nCT);
    if (rb != cur_rb) {  // the right product never reads KR_l: flush and go on
      if (cur_rb >= 0) flush(cur_rb);
      cur_rb = rb;
    }
    const unsigned long long w0 = clock64();
    mbar_wait(&q.full[s], (k / q.stages) & 1);
    cw += clock64() - w0;
    const double* ya = q.Ys + s * kTJ * LDY + warp * 8 + g + t * LDY;
    const double* kb = q.KRr + s * kTJ * LDK + t * LDK + g;
    double a[2][MC > 0 ? MC : 1], b[2][NT];
#pragma unroll
    for (int m = 0; m < MC; ++m) a[0][m] = ya[W * 8 * m];
#pragma unroll
    for (int nb = 0; nb < NT; ++nb) b[0][nb] = kb[nb * 8];
#pragma unroll
    for (int ks = 0; ks < kTJ / 4; ++ks) {
      const int cur = ks & 1, nxt = cur ^ 1;
      if (ks + 1 < kTJ / 4) {
#pragma unroll
        for (int m = 0; m < MC; ++m) a[nxt][m] = ya[(ks + 1) * 4 * LDY + W * 8 * m];
#pragma unroll
        for (int nb = 0; nb < NT; ++nb) b[nxt][nb] = kb[(ks + 1) * 4 * LDK + nb * 8];
      }
#pragma unroll
      for (int m = 0; m < MC; ++m)
#pragma unroll
        for (int nb = 0; nb < NT; ++nb) dmma(acc[m][nb], a[cur][m], b[cur][nb]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&q.empty[s]);
  }
  if (cur_rb >= 0) flush(cur_rb);
}

// Left product of the fused pass, alternating tiles between two warp pairs:
// pair (k & 1) takes tile k, warp c of the pair the 8-column fragments 2c and
// 2c + 1 over the full K = TI rows.  A k-step costs two Y fragment loads and NT
// Khatri-Rao fragment loads for 2 NT DMMAs; two k-interleaved accumulator sets
// give 4 NT independent chains.  No per-tile synchronisation: every tile is
// released by the four right warps and the two warps of its pair (the empty
// barriers count 6 arrivals in MODE 3).  All four left warps walk every tile
// index so they meet at each row-block change to refresh KR_l.
template <int NT>
__device__ void left_pair_role(const SeedParams& p, const Ring& q, int64_t t0, int ntiles, int lw, int lane,
                               unsigned long long& cw) {
  constexpr int LDK = seed_ldk(NT);
  const int g = lane >> 2, t = lane & 3;
  const int LDY = q.LDY, TI = q.TI;
  const int ksteps = TI >> 2;  // even: TI is a multiple of 8
  const int pair = lw >> 1, c = lw & 1;
  int64_t cur_rb = -1;
  for (int k = 0; k < ntiles; ++k) {
    const int64_t tile = t0 + k;
    const int64_t rb = tile_rb(tile, p.nCT), ct = tile - rb * p.nCT;
    if (rb != cur_rb) {
      asm volatile("bar.sync 2, 128;\n" ::: "memory");
      load_krl(p, q, rb, lw * 32 + lane, 128);
      asm volatile("bar.sync 2, 128;\n" ::: "memory");
      cur_rb = rb;
    }
    if ((k & 1) != pair) continue;
    const int s = k % q.stages;
    const unsigned long long w0 = clock64();
    mbar_wait(&q.full[s], (k / q.stages) & 1);
    cw += clock64() - w0;
    // B fragments: Y[ks 4 + t][(2c + f) 8 + g]; A fragments: KR_l[ks 4 + t][nb 8 + g]
    const double* yb = q.Ys + s * kTJ * LDY + (c * 16 + g) * LDY + t;
    const double* kl = q.KRl + t * LDK + g;
    double acc[2][2][NT][2];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int f = 0; f < 2; ++f)
#pragma unroll
        for (int nb = 0; nb < NT; ++nb) acc[h][f][nb][0] = acc[h][f][nb][1] = 0.0;
    double y[2][2][2], l[2][2][NT];  // [buffer][k-step of the pair][...]
    auto load = [&](int buf, int ks) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int f = 0; f < 2; ++f) y[buf][h][f] = yb[f * 8 * LDY + (ks + h) * 4];
#pragma unroll
        for (int nb = 0; nb < NT; ++nb) l[buf][h][nb] = kl[(ks + h) * 4 * LDK + nb * 8];
      }
    };
    load(0, 0);
    for (int ks = 0; ks < ksteps; ks += 4) {
      if (ks + 2 < ksteps) load(1, ks + 2);
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int nb = 0; nb < NT; ++nb)
#pragma unroll
          for (int f = 0; f < 2; ++f) dmma(acc[h][f][nb], l[0][h][nb], y[0][h][f]);
      if (ks + 2 >= ksteps) break;
      if (ks + 4 < ksteps) load(0, ks + 4);
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int nb = 0; nb < NT; ++nb)
#pragma unroll
          for (int f = 0; f < 2; ++f) dmma(acc[h][f][nb], l[1][h][nb], y[1][h][f]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&q.empty[s]);
    double* dst = p.Lpart + rb * static_cast<int64_t>(p.R) * p.K;
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      const int64_t col = ct * kTJ + (c * 2 + f) * 8 + 2 * t;
#pragma unroll
      for (int nb = 0; nb < NT; ++nb) {
        const int r = nb * 8 + g;
        if (r < p.R) {
          if (col < p.K) dst[r * p.K + col] = acc[0][f][nb][0] + acc[1][f][nb][0];
          if (col + 1 < p.K) dst[r * p.K + col + 1] = acc[0][f][nb][1] + acc[1][f][nb][1];
        }
      }
    }
  }
}

// Left product only (ALS second pass): 4 column fragments x 2 halves of K,
// combined through shared memory.
template <int NT>
__device__ void left_only_role(const SeedParams& p, const Ring& q, int64_t t0, int ntiles, int warp, int lane,
                               int tid, unsigned long long& cw) {
  const int g = lane >> 2, t = lane & 3;
  constexpr int LDK = seed_ldk(NT);
  const int LDY = q.LDY, TI = q.TI;
  const int nf = warp & 3, h = warp >> 2;
  const int ksteps = TI >> 2, kh = ((ksteps >> 1) + 1) & ~1;
  const int ks0 = h * kh, ks1 = min(ksteps, ks0 + kh);
  int64_t cur_rb = -1;
  auto noflush = [](int64_t) {};
  for (int k = 0; k < ntiles; ++k) {
    const int s = k % q.stages;
    const int64_t tile = t0 + k;
    const int64_t rb = tile_rb(tile, p.nCT), ct = tile - rb * p.nCT;
    if (rb != cur_rb) row_block_change(p, q, rb, cur_rb, true, tid, [](int64_t) {});
    const unsigned long long w0 = clock64();
    mbar_wait(&q.full[s], (k / q.stages) & 1);
    cw += clock64() - w0;
    const double* yb = q.Ys + s * kTJ * LDY + (nf * 8 + g) * LDY + t;
    const double* kl = q.KRl + t * LDK + g;
    double accA[NT][2], accB[NT][2];
#pragma unroll
    for (int nb = 0; nb < NT; ++nb) accA[nb][0] = accA[nb][1] = accB[nb][0] = accB[nb][1] = 0.0;
#pragma unroll 2
    for (int ks = ks0; ks < ks1; ks += 2) {
      const bool two = ks + 1 < ks1;
      const double y0 = yb[ks * 4];
      const double y1 = two ? yb[(ks + 1) * 4] : 0.0;
      double l0[NT], l1[NT];
#pragma unroll
      for (int nb = 0; nb < NT; ++nb) {
        l0[nb] = kl[ks * 4 * LDK + nb * 8];
        l1[nb] = two ? kl[(ks + 1) * 4 * LDK + nb * 8] : 0.0;
      }
#pragma unroll
      for (int nb = 0; nb < NT; ++nb) {
        dmma(accA[nb], l0[nb], y0);
        dmma(accB[nb], l1[nb], y1);
      }
    }
    double* rd = q.red + (k & 1) * (4 * 32 * NT * 2);
    if (h == 1) {
#pragma unroll
      for (int nb = 0; nb < NT; ++nb) {
        rd[(nf * 32 + lane) * NT * 2 + nb * 2] = accA[nb][0] + accB[nb][0];
        rd[(nf * 32 + lane) * NT * 2 + nb * 2 + 1] = accA[nb][1] + accB[nb][1];
      }
    }
    consumer_sync();
    if (h == 0) {
      const int64_t col = ct * kTJ + nf * 8 + 2 * t;
      double* dst = p.Lpart + rb * static_cast<int64_t>(p.R) * p.K;
#pragma unroll
      for (int nb = 0; nb < NT; ++nb) {
        const int r = nb * 8 + g;
        if (r < p.R) {
          const double v0 = accA[nb][0] + accB[nb][0] + rd[(nf * 32 + lane) * NT * 2 + nb * 2];
          const double v1 = accA[nb][1] + accB[nb][1] + rd[(nf * 32 + lane) * NT * 2 + nb * 2 + 1];
          if (col < p.K) dst[r * p.K + col] = v0;
          if (col + 1 < p.K) dst[r * p.K + col + 1] = v1;
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&q.empty[s]);
  }
}

// Dispatch the right role on this warp's (static) fragment count.
template <int NT, int W, int MAXMC>
__device__ void right_dispatch(int mc, const SeedParams& p, const Ring& q, int64_t t0, int ntiles, int cta, int warp,
                               int lane, int tid, bool need_krl, unsigned long long& cw) {
  if constexpr (MAXMC >= 1) {
    if (mc == MAXMC) {
      right_role<NT, MAXMC, W>(p, q, t0, ntiles, cta, warp, lane, tid, need_krl, cw);
      return;
    }
    right_dispatch<NT, W, MAXMC - 1>(mc, p, q, t0, ntiles, cta, warp, lane, tid, need_krl, cw);
  } else {
    right_role<NT, 0, W>(p, q, t0, ntiles, cta, warp, lane, tid, need_krl, cw);
  }
}

template <int NT, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
    seed_f64_kernel(const SeedParams p, const __grid_constant__ CUtensorMap tmap,
                    const __grid_constant__ CUtensorMap kmap) {
  constexpr int RP = NT * 8;
  // right-product row fragments per warp: 4 warps in MODE 3, 8 in MODE 1
  // register budget: 9 warps put 3 on one SMSP -> <= 168 registers per thread
  constexpr int kMaxMF = (MODE == 3) ? (NT <= 2 ? 7 : (NT == 3 ? 6 : 5)) : 4;
  const unsigned long long g_entry = p.trace ? gtime() : 0;
  tl_begin(p.tl, p.tl_slot);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int cta = blockIdx.x;
  const int64_t t0 = (static_cast<int64_t>(cta) * p.T) / p.P;
  const int64_t t1 = (static_cast<int64_t>(cta + 1) * p.T) / p.P;
  if (t0 >= t1) return;
  const int ntiles = static_cast<int>(t1 - t0);
  const int TI = p.TI, LDY = p.LDY, LDK = p.LDK;
  const int STAGES = p.stages;
  const int nMF = TI >> 3;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  // TMA destinations need 128-byte alignment: align the carve-out base
  unsigned char* base = smem_raw + ((128 - (smem_u32(smem_raw) & 127)) & 127);
  uint64_t* full = reinterpret_cast<uint64_t*>(base);   // [3]
  uint64_t* empty = full + 3;                            // [3]
  double* Ys = reinterpret_cast<double*>(base + 128);    // [STAGES][kTJ * LDY]
  double* KRr = Ys + STAGES * kTJ * LDY;                 // [STAGES][kTJ * LDK]
  double* KRl = KRr + STAGES * kTJ * LDK;                // [TI * LDK]
  // MODE 2: [2][4 * 32 * NT * 2] after KR_l; MODE 3 keeps KR_l in registers and
  // uses the space for the left slices' reduction ([2][4][3][NT][2][32])
  double* red = KRl + ((MODE & 2) ? TI * LDK : 0);

  // plain-copy path: zero the stage buffers once (edge tiles are cleared below)
  if (!p.use_tma)
    for (int e = tid; e < STAGES * kTJ * LDY; e += kThreads) Ys[e] = 0.0;
  if (p.use_tma && warp == kConsumers && lane == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
    if (MODE & 1) asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&kmap)) : "memory");
  }
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MODE == 3 ? 6 : kConsumers);  // MODE 3: 4 right + the tile's left pair
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();

  // ------------------------------------------------------------------ producer
  if (warp == kConsumers) {
    unsigned long long tw = 0, tstart = clock64();
    // Y does not depend on the preceding kernel (PDL): the first stages' Y tiles
    // are requested before the wait, their Khatri-Rao rows after it.
    const int early = p.use_tma ? min(STAGES, ntiles) : 0;
    if (lane == 0)
      for (int k = 0; k < early; ++k) {
        const int64_t tile = t0 + k;
        const int64_t rb = tile_rb(tile, p.nCT), ct = tile - rb * p.nCT;
        mbar_arrive_tx(&full[k], LDY * kTJ * 8 + ((MODE & 1) ? kTJ * LDK * 8 : 0));
        tma_load_2d(Ys + k * kTJ * LDY, &tmap, static_cast<int>(rb * TI), static_cast<int>(ct * kTJ), &full[k], true);
      }
    pdl_wait();
    const unsigned long long g_pdl = p.trace ? gtime() : 0;
    if (lane == 0 && (MODE & 1))
      for (int k = 0; k < early; ++k) {
        const int64_t ct = (t0 + k) - tile_rb(t0 + k, p.nCT) * p.nCT;
        tma_load_2d(KRr + k * kTJ * LDK, &kmap, 0, static_cast<int>(ct * kTJ), &full[k]);
      }
    for (int k = early; k < ntiles; ++k) {
      const int s = k % STAGES;
      if (k >= STAGES) {
        const unsigned long long a = clock64();
        mbar_wait(&empty[s], ((k / STAGES) - 1) & 1);
        tw += clock64() - a;
      }
      const int64_t tile = t0 + k;
      const int64_t rb = tile_rb(tile, p.nCT), ct = tile - rb * p.nCT;
      const int64_t row0 = rb * TI, col0 = ct * kTJ;
      double* ys = Ys + s * kTJ * LDY;
      double* kr = KRr + s * kTJ * LDK;
      if (p.use_tma) {  // Y tile + its Khatri-Rao rows, one transaction count
        if (lane == 0) {
          const uint32_t bytes = LDY * kTJ * 8 + ((MODE & 1) ? kTJ * LDK * 8 : 0);
          mbar_arrive_tx(&full[s], bytes);
          tma_load_2d(ys, &tmap, static_cast<int>(row0), static_cast<int>(col0), &full[s], true);
          if (MODE & 1) tma_load_2d(kr, &kmap, 0, static_cast<int>(col0), &full[s]);
        }
      } else {  // unaligned leading extent: plain loads (rare shapes)
        const int rows = static_cast<int>(min64(TI, p.J - row0));
        const int cols = static_cast<int>(min64(kTJ, p.K - col0));
        for (int c = 0; c < kTJ; ++c)
          for (int q = lane; q < TI; q += 32)
            ys[c * LDY + q] = (c < cols && q < rows) ? p.Y[row0 + q + p.J * (col0 + c)] : 0.0;
        if (MODE & 1)
          for (int e = lane; e < kTJ * LDK; e += 32) {
            const int jj = e / LDK;
            kr[e] = jj < cols ? p.KRr_g[(col0 + jj) * LDK + (e - jj * LDK)] : 0.0;
          }
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[s]);
      }
    }
    if (p.trace && lane == 0) {
      unsigned long long* tr = p.trace + (static_cast<int64_t>(cta) * 9 + warp) * 8;
      tr[0] = tw; tr[1] = g_entry; tr[2] = clock64() - tstart; tr[3] = ntiles; tr[4] = g_pdl; tr[6] = gtime();
    }
    tl_end(p.tl, p.tl_slot);
    return;
  }

  // ------------------------------------------------------------------ consumers
  pdl_wait();  // Khatri-Rao rows and the partial buffers belong to the preceding kernels
  const unsigned long long g_pdl = p.trace ? gtime() : 0;
  if (warp == 0) tl_mid(p.tl, p.tl_slot);
  const Ring q{full, empty, Ys, KRr, KRl, red, STAGES, TI, LDY, LDK};
  unsigned long long cw = 0;
  const unsigned long long cstart = clock64();
  if (MODE == 3) {
    if (warp < 4) {
      const int mc = (nMF - warp + 3) / 4;
      right_dispatch<NT, 4, kMaxMF>(mc, p, q, t0, ntiles, cta, warp, lane, tid, true, cw);
    } else {
      left_pair_role<NT>(p, q, t0, ntiles, warp - 4, lane, cw);
    }
  } else if (MODE == 1) {
    const int mc = (nMF - warp + 7) / 8;
    right_dispatch<NT, 8, kMaxMF>(mc, p, q, t0, ntiles, cta, warp, lane, tid, false, cw);
  } else {
    left_only_role<NT>(p, q, t0, ntiles, warp, lane, tid, cw);
  }
  if (p.trace && lane == 0) {
    unsigned long long* tr = p.trace + (static_cast<int64_t>(cta) * 9 + warp) * 8;
    tr[0] = cw; tr[1] = g_entry; tr[2] = clock64() - cstart; tr[3] = ntiles; tr[4] = g_pdl; tr[6] = gtime();
  }
  tl_end(p.tl, p.tl_slot);
}

// ---- left seed with column-block accumulation (ALS / hook second pass) -----------
// Ls[j, r] = sum_i Y[i, j] KR_l[i, r] with the MMA's M = j: a block of TJ columns
// is walked down the rows in 32-row stages and its accumulators persist across
// the rows, flushed once per block into the CTA's partial slot (MODE 2 wrote a
// partial per tile and reduced four K slices per tile through shared memory).
// Y stages arrive as two 16-row halves with 128-byte swizzle ([TJ][16] doubles,
// 16-byte chunk c of column j at c ^ (j % 8)): conflict-free Y^T fragments.
// The Khatri-Rao rows of each stage (32 x LDK) come by TMA like KR_r in MODE 1.
// SeedParams reuse: TI = TJ, nRB = column blocks, nCT = 32-row stages per block,
// T = units, Rpart = partial slots [P * slots][8 NT][TJ].
template <int NT, int MC>
__global__ void __launch_bounds__(kThreads, 1)
    seed_left_cols_kernel(const SeedParams p, const __grid_constant__ CUtensorMap ymap,
                          const __grid_constant__ CUtensorMap kmap) {
  constexpr int RP = NT * 8;
  constexpr int LDK = seed_ldk(NT);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int cta = blockIdx.x;
  const int64_t t0 = (static_cast<int64_t>(cta) * p.T) / p.P;
  const int64_t t1 = (static_cast<int64_t>(cta + 1) * p.T) / p.P;
  if (t0 >= t1) return;
  const int ntiles = static_cast<int>(t1 - t0);
  const int TJ = p.TI, STAGES = p.stages;

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  double* Ys = reinterpret_cast<double*>(base);                  // [STAGES][2][TJ][16]
  double* KRs = Ys + STAGES * kTJ * TJ;                           // [STAGES][32][LDK]
  uint64_t* full = reinterpret_cast<uint64_t*>(KRs + STAGES * kTJ * LDK);
  uint64_t* empty = full + 4;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == kConsumers && lane == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&ymap)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&kmap)) : "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();

  if (warp == kConsumers) {
    // ------------------------------------------------------------------ producer
    if (lane == 0) {
      const uint32_t bytes = kTJ * TJ * 8 + kTJ * LDK * 8;
      auto load_y = [&](int k, int s) {
        const int64_t u = t0 + k, cb = tile_rb(u, p.nCT), rt = u - cb * p.nCT;
        double* ys = Ys + s * kTJ * TJ;
        tma_load_2d(ys, &ymap, static_cast<int>(rt * kTJ), static_cast<int>(cb * TJ), &full[s], true);
        tma_load_2d(ys + 16 * TJ, &ymap, static_cast<int>(rt * kTJ + 16), static_cast<int>(cb * TJ), &full[s], true);
      };
      auto load_k = [&](int k, int s) {
        const int64_t u = t0 + k, rt = u - tile_rb(u, p.nCT) * p.nCT;
        tma_load_2d(KRs + s * kTJ * LDK, &kmap, 0, static_cast<int>(rt * kTJ), &full[s]);
      };
      const int early = min(STAGES, ntiles);
      for (int k = 0; k < early; ++k) {  // Y does not depend on the preceding kernel (PDL)
        mbar_arrive_tx(&full[k], bytes);
        load_y(k, k);
      }
      pdl_wait();
      for (int k = 0; k < early; ++k) load_k(k, k);
      for (int k = early; k < ntiles; ++k) {
        const int s = k % STAGES;
        mbar_wait(&empty[s], ((k / STAGES) - 1) & 1);
        mbar_arrive_tx(&full[s], bytes);
        load_y(k, s);
        load_k(k, s);
      }
    }
    return;
  }

  // ------------------------------------------------------------------ consumers
  pdl_wait();
  double acc[MC > 0 ? MC : 1][NT][2];
#pragma unroll
  for (int m = 0; m < MC; ++m)
#pragma unroll
    for (int nb = 0; nb < NT; ++nb) acc[m][nb][0] = acc[m][nb][1] = 0.0;
  const int64_t slot_cb0 = t0 / p.nCT;
  auto flush = [&](int64_t cb) {
    double* dst = p.Rpart + (static_cast<int64_t>(cta) * p.slots + (cb - slot_cb0)) * RP * TJ;
#pragma unroll
    for (int m = 0; m < MC; ++m) {
      const int j = (warp + kConsumers * m) * 8 + g;
#pragma unroll
      for (int nb = 0; nb < NT; ++nb) {
        const int r = nb * 8 + 2 * t;
        dst[r * TJ + j] = acc[m][nb][0];
        dst[(r + 1) * TJ + j] = acc[m][nb][1];
        acc[m][nb][0] = acc[m][nb][1] = 0.0;
      }
    }
  };
  // byte offset of Y^T fragment element (k-step ks, row-fragment m) inside a stage
  auto yoff = [&](int ks, int m) {
    const int j = (warp + kConsumers * m) * 8 + g;
    const int ip = (4 * ks + t) & 15;
    return (ks >> 2) * (16 * TJ * 8) + j * 128 + (((ip >> 1) ^ (j & 7)) << 4) + (ip & 1) * 8;
  };
  int64_t cur_cb = -1;
  for (int k = 0; k < ntiles; ++k) {
    const int s = k % STAGES;
    const int64_t cb = tile_rb(t0 + k, p.nCT);
    if (cb != cur_cb) {
      if (cur_cb >= 0) flush(cur_cb);
      cur_cb = cb;
    }
    mbar_wait(&full[s], (k / STAGES) & 1);
    const unsigned char* ys = reinterpret_cast<const unsigned char*>(Ys + s * kTJ * TJ);
    const double* kb = KRs + s * kTJ * LDK + t * LDK + g;
    double a[2][MC > 0 ? MC : 1], b[2][NT];
#pragma unroll
    for (int m = 0; m < MC; ++m) a[0][m] = *reinterpret_cast<const double*>(ys + yoff(0, m));
#pragma unroll
    for (int nb = 0; nb < NT; ++nb) b[0][nb] = kb[nb * 8];
#pragma unroll
    for (int ks = 0; ks < kTJ / 4; ++ks) {
      const int cur = ks & 1, nxt = cur ^ 1;
      if (ks + 1 < kTJ / 4) {
#pragma unroll
        for (int m = 0; m < MC; ++m) a[nxt][m] = *reinterpret_cast<const double*>(ys + yoff(ks + 1, m));
#pragma unroll
        for (int nb = 0; nb < NT; ++nb) b[nxt][nb] = kb[(ks + 1) * 4 * LDK + nb * 8];
      }
#pragma unroll
      for (int m = 0; m < MC; ++m)
#pragma unroll
        for (int nb = 0; nb < NT; ++nb) dmma(acc[m][nb], a[cur][m], b[cur][nb]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (cur_cb >= 0) flush(cur_cb);
}

template <int NT, int MODE>
void launch_one(const SeedParams& p, const CUtensorMap& tmap, const CUtensorMap& kmap, cudaStream_t s,
                size_t smem) {
  auto fn = seed_f64_kernel<NT, MODE>;
  static unsigned long long configured = 0;  // devices done, per instantiation
  set_smem_attr(fn, 232448, configured);
  launch_k(fn, dim3(p.P), dim3(kThreads), smem, s, pdl_enabled(), p, tmap, kmap);
}

template <int NT>
void launch_nt(const SeedParams& p, const CUtensorMap& tmap, const CUtensorMap& kmap, int mode, cudaStream_t s,
               size_t smem) {
  if (mode == 1) launch_one<NT, 1>(p, tmap, kmap, s, smem);
  else if (mode == 2) launch_one<NT, 2>(p, tmap, kmap, s, smem);
  else launch_one<NT, 3>(p, tmap, kmap, s, smem);
}

}  // namespace

int seed_f64_max_ti(int NT) { return NT <= 2 ? 208 : (NT == 3 ? 192 : 160); }

size_t seed_f64_smem_bytes(int NT, int TI, int LDY, int LDK, int mode, int stages, int64_t fac_doubles) {
  size_t d = static_cast<size_t>(stages) * kTJ * LDY + static_cast<size_t>(stages) * kTJ * LDK;
  if (mode & 2) d += static_cast<size_t>(TI) * LDK;
  if (mode == 2) d += 2 * 4 * 32 * NT * 2;
  if (mode & 1) d += static_cast<size_t>(fac_doubles);
  return 256 + d * sizeof(double);  // barriers + 128-byte alignment slack
}

size_t seed_left_cols_smem_bytes(int NT, int TJ, int stages) {
  const int LDK = seed_ldk(NT);
  return 1024 + static_cast<size_t>(stages) * kTJ * (TJ + LDK) * sizeof(double) + 64;
}

template <int NT>
void launch_lc(const SeedParams& p, const CUtensorMap& ym, const CUtensorMap& km, cudaStream_t s, size_t smem) {
  constexpr int MC = 4;  // TJ = 8 warps x 4 fragments x 8 = 256 columns
  auto fn = seed_left_cols_kernel<NT, MC>;
  static unsigned long long configured = 0;
  set_smem_attr(fn, 232448, configured);
  launch_k(fn, dim3(p.P), dim3(kThreads), smem, s, pdl_enabled(), p, ym, km);
}

int launch_seed_left_cols(const SeedParams& p, const CUtensorMap* ymap, const CUtensorMap* kmap, int NT,
                          cudaStream_t s) {
  const size_t smem = seed_left_cols_smem_bytes(NT, p.TI, p.stages);
  switch (NT) {
    case 1: launch_lc<1>(p, *ymap, *kmap, s, smem); break;
    case 2: launch_lc<2>(p, *ymap, *kmap, s, smem); break;
    case 3: launch_lc<3>(p, *ymap, *kmap, s, smem); break;
    case 4: launch_lc<4>(p, *ymap, *kmap, s, smem); break;
    default: return 0;
  }
  return 1;
}

int launch_seed_f64(const SeedParams& p, const CUtensorMap* tmap, const CUtensorMap* kmap, int NT, int mode,
                    cudaStream_t s) {
  CUtensorMap dummy;
  std::memset(&dummy, 0, sizeof dummy);
  const CUtensorMap& m = (p.use_tma && tmap) ? *tmap : dummy;
  const CUtensorMap& km = (p.use_tma && kmap) ? *kmap : dummy;
  const size_t smem = seed_f64_smem_bytes(NT, p.TI, p.LDY, p.LDK, mode, p.stages, 0);
  switch (NT) {
    case 1: launch_nt<1>(p, m, km, mode, s, smem); break;
    case 2: launch_nt<2>(p, m, km, mode, s, smem); break;
    case 3: launch_nt<3>(p, m, km, mode, s, smem); break;
    case 4: launch_nt<4>(p, m, km, mode, s, smem); break;
    default: return 0;
  }
  return 1;
}

bool make_tensor_map_2d(CUtensorMap* out, const void* base, CUtensorMapDataType dtype, int elem_bytes,
                        uint64_t dim0, uint64_t dim1, uint64_t stride1_bytes, uint32_t box0, uint32_t box1,
                        bool swizzle128, int promote) {
  static PFN_cuTensorMapEncodeTiled encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return false;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
  }
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (stride1_bytes & 15) || ((box0 * elem_bytes) & 15) ||
      box0 > 256 || box1 > 256 || dim0 >= (1ull << 32) || dim1 >= (1ull << 32))
    return false;
  const cuuint64_t gdim[2] = {dim0, dim1};
  const cuuint64_t gstride[1] = {stride1_bytes};
  const cuuint32_t box[2] = {box0, box1};
  const cuuint32_t estride[2] = {1, 1};
  return encode(out, dtype, 2, const_cast<void*>(base), gdim, gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
                swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                promote >= 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                : promote >= 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                : promote >= 64  ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                : promote == 1   ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B  // bool true from older callers
                                 : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace cpdgpu
