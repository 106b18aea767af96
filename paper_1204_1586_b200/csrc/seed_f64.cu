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
//  * Y tiles of TI rows x 32 columns stream HBM -> shared memory with
//    cp.async (16-byte LDGSTS, zero-filled at the edges), STAGES deep.
//  * Khatri-Rao rows are never materialised in HBM: the KR(p+1..N) rows of a
//    tile (32 x RP) and the KR(1..p) rows of a row block (TI x RP) are
//    generated in shared memory from factor rows (kron_range_column,
//    kron.cpp:54-68, later modes outermost).
//  * Right product (M = rows, N = rank, K = columns) and left product computed
//    as  L^T = KR^T * Y  (M = rank, N = columns, K = rows) with
//    mma.sync.m8n8k4.f64 (DMMA): measured 37.1 TF/s on B200 vs 36.7 TF/s for
//    DFMA at full occupancy, with ~1/16 of the issue slots.
//  * Each persistent CTA owns a contiguous range of the row-block-major tile
//    space.  Right partials persist in registers across a row block and are
//    written once per (CTA, row block) slot; left partials are written per tile
//    per row block.  A deterministic reduction (tail.cu) sums them in a fixed
//    order, so results are bitwise reproducible run to run.
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace cpdgpu {
namespace {

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

constexpr int kTJ = 32;       // columns per tile
constexpr int kThreads = 256;  // 8 warps
constexpr int kMaxMF = 4;      // row fragments per warp (TI <= 8 * 8 * 4 = 256)

template <int NT, int STAGES, bool VEC16, int MODE>
__global__ void __launch_bounds__(kThreads, 1) seed_f64_kernel(const SeedParams p) {
  constexpr int RP = NT * 8;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int cta = blockIdx.x;
  const int64_t t0 = (static_cast<int64_t>(cta) * p.T) / p.P;
  const int64_t t1 = (static_cast<int64_t>(cta + 1) * p.T) / p.P;
  if (t0 >= t1) return;
  const int ntiles = static_cast<int>(t1 - t0);
  const int TI = p.TI, LDY = p.LDY, LDK = p.LDK;
  const int nMF = TI >> 3;

  extern __shared__ __align__(16) double smem[];
  double* Ys = smem;                                   // [STAGES][kTJ * LDY]
  double* KRr = Ys + STAGES * kTJ * LDY;               // [STAGES][kTJ * LDK]
  double* KRl = KRr + STAGES * kTJ * LDK;              // [TI * LDK]
  double* red = KRl + ((MODE & 2) ? TI * LDK : 0);     // [4 * 32 * NT * 2]

  auto issue_tile = [&](int64_t tile, int stage) {
    const int64_t rb = tile / p.nCT, ct = tile - rb * p.nCT;
    const int64_t row0 = rb * TI, col0 = ct * kTJ;
    const int rows = static_cast<int>(min64(TI, p.J - row0));
    const int cols = static_cast<int>(min64(kTJ, p.K - col0));
    double* dst = Ys + stage * kTJ * LDY;
    if (VEC16) {
      const int half = TI >> 1;
      for (int e = tid; e < kTJ * half; e += kThreads) {
        const int c = e / half, q = e - c * half;
        const int row = 2 * q;
        int bytes = 0;
        const double* src = p.Y;
        if (c < cols && row < rows) {
          bytes = (rows - row) >= 2 ? 16 : 8;
          src = p.Y + (row0 + row) + p.J * (col0 + c);
        }
        cp_async16(dst + c * LDY + row, src, bytes);
      }
    } else {
      for (int e = tid; e < kTJ * TI; e += kThreads) {
        const int c = e / TI, row = e - c * TI;
        int bytes = 0;
        const double* src = p.Y;
        if (c < cols && row < rows) {
          bytes = 8;
          src = p.Y + (row0 + row) + p.J * (col0 + c);
        }
        cp_async8(dst + c * LDY + row, src, bytes);
      }
    }
    if (MODE & 1) {  // KR(p+1..N) rows of this tile's columns
      double* kr = KRr + stage * kTJ * LDK;
      for (int e = tid; e < kTJ * RP; e += kThreads) {
        const int jj = e / RP, r = e - jj * RP;
        double v = 0.0;
        if (jj < cols && r < p.R)
          v = p.use32 ? kr_entry32(p.right, static_cast<uint32_t>(col0 + jj), r)
                      : kr_entry(p.right, col0 + jj, r);
        kr[jj * LDK + r] = v;
      }
    }
  };

  auto load_krl = [&](int64_t rb) {  // KR(1..p) rows of a row block
    const int64_t row0 = rb * TI;
    const int rows = static_cast<int>(min64(TI, p.J - row0));
    for (int e = tid; e < TI * RP; e += kThreads) {
      const int i = e / RP, r = e - i * RP;
      double v = 0.0;
      if (i < rows && r < p.R)
        v = p.use32 ? kr_entry32(p.left, static_cast<uint32_t>(row0 + i), r)
                    : kr_entry(p.left, row0 + i, r);
      KRl[i * LDK + r] = v;
    }
  };

  double acc1[kMaxMF][NT][2];
#pragma unroll
  for (int m = 0; m < kMaxMF; ++m)
#pragma unroll
    for (int nb = 0; nb < NT; ++nb) acc1[m][nb][0] = acc1[m][nb][1] = 0.0;

  const int64_t slot_rb0 = t0 / p.nCT;
  auto flush_right = [&](int64_t rb) {
    double* dst = p.Rpart + (static_cast<int64_t>(cta) * p.slots + (rb - slot_rb0)) * RP * TI;
#pragma unroll
    for (int m = 0; m < kMaxMF; ++m) {
      const int mf = warp + 8 * m;
      if (mf < nMF) {
        const int i = mf * 8 + g;
#pragma unroll
        for (int nb = 0; nb < NT; ++nb) {
          const int r = nb * 8 + 2 * t;
          dst[r * TI + i] = acc1[m][nb][0];
          dst[(r + 1) * TI + i] = acc1[m][nb][1];
          acc1[m][nb][0] = acc1[m][nb][1] = 0.0;
        }
      }
    }
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ntiles) issue_tile(t0 + s, s);
    cp_async_commit();
  }

  int64_t cur_rb = -1;
  for (int k = 0; k < ntiles; ++k) {
    const int64_t tile = t0 + k;
    const int64_t rb = tile / p.nCT, ct = tile - rb * p.nCT;
    if (k + STAGES - 1 < ntiles) issue_tile(tile + STAGES - 1, (k + STAGES - 1) % STAGES);
    cp_async_commit();
    if (rb != cur_rb) {
      if ((MODE & 1) && cur_rb >= 0) flush_right(cur_rb);
      if (MODE & 2) load_krl(rb);
      cur_rb = rb;
    }
    cp_async_wait<STAGES - 1>();
    __syncthreads();

    const int stage = k % STAGES;
    const double* Yst = Ys + stage * kTJ * LDY;
    if (MODE & 1) {  // right: Rs[i, r] += sum_j Y[i, j] KR_r[j, r]
      const double* kr = KRr + stage * kTJ * LDK;
#pragma unroll
      for (int ks = 0; ks < kTJ / 4; ++ks) {
        double b[NT];
#pragma unroll
        for (int nb = 0; nb < NT; ++nb) b[nb] = kr[(ks * 4 + t) * LDK + nb * 8 + g];
#pragma unroll
        for (int m = 0; m < kMaxMF; ++m) {
          const int mf = warp + 8 * m;
          if (mf < nMF) {
            const double a = Yst[(mf * 8 + g) + (ks * 4 + t) * LDY];
#pragma unroll
            for (int nb = 0; nb < NT; ++nb) dmma(acc1[m][nb], a, b[nb]);
          }
        }
      }
    }
    double acc2[NT][2];
    if (MODE & 2) {  // left: Ls^T[r, j] += sum_i KR_l^T[r, i] Y[i, j]
#pragma unroll
      for (int nb = 0; nb < NT; ++nb) acc2[nb][0] = acc2[nb][1] = 0.0;
      const int nf = warp & 3, h = warp >> 2;
      const int ksteps = TI >> 2, kh = (ksteps + 1) >> 1;
      const int ks0 = h * kh, ks1 = min(ksteps, ks0 + kh);
#pragma unroll 4
      for (int ks = ks0; ks < ks1; ++ks) {
        const double by = Yst[(ks * 4 + t) + (nf * 8 + g) * LDY];
#pragma unroll
        for (int nb = 0; nb < NT; ++nb) dmma(acc2[nb], KRl[(ks * 4 + t) * LDK + nb * 8 + g], by);
      }
      if (warp >= 4) {
        double* rd = red + ((warp - 4) * 32 + lane) * NT * 2;
#pragma unroll
        for (int nb = 0; nb < NT; ++nb) {
          rd[nb * 2] = acc2[nb][0];
          rd[nb * 2 + 1] = acc2[nb][1];
        }
      }
    }
    __syncthreads();
    if ((MODE & 2) && warp < 4) {
      const double* rd = red + (warp * 32 + lane) * NT * 2;
      const int nf = warp;
      const int64_t col = ct * kTJ + nf * 8 + 2 * t;
      double* dst = p.Lpart + rb * static_cast<int64_t>(p.R) * p.K;
#pragma unroll
      for (int nb = 0; nb < NT; ++nb) {
        const int r = nb * 8 + g;
        if (r < p.R) {
          if (col < p.K) dst[r * p.K + col] = acc2[nb][0] + rd[nb * 2];
          if (col + 1 < p.K) dst[r * p.K + col + 1] = acc2[nb][1] + rd[nb * 2 + 1];
        }
      }
    }
  }
  if (MODE & 1) flush_right(cur_rb);
}

template <int NT, int STAGES, bool VEC16, int MODE>
void launch_one(const SeedParams& p, cudaStream_t s, size_t smem) {
  auto fn = seed_f64_kernel<NT, STAGES, VEC16, MODE>;
  static bool configured = false;  // one attribute call per instantiation
  if (!configured) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    configured = true;
  }
  fn<<<p.P, kThreads, smem, s>>>(p);
}

template <int NT, int STAGES>
void launch_nt(const SeedParams& p, int mode, bool vec16, cudaStream_t s, size_t smem) {
  if (vec16) {
    if (mode == 1) launch_one<NT, STAGES, true, 1>(p, s, smem);
    else if (mode == 2) launch_one<NT, STAGES, true, 2>(p, s, smem);
    else launch_one<NT, STAGES, true, 3>(p, s, smem);
  } else {
    if (mode == 1) launch_one<NT, STAGES, false, 1>(p, s, smem);
    else if (mode == 2) launch_one<NT, STAGES, false, 2>(p, s, smem);
    else launch_one<NT, STAGES, false, 3>(p, s, smem);
  }
}

}  // namespace

int seed_f64_stages(int NT) { return NT <= 3 ? 3 : 2; }

size_t seed_f64_smem_bytes(int NT, int TI, int LDY, int LDK, int mode) {
  const int stages = seed_f64_stages(NT);
  size_t d = static_cast<size_t>(stages) * kTJ * LDY + static_cast<size_t>(stages) * kTJ * LDK;
  if (mode & 2) d += static_cast<size_t>(TI) * LDK + 4 * 32 * NT * 2;
  return d * sizeof(double);
}

int launch_seed_f64(const SeedParams& p, int NT, int mode, cudaStream_t s) {
  const bool vec16 = (p.J % 2 == 0);
  const size_t smem = seed_f64_smem_bytes(NT, p.TI, p.LDY, p.LDK, mode);
  switch (NT) {
    case 1: launch_nt<1, 3>(p, mode, vec16, s, smem); break;
    case 2: launch_nt<2, 3>(p, mode, vec16, s, smem); break;
    case 3: launch_nt<3, 3>(p, mode, vec16, s, smem); break;
    case 4: launch_nt<4, 2>(p, mode, vec16, s, smem); break;
    default: return 0;
  }
  return 1;
}

}  // namespace cpdgpu
