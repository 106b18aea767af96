// tail.cu — everything around the seed contraction: the prologue (factor
// gather + Khatri-Rao rows for K1), the deterministic seed-partial reductions
// and the rank-batched TTV recursion tail.
//
// Reference: the right phase  (mttkrp.cpp:165-193; Eq 3.20 recursion, Eq 3.12
// extraction) and the left phase (mttkrp.cpp:212-241; Eq 3.22 recursion,
// Eq 3.16 extraction).  The reference runs one GEMV per rank column r; here a
// single launch ("tail step") covers every rank column of every contraction
// that can run at the same recursion level — the right phase's extraction of
// mode j and recursion to mode j-1 read the same R^(j), the left phase is
// independent of the right — so a gradient costs 1 + max(p, N - p) tail
// launches.  Every output is produced by one warp in a fixed order, so results
// are bitwise reproducible.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "kernels.h"

namespace cpdgpu {
namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double kr_at(const KRSpec& s, int64_t q, int r) {
  if (s.n == 0) return 1.0;
  if (s.n == 1) return __ldg(s.A[0] + q + s.dims[0] * r);  // one factor: no digits
  return q < (1LL << 31) ? kr_entry32(s, static_cast<uint32_t>(q), r) : kr_entry(s, q, r);
}

// sum_{x = lane, lane + 32, ... < n} z[x * stride] * KR(s)[x, r], four
// independent partial sums in flight (latency of the L2-resident operands).
__device__ __forceinline__ double strided_dot(const double* z, int64_t stride, int64_t n, const KRSpec& s, int r,
                                              int lane) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int64_t x = lane;
  for (; x + 96 < n; x += 128) {
    s0 += z[x * stride] * kr_at(s, x, r);
    s1 += z[(x + 32) * stride] * kr_at(s, x + 32, r);
    s2 += z[(x + 64) * stride] * kr_at(s, x + 64, r);
    s3 += z[(x + 96) * stride] * kr_at(s, x + 96, r);
  }
  for (; x < n; x += 32) s0 += z[x * stride] * kr_at(s, x, r);
  return (s0 + s1) + (s2 + s3);
}

// Contractions at least this long run one output per CTA (256 threads and a
// fixed-order block reduction) instead of one per warp: the top extraction of a
// high-order tensor has few outputs, each a dot product over thousands of terms.
constexpr int64_t kCtaContractLen = 1024;

__host__ __device__ inline int64_t contract_len(const TailOp& o) {
  return o.type == kOpContractA ? o.M : (o.type == kOpContractB ? o.B : 0);
}

// Number of CTA work units of an op (one per output of a long contraction).
__host__ __device__ inline int64_t op_cta_units(const TailOp& o) {
  if (!o.cta) return 0;
  return o.type == kOpContractA ? o.B * o.R : o.M * o.R;
}

// Number of warp work units of an op.
__host__ __device__ inline int64_t op_units(const TailOp& o) {
  if (o.cta) return 0;
  switch (o.type) {
    case kOpContractA: return o.B * o.R;                       // warp per output (b, r)
    case kOpContractB: return o.M * o.R;                       // warp per output (a, r)
    case kOpReduceRight:                                       // B == 1: warp per output (lanes over slots)
      return o.B == 1 ? o.M * o.R : ((o.M + 31) / 32) * o.R;   // else 32 rows per warp
    case kOpReduceLeft: return ((o.M + 31) / 32) * o.R;        // 32 columns per warp
    default: return 0;
  }
}

__device__ __forceinline__ double* op_out(const TailOp& o, double* const* gtab) {
  return o.out_slot >= 0 ? gtab[o.out_slot] + o.out_off : o.out;
}

__device__ void run_unit(const TailOp& o, int64_t u, int lane, double* const* gtab) {
  double* out = op_out(o, gtab);
  if (o.type == kOpContractA) {  // out[r][b] = sum_a Z[r][a + M b] KR_v[a, r]
    const int r = static_cast<int>(u / o.B);
    const int64_t b = u - r * o.B;
    const double s = warp_sum(strided_dot(o.Z + r * o.ldz + o.M * b, 1, o.M, o.kr, r, lane));
    if (lane == 0) out[r * o.ldo + b] = s;
  } else if (o.type == kOpContractB) {  // out[r][a] = sum_b Z[r][a + M b] KR_w[b, r]
    const int r = static_cast<int>(u / o.M);
    const int64_t a = u - r * o.M;
    const double s = warp_sum(strided_dot(o.Z + r * o.ldz + a, o.M, o.B, o.kr, r, lane));
    if (lane == 0) out[r * o.ldo + a] = s;
  } else if (o.type == kOpReduceRight && o.B == 1) {  // many slots: lanes over slots, fixed tree
    const int r = static_cast<int>(u / o.M);
    const int64_t i = u - r * o.M;
    const int64_t rb = i / o.TI, il = i - rb * o.TI;
    double s = 0.0;
    for (int q = o.rb_ptr[rb] + lane; q < o.rb_ptr[rb + 1]; q += 32)
      s += o.Z[(static_cast<int64_t>(o.slot_list[q]) * o.RP + r) * o.TI + il];
    s = warp_sum(s);
    if (lane == 0) out[r * o.ldo + i] = s;
  } else if (o.type == kOpReduceRight) {  // Rs[r][i] = sum of the slots of row block rb(i)
    const int64_t chunks = (o.M + 31) / 32;
    const int r = static_cast<int>(u / chunks);
    const int64_t i = (u - r * chunks) * 32 + lane;
    if (i < o.M) {
      const int64_t rb = i / o.TI, il = i - rb * o.TI;
      double s = 0.0;
      for (int q = o.rb_ptr[rb]; q < o.rb_ptr[rb + 1]; ++q)
        s += o.Z[(static_cast<int64_t>(o.slot_list[q]) * o.RP + r) * o.TI + il];
      out[r * o.ldo + i] = s;
    }
  } else if (o.type == kOpReduceLeft) {  // Ls[r][j] = sum_rb Lpart[rb][r][j]
    const int64_t chunks = (o.M + 31) / 32;
    const int r = static_cast<int>(u / chunks);
    const int64_t j = (u - r * chunks) * 32 + lane;
    if (j < o.M) {
      const int64_t stride = static_cast<int64_t>(o.R) * o.M;
      const double* z = o.Z + r * o.M + j;
      double s = 0.0;
      for (int64_t rb = 0; rb < o.B; ++rb) s += z[rb * stride];
      out[r * o.ldo + j] = s;
    }
  }
}

// One output of a long contraction on the whole CTA: 256 threads stride over the
// contraction with four partial sums each, then warp sums and the eight warp
// totals are added in warp order (bitwise reproducible).
__device__ void run_cta_unit(const TailOp& o, int64_t u, double* red, double* const* gtab) {
  double* out = op_out(o, gtab);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int r;
  int64_t n, stride, oidx;
  const double* z;
  if (o.type == kOpContractA) {  // out[r][b] = sum_a Z[r][a + M b] KR_v[a, r]
    r = static_cast<int>(u / o.B);
    const int64_t b = u - r * o.B;
    z = o.Z + r * o.ldz + o.M * b;
    n = o.M;
    stride = 1;
    oidx = r * o.ldo + b;
  } else {  // out[r][a] = sum_b Z[r][a + M b] KR_w[b, r]
    r = static_cast<int>(u / o.M);
    const int64_t a = u - r * o.M;
    z = o.Z + r * o.ldz + a;
    n = o.B;
    stride = o.M;
    oidx = r * o.ldo + a;
  }
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int64_t x = tid;
  for (; x + 768 < n; x += 1024) {
    s0 += z[x * stride] * kr_at(o.kr, x, r);
    s1 += z[(x + 256) * stride] * kr_at(o.kr, x + 256, r);
    s2 += z[(x + 512) * stride] * kr_at(o.kr, x + 512, r);
    s3 += z[(x + 768) * stride] * kr_at(o.kr, x + 768, r);
  }
  for (; x < n; x += 256) s0 += z[x * stride] * kr_at(o.kr, x, r);
  const double v = warp_sum((s0 + s1) + (s2 + s3));
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w];
    out[oidx] = t;
  }
  __syncthreads();
}

// One recursion level.  CTA = false: every op is warp-granular (the common
// case, kept lean); CTA = true: the step holds long contractions, whose outputs
// run one per CTA before the warp units.
template <bool CTA>
__global__ void __launch_bounds__(256) tail_step_kernel(const TailStep st, double* const* gtab) {
  tl_begin(st.tl, st.tl_slot);
  pdl_wait();     // inputs come from the previous step / seed
  tl_mid(st.tl, st.tl_slot);
  pdl_trigger();  // the next step may launch and wait
  if constexpr (CTA) {  // block-uniform loop over the CTA units
    __shared__ double red[8];
    int64_t cstart[kMaxTailOps + 1];
    cstart[0] = 0;
    for (int i = 0; i < st.n; ++i) cstart[i + 1] = cstart[i] + op_cta_units(st.op[i]);
    for (int64_t cu = blockIdx.x; cu < cstart[st.n]; cu += gridDim.x) {
      int i = 0;
      while (cu >= cstart[i + 1]) ++i;
      run_cta_unit(st.op[i], cu - cstart[i], red, gtab);
    }
  }
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  int64_t start[kMaxTailOps + 1];
  start[0] = 0;
  for (int i = 0; i < st.n; ++i) start[i + 1] = start[i] + op_units(st.op[i]);
  for (int64_t w = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; w < start[st.n];
       w += nwarps) {
    int i = 0;
    while (w >= start[i + 1]) ++i;
    run_unit(st.op[i], w - start[i], lane, gtab);
  }
  tl_end(st.tl, st.tl_slot);
}

// Prologue: sorted factors Fs[j] <- input block perm[j]; output pointer table;
// Khatri-Rao rows of every K1 chunk: out[q * LDK + r] = KR(spec)[q, r], one
// thread per entry (one dependent load per mode: latency, not bandwidth, is the
// cost of this small kernel).
__device__ void kr_rows(const KRJob& k, int64_t t, int64_t nt) {
  const int64_t total = k.L * k.LDK;
  for (int64_t e = t; e < total; e += nt) {
    const int64_t q = e / k.LDK;
    const int r = static_cast<int>(e - q * k.LDK);
    double v = r < k.R ? 1.0 : 0.0;
    if (r < k.R) {
      int64_t rem = q;
      for (int m = 0; m < k.spec.n; ++m) {
        const int64_t I = k.spec.dims[m];
        const int64_t d = rem % I;
        rem /= I;
        v *= __ldg(k.spec.A[m] + d + I * r);
      }
    }
    k.out[e] = v;
  }
}

__global__ void __launch_bounds__(256) prologue_kernel(const Prologue pr, double** gtab) {
  tl_begin(pr.tl, 0);
  tl_mid(pr.tl, 0);
  pdl_trigger();  // the seed contraction may start streaming Y now
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t nt = static_cast<int64_t>(gridDim.x) * blockDim.x;
  if (t < kMaxModes && t < pr.N) gtab[t] = pr.gout[t];
  for (int64_t e = t; e < pr.zero_n; e += nt) pr.zero[e] = 0.0;
  if (pr.Fs)
    for (int j = 0; j < pr.N; ++j)
      for (int64_t e = t; e < pr.len[j]; e += nt) pr.Fs[pr.dst_off[j] + e] = pr.fin[pr.src_off[j] + e];
  for (int c = 0; c < pr.nkr; ++c) kr_rows(pr.kr[c], t, nt);
  tl_end(pr.tl, 0);
}

// ---- first level fused with the seed reduction (see L0Side in kernels.h) ----------
__global__ void __launch_bounds__(kL0Threads) l0_kernel(const L0Step st, double* const* gtab) {
  tl_begin(st.tl, st.tl_slot);
  pdl_wait();
  tl_mid(st.tl, st.tl_slot);
  pdl_trigger();
  extern __shared__ double zs[];  // [bq][M]
  __shared__ unsigned last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // block -> (side, r, chunk)
  int bid = blockIdx.x, si = 0;
  const int n0 = st.side[0].nq * st.R;
  if (st.nsides > 1 && bid >= n0) {
    si = 1;
    bid -= n0;
  }
  const L0Side& sd = st.side[si];
  const int r = bid / sd.nq, qc = bid - r * sd.nq;
  const int64_t b0 = static_cast<int64_t>(qc) * sd.bq;
  const int64_t b1 = min(sd.B, b0 + sd.bq);
  const int64_t M = sd.M, rows = (b1 - b0) * M;
  // 1. this chunk's rows of Z (contiguous: idx = a + M b) into shared memory;
  //    two rows per thread and step, each summed from batches of eight
  //    partial loads issued together (order of the reduction ops kept)
  const int64_t base = b0 * M;
  if (sd.zsrc == 1) {
    // slot partials [slot][RP][TI] listed per row tile (CSR).  Four rows per thread and
    // step, so a chunk of up to 1024 rows is one step: the row-tile pointer, slot list
    // and partial loads are three dependent round trips per STEP, and a second step
    // doubled them (each CTA's life is this latency chain).  Fields hoisted out of the
    // dynamically indexed parameter struct; two partial loads per row in flight (a row
    // tile has 1-3 slots at c5, ~6 at c2); the sum runs in slot-list order.
    const double* __restrict__ Zp = sd.Z;
    const int* __restrict__ sl = sd.slot_list;
    const int* __restrict__ rbp = sd.rb_ptr;
    const uint32_t TI = static_cast<uint32_t>(sd.TI);
    const int64_t sstride = static_cast<int64_t>(sd.RP) * sd.TI;
    for (int64_t e0 = tid; e0 < rows; e0 += 4 * kL0Threads) {
      double sum[4] = {0.0, 0.0, 0.0, 0.0};
      int q0[4], q1[4];
      const double* pk[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int64_t e = e0 + k * kL0Threads;
        const bool has = e < rows;
        const int64_t idx = base + (has ? e : e0);
        const uint32_t rb = static_cast<uint32_t>(idx) / TI;
        pk[k] = Zp + static_cast<int64_t>(r) * TI + (idx - static_cast<int64_t>(rb) * TI);
        q0[k] = rbp[rb];
        q1[k] = has ? rbp[rb + 1] : q0[k];
      }
      const int nmax = max(max(q1[0] - q0[0], q1[1] - q0[1]), max(q1[2] - q0[2], q1[3] - q0[3]));
      for (int qq = 0; qq < nmax; qq += 2) {
        double v[4][2];
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int q = q0[k] + qq + u;
            v[k][u] = q < q1[k] ? pk[k][static_cast<int64_t>(sl[q]) * sstride] : 0.0;
          }
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int u = 0; u < 2; ++u)
            if (q0[k] + qq + u < q1[k]) sum[k] += v[k][u];
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (e0 + k * kL0Threads < rows) zs[e0 + k * kL0Threads] = sum[k];
    }
  } else
  for (int64_t e0 = tid; e0 < rows; e0 += 2 * kL0Threads) {
    const int64_t e1 = e0 + kL0Threads;
    const bool has1 = e1 < rows;
    if (sd.zsrc == 0) {
      zs[e0] = sd.Z[r * sd.ldz + base + e0];
      if (has1) zs[e1] = sd.Z[r * sd.ldz + base + e1];
    } else {
      double sum[2] = {0.0, 0.0};
      // row-block partials: plane stride ldz, fields hoisted out of the
      // (dynamically indexed) parameter struct
      const int pcount = sd.pcount;
      const int64_t ldz = sd.ldz;
      const double* z0 = sd.Z + r * sd.pK + base + e0;
      const double* z1 = sd.Z + r * sd.pK + base + (has1 ? e1 : e0);
      for (int rb0 = 0; rb0 < pcount; rb0 += 8) {
        double v0[8], v1[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const bool ok = rb0 + u < pcount;
          v0[u] = ok ? z0[(rb0 + u) * ldz] : 0.0;
          v1[u] = ok ? z1[(rb0 + u) * ldz] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (rb0 + u < pcount) {
            sum[0] += v0[u];
            sum[1] += v1[u];
          }
      }
      zs[e0] = sum[0];
      if (has1) zs[e1] = sum[1];
    }
  }
  // Khatri-Rao values of this (r, chunk): KR_A[a, r] for every a, KR_B[b, r] for the chunk's b
  double* kra = zs + rows;
  double* krb = kra + M;
  double* gp = krb + (b1 - b0);  // group partials of opB [groups][M]
  for (int64_t x = tid; x < M; x += kL0Threads) kra[x] = kr_at(sd.krA, x, r);
  for (int64_t x = tid; x < b1 - b0; x += kL0Threads) krb[x] = kr_at(sd.krB, b0 + x, r);
  __syncthreads();
  // 2. opA, complete for b in [b0, b1): warp per b
  double* outA = sd.outA ? sd.outA : gtab[sd.slotA];
  for (int64_t b = b0 + warp; b < b1; b += kL0Threads / 32) {
    const double* z = zs + (b - b0) * M;
    double s0 = 0.0, s1 = 0.0;
    int64_t a = lane;
    for (; a + 32 < M; a += 64) {
      s0 += z[a] * kra[a];
      s1 += z[a + 32] * kra[a + 32];
    }
    for (; a < M; a += 32) s0 += z[a] * kra[a];
    const double v = warp_sum(s0 + s1);
    if (lane == 0) outA[r * sd.ldoA + b] = v;
  }
  // 3. opB partial over this chunk's b: thread per a, or G groups of threads
  //    splitting the b's when M is small (group sums added in group order)
  double* part = sd.scratch + (static_cast<int64_t>(r) * sd.nq + qc) * M;
  const int64_t nb = b1 - b0;
  const int64_t gmax = kL0Threads / M;
  const int G = M >= kL0Threads ? 1 : static_cast<int>(gmax < nb ? gmax : nb);
  if (G == 1) {
    for (int64_t a = tid; a < M; a += kL0Threads) {
      double s = 0.0;
      for (int64_t b = 0; b < nb; ++b) s += zs[b * M + a] * krb[b];
      part[a] = s;
    }
  } else {
    const int g = tid / static_cast<int>(M);
    const int64_t a = tid - static_cast<int64_t>(g) * M;
    if (g < G) {
      double s = 0.0;
      for (int64_t b = g; b < nb; b += G) s += zs[b * M + a] * krb[b];
      gp[g * M + a] = s;
    }
    __syncthreads();
    if (tid < M) {
      double s = 0.0;
      for (int q = 0; q < G; ++q) s += gp[q * M + tid];
      part[tid] = s;
    }
  }
  // 4. the last chunk CTA of (side, r) adds the partials in chunk order
  __threadfence();
  __syncthreads();
  if (tid == 0) last = atomicAdd(sd.tickets + r, 1u) == static_cast<unsigned>(sd.nq - 1);
  __syncthreads();
  if (last) {
    __threadfence();
    double* outB = sd.outB ? sd.outB : gtab[sd.slotB];
    const double* p0 = sd.scratch + static_cast<int64_t>(r) * sd.nq * M;
    for (int64_t a = tid; a < M; a += kL0Threads) {
      double s = 0.0;
      int q = 0;
      for (; q + 8 <= sd.nq; q += 8) {  // eight loads in flight, added in chunk order
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcg(p0 + static_cast<int64_t>(q + u) * M + a);
#pragma unroll
        for (int u = 0; u < 8; ++u) s += v[u];
      }
      for (; q < sd.nq; ++q) s += __ldcg(p0 + static_cast<int64_t>(q) * M + a);
      outB[r * sd.ldoB + a] = s;
    }
    if (tid == 0) sd.tickets[r] = 0u;  // ready for the next replay
  }
  tl_end(st.tl, st.tl_slot);
}

int grid_for(int64_t work, int threads, int cap) {
  const int64_t b = (work + threads - 1) / threads;
  return static_cast<int>(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace

int64_t tail_step_units(const TailStep& st) {
  int64_t n = 0;
  for (int i = 0; i < st.n; ++i) n += op_units(st.op[i]);
  return n;
}

static int64_t tail_step_cta_units(const TailStep& st) {
  int64_t n = 0;
  for (int i = 0; i < st.n; ++i) n += op_cta_units(st.op[i]);
  return n;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("CPDGPU_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// fp32 left partials of the fused fp32 seed, [band][column tile][64 r][64 j] in
// scaled units: Ls[r][j] = us_y us_r[r] sum_b Z[b][j / 64][r][j % 64] (chunked = 1,
// the operand-image kernel's staging layout: [band][column tile][16 column quads][64 r][4 j]).  Thread =
// four columns of one rank; eight bands' 16-byte loads in flight per thread, the
// bands summed in a fixed order (b % 2 into two fp64 sums, then added).
__global__ void __launch_bounds__(256) reduce_left32_kernel(const float* __restrict__ Z, int64_t nB, int64_t nC,
                                                            int64_t M, int R, const double* __restrict__ us_y,
                                                            const double* __restrict__ us_r, double* out,
                                                            double* const* gtab, int out_slot, int64_t ldo,
                                                            int chunked) {
  pdl_wait();
  if (out_slot >= 0) out = gtab[out_slot];  // the left seed is G(N): written in place
  const int64_t quads = (M + 3) / 4;
  const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (e >= quads * R) return;
  const int r = static_cast<int>(e / quads);
  const int64_t j0 = (e - r * quads) * 4;  // the four columns share a 64-column tile (padded past M)
  const int64_t jj = j0 & 63;
  const float4* z = reinterpret_cast<const float4*>(
      chunked ? Z + (((j0 >> 6) * 16 + (jj >> 2)) * 64 + r) * 4 : Z + ((j0 >> 6) * 64 + r) * 64 + jj);
  const int64_t stride = nC * 64 * 64 / 4;  // one band
  double a[4] = {0.0, 0.0, 0.0, 0.0}, b[4] = {0.0, 0.0, 0.0, 0.0};
  int64_t k = 0;
  for (; k + 7 < nB; k += 8) {
    float4 v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = __ldcs(z + (k + q) * stride);
#pragma unroll
    for (int q = 0; q < 8; q += 2) {
      a[0] += v[q].x; a[1] += v[q].y; a[2] += v[q].z; a[3] += v[q].w;
      b[0] += v[q + 1].x; b[1] += v[q + 1].y; b[2] += v[q + 1].z; b[3] += v[q + 1].w;
    }
  }
  for (; k < nB; ++k) {
    const float4 v = __ldcs(z + k * stride);
    double* d = (k & 1) ? b : a;
    d[0] += v.x; d[1] += v.y; d[2] += v.z; d[3] += v.w;
  }
  const double us = us_y[0] * us_r[r];
#pragma unroll
  for (int c = 0; c < 4; ++c)
    if (j0 + c < M) out[r * ldo + j0 + c] = (a[c] + b[c]) * us;
}

int launch_reduce_left32(const float* Z, int64_t nB, int64_t nC, int64_t M, int R, const double* us_y,
                         const double* us_r, double* out, double* const* gtab, int out_slot, int64_t ldo,
                         int chunked, cudaStream_t s) {
  const int64_t threads = ((M + 3) / 4) * R;
  launch_k(reduce_left32_kernel, dim3(static_cast<unsigned>((threads + 255) / 256)), dim3(256), 0, s, pdl_enabled(),
           Z, nB, nC, M, R, us_y, us_r, out, gtab, out_slot, ldo, chunked);
  return 1;
}

int launch_tail_step(const TailStep& st0, double* const* gtab, int num_sms, cudaStream_t s) {
  if (st0.n == 0) return 0;
  TailStep st = st0;
  for (int i = 0; i < st.n; ++i) st.op[i].cta = contract_len(st.op[i]) >= kCtaContractLen ? 1 : 0;
  const int64_t warps = tail_step_units(st), ctas = tail_step_cta_units(st);
  static const bool dbg = std::getenv("CPDGPU_TAIL_DEBUG") != nullptr;
  if (dbg) {
    std::fprintf(stderr, "[tail step] warps %lld ctas %lld:", static_cast<long long>(warps), static_cast<long long>(ctas));
    for (int i = 0; i < st.n; ++i)
      std::fprintf(stderr, " (type %d M %lld B %lld R %d cta %d)", st.op[i].type, static_cast<long long>(st.op[i].M),
                   static_cast<long long>(st.op[i].B), st.op[i].R, st.op[i].cta);
    std::fprintf(stderr, "\n");
  }
  const int grid = std::max(grid_for(warps * 32, 256, num_sms * 8), grid_for(ctas * 256, 256, num_sms * 8));
  if (ctas > 0)
    launch_k(tail_step_kernel<true>, dim3(grid), dim3(256), 0, s, pdl_enabled(), st, gtab);
  else
    launch_k(tail_step_kernel<false>, dim3(grid), dim3(256), 0, s, pdl_enabled(), st, gtab);
  return 1;
}

const void* prologue_kernel_fn() { return reinterpret_cast<const void*>(prologue_kernel); }

void prologue_geometry(const Prologue& pr, int num_sms, dim3* grid, dim3* block) {
  int64_t work = 0;
  for (int j = 0; j < pr.N; ++j) work = work > pr.len[j] ? work : pr.len[j];
  for (int c = 0; c < pr.nkr; ++c) work = work > pr.kr[c].L * pr.kr[c].LDK ? work : pr.kr[c].L * pr.kr[c].LDK;
  work = work > pr.zero_n / 4 ? work : pr.zero_n / 4;
  *grid = dim3(static_cast<unsigned>(grid_for(work, 256, num_sms * 8)));
  *block = dim3(256);
}

int launch_l0_step(const L0Step& st, double* const* gtab, cudaStream_t s) {
  int blocks = 0;
  int64_t rows = 0;
  for (int i = 0; i < st.nsides; ++i) {
    blocks += st.side[i].nq * st.R;
    rows = std::max<int64_t>(rows, static_cast<int64_t>(st.side[i].bq) * st.side[i].M);
  }
  int64_t extra = 0;  // KR values and opB group partials
  for (int i = 0; i < st.nsides; ++i) extra = std::max<int64_t>(extra, st.side[i].M + st.side[i].bq + kL0Threads);
  const size_t smem = static_cast<size_t>(rows + extra) * sizeof(double);
  static unsigned long long configured = 0;
  set_smem_attr(l0_kernel, static_cast<int>((3 * kL0MaxRows + kL0Threads) * sizeof(double)), configured);
  launch_k(l0_kernel, dim3(blocks), dim3(kL0Threads), smem, s, pdl_enabled(), st, gtab);
  return 1;
}

int launch_prologue(const Prologue& pr, double** gtab, int num_sms, cudaStream_t s) {
  dim3 grid, block;
  prologue_geometry(pr, num_sms, &grid, &block);
  prologue_kernel<<<grid, block, 0, s>>>(pr, gtab);
  return 1;
}

}  // namespace cpdgpu
