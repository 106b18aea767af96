// tail.cu — seed-partial reductions and the rank-batched TTV recursion tail.
//
// Reference: the right phase  (mttkrp.cpp:165-193; Eq 3.20 recursion, Eq 3.12
// extraction) and the left phase (mttkrp.cpp:212-241; Eq 3.22 recursion,
// Eq 3.16 extraction).  The reference runs one GEMV per rank column r; here
// every launch covers all R columns at once ("rank-batched"), with the
// Khatri-Rao vector generated on the fly from factor rows.
#include "kernels.h"

namespace cpdgpu {
namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// CTA whose tile range [t0, t1) contains tile t (t0(c) = floor(c T / P)).
__device__ __forceinline__ int64_t cta_of(int64_t t, int64_t T, int64_t P) {
  return ((t + 1) * P + T - 1) / T - 1;
}

__global__ void reduce_right_kernel(const SeedParams p, int RP, double* Rs, int64_t ldo) {
  const int64_t total = p.J * p.R;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(e / p.J);
    const int64_t i = e - r * p.J;
    const int64_t rb = i / p.TI, il = i - rb * p.TI;
    const int64_t c0 = cta_of(rb * p.nCT, p.T, p.P);
    const int64_t c1 = cta_of((rb + 1) * p.nCT - 1, p.T, p.P);
    double s = 0.0;
    for (int64_t c = c0; c <= c1; ++c) {
      const int64_t ta = (c * p.T) / p.P, tb = ((c + 1) * p.T) / p.P;
      if (ta >= tb) continue;
      const int64_t slot = c * p.slots + (rb - ta / p.nCT);
      s += p.Rpart[(slot * RP + r) * p.TI + il];
    }
    Rs[r * ldo + i] = s;
  }
}

__global__ void reduce_left_kernel(const double* Lpart, int64_t nRB, int R, int64_t K, double* Ls,
                                   int64_t ldo) {
  const int64_t total = K * R;
  const int64_t stride = static_cast<int64_t>(R) * K;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(e / K);
    const int64_t j = e - r * K;
    double s = 0.0;
    for (int64_t rb = 0; rb < nRB; ++rb) s += Lpart[rb * stride + e];
    Ls[r * ldo + j] = s;
  }
}

// One warp per output (b, r): a contiguous dot product of length M.
__global__ void contract_a_kernel(const double* __restrict__ Z, int64_t ldz, int64_t M, int64_t B,
                                  int R, const KRSpec v, double* __restrict__ out, int64_t ldo) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t w = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; w < B * R;
       w += nw) {
    const int r = static_cast<int>(w / B);
    const int64_t b = w - r * B;
    const double* z = Z + r * ldz + M * b;
    double s = 0.0;
    for (int64_t a = lane; a < M; a += 32) s += z[a] * kr_entry(v, a, r);
    s = warp_sum(s);
    if (lane == 0) out[r * ldo + b] = s;
  }
}

// out[r][a] = sum_b Z[r][a + M b] w[b, r]: threads over a (coalesced), groups
// over b, fixed-order shared-memory reduction, optional split of the b range
// with a second deterministic pass.
constexpr int kCB = 256;

__global__ void contract_b_kernel(const double* __restrict__ Z, int64_t ldz, int64_t M, int64_t B,
                                  int R, const KRSpec w, double* __restrict__ out, int64_t ldo,
                                  int TA, int64_t nAB, int S, double* __restrict__ part) {
  __shared__ double red[kCB];
  const int NB = kCB / TA;
  const int tid = threadIdx.x;
  const int al = tid % TA, bg = tid / TA;
  const int64_t ab = blockIdx.x % nAB;
  const int s = static_cast<int>(blockIdx.x / nAB);
  const int r = blockIdx.y;
  const int64_t a = ab * TA + al;
  const int64_t b0 = (B * s) / S, b1 = (B * (s + 1)) / S;
  double acc = 0.0;
  if (a < M) {
    const double* z = Z + r * ldz + a;
    for (int64_t b = b0 + bg; b < b1; b += NB) acc += z[M * b] * kr_entry(w, b, r);
  }
  red[tid] = acc;
  __syncthreads();
  if (bg == 0 && a < M) {
    double tot = 0.0;
    for (int q = 0; q < NB; ++q) tot += red[q * TA + al];
    if (S == 1) out[r * ldo + a] = tot;
    else part[(static_cast<int64_t>(s) * R + r) * M + a] = tot;
  }
}

__global__ void contract_b_finish(const double* __restrict__ part, int64_t M, int R, int S,
                                  double* __restrict__ out, int64_t ldo) {
  const int64_t total = M * R;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(e / M);
    const int64_t a = e - r * M;
    double tot = 0.0;
    for (int s = 0; s < S; ++s) tot += part[(static_cast<int64_t>(s) * R + r) * M + a];
    out[r * ldo + a] = tot;
  }
}

int grid_for(int64_t work, int threads) {
  const int64_t b = (work + threads - 1) / threads;
  return static_cast<int>(b < 1 ? 1 : (b > 65535 * 16 ? 65535 * 16 : b));
}

void contract_b_shape(int64_t M, int64_t B, int R, int num_sms, int* TA, int64_t* nAB, int* S) {
  int ta = 32;
  while (ta < M && ta < kCB) ta *= 2;
  *TA = ta;
  *nAB = (M + ta - 1) / ta;
  const int64_t base = *nAB * R;
  const int64_t want = 2LL * num_sms;
  int64_t s = base >= want ? 1 : (want + base - 1) / base;
  const int64_t per = (kCB / ta);  // b-groups per CTA
  const int64_t smax = (B + per * 8 - 1) / (per * 8);  // keep >= 8 b per group
  if (s > smax) s = smax;
  if (s < 1) s = 1;
  *S = static_cast<int>(s);
}

}  // namespace

int launch_reduce_right(const SeedParams& p, int RP, double* Rs, int64_t ldo, cudaStream_t s) {
  const int64_t work = p.J * p.R;
  reduce_right_kernel<<<grid_for(work, 256), 256, 0, s>>>(p, RP, Rs, ldo);
  return 1;
}

int launch_reduce_left(const double* Lpart, int64_t nRB, int R, int64_t K, double* Ls,
                        int64_t ldo, cudaStream_t s) {
  reduce_left_kernel<<<grid_for(K * R, 256), 256, 0, s>>>(Lpart, nRB, R, K, Ls, ldo);
  return 1;
}

int launch_contract_a(const double* Z, int64_t ldz, int64_t M, int64_t B, int R,
                       const KRSpec& v, double* out, int64_t ldo, cudaStream_t s) {
  const int64_t warps = B * R;
  contract_a_kernel<<<grid_for(warps * 32, 256), 256, 0, s>>>(Z, ldz, M, B, R, v, out, ldo);
  return 1;
}

size_t contract_b_scratch(int64_t M, int64_t B, int R, int num_sms) {
  int TA, S;
  int64_t nAB;
  contract_b_shape(M, B, R, num_sms, &TA, &nAB, &S);
  return S > 1 ? static_cast<size_t>(S) * R * M : 0;
}

int launch_contract_b(const double* Z, int64_t ldz, int64_t M, int64_t B, int R,
                       const KRSpec& w, double* out, int64_t ldo, double* part, int num_sms,
                       cudaStream_t s) {
  int TA, S;
  int64_t nAB;
  contract_b_shape(M, B, R, num_sms, &TA, &nAB, &S);
  dim3 grid(static_cast<unsigned>(nAB * S), static_cast<unsigned>(R));
  contract_b_kernel<<<grid, kCB, 0, s>>>(Z, ldz, M, B, R, w, out, ldo, TA, nAB, S, part);
  if (S > 1) contract_b_finish<<<grid_for(M * R, 256), 256, 0, s>>>(part, M, R, S, out, ldo);
  return S > 1 ? 2 : 1;
}

}  // namespace cpdgpu
