// DMMA (mma.sync.m8n8k4.f64) latency / throughput under different operand and
// ILP patterns on B200 — used to size the K1 consumer loops.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

// CH independent accumulator chains, operands from registers (varying a per chain)
template <int CH>
__global__ void chains(double* out, int iters) {
  double c[CH][2];
  double a[CH], b = 1.0 + threadIdx.x * 1e-9;
  for (int i = 0; i < CH; ++i) { c[i][0] = c[i][1] = 0; a[i] = 1e-3 * (i + threadIdx.x); }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) dmma(c[i], a[i], b);
  }
  double s = 0;
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}

// operands streamed from shared memory like the GEMM1 loop: per k-step NB b-frags,
// MF a-frags, MF*NB DMMAs
template <int MF, int NB>
__global__ void smem_gemm(double* out, int iters) {
  __shared__ double sm[64 * 64];
  for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) sm[i] = 1e-3 * i;
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double c[MF][NB][2];
  for (int m = 0; m < MF; ++m) for (int n = 0; n < NB; ++n) c[m][n][0] = c[m][n][1] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 2
    for (int ks = 0; ks < 8; ++ks) {
      double b[NB];
#pragma unroll
      for (int n = 0; n < NB; ++n) b[n] = sm[(ks * 4 + t) * 24 + n * 8 + g];
#pragma unroll
      for (int m = 0; m < MF; ++m) {
        const double a = sm[1024 + (m * 8 + g) + (ks * 4 + t) * 200 % 2048];
#pragma unroll
        for (int n = 0; n < NB; ++n) dmma(c[m][n], a, b[n]);
      }
    }
  }
  double s = 0;
  for (int m = 0; m < MF; ++m) for (int n = 0; n < NB; ++n) s += c[m][n][0] + c[m][n][1];
  if (s == 1.2345) out[0] = s;
}

// every DMMA with fresh A and B registers (no operand reuse between neighbours)
template <int CH>
__global__ void noreuse(double* out, int iters) {
  double c[CH][2], a[CH], b[CH];
  for (int i = 0; i < CH; ++i) { c[i][0] = c[i][1] = 0; a[i] = 1e-3 * (i + threadIdx.x); b[i] = 1.0 + 1e-6 * i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) dmma(c[i], a[i], b[i]);
  }
  double s = 0;
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}

template <typename F>
float timeit(F f) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f();
  cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); return ms;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 8);
  const int iters = 4000;
  auto report = [&](const char* name, int warps_per_sm, double dmma_per_warp, float ms) {
    double fl = 2.0 * 256 * dmma_per_warp * warps_per_sm * sms * 32 / 32;  // per warp 256 FMA
    printf("%-34s warps/SM %2d: %6.2f TF/s  (%.1f cycles/DMMA/SMSP at 1.965 GHz)\n", name, warps_per_sm,
           fl / ms / 1e9, (ms * 1e-3 * 1.965e9) / (dmma_per_warp * warps_per_sm / 4));
  };
#define CH(N)                                                                                         \
  for (int w : {4, 8}) {                                                                              \
    float ms = timeit([&] { chains<N><<<sms, 32 * w>>>(out, iters); });                              \
    report("chains<" #N ">", w, (double)N * iters, ms);                                              \
  }
  CH(1) CH(2) CH(4) CH(6) CH(8) CH(16)
#define SG(M, N)                                                                                      \
  for (int w : {4, 8}) {                                                                              \
    float ms = timeit([&] { smem_gemm<M, N><<<sms, 32 * w>>>(out, iters / 8); });                    \
    report("smem_gemm<" #M "," #N ">", w, (double)M * N * 8 * (iters / 8), ms);                       \
  }
  SG(6, 3) SG(7, 2) SG(4, 3) SG(2, 3) SG(1, 3)
#define NR(N)                                                                                         \
  for (int w : {4, 8, 16}) {                                                                          \
    float ms = timeit([&] { noreuse<N><<<sms, 32 * w>>>(out, iters); });                             \
    report("noreuse<" #N ">", w, (double)N * iters, ms);                                             \
  }
  NR(4) NR(8) NR(12)
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
}
