// Microbenchmark: FP64 DFMA vs DMMA (mma.sync.m8n8k4.f64) throughput on B200,
// plus a plain HBM read-stream. Used to choose the fp64 seed-kernel design.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 1.0000001, c = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.0) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
  double c[8][2];
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void read_kernel(const double2* __restrict__ in, size_t n, double* out) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldg(in + i);
    s += v.x + v.y;
  }
  if (s == 12345.0) out[0] = s;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d, max clock %d kHz\n", sms, clk);
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int occ : {4, 8, 16, 32}) {
    dfma_kernel<<<sms, 32 * occ>>>(out, 100);
    cudaEventRecord(e0);
    dfma_kernel<<<sms, 32 * occ>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * iters * 32.0 * occ * sms;
    printf("DFMA warps/SM %2d: %.2f TFLOP/s\n", occ, flops / ms / 1e9);
  }
  for (int occ : {4, 8, 16, 32}) {
    dmma_kernel<<<sms, 32 * occ>>>(out, 100);
    cudaEventRecord(e0);
    dmma_kernel<<<sms, 32 * occ>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 8 * (double)iters * occ * sms;
    printf("DMMA warps/SM %2d: %.2f TFLOP/s\n", occ, flops / ms / 1e9);
  }
  size_t n = (size_t)1 << 28;  // 4 GiB of double2? no: 2^28 * 16 B = 4 GiB
  double2* buf; cudaMalloc(&buf, n * sizeof(double2));
  cudaMemset(buf, 0, n * sizeof(double2));
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    read_kernel<<<sms * 8, 256>>>(buf, n, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("read stream: %.1f GB/s\n", n * 16.0 / ms / 1e6);
  }
  cudaError_t err = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
