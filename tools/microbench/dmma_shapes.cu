// Microbenchmark: fp64 mma.sync shapes on B200 (m8n8k4 vs m16n8k4 / k8 / k16):
// throughput with independent accumulator chains, 4 and 8 warps per SM.
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void m8n8k4(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
  double c[CH][2] = {};
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  double s = 0;
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}
template <int CH>
__global__ void m16n8k4(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 + threadIdx.x * 1e-6;
  double c[CH][4] = {};
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  double s = 0;
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.0) out[0] = s;
}
template <int CH>
__global__ void m16n8k8(double* out, int iters) {
  double a[4], b0 = 1.0 + threadIdx.x * 1e-6, b1 = b0 + 1;
  for (int i = 0; i < 4; ++i) a[i] = threadIdx.x * 1e-3 + i;
  double c[CH][4] = {};
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b0), "d"(b1));
  double s = 0;
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.0) out[0] = s;
}
template <int CH>
__global__ void m16n8k16(double* out, int iters) {
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + i * 1e-6;
  double c[CH][4] = {};
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
                   "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  double s = 0;
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.0) out[0] = s;
}

template <typename K>
void run(const char* name, K k, double flop_per_mma, int ch, int iters) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w : {4, 8}) {
    k<<<sms, 32 * w>>>(out, 10);
    cudaEventRecord(e0);
    k<<<sms, 32 * w>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double flops = flop_per_mma * ch * (double)iters * w * sms;
    printf("%-10s chains %d warps/SM %d: %.2f TF/s  (%s)\n", name, ch, w, flops / ms / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  cudaFree(out);
}

int main() {
  run("m8n8k4", m8n8k4<8>, 2.0 * 8 * 8 * 4, 8, 20000);
  run("m16n8k4", m16n8k4<8>, 2.0 * 16 * 8 * 4, 8, 10000);
  run("m16n8k8", m16n8k8<8>, 2.0 * 16 * 8 * 8, 8, 5000);
  run("m16n8k16", m16n8k16<4>, 2.0 * 16 * 8 * 16, 4, 5000);
  run("m16n8k16", m16n8k16<8>, 2.0 * 16 * 8 * 16, 8, 2500);
  return 0;
}
