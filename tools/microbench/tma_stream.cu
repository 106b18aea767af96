// TMA streaming throughput on B200: a J x K fp64 column-major matrix streamed
// through shared memory in {rows x cols} boxes, `stages`-deep mbarrier ring,
// one persistent CTA per SM, one elected issuer.  Used to size the K1 tile.
#include <cstdio>
#include <cstring>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ void arrive_tx(uint64_t* b, uint32_t tx) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(tx) : "memory"); }
__device__ void wait(uint64_t* b, uint32_t par) {
  uint32_t done = 0;
  while (!done) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(su32(b)), "r"(par) : "memory");
}
__device__ void tma(void* dst, const CUtensorMap* m, int c0, int c1, uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               ::"r"(su32(dst)), "l"((uint64_t)m), "r"(c0), "r"(c1), "r"(su32(bar)) : "memory");
}

__global__ void stream(const __grid_constant__ CUtensorMap map, int J, int K, int rows, int cols, int stages, int warps, double* out, int delay) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* full = (uint64_t*)sm; uint64_t* empty = full + 16;
  double* buf = (double*)(sm + 1024);
  const int nRB = (J + rows - 1) / rows, nCT = (K + cols - 1) / cols;
  const long T = (long)nRB * nCT;
  const long t0 = blockIdx.x * T / gridDim.x, t1 = (blockIdx.x + 1) * T / gridDim.x;
  const int nt = (int)(t1 - t0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], warps); } asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  const uint32_t bytes = rows * cols * 8;
  auto issue = [&](int k) { long tile = t0 + k; int rb = tile / nCT, ct = tile % nCT; int s = k % stages;
    arrive_tx(&full[s], bytes); tma(buf + (size_t)s * rows * cols, &map, rb * rows, ct * cols, &full[s]); };
  if (threadIdx.x == 0) for (int k = 0; k < stages && k < nt; ++k) issue(k);
  double acc = 0;
  for (int k = 0; k < nt; ++k) {
    if (threadIdx.x == 0 && k > 0 && k - 1 + stages < nt) { wait(&empty[(k - 1) % stages], ((k - 1) / stages) & 1); issue(k - 1 + stages); }
    const int s = k % stages;
    wait(&full[s], (k / stages) & 1);
    acc += buf[(size_t)s * rows * cols + threadIdx.x];
    if (delay) { long long t0c = clock64(); while (clock64() - t0c < delay) acc += 1e-300; }
    __syncwarp();
    if (lane == 0) arrive(&empty[s]);
  }
  if (acc == 1.234) out[0] = acc;
}


// variant: dedicated producer warp (warp `warps`), consumers spin `delay` cycles per tile
__global__ void stream_prod(const __grid_constant__ CUtensorMap map, int J, int K, int rows, int cols, int stages, int warps, double* out, int delay) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* full = (uint64_t*)sm; uint64_t* empty = full + 16;
  double* buf = (double*)(sm + 1024);
  const int nRB = (J + rows - 1) / rows, nCT = (K + cols - 1) / cols;
  const long T = (long)nRB * nCT;
  const long t0 = blockIdx.x * T / gridDim.x, t1 = (blockIdx.x + 1) * T / gridDim.x;
  const int nt = (int)(t1 - t0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], warps); } asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  const uint32_t bytes = rows * cols * 8;
  if (warp == warps) {
    if (lane == 0)
      for (int k = 0; k < nt; ++k) {
        const int s = k % stages;
        if (k >= stages) wait(&empty[s], ((k / stages) - 1) & 1);
        long tile = t0 + k; int rb = tile / nCT, ct = tile % nCT;
        arrive_tx(&full[s], bytes); tma(buf + (size_t)s * rows * cols, &map, rb * rows, ct * cols, &full[s]);
      }
    return;
  }
  double acc = 0;
  long long wsum = 0, tstart = clock64();
  for (int k = 0; k < nt; ++k) {
    const int s = k % stages;
    long long w0 = clock64();
    wait(&full[s], (k / stages) & 1);
    wsum += clock64() - w0;
    acc += buf[(size_t)s * rows * cols + threadIdx.x];
    if (delay) { long long t0c = clock64(); while (clock64() - t0c < delay) acc += 1e-300; }
    __syncwarp();
    if (lane == 0) arrive(&empty[s]);
  }
  if (acc == 1.234) out[0] = acc;
  if (blockIdx.x == 0 && lane == 0 && warp < 4) printf("  warp %d: wait %lld of %lld cycles over %d tiles\n", warp, wsum, clock64() - tstart, nt);
}

int main() {
  PFN_cuTensorMapEncodeTiled enc; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int J = 3600; const long K = 36000;  // 1.04 GB
  double* y; cudaMalloc(&y, (size_t)J * K * 8); cudaMemset(y, 0, (size_t)J * K * 8);
  double* out; cudaMalloc(&out, 8);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448); cudaFuncSetAttribute(stream_prod, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
  struct Cfg { int rows, cols, stages, warps; };
  Cfg cfgs[] = {{188, 32, 3, -16}};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (auto c : cfgs) {
    CUtensorMap map;
    cuuint64_t gd[2] = {(cuuint64_t)J, (cuuint64_t)K}; cuuint64_t gs[1] = {(cuuint64_t)J * 8};
    cuuint32_t box[2] = {(cuuint32_t)c.rows, (cuuint32_t)c.cols}; cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, y, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    size_t smem = 1024 + (size_t)c.stages * c.rows * c.cols * 8;
    if (r != CUDA_SUCCESS || smem > 232448) { printf("skip %d %d %d\n", c.rows, c.cols, c.stages); continue; }
    for (int delay : {3000}) {
     int d = delay * c.rows * c.cols / (188 * 32);
     for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (c.warps < 0) stream_prod<<<sms, 32 * (-c.warps + 1), smem>>>(map, J, (int)K, c.rows, c.cols, c.stages, -c.warps, out, d);
      else stream<<<sms, 32 * c.warps, smem>>>(map, J, (int)K, c.rows, c.cols, c.stages, c.warps, out, d);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      long tiles = (long)((J + c.rows - 1) / c.rows) * ((K + c.cols - 1) / c.cols);
      if (rep == 1) printf("box %3d x %2d stages %d delay %5d cyc/tile: %7.1f GB/s, %6.0f cycles/tile (1.965 GHz)\n", c.rows, c.cols, c.stages, d,
                           (double)J * K * 8 / ms / 1e6, ms * 1e-3 * 1.965e9 / (tiles / (double)sms));
     }
    }
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
}
