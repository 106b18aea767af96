// Microbenchmark: TMA streaming rate of Y (60^4 view, 3600 x 3600 fp64 reused as
// a 3600 x 36000 matrix) for the int8 seed's slot shapes and visit orders.
// One producer thread per CTA keeps `stages` boxes in flight; four consumer
// warps only wait and release (no compute), so the number is the delivery rate.
//   A: box 16 i x 64 j, 128B swizzle, row chunks c fastest (seed_i8.cu order)
//   B: box 128 i x 8 j, no swizzle (whole 1 KB column runs per request)
//   C: 3-D view (16, J/16, K), box 16 x 8 x 8 (same bytes as B, swizzled rows)
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void wait(unsigned long long* b, unsigned par) {
  unsigned done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                 : "=r"(done) : "r"(smem_u32(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void arrive_tx(unsigned long long* b, unsigned tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}

template <int MODE>
__global__ void stream(const __grid_constant__ CUtensorMap map, int J, int K, int stages, long total, int sbytes, int cw, const unsigned char* img, int bulk) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  unsigned long long* full = (unsigned long long*)(base + stages * sbytes);
  unsigned long long* empty = full + stages;
  unsigned long long* bfull = empty + stages;
  unsigned char* bbuf = base + stages * sbytes + 1024;  // bulk image landing area (12 KB)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], cw); }
    mbar_init(bfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const long a0 = blockIdx.x * total / gridDim.x, a1 = (blockIdx.x + 1) * total / gridDim.x;
  const int n = (int)(a1 - a0);
  const int nCT = (K + 127) / 128;
  if (warp == cw) {
    if (lane == 0) {
      for (int q = 0; q < n; ++q) {
        const int s = q % stages;
        if (q >= stages) wait(&empty[s], ((q / stages) - 1) & 1);
        const long u = a0 + q;
        if (bulk && (q & 7) == 0) {  // per-tile 12 KB image from L2 (as seed_i8's Khatri-Rao digits)
          if (q >= 8) wait(bfull, ((q >> 3) - 1) & 1);
          arrive_tx(bfull, 12288);
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 12288, [%2];"
                       ::"r"(smem_u32(bbuf)), "l"(img + ((u >> 3) % 301) * 12288), "r"(smem_u32(bfull)) : "memory");
        }
        arrive_tx(&full[s], sbytes);
        unsigned dst = smem_u32(base + s * sbytes), bar = smem_u32(&full[s]);
        if (MODE == 0) {  // slot = (tile, half, chunk): c fastest
          const long tile = u >> 4; const int h = (u >> 3) & 1, c = u & 7;
          const int rb = tile / nCT, ct = tile % nCT;
          int i = rb * 128 + 16 * c, j = ct * 128 + 64 * h;
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                       ::"r"(dst), "l"(&map), "r"(i), "r"(j), "r"(bar) : "memory");
        } else if (MODE == 3) {  // 16 rows x 128 columns (16 KB), c fastest
          const long tile = u >> 3; const int c = u & 7;
          const int rb = tile / nCT, ct = tile % nCT;
          int i = rb * 128 + 16 * c, j = ct * 128;
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                       ::"r"(dst), "l"(&map), "r"(i), "r"(j), "r"(bar) : "memory");
        } else if (MODE == 4) {  // 128 rows x 32 columns (32 KB)
          const long tile = u >> 2; const int s4 = u & 3;
          const int rb = tile / nCT, ct = tile % nCT;
          int i = rb * 128, j = ct * 128 + 32 * s4;
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                       ::"r"(dst), "l"(&map), "r"(i), "r"(j), "r"(bar) : "memory");
        } else if (MODE == 1) {  // 128 rows x 8 columns
          const long tile = u >> 4; const int s8 = u & 15;
          const int rb = tile / nCT, ct = tile % nCT;
          int i = rb * 128, j = ct * 128 + 8 * s8;
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                       ::"r"(dst), "l"(&map), "r"(i), "r"(j), "r"(bar) : "memory");
        } else {  // 3-D: (16 i_in, 8 i_out, 8 j)
          const long tile = u >> 4; const int s8 = u & 15;
          const int rb = tile / nCT, ct = tile % nCT;
          int io = rb * 8, j = ct * 128 + 8 * s8;
          asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                       ::"r"(dst), "l"(&map), "r"(0), "r"(io), "r"(j), "r"(bar) : "memory");
        }
      }
    }
  } else if (warp < cw) {
    for (int q = 0; q < n; ++q) {
      const int s = q % stages;
      wait(&full[s], (q / stages) & 1);
      __syncwarp();
      if (lane == 0) arrive(&empty[s]);
    }
  }
}

int main() {
  PFN_cuTensorMapEncodeTiled enc; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int J = getenv("TJ") ? atoi(getenv("TJ")) : 3584; const long K = getenv("TK") ? atol(getenv("TK")) : 36000;
  double* y; cudaMalloc(&y, (size_t)J * K * 8); cudaMemset(y, 0, (size_t)J * K * 8);
  const long tiles = (long)((J + 127) / 128) * ((K + 127) / 128);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct Cfg { int mode, rows, cols, sw, stages, cw, bulk; };
  Cfg cfgs[] = {{3, 16, 128, 1, 6, 8, 1}};
  unsigned char* img; cudaMalloc(&img, 301 * 12288); cudaMemset(img, 0, 301 * 12288);
  for (auto c : cfgs) {
    CUtensorMap map;
    cuuint64_t gd[2] = {(cuuint64_t)J, (cuuint64_t)K}; cuuint64_t gs[1] = {(cuuint64_t)J * 8};
    cuuint32_t box[2] = {(cuuint32_t)c.rows, (cuuint32_t)c.cols}; cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, y, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     c.sw ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed\n"); continue; }
    const int sbytes = c.rows * c.cols * 8;
    const long nslots = tiles * (131072 / sbytes);
    const size_t smem = 1024 + (size_t)c.stages * sbytes + 1024 + 12288 + 512;
    auto fn = c.mode == 0 ? stream<0> : (c.mode == 1 ? stream<1> : (c.mode == 3 ? stream<3> : stream<4>));
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      fn<<<sms, 32 * (c.cw + 1), smem>>>(map, J, (int)K, c.stages, nslots, sbytes, c.cw, img, c.bulk);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 1) printf("box %3d x %3d sw %d stages %2d (%3d KB in flight) consumers %d bulk %d: %7.1f GB/s\n", c.rows,
                           c.cols, c.sw, c.stages, c.stages * sbytes / 1024, c.cw, c.bulk, (double)J * K * 8 / ms / 1e6);
    }
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
}
