// tcgen05.mma kind::f16 issue-to-completion throughput per shape and operand source
// (one CTA per SM, one thread issues `n` MMAs back to back into one accumulator,
// commit, wait; cycles per MMA from clock64).  Build: nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -o mma_rate mma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFFu) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc_f16(bool a_mn, bool b_mn, int M, int N) {
  return (1u << 4) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}
__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile("{\n .reg .pred P;\n elect.sync _|P, 0xffffffff;\n selp.u32 %0, 1, 0, P;\n}\n" : "=r"(p));
  return p != 0;
}

template <int MODE>  // 0: SS (A smem, B smem), 1: TS (A tmem, B smem)
__global__ void __launch_bounds__(128, 1) k(int n, uint32_t idesc, int bbytes_step, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tslot;
  const uint32_t base = smem_u32(sm);
  const uint64_t a0 = sdesc(base, 8192, 1024), b0 = sdesc(base + 32768, 16, 1024);
  if (warp == 0) {
    long long t0 = clock64();
    if (elect_one()) {
      for (int i = 0; i < n; ++i) {
        const uint64_t a = a0 + ((i & 3) * 128), b = b0 + ((i & 3) * (bbytes_step >> 4));
        if (MODE == 0)
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(tmem), "l"(a), "l"(b), "r"(idesc), "r"(1));
        else
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                       ::"r"(tmem), "r"(tmem + 256 + 8 * (i & 3)), "l"(b), "r"(idesc), "r"(1));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)) : "memory");
    }
    __syncwarp();
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done) : "r"(smem_u32(&bar)) : "memory");
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  long long h[148];
  const int n = 4096;
  struct C { const char* name; int mode, M, N; bool amn, bmn; } cs[] = {
      {"SS M128 N64  A mn", 0, 128, 64, true, false},  {"SS M128 N64  A k ", 0, 128, 64, false, false},
      {"SS M128 N128 A mn", 0, 128, 128, true, false}, {"SS M128 N256 A mn", 0, 128, 256, true, false},
      {"TS M128 N64      ", 1, 128, 64, false, false}, {"TS M128 N128     ", 1, 128, 128, false, false},
      {"TS M128 N256     ", 1, 128, 256, false, false}, {"TS M128 N64 B mn ", 1, 128, 64, false, true},
      {"TS M128 N128 B mn", 1, 128, 128, false, true}, {"SS M64 N64   A k ", 0, 64, 64, false, false},
      {"TS M64 N64       ", 1, 64, 64, false, false},  {"TS M64 N128      ", 1, 64, 128, false, false},
      {"SS M128 N128 A k ", 0, 128, 128, false, false}, {"SS M128 N32  A k ", 0, 128, 32, false, false},
      {"TS M128 N32      ", 1, 128, 32, false, false},
  };
  for (int grid : {1, 148}) {
    for (auto& c : cs) {
      const uint32_t id = idesc_f16(c.amn, c.bmn, c.M, c.N);
      auto fn = c.mode == 0 ? k<0> : k<1>;
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
      for (int rep = 0; rep < 2; ++rep) fn<<<grid, 128, 100 * 1024>>>(n, id, 32, d);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < grid; ++i) avg += h[i];
      avg /= grid;
      const double flop = 2.0 * c.M * c.N * 16;
      printf("grid %3d %s : %6.1f cyc/MMA  (%5.0f flop/cyc/SM) %s\n", grid, c.name, avg / n, flop * n / avg,
             e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  return 0;
}
