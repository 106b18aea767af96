// Per-tile tcgen05 cost of the fused fp32 seed's MMA sequence (seed_f32i_kernel)
// and of alternative sequences, with no data movement: one CTA per SM, one
// elected lane issues T tiles back to back, one commit per tile (as the kernel's
// ring-slot release), cycles per tile from clock64.  Optional drain warps read
// TMEM columns continuously (the kernel's drains) to measure TMEM-read contention.
//
//   0 kernel:   right 4 x (SS hh, SS hl, SS lh) M128 N64 into D_R[t % 3],
//               left 8 x (TS h, TS l) M128 N64 into D_L[u & 1]
//   1 right only (SS part of 0)          2 left only (TS part of 0)
//   3 stacked:  right 4 x (SS h*[h|l] N128, SS l*h N64), left as 0
//   4 transposed right: 4 x (TS N128 B=Y_h mn, TS N128 B=Y_l mn), left as 0
//   5 kernel sequence, right and left interleaved per K step
//   6 kernel sequence + the MMA warp's per-tile / per-unit barrier waits (on
//     completed barriers), fences and commits (one warp)
//   7 as 6, right MMAs issued by warp 0 and left MMAs by warp 1
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_mix mma_mix.cu
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
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
               ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
               ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

constexpr int kPlane = 16384;
__device__ __forceinline__ void wait_done(uint64_t* bar) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(smem_u32(bar)) : "memory");
}
template <int V>
__global__ void __launch_bounds__(256, 1) k(int tiles, int drains, long long* out, unsigned* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tslot;
  __shared__ volatile int stop, stop2;
  const int warp = threadIdx.x >> 5;
  uint32_t x = 0x9E3779B9u * (threadIdx.x + 1) + blockIdx.x;
  for (int i = threadIdx.x; i < 128 * 1024 / 4; i += blockDim.x) {  // random fp16 pairs in [-1, 1]
    x ^= x << 13; x ^= x >> 17; x ^= x << 5;
    const uint32_t lo = 0x3800u | (x & 0x3FFu) | ((x >> 10) & 1u) << 15, hi = 0x3800u | ((x >> 11) & 0x3FFu) | ((x >> 21) & 1u) << 15;
    reinterpret_cast<uint32_t*>(sm)[i] = lo | (hi << 16);
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar[i])));
    stop = 0;
    stop2 = 0;
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&bar[2])) : "memory");  // phase 0 done
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
  if (warp == 0) {
    const uint32_t id_r = idesc_f16(true, false, 128, 64), id_r128 = idesc_f16(true, false, 128, 128);
    const uint32_t id_l = idesc_f16(false, false, 128, 64), id_t = idesc_f16(false, true, 128, 128);
    const uint64_t dA0 = sdesc(base, 8192, 1024), dB0 = sdesc(base + 2 * 32768, 16, 1024), dL0 = sdesc(base, 16, 1024);
    long long t0 = clock64();
    for (int u = 0; u < tiles; ++u) {
      const int s = u & 1, t = u % 3;
      const uint64_t pa = static_cast<uint64_t>((s * 2 * kPlane) >> 4);
      const uint64_t aH = dA0 + pa, aL = aH + (kPlane >> 4), lH = dL0 + pa, lL = lH + (kPlane >> 4);
      const uint64_t kb = dB0;
      const uint32_t dR = tmem + 64 * t, aK = tmem + 192 + 64 * t, dL = tmem + 384 + 64 * ((u / 3) & 1);
      if (elect_one()) {
        if (V == 0 || V == 1) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            mma_ss(dR, aH + q * 128, kb + q * 2, id_r, q != 0);
            mma_ss(dR, aH + q * 128, kb + 512 + q * 2, id_r, 1u);
            mma_ss(dR, aL + q * 128, kb + q * 2, id_r, 1u);
          }
        }
        if (V == 3) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            mma_ss(tmem + 128 * (t & 1), aH + q * 128, kb + q * 2, id_r128, q != 0);
            mma_ss(tmem + 128 * (t & 1), aL + q * 128, kb + q * 2, id_r, 1u);
          }
        }
        if (V == 4) {  // D^T[m][i] += KRr^T[m][j] Y[i][j]: A in TMEM (cols 192..), B = plane MN-major (i contiguous)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            mma_ts(tmem + 128 * (t & 1), aK + 8 * q, aH + q * 128, id_t, q != 0);
            mma_ts(tmem + 128 * (t & 1), aK + 8 * q, aL + q * 128, id_t, 1u);
          }
        }
        if (V == 0 || V == 2 || V == 3 || V == 4) {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const uint32_t off = ((q >> 2) * 8192 + (q & 3) * 32) >> 4;
            mma_ts(dL, aK + 8 * q, lH + off, id_l, q != 0);
            mma_ts(dL, aK + 8 * q, lL + off, id_l, 1u);
          }
        }
        if (V == 5) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            mma_ss(dR, aH + q * 128, kb + q * 2, id_r, q != 0);
            mma_ss(dR, aH + q * 128, kb + 512 + q * 2, id_r, 1u);
            mma_ss(dR, aL + q * 128, kb + q * 2, id_r, 1u);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int ql = 2 * q + h;
              const uint32_t off = ((ql >> 2) * 8192 + (ql & 3) * 32) >> 4;
              mma_ts(dL, aK + 8 * ql, lH + off, id_l, ql != 0);
              mma_ts(dL, aK + 8 * ql, lL + off, id_l, 1u);
            }
          }
        }
        if (V == 6 || V == 7) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            mma_ss(dR, aH + q * 128, kb + q * 2, id_r, q != 0);
            mma_ss(dR, aH + q * 128, kb + 512 + q * 2, id_r, 1u);
            mma_ss(dR, aL + q * 128, kb + q * 2, id_r, 1u);
          }
          if (V == 6) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const uint32_t off = ((q >> 2) * 8192 + (q & 3) * 32) >> 4;
              mma_ts(dL, aK + 8 * q, lH + off, id_l, q != 0);
              mma_ts(dL, aK + 8 * q, lL + off, id_l, 1u);
            }
          }
        }
        commit(&bar[0]);
        if ((V == 6 || V == 7) && t == 2) {
          commit(&bar[3]);
          commit(&bar[3]);
        }
      }
      __syncwarp();
      if (V == 6 || V == 7) {  // the kernel's waits (all on completed barriers) and fences
        wait_done(&bar[2]);
        if (t == 2) {
          wait_done(&bar[2]);
          wait_done(&bar[2]);
          wait_done(&bar[2]);
        }
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      }
    }
    if (elect_one()) commit(&bar[1]);
    __syncwarp();
    if (V == 7) {
      while (!stop2) {}
    }
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done) : "r"(smem_u32(&bar[1])) : "memory");
    long long t1 = clock64();
    if (threadIdx.x == 0) {
      out[blockIdx.x] = t1 - t0;
      stop = 1;
    }
  } else if (V == 7 && warp == 1) {  // left MMAs of variant 7
    const uint32_t id_l = idesc_f16(false, false, 128, 64);
    const uint64_t dL0 = sdesc(base, 16, 1024);
    for (int u = 0; u < tiles; ++u) {
      const int s = u & 1, t = u % 3;
      const uint64_t lH = dL0 + static_cast<uint64_t>((s * 2 * kPlane) >> 4), lL = lH + (kPlane >> 4);
      const uint32_t aK = tmem + 192 + 64 * t, dL = tmem + 384 + 64 * ((u / 3) & 1);
      if (elect_one()) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint32_t off = ((q >> 2) * 8192 + (q & 3) * 32) >> 4;
          mma_ts(dL, aK + 8 * q, lH + off, id_l, q != 0);
          mma_ts(dL, aK + 8 * q, lL + off, id_l, 1u);
        }
        commit(&bar[0]);
        if (t == 2) commit(&bar[3]);
      }
      __syncwarp();
      wait_done(&bar[2]);
      if (t == 2) {
        wait_done(&bar[2]);
        wait_done(&bar[2]);
      }
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    }
    if (elect_one()) commit(&bar[2 + 1]);
    __syncwarp();
    if (threadIdx.x == 32) stop2 = 1;
  } else if (warp >= 4 && warp < 4 + drains) {  // TMEM readers: the lane quarter warp % 4
    const uint32_t lanes = static_cast<uint32_t>((warp & 3) * 32) << 16;
    uint32_t acc = 0;
    int it = 0;
    while (!stop) {
      uint32_t v[16];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];\n"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                     "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                   : "r"(tmem + lanes + 384 + 16 * (it & 7)));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      for (int e = 0; e < 16; ++e) acc += v[e];
      ++it;
      for (int d = 0; d < 64; ++d) __nanosleep(0);
    }
    if (acc == 0x12345678u) sink[0] = acc;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

int main() {
  long long* d;
  unsigned* sink;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaMalloc(&sink, 4);
  long long h[148];
  const int tiles = 6000;
  const char* names[] = {"kernel seq (12 SS + 16 TS)", "right only (12 SS N64)", "left only (16 TS N64)",
                         "stacked right (4 SS N128 + 4 SS N64) + left", "transposed right (8 TS N128 B mn) + left",
                         "kernel seq interleaved per K step", "kernel seq + waits/fences/commits, 1 warp",
                         "kernel seq + waits/fences/commits, 2 warps"};
  auto run = [&](auto fn, int v, int drains) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 130 * 1024);
    for (int rep = 0; rep < 2; ++rep) fn<<<148, 256, 130 * 1024>>>(tiles, drains, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 148 * sizeof(long long), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    printf("%-46s drains %d : %7.1f cyc/tile %s\n", names[v], drains, avg / tiles, e == cudaSuccess ? "" : cudaGetErrorString(e));
  };
  for (int drains : {0, 4}) {
    run(k<0>, 0, drains);
    run(k<1>, 1, drains);
    run(k<2>, 2, drains);
    run(k<3>, 3, drains);
    run(k<4>, 4, drains);
    run(k<5>, 5, drains);
    run(k<6>, 6, drains);
    run(k<7>, 7, drains);
  }
  return 0;
}
