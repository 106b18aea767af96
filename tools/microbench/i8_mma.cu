// Microbenchmark + layout check: tcgen05.mma kind::i8 on B200 for the digit
// planes of the int8 fp64 seed (seed_i8.cu).  One 128 x 128 int8 plane stored
// as rows j of 128 bytes (i contiguous, 128-byte swizzle) serves
//   right: D_R[i][r] = sum_j P[i][j] B_R[r][j]   (A = P, M = i, MN-major)
//   left:  D_L[j][r] = sum_i P[i][j] B_L[r][i]   (A = P^T, M = j, K-major)
// Part 1 checks both products against host integer math; part 2 times the
// per-tile MMA schedule (21 digit pairs x both products) on every SM.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__host__ __device__ inline int swz(int row, int col) { return row * 128 + ((((col >> 4) ^ (row & 7))) << 4) + (col & 15); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFFu) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc_i8(bool a_mn, int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | (static_cast<uint32_t>(n >> 3) << 17) |
         (8u << 24);
}
// M = 64 probe: left product for rows j 0..63 only; dump all 128 lanes x N columns
__host__ __device__ constexpr uint32_t idesc_i8_m(bool a_mn, int n, int m) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}
__host__ __device__ inline int8_t val(uint32_t seed, uint32_t idx) {
  uint32_t x = seed * 0x9E3779B9u + idx;
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return static_cast<int8_t>(x & 0xFF);
}

template <int N>
__global__ void __launch_bounds__(128, 1) check(int32_t* outR, int32_t* outL) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  unsigned char* P = base;             // [128 j][128 i]
  unsigned char* BR = P + 16384;       // [N r][128 j]
  unsigned char* BL = BR + N * 128;    // [N r][128 i]
  uint64_t* bar = reinterpret_cast<uint64_t*>(BL + N * 128);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < 128 * 128; e += 128) {
    const int i = e & 127, j = e >> 7;
    P[swz(j, i)] = static_cast<unsigned char>(val(1, i + 128 * j));
  }
  for (int e = tid; e < N * 128; e += 128) {
    const int k = e & 127, r = e >> 7;
    BR[swz(r, k)] = static_cast<unsigned char>(val(2, k + 128 * r));
    BL[swz(r, k)] = static_cast<unsigned char>(val(3, k + 128 * r));
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;\n" ::"r"(smem_u32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *slot;
  if (tid == 0) {
    const uint32_t p = smem_u32(P), br = smem_u32(BR), bl = smem_u32(BL);
    for (int ks = 0; ks < 4; ++ks) {
      // right: A MN-major, K step 32 j = 4 KB; B K-major, +32 B per step
      mma_i8(tmem, desc(p + ks * 4096, 16384, 1024), desc(br + ks * 32, 16, 1024), idesc_i8(true, N), ks > 0);
      // left: A K-major (rows j), +32 B per step
      mma_i8(tmem + N, desc(p + ks * 32, 16, 1024), desc(bl + ks * 32, 16, 1024), idesc_i8(false, N), ks > 0);
    }
    commit(bar);
  }
  mbar_wait(bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const int row = warp * 32 + (tid & 31);
  for (int c = 0; c < 2 * N; ++c) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(v)
                 : "r"(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    if (c < N) outR[row * N + c] = static_cast<int32_t>(v);
    else outL[row * N + c - N] = static_cast<int32_t>(v);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;\n" ::"r"(tmem));
}

// Timing: per "tile" 21 digit pairs x (right 4 K-steps + left 4 K-steps), 6 + 6
// accumulators of N columns; commit + wait per tile.
template <int N, bool STACK, bool HALF = false>
__global__ void __launch_bounds__(128, 1) timing(int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  unsigned char* P = base;                 // 6 planes [128][128]
  unsigned char* BR = P + 6 * 16384;       // 6 planes [N][128]
  unsigned char* BL = BR + 6 * N * 128;
  uint64_t* bar = reinterpret_cast<uint64_t*>(BL + 6 * N * 128);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < (6 * 16384 + 12 * N * 128) / 4; e += 128) reinterpret_cast<uint32_t*>(P)[e] = hsh(e);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *slot;
  if (tid == 0) {
    const unsigned long long t0 = clock64();
    const uint32_t p = smem_u32(P), br = smem_u32(BR), bl = smem_u32(BL);
    for (int it = 0; it < iters; ++it) {
      if (HALF) {
#pragma unroll 1
        for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
          for (int ks = 0; ks < 2; ++ks)
#pragma unroll
            for (int a = 0; a < 6; ++a)
              mma_i8(tmem + a * N, desc(p + a * 16384 + hh * 8192 + ks * 4096, 16384, 1024),
                     desc(br + hh * 64 + ks * 32, 16, 1024), idesc_i8(true, N * (6 - a)), (ks > 0 || a > 0 || hh > 0) ? 1u : 0u);
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
#pragma unroll
            for (int a = 0; a < 6; ++a)
              mma_i8(tmem + (static_cast<uint32_t>(16 * hh) << 16) + 6 * N + a * N,
                     desc(p + a * 16384 + hh * 8192 + ks * 32, 16, 1024), desc(bl + ks * 32, 16, 1024),
                     idesc_i8_m(false, N * (6 - a), 64), (ks > 0 || a > 0) ? 1u : 0u);
        }
      } else if (STACK) {
        // one MMA per Y plane a and K step: B planes b = 0..5-a stacked along N,
        // D starts at diagonal a (column block b -> diagonal a + b)
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
#pragma unroll
          for (int a = 0; a < 6; ++a) {
            const uint32_t pa = p + a * 16384;
            mma_i8(tmem + a * N, desc(pa + ks * 4096, 16384, 1024), desc(br + ks * 32, 16, 1024),
                   idesc_i8(true, N * (6 - a)), (ks > 0 || a > 0) ? 1u : 0u);
            mma_i8(tmem + 6 * N + a * N, desc(pa + ks * 32, 16, 1024), desc(bl + ks * 32, 16, 1024),
                   idesc_i8(false, N * (6 - a)), (ks > 0 || a > 0) ? 1u : 0u);
          }
      } else {
      for (int a = 0; a < 6; ++a)
        for (int b = 0; b < 6 - a; ++b) {
          const uint32_t dR = tmem + (a + b) * N, dL = tmem + 6 * N + (a + b) * N;
          const uint32_t pa = p + a * 16384;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            mma_i8(dR, desc(pa + ks * 4096, 16384, 1024), desc(br + b * N * 128 + ks * 32, 16, 1024),
                   idesc_i8(true, N), (ks > 0 || b > 0) ? 1u : 0u);
            mma_i8(dL, desc(pa + ks * 32, 16, 1024), desc(bl + b * N * 128 + ks * 32, 16, 1024), idesc_i8(false, N),
                   (ks > 0 || b > 0) ? 1u : 0u);
          }
        }
      }
      commit(bar);
      mbar_wait(bar, it & 1);
    }
    cyc[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}


template <int N>
__global__ void __launch_bounds__(128, 1) probe_m64(int32_t* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  unsigned char* P = base;
  unsigned char* BL = P + 16384;
  uint64_t* bar = reinterpret_cast<uint64_t*>(BL + N * 128);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < 128 * 128; e += 128) {
    const int i = e & 127, j = e >> 7;
    P[swz(j, i)] = static_cast<unsigned char>(val(1, i + 128 * j));
  }
  for (int e = tid; e < N * 128; e += 128) {
    const int k = e & 127, r = e >> 7;
    BL[swz(r, k)] = static_cast<unsigned char>(val(3, k + 128 * r));
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;\n" ::"r"(smem_u32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *slot;
  // zero all 128 lanes x 2N columns first
  {
    uint32_t z = 0;
    for (int c = 0; c < 2 * N; ++c)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};\n" ::"r"(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c), "r"(z));
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (tid == 0) {
    const uint32_t p = smem_u32(P), bl = smem_u32(BL);
    for (int ks = 0; ks < 4; ++ks)
      mma_i8(tmem, desc(p + ks * 32, 16, 1024), desc(bl + ks * 32, 16, 1024), idesc_i8_m(false, N, 64), ks > 0);
    // second half rows 64..127 into columns N.. (same lanes as the first)
    for (int ks = 0; ks < 4; ++ks)
      mma_i8(tmem + (16u << 16) + N, desc(p + 8192 + ks * 32, 16, 1024), desc(bl + ks * 32, 16, 1024), idesc_i8_m(false, N, 64), ks > 0);
    commit(bar);
  }
  mbar_wait(bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  for (int c = 0; c < 2 * N; ++c) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(v)
                 : "r"(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    out[tid * 2 * N + c] = static_cast<int32_t>(v);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;\n" ::"r"(tmem));
}
template <int N>
void run_probe() {
  int32_t* d;
  cudaMalloc(&d, 128 * 2 * N * 4);
  const int smem = 16384 + N * 128 + 64 + 1024;
  cudaFuncSetAttribute(probe_m64<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe_m64<N><<<1, 128, smem>>>(d);
  std::vector<int32_t> h(128 * 2 * N);
  cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
  std::printf("M=64 probe N=%d: %s\n", N, cudaGetErrorString(cudaDeviceSynchronize()));
  // expected left value for row j, column r
  auto want = [](int j, int r) {
    int64_t s = 0;
    for (int k = 0; k < 128; ++k) s += static_cast<int64_t>(val(1, k + 128 * j)) * val(3, k + 128 * r);
    return s;
  };
  // for each lane and column block (0: rows 0..63 MMA, 1: rows 64..127 MMA) find the matching row
  for (int blk = 0; blk < 2; ++blk) {
    std::printf(" block %d lanes->rows:", blk);
    for (int lane = 0; lane < 128; ++lane) {
      int found = -1, col_off = -1;
      for (int j = 0; j < 128 && found < 0; ++j)
        for (int c0 = 0; c0 < N && found < 0; c0 += 8)
          if (h[lane * 2 * N + blk * N + c0] == want(j, c0) && want(j, c0) != 0) { found = j; col_off = c0; }
      if (lane % 8 == 0) std::printf(" [%d]", lane);
      std::printf(" %d", found);
    }
    std::printf("\n");
  }
}

template <int N>
int run_check() {
  int32_t *dR, *dL;
  cudaMalloc(&dR, 128 * N * 4);
  cudaMalloc(&dL, 128 * N * 4);
  const int smem = 16384 + 2 * N * 128 + 64 + 1024;
  cudaFuncSetAttribute(check<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  check<N><<<1, 128, smem>>>(dR, dL);
  std::vector<int32_t> hR(128 * N), hL(128 * N);
  cudaMemcpy(hR.data(), dR, hR.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hL.data(), dL, hL.size() * 4, cudaMemcpyDeviceToHost);
  if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
    std::printf("N=%d check: CUDA error %s\n", N, cudaGetErrorString(cudaGetLastError()));
    return 1;
  }
  int badR = 0, badL = 0;
  for (int i = 0; i < 128; ++i)
    for (int r = 0; r < N; ++r) {
      int64_t sR = 0, sL = 0;
      for (int k = 0; k < 128; ++k) {
        sR += static_cast<int64_t>(val(1, i + 128 * k)) * val(2, k + 128 * r);  // i = row of P, j = k
        sL += static_cast<int64_t>(val(1, k + 128 * i)) * val(3, k + 128 * r);  // j = i (row), sum over i = k
      }
      badR += (sR != hR[i * N + r]);
      badL += (sL != hL[i * N + r]);
      if ((sR != hR[i * N + r] || sL != hL[i * N + r]) && badR + badL < 4)
        std::printf("  mismatch i=%d r=%d: R %lld vs %d, L %lld vs %d\n", i, r, (long long)sR, hR[i * N + r],
                    (long long)sL, hL[i * N + r]);
    }
  std::printf("N=%d check: right (MN-major A) %d bad, left (K-major A) %d bad of %d\n", N, badR, badL, 128 * N);
  return badR + badL;
}

template <int N, bool STACK, bool HALF = false>
void run_timing(int sms) {
  const int smem = 6 * 16384 + 12 * N * 128 + 64 + 1024;
  cudaFuncSetAttribute(timing<N, STACK, HALF>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* cyc;
  cudaMalloc(&cyc, sms * 8);
  const int iters = 200;
  timing<N, STACK, HALF><<<sms, 128, smem>>>(10, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  timing<N, STACK, HALF><<<sms, 128, smem>>>(iters, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<unsigned long long> h(sms);
  cudaMemcpy(h.data(), cyc, sms * 8, cudaMemcpyDeviceToHost);
  const double macs_tile = 2.0 * 21 * 128.0 * N * 128;
  std::printf("%s N=%d: %.1f cycles per tile (21 pairs x 2 products, 128x128 tile), %.0f MAC/clk/SM, %.3f us/tile, "
              "%.1f TOPS chip\n", HALF ? "halves " : (STACK ? "stacked" : "pairs  "), N, static_cast<double>(h[0]) / iters, macs_tile * iters / h[0], ms * 1e3 / iters,
              2.0 * macs_tile * iters * sms / (ms * 1e-3) / 1e12);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run_probe<32>();
  int bad = run_check<16>() + run_check<32>();
  run_timing<16, false>(sms);
  run_timing<32, false>(sms);
  run_timing<16, true>(sms);
  run_timing<32, true>(sms);
  run_timing<16, true, true>(sms);
  run_timing<32, true, true>(sms);
  std::printf("status %s\n", bad ? "MISMATCH" : "ok");
  return 0;
}
