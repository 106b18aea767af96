// common.cuh — shared device-side types for the B200 all-mode CP gradient.
//
// The index vocabulary follows the reference (SURVEY.md shorthand): Y is the
// dense column-major tensor in the ascending-sorted mode frame, p the pivot,
// J_n / K_n the prefix / suffix products, the right seed J_p x R and the left
// seed K_p x R (mttkrp.cpp:149-210).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace cpdgpu {

constexpr int kMaxModes = 16;  // modes per Khatri-Rao range

// Programmatic dependent launch: a kernel launched with the programmatic
// stream-serialization attribute may start while its predecessor runs; it must
// pdl_wait() before touching anything the predecessor writes.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// Launch timeline (diagnostics only; compiled in with -DCPDGPU_TIMELINE, enabled
// at run time by CPDGPU_TIMELINE=1): per launch slot, the earliest CTA entry,
// the earliest return from the dependency wait and the last warp exit, in
// globaltimer nanoseconds.  Compiled out by default: even the null-pointer
// checks measurably delayed the small latency-bound kernels (c1: +2 us/step).
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
  return v;
}
#ifndef CPDGPU_TIMELINE
__device__ __forceinline__ void tl_begin(unsigned long long*, int) {}
__device__ __forceinline__ void tl_mid(unsigned long long*, int) {}
__device__ __forceinline__ void tl_end(unsigned long long*, int) {}
#else
__device__ __forceinline__ void tl_begin(unsigned long long* tl, int slot) {
  if (tl && threadIdx.x == 0) atomicMin(tl + 3 * slot, gtimer());
}
__device__ __forceinline__ void tl_mid(unsigned long long* tl, int slot) {
  if (tl && threadIdx.x == 0) atomicMin(tl + 3 * slot + 1, gtimer());
}
__device__ __forceinline__ void tl_end(unsigned long long* tl, int slot) {
  if (tl && (threadIdx.x & 31) == 0) atomicMax(tl + 3 * slot + 2, gtimer());
}
#endif

// Host: launch with (pdl = true) or without the programmatic attribute.
template <typename... Exp, typename... Act>
inline cudaError_t launch_k(void (*kernel)(Exp...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl,
                            Act&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<Act&&>(args)...);
}
bool pdl_enabled();  // CPDGPU_PDL=0 disables (default on)

// Dynamic shared memory above 48 KB: cudaFuncSetAttribute applies to the current
// device only, so it is set once per (kernel, device); `mask` is the caller's
// per-kernel record of the devices done.
template <typename K>
inline void set_smem_attr(K kernel, int bytes, unsigned long long& mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = dev < 64 ? (1ull << dev) : 0ull;
  if (bit && (mask & bit)) return;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  mask |= bit;
}

// A contiguous range of modes lo..hi of the sorted frame whose factor columns
// form a Khatri-Rao row on the fly: row index q has mixed-radix digits
// d_k (first mode fastest) and  KR[q, r] = prod_k A_k[d_k + I_k r]
// (kron_range_column, kron.cpp:54-68: later modes outermost).
struct KRSpec {
  int n;                           // number of modes in the range (0 => KR == 1)
  int64_t dims[kMaxModes];         // I_k
  const double* A[kMaxModes];      // device factor k, column-major I_k x R
};

__device__ __forceinline__ double kr_entry(const KRSpec& s, int64_t q, int r) {
  double prod = 1.0;
#pragma unroll 1
  for (int k = 0; k < s.n; ++k) {
    const int64_t I = s.dims[k];
    const int64_t d = q % I;
    q /= I;
    prod *= __ldg(s.A[k] + d + I * r);
  }
  return prod;
}

// 32-bit fast path when every intermediate fits (the common case).
__device__ __forceinline__ double kr_entry32(const KRSpec& s, uint32_t q, int r) {
  double prod = 1.0;
#pragma unroll 1
  for (int k = 0; k < s.n; ++k) {
    const uint32_t I = static_cast<uint32_t>(s.dims[k]);
    const uint32_t d = q % I;
    q /= I;
    prod *= __ldg(s.A[k] + d + static_cast<int64_t>(I) * r);
  }
  return prod;
}


__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace cpdgpu
