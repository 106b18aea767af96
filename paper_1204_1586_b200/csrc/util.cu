// util.cu — data-movement helpers: factor gather, mode permutation
// (sort_modes/permute, mttkrp.cpp:67-90 / tensor_ops.cpp:39-71), the
// counter-based synthetic generator, model materialisation (full,
// kruskal.cpp:23-31) and the squared Frobenius norm (dense_tensor.cpp:32-34).
#include "kernels.h"

namespace cpdgpu {
namespace {

struct GatherArgs {
  int N;
  int64_t src_off[kMaxModes], dst_off[kMaxModes], len[kMaxModes];
};

__global__ void gather_blocks_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                     const GatherArgs a) {
  for (int j = 0; j < a.N; ++j)
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < a.len[j];
         e += static_cast<int64_t>(gridDim.x) * blockDim.x)
      dst[a.dst_off[j] + e] = src[a.src_off[j] + e];
}

struct PermArgs {
  int N;
  int64_t od[kMaxModes];       // output dims
  int64_t sstride[kMaxModes];  // source stride of output axis k
  int64_t total;
};

template <typename T>
__global__ void permute_kernel(const T* __restrict__ in, T* __restrict__ out, const PermArgs a) {
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < a.total;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t rem = q, src = 0;
    for (int k = 0; k < a.N; ++k) {
      const int64_t d = rem % a.od[k];
      rem /= a.od[k];
      src += d * a.sstride[k];
    }
    out[q] = in[src];
  }
}

__device__ __forceinline__ uint64_t hash64(uint64_t seed, uint64_t idx) {
  uint64_t x = seed * 0xD1B54A32D192ED03ull + idx * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

template <typename T>
__global__ void generate_kernel(T* __restrict__ out, int64_t n, int dist, uint64_t seed,
                                int64_t offset) {
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t i = static_cast<uint64_t>(offset + q);
    double v;
    if (dist == 0) {
      const double u1 = (static_cast<double>(hash64(seed, 2 * i) >> 11) + 0.5) * 0x1.0p-53;
      const double u2 = static_cast<double>(hash64(seed, 2 * i + 1) >> 11) * 0x1.0p-53;
      v = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
    } else {
      const uint64_t h = hash64(seed, i);
      v = static_cast<double>(static_cast<int32_t>(h >> 40) - 8388608) * 0x1.0p-23;
    }
    out[q] = static_cast<T>(v);
  }
}

template <typename T>
__global__ void axpby_kruskal_kernel(T* __restrict__ Y, const KRSpec s, int R, double alpha,
                                     double beta, int64_t total) {
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < total;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t d[kMaxModes];
    int64_t rem = q;
    for (int k = 0; k < s.n; ++k) {
      d[k] = rem % s.dims[k];
      rem /= s.dims[k];
    }
    double acc = 0.0;
    for (int r = 0; r < R; ++r) {
      double prod = 1.0;
      for (int k = 0; k < s.n; ++k) prod *= __ldg(s.A[k] + d[k] + s.dims[k] * r);
      acc += prod;
    }
    const double y = static_cast<double>(Y[q]);
    Y[q] = static_cast<T>(alpha * y + beta * acc);
  }
}

constexpr int kNormBlocks = 1184;  // 8 per SM

template <typename T>
__global__ void norm2_partial(const T* __restrict__ Y, int64_t n, double* __restrict__ part) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double v = static_cast<double>(Y[q]);
    s += v * v;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void norm2_final(const double* __restrict__ part, int nb, double* out) {
  __shared__ double red[256];
  double s = 0.0;
  for (int q = threadIdx.x; q < nb; q += blockDim.x) s += part[q];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0];
}

int grid_for(int64_t work, int threads, int cap = 148 * 32) {
  const int64_t b = (work + threads - 1) / threads;
  return static_cast<int>(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace

int launch_gather_blocks(const double* src, double* dst, int N, const int64_t* src_off,
                          const int64_t* dst_off, const int64_t* len, cudaStream_t s) {
  GatherArgs a;
  a.N = N;
  int64_t mx = 1;
  for (int j = 0; j < N; ++j) {
    a.src_off[j] = src_off[j];
    a.dst_off[j] = dst_off[j];
    a.len[j] = len[j];
    mx = len[j] > mx ? len[j] : mx;
  }
  gather_blocks_kernel<<<grid_for(mx, 256), 256, 0, s>>>(src, dst, a);
  return 1;
}

int launch_permute(const void* in, void* out, int elem_bytes, int N, const int64_t* dims,
                    const int* perm, cudaStream_t s) {
  PermArgs a;
  a.N = N;
  int64_t J[kMaxModes + 1];
  J[0] = 1;
  for (int k = 0; k < N; ++k) J[k + 1] = J[k] * dims[k];
  a.total = J[N];
  for (int k = 0; k < N; ++k) {
    a.od[k] = dims[perm[k] - 1];
    a.sstride[k] = J[perm[k] - 1];
  }
  if (elem_bytes == 8)
    permute_kernel<double><<<grid_for(a.total, 256), 256, 0, s>>>(
        static_cast<const double*>(in), static_cast<double*>(out), a);
  else
    permute_kernel<float><<<grid_for(a.total, 256), 256, 0, s>>>(
        static_cast<const float*>(in), static_cast<float*>(out), a);
  return 1;
}

int launch_generate(void* out, int elem_bytes, int64_t n, int dist, uint64_t seed,
                     int64_t offset, cudaStream_t s) {
  if (elem_bytes == 8)
    generate_kernel<double><<<grid_for(n, 256), 256, 0, s>>>(static_cast<double*>(out), n, dist,
                                                             seed, offset);
  else
    generate_kernel<float><<<grid_for(n, 256), 256, 0, s>>>(static_cast<float*>(out), n, dist,
                                                            seed, offset);
  return 1;
}

int launch_axpby_kruskal(void* Y, int elem_bytes, int N, const int64_t* dims, const KRSpec& all,
                          int R, double alpha, double beta, cudaStream_t s) {
  int64_t total = 1;
  for (int k = 0; k < N; ++k) total *= dims[k];
  if (elem_bytes == 8)
    axpby_kruskal_kernel<double><<<grid_for(total, 256), 256, 0, s>>>(static_cast<double*>(Y),
                                                                      all, R, alpha, beta, total);
  else
    axpby_kruskal_kernel<float><<<grid_for(total, 256), 256, 0, s>>>(static_cast<float*>(Y), all,
                                                                     R, alpha, beta, total);
  return 1;
}

int launch_norm2(const void* Y, int elem_bytes, int64_t n, double* scratch, double* out,
                  cudaStream_t s) {
  if (elem_bytes == 8)
    norm2_partial<double><<<kNormBlocks, 256, 0, s>>>(static_cast<const double*>(Y), n, scratch);
  else
    norm2_partial<float><<<kNormBlocks, 256, 0, s>>>(static_cast<const float*>(Y), n, scratch);
  norm2_final<<<1, 256, 0, s>>>(scratch, kNormBlocks, out);
  return 2;
}

}  // namespace cpdgpu
