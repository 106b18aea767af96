// als.cu — the R x R part of the fast CP_ALS update on the device.
//
// Reference: gram_hadamard_skip (kron.cpp:124-134), pinv_psd (als.cpp:34-47),
// als_update_mode (als.cpp:49-56) and the Gram identity of cost()
// (kruskal.cpp:58-77).  Differences from the reference, all value-preserving:
//  * the per-factor Grams A_k^T A_k are cached on the device and only the
//    updated mode's Gram is recomputed (the reference recomputes all N-1);
//  * the symmetric eigendecomposition is a parallel cyclic Jacobi in fp64
//    shared memory (round-robin pairing, R/2 disjoint rotations per step)
//    instead of Eigen's tridiagonal QR; the pseudo-inverse keeps the
//    reference's cutoff rule (lambda <= rtol*max|lambda| or lambda <= 0 -> 0);
//  * inside the ALS update a Cholesky inverse replaces the eigensolve when the
//    matrix is certified positive definite with no eigenvalue near the cutoff
//    (then pinv_psd(W) = W^{-1}); anything else takes the Jacobi route;
//  * <Y, Yhat> comes from sum(A_L .* G_L) of the last updated mode L (exact:
//    G_L was computed from the final factors of every other mode), so the fit
//    needs no extra pass over Y.
#include "kernels.h"

namespace cpdgpu {
namespace {

constexpr int kAlsThreads = 256;
constexpr int64_t kAlsStage = 4096;  // I x R doubles of G (and of A) staged in shared memory

__global__ void gram_kernel(const double* __restrict__ A, int64_t I, int R,
                            double* __restrict__ gram) {
  for (int e = threadIdx.x + blockIdx.x * blockDim.x; e < R * R; e += blockDim.x * gridDim.x) {
    const int a = e % R, c = e / R;
    if (a > c) continue;
    double s = 0.0;
    for (int64_t i = 0; i < I; ++i) s += A[i + I * a] * A[i + I * c];
    gram[a + R * c] = s;
    gram[c + R * a] = s;
  }
}

// Parallel cyclic Jacobi on the Rp x Rp (Rp even) matrix in M; V receives the
// eigenvectors (columns).  A pair is rotated while |a_pq| is above both the
// relative-accuracy level eps sqrt(|a_pp a_qq|) and the rounding floor of the
// matrix, eps max_k |a_kk| (backward-stable accuracy, as a QR-based solver);
// below the floor a rotation only shuffles rounding noise and the sweep loop
// would never see a rotation-free sweep.  The loop stops after such a sweep.
// M2 / V2 are ping-pong buffers; the eigenvalues are left on the diagonal of M.
__device__ void jacobi_eig(double* M, double* M2, double* V, double* V2, double* cs, int* partner,
                           int Rp) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int RR = Rp * Rp;
  for (int e = tid; e < RR; e += nt) V[e] = (e % Rp == e / Rp) ? 1.0 : 0.0;
  __shared__ int s_rot;
  __shared__ double s_floor;
  if (tid == 0) {
    double mx = 0.0;
    for (int x = 0; x < Rp; ++x) mx = fmax(mx, fabs(M[x + Rp * x]));
    s_floor = 2.2e-16 * mx;  // trace-scale rounding floor (diagonal max of a PSD matrix)
  }
  __syncthreads();
  const double floor_abs = s_floor;
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (tid == 0) s_rot = 0;
    __syncthreads();
    for (int step = 0; step < Rp - 1; ++step) {
      // round-robin pairs: L[0] = 0, L[k] = (k - 1 + step) % (Rp - 1) + 1
      for (int i = tid; i < Rp / 2; i += nt) {
        const int a = (i == 0) ? 0 : ((i - 1 + step) % (Rp - 1)) + 1;
        const int k = Rp - 1 - i;
        const int b = ((k - 1 + step) % (Rp - 1)) + 1;
        const int p = a < b ? a : b, q = a < b ? b : a;
        const double apq = M[p + Rp * q];
        const double app = M[p + Rp * p], aqq = M[q + Rp * q];
        double c = 1.0, s = 0.0;
        if (apq != 0.0 && fabs(apq) > 1e-16 * sqrt(fabs(app * aqq)) && fabs(apq) > floor_abs) {
          const double theta = (aqq - app) / (2.0 * apq);
          const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
          c = 1.0 / sqrt(t * t + 1.0);
          s = t * c;
          s_rot = 1;
        }
        partner[p] = q;
        partner[q] = p;
        cs[2 * p] = c;       // J[p][p]
        cs[2 * p + 1] = -s;  // J[q][p]
        cs[2 * q] = c;       // J[q][q]
        cs[2 * q + 1] = s;   // J[p][q]
      }
      __syncthreads();
      for (int e = tid; e < RR; e += nt) {
        const int x = e % Rp, y = e / Rp;
        const int px = partner[x], py = partner[y];
        const double cx = cs[2 * x], ox = cs[2 * x + 1], cy = cs[2 * y], oy = cs[2 * y + 1];
        double v = cx * cy * M[x + Rp * y] + cx * oy * M[x + Rp * py] +
                   ox * cy * M[px + Rp * y] + ox * oy * M[px + Rp * py];
        if (y == px) v = 0.0;  // the annihilated pair
        M2[e] = v;
        V2[e] = V[x + Rp * y] * cy + V[x + Rp * py] * oy;
      }
      __syncthreads();
      for (int e = tid; e < RR; e += nt) {
        M[e] = M2[e];
        V[e] = V2[e];
      }
      __syncthreads();
    }
    if (!s_rot) break;
    __syncthreads();
  }
}

// P = V diag(inv) V^T with the pinv_psd cutoff rule; writes P (R x R, ld R).
__device__ void pinv_from_eig(const double* M, const double* V, double* inv, int R, int Rp,
                              double rtol, double* P) {
  const int tid = threadIdx.x, nt = blockDim.x;
  __shared__ double s_max;
  if (tid == 0) {
    double mx = 0.0;
    for (int x = 0; x < R; ++x) mx = fmax(mx, fabs(M[x + Rp * x]));
    s_max = mx;
  }
  __syncthreads();
  const double cutoff = rtol * s_max;
  for (int x = tid; x < R; x += nt) {
    const double ev = M[x + Rp * x];
    inv[x] = (ev > cutoff && ev > 0.0) ? 1.0 / ev : 0.0;
  }
  __syncthreads();
  for (int e = tid; e < R * R; e += nt) {
    const int a = e % R, c = e / R;
    double acc = 0.0;
    for (int x = 0; x < R; ++x) acc += V[a + Rp * x] * inv[x] * V[c + Rp * x];
    P[a + R * c] = acc;
  }
  __syncthreads();
}

// Fast path of pinv_psd for a certified well-conditioned PD matrix: X = W^{-1}
// by Gauss-Jordan elimination without pivoting (stable for symmetric positive
// definite W, the pivots are its Schur complements), all R x R entries updated
// in parallel per pivot step (R steps; the former Cholesky + per-column
// triangular solves ran R^2 dependent steps on R threads).  Accepted only when
// every pivot was positive and lambda_min >= 1 / ||X||_inf exceeds
// 10 rtol ||W||_inf >= 10 rtol lambda_max: then no eigenvalue reaches the
// pinv_psd cutoff and the pseudo-inverse IS the inverse.  Otherwise the caller
// runs the Jacobi eigensolver.  X and its ping-pong partner use the M2 / V2
// scratch (ld Rp).
__device__ bool chol_inverse(const double* W, double* X, double* X2, int R, int Rp, double rtol, double* P) {
  const int tid = threadIdx.x, nt = blockDim.x;
  __shared__ int s_fail;
  __shared__ double s_wn, s_xn;
  if (tid == 0) {
    s_fail = 0;
    s_wn = 0.0;
    s_xn = 0.0;
  }
  for (int e = tid; e < Rp * Rp; e += nt) X[e] = W[e];
  __syncthreads();
  double* cur = X;
  double* nxt = X2;
  for (int k = 0; k < R; ++k) {
    const double piv = cur[k + Rp * k];
    if (!(piv > 0.0)) {  // uniform: every thread reads the same pivot
      if (tid == 0) s_fail = 1;
      break;
    }
    const double ip = 1.0 / piv;
    for (int e = tid; e < R * R; e += nt) {
      const int i = e % R, j = e / R;
      double v;
      if (i == k && j == k)
        v = ip;
      else if (i == k)
        v = cur[k + Rp * j] * ip;
      else if (j == k)
        v = -cur[i + Rp * k] * ip;
      else
        v = cur[i + Rp * j] - cur[i + Rp * k] * cur[k + Rp * j] * ip;
      nxt[i + Rp * j] = v;
    }
    __syncthreads();
    double* t = cur;
    cur = nxt;
    nxt = t;
  }
  __syncthreads();
  if (s_fail) return false;
  for (int a = tid; a < R; a += nt) {  // infinity norms (row sums)
    double w = 0.0, x = 0.0;
    for (int c = 0; c < R; ++c) {
      w += fabs(W[a + Rp * c]);
      x += fabs(cur[a + Rp * c]);
    }
    atomicMax(reinterpret_cast<unsigned long long*>(&s_wn), __double_as_longlong(w));
    atomicMax(reinterpret_cast<unsigned long long*>(&s_xn), __double_as_longlong(x));
  }
  __syncthreads();
  const bool ok = s_xn > 0.0 && (1.0 / s_xn) > 10.0 * rtol * s_wn;
  if (ok)
    for (int e = tid; e < R * R; e += nt) {
      const int a = e % R, c = e / R;
      P[a + R * c] = 0.5 * (cur[a + Rp * c] + cur[c + Rp * a]);
    }
  __syncthreads();
  return ok;
}
struct EigSmem {
  double *M, *M2, *V, *V2, *cs, *inv, *P;
  int* partner;
};

__device__ EigSmem carve(double* smem, int R, int Rp) {
  EigSmem e;
  const int RR = Rp * Rp;
  e.M = smem;
  e.M2 = e.M + RR;
  e.V = e.M2 + RR;
  e.V2 = e.V + RR;
  e.P = e.V2 + RR;
  e.cs = e.P + R * R;
  e.inv = e.cs + 2 * Rp;
  e.partner = reinterpret_cast<int*>(e.inv + Rp);
  return e;
}

size_t eig_smem_bytes(int R) {
  const int Rp = R + (R & 1);
  return (4 * static_cast<size_t>(Rp) * Rp + static_cast<size_t>(R) * R + 3 * Rp) * sizeof(double) +
         Rp * sizeof(int) + 64;
}

__global__ void __launch_bounds__(kAlsThreads, 1)
    als_update_kernel(const double* __restrict__ G, int64_t I, int R,
                      const double* __restrict__ grams, int N, int n, double rtol,
                      double* __restrict__ A, double* __restrict__ gram_n, int* status) {
  extern __shared__ double smem[];
  const int Rp = R + (R & 1);
  EigSmem s = carve(smem, R, Rp);
  const int tid = threadIdx.x, nt = blockDim.x;
  // non-finite check (als.cpp:53-54)
  int bad = 0;
  for (int64_t e = tid; e < I * R; e += nt) bad |= !isfinite(G[e]);
  if (__syncthreads_or(bad)) {
    if (tid == 0) status[0] = 4;
    return;
  }
  // W = hadamard_{k != n} gram_k  (kron.cpp:124-134), zero-padded to Rp
  for (int e = tid; e < Rp * Rp; e += nt) {
    const int a = e % Rp, c = e / Rp;
    double w = 0.0;
    if (a < R && c < R) {
      w = 1.0;
      for (int k = 0; k < N; ++k)
        if (k != n) w *= grams[static_cast<int64_t>(k) * R * R + a + R * c];
    }
    s.M[e] = w;
  }
  __syncthreads();
  if (!chol_inverse(s.M, s.M2, s.V2, R, Rp, rtol, s.P)) {
    jacobi_eig(s.M, s.M2, s.V, s.V2, s.cs, s.partner, Rp);
    pinv_from_eig(s.M, s.V, s.inv, R, Rp, rtol, s.P);
  }
  // A_n = G * P  (als.cpp:55); G staged in shared memory (after the eigen scratch)
  // when it fits, so the products and the new Gram read shared memory
  double* gs = s.partner ? reinterpret_cast<double*>(s.partner + Rp) : nullptr;
  gs = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(gs) + 15) & ~static_cast<uintptr_t>(15));
  const bool staged = I * R <= kAlsStage;
  if (staged) {
    double* as = gs + I * R;
    for (int64_t e = tid; e < I * R; e += nt) gs[e] = G[e];
    __syncthreads();
    for (int64_t e = tid; e < I * R; e += nt) {
      const int64_t i = e % I;
      const int c = static_cast<int>(e / I);
      double acc = 0.0;
      for (int k = 0; k < R; ++k) acc += gs[i + I * k] * s.P[k + R * c];
      as[e] = acc;
      A[e] = acc;
    }
    __syncthreads();
    for (int e = tid; e < R * R; e += nt) {
      const int a = e % R, c = e / R;
      double acc = 0.0;
      for (int64_t i = 0; i < I; ++i) acc += as[i + I * a] * as[i + I * c];
      gram_n[e] = acc;
    }
    return;
  }
  for (int64_t e = tid; e < I * R; e += nt) {
    const int64_t i = e % I;
    const int c = static_cast<int>(e / I);
    double acc = 0.0;
    for (int k = 0; k < R; ++k) acc += G[i + I * k] * s.P[k + R * c];
    A[e] = acc;
  }
  __threadfence_block();
  __syncthreads();
  for (int e = tid; e < R * R; e += nt) {
    const int a = e % R, c = e / R;
    double acc = 0.0;
    for (int64_t i = 0; i < I; ++i) acc += A[i + I * a] * A[i + I * c];
    gram_n[e] = acc;
  }
}

// mu_sweep's update (als.cpp:84-90): A <- A .* G ./ (A W + eps), W = hadamard of the
// other modes' Grams (current factors); then gram_n <- A^T A.  A thread owns whole
// rows (in-place safe: row i of the new A needs only row i of the old one).
__global__ void __launch_bounds__(kAlsThreads, 1)
    mu_update_kernel(const double* __restrict__ G, int64_t I, int R, const double* __restrict__ grams, int N, int n,
                     double eps, double* __restrict__ A, double* __restrict__ gram_n) {
  extern __shared__ double W[];  // R x R
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < R * R; e += nt) {
    double w = 1.0;
    for (int k = 0; k < N; ++k)
      if (k != n) w *= grams[static_cast<int64_t>(k) * R * R + e];
    W[e] = w;
  }
  __syncthreads();
  for (int64_t i = tid; i < I; i += nt) {
    double row[64];
    for (int k = 0; k < R; ++k) row[k] = A[i + I * k];
    for (int c = 0; c < R; ++c) {
      double den = 0.0;
      for (int k = 0; k < R; ++k) den += row[k] * W[k + R * c];
      A[i + I * c] = row[c] * G[i + I * c] / (den + eps);
    }
  }
  __threadfence_block();
  __syncthreads();
  for (int e = tid; e < R * R; e += nt) {
    const int a = e % R, c = e / R;
    double acc = 0.0;
    for (int64_t i = 0; i < I; ++i) acc += A[i + I * a] * A[i + I * c];
    gram_n[e] = acc;
  }
}

// gd_step's update for one mode (als.cpp:93-101): A += 2 eta (G - A W) with W from
// the pre-step Grams (the caller recomputes every Gram after all modes).
__global__ void gd_update_kernel(const double* __restrict__ G, int64_t I, int R, const double* __restrict__ grams,
                                 int N, int n, double eta, double* __restrict__ A) {
  extern __shared__ double W[];
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    double w = 1.0;
    for (int k = 0; k < N; ++k)
      if (k != n) w *= grams[static_cast<int64_t>(k) * R * R + e];
    W[e] = w;
  }
  __syncthreads();
  // each thread owns rows i (all R columns), so the in-place update reads its own old row
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < I;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double row[64];
    for (int k = 0; k < R; ++k) row[k] = A[i + I * k];
    for (int c = 0; c < R; ++c) {
      double aw = 0.0;
      for (int k = 0; k < R; ++k) aw += row[k] * W[k + R * c];
      A[i + I * c] = row[c] + 2.0 * eta * (G[i + I * c] - aw);
    }
  }
}

// status[0] <- 5 (DomainError) when any entry is negative (mu_sweep's check_nonnegative).
template <typename T>
__global__ void nonneg_kernel(const T* __restrict__ y, int64_t n, int* status) {
  int bad = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    bad |= y[i] < T(0);
  if (__syncthreads_or(bad) && threadIdx.x == 0) status[0] = 5;
}

__global__ void __launch_bounds__(kAlsThreads, 1)
    pinv_kernel(const double* __restrict__ S, int R, double rtol, double* __restrict__ out) {
  extern __shared__ double smem[];
  const int Rp = R + (R & 1);
  EigSmem s = carve(smem, R, Rp);
  for (int e = threadIdx.x; e < Rp * Rp; e += blockDim.x) {
    const int a = e % Rp, c = e / Rp;
    s.M[e] = (a < R && c < R) ? S[a + R * c] : 0.0;
  }
  __syncthreads();
  jacobi_eig(s.M, s.M2, s.V, s.V2, s.cs, s.partner, Rp);
  pinv_from_eig(s.M, s.V, s.inv, R, Rp, rtol, s.P);
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) out[e] = s.P[e];
}

__global__ void als_cost_kernel(const double* __restrict__ A, const double* __restrict__ G,
                                int64_t I, int R, const double* __restrict__ grams, int N,
                                const double* ynorm2, double* cost_out) {
  __shared__ double red[kAlsThreads];
  __shared__ double red2[kAlsThreads];
  double inner = 0.0, gs = 0.0;
  for (int64_t e = threadIdx.x; e < I * R; e += blockDim.x) inner += A[e] * G[e];
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    double w = 1.0;
    for (int k = 0; k < N; ++k) w *= grams[static_cast<int64_t>(k) * R * R + e];
    gs += w;
  }
  red[threadIdx.x] = inner;
  red2[threadIdx.x] = gs;
  __syncthreads();
  for (int o = kAlsThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      red[threadIdx.x] += red[threadIdx.x + o];
      red2[threadIdx.x] += red2[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double d = ynorm2[0] - 2.0 * red[0] + red2[0];
    cost_out[0] = d < 0.0 ? 0.0 : d;  // kruskal.cpp:76
  }
}

// Opt-in dynamic shared memory, once per (kernel, size): never inside a graph capture.
void set_smem(const void* fn, size_t bytes) {
  static const void* done_fn[8] = {nullptr};
  static size_t done_bytes[8] = {0};
  if (bytes <= 48 * 1024) return;
  for (int i = 0; i < 8; ++i)
    if (done_fn[i] == fn && done_bytes[i] >= bytes) return;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
  for (int i = 0; i < 8; ++i)
    if (done_fn[i] == fn || done_fn[i] == nullptr) {
      done_fn[i] = fn;
      done_bytes[i] = bytes;
      return;
    }
}

}  // namespace

int launch_gram(const double* A, int64_t I, int R, double* gram, cudaStream_t s) {
  gram_kernel<<<1, kAlsThreads, 0, s>>>(A, I, R, gram);
  return 1;
}

int launch_als_update(const double* G, int64_t I, int R, const double* grams, int N, int n,
                       double rtol, double* A, double* gram_n, int* status, cudaStream_t s) {
  const size_t bytes = eig_smem_bytes(R) + 16 + (I * R <= kAlsStage ? 2 * static_cast<size_t>(I) * R * sizeof(double) : 0);
  set_smem(reinterpret_cast<const void*>(als_update_kernel), bytes);
  als_update_kernel<<<1, kAlsThreads, bytes, s>>>(G, I, R, grams, N, n, rtol, A, gram_n, status);
  return 1;
}

int launch_mu_update(const double* G, int64_t I, int R, const double* grams, int N, int n, double eps, double* A,
                     double* gram_n, cudaStream_t s) {
  const size_t bytes = static_cast<size_t>(R) * R * sizeof(double);
  mu_update_kernel<<<1, kAlsThreads, bytes, s>>>(G, I, R, grams, N, n, eps, A, gram_n);
  return 1;
}

int launch_gd_update(const double* G, int64_t I, int R, const double* grams, int N, int n, double eta, double* A,
                     cudaStream_t s) {
  const int blocks = static_cast<int>(I / 128 + 1 < 148 ? I / 128 + 1 : 148);
  gd_update_kernel<<<blocks, 128, static_cast<size_t>(R) * R * sizeof(double), s>>>(G, I, R, grams, N, n, eta, A);
  return 1;
}

int launch_nonneg_check(const void* y, int elem_bytes, int64_t n, int* status, cudaStream_t s) {
  if (elem_bytes == 8)
    nonneg_kernel<double><<<148 * 4, 256, 0, s>>>(static_cast<const double*>(y), n, status);
  else
    nonneg_kernel<float><<<148 * 4, 256, 0, s>>>(static_cast<const float*>(y), n, status);
  return 1;
}

int launch_pinv_psd(const double* S, int R, double rtol, double* out, cudaStream_t s) {
  const size_t bytes = eig_smem_bytes(R);
  set_smem(reinterpret_cast<const void*>(pinv_kernel), bytes);
  pinv_kernel<<<1, kAlsThreads, bytes, s>>>(S, R, rtol, out);
  return 1;
}

int launch_als_cost(const double* A, const double* G, int64_t I, int R, const double* grams,
                     int N, const double* ynorm2, double* cost_out, cudaStream_t s) {
  als_cost_kernel<<<1, kAlsThreads, 0, s>>>(A, G, I, R, grams, N, ynorm2, cost_out);
  return 1;
}

}  // namespace cpdgpu
