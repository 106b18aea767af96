// kernels.h — host-visible launch interface of the device kernels.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace cpdgpu {

// ---- K1: fp64 seed contraction (seed_f64.cu) --------------------------------
struct SeedParams {
  const double* Y;  // sorted-frame tensor viewed as J x K column-major (ld J)
  int64_t J, K;     // J_p, K_p
  int R;            // rank handled by this launch (<= 8 * NT)
  int TI;           // rows per row block (multiple of 8, <= 256)
  int LDY, LDK;     // shared-memory leading dimensions (bank-conflict-free)
  int64_t nRB, nCT; // row blocks, 32-column tiles
  int64_t T;        // nRB * nCT
  int P;            // CTAs (persistent)
  int slots;        // right-partial slots per CTA
  int use32;        // all KR row indices fit in 32 bits
  KRSpec left;      // modes 1..p   (rows of the view)
  KRSpec right;     // modes p+1..N (columns of the view)
  double* Rpart;    // [P * slots][R8][TI]
  double* Lpart;    // [nRB][R][K]
};
int seed_f64_stages(int NT);
size_t seed_f64_smem_bytes(int NT, int TI, int LDY, int LDK, int mode);
int launch_seed_f64(const SeedParams& p, int NT, int mode, cudaStream_t s);

// ---- reductions of the seed partials (tail.cu) ------------------------------
// Rs[r * ldo + i] = sum over the (CTA, row block) slots covering row i.
int launch_reduce_right(const SeedParams& p, int RP, double* Rs, int64_t ldo, cudaStream_t s);
// Ls[r * ldo + j] = sum_rb Lpart[rb][r][j]
int launch_reduce_left(const double* Lpart, int64_t nRB, int R, int64_t K, double* Ls,
                        int64_t ldo, cudaStream_t s);

// ---- K2: rank-batched TTV contractions of the recursion tail (tail.cu) -------
// out[r*ldo + b] = sum_{a<M} Z[r*ldz + a + M*b] * KR_v[a, r]      (Eq 3.12 / 3.22)
int launch_contract_a(const double* Z, int64_t ldz, int64_t M, int64_t B, int R,
                       const KRSpec& v, double* out, int64_t ldo, cudaStream_t s);
// out[r*ldo + a] = sum_{b<B} Z[r*ldz + a + M*b] * KR_w[b, r]      (Eq 3.20 / 3.16)
// part: scratch of at least contract_b_scratch(M, B, R) doubles.
size_t contract_b_scratch(int64_t M, int64_t B, int R, int num_sms);
int launch_contract_b(const double* Z, int64_t ldz, int64_t M, int64_t B, int R,
                       const KRSpec& w, double* out, int64_t ldo, double* part, int num_sms,
                       cudaStream_t s);

// ---- utilities (util.cu) -----------------------------------------------------
// packed factor gather: dst block j <- src block perm[j]-1 (sorted frame)
int launch_gather_blocks(const double* src, double* dst, int N, const int64_t* src_off,
                          const int64_t* dst_off, const int64_t* len, cudaStream_t s);
// out (sorted frame) <- permute(in, perm) (tensor_ops.cpp:39-71), dtype size 4 or 8
int launch_permute(const void* in, void* out, int elem_bytes, int N, const int64_t* dims,
                    const int* perm, cudaStream_t s);
int launch_generate(void* out, int elem_bytes, int64_t n, int dist, uint64_t seed,
                     int64_t offset, cudaStream_t s);
// Y <- alpha Y + beta full(model), fp64 or fp32 storage
int launch_axpby_kruskal(void* Y, int elem_bytes, int N, const int64_t* dims, const KRSpec& all,
                          int R, double alpha, double beta, cudaStream_t s);
// partial sums of squares -> out[0] (two-stage, deterministic)
int launch_norm2(const void* Y, int elem_bytes, int64_t n, double* scratch, double* out,
                  cudaStream_t s);

// ---- ALS (als.cu) -------------------------------------------------------------
// gram[a + R c] = sum_i A[i + I a] A[i + I c]
int launch_gram(const double* A, int64_t I, int R, double* gram, cudaStream_t s);
// A_n <- G * pinv_psd(hadamard_{k != n} grams[k], rtol); gram_n <- A_n^T A_n.
// status[0] set to 4 (NumericError) when G holds a non-finite value.
int launch_als_update(const double* G, int64_t I, int R, const double* grams, int N, int n,
                       double rtol, double* A, double* gram_n, int* status, cudaStream_t s);
// standalone pinv_psd of a device R x R matrix
int launch_pinv_psd(const double* S, int R, double rtol, double* out, cudaStream_t s);
// cost = ynorm2 - 2 sum(A_L .* G_L) + 1^T (hadamard of all grams) 1, clamped at 0
int launch_als_cost(const double* A, const double* G, int64_t I, int R, const double* grams,
                     int N, const double* ynorm2, double* cost_out, cudaStream_t s);

}  // namespace cpdgpu
