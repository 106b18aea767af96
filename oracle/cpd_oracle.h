/* cpd_oracle.h — CPU restatement of the reference's all-mode CP gradient and
 * fast CP_ALS (arXiv 1204.1586; /root/reference/proj/core/src/{mttkrp,kron,als,
 * kruskal,shape,tensor_ops}.cpp).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library, and only as the
 * checker or the CPU baseline.  The product path (paper_1204_1586_b200/) never
 * links, imports or calls it.
 *
 * Conventions follow the reference: every tensor is column-major (first index
 * fastest, dense_tensor.hpp:12-14); factor n is I_n x R column-major
 * (kron.hpp:13-14); modes are 1-based in the public arguments; results come
 * back in the caller's (original) mode order (mttkrp.cpp:134-136).
 *
 * Status codes are the C-ABI's (include/cpdgpu.h): 0 ok, 1 ShapeError,
 * 2 IndexError, 3 ArgumentError, 4 NumericError.
 */
#ifndef CPD_ORACLE_H
#define CPD_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef int64_t ora_index;

/* hook(user, original 1-based mode, G (rows x R), rows, R); may overwrite the
 * caller's factor for that mode, which the sweep re-reads (mttkrp.cpp:137-144). */
typedef void (*ora_hook_fn)(void* user, int mode, const double* g, ora_index rows, ora_index R);

int ora_select_pivot(int N, const ora_index* dims);
int ora_sort_perm(int N, const ora_index* dims, int* perm, int* inverse);
int ora_fast_update_order(int N, const ora_index* dims, int* order);
int ora_permute(int N, const ora_index* dims, const double* y, const int* perm, double* out);
uint64_t ora_fast_count_realized(int N, const ora_index* dims, ora_index R, int n);
uint64_t ora_predicted_mult_count(int N, const ora_index* dims, ora_index R, int n, int variant);

/* Algorithm 2 (mttkrp.cpp:113-253).  factors[k] points at the caller's I_k x R
 * factor (may be modified by the hook); g_out[k] receives G^(k+1).  counter and
 * peak_ws are optional.  pivot = 0 selects p* (select_pivot); a positive value
 * forces the split point (used for slab shards).  nthreads <= 0: all cores. */
int ora_cp_gradient_all(int N, const ora_index* dims, const double* y, ora_index R,
                        double* const* factors, double* const* g_out,
                        ora_hook_fn hook, void* user, uint64_t* counter,
                        int64_t* peak_ws, int pivot, int nthreads);

/* entrywise definition (test_util.hpp:44-60) */
/* The same all-mode gradient of a GENERATED fp32 tensor, in the caller frame
 * (no mode sort: ascending dims, or a last-mode slab with a forced pivot):
 * Y[q] = U(-1,1) from (seed, offset + q) as ora_fill_upm1_f32, upcast to fp64,
 * streamed through the two seeds so host memory stays O(R (J_p + K_p)) —
 * config 5 (300^4, 32.4 GB in fp32) at full size.  offset = first global index
 * of a last-mode slab. */
int ora_cp_gradient_all_upm1_f32(int N, const ora_index* dims, uint64_t seed, ora_index offset, ora_index R,
                                 double* const* factors, double* const* g_out, int pivot, int nthreads);
int ora_brute_mttkrp(int N, const ora_index* dims, const double* y, ora_index R,
                     const double* const* factors, int n, double* out);

int ora_gram_hadamard_skip(int N, const ora_index* dims, ora_index R,
                           const double* const* factors, int n, double* w);
int ora_pinv_psd(ora_index R, const double* s, double rtol, double* out);
int ora_als_update_mode(int N, const ora_index* dims, ora_index R, const double* m,
                        const double* const* factors, int n, double rtol, double* out);
int ora_als_sweep_fast(int N, const ora_index* dims, const double* y, ora_index R,
                       double* const* factors, double rtol, uint64_t* counter, int nthreads);
double ora_cost(int N, const ora_index* dims, const double* y, ora_index R,
                const double* const* factors, ora_index materialize_limit, int nthreads);
int ora_full(int N, const ora_index* dims, ora_index R, const double* const* factors, double* out);
/* run(y, init, als_fast, opts) (als.cpp:147-210); factors in/out. */
int ora_run_als_fast(int N, const ora_index* dims, const double* y, ora_index R,
                     double* const* factors, int max_iters, double tol, double pinv_rtol,
                     double* cost_trace, double* rel_trace, double* sec_trace,
                     uint64_t* mults_trace, int* iters_run, int nthreads);

/* Uniform01 stream of the reference's fixtures (rng.hpp:9-26). */
int ora_als_sweep_direct(int N, const ora_index* dims, const double* y, ora_index R,
                         double* const* factors, const int* order, int norder, double rtol,
                         uint64_t* counter);
int ora_mu_sweep(int N, const ora_index* dims, const double* y, ora_index R, double* const* factors,
                 double eps, uint64_t* counter, int nthreads);
int ora_gd_step(int N, const ora_index* dims, const double* y, ora_index R, double* const* factors,
                double eta, uint64_t* counter, int nthreads);
int ora_run(int N, const ora_index* dims, const double* y, ora_index R, double* const* factors, int algo,
            int order_pivot, int max_iters, double tol, double pinv_rtol, double mu_eps, double gd_eta,
            double* cost_trace, double* rel_trace, uint64_t* mults_trace, int* iters_run, int nthreads);

void ora_uniform01_fill(uint64_t seed, ora_index n, double* out);
/* Counter-based generator shared with the product's device generator
 * (DESIGN.md "Synthetic inputs"): hash of (seed, linear index). */
uint64_t ora_hash64(uint64_t seed, uint64_t idx);
void ora_fill_normal(uint64_t seed, ora_index offset, ora_index n, double* out, int nthreads);
void ora_fill_upm1_f32(uint64_t seed, ora_index offset, ora_index n, float* out, int nthreads);

#ifdef __cplusplus
}
#endif
#endif
