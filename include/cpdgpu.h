/* cpdgpu.h — C-ABI of the B200-native all-mode CP gradient / fast CP_ALS.
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/proj/core).  Each entry point names the reference
 * interface it replaces (file:line, relative to /root/reference/proj/core).
 * Plain pointers and sizes only: no C++ types, no torch types, no exceptions.
 *
 * Conventions (identical to the reference):
 *   - tensors are dense, column-major (first index fastest; dense_tensor.hpp:12-14);
 *   - factor n is an I_n x R column-major fp64 matrix (kron.hpp:13-14);
 *   - modes are 1-based; results come back in the caller's mode order
 *     (mttkrp.cpp:134-136);
 *   - every call returns a cpdgpu_status; the message of the last failure is
 *     cpdgpu_last_error(ctx).  Statuses map 1:1 onto the reference exception
 *     types (errors.hpp:8-35); see INTEGRATION.md.
 *   - one host thread per context; calls are synchronous with respect to the
 *     host unless they take device pointers (the *_device variants), which are
 *     ordered on the context's stream (cpdgpu_set_stream).
 */
#ifndef CPDGPU_H
#define CPDGPU_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CPDGPU_OK = 0,
  CPDGPU_SHAPE_ERROR = 1,    /* cpd::ShapeError    (errors.hpp:9-11)  */
  CPDGPU_INDEX_ERROR = 2,    /* cpd::IndexError    (errors.hpp:14-16) */
  CPDGPU_ARGUMENT_ERROR = 3, /* cpd::ArgumentError (errors.hpp:19-21) */
  CPDGPU_NUMERIC_ERROR = 4,  /* cpd::NumericError  (errors.hpp:29-31) */
  CPDGPU_DOMAIN_ERROR = 5,   /* cpd::DomainError   (errors.hpp:24-26) */
  CPDGPU_CUDA_ERROR = 6,     /* device / driver failure                */
  CPDGPU_NO_MEMORY = 7,      /* device allocation failed               */
  CPDGPU_PARSE_ERROR = 8,    /* cpd::ParseError    (errors.hpp:33-36) */
  CPDGPU_HOOK_ABORTED = 9    /* the caller's mode hook failed; the caller holds
                                its exception and rethrows it unchanged   */
} cpdgpu_status;

typedef enum { CPDGPU_F64 = 0, CPDGPU_F32 = 1 } cpdgpu_dtype;
typedef enum { CPDGPU_DIST_NORMAL = 0, CPDGPU_DIST_UNIFORM_PM1 = 1 } cpdgpu_dist;

typedef struct cpdgpu_ctx cpdgpu_ctx;
typedef struct cpdgpu_tensor cpdgpu_tensor;

/* Per-mode callback for the generic ModeHook (mttkrp.hpp:49-51): called right
 * after G^(mode) is ready (rows x R, column-major, host memory) and after the
 * mode's multiplication count has been reported through `mults`.  It may
 * overwrite the caller's factor for `mode` (the buffer passed in `factors`),
 * which the sweep re-reads before moving on (mttkrp.cpp:137-144).  A non-zero
 * return aborts the sweep with that status (CPDGPU_HOOK_ABORTED when the hook
 * threw: the adapter rethrows the hook's own exception). */
typedef int (*cpdgpu_mode_hook)(void* user, int mode, const double* gradient, int64_t rows,
                                int64_t rank, uint64_t mults);

/* ---- context ------------------------------------------------------------ */
int cpdgpu_create(cpdgpu_ctx** ctx, int device);
int cpdgpu_destroy(cpdgpu_ctx* ctx);
const char* cpdgpu_last_error(const cpdgpu_ctx* ctx);
/* cudaStream_t as void*; NULL = the context's own stream. */
int cpdgpu_set_stream(cpdgpu_ctx* ctx, void* stream);
int cpdgpu_synchronize(cpdgpu_ctx* ctx);
/* 1 = capture the per-gradient launch sequence into a CUDA graph (default 1). */
int cpdgpu_set_graphs(cpdgpu_ctx* ctx, int enabled);
/* 1 = bitwise-reproducible results run to run (default 0; CPDGPU_DETERMINISTIC=1
 * sets the default).  Two seed passes differ: by default the drains of the
 * fused fp32 seed and of the int8 fp64 seed add their per-band / per-row-block
 * left partials in L2 (red.add; the addition order varies, so repeats differ in
 * the last bits: ~1e-7 relative for fp32, ~1e-16 for fp64); deterministic mode
 * stores one partial slot per band / row block and sums them in a fixed order
 * (c5: +0.9 ms per gradient).  The DMMA and split fp32 passes are always
 * deterministic. */
int cpdgpu_set_deterministic(cpdgpu_ctx* ctx, int enabled);
/* Kernels launched by this context so far (evidence counter for bench.py). */
uint64_t cpdgpu_launch_count(const cpdgpu_ctx* ctx);
/* 1 = bracket every seed-contraction launch (K1) with CUDA events on the
 * context stream; cpdgpu_last_seed_ms then returns the summed K1 device time
 * of the most recent gradient / sweep call (synchronises on the last event). */
int cpdgpu_set_timing(cpdgpu_ctx* ctx, int enabled);
int cpdgpu_last_seed_ms(cpdgpu_ctx* ctx, double* ms);
/* Seed path of the most recent hook-free fp64 gradient: 0 = fp64 DMMA pass,
 * 1 = fused pass on the int8 tensor cores (default for large fp64 tensors; CPDGPU_I8=1/0
 * forces it on/off), 2 = fp32 two passes, 3 = fp32 one fused pass splitting Y in
 * the kernel, 4 = fp32 one fused pass over the tensor's cached fp16 operand image
 * (the default; CPDGPU_F32_IMAGE=0 / CPDGPU_F32_FUSED=0 select 3 / 2). */
int cpdgpu_last_seed_path(const cpdgpu_ctx* ctx);

/* ---- tensors (DenseTensor, dense_tensor.hpp:15-47) -------------------------
 * A tensor is immutable once created, as the reference's is; the context may
 * cache a mode-sorted copy (sort_modes, mttkrp.cpp:67-90) for its lifetime. */
int cpdgpu_tensor_upload(cpdgpu_ctx* ctx, const void* host, cpdgpu_dtype dtype, int N,
                         const int64_t* dims, cpdgpu_tensor** out);
/* Zero-copy view of caller-owned device memory (not freed by the library). */
int cpdgpu_tensor_wrap_device(cpdgpu_ctx* ctx, void* device_ptr, cpdgpu_dtype dtype, int N,
                              const int64_t* dims, cpdgpu_tensor** out);
/* Device-side generation: entry at global linear index (offset + q) is drawn
 * from the counter-based generator of DESIGN.md "Synthetic inputs". */
int cpdgpu_tensor_generate(cpdgpu_ctx* ctx, cpdgpu_dtype dtype, int N, const int64_t* dims,
                           cpdgpu_dist dist, uint64_t seed, int64_t offset, cpdgpu_tensor** out);
/* Y <- alpha * Y + beta * full(model)  (full: kruskal.cpp:23-31). */
int cpdgpu_tensor_axpby_kruskal(cpdgpu_ctx* ctx, cpdgpu_tensor* t, double alpha, double beta,
                                const double* const* factors, int64_t R);
/* Refresh an existing tensor's values from host memory (same dims/dtype);
 * the H2D copy of the end-to-end path.  Pinned host memory copies at full
 * PCIe/C2C rate; drops the cached norm and sorted copy. */
int cpdgpu_tensor_update(cpdgpu_ctx* ctx, cpdgpu_tensor* t, const void* host);
int cpdgpu_tensor_download(cpdgpu_ctx* ctx, const cpdgpu_tensor* t, void* host);
/* |Y|_F^2 in fp64 (DenseTensor::norm, dense_tensor.cpp:32-34, squared). */
int cpdgpu_tensor_norm2(cpdgpu_ctx* ctx, cpdgpu_tensor* t, double* out);
int cpdgpu_tensor_device_ptr(const cpdgpu_tensor* t, void** device_ptr);
int cpdgpu_tensor_free(cpdgpu_tensor* t);

/* ---- problem generation and cost (rng.hpp:9-26, kruskal.cpp:58-77) -------
 * uniform01_fill: the reference's Uniform01 stream (mt19937_64, splitmix seed),
 * host-side and bitwise identical; generate_problem / random_init draw from it.
 * cost: |Y - full(model)|^2 on the device by the Gram identity. */
int cpdgpu_uniform01_fill(uint64_t seed, int64_t n, double* out);
int cpdgpu_cost(cpdgpu_ctx* ctx, cpdgpu_tensor* y, int64_t R, const double* const* factors, double* out);

/* ---- TDNB tensor files (io.hpp:10-12, io.cpp:162-216) --------------------
 * Binary form "TDNB" + u32 LE N + u32 LE dims + f64 LE values (vec order).
 * load: streams the file through pinned double buffers straight to the device;
 * slab_hi > slab_lo loads only last-mode slices [slab_lo, slab_hi) (a rank's
 * shard), else the whole tensor.  Malformed files -> CPDGPU_PARSE_ERROR with the
 * byte offset in the message.  save: f64 LE (fp32 tensors are widened exactly). */
int cpdgpu_tensor_load_tdnb(cpdgpu_ctx* ctx, const char* path, int64_t slab_lo, int64_t slab_hi,
                            cpdgpu_tensor** out);
int cpdgpu_tensor_save_tdnb(cpdgpu_ctx* ctx, const cpdgpu_tensor* t, const char* path);

/* ---- ordering helpers (mttkrp.hpp:24,35,73) ----------------------------- */
int cpdgpu_select_pivot(int N, const int64_t* dims, int* pivot);            /* mttkrp.cpp:56-65  */
int cpdgpu_sort_modes(int N, const int64_t* dims, int* perm, int* inverse); /* mttkrp.cpp:67-90  */
int cpdgpu_fast_update_order(int N, const int64_t* dims, int* order);       /* mttkrp.cpp:92-111 */
/* mttkrp.cpp:292-320 (dims must be ascending); 0 on bad input. */
uint64_t cpdgpu_fast_count_realized(int N, const int64_t* dims, int64_t R, int n);
/* predicted_mult_count (mttkrp.hpp:85-86, mttkrp.cpp:255-290): the analytic
 * count of one mode, variant 0 direct, 1 fast (compressed closed form), 2
 * fast_derived (CountVariant order).  Ascending dims; status 2 (IndexError) for a
 * mode outside 1..N, 3 (ArgumentError) for R < 1 or unsorted dims. */
int cpdgpu_predicted_mult_count(int N, const int64_t* dims, int64_t R, int n, int variant, uint64_t* out);
/* FastStats::peak_workspace_doubles (mttkrp.hpp:37-47) as the reference's
 * cp_gradient_all tracks it (mttkrp.cpp:127-131,147-243) for ascending dims: the
 * figure every gradient entry point reports through peak_workspace (host only). */
int cpdgpu_reference_workspace(int N, const int64_t* dims, int64_t R, int64_t* out);
/* The DEVICE workspace this implementation holds, in bytes: seed partials, Khatri-Rao
 * operands, operand images, padded / sorted copies and tables of every live plan and
 * tensor of the process (not the tensors' own values) -- now and at its high-water mark.
 * This is what FastStats::peak_workspace_doubles (mttkrp.hpp:37-47, tracked at
 * mttkrp.cpp:127-131,243) measures for the reference; the gradient entry points keep
 * reporting the reference algorithm's figure (above) so the bound its tests check
 * (test_mttkrp.cpp:188-198) holds, and this call reports the real one. */
int cpdgpu_device_workspace(cpdgpu_ctx* ctx, int64_t* current_bytes, int64_t* peak_bytes);

/* ---- all-mode CP gradient (cp_gradient_all, mttkrp.hpp:59-69, mttkrp.cpp:113-253)
 * factors[k] / gradients[k]: host I_{k+1} x R column-major fp64 buffers in the
 * caller's mode order.  mults_per_mode (N entries, optional) receives the
 * reference's per-mode multiplication charges (fast_count_realized);
 * peak_workspace (optional) the FastStats::peak_workspace_doubles figure. */
int cpdgpu_cp_gradient_all(cpdgpu_ctx* ctx, cpdgpu_tensor* y, int64_t R,
                           const double* const* factors, double* const* gradients,
                           uint64_t* mults_per_mode, int64_t* peak_workspace);
/* Hook form (mttkrp.hpp:59-63): factors[] are mutable; hook runs per mode in
 * fast_update_order and the sweep reads back any factor it replaced. */
int cpdgpu_cp_gradient_all_hook(cpdgpu_ctx* ctx, cpdgpu_tensor* y, int64_t R,
                                double* const* factors, double* const* gradients,
                                cpdgpu_mode_hook hook, void* user, int64_t* peak_workspace);
/* Device form: factors_dev / gradients_dev are device buffers holding the N
 * factor (gradient) matrices packed back to back in the caller's mode order
 * (sum_n I_n x R doubles).  pivot = 0 selects p*; a positive pivot forces the
 * split point (slab shards of a larger tensor use the global p*).  Ordered on
 * the context stream; no host synchronisation. */
int cpdgpu_cp_gradient_all_device(cpdgpu_ctx* ctx, cpdgpu_tensor* y, int64_t R,
                                  const double* factors_dev, double* gradients_dev, int pivot);

/* ---- multi-GPU: last-mode slab sharding ----------------------
 * Replaces running cp_gradient_all (mttkrp.hpp:59-69) on one huge tensor: each
 * rank (one process per GPU) holds the contiguous last-mode slab [lo, hi) of a
 * global tensor whose dims are ascending, computes its slab's gradient with the
 * GLOBAL pivot p* (the right seed and G(1..N-1) are linear sums over slabs, the
 * rows of G(N) belong to the slab), and ONE all-reduce(sum) of
 * [partial G(1..N-1) | G(N) rows at the slab's offset, zeros elsewhere]
 * finishes it inside the library.  The collective is NCCL (dlopen'ed
 * libnccl.so.2, in-place ncclAllReduce on the context stream over NVLink) or a
 * caller-supplied host all-reduce (e.g. MPI or gloo). */
#define CPDGPU_COMM_ID_BYTES 128
/* Host all-reduce: sum `count` doubles of `buf` across the ranks, in place. */
typedef int (*cpdgpu_allreduce_fn)(void* user, double* buf, int64_t count);
/* Rank 0 creates the id (ncclGetUniqueId) and the caller broadcasts it. */
int cpdgpu_comm_unique_id(unsigned char* id /* CPDGPU_COMM_ID_BYTES */);
/* Joins the NCCL communicator on the context's device (ncclCommInitRank). */
int cpdgpu_comm_init(cpdgpu_ctx* ctx, const unsigned char* id, int nranks, int rank);
/* The exchange runs through `fn` on host memory instead of NCCL. */
int cpdgpu_comm_init_host(cpdgpu_ctx* ctx, int nranks, int rank, cpdgpu_allreduce_fn fn, void* user);
int cpdgpu_comm_destroy(cpdgpu_ctx* ctx);
/* Balanced contiguous split of the last mode (sizes differ by at most one:
 * 300 over 8 ranks -> 38,38,38,38,37,37,37,37). */
int cpdgpu_slab_bounds(int64_t extent, int nranks, int rank, int64_t* lo, int64_t* hi);
/* Sharded all-mode gradient.  slab: this rank's tensor, dims = global_dims
 * except the last (hi - lo, with [lo, hi) = cpdgpu_slab_bounds of the
 * communicator's rank).  factors / gradients: the GLOBAL I_n x R matrices
 * (host, caller's mode order); every rank receives the full gradients.
 * mults (optional, N entries): the per-mode charges of the unsharded call
 * (fast_count_realized on global_dims). */
int cpdgpu_cp_gradient_all_sharded(cpdgpu_ctx* ctx, cpdgpu_tensor* slab, int N, const int64_t* global_dims,
                                   int64_t R, const double* const* factors, double* const* gradients,
                                   uint64_t* mults);
/* Device form, ordered on the context stream: factors_dev = the slab's packed
 * factors (modes 1..N-1 whole, rows [lo, hi) of mode N); out_dev = the packed
 * GLOBAL result, (sum_{n<N} I_n + I_N) x R doubles: G(1..N-1) then G(N). */
int cpdgpu_cp_gradient_all_sharded_device(cpdgpu_ctx* ctx, cpdgpu_tensor* slab, int N, const int64_t* global_dims,
                                          int64_t R, const double* factors_dev, double* out_dev);
/* Sharded als_sweep_fast (als.cpp:69-78) in the global sweep order: all-reduce
 * of each G(n), n < N, before A_n's update (I_n x R), of A_N's Gram after its
 * row-local update (R x R), and of [A_N | G(N)] rows for the cost and the
 * caller's whole A_N (2 I_N x R).  factors: the GLOBAL matrices, updated in
 * place identically on every rank.  A NumericError on any rank fails the call on
 * every rank.  cost_out / mults optional (mults: the unsharded sweep's charge). */
int cpdgpu_als_sweep_sharded(cpdgpu_ctx* ctx, cpdgpu_tensor* slab, int N, const int64_t* global_dims, int64_t R,
                             double* const* factors, double pinv_rtol, double* cost_out, uint64_t* mults);
/* run(y, init, Algorithm::als_fast, opts) (als.cpp:147-210) over slabs; traces
 * as cpdgpu_als_run (the cost and fit are global; every rank stops together). */
int cpdgpu_als_run_sharded(cpdgpu_ctx* ctx, cpdgpu_tensor* slab, int N, const int64_t* global_dims, int64_t R,
                           double* const* factors, int max_iters, double tol, double pinv_rtol, double* cost_trace,
                           double* rel_trace, double* sec_trace, uint64_t* mults_trace, int* iters_run);

/* ---- direct MTTKRP (Algorithm 1 cost model; mttkrp.hpp:19-20, mttkrp.cpp:29-54)
 * One pass over Y for one mode: out = Y_(n) (KR_{k != n} A(k)), I_n x R column-major,
 * caller's mode order; mults (optional) receives the reference's charge. */
int cpdgpu_mttkrp_direct(cpdgpu_ctx* ctx, cpdgpu_tensor* y, int64_t R, const double* const* factors, int n,
                         double* out, uint64_t* mults);
/* Device form: packed factors in, block n of the packed gradient buffer written. */
int cpdgpu_mttkrp_direct_device(cpdgpu_ctx* ctx, cpdgpu_tensor* y, int64_t R, const double* factors_dev, int n,
                                double* gradients_dev);
/* als_sweep_direct (als.hpp:58-60, als.cpp:58-67): modes in `order` (1-based), each
 * update sees the previous ones; factors updated in place. */
int cpdgpu_als_sweep_direct(cpdgpu_ctx* ctx, cpdgpu_tensor* y, int64_t R, double* const* factors, const int* order,
                            int norder, double pinv_rtol, uint64_t* mults);

/* ---- fast CP_ALS (als.hpp:48-93) ----------------------------------------- */
/* pinv_psd (als.cpp:34-47) of a host R x R symmetric matrix, on the device. */
int cpdgpu_pinv_psd(cpdgpu_ctx* ctx, int64_t R, const double* s, double rtol, double* out);
/* als_update_mode (als.cpp:49-56): out = m * pinv_psd(gram_hadamard_skip(factors, n)). */
int cpdgpu_als_update_mode(cpdgpu_ctx* ctx, int N, const int64_t* dims, int64_t R,
                           const double* m, const double* const* factors, int n, double rtol,
                           double* out);
/* als_sweep_fast (als.cpp:69-78): factors updated in place; the whole sweep
 * (gradients, Gram/Hadamard, pseudo-inverse, update) runs on the device.
 * cost_out (optional) receives cost(y, model) after the sweep (kruskal.cpp:58-77). */
int cpdgpu_als_sweep(cpdgpu_ctx* ctx, cpdgpu_tensor* y, int64_t R, double* const* factors,
                     double pinv_rtol, double* cost_out, uint64_t* mults);
/* mu_sweep (als.cpp:80-91): A <- A .* G ./ (A W + eps) per mode through the
 * Gauss-Seidel sweep; negative tensor / factor entries -> DomainError. */
int cpdgpu_mu_sweep(cpdgpu_ctx* ctx, cpdgpu_tensor* y, int64_t R, double* const* factors, double eps,
                    uint64_t* mults);
/* gd_step (als.cpp:93-101): a <- a + 2 eta (M - A W) for all modes at the pre-step factors. */
int cpdgpu_gd_step(cpdgpu_ctx* ctx, cpdgpu_tensor* y, int64_t R, double* const* factors, double eta,
                   uint64_t* mults);
/* run(y, init, algo, opts) (als.cpp:147-210) for every Algorithm: 0 als_direct
 * (order_pivot != 0: fast_update_order, else 1..N), 1 als_fast, 2 mu, 3 gd. */
int cpdgpu_run_algo(cpdgpu_ctx* ctx, cpdgpu_tensor* y, int64_t R, double* const* factors, int algo,
                    int order_pivot, int max_iters, double tol, double pinv_rtol, double mu_eps, double gd_eta,
                    double* cost_trace, double* rel_trace, double* sec_trace, uint64_t* mults_trace,
                    int* iters_run);
/* run(y, init, Algorithm::als_fast, opts) (als.cpp:147-210).  Traces hold
 * max_iters entries; sec_trace times each sweep on the device (CUDA events). */
int cpdgpu_als_run(cpdgpu_ctx* ctx, cpdgpu_tensor* y, int64_t R, double* const* factors,
                   int max_iters, double tol, double pinv_rtol, double* cost_trace,
                   double* rel_trace, double* sec_trace, uint64_t* mults_trace, int* iters_run);

#ifdef __cplusplus
}
#endif
#endif /* CPDGPU_H */
