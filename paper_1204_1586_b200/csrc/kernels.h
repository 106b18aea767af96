// kernels.h — host-visible launch interface of the device kernels.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda.h>
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
  int use_tma;      // Y tiles arrive by 2-D TMA (dense LDY == TI); else plain copies
  int stages;       // pipeline depth (2 or 3)
  KRSpec left;      // modes 1..p   (rows of the view)
  KRSpec right;     // modes p+1..N (columns of the view)
  const double* KRl_g;  // Khatri-Rao rows of the view's rows    [J][LDK] (kr_materialize)
  const double* KRr_g;  // Khatri-Rao rows of the view's columns [K][LDK]
  unsigned long long* trace;  // optional per-warp counters [P][9][8] (CPDGPU_SEED_TRACE)
  unsigned long long* tl;     // launch timeline (CPDGPU_TIMELINE) and this launch's slot
  int tl_slot;
  double* Rpart;    // [P * slots][R8][TI]
  double* Lpart;    // [nRB][R][K]
};
// Row stride (doubles) of the Khatri-Rao row buffers and their shared-memory
// tiles: == 4 mod 8, so the DMMA fragment loads (lane (g, t) reads row t,
// column g) of a half-warp hit 16 distinct 8-byte banks.
__host__ __device__ constexpr int seed_ldk(int NT) { return NT * 8 + 4; }
// largest row block the fused kernel can hold in registers for this NT
int seed_f64_max_ti(int NT);
size_t seed_f64_smem_bytes(int NT, int TI, int LDY, int LDK, int mode, int stages, int64_t fac_doubles);
constexpr size_t kSeedSmemLimit = 232448 - 1024;  // per-block opt-in limit, minus slack
// tmap: 2-D tensor map of Y (dim0 = rows J, dim1 = columns K, box TI x 32), or
// nullptr when p.use_tma == 0.
// kmap: 2-D tensor map of KRr_g (dim0 = LDK, dim1 = K, box LDK x 32).
int launch_seed_f64(const SeedParams& p, const CUtensorMap* tmap, const CUtensorMap* kmap, int NT, int mode,
                    cudaStream_t s);

// Host helper: 2-D tiled tensor map (driver entry point, no -lcuda link).
bool make_tensor_map_2d(CUtensorMap* out, const void* base, CUtensorMapDataType dtype, int elem_bytes,
                        uint64_t dim0, uint64_t dim1, uint64_t stride1_bytes, uint32_t box0, uint32_t box1,
                        bool swizzle128 = false, int promote = true);
// Left seed alone with column-block accumulation (ALS / hook second pass): TI =
// columns per block (256), nRB = column blocks, nCT = 32-row stages per block,
// Rpart = partial slots [P * slots][8 NT][TI].  ymap: Y (dim0 J, dim1 K), box
// 16 x TI, 128-byte swizzle; kmap: KR_l rows (dim0 LDK, dim1 J), box LDK x 32.
int launch_seed_left_cols(const SeedParams& p, const CUtensorMap* ymap, const CUtensorMap* kmap, int NT,
                          cudaStream_t s);
size_t seed_left_cols_smem_bytes(int NT, int TJ, int stages);

// ---- K1 fp64 fused on the int8 tensor cores (seed_i8.cu) ---------------------
// Both seeds in one pass over Y, 128 x 128 tiles, tile = rb * nCT + ct, CTA c owns
// [c T / P, (c + 1) T / P).  Right partials: Rpart[(c * slots + rb - rb0)][RP][128];
// left partials: Lpart[(rb * R + r) * K + j] (the fp64 path's formats, TI = 128).
struct SeedI8Params {
  int64_t J, K;          // J_p, K_p
  int R, RP, N, NL;      // rank columns, Rpart row stride (8 NT), right / left MMA rank blocks
  int64_t nRB, nCT, T;   // 128-row blocks, 128-column tiles, nRB * nCT
  int P, slots;
  const unsigned char* img_r;  // [nCT][6][N][128] Khatri-Rao digits of the view's columns
  const unsigned char* img_l;  // [nRB][6][N][128]                 ... of the view's rows
  const double* w_r;           // [nCT][N] column weights 2^(eY + e_r - 52)
  const double* w_l;           // [nRB][N]
  const double* yscale;        // tensor scale record: [0] 2^(46 - eY), [1] eY, [2] max |Y|
  double* Rpart;
  double* Lpart;
  unsigned* progress;  // CPDGPU_I8_DEBUG: [P][16] per-warp positions for the watchdog report
  unsigned long long* trace;  // CPDGPU_SEED_TRACE: [P][14][6] per-warp wait cycles, total, tiles
  int knobs;                  // CPDGPU_I8_KNOBS experiments (bit 0: no digit stores)
  int lred;                   // left partials red.add'ed into row-block slot 0 (zeroed by the host)
  int rhalf;                  // right product as two M = 64 row halves issued while the split runs (CPDGPU_I8_RHALF)
  int* fault;                 // context fault word: the watchdog's report (no trap)
  int stall;                  // tests: force a pipeline stall (CPDGPU_FORCE_STALL)
  int watchdog;               // bounded barrier waits (CPDGPU_WATCHDOG=1; implied by stall)
};
// left rank block for a right block N and rank R (24 when it lets the left accumulators
// double-buffer in TMEM), and the left digit image bytes per row block
int i8_left_block(int N, int R);
size_t i8_left_image_bytes(int NL);
size_t i8_right_image_bytes(int N, int NL);
// ymap: Y (dim0 J, dim1 K) fp64, box 16 x 128, 128-byte swizzle
int launch_seed_i8(const SeedI8Params& p, const CUtensorMap* ymap, cudaStream_t s);
// int8 factor-range guard (both sides' Khatri-Rao columns): *flag |= 1 when a column's
// max / rms product exceeds `limit` or a factor entry is not finite
int launch_i8_factor_guard(const KRSpec& right, const KRSpec& left, int R, double limit, int* flag, cudaStream_t s);
// Khatri-Rao rows [L][ldk] -> digit images [ceil(L / 128)][6][N][128] + weights [.][N]
// Khatri-Rao digit images [tiles][6][N][128] + column weights [tiles][N] of both
// sides, from the factors (right: K_p rows, left: J_p rows; one launch)
// numel / budget / fault: the error-budget check of the call's factors (tile 0 of
// each side; *fault = 3000 when prod_m max / rms > budget mean|Y| / max|Y|)
int launch_kr_digits(const KRSpec& right, int64_t Kp, const KRSpec& left, int64_t Jp, int R, int N, int NL,
                     const double* yscale, void* img_r, double* w_r, void* img_l, double* w_l, int64_t numel,
                     double budget, int* fault, cudaStream_t s);
// fp64 tensor scale record [2^(46-eY), eY, max|Y|, sum|Y|] (bitwise reproducible);
// scratch >= 16 * y_scale_f64_blocks(n, num_sms) bytes
int y_scale_f64_blocks(int64_t n, int num_sms);
int launch_y_scale_f64(const double* y, int64_t n, void* scratch, double* out, int num_sms, cudaStream_t s);

// ---- K1 for fp32 tensors: tcgen05 split-fp16 seed contraction (seed_f32.cu) ---
// One pass computes ONE seed (right: blocks over the view's rows i, k-tiles over
// columns j; left: blocks over columns j, k-tiles over rows i) for up to 64 rank
// columns.  CTA c owns units [c U / P, (c + 1) U / P) of unit = block * nK + tile
// and writes one fp64 partial [64][128] per block it touches (slot c * slots + s).
struct Seed32Params {
  const unsigned char* kr_tiles;  // [nK][16 KB] scaled fp16 hi / lo Khatri-Rao tiles
  const float* scale_y;           // [1] power-of-two Y scale
  const double* inv_scale_y;      // [1]
  const double* inv_scale_kr;     // [64] Khatri-Rao column unscales of this side
  double* part;                   // [P * slots][64][128]
  int64_t nK, units;
  int P, slots, chunk;
  int debug;  // experiment knobs (CPDGPU_F32_DEBUG): bit 0 one MMA per k-step, bit 1 no split work
  unsigned long long* trace;  // optional [P][10][4] per-warp cycle counters (CPDGPU_SEED_TRACE)
};
size_t seed_f32_smem_bytes();
int seed_f32_rank_cols();         // 64
int64_t seed_f32_tile_bytes();    // bytes of one Khatri-Rao tile (64 rows)
int launch_seed_f32(const Seed32Params& p, const CUtensorMap* ymap, int left, cudaStream_t s);
// ---- K1 for fp32 tensors, both seeds in one HBM pass (seed_f32f.cu) ------------
// unit = (band of seed_f32f_band_tiles() 128-row tiles, one 64-column tile); CTA c
// owns units [c U / P, (c + 1) U / P) band-major.  Outputs: the right seed as
// fp64 partial blocks [slot][64 r][128 i] (slot = (c slots + band - first band) 3
// + row tile in band; CSR per row tile for the tail), the left seed as fp32
// partials [band][column tile][64 r][64 j] in scaled units (kOpReduceLeft32 sums
// the bands).
struct Seed32FParams {
  const unsigned char* kr_tiles;  // [nC][16 KB] right Khatri-Rao tiles (kr_split layout)
  const void* krl_img;            // [nRT][128][128] fp16 KRl^T image (launch_krl_image)
  const float* scale_y;           // [1] power-of-two Y scale
  const double* inv_scale_y;      // [1]
  const double* inv_scale_kr;     // [64] right Khatri-Rao column unscales
  double* rpart;
  float* lpart;
  int64_t nRT, nC, units;
  int P, slots, window;
  unsigned long long* trace;  // CPDGPU_SEED_TRACE: [P][16 warps][8] cycle counters (image kernel)
  int knobs;  // CPDGPU_F32F_KNOBS timing experiments (wrong results): 1 no split stores,
              // 2 one right MMA per k-step, 4 one left MMA per k-step, 8 no left partial stores,
              // 16 (image kernel) no plane refills after the first ring, 32 (image kernel) no MMAs
  int* fault;  // context fault word: the watchdog's report (no trap)
  int stall;   // tests: force a pipeline stall (CPDGPU_FORCE_STALL)
  int watchdog;  // image kernel: bounded barrier waits (CPDGPU_WATCHDOG=1; implied by stall)
  int band_tiles;  // row tiles per band: 3, or 2 (image kernel only: stacked right product)
  int left_m64;    // image kernel: the left Y_lo MMA with M = 64 (hi parts only, no lo * lo product)
};
int seed_f32f_band_tiles();  // 3 (the in-kernel-split variant)
// ymap: the right pass's map (box 128 i x 64 j, no swizzle)
int launch_seed_f32f(const Seed32FParams& p, const CUtensorMap* ymap, cudaStream_t s);
// The same kernel reading a cached operand image of the tensor instead of the fp32
// values (no split stage).  imap: make_tensor_map_f16_image of that image.
int launch_seed_f32i(const Seed32FParams& p, const CUtensorMap* imap, cudaStream_t s);
// operand image of an fp32 view (J x K, leading dimension ldy): [2][K][LD] fp16
// planes hi = fp16(s y), lo = fp16(s y - hi), LD = f16_image_ld(J) (rows past J zero).
// (A unit-ordered, pre-swizzled 32 KB-tile layout moved by bulk copies streamed
// faster alone but made the fused pass 0.6 ms slower at c5: measured and dropped.)
int64_t f16_image_ld(int64_t J);
int launch_build_f16_image(const float* y, int64_t J, int64_t ldy, int64_t K, const float* scale, void* img,
                           int num_sms, int chunked, cudaStream_t s);
bool make_tensor_map_f16_image(CUtensorMap* out, const void* img, int64_t J, int64_t K, int chunked);
// fused pass: column scales, right B tiles and the KRl^T image straight from the
// sorted factors (two launches, no fp64 Khatri-Rao rows)
// (lane_halves: the KRl^T slot of (rank r, part) is 32 (r / 16) + 16 part + r % 16, the
// operand-image kernel's TMEM lane layout, instead of 2 r + part)
int launch_kr_fused_operands(const KRSpec& right, int64_t Kp, const KRSpec& left, int64_t Jp, int R, double* scale,
                             double* inv, void* rtiles, void* limg, int lane_halves, cudaStream_t s);
// column scales of the right (scale[0..63]) and left (scale[64..127]) Khatri-Rao rows
int launch_kr_scale(const KRSpec& right, const KRSpec& left, int R, double* scale, double* inv, cudaStream_t s);
// fp64 rows [L][ld] (ld <= 64) -> tiles (see Seed32Params::kr_tiles)
int launch_kr_split(const double* rows, int64_t L, int ld, const double* scale, void* tiles, cudaStream_t s);
int launch_y_scale(const float* y, int64_t n, unsigned int* amax_scratch, float* scale, double* inv, int num_sms,
                   cudaStream_t s);
// fp64 view J x K (leading dimension J) -> leading dimension LD (even, >= J), rows past J zero
int launch_pad_rows_f64(const double* src, double* dst, int64_t J, int64_t LD, int64_t K, int num_sms,
                        cudaStream_t s);
int launch_pad_rows_f32(const float* src, float* dst, int64_t J, int64_t J8, int64_t K, int num_sms,
                        cudaStream_t s);
// 2-D map of a J8 x K column-major fp32 matrix; box for the right (128 i x 64 j)
// or left (64 i x 128 j) pass.  J8 % 8 == 0.
bool make_tensor_map_y32(CUtensorMap* out, const void* base, int64_t J8, int64_t K, int left);

// ---- prologue + recursion tail (tail.cu) ------------------------------------
enum TailOpType {
  kOpNone = 0,
  kOpContractA = 1,
  kOpContractB = 2,
  kOpReduceRight = 3,
  kOpReduceLeft = 4
};

// One rank-batched contraction / reduction (all R columns):
//  ContractA: out[r*ldo + b] = sum_{a<M} Z[r*ldz + a + M*b] * KR(kr)[a, r]   (Eq 3.12 / 3.22)
//  ContractB: out[r*ldo + a] = sum_{b<B} Z[r*ldz + a + M*b] * KR(kr)[b, r]   (Eq 3.20 / 3.16)
//  ReduceRight: out[r*ldo + i] = sum over the right-partial slots of row block i / TI
//               (Z = Rpart [slots][RP][TI], M = J rows, CSR rb_ptr / slot_list)
//  ReduceLeft:  out[r*ldo + j] = sum_{rb < B} Z[(rb*R + r)*M + j]  (M = K columns)
// out_slot >= 0 writes through the device pointer table instead of `out`.
struct TailOp {
  int type;
  int R;
  const double* Z;
  int64_t ldz, M, B;
  KRSpec kr;
  double* out;
  int64_t ldo;
  int out_slot;
  int64_t out_off;
  int RP, TI;
  const int* rb_ptr;
  const int* slot_list;
  int cta;  // set by launch_tail_step: long contractions run one output per CTA
};
constexpr int kMaxTailOps = 8;
struct TailStep {
  int n;
  TailOp op[kMaxTailOps];
  unsigned long long* tl = nullptr;  // launch timeline (CPDGPU_TIMELINE)
  int tl_slot = 0;
};
// First recursion level fused with the seed-partial reduction.  A side pairs
// the two contractions of one seed Z (rows a + M b, a < M, b < B):
//   opA: outA[r][b] = sum_a Z[a + M b, r] KR_A[a, r]   (complete per b)
//   opB: outB[r][a] = sum_b Z[a + M b, r] KR_B[b, r]   (partial per b-chunk)
// One CTA per (side, r, chunk of b): it sums its rows of Z from the partials
// (zsrc as TailOp) into shared memory, writes opA's outputs and its opB partial;
// the last CTA of (side, r) to finish (ticket counter) adds the chunk partials in
// chunk order.  Right side: opA = extraction G(p), opB = recursion R^(p-1);
// left side: opA = recursion L^(p+2), opB = extraction G(p+1).
struct L0Side {
  int zsrc;  // 0 direct (Z[r ldz + idx]), 1 right slots, 2 left row blocks (ldz = R pK)
  const double* Z;
  int64_t ldz;
  int RP, TI;
  const int* rb_ptr;
  const int* slot_list;
  int pcount;
  int64_t pK;
  int64_t M, B;
  int nq, bq;  // b-chunks and b per chunk
  KRSpec krA, krB;
  double* outA;  // nullptr: gtab[slotA] + 0 (ld ldoA)
  int slotA;
  int64_t ldoA;
  double* outB;
  int slotB;
  int64_t ldoB;
  double* scratch;    // [R][nq][M]
  unsigned* tickets;  // [R], zero between calls
};
struct L0Step {
  int nsides, R;
  L0Side side[2];
  unsigned long long* tl = nullptr;
  int tl_slot = 0;
};
constexpr int kL0Threads = 256;
constexpr int64_t kL0MaxRows = 6144;  // Z rows per CTA staged in shared memory (48 KB)
int launch_l0_step(const L0Step& st, double* const* gtab, cudaStream_t s);

int64_t tail_step_units(const TailStep& st);
// fused fp32 seed: Ls[r][j] = us_y[0] us_r[r] sum_b Z[((b nC + j / 64) 64 + r) 64 + j % 64]
// into out, or into gtab[out_slot] when out_slot >= 0 (the left seed is a gradient);
// chunked = 1: the operand-image kernel's layout Z[(((b nC + j / 64) 16 + j % 64 / 4) 64 + r) 4 + j % 4]
int launch_reduce_left32(const float* Z, int64_t nB, int64_t nC, int64_t M, int R, const double* us_y,
                         const double* us_r, double* out, double* const* gtab, int out_slot, int64_t ldo,
                         int chunked, cudaStream_t s);
int launch_tail_step(const TailStep& st, double* const* gtab, int num_sms, cudaStream_t s);

// Khatri-Rao rows for K1: out[q*LDK + r] = KR(spec)[q, r] for q < L (zero past R).
struct KRJob {
  KRSpec spec;
  int64_t L;
  int R, NT, LDK;
  double* out;
};
constexpr int kMaxKRJobs = 8;
// Prologue of a gradient: Fs block j <- fin block (src_off[j]) (skipped when Fs
// is null), gtab[m] <- gout[m], then every KR job.
struct Prologue {
  int N;
  const double* fin;
  double* Fs;
  int64_t src_off[kMaxModes], dst_off[kMaxModes], len[kMaxModes];
  double* gout[kMaxModes];
  int nkr;
  KRJob kr[kMaxKRJobs];
  unsigned long long* tl = nullptr;  // launch timeline (CPDGPU_TIMELINE), slot 0
  double* zero = nullptr;            // zeroed here: the int8 seed's red.add left-partial slot
  int64_t zero_n = 0;
};
int launch_prologue(const Prologue& pr, double** gtab, int num_sms, cudaStream_t s);
const void* prologue_kernel_fn();
void prologue_geometry(const Prologue& pr, int num_sms, dim3* grid, dim3* block);

// ---- utilities (util.cu) -----------------------------------------------------
// packed factor gather: dst block j <- src block (src_off[j]); plain block copies
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
// mu_sweep update (als.cpp:84-90) of mode n: A <- A .* G ./ (A W + eps); gram_n <- A^T A.
int launch_mu_update(const double* G, int64_t I, int R, const double* grams, int N, int n, double eps, double* A,
                     double* gram_n, cudaStream_t s);
// gd_step update of mode n (als.cpp:93-101): A += 2 eta (G - A W), W from the old Grams.
int launch_gd_update(const double* G, int64_t I, int R, const double* grams, int N, int n, double eta, double* A,
                     cudaStream_t s);
// status[0] <- 5 when the fp64 / fp32 tensor has a negative entry.
int launch_nonneg_check(const void* y, int elem_bytes, int64_t n, int* status, cudaStream_t s);
// standalone pinv_psd of a device R x R matrix
int launch_pinv_psd(const double* S, int R, double rtol, double* out, cudaStream_t s);
// cost = ynorm2 - 2 sum(A_L .* G_L) + 1^T (hadamard of all grams) 1, clamped at 0
int launch_als_cost(const double* A, const double* G, int64_t I, int R, const double* grams,
                     int N, const double* ynorm2, double* cost_out, cudaStream_t s);

}  // namespace cpdgpu
