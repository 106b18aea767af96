/* cpd_oracle.c — CPU restatement of the reference's hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see cpd_oracle.h).  Every function cites the
 * reference file:line it restates (paths relative to /root/reference/proj/core).
 * The reference itself cannot be compiled in this image: it needs Eigen >= 3.3,
 * which is neither vendored nor installed, so this is a
 * restatement pinned against the reference tests' known-answer vectors and the
 * entrywise definition (tests/test_oracle.py).
 */
#include "cpd_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { ORA_OK = 0, ORA_SHAPE = 1, ORA_INDEX = 2, ORA_ARG = 3, ORA_NUMERIC = 4, ORA_DOMAIN = 5 };
#define MAXN 64

/* ---- shape arithmetic (shape.cpp:8-36, shape.hpp:27-32) ------------------ */

static void prefix_products(int N, const ora_index* dims, ora_index* J) {
  J[0] = 1;
  for (int k = 0; k < N; ++k) J[k + 1] = J[k] * dims[k];
}

static int set_threads(int nthreads) {
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_num_procs();
  return nthreads;
#else
  (void)nthreads;
  return 1;
#endif
}

/* select_pivot: max{n : J_n <= K_n}, ties to the larger n (mttkrp.cpp:56-65). */
int ora_select_pivot(int N, const ora_index* dims) {
  if (N < 2 || N > MAXN) return -ORA_ARG;
  ora_index J[MAXN + 1];
  prefix_products(N, dims, J);
  int pivot = 0;
  for (int n = 1; n <= N; ++n)
    if (J[n] <= J[N] / J[n]) pivot = n;
  if (pivot == 0) return -ORA_SHAPE;
  return pivot;
}

/* stable ascending sort of modes (mttkrp.cpp:67-90); returns 1 when identity. */
int ora_sort_perm(int N, const ora_index* dims, int* perm, int* inverse) {
  for (int j = 0; j < N; ++j) perm[j] = j + 1;
  for (int a = 1; a < N; ++a) { /* insertion sort == stable */
    int v = perm[a], b = a - 1;
    while (b >= 0 && dims[perm[b] - 1] > dims[v - 1]) {
      perm[b + 1] = perm[b];
      --b;
    }
    perm[b + 1] = v;
  }
  int identity = 1;
  for (int j = 1; j <= N; ++j) {
    if (inverse) inverse[perm[j - 1] - 1] = j;
    identity &= (perm[j - 1] == j);
  }
  return identity;
}

/* fast_update_order (mttkrp.cpp:92-111). */
int ora_fast_update_order(int N, const ora_index* dims, int* order) {
  if (N < 2 || N > MAXN) return ORA_ARG;
  int perm[MAXN];
  ora_index sd[MAXN];
  ora_sort_perm(N, dims, perm, NULL);
  for (int j = 0; j < N; ++j) sd[j] = dims[perm[j] - 1];
  const int p = ora_select_pivot(N, sd);
  if (p < 0) return -p;
  int at = 0;
  for (int j = p; j >= 1; --j) order[at++] = perm[j - 1];
  for (int j = p + 1; j <= N; ++j) order[at++] = perm[j - 1];
  return ORA_OK;
}

/* permute: new axis k = old mode perm[k] (tensor_ops.cpp:39-71). */
int ora_permute(int N, const ora_index* dims, const double* y, const int* perm, double* out) {
  ora_index od[MAXN], oJ[MAXN + 1], ostride[MAXN], cnt[MAXN];
  for (int k = 0; k < N; ++k) od[k] = dims[perm[k] - 1];
  prefix_products(N, od, oJ);
  for (int k = 0; k < N; ++k) ostride[perm[k] - 1] = oJ[k];
  const ora_index total = oJ[N];
  memset(cnt, 0, sizeof cnt);
  ora_index dst = 0;
  for (ora_index s = 0; s < total; ++s) {
    out[dst] = y[s];
    for (int m = 0; m < N; ++m) {
      dst += ostride[m];
      if (++cnt[m] < dims[m]) break;
      dst -= ostride[m] * dims[m];
      cnt[m] = 0;
    }
  }
  return ORA_OK;
}

/* ---- multiplication-count model (mttkrp.cpp:255-320) -------------------- */

static uint64_t sum_j(const ora_index* J, int lo, int hi, ora_index div) {
  uint64_t t = 0;
  for (int k = lo < 0 ? 0 : lo; k <= hi; ++k) t += (uint64_t)(J[k] / div);
  return t;
}

uint64_t ora_fast_count_realized(int N, const ora_index* dims, ora_index R, int n) {
  ora_index J[MAXN + 1];
  prefix_products(N, dims, J);
  const int p = ora_select_pivot(N, dims);
  const uint64_t uR = (uint64_t)R;
#define KS(m) (J[N] / J[(m)])
  if (n == p)
    return uR * ((uint64_t)J[N] + sum_j(J, n + 2, N, J[n]) + sum_j(J, 2, n - 1, 1) + (uint64_t)J[n]);
  if (n == p + 1)
    return uR * ((uint64_t)J[N] + sum_j(J, 2, n - 1, 1) + sum_j(J, n + 2, N, J[n]) + (uint64_t)KS(n - 1));
  if (n < p) return uR * ((uint64_t)J[n + 1] + sum_j(J, 2, n - 1, 1) + (uint64_t)J[n]);
  return uR * ((uint64_t)KS(n - 2) + sum_j(J, n + 2, N, J[n]) + (uint64_t)KS(n - 1));
}

/* variant: 0 direct, 1 fast, 2 fast_derived (mttkrp.cpp:255-290). */
uint64_t ora_predicted_mult_count(int N, const ora_index* dims, ora_index R, int n, int variant) {
  ora_index J[MAXN + 1];
  prefix_products(N, dims, J);
  const uint64_t uR = (uint64_t)R;
  if (variant == 0)
    return uR * ((uint64_t)J[N] + sum_j(J, 2, n - 1, 1) + sum_j(J, n + 1, N, dims[n - 1]));
  const int p = ora_select_pivot(N, dims);
  if (n == p || n == p + 1) {
    const ora_index a = J[n], b = KS(n - 1);
    const uint64_t pivot_term = (uint64_t)(a < b ? a : b);
    return uR * (sum_j(J, 2, n - 1, 1) + pivot_term + sum_j(J, n + 2, N, J[n]) + (uint64_t)J[N]);
  }
  if (n < p) return uR * sum_j(J, 2, n + 1, 1);
  const uint64_t tail = variant == 1 ? sum_j(J, n + 2, N, 1) : sum_j(J, n + 2, N, J[n]);
  return uR * ((uint64_t)KS(n - 2) + (uint64_t)KS(n - 1) + tail);
#undef KS
}

/* ---- Khatri-Rao column (kron.cpp:47-68) ---------------------------------- */

/* t = a_r^(hi) kron ... kron a_r^(lo) (lo fastest) over the sorted factors
 * sf[0..N-1]; returns |t|.  Empty range -> [1].  Charges |a|*|t| per fold. */
static ora_index kron_range_column(const ora_index* dims, double* const* sf, int lo, int hi,
                                   ora_index r, double* t, uint64_t* counter) {
  if (lo > hi) {
    t[0] = 1.0;
    return 1;
  }
  ora_index len = dims[lo - 1];
  memcpy(t, sf[lo - 1] + r * dims[lo - 1], (size_t)len * sizeof(double));
  for (int k = lo + 1; k <= hi; ++k) {
    const ora_index ia = dims[k - 1];
    const double* a = sf[k - 1] + r * ia;
    if (counter) *counter += (uint64_t)ia * (uint64_t)len;
    for (ora_index i = ia - 1; i >= 0; --i) /* in place, outermost block last */
      for (ora_index q = len - 1; q >= 0; --q) t[i * len + q] = a[i] * t[q];
    len *= ia;
  }
  return len;
}

/* ---- Algorithm 2: all-mode gradient (mttkrp.cpp:113-253) ----------------- */

typedef struct {
  int64_t live, peak;
} ws_track;
static void track(ws_track* w, int64_t d) {
  w->live += d;
  if (w->live > w->peak) w->peak = w->live;
}

/* right[i + Jp r] = sum_c Y[i + Jp c] KR[c + Kp r]   (mttkrp.cpp:160) */
static void seed_right(const double* y, ora_index Jp, ora_index Kp, ora_index R, const double* KR,
                       double* right, int nth) {
  const size_t per = (size_t)Jp * (size_t)R;
  double* priv = (double*)calloc((size_t)nth * per, sizeof(double));
#pragma omp parallel num_threads(nth)
  {
    int tid = 0;
#ifdef _OPENMP
    tid = omp_get_thread_num();
#endif
    double* acc = priv + (size_t)tid * per;
#pragma omp for schedule(static)
    for (ora_index c = 0; c < Kp; ++c) {
      const double* col = y + (size_t)c * (size_t)Jp;
      for (ora_index r = 0; r < R; ++r) {
        const double k = KR[c + Kp * r];
        double* out = acc + (size_t)r * (size_t)Jp;
        for (ora_index i = 0; i < Jp; ++i) out[i] += col[i] * k;
      }
    }
  }
  memset(right, 0, per * sizeof(double));
  for (int t = 0; t < nth; ++t)
    for (size_t q = 0; q < per; ++q) right[q] += priv[(size_t)t * per + q];
  free(priv);
}

/* left[c + Kp r] = sum_i Y[i + Jp c] KR[i + Jp r]   (mttkrp.cpp:207) */
static void seed_left(const double* y, ora_index Jp, ora_index Kp, ora_index R, const double* KR,
                      double* left, int nth) {
#pragma omp parallel for num_threads(nth) schedule(static)
  for (ora_index c = 0; c < Kp; ++c) {
    const double* col = y + (size_t)c * (size_t)Jp;
    for (ora_index r = 0; r < R; ++r) {
      const double* k = KR + (size_t)r * (size_t)Jp;
      double s = 0.0;
      for (ora_index i = 0; i < Jp; ++i) s += col[i] * k[i];
      left[c + Kp * r] = s;
    }
  }
}

/* ---- streaming seeds over a generated fp32 tensor (config 5) ---------------
 * Y entries are never held: Y[q] = U(-1,1) fp32 from (seed, offset + q), the
 * ora_fill_upm1_f32 formula, upcast to fp64; the two seed products of
 * mttkrp.cpp:160 and :207 are accumulated in fp64 over cache-sized tiles.
 * Host memory is O(R (J_p + K_p)), so the 32.4 GB fp32 tensor of config 5 is
 * checked at full size. */
typedef struct {
  const double* y; /* in-memory values (column-major), or NULL: generated */
  uint64_t seed;
  ora_index offset;
} ysrc;

static inline double gen_upm1(uint64_t seed, uint64_t idx) {
  const uint64_t h = ora_hash64(seed, idx);
  return (double)((float)((int32_t)(h >> 40) - 8388608) * 0x1.0p-23f);
}

enum { GB_I = 256, GB_C = 64 };

/* right[i + Jp r] = sum_c Y[i + Jp c] KR[c + Kp r]: thread = block of GB_I rows,
 * accumulators [GB_I][R] (rank fastest), Khatri-Rao rows transposed [Kp][R]. */
static void seed_right_gen(const ysrc* src, ora_index Jp, ora_index Kp, ora_index R, const double* KR,
                           double* right, int nth) {
  double* KT = (double*)malloc((size_t)Kp * (size_t)R * sizeof(double));
  for (ora_index c = 0; c < Kp; ++c)
    for (ora_index r = 0; r < R; ++r) KT[c * R + r] = KR[c + Kp * r];
  const ora_index nb = (Jp + GB_I - 1) / GB_I;
#pragma omp parallel num_threads(nth)
  {
    double* acc = (double*)malloc((size_t)GB_I * (size_t)R * sizeof(double));
    double yb[GB_I];
#pragma omp for schedule(dynamic, 1)
    for (ora_index b = 0; b < nb; ++b) {
      const ora_index i0 = b * GB_I, ni = (Jp - i0) < GB_I ? (Jp - i0) : GB_I;
      memset(acc, 0, (size_t)GB_I * (size_t)R * sizeof(double));
      for (ora_index c = 0; c < Kp; ++c) {
        const uint64_t base = (uint64_t)(src->offset + i0 + Jp * c);
        for (ora_index i = 0; i < ni; ++i) yb[i] = gen_upm1(src->seed, base + (uint64_t)i);
        const double* k = KT + (size_t)c * (size_t)R;
        for (ora_index i = 0; i < ni; ++i) {
          double* a = acc + (size_t)i * (size_t)R;
          const double v = yb[i];
          for (ora_index r = 0; r < R; ++r) a[r] += v * k[r];
        }
      }
      for (ora_index i = 0; i < ni; ++i)
        for (ora_index r = 0; r < R; ++r) right[i0 + i + Jp * r] = acc[(size_t)i * (size_t)R + r];
    }
    free(acc);
  }
  free(KT);
}

/* left[c + Kp r] = sum_i Y[i + Jp c] KR[i + Jp r]: thread = block of GB_C
 * columns, rows in chunks of GB_I (Khatri-Rao rows transposed [Jp][R]). */
static void seed_left_gen(const ysrc* src, ora_index Jp, ora_index Kp, ora_index R, const double* KR,
                          double* left, int nth) {
  double* KT = (double*)malloc((size_t)Jp * (size_t)R * sizeof(double));
  for (ora_index i = 0; i < Jp; ++i)
    for (ora_index r = 0; r < R; ++r) KT[i * R + r] = KR[i + Jp * r];
  const ora_index nb = (Kp + GB_C - 1) / GB_C;
#pragma omp parallel num_threads(nth)
  {
    double* acc = (double*)malloc((size_t)GB_C * (size_t)R * sizeof(double));
    double* yb = (double*)malloc((size_t)GB_C * GB_I * sizeof(double));
#pragma omp for schedule(dynamic, 1)
    for (ora_index b = 0; b < nb; ++b) {
      const ora_index c0 = b * GB_C, nc = (Kp - c0) < GB_C ? (Kp - c0) : GB_C;
      memset(acc, 0, (size_t)GB_C * (size_t)R * sizeof(double));
      for (ora_index i0 = 0; i0 < Jp; i0 += GB_I) {
        const ora_index ni = (Jp - i0) < GB_I ? (Jp - i0) : GB_I;
        for (ora_index c = 0; c < nc; ++c) {
          const uint64_t base = (uint64_t)(src->offset + i0 + Jp * (c0 + c));
          for (ora_index i = 0; i < ni; ++i) yb[c * GB_I + i] = gen_upm1(src->seed, base + (uint64_t)i);
        }
        for (ora_index i = 0; i < ni; ++i) {
          const double* k = KT + (size_t)(i0 + i) * (size_t)R;
          for (ora_index c = 0; c < nc; ++c) {
            double* a = acc + (size_t)c * (size_t)R;
            const double v = yb[c * GB_I + i];
            for (ora_index r = 0; r < R; ++r) a[r] += v * k[r];
          }
        }
      }
      for (ora_index c = 0; c < nc; ++c)
        for (ora_index r = 0; r < R; ++r) left[c0 + c + Kp * r] = acc[(size_t)c * (size_t)R + r];
    }
    free(yb);
    free(acc);
  }
  free(KT);
}

static int cp_gradient_core(int N, const ora_index* dims, const ysrc* src, ora_index R,
                            double* const* factors, double* const* g_out, ora_hook_fn hook,
                            void* user, uint64_t* counter, int64_t* peak_ws, int pivot, int nthreads);

int ora_cp_gradient_all(int N, const ora_index* dims, const double* y, ora_index R,
                        double* const* factors, double* const* g_out, ora_hook_fn hook,
                        void* user, uint64_t* counter, int64_t* peak_ws, int pivot,
                        int nthreads) {
  const ysrc src = {y, 0, 0};
  return cp_gradient_core(N, dims, &src, R, factors, g_out, hook, user, counter, peak_ws, pivot, nthreads);
}

int ora_cp_gradient_all_upm1_f32(int N, const ora_index* dims, uint64_t seed, ora_index offset, ora_index R,
                                 double* const* factors, double* const* g_out, int pivot, int nthreads) {
  if (N < 2 || N > MAXN) return ORA_ARG;
  const ysrc src = {NULL, seed, offset};
  return cp_gradient_core(N, dims, &src, R, factors, g_out, NULL, NULL, NULL, NULL, pivot, nthreads);
}

static int cp_gradient_core(int N, const ora_index* dims, const ysrc* src, ora_index R,
                            double* const* factors, double* const* g_out, ora_hook_fn hook,
                            void* user, uint64_t* counter, int64_t* peak_ws, int pivot, int nthreads) {
  const double* y = src->y;
  if (N < 2) return ORA_ARG; /* mttkrp.cpp:119 */
  if (N > MAXN || R < 1) return ORA_ARG;
  const int nth = set_threads(nthreads);
  int perm[MAXN];
  int identity = ora_sort_perm(N, dims, perm, NULL); /* mttkrp.cpp:123 */
  if (!y) { /* generated Y is read in the caller's frame (a slab of an ascending tensor) */
    for (int j = 0; j < N; ++j) perm[j] = j + 1;
    identity = 1;
  }
  ora_index sd[MAXN], J[MAXN + 1];
  for (int j = 0; j < N; ++j) sd[j] = dims[perm[j] - 1];
  prefix_products(N, sd, J);
  const double* ys = y;
  double* yperm = NULL;
  if (!identity && y) {
    yperm = (double*)malloc((size_t)J[N] * sizeof(double));
    ora_permute(N, dims, y, perm, yperm);
    ys = yperm;
  }
  double* sf[MAXN]; /* s.factors: sorted copies (mttkrp.cpp:80-82) */
  for (int j = 0; j < N; ++j) {
    sf[j] = (double*)malloc((size_t)sd[j] * (size_t)R * sizeof(double));
    memcpy(sf[j], factors[perm[j] - 1], (size_t)sd[j] * (size_t)R * sizeof(double));
  }
  int p = pivot > 0 ? pivot : ora_select_pivot(N, sd); /* mttkrp.cpp:125 */
  if (p < 0) {
    for (int j = 0; j < N; ++j) free(sf[j]);
    free(yperm);
    return -p;
  }
  ws_track ws = {0, 0};
  ora_index maxdim = 1;
  for (int j = 0; j < N; ++j) maxdim = sd[j] > maxdim ? sd[j] : maxdim;
  const ora_index Jp = J[p], Kp = J[N] / J[p];
  /* extraction kron columns: |t| <= J_{p-1} (right) or K_{p+1} (left) */
  ora_index tcap = J[p - 1];
  if (p + 1 <= N && J[N] / J[p + 1] > tcap) tcap = J[N] / J[p + 1];
  double* t = (double*)malloc((size_t)(tcap > 1 ? tcap : 1) * sizeof(double) + 64);
  double* G = (double*)malloc((size_t)maxdim * (size_t)R * sizeof(double));

#define EMIT(jj, rows)                                                                     \
  do {                                                                                     \
    const int orig = perm[(jj)-1];                                                         \
    memcpy(g_out[orig - 1], G, (size_t)(rows) * (size_t)R * sizeof(double));               \
    if (hook) {                                                                            \
      hook(user, orig, g_out[orig - 1], (rows), R);                                        \
      memcpy(sf[(jj)-1], factors[orig - 1], (size_t)(rows) * (size_t)R * sizeof(double)); \
    }                                                                                      \
  } while (0)

  /* Right phase (mttkrp.cpp:149-193). */
  double* right = (double*)malloc((size_t)Jp * (size_t)R * sizeof(double));
  {
    double* KR = (double*)malloc((size_t)Kp * (size_t)R * sizeof(double));
    track(&ws, Kp * R);
    for (ora_index r = 0; r < R; ++r)
      kron_range_column(sd, sf, p + 1, N, r, KR + (size_t)r * (size_t)Kp, counter);
    track(&ws, Jp * R);
    if (counter) *counter += (uint64_t)Jp * (uint64_t)Kp * (uint64_t)R;
    if (ys)
      seed_right(ys, Jp, Kp, R, KR, right, nth);
    else
      seed_right_gen(src, Jp, Kp, R, KR, right, nth);
    free(KR);
    track(&ws, -Kp * R);
  }
  ora_index scr_len = J[p - 1] > 1 ? J[p - 1] : 1;
  double* scratch = (double*)malloc((size_t)(Jp > Kp ? Jp : Kp) * sizeof(double) + 64);
  track(&ws, scr_len);
  for (int j = p; j >= 1; --j) {
    if (j < p) { /* Eq 3.20: R^(r,j) = reshape(R^(r,j+1), [J_j, I_{j+1}]) a_r^(j+1) */
      const ora_index Jj = J[j], In = sd[j];
      for (ora_index r = 0; r < R; ++r) {
        const double* Z = right + (size_t)r * (size_t)Jp;
        const double* a = sf[j] + r * In;
        if (counter) *counter += (uint64_t)Jj * (uint64_t)In;
        for (ora_index q = 0; q < Jj; ++q) scratch[q] = 0.0;
        for (ora_index b = 0; b < In; ++b)
          for (ora_index q = 0; q < Jj; ++q) scratch[q] += Z[q + Jj * b] * a[b];
        memcpy(right + (size_t)r * (size_t)Jp, scratch, (size_t)Jj * sizeof(double));
      }
    }
    /* Eq 3.12: g_r = reshape(R^(r,j), [J_{j-1}, I_j])^T kron(a^(j-1..1)) */
    const ora_index Jm1 = J[j - 1], Ij = sd[j - 1];
    for (ora_index r = 0; r < R; ++r) {
      const ora_index tl = kron_range_column(sd, sf, 1, j - 1, r, t, counter);
      track(&ws, tl);
      const double* Z = right + (size_t)r * (size_t)Jp;
      if (counter) *counter += (uint64_t)Ij * (uint64_t)Jm1;
      for (ora_index b = 0; b < Ij; ++b) {
        double s = 0.0;
        for (ora_index a = 0; a < Jm1; ++a) s += Z[a + Jm1 * b] * t[a];
        G[b + Ij * r] = s;
      }
      track(&ws, -tl);
    }
    EMIT(j, Ij);
  }
  track(&ws, -scr_len);
  track(&ws, -Jp * R);
  free(right);

  /* Left phase (mttkrp.cpp:195-241). */
  if (p + 1 <= N) {
    double* left = (double*)malloc((size_t)Kp * (size_t)R * sizeof(double));
    {
      double* KR = (double*)malloc((size_t)Jp * (size_t)R * sizeof(double));
      track(&ws, Jp * R);
      for (ora_index r = 0; r < R; ++r)
        kron_range_column(sd, sf, 1, p, r, KR + (size_t)r * (size_t)Jp, counter);
      track(&ws, Kp * R);
      if (counter) *counter += (uint64_t)Kp * (uint64_t)Jp * (uint64_t)R;
      if (ys)
        seed_left(ys, Jp, Kp, R, KR, left, nth);
      else
        seed_left_gen(src, Jp, Kp, R, KR, left, nth);
      free(KR);
      track(&ws, -Jp * R);
    }
    scr_len = J[N] / J[p + 1] > 1 ? J[N] / J[p + 1] : 1;
    track(&ws, scr_len);
    for (int j = p + 1; j <= N; ++j) {
      if (j > p + 1) { /* Eq 3.22: L^(r,j) = reshape(L^(r,j-1), [I_{j-1}, K_{j-1}])^T a_r^(j-1) */
        const ora_index Ip = sd[j - 2], Km1 = J[N] / J[j - 1];
        for (ora_index r = 0; r < R; ++r) {
          const double* Z = left + (size_t)r * (size_t)Kp;
          const double* a = sf[j - 2] + r * Ip;
          if (counter) *counter += (uint64_t)Km1 * (uint64_t)Ip;
          for (ora_index c = 0; c < Km1; ++c) {
            double s = 0.0;
            for (ora_index b = 0; b < Ip; ++b) s += Z[b + Ip * c] * a[b];
            scratch[c] = s;
          }
          memcpy(left + (size_t)r * (size_t)Kp, scratch, (size_t)Km1 * sizeof(double));
        }
      }
      /* Eq 3.16: g_r = reshape(L^(r,j), [I_j, K_j]) kron(a^(N..j+1)) */
      const ora_index Ij = sd[j - 1], Kj = J[N] / J[j];
      for (ora_index r = 0; r < R; ++r) {
        const ora_index tl = kron_range_column(sd, sf, j + 1, N, r, t, counter);
        track(&ws, tl);
        const double* Z = left + (size_t)r * (size_t)Kp;
        if (counter) *counter += (uint64_t)Ij * (uint64_t)Kj;
        for (ora_index b = 0; b < Ij; ++b) G[b + Ij * r] = 0.0;
        for (ora_index c = 0; c < Kj; ++c)
          for (ora_index b = 0; b < Ij; ++b) G[b + Ij * r] += Z[b + Ij * c] * t[c];
        track(&ws, -tl);
      }
      EMIT(j, Ij);
    }
    track(&ws, -scr_len);
    track(&ws, -Kp * R);
    free(left);
  }
#undef EMIT
  if (peak_ws) *peak_ws = ws.peak;
  free(scratch);
  free(G);
  free(t);
  for (int j = 0; j < N; ++j) free(sf[j]);
  free(yperm);
  return ORA_OK;
}

/* ---- entrywise oracle (tests/test_util.hpp:44-60) ------------------------ */

int ora_brute_mttkrp(int N, const ora_index* dims, const double* y, ora_index R,
                     const double* const* f, int n, double* out) {
  if (n < 1 || n > N) return ORA_INDEX;
  ora_index J[MAXN + 1], mi[MAXN];
  prefix_products(N, dims, J);
  memset(out, 0, (size_t)dims[n - 1] * (size_t)R * sizeof(double));
  for (ora_index lin = 0; lin < J[N]; ++lin) {
    ora_index rem = lin;
    for (int k = 0; k < N; ++k) {
      mi[k] = rem % dims[k];
      rem /= dims[k];
    }
    const double v = y[lin];
    for (ora_index r = 0; r < R; ++r) {
      double prod = 1.0;
      for (int k = 0; k < N; ++k)
        if (k != n - 1) prod *= f[k][mi[k] + dims[k] * r];
      out[mi[n - 1] + dims[n - 1] * r] += v * prod;
    }
  }
  return ORA_OK;
}

/* ---- ALS pieces (kron.cpp:124-134, als.cpp:34-78) ------------------------ */

int ora_gram_hadamard_skip(int N, const ora_index* dims, ora_index R,
                           const double* const* f, int n, double* w) {
  if (n < 1 || n > N) return ORA_INDEX;
  for (ora_index q = 0; q < R * R; ++q) w[q] = 1.0;
  for (int k = 1; k <= N; ++k) {
    if (k == n) continue;
    const double* A = f[k - 1];
    const ora_index I = dims[k - 1];
    for (ora_index c = 0; c < R; ++c)
      for (ora_index a = 0; a < R; ++a) {
        double s = 0.0;
        for (ora_index i = 0; i < I; ++i) s += A[i + I * a] * A[i + I * c];
        w[a + R * c] *= s;
      }
  }
  return ORA_OK;
}

/* Symmetric eigendecomposition by cyclic Jacobi (the reference uses Eigen's
 * SelfAdjointEigenSolver; any backward-stable symmetric solver restates it). */
static int sym_eig(ora_index n, double* a, double* v, double* ev) {
  for (ora_index i = 0; i < n * n; ++i) v[i] = 0.0;
  for (ora_index i = 0; i < n; ++i) v[i + n * i] = 1.0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    int rotated = 0;
    for (ora_index p = 0; p < n - 1; ++p)
      for (ora_index q = p + 1; q < n; ++q) {
        const double apq = a[p + n * q];
        const double app = a[p + n * p], aqq = a[q + n * q];
        if (apq == 0.0 || fabs(apq) <= 1e-16 * sqrt(fabs(app * aqq))) continue;
        rotated = 1;
        const double theta = (aqq - app) / (2.0 * apq);
        const double tt = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(tt * tt + 1.0), s = tt * c;
        for (ora_index k = 0; k < n; ++k) { /* A <- A J (columns p,q) */
          const double akp = a[k + n * p], akq = a[k + n * q];
          a[k + n * p] = c * akp - s * akq;
          a[k + n * q] = s * akp + c * akq;
        }
        for (ora_index k = 0; k < n; ++k) { /* A <- J^T A (rows p,q) */
          const double apk = a[p + n * k], aqk = a[q + n * k];
          a[p + n * k] = c * apk - s * aqk;
          a[q + n * k] = s * apk + c * aqk;
        }
        a[p + n * q] = a[q + n * p] = 0.0;
        for (ora_index k = 0; k < n; ++k) {
          const double vkp = v[k + n * p], vkq = v[k + n * q];
          v[k + n * p] = c * vkp - s * vkq;
          v[k + n * q] = s * vkp + c * vkq;
        }
      }
    if (!rotated) break;
  }
  for (ora_index i = 0; i < n; ++i) ev[i] = a[i + n * i];
  return ORA_OK;
}

/* pinv_psd (als.cpp:34-47): eigenvalues <= rtol*max|lambda| (or <= 0) dropped. */
int ora_pinv_psd(ora_index R, const double* s, double rtol, double* out) {
  if (rtol < 0.0) return ORA_ARG;
  double* a = (double*)malloc((size_t)(R * R) * sizeof(double));
  double* v = (double*)malloc((size_t)(R * R) * sizeof(double));
  double* ev = (double*)malloc((size_t)(R > 0 ? R : 1) * sizeof(double));
  memcpy(a, s, (size_t)(R * R) * sizeof(double));
  sym_eig(R, a, v, ev);
  double mx = 0.0;
  for (ora_index i = 0; i < R; ++i) mx = fabs(ev[i]) > mx ? fabs(ev[i]) : mx;
  const double cutoff = R > 0 ? rtol * mx : 0.0;
  for (ora_index i = 0; i < R; ++i) ev[i] = (ev[i] > cutoff && ev[i] > 0.0) ? 1.0 / ev[i] : 0.0;
  for (ora_index c = 0; c < R; ++c)
    for (ora_index r = 0; r < R; ++r) {
      double acc = 0.0;
      for (ora_index k = 0; k < R; ++k) acc += v[r + R * k] * ev[k] * v[c + R * k];
      out[r + R * c] = acc;
    }
  free(a);
  free(v);
  free(ev);
  return ORA_OK;
}

/* als_update_mode (als.cpp:49-56): M * pinv_psd(gram_hadamard_skip). */
int ora_als_update_mode(int N, const ora_index* dims, ora_index R, const double* m,
                        const double* const* f, int n, double rtol, double* out) {
  if (n < 1 || n > N) return ORA_INDEX;
  const ora_index I = dims[n - 1];
  for (ora_index q = 0; q < I * R; ++q)
    if (!isfinite(m[q])) return ORA_NUMERIC;
  double* w = (double*)malloc((size_t)(R * R) * sizeof(double));
  double* pw = (double*)malloc((size_t)(R * R) * sizeof(double));
  ora_gram_hadamard_skip(N, dims, R, f, n, w);
  int st = ora_pinv_psd(R, w, rtol, pw);
  if (st == ORA_OK)
    for (ora_index c = 0; c < R; ++c)
      for (ora_index i = 0; i < I; ++i) {
        double acc = 0.0;
        for (ora_index k = 0; k < R; ++k) acc += m[i + I * k] * pw[k + R * c];
        out[i + I * c] = acc;
      }
  free(w);
  free(pw);
  return st;
}

typedef struct {
  int N;
  const ora_index* dims;
  ora_index R;
  double* const* factors;
  double rtol;
  int status;
} als_ctx;

static void als_hook(void* user, int n, const double* g, ora_index rows, ora_index R) {
  als_ctx* c = (als_ctx*)user;
  double* upd = (double*)malloc((size_t)(rows * R) * sizeof(double));
  int st = ora_als_update_mode(c->N, c->dims, c->R, g, (const double* const*)c->factors, n,
                               c->rtol, upd);
  if (st == ORA_OK)
    memcpy(c->factors[n - 1], upd, (size_t)(rows * R) * sizeof(double));
  else if (c->status == ORA_OK)
    c->status = st;
  free(upd);
}

/* als_sweep_fast (als.cpp:69-78). */
int ora_als_sweep_fast(int N, const ora_index* dims, const double* y, ora_index R,
                       double* const* factors, double rtol, uint64_t* counter, int nthreads) {
  als_ctx c = {N, dims, R, factors, rtol, ORA_OK};
  double* g[MAXN] = {0};
  for (int k = 0; k < N; ++k) g[k] = (double*)malloc((size_t)(dims[k] * R) * sizeof(double));
  int st = ora_cp_gradient_all(N, dims, y, R, factors, g, als_hook, &c, counter, NULL, 0, nthreads);
  for (int k = 0; k < N; ++k) free(g[k]);
  return st != ORA_OK ? st : c.status;
}

/* full (kruskal.cpp:23-31). */
int ora_full(int N, const ora_index* dims, ora_index R, const double* const* f, double* out) {
  ora_index J[MAXN + 1];
  prefix_products(N, dims, J);
  double* t = (double*)malloc((size_t)J[N] * sizeof(double));
  memset(out, 0, (size_t)J[N] * sizeof(double));
  for (ora_index r = 0; r < R; ++r) {
    kron_range_column(dims, (double* const*)f, 1, N, r, t, NULL);
    for (ora_index q = 0; q < J[N]; ++q) out[q] += t[q];
  }
  free(t);
  return ORA_OK;
}

/* cost (kruskal.cpp:42-77): materialise up to the limit, else the Gram
 * identity |Y|^2 - 2<Y,Yhat> + 1^T(hadamard of Grams)1 with <Y,Yhat> from
 * inner_with_model.  All R columns are accumulated in one pass over Y (the
 * reference makes R passes; the arithmetic per column is the same). */
double ora_cost(int N, const ora_index* dims, const double* y, ora_index R,
                const double* const* f, ora_index materialize_limit, int nthreads) {
  const int nth = set_threads(nthreads);
  ora_index J[MAXN + 1];
  prefix_products(N, dims, J);
  if (J[N] <= materialize_limit) {
    double* yh = (double*)malloc((size_t)J[N] * sizeof(double));
    ora_full(N, dims, R, f, yh);
    double d = 0.0;
    for (ora_index q = 0; q < J[N]; ++q) d += (y[q] - yh[q]) * (y[q] - yh[q]);
    free(yh);
    return d;
  }
  double* W = (double*)malloc((size_t)(R * R) * sizeof(double));
  for (ora_index q = 0; q < R * R; ++q) W[q] = 1.0;
  for (int n = 0; n < N; ++n)
    for (ora_index c = 0; c < R; ++c)
      for (ora_index a = 0; a < R; ++a) {
        double s = 0.0;
        for (ora_index i = 0; i < dims[n]; ++i) s += f[n][i + dims[n] * a] * f[n][i + dims[n] * c];
        W[a + R * c] *= s;
      }
  double wsum = 0.0;
  for (ora_index q = 0; q < R * R; ++q) wsum += W[q];
  free(W);
  double yy = 0.0;
#pragma omp parallel for num_threads(nth) reduction(+ : yy) schedule(static)
  for (ora_index q = 0; q < J[N]; ++q) yy += y[q] * y[q];
  /* inner_with_model (kruskal.cpp:42-54): Ypref = J_{N-1} x I_N. */
  double inner = 0.0;
  const ora_index Jn1 = J[N - 1], IN = dims[N - 1];
  double* T = (double*)malloc((size_t)(Jn1 * R) * sizeof(double));
  for (ora_index r = 0; r < R; ++r)
    kron_range_column(dims, (double* const*)f, 1, N - 1, r, T + (size_t)(r * Jn1), NULL);
  double* perr = (double*)calloc((size_t)R, sizeof(double));
  for (ora_index r = 0; r < R; ++r) {
    double dot = 0.0;
#pragma omp parallel for num_threads(nth) reduction(+ : dot) schedule(static)
    for (ora_index c = 0; c < IN; ++c) {
      const double* col = y + (size_t)(c * Jn1);
      const double* t = T + (size_t)(r * Jn1);
      double s = 0.0;
      for (ora_index i = 0; i < Jn1; ++i) s += col[i] * t[i];
      dot += f[N - 1][c + IN * r] * s;
    }
    perr[r] = dot;
  }
  for (ora_index r = 0; r < R; ++r) inner += perr[r];
  free(perr);
  free(T);
  const double d = yy - 2.0 * inner + wsum;
  return d < 0.0 ? 0.0 : d;
}

static double now_seconds(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* run(y, init, als_fast, opts) (als.cpp:147-210). */
int ora_run_als_fast(int N, const ora_index* dims, const double* y, ora_index R,
                     double* const* factors, int max_iters, double tol, double pinv_rtol,
                     double* cost_trace, double* rel_trace, double* sec_trace,
                     uint64_t* mults_trace, int* iters_run, int nthreads) {
  if (max_iters < 1) return ORA_ARG;
  if (tol < 0.0 || pinv_rtol < 0.0) return ORA_ARG;
  int perm[MAXN];
  const int identity = ora_sort_perm(N, dims, perm, NULL);
  ora_index sd[MAXN], J[MAXN + 1];
  for (int j = 0; j < N; ++j) sd[j] = dims[perm[j] - 1];
  prefix_products(N, sd, J);
  const double* work = y;
  double* yperm = NULL;
  double* sf[MAXN];
  for (int j = 0; j < N; ++j) {
    sf[j] = (double*)malloc((size_t)(sd[j] * R) * sizeof(double));
    memcpy(sf[j], factors[perm[j] - 1], (size_t)(sd[j] * R) * sizeof(double));
  }
  if (!identity) { /* hoisted sort (als.cpp:159-165) */
    yperm = (double*)malloc((size_t)J[N] * sizeof(double));
    ora_permute(N, dims, y, perm, yperm);
    work = yperm;
  }
  double yn = 0.0;
  for (ora_index q = 0; q < J[N]; ++q) yn += work[q] * work[q];
  yn = sqrt(yn);
  uint64_t counter = 0;
  double prev = NAN;
  int st = ORA_OK, it;
  int done = 0;
  for (it = 1; it <= max_iters; ++it) {
    const double t0 = now_seconds();
    st = ora_als_sweep_fast(N, sd, work, R, sf, pinv_rtol, &counter, nthreads);
    const double t1 = now_seconds();
    if (st != ORA_OK) break;
    sec_trace[it - 1] = t1 - t0;
    if (mults_trace) mults_trace[it - 1] = counter;
    ++done;
    const double d = ora_cost(N, sd, work, R, (const double* const*)sf, 1000000, nthreads);
    cost_trace[it - 1] = d;
    rel_trace[it - 1] = yn > 0.0 ? sqrt(d) / yn : sqrt(d);
    if (tol > 0.0 && it > 1 && fabs(d - prev) / (prev > 1e-15 ? prev : 1e-15) < tol) break;
    prev = d;
  }
  *iters_run = done;
  for (int j = 0; j < N; ++j) { /* un-permute (als.cpp:206-208) */
    memcpy(factors[perm[j] - 1], sf[j], (size_t)(sd[j] * R) * sizeof(double));
    free(sf[j]);
  }
  free(yperm);
  return st;
}

/* ---- the other consumers of the gradient (als.cpp:58-101) ------------------- */

/* mttkrp_direct's charge (mttkrp.cpp:29-54 with skip_kron_column, kron.cpp:85-93). */
static uint64_t direct_charge(int N, const ora_index* dims, ora_index R, int n) {
  ora_index J[MAXN + 1];
  prefix_products(N, dims, J);
  uint64_t s = (uint64_t)J[N];
  for (int k = 2; k <= n - 1; ++k) s += (uint64_t)J[k];
  for (int k = n + 1; k <= N; ++k) s += (uint64_t)(J[k] / dims[n - 1]);
  return (uint64_t)R * s;
}

/* als_sweep_direct (als.cpp:58-67): direct MTTKRP + update per mode of order. */
int ora_als_sweep_direct(int N, const ora_index* dims, const double* y, ora_index R,
                         double* const* factors, const int* order, int norder, double rtol,
                         uint64_t* counter) {
  for (int i = 0; i < norder; ++i) {
    const int n = order[i];
    if (n < 1 || n > N) return ORA_INDEX;
    const ora_index I = dims[n - 1];
    double* m = (double*)malloc((size_t)(I * R) * sizeof(double));
    double* upd = (double*)malloc((size_t)(I * R) * sizeof(double));
    ora_brute_mttkrp(N, dims, y, R, (const double* const*)factors, n, m);
    if (counter) *counter += direct_charge(N, dims, R, n);
    const int st = ora_als_update_mode(N, dims, R, m, (const double* const*)factors, n, rtol, upd);
    if (st == ORA_OK) memcpy(factors[n - 1], upd, (size_t)(I * R) * sizeof(double));
    free(m);
    free(upd);
    if (st != ORA_OK) return st;
  }
  return ORA_OK;
}

typedef struct {
  int N;
  const ora_index* dims;
  ora_index R;
  double* const* factors;
  double eps;
} mu_ctx;

/* mu_sweep's hook (als.cpp:84-90): A <- A .* G ./ (A W + eps), W from the current factors. */
static void mu_hook(void* user, int n, const double* g, ora_index rows, ora_index R) {
  mu_ctx* c = (mu_ctx*)user;
  double* w = (double*)malloc((size_t)(R * R) * sizeof(double));
  ora_gram_hadamard_skip(c->N, c->dims, R, (const double* const*)c->factors, n, w);
  double* a = c->factors[n - 1];
  double* na = (double*)malloc((size_t)(rows * R) * sizeof(double));
  for (ora_index col = 0; col < R; ++col)
    for (ora_index i = 0; i < rows; ++i) {
      double den = 0.0;
      for (ora_index k = 0; k < R; ++k) den += a[i + rows * k] * w[k + R * col];
      na[i + rows * col] = a[i + rows * col] * g[i + rows * col] / (den + c->eps);
    }
  memcpy(a, na, (size_t)(rows * R) * sizeof(double));
  free(na);
  free(w);
}

/* mu_sweep (als.cpp:80-91). */
int ora_mu_sweep(int N, const ora_index* dims, const double* y, ora_index R, double* const* factors,
                 double eps, uint64_t* counter, int nthreads) {
  if (eps < 0.0) return ORA_ARG;
  ora_index J[MAXN + 1];
  prefix_products(N, dims, J);
  for (ora_index q = 0; q < J[N]; ++q) /* check_nonnegative (als.cpp:24-30) */
    if (y[q] < 0.0) return ORA_DOMAIN;
  for (int k = 0; k < N; ++k)
    for (ora_index q = 0; q < dims[k] * R; ++q)
      if (factors[k][q] < 0.0) return ORA_DOMAIN;
  mu_ctx c = {N, dims, R, factors, eps};
  double* g[MAXN] = {0};
  for (int k = 0; k < N; ++k) g[k] = (double*)malloc((size_t)(dims[k] * R) * sizeof(double));
  const int st = ora_cp_gradient_all(N, dims, y, R, factors, g, mu_hook, &c, counter, NULL, 0, nthreads);
  for (int k = 0; k < N; ++k) free(g[k]);
  return st;
}

/* gd_step (als.cpp:93-101, kruskal.cpp:83-101): M = all-mode gradient at the
 * pre-step factors, G(n) = M(n) - A(n) W(n), then a(n) += 2 eta G(n) for all n. */
int ora_gd_step(int N, const ora_index* dims, const double* y, ora_index R, double* const* factors,
                double eta, uint64_t* counter, int nthreads) {
  if (!(eta >= 0.0)) return ORA_ARG;
  double* m[MAXN] = {0};
  for (int k = 0; k < N; ++k) m[k] = (double*)malloc((size_t)(dims[k] * R) * sizeof(double));
  const int st = ora_cp_gradient_all(N, dims, y, R, factors, m, NULL, NULL, counter, NULL, 0, nthreads);
  if (st == ORA_OK) {
    double* w = (double*)malloc((size_t)(R * R) * sizeof(double));
    for (int k = 0; k < N; ++k) { /* G(n) in place of M(n), all from the old factors */
      ora_gram_hadamard_skip(N, dims, R, (const double* const*)factors, k + 1, w);
      const ora_index I = dims[k];
      const double* a = factors[k];
      double* gk = m[k];
      for (ora_index col = 0; col < R; ++col)
        for (ora_index i = 0; i < I; ++i) {
          double aw = 0.0;
          for (ora_index q = 0; q < R; ++q) aw += a[i + I * q] * w[q + R * col];
          gk[i + I * col] -= aw;
        }
    }
    free(w);
    for (int k = 0; k < N; ++k)
      for (ora_index q = 0; q < dims[k] * R; ++q) factors[k][q] += 2.0 * eta * m[k][q];
  }
  for (int k = 0; k < N; ++k) free(m[k]);
  return st;
}

/* run(y, init, algo, opts) for every Algorithm (als.cpp:147-210): algo 0 als_direct
 * (order_pivot: fast_update_order, else 1..N), 1 als_fast, 2 mu, 3 gd.  als_fast and
 * mu run in the ascending-sorted frame. */
int ora_run(int N, const ora_index* dims, const double* y, ora_index R, double* const* factors, int algo,
            int order_pivot, int max_iters, double tol, double pinv_rtol, double mu_eps, double gd_eta,
            double* cost_trace, double* rel_trace, uint64_t* mults_trace, int* iters_run, int nthreads) {
  if (max_iters < 1 || tol < 0.0 || pinv_rtol < 0.0 || mu_eps < 0.0) return ORA_ARG;
  if (algo < 0 || algo > 3) return ORA_ARG;
  int perm[MAXN];
  const int wants_sorted = (algo == 1 || algo == 2);
  int identity = 1;
  if (wants_sorted) identity = ora_sort_perm(N, dims, perm, NULL);
  if (identity)
    for (int j = 0; j < N; ++j) perm[j] = j + 1;
  ora_index sd[MAXN], J[MAXN + 1];
  for (int j = 0; j < N; ++j) sd[j] = dims[perm[j] - 1];
  prefix_products(N, sd, J);
  const double* work = y;
  double* yperm = NULL;
  if (!identity) {
    yperm = (double*)malloc((size_t)J[N] * sizeof(double));
    ora_permute(N, dims, y, perm, yperm);
    work = yperm;
  }
  double* sf[MAXN];
  for (int j = 0; j < N; ++j) {
    sf[j] = (double*)malloc((size_t)(sd[j] * R) * sizeof(double));
    memcpy(sf[j], factors[perm[j] - 1], (size_t)(sd[j] * R) * sizeof(double));
  }
  int order[MAXN];
  if (algo == 0) {
    if (order_pivot) ora_fast_update_order(N, sd, order);
    else
      for (int j = 0; j < N; ++j) order[j] = j + 1;
  }
  double yn = 0.0;
  for (ora_index q = 0; q < J[N]; ++q) yn += work[q] * work[q];
  yn = sqrt(yn);
  uint64_t counter = 0;
  double prev = NAN;
  int st = ORA_OK, done = 0;
  for (int it = 1; it <= max_iters; ++it) {
    switch (algo) {
      case 0: st = ora_als_sweep_direct(N, sd, work, R, sf, order, N, pinv_rtol, &counter); break;
      case 1: st = ora_als_sweep_fast(N, sd, work, R, sf, pinv_rtol, &counter, nthreads); break;
      case 2: st = ora_mu_sweep(N, sd, work, R, sf, mu_eps, &counter, nthreads); break;
      default: st = ora_gd_step(N, sd, work, R, sf, gd_eta, &counter, nthreads); break;
    }
    if (st != ORA_OK) break;
    if (mults_trace) mults_trace[it - 1] = counter;
    ++done;
    const double d = ora_cost(N, sd, work, R, (const double* const*)sf, 1000000, nthreads);
    cost_trace[it - 1] = d;
    rel_trace[it - 1] = yn > 0.0 ? sqrt(d) / yn : sqrt(d);
    if (tol > 0.0 && it > 1 && fabs(d - prev) / (prev > 1e-15 ? prev : 1e-15) < tol) break;
    prev = d;
  }
  *iters_run = done;
  for (int j = 0; j < N; ++j) {
    memcpy(factors[perm[j] - 1], sf[j], (size_t)(sd[j] * R) * sizeof(double));
    free(sf[j]);
  }
  free(yperm);
  return st;
}

/* ---- generators ------------------------------------------------------------ */

/* Uniform01 (rng.hpp:9-26): mt19937_64 seeded with mix_seed(seed). */
static uint64_t mix_seed(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

void ora_uniform01_fill(uint64_t seed, ora_index n, double* out) {
  enum { NN = 312, MM = 156 };
  uint64_t mt[NN];
  int mti;
  mt[0] = mix_seed(seed);
  for (mti = 1; mti < NN; ++mti)
    mt[mti] = 6364136223846793005ull * (mt[mti - 1] ^ (mt[mti - 1] >> 62)) + (uint64_t)mti;
  static const uint64_t mag01[2] = {0ull, 0xB5026F5AA96619E9ull};
  const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
  for (ora_index q = 0; q < n; ++q) {
    if (mti >= NN) {
      int i;
      uint64_t x;
      for (i = 0; i < NN - MM; ++i) {
        x = (mt[i] & UM) | (mt[i + 1] & LM);
        mt[i] = mt[i + MM] ^ (x >> 1) ^ mag01[(int)(x & 1ull)];
      }
      for (; i < NN - 1; ++i) {
        x = (mt[i] & UM) | (mt[i + 1] & LM);
        mt[i] = mt[i + (MM - NN)] ^ (x >> 1) ^ mag01[(int)(x & 1ull)];
      }
      x = (mt[NN - 1] & UM) | (mt[0] & LM);
      mt[NN - 1] = mt[MM - 1] ^ (x >> 1) ^ mag01[(int)(x & 1ull)];
      mti = 0;
    }
    uint64_t x = mt[mti++];
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= (x >> 43);
    out[q] = (double)(x >> 11) * 0x1.0p-53;
  }
}

/* Counter-based generator; the product's
 * device generator implements the same formula independently. */
uint64_t ora_hash64(uint64_t seed, uint64_t idx) {
  uint64_t x = seed * 0xD1B54A32D192ED03ull + idx * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

void ora_fill_normal(uint64_t seed, ora_index offset, ora_index n, double* out, int nthreads) {
  const int nth = set_threads(nthreads);
#pragma omp parallel for num_threads(nth) schedule(static)
  for (ora_index q = 0; q < n; ++q) {
    const uint64_t i = (uint64_t)(offset + q);
    const double u1 = ((double)(ora_hash64(seed, 2 * i) >> 11) + 0.5) * 0x1.0p-53;
    const double u2 = (double)(ora_hash64(seed, 2 * i + 1) >> 11) * 0x1.0p-53;
    out[q] = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
  }
}

void ora_fill_upm1_f32(uint64_t seed, ora_index offset, ora_index n, float* out, int nthreads) {
  const int nth = set_threads(nthreads);
#pragma omp parallel for num_threads(nth) schedule(static)
  for (ora_index q = 0; q < n; ++q) {
    const uint64_t h = ora_hash64(seed, (uint64_t)(offset + q));
    out[q] = (float)((int32_t)(h >> 40) - 8388608) * 0x1.0p-23f;
  }
}
