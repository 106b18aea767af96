// cpdgpu.cu — host orchestration and the C-ABI (include/cpdgpu.h).
//
// Drives Algorithm 2 of the reference (cp_gradient_all, mttkrp.cpp:113-253)
// and the fast ALS sweep / driver (als.cpp:69-78, 147-210) on one B200:
//   sort_modes (hoisted, cached per tensor) -> K1 seed contraction(s) ->
//   deterministic partial reduction -> rank-batched recursion tail -> ALS
//   update (on device) / gradients out.
// Everything below the C-ABI is sm_100a device code; there is no CPU fallback.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl.so.2 is opened at run time (cpdgpu_comm_init)

#include "../../include/cpdgpu.h"
#include "kernels.h"

namespace {

using cpdgpu::KRSpec;
using cpdgpu::kMaxModes;

struct Failure : std::exception {
  int code;
  std::string msg;
  Failure(int c, std::string m) : code(c), msg(std::move(m)) {}
  const char* what() const noexcept override { return msg.c_str(); }
};

[[noreturn]] void fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  throw Failure(code, buf);
}

void cuda_check(cudaError_t e, const char* what) {
  if (e == cudaErrorMemoryAllocation) fail(CPDGPU_NO_MEMORY, "%s: %s", what, cudaGetErrorString(e));
  if (e != cudaSuccess) fail(CPDGPU_CUDA_ERROR, "%s: %s", what, cudaGetErrorString(e));
}
#define CK(x) cuda_check((x), #x)

// Device workspace the library itself holds (seed partials, Khatri-Rao operands, operand
// images, padded / sorted copies, tables: everything but the tensors' own values), bytes in
// use and the high-water mark, per process: what FastStats::peak_workspace_doubles
// (mttkrp.cpp:127-131,243) would be for THIS implementation (cpdgpu_device_workspace).
std::atomic<long long> g_ws_cur{0}, g_ws_peak{0};
void ws_add(long long b) {
  const long long now = g_ws_cur.fetch_add(b) + b;
  long long pk = g_ws_peak.load();
  while (now > pk && !g_ws_peak.compare_exchange_weak(pk, now)) {
  }
}

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) {
      cudaFree(p);
      ws_add(-static_cast<long long>(bytes));
    }
  }
  void ensure(size_t b) {
    if (b <= bytes) return;
    if (p) {
      cudaFree(p);
      ws_add(-static_cast<long long>(bytes));
    }
    p = nullptr;
    bytes = 0;
    CK(cudaMalloc(&p, b));
    bytes = b;
    ws_add(static_cast<long long>(b));
  }
  double* d() const { return static_cast<double*>(p); }
};

struct HostBuf {
  void* p = nullptr;
  size_t bytes = 0;
  HostBuf() = default;
  HostBuf(const HostBuf&) = delete;
  HostBuf& operator=(const HostBuf&) = delete;
  ~HostBuf() {
    if (p) cudaFreeHost(p);
  }
  void ensure(size_t b) {
    if (b <= bytes) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
    CK(cudaHostAlloc(&p, b, cudaHostAllocDefault));
    bytes = b;
  }
  double* d() const { return static_cast<double*>(p); }
};

// ---- shape arithmetic (shape.cpp:8-36) ---------------------------------------

std::vector<int64_t> prefix(const std::vector<int64_t>& dims) {
  std::vector<int64_t> J(dims.size() + 1, 1);
  for (size_t k = 0; k < dims.size(); ++k) {
    if (dims[k] < 1)
      fail(CPDGPU_SHAPE_ERROR, "shape: mode %zu has nonpositive extent %lld", k + 1,
           static_cast<long long>(dims[k]));
    int64_t next;
    if (__builtin_mul_overflow(J[k], dims[k], &next))
      fail(CPDGPU_SHAPE_ERROR, "shape: entry count overflows at mode %zu", k + 1);
    J[k + 1] = next;
  }
  return J;
}

// select_pivot (mttkrp.cpp:56-65): max{n : J_n <= K_n}, ties to the larger n.
int select_pivot(const std::vector<int64_t>& dims) {
  const int N = static_cast<int>(dims.size());
  if (N < 2) fail(CPDGPU_ARGUMENT_ERROR, "select_pivot: need an order-2 or higher shape");
  const auto J = prefix(dims);
  int pivot = 0;
  for (int n = 1; n <= N; ++n)
    if (J[n] <= J[N] / J[n]) pivot = n;
  if (pivot == 0)
    fail(CPDGPU_SHAPE_ERROR, "select_pivot: no mode satisfies J_n <= K_n; sort modes first");
  return pivot;
}

// stable ascending sort (mttkrp.cpp:67-90); perm[j] = original mode at sorted j (1-based)
std::vector<int> sort_perm(const std::vector<int64_t>& dims) {
  std::vector<int> perm(dims.size());
  for (size_t j = 0; j < dims.size(); ++j) perm[j] = static_cast<int>(j) + 1;
  std::stable_sort(perm.begin(), perm.end(),
                   [&](int a, int b) { return dims[a - 1] < dims[b - 1]; });
  return perm;
}

bool ascending(const std::vector<int64_t>& dims) {
  for (size_t k = 1; k < dims.size(); ++k)
    if (dims[k] < dims[k - 1]) return false;
  return true;
}

// fast_count_realized (mttkrp.cpp:292-320), ascending dims.
uint64_t count_realized(const std::vector<int64_t>& dims, int64_t R, int n) {
  const int N = static_cast<int>(dims.size());
  const auto J = prefix(dims);
  const int p = select_pivot(dims);
  auto sumj = [&](int lo, int hi, int64_t div) {
    uint64_t t = 0;
    for (int k = std::max(lo, 0); k <= hi; ++k) t += static_cast<uint64_t>(J[k] / div);
    return t;
  };
  auto K = [&](int m) { return static_cast<uint64_t>(J[N] / J[m]); };
  const uint64_t uR = static_cast<uint64_t>(R);
  if (n == p)
    return uR * (static_cast<uint64_t>(J[N]) + sumj(n + 2, N, J[n]) + sumj(2, n - 1, 1) +
                 static_cast<uint64_t>(J[n]));
  if (n == p + 1)
    return uR * (static_cast<uint64_t>(J[N]) + sumj(2, n - 1, 1) + sumj(n + 2, N, J[n]) + K(n - 1));
  if (n < p) return uR * (static_cast<uint64_t>(J[n + 1]) + sumj(2, n - 1, 1) + static_cast<uint64_t>(J[n]));
  return uR * (K(n - 2) + sumj(n + 2, N, J[n]) + K(n - 1));
}

// FastStats::peak_workspace_doubles as the reference tracks it (mttkrp.cpp:127-131,
// 147-243): seeds, Khatri-Rao staging and recursion scratch, outputs excluded.
int64_t reference_peak_workspace(const std::vector<int64_t>& sd, int p, int64_t R) {
  const int N = static_cast<int>(sd.size());
  const auto J = prefix(sd);
  const int64_t Jp = J[p], Kp = J[N] / J[p];
  int64_t live = 0, peak = 0;
  auto track = [&](int64_t d) {
    live += d;
    peak = std::max(peak, live);
  };
  track(Kp * R);
  track(Jp * R);
  track(-Kp * R);
  int64_t scr = std::max<int64_t>(J[p - 1], 1);
  track(scr);
  for (int j = p; j >= 1; --j) {
    track(J[j - 1]);
    track(-J[j - 1]);
  }
  track(-scr);
  track(-Jp * R);
  if (p + 1 <= N) {
    track(Jp * R);
    track(Kp * R);
    track(-Jp * R);
    scr = std::max<int64_t>(J[N] / J[p + 1], 1);
    track(scr);
    for (int j = p + 1; j <= N; ++j) {
      const int64_t t = J[N] / J[j];
      track(t);
      track(-t);
    }
    track(-scr);
    track(-Kp * R);
  }
  return peak;
}

}  // namespace

// ---- objects -----------------------------------------------------------------

struct Plan;

struct cpdgpu_tensor {
  cpdgpu_ctx* ctx = nullptr;
  cpdgpu_dtype dtype = CPDGPU_F64;
  std::vector<int64_t> dims;  // caller's mode order
  int64_t numel = 0;
  void* data = nullptr;
  bool owned = false;
  std::vector<int> perm;      // sorted position -> original mode (1-based)
  bool identity = true;
  void* sorted = nullptr;     // mode-sorted copy (== data when identity)
  bool sorted_ready = false;
  double norm2 = -1.0;
  uint64_t id = 0;
  uint64_t version = 0;              // bumped whenever the values change
  DevBuf yscale;                     // fp32: [float scale | double inv | uint amax] (seed_f32.cu)
  uint64_t scale_version = ~0ull;
  DevBuf yscale8;                    // fp64: int8 seed scale record [2^(46-eY), eY, max|Y|] + scratch
  uint64_t scale8_version = ~0ull;
  double amax8 = -1.0, amean8 = 0.0;
  bool scale8_ok = false;
  size_t elem() const { return dtype == CPDGPU_F64 ? 8 : 4; }
  ~cpdgpu_tensor() {
    if (sorted && sorted != data) {
      cudaFree(sorted);
      ws_add(-static_cast<long long>(numel * static_cast<int64_t>(elem())));
    }
    if (owned && data) cudaFree(data);
  }
};

struct Plan {
  // sorted frame
  int N = 0, p = 0;
  int64_t R = 0;
  std::vector<int64_t> sd, J;
  int64_t Jp = 0, Kp = 0;
  std::vector<int> perm;  // sorted j (0-based) -> original mode (1-based)
  std::vector<int64_t> off_sorted, off_orig;
  int64_t total_factor = 0;
  // K1 chunks over the rank (<= 32 columns per pass)
  struct Chunk {
    int r0, Rc, NT;
    int64_t rpart_off = 0, lpart_off = 0;
    cpdgpu::SeedParams sp;
    std::unique_ptr<DevBuf> KRr, KRl;  // pre-built Khatri-Rao rows [K][LDK], [J][LDK]
    CUtensorMap kmap{};
    bool kmap_ok = false;
    std::unique_ptr<DevBuf> KRr16, KRl16, scales;  // fp32 path: split tiles, [scale 128 | inv 128]
    CUtensorMap kmapL{};                           // KR_l rows for the column-block left pass
    int64_t lc_off = 0;
  };
  std::vector<Chunk> chunks;
  bool lpart_direct = false;  // one row block: the left partial is the seed itself
  // left seed alone (ALS / hook second pass): column-block kernel
  bool use_lc = false;
  int64_t lc_TJ = 256, lc_nCB = 0, lc_nRT = 0, lc_U = 0;
  int lc_P = 0, lc_slots = 0, lc_tab_len = 0, lc_tab_max = 0;
  DevBuf lc_tab, LCpart;
  CUtensorMap ymapL{};
  const void* ymapL_base = nullptr;
  bool raw_frame = false;     // forced pivot: the caller's frame is used unsorted
  bool tma_ok = false;        // Y tiles by 2-D TMA (even leading extent)
  CUtensorMap tmap{};         // bound to the tensor's device address
  const void* tmap_base = nullptr;
  DevBuf Fs, Forig, Gorig, Rpart, Lpart, Rs, Ls, Rtmp, Ltmp, grams, costs, status, norm;
  DevBuf l0_scratch, l0_tickets;  // fused first level: chunk partials, self-resetting tickets
  DevBuf slot_tab;            // CSR of right-partial slots per row block: [nRB + 1] + [slots]
  int slot_tab_ptr_len = 0;
  int slot_tab_max = 0;         // most slots any row block has
  // fp64 fused gradient on the int8 tensor cores (seed_i8.cu): its own 128 x 128
  // tile geometry; gradient_body swaps it in for the seed partials' consumers.
  struct I8 {
    bool ok = false;   // geometry built (one rank chunk, both seeds, even J_p)
    bool on = false;   // tensor_ok && factors_ok: the gradient runs the int8 pass
    bool tensor_ok = false;   // bound tensor passed the range guard and has a TMA view
    bool factors_ok = true;   // the call's factors passed the Khatri-Rao range guard
    const void* guard_fdev = nullptr;  // device factors the last synchronous guard checked
    int N = 0;         // MMA rank block (16 or 32)
    int NL = 0;        // left rank block (24 when R <= 24 < N)
    int64_t nRB = 0, nCT = 0, T = 0;
    int P = 0, slots = 0;
    DevBuf img_r, img_l, w_r, w_l;
    CUtensorMap ymap{};
    const void* ymap_base = nullptr;
    // 128-byte-aligned column copy of Y when J_p * 8 is not a multiple of 128 (per
    // tensor version): the 16-row TMA boxes then stream at full rate
    DevBuf ypad;
    int64_t ld = 0;
    uint64_t ypad_version = ~0ull;
    uint64_t seen_version = ~0ull;  // tensor version of the last int8 gradient
    // swapped with the fp64 geometry while an int8 gradient is recorded
    int TI_s = 128;
    int64_t nRB_s = 0;
    DevBuf tab;
    int tab_len = 0, tab_max = 0;
    bool lpart_direct = false;
    // left partials added in L2 (red.add.f64) into one row-block slot (not in
    // deterministic mode): the tail then reads one partial instead of nRB
    bool lred = false;
  } i8;
  HostBuf hF, hG;
  // fp32 tensors: tcgen05 seed passes (seed_f32.cu), one per side
  bool f32 = false;
  const cpdgpu_tensor* tensor = nullptr;  // the tensor this plan belongs to
  struct F32Pass {
    int64_t nB = 0, nK = 0, U = 0;
    int P = 0, slots = 0, tab_len = 0, tab_max = 0;
    DevBuf tab;  // CSR of partial slots per output block
  };
  F32Pass fr, fl;
  // hook-free fp32 gradients with R <= 64: both seeds in one pass (seed_f32f.cu)
  struct F32Fused {
    bool on = false;
    int64_t nRT = 0, nB = 0, nC = 0, U = 0;
    int P = 0, slots = 0, window = 4;
    int band = 3;  // row tiles per band (2: the image kernel's stacked right product)
    DevBuf tab;  // CSR of right-partial slots per 128-row tile
    int tab_len = 0, tab_max = 0;
    DevBuf krl_img, lpart32;
    // the tensor's fp16 hi / lo operand image (built once per tensor version; the
    // kernel then has no split stage); off when it does not fit in memory
    bool img_on = false, img_failed = false;
    bool lred = false;  // left partials added in L2 (red.add) into one band slot
    void* img = nullptr;
    size_t img_bytes = 0;
    CUtensorMap imap{};
    uint64_t img_version = ~0ull;
    ~F32Fused() {
      if (img) {
        cudaFree(img);
        ws_add(-static_cast<long long>(img_bytes));
      }
    }
  } ff;
  int64_t J8 = 0;               // J_p rounded up to 8 (3-D TMA view)
  DevBuf ypad;                  // padded copy when J_p % 8 != 0
  CUtensorMap ymap_r{}, ymap_l{};
  const void* ymap_base = nullptr;
  uint64_t ypad_version = ~0ull;
  DevBuf gtab;                              // device table of the N output pointers
  cudaGraph_t grad_graph = nullptr;         // hook-free gradient
  cudaGraphExec_t grad_exec = nullptr;
  cudaGraphNode_t prologue_node = nullptr;  // patched per call (inputs / outputs)
  uint64_t grad_graph_launches = 0;
  bool grad_warm = false;
  cudaGraphExec_t als_exec = nullptr;       // one fast ALS sweep
  uint64_t als_graph_launches = 0;
  bool als_warm = false;
  double als_rtol = -1.0;
  const void* graph_ybase = nullptr;       // Y address the recorded graphs read
  ~Plan() { drop_graphs(); }
  // The recorded graphs hold Y's address and its TMA views by value: they are
  // re-recorded whenever either changes (e.g. a re-permuted sorted copy).
  void drop_graphs() {
    if (grad_exec) cudaGraphExecDestroy(grad_exec);
    if (grad_graph) cudaGraphDestroy(grad_graph);
    if (als_exec) cudaGraphExecDestroy(als_exec);
    grad_exec = nullptr;
    grad_graph = nullptr;
    als_exec = nullptr;
    grad_warm = false;
    als_warm = false;
  }

  KRSpec spec(int lo, int hi, int r0) const {  // 1-based sorted modes lo..hi
    KRSpec s{};
    s.n = lo > hi ? 0 : hi - lo + 1;
    for (int k = 0; k < s.n; ++k) {
      const int j = lo - 1 + k;
      s.dims[k] = sd[j];
      s.A[k] = Fs.d() + off_sorted[j] + sd[j] * r0;
    }
    return s;
  }
  double* factor(int j) const { return Fs.d() + off_sorted[j - 1]; }  // sorted 1-based
  int64_t K(int m) const { return J[N] / J[m]; }
};

// Communicator of the sharded gradient: NCCL (in-place all-reduce on the context
// stream) or the caller's host all-reduce.  libnccl.so.2 is dlopen'ed on first
// use, so the library has no link-time NCCL dependency (and shares the process's
// already-loaded NCCL, e.g. torch's, when there is one).
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};
NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("libnccl.so.2 not found: ") + dlerror();
      return a;
    }
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    a.init_rank = reinterpret_cast<decltype(a.init_rank)>(dlsym(h, "ncclCommInitRank"));
    a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
    a.destroy = reinterpret_cast<decltype(a.destroy)>(dlsym(h, "ncclCommDestroy"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.get_unique_id && a.init_rank && a.all_reduce && a.destroy && a.error_string;
    if (!a.ok) a.why = "libnccl.so.2 lacks the expected entry points";
    return a;
  }();
  return api;
}
struct Comm {
  int nranks = 1, rank = 0;
  ncclComm_t nccl = nullptr;
  cpdgpu_allreduce_fn host_fn = nullptr;
  void* user = nullptr;
  DevBuf fbuf;   // packed slab factors (host entry)
  DevBuf xbuf;   // exchange / packed global result (host entry)
  DevBuf lbuf;   // packed slab gradients
  HostBuf hbuf;  // host exchange staging
  ~Comm() {
    if (nccl) nccl_api().destroy(nccl);
  }
};

struct HostStager;
struct cpdgpu_ctx {
  int device = 0;
  std::shared_ptr<HostStager> stager;  // pinned staging buffers for uploads from pageable memory
  std::unique_ptr<Comm> comm;
  int num_sms = 148;
  cudaStream_t own = nullptr, stream = nullptr;
  std::string err;
  bool graphs = true;
  // bitwise-reproducible results (cpdgpu_set_deterministic / CPDGPU_DETERMINISTIC=1)
  bool deterministic = [] {
    const char* e = std::getenv("CPDGPU_DETERMINISTIC");
    return e && e[0] == '1';
  }();
  uint64_t launches = 0;
  int last_seed_path = 0;  // cpdgpu_last_seed_path
  uint64_t next_id = 1;
  std::map<std::tuple<uint64_t, int64_t, int>, std::unique_ptr<Plan>> plans;
  DevBuf scratch;
  bool timing = false;
  std::vector<cudaEvent_t> seed_events;  // pairs around K1 launches
  size_t seed_used = 0;                  // events used by the current call
  // launch timeline (CPDGPU_TIMELINE=1, diagnostics): [slot][entry, wait return, exit]
  bool tl_on = std::getenv("CPDGPU_TIMELINE") != nullptr;
  DevBuf tl;
  int tl_next = 0;
  unsigned long long* tl_ptr() {
    if (!tl_on) return nullptr;
    tl.ensure(64 * 3 * sizeof(unsigned long long));
    return static_cast<unsigned long long*>(tl.p);
  }
  int tl_slot() { return tl_next < 64 ? tl_next++ : 63; }
  // pipeline watchdog (seed kernels): a barrier wait that never completes sets this
  // word (mapped pinned host memory, so the host reads it without a copy) and the
  // kernel unwinds instead of trapping; the next API return reports it
  volatile int* fault_host = nullptr;
  int* fault_dev = nullptr;
  volatile int* guard_host = nullptr;  // int8 factor-range guard result (mapped)
  int* guard_dev = nullptr;
  std::tuple<uint64_t, int64_t, int> i8_last_key{0, 0, 0};  // plan of the last int8 launch
  ~cpdgpu_ctx() {
    for (auto e : seed_events) cudaEventDestroy(e);
    if (fault_host) cudaFreeHost(const_cast<int*>(fault_host));
    if (guard_host) cudaFreeHost(const_cast<int*>(guard_host));
  }
};

namespace {

int set_error(cpdgpu_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

void set_i8_on(Plan& pl);
// kr_digits_kernel found the int8 error budget exceeded (fault code 3000): the plan
// forgets its checked factor buffer, so its next device call re-runs the guard
int i8_budget_fault(cpdgpu_ctx* ctx) {
  auto it = ctx->plans.find(ctx->i8_last_key);
  if (it != ctx->plans.end()) {
    it->second->i8.factors_ok = false;
    it->second->i8.guard_fdev = nullptr;
    set_i8_on(*it->second);
  }
  return set_error(ctx, CPDGPU_NUMERIC_ERROR,
                   "cp_gradient_all: the device factors exceed the int8 pass's error budget "
                   "((max|Y| / mean|Y|) x max_r S_r / rms KR_r > 2^11); this result is invalid and later calls of "
                   "this tensor run the fp64 DMMA pass until the factors pass the guard again");
}

template <typename F>
int guarded(cpdgpu_ctx* ctx, F&& f) {
  try {
    f();
    if (ctx && ctx->fault_host && *ctx->fault_host) {  // a seed kernel's watchdog fired
      const int code = *ctx->fault_host;
      *ctx->fault_host = 0;
      if (code == 3000) return i8_budget_fault(ctx);
      return set_error(ctx, CPDGPU_CUDA_ERROR,
                       "seed pipeline stalled (watchdog code " + std::to_string(code) +
                           "): the kernel unwound, results of the calls since the last check are invalid");
    }
    if (ctx) ctx->err.clear();
    return CPDGPU_OK;
  } catch (const Failure& e) {
    return set_error(ctx, e.code, e.msg);
  } catch (const std::exception& e) {
    return set_error(ctx, CPDGPU_CUDA_ERROR, e.what());
  }
}

void use_device(cpdgpu_ctx* ctx) { CK(cudaSetDevice(ctx->device)); }

void ensure_sorted(cpdgpu_ctx* ctx, cpdgpu_tensor* t) {
  if (t->sorted_ready) return;
  if (t->identity) {
    t->sorted = t->data;
  } else {  // hoisted sort_modes copy (als.cpp:159-165)
    CK(cudaMalloc(&t->sorted, static_cast<size_t>(t->numel) * t->elem()));
    ws_add(static_cast<long long>(t->numel * static_cast<int64_t>(t->elem())));
    ctx->launches += cpdgpu::launch_permute(t->data, t->sorted, static_cast<int>(t->elem()),
                                            static_cast<int>(t->dims.size()), t->dims.data(),
                                            t->perm.data(), ctx->stream);
    CK(cudaGetLastError());
  }
  t->sorted_ready = true;
}

int pick_nt(int64_t Rc) { return static_cast<int>((Rc + 7) / 8); }

// CSR of partial slots per output block for a persistent launch: CTA c owns
// units [c T / P, (c + 1) T / P) of unit = block * nCT + tile, one slot per block.
void build_slot_tab(DevBuf& buf, int64_t nB, int64_t nCT, int64_t T, int P, int slots, int* ptr_len, int* tab_max) {
  std::vector<std::vector<int>> per(static_cast<size_t>(nB));
  for (int64_t c = 0; c < P; ++c) {
    const int64_t a = c * T / P, b = (c + 1) * T / P;
    if (a >= b) continue;
    for (int64_t rb = a / nCT; rb <= (b - 1) / nCT; ++rb)
      per[static_cast<size_t>(rb)].push_back(static_cast<int>(c * slots + (rb - a / nCT)));
  }
  std::vector<int> tab(static_cast<size_t>(nB) + 1, 0);
  int mx = 0;
  for (int64_t rb = 0; rb < nB; ++rb) {
    tab[rb + 1] = tab[rb] + static_cast<int>(per[rb].size());
    mx = std::max(mx, static_cast<int>(per[rb].size()));
  }
  for (auto& v : per) tab.insert(tab.end(), v.begin(), v.end());
  buf.ensure(tab.size() * sizeof(int));
  CK(cudaMemcpy(buf.p, tab.data(), tab.size() * sizeof(int), cudaMemcpyHostToDevice));
  *ptr_len = static_cast<int>(nB) + 1;
  *tab_max = mx;
}

void build_f64_geometry(cpdgpu_ctx* ctx, Plan& pl) {
  const int64_t R = pl.R;
  // K1 geometry
  const int64_t Jp = pl.Jp, Kp = pl.Kp;
  // Row block TI: a multiple of 8 (DMMA fragments); the TMA box is TI + 4 rows
  // (LDY == 4 or 12 mod 16: conflict-free fragment loads for both products).
  // When the columns start on 128-byte lines (J_p % 16 == 0) TI is a multiple of
  // 16 as well, so row blocks never share a line with a neighbour that another
  // CTA streams later (a shared line is fetched from HBM twice); among those the
  // largest TI whose last row block wastes <= 2 % of J_p is taken.
  int ti_max = 208;
  for (int64_t r0 = 0; r0 < R; r0 += 32)
    ti_max = std::min(ti_max, cpdgpu::seed_f64_max_ti(pick_nt(std::min<int64_t>(32, R - r0))));
  int64_t nRB = 0;
  int TI = 0;
  if (Jp % 16 == 0 && Jp >= 96) {
    int best = 0;
    double best_waste = 1e30;
    for (int ti = ti_max / 16 * 16; ti >= 96; ti -= 16) {
      const double waste = static_cast<double>(cpdgpu::ceil_div(Jp, ti) * ti - Jp) / static_cast<double>(Jp);
      if (waste <= 0.02) {
        best = ti;
        break;
      }
      if (waste < best_waste) {
        best_waste = waste;
        best = ti;
      }
    }
    TI = best;
    nRB = cpdgpu::ceil_div(Jp, TI);
  } else {
    if (ti_max % 16 != 8) ti_max -= 8;
    auto ti_for = [](int64_t rows) {
      int64_t ti = (rows + 7) / 8 * 8;
      if (ti % 16 == 0) ti += 8;
      return static_cast<int>(ti);
    };
    nRB = cpdgpu::ceil_div(Jp, ti_max);
    TI = ti_for(cpdgpu::ceil_div(Jp, nRB));
    while (TI > ti_max) {
      ++nRB;
      TI = ti_for(cpdgpu::ceil_div(Jp, nRB));
    }
  }
  pl.tma_ok = (Jp % 2 == 0);
  // TMA box rows TI + 4 (== 12 mod 16): conflict-free fragment loads for both products
  const int LDY = pl.tma_ok ? TI + 4 : TI + 12;
  const int64_t nCT = cpdgpu::ceil_div(Kp, 32);
  const int64_t T = nRB * nCT;
  const int P = static_cast<int>(std::min<int64_t>(ctx->num_sms, T));
  const int64_t per = cpdgpu::ceil_div(T, P);
  const int slots = static_cast<int>(cpdgpu::ceil_div(per, nCT) + 1);
  pl.lpart_direct = (nRB == 1);
  size_t rpart = 0, lpart = 0;
  for (int64_t r0 = 0; r0 < R; r0 += 32) {
    Plan::Chunk c;
    c.r0 = static_cast<int>(r0);
    c.Rc = static_cast<int>(std::min<int64_t>(32, R - r0));
    c.NT = pick_nt(c.Rc);
    auto& sp = c.sp;
    sp = cpdgpu::SeedParams{};
    sp.J = Jp;
    sp.K = Kp;
    sp.R = c.Rc;
    sp.TI = TI;
    sp.LDY = LDY;
    sp.LDK = cpdgpu::seed_ldk(c.NT);
    sp.nRB = nRB;
    sp.nCT = nCT;
    sp.T = T;
    sp.P = P;
    sp.slots = slots;
    sp.use32 = (Jp < (1LL << 31) && Kp < (1LL << 31)) ? 1 : 0;
    const int lk = cpdgpu::seed_ldk(c.NT);
    const size_t ldy = pl.tma_ok ? TI + 4 : TI + 12;
    sp.stages = std::max(cpdgpu::seed_f64_smem_bytes(c.NT, TI, ldy, lk, 3, 3, 0),
                         cpdgpu::seed_f64_smem_bytes(c.NT, TI, ldy, lk, 2, 3, 0)) <= cpdgpu::kSeedSmemLimit
                    ? 3 : 2;
    if (const char* e = std::getenv("CPDGPU_SEED_STAGES")) sp.stages = std::atoi(e);
    c.KRr = std::make_unique<DevBuf>();
    c.KRl = std::make_unique<DevBuf>();
    c.KRr->ensure(static_cast<size_t>(Kp) * lk * sizeof(double));
    c.KRl->ensure(static_cast<size_t>(Jp) * lk * sizeof(double));
    sp.KRr_g = c.KRr->d();
    sp.KRl_g = c.KRl->d();
    c.kmap_ok = pl.tma_ok && cpdgpu::make_tensor_map_2d(&c.kmap, c.KRr->p, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8,
                                                       static_cast<uint64_t>(lk), static_cast<uint64_t>(Kp),
                                                       static_cast<uint64_t>(lk) * 8, static_cast<uint32_t>(lk), 32);
    c.rpart_off = static_cast<int64_t>(rpart);  // per-chunk partials: all chunks run before the reduction
    c.lpart_off = static_cast<int64_t>(lpart);
    rpart += static_cast<size_t>(P) * slots * c.NT * 8 * TI;
    lpart += static_cast<size_t>(nRB) * c.Rc * Kp;
    pl.chunks.push_back(std::move(c));
  }
  pl.Rpart.ensure(rpart * sizeof(double));
  build_slot_tab(pl.slot_tab, nRB, nCT, T, P, slots, &pl.slot_tab_ptr_len, &pl.slot_tab_max);
  // column-block left pass (needs the TMA views of Y and of the KR_l rows)
  if (pl.tma_ok && std::getenv("CPDGPU_NO_LC") == nullptr) {
    pl.lc_nCB = cpdgpu::ceil_div(Kp, pl.lc_TJ);
    pl.lc_nRT = cpdgpu::ceil_div(Jp, 32);
    pl.lc_U = pl.lc_nCB * pl.lc_nRT;
    pl.lc_P = static_cast<int>(std::min<int64_t>(ctx->num_sms, pl.lc_U));
    pl.lc_slots = static_cast<int>(cpdgpu::ceil_div(cpdgpu::ceil_div(pl.lc_U, pl.lc_P), pl.lc_nRT) + 1);
    build_slot_tab(pl.lc_tab, pl.lc_nCB, pl.lc_nRT, pl.lc_U, pl.lc_P, pl.lc_slots, &pl.lc_tab_len, &pl.lc_tab_max);
    size_t lc = 0;
    bool ok = true;
    for (auto& c : pl.chunks) {
      c.lc_off = static_cast<int64_t>(lc);
      lc += static_cast<size_t>(pl.lc_P) * pl.lc_slots * c.NT * 8 * pl.lc_TJ;
      ok = ok && cpdgpu::make_tensor_map_2d(&c.kmapL, c.KRl->p, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8,
                                            static_cast<uint64_t>(c.sp.LDK), static_cast<uint64_t>(Jp),
                                            static_cast<uint64_t>(c.sp.LDK) * 8, static_cast<uint32_t>(c.sp.LDK), 32);
    }
    if (ok) {
      pl.LCpart.ensure(lc * sizeof(double));
      pl.use_lc = true;
    }
  }
  if (!pl.lpart_direct) pl.Lpart.ensure(lpart * sizeof(double));
  // int8 fused seed: one rank chunk of <= 32 columns, both seeds, Y rows 16-byte
  // aligned for the 2-D TMA view
  pl.i8.ok = false;
  // Default: the int8 pass where it measured faster than the DMMA pass on B200 (large
  // tensors whose 128 x 128 tiles waste <= 10 % of either side: c2, c3; not c1's
  // 200-row view); CPDGPU_I8=1 / 0 forces it on / off.
  const char* i8env = std::getenv("CPDGPU_I8");
  const auto waste = [](int64_t L) {
    return static_cast<double>(cpdgpu::ceil_div(L, 128) * 128 - L) / static_cast<double>(L);
  };
  const bool i8_want = i8env ? i8env[0] == '1'
                             : (pl.J[pl.N] >= (int64_t{8} << 20) && waste(Jp) <= 0.10 && waste(Kp) <= 0.10);
  if (i8_want && pl.chunks.size() == 1 && pl.p + 1 <= pl.N && Jp % 2 == 0 &&
      Jp < (1LL << 31) && Kp < (1LL << 31)) {
    Plan::I8& g = pl.i8;
    const Plan::Chunk& c = pl.chunks[0];
    g.N = c.Rc <= 16 ? 16 : 32;
    g.NL = cpdgpu::i8_left_block(g.N, c.Rc);
    g.nRB = cpdgpu::ceil_div(Jp, 128);
    g.nCT = cpdgpu::ceil_div(Kp, 128);
    g.T = g.nRB * g.nCT;
    g.P = static_cast<int>(std::min<int64_t>(ctx->num_sms, g.T));
    g.slots = static_cast<int>(cpdgpu::ceil_div(cpdgpu::ceil_div(g.T, g.P), g.nCT) + 1);
    build_slot_tab(g.tab, g.nRB, g.nCT, g.T, g.P, g.slots, &g.tab_len, &g.tab_max);
    g.TI_s = 128;
    g.nRB_s = g.nRB;
    g.lpart_direct = g.nRB == 1;
    pl.Rpart.ensure(std::max(pl.Rpart.bytes, static_cast<size_t>(g.P) * g.slots * c.NT * 8 * 128 * sizeof(double)));
    if (!g.lpart_direct)
      pl.Lpart.ensure(std::max(pl.Lpart.bytes, static_cast<size_t>(g.nRB) * c.Rc * Kp * sizeof(double)));
    g.img_r.ensure(static_cast<size_t>(g.nCT) * cpdgpu::i8_right_image_bytes(g.N, g.NL));
    g.img_l.ensure(static_cast<size_t>(g.nRB) * cpdgpu::i8_left_image_bytes(g.NL));
    g.w_r.ensure(static_cast<size_t>(g.nCT) * g.N * sizeof(double));
    g.w_l.ensure(static_cast<size_t>(g.nRB) * g.N * sizeof(double));
    g.ok = true;
  }
}

// fp32 tensors: one tcgen05 pass per seed, 64 rank columns per chunk.
void build_f32_geometry(cpdgpu_ctx* ctx, Plan& pl) {
  pl.f32 = true;
  pl.lpart_direct = false;
  const int64_t Jp = pl.Jp, Kp = pl.Kp;
  const int RPc = cpdgpu::seed_f32_rank_cols();
  // Leading dimension of the fp32 view: a multiple of 8 rows for the MMA tiles; for
  // tensors far beyond L2 a multiple of 32 (128-byte column starts), because the
  // right pass's row blocks belong to different CTAs and a 128-byte line straddling
  // two of them is otherwise fetched from HBM twice (measured: +12 % DRAM reads at
  // 300^4).  The padded copy is made once per tensor version (bind_f32_inputs).
  const bool big = static_cast<double>(Jp) * static_cast<double>(Kp) * 4.0 > 1024.0 * 1024.0 * 1024.0;
  pl.J8 = big ? (Jp + 31) / 32 * 32 : (Jp + 7) / 8 * 8;
  auto pass = [&](Plan::F32Pass& f, int64_t rows, int64_t kdim) {
    f.nB = cpdgpu::ceil_div(rows, 128);
    f.nK = cpdgpu::ceil_div(kdim, 64);
    f.U = f.nB * f.nK;
    f.P = static_cast<int>(std::min<int64_t>(ctx->num_sms, f.U));
    f.slots = static_cast<int>(cpdgpu::ceil_div(cpdgpu::ceil_div(f.U, f.P), f.nK) + 1);
    build_slot_tab(f.tab, f.nB, f.nK, f.U, f.P, f.slots, &f.tab_len, &f.tab_max);
  };
  pass(pl.fr, Jp, Kp);
  pass(pl.fl, Kp, Jp);
  size_t rpart = 0, lpart = 0;
  for (int64_t r0 = 0; r0 < pl.R; r0 += RPc) {
    Plan::Chunk c;
    c.r0 = static_cast<int>(r0);
    c.Rc = static_cast<int>(std::min<int64_t>(RPc, pl.R - r0));
    c.NT = RPc / 8;
    c.sp = cpdgpu::SeedParams{};
    c.sp.LDK = RPc;
    c.KRr = std::make_unique<DevBuf>();
    c.KRl = std::make_unique<DevBuf>();
    c.KRr16 = std::make_unique<DevBuf>();
    c.KRl16 = std::make_unique<DevBuf>();
    c.scales = std::make_unique<DevBuf>();
    c.KRr->ensure(static_cast<size_t>(Kp) * RPc * sizeof(double));
    c.KRl->ensure(static_cast<size_t>(Jp) * RPc * sizeof(double));
    c.KRr16->ensure(static_cast<size_t>(pl.fr.nK * cpdgpu::seed_f32_tile_bytes()));
    c.KRl16->ensure(static_cast<size_t>(pl.fl.nK * cpdgpu::seed_f32_tile_bytes()));
    c.scales->ensure(4 * RPc * sizeof(double));
    c.rpart_off = static_cast<int64_t>(rpart);
    c.lpart_off = static_cast<int64_t>(lpart);
    rpart += static_cast<size_t>(pl.fr.P) * pl.fr.slots * RPc * 128;
    lpart += static_cast<size_t>(pl.fl.P) * pl.fl.slots * RPc * 128;
    pl.chunks.push_back(std::move(c));
  }
  // fused single pass (hook-free gradients): bands of kA row tiles x 64-column tiles
  Plan::F32Fused& ff = pl.ff;
  static const char* fused_env = std::getenv("CPDGPU_F32_FUSED");
  ff.on = pl.chunks.size() == 1 && pl.p < pl.N && !(fused_env && std::atoi(fused_env) == 0);
  if (ff.on) {
    // bands of 3 row tiles; CPDGPU_F32_BAND=2: bands of 2 with the operand-image kernel's
    // stacked right product (fewer tensor-pipe cycles, 1.5x the left partial traffic:
    // the same time within noise at c5, profiles/r02_f32i_band2.txt)
    static const char* band_env = std::getenv("CPDGPU_F32_BAND");
    static const char* img_env = std::getenv("CPDGPU_F32_IMAGE");
    const bool img_off = img_env && std::atoi(img_env) == 0;
    ff.band = !img_off && band_env && std::atoi(band_env) == 2 ? 2 : cpdgpu::seed_f32f_band_tiles();
    const int kA = ff.band;
    ff.nRT = cpdgpu::ceil_div(Jp, 128);
    ff.nB = cpdgpu::ceil_div(ff.nRT, kA);
    ff.nC = cpdgpu::ceil_div(Kp, 64);
    ff.U = ff.nB * ff.nC;
    ff.P = static_cast<int>(std::min<int64_t>(ctx->num_sms, ff.U));
    ff.slots = static_cast<int>(cpdgpu::ceil_div(cpdgpu::ceil_div(ff.U, ff.P), ff.nC) + 1);
    static const char* win_env = std::getenv("CPDGPU_F32_WINDOW");
    ff.window = win_env && std::atoi(win_env) > 0 ? std::atoi(win_env) : 4;
    std::vector<std::vector<int>> per(static_cast<size_t>(ff.nRT));
    for (int64_t c = 0; c < ff.P; ++c) {
      const int64_t a = c * ff.U / ff.P, b = (c + 1) * ff.U / ff.P;
      if (a >= b) continue;
      for (int64_t band = a / ff.nC; band <= (b - 1) / ff.nC; ++band)
        for (int t = 0; t < kA && band * kA + t < ff.nRT; ++t)
          per[static_cast<size_t>(band * kA + t)].push_back(
              static_cast<int>((c * ff.slots + (band - a / ff.nC)) * kA + t));
    }
    std::vector<int> tab(static_cast<size_t>(ff.nRT) + 1, 0);
    for (int64_t rt = 0; rt < ff.nRT; ++rt) {
      tab[rt + 1] = tab[rt] + static_cast<int>(per[static_cast<size_t>(rt)].size());
      ff.tab_max = std::max(ff.tab_max, static_cast<int>(per[static_cast<size_t>(rt)].size()));
    }
    for (auto& v : per) tab.insert(tab.end(), v.begin(), v.end());
    ff.tab.ensure(tab.size() * sizeof(int));
    CK(cudaMemcpy(ff.tab.p, tab.data(), tab.size() * sizeof(int), cudaMemcpyHostToDevice));
    ff.tab_len = static_cast<int>(ff.nRT) + 1;
    ff.krl_img.ensure(static_cast<size_t>(ff.nRT) * 128 * 128 * 2);
    ff.lpart32.ensure(static_cast<size_t>(ff.nB * ff.nC) * 64 * 64 * sizeof(float));
    rpart = std::max(rpart, static_cast<size_t>(ff.P) * ff.slots * kA * RPc * 128);
  }
  pl.Rpart.ensure(rpart * sizeof(double));
  pl.Lpart.ensure(lpart * sizeof(double));
}

Plan* get_plan(cpdgpu_ctx* ctx, cpdgpu_tensor* t, int64_t R, int pivot) {
  auto key = std::make_tuple(t->id, R, pivot);
  auto it = ctx->plans.find(key);
  if (it != ctx->plans.end()) return it->second.get();
  auto holder = std::make_unique<Plan>();
  Plan& pl = *holder;
  pl.N = static_cast<int>(t->dims.size());
  pl.R = R;
  pl.tensor = t;
  pl.raw_frame = pivot > 0;
  if (pl.raw_frame) {  // slab shards: the caller's (global, sorted) frame as is
    pl.perm.resize(pl.N);
    for (int j = 0; j < pl.N; ++j) pl.perm[j] = j + 1;
  } else {
    pl.perm = t->perm;
  }
  pl.sd.resize(pl.N);
  for (int j = 0; j < pl.N; ++j) pl.sd[j] = t->dims[pl.perm[j] - 1];
  pl.J = prefix(pl.sd);
  pl.p = pivot > 0 ? pivot : select_pivot(pl.sd);
  if (pl.p < 1 || pl.p > pl.N) fail(CPDGPU_ARGUMENT_ERROR, "pivot %d outside 1..%d", pl.p, pl.N);
  pl.Jp = pl.J[pl.p];
  pl.Kp = pl.J[pl.N] / pl.Jp;
  pl.off_sorted.resize(pl.N);
  pl.off_orig.resize(pl.N);
  int64_t off = 0;
  for (int m = 0; m < pl.N; ++m) {
    pl.off_orig[m] = off;
    off += t->dims[m] * R;
  }
  pl.total_factor = off;
  off = 0;
  for (int j = 0; j < pl.N; ++j) {
    pl.off_sorted[j] = off;
    off += pl.sd[j] * R;
  }
  const size_t fbytes = static_cast<size_t>(pl.total_factor) * sizeof(double);
  pl.Fs.ensure(fbytes);
  pl.Forig.ensure(fbytes);
  pl.Gorig.ensure(fbytes);
  pl.hF.ensure(fbytes);
  pl.hG.ensure(fbytes);

  if (t->dtype == CPDGPU_F32)
    build_f32_geometry(ctx, pl);
  else
    build_f64_geometry(ctx, pl);
  const int64_t Jp = pl.Jp, Kp = pl.Kp;
  pl.Rs.ensure(static_cast<size_t>(Jp * R) * sizeof(double));
  pl.Ls.ensure(static_cast<size_t>(Kp * R) * sizeof(double));
  pl.Rtmp.ensure(static_cast<size_t>(Jp * R) * sizeof(double));
  pl.Ltmp.ensure(static_cast<size_t>(Kp * R) * sizeof(double));
  pl.grams.ensure(static_cast<size_t>(pl.N) * R * R * sizeof(double));
  pl.gtab.ensure(kMaxModes * sizeof(double*));
  pl.status.ensure(sizeof(int) * 4);
  pl.norm.ensure(sizeof(double) * 4);
  Plan* raw = holder.get();
  ctx->plans.emplace(key, std::move(holder));
  return raw;
}

// Operand image layout of the fused fp32 seed: 64-row chunks of the columns side
// by side (CPDGPU_F32_IMG_CHUNK=1) or whole columns (0)
int f32_image_chunked() {
  static const int v = [] {
    const char* e = std::getenv("CPDGPU_F32_IMG_CHUNK");
    return e ? (std::atoi(e) != 0 ? 1 : 0) : 1;
  }();
  return v;
}

// fp32: power-of-two Y scale (cached per tensor version), then either the fp16
// operand image (hook-free gradients on the fused pass: the only view that pass
// reads) or the split passes' view: rows padded to J8 when needed and the two 3-D
// TMA maps.  Each is built lazily, once per tensor version, eagerly (outside any
// graph capture): a fused-gradient caller never makes the padded copy (at 300^4
// that is 32 GB of HBM and a 29 ms copy the fused pass would not read).
void bind_f32_inputs(cpdgpu_ctx* ctx, Plan& pl, cpdgpu_tensor* t, bool fused_gradient) {
  const float* src = static_cast<const float*>(pl.raw_frame ? t->data : t->sorted);
  if (t->scale_version != t->version) {
    t->yscale.ensure(32);
    char* b = static_cast<char*>(t->yscale.p);
    ctx->launches += cpdgpu::launch_y_scale(static_cast<const float*>(t->data), t->numel,
                                            reinterpret_cast<unsigned int*>(b + 16), reinterpret_cast<float*>(b),
                                            reinterpret_cast<double*>(b + 8), ctx->num_sms, ctx->stream);
    CK(cudaGetLastError());
    t->scale_version = t->version;
  }
  if (pl.ff.on && fused_gradient) {  // operand image for the fused seed (CPDGPU_F32_IMAGE=0: split in the kernel)
    static const char* img_env = std::getenv("CPDGPU_F32_IMAGE");
    Plan::F32Fused& ff = pl.ff;
    if (!ff.img && !ff.img_failed && !(img_env && std::atoi(img_env) == 0)) {
      const size_t bytes = static_cast<size_t>(2 * cpdgpu::f16_image_ld(pl.Jp) * pl.Kp) * 2;
      if (cudaMalloc(&ff.img, bytes) != cudaSuccess) {
        cudaGetLastError();  // out of memory: the split-in-kernel path (bands of 3) or two passes
        ff.img = nullptr;
        ff.img_failed = true;
      } else if (!cpdgpu::make_tensor_map_f16_image(&ff.imap, ff.img, pl.Jp, pl.Kp, f32_image_chunked())) {
        cudaFree(ff.img);
        ff.img = nullptr;
        ff.img_failed = true;
      } else {
        ff.img_bytes = bytes;
        ws_add(static_cast<long long>(bytes));
      }
    }
    ff.img_on = ff.img != nullptr;
    if (ff.img_on && ff.img_version != t->version) {
      ctx->launches += cpdgpu::launch_build_f16_image(src, pl.Jp, pl.Jp, pl.Kp, static_cast<const float*>(t->yscale.p),
                                                      ff.img, ctx->num_sms, f32_image_chunked(), ctx->stream);
      CK(cudaGetLastError());
      ff.img_version = t->version;
    }
    if (ff.img_on) {
      // left partials: summed in L2 by red.add (fast; the fp32 addition order varies
      // run to run) unless the context asks for bitwise-reproducible results
      const bool lred = !ctx->deterministic;
      if (lred != ff.lred) pl.drop_graphs();
      ff.lred = lred;
      return;
    }
  }
  const void* base = src;
  if (pl.J8 != pl.Jp) {
    if (pl.ypad_version != t->version || !pl.ypad.p) {
      pl.ypad.ensure(static_cast<size_t>(pl.J8 * pl.Kp) * sizeof(float));
      ctx->launches += cpdgpu::launch_pad_rows_f32(src, static_cast<float*>(pl.ypad.p), pl.Jp, pl.J8, pl.Kp,
                                                   ctx->num_sms, ctx->stream);
      CK(cudaGetLastError());
      pl.ypad_version = t->version;
    }
    base = pl.ypad.p;
  }
  if (pl.ymap_base != base) {
    if (!cpdgpu::make_tensor_map_y32(&pl.ymap_r, base, pl.J8, pl.Kp, 0) ||
        !cpdgpu::make_tensor_map_y32(&pl.ymap_l, base, pl.J8, pl.Kp, 1))
      fail(CPDGPU_ARGUMENT_ERROR, "cp_gradient_all: fp32 tensor view not addressable by TMA");
    pl.ymap_base = base;
  }
}

void set_i8_on(Plan& pl) {
  const bool on = pl.i8.tensor_ok && pl.i8.factors_ok;
  if (on != pl.i8.on) pl.drop_graphs();  // the recorded gradient used the other seed path
  pl.i8.on = on;
}

// int8 fused seed: the tensor's scale record (cached per tensor version), the
// range guard and the swizzled TMA view.  Digits are scaled to max |Y|, so the
// path is kept to tensors whose largest entry is within 2^12 of their mean
// magnitude (a wider range would cost the typical entries precision) and that
// hold no Inf / NaN; everything else runs the fp64 DMMA pass.
void bind_i8(cpdgpu_ctx* ctx, Plan& pl, cpdgpu_tensor* t, const void* ybase) {
  if (t->scale8_version != t->version) {
    t->yscale8.ensure(32 + 16 * static_cast<size_t>(cpdgpu::y_scale_f64_blocks(t->numel, ctx->num_sms)));
    double* rec = t->yscale8.d();
    ctx->launches += cpdgpu::launch_y_scale_f64(static_cast<const double*>(ybase), t->numel, rec + 4, rec,
                                                ctx->num_sms, ctx->stream);
    double h[4] = {0, 0, 0, 0};
    CK(cudaMemcpyAsync(h, rec, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    t->amax8 = h[2];
    t->amean8 = t->numel > 0 ? h[3] / static_cast<double>(t->numel) : 0.0;
    // the digit scale 2^(46 - eY) must be a finite normal double
    t->scale8_ok = std::isfinite(h[0]) && h[0] >= 0x1p-1000;
    t->scale8_version = t->version;
  }
  bool on = t->scale8_ok && std::isfinite(t->amax8) && std::isfinite(t->amean8) &&
            (t->amax8 == 0.0 || t->amax8 <= 4096.0 * t->amean8);
  // columns whose starts are not 128-byte aligned (c3: 2744 rows) stream from a
  // padded copy made once per tensor version (CPDGPU_I8_PAD=0 reads Y in place) --
  // from the SECOND gradient on the same values on: the copy costs a pass over Y
  // (0.26 ms at c3) and saves 4 us per gradient, so values used once are read in place
  // (CPDGPU_I8_PAD=2 pads at once)
  static const char* pad_env = std::getenv("CPDGPU_I8_PAD");
  static const int pad_mode = pad_env ? std::atoi(pad_env) : 1;
  const bool fresh = pl.i8.seen_version != t->version;
  pl.i8.seen_version = t->version;
  const void* view = ybase;
  pl.i8.ld = pl.Jp;
  if (on && (pl.Jp * 8) % 128 != 0 && pad_mode != 0 && (!fresh || pad_mode == 2)) {
    const int64_t ld = cpdgpu::ceil_div(pl.Jp, 16) * 16;
    if (!pl.i8.ypad.p || pl.i8.ypad_version != t->version) {
      pl.i8.ypad.ensure(static_cast<size_t>(ld * pl.Kp) * sizeof(double));
      ctx->launches += cpdgpu::launch_pad_rows_f64(static_cast<const double*>(ybase), pl.i8.ypad.d(), pl.Jp, ld, pl.Kp,
                                                   ctx->num_sms, ctx->stream);
      CK(cudaGetLastError());
      pl.i8.ypad_version = t->version;
    }
    view = pl.i8.ypad.p;
    pl.i8.ld = ld;
  }
  if (on && pl.i8.ymap_base != view) {
    // L2 promotion of the 16-row boxes: 256 B (default) or CPDGPU_I8_PROMO = 0 / 64 / 128
    static const char* promo_env = std::getenv("CPDGPU_I8_PROMO");
    const int promo = promo_env ? std::atoi(promo_env) : 256;
    on = cpdgpu::make_tensor_map_2d(&pl.i8.ymap, view, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8,
                                    static_cast<uint64_t>(pl.Jp), static_cast<uint64_t>(pl.Kp),
                                    static_cast<uint64_t>(pl.i8.ld) * 8, 16, 128, true, promo);
    pl.i8.ymap_base = on ? view : nullptr;
    pl.drop_graphs();  // a recorded gradient holds the old map (in-place <-> padded view)
  }
  pl.i8.tensor_ok = on;
  const bool lred = !ctx->deterministic && pl.i8.nRB > 1;
  if (lred != pl.i8.lred) pl.drop_graphs();
  pl.i8.lred = lred;
  set_i8_on(pl);
}

// int8 range guard for the call's factors.  The pass holds every product to ~2^-47
// max|Y| S_r absolute (48-bit digits of Y scaled by max|Y| and of each Khatri-Rao
// column by S_r = prod_m max_i |A_m[i, r]|, kr_digits_kernel; 21 of 36 digit
// pairs), while a gradient entry is ~ rms(Y) rms(KR_r) per term, so the relative
// error is ~2^-47 (max|Y| / mean|Y|) (S_r / rms KR_r) with rms KR_r =
// prod_m rms_i A_m[i, r] (mean |Y| <= rms |Y|: conservative).  The pass runs only
// while that product stays <= 2^11 (<= ~1.5e-11, under the 1e-10 gate): N(0,1)
// data sits near 2^7 (c2 ~110, c3 ~60).  Otherwise, and for non-finite factors,
// the call runs the fp64 DMMA pass (kron.cpp:54-68 products, mttkrp.cpp:160,207).
constexpr double kI8ErrorBudget = 2048.0;
double i8_factor_limit(const cpdgpu_tensor* t) {
  return t->amax8 > 0.0 ? kI8ErrorBudget * t->amean8 / t->amax8 : kI8ErrorBudget;
}
bool i8_factors_ok_host(const Plan& pl, const double* const* mode_factors, bool caller_order, double limit) {
  for (int side = 0; side < 2; ++side) {
    const int lo = side == 0 ? pl.p + 1 : 1, hi = side == 0 ? pl.N : pl.p;
    for (int64_t r = 0; r < pl.R; ++r) {
      double ratio = 1.0;
      for (int j = lo; j <= hi; ++j) {
        const int m = caller_order ? pl.perm[j - 1] - 1 : j - 1;
        const int64_t I = pl.sd[j - 1];
        const double* col = mode_factors[m] + I * r;
        double mx = 0.0, ss = 0.0;
        for (int64_t i = 0; i < I; ++i) {
          const double a = std::abs(col[i]);
          if (!std::isfinite(a)) return false;
          mx = std::max(mx, a);
          ss += a * a;
        }
        if (mx == 0.0) {  // a zero column: its Khatri-Rao column is exactly 0
          ratio = 0.0;
          break;
        }
        ratio *= mx / std::sqrt(ss / static_cast<double>(I));
      }
      if (!(ratio <= limit)) return false;
    }
  }
  return true;
}

KRSpec spec_over(const Plan& pl, const double* base, bool orig, int lo, int hi, int r0);

// The same guard on device-resident factors (the packed caller-order buffer of the
// device entry points): one tiny kernel into mapped host memory and a stream sync,
// paid only by calls that would otherwise take the int8 pass.
bool i8_factors_ok_device(cpdgpu_ctx* ctx, const Plan& pl, const double* fdev, double limit) {
  *ctx->guard_host = 0;
  ctx->launches += cpdgpu::launch_i8_factor_guard(spec_over(pl, fdev, true, pl.p + 1, pl.N, 0),
                                                  spec_over(pl, fdev, true, 1, pl.p, 0), static_cast<int>(pl.R),
                                                  limit, ctx->guard_dev, ctx->stream);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(ctx->stream));
  return *ctx->guard_host == 0;
}

void i8_apply_factor_guard(Plan& pl, bool ok) {
  pl.i8.factors_ok = ok;
  set_i8_on(pl);
}

// Device entry points: the synchronous guard runs when the factor buffer is new to
// the plan; repeated calls on the same buffer rely on the device's own check
// (kr_digits_kernel, fault code 3000), which turns a later out-of-budget call into a
// reported error rather than a silently inaccurate result and sends the plan back
// through the synchronous guard.
void i8_device_guard(cpdgpu_ctx* ctx, Plan& pl, const double* fdev, const cpdgpu_tensor* t) {
  if (!pl.i8.tensor_ok || fdev == pl.i8.guard_fdev) return;
  i8_apply_factor_guard(pl, i8_factors_ok_device(ctx, pl, fdev, i8_factor_limit(t)));
  pl.i8.guard_fdev = fdev;
}

// fused_gradient: the caller runs a hook-free all-mode gradient (the fp32 fused
// pass reads the operand image, not the split passes' view)
void bind_seed_inputs(cpdgpu_ctx* ctx, Plan& pl, cpdgpu_tensor* t, bool fused_gradient = false) {
  if (pl.f32) {
    bind_f32_inputs(ctx, pl, t, fused_gradient);
    // a recorded gradient follows the view it read (the image buffer is stable)
    const void* gb = fused_gradient && pl.ff.img_on ? pl.ff.img : pl.ymap_base;
    if (pl.graph_ybase != gb) {
      pl.drop_graphs();
      pl.graph_ybase = gb;
    }
    return;
  }
  const void* ybase = pl.raw_frame ? t->data : t->sorted;
  if (pl.graph_ybase != ybase) {
    pl.drop_graphs();
    pl.graph_ybase = ybase;
  }
  if (pl.use_lc && pl.ymapL_base != ybase) {
    if (!cpdgpu::make_tensor_map_2d(&pl.ymapL, ybase, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8,
                                    static_cast<uint64_t>(pl.Jp), static_cast<uint64_t>(pl.Kp),
                                    static_cast<uint64_t>(pl.Jp) * 8, 16, static_cast<uint32_t>(pl.lc_TJ), true))
      pl.use_lc = false;
    else
      pl.ymapL_base = ybase;
  }
  bool tma = pl.tma_ok;
  if (tma && pl.tmap_base != ybase) {
    // no 256 B L2 promotion for Y: row-block starts are not line aligned and the
    // promoted neighbour lines belong to another CTA's (later) tiles
    tma = cpdgpu::make_tensor_map_2d(&pl.tmap, ybase, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8,
                                     static_cast<uint64_t>(pl.Jp), static_cast<uint64_t>(pl.Kp),
                                     static_cast<uint64_t>(pl.Jp) * 8,
                                     static_cast<uint32_t>(pl.chunks[0].sp.TI + 4), 32, false, false);
    pl.tmap_base = tma ? ybase : nullptr;
  }
  tma = tma && pl.tmap_base == ybase;
  for (auto& c : pl.chunks) {
    c.sp.use_tma = (tma && c.kmap_ok) ? 1 : 0;
    c.sp.LDY = c.sp.use_tma ? c.sp.TI + 4 : c.sp.TI + 12;
    c.sp.Y = static_cast<const double*>(ybase);
    c.sp.left = pl.spec(1, pl.p, c.r0);
    c.sp.right = pl.spec(pl.p + 1, pl.N, c.r0);
    c.sp.Rpart = pl.Rpart.d() + c.rpart_off;
    c.sp.Lpart = pl.lpart_direct ? pl.Ls.d() + static_cast<int64_t>(c.r0) * pl.Kp : pl.Lpart.d() + c.lpart_off;
  }
  if (pl.i8.ok) bind_i8(ctx, pl, t, ybase);
}

// Tests only: CPDGPU_FORCE_STALL=1 makes the next seed launches stall on purpose so
// the watchdog path (fault word, no trap) can be exercised; read per launch.
int force_stall() {
  const char* e = std::getenv("CPDGPU_FORCE_STALL");
  return e && std::atoi(e) != 0 ? 1 : 0;
}
// CPDGPU_WATCHDOG=1: the seed kernels' bounded-wait build (a stuck pipeline is
// reported as CPDGPU_CUDA_ERROR and unwinds; costs 5-30 % on the int8 pass, so off
// by default); read per launch
int watchdog_on(int stall) {
  const char* e = std::getenv("CPDGPU_WATCHDOG");
  return stall || (e && std::atoi(e) != 0) ? 1 : 0;
}

// ---- K1 launches ---------------------------------------------------------------
cudaEvent_t seed_event(cpdgpu_ctx* ctx) {
  if (ctx->seed_used == ctx->seed_events.size()) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    ctx->seed_events.push_back(e);
  }
  return ctx->seed_events[ctx->seed_used++];
}

// K1 seed contraction(s).  mode 1: right seed, 2: left seed, 3: both (one HBM pass).
// The Khatri-Rao rows must already be in the chunks' KRr / KRl buffers.
// fp32 seeds: Khatri-Rao column scales and split tiles from the sorted factors
// (Fs), then one tcgen05 pass per requested side.
void run_seeds_f32(cpdgpu_ctx* ctx, Plan& pl, int mode, const cpdgpu_tensor* t) {
  cudaStream_t s = ctx->stream;
  const int RPc = cpdgpu::seed_f32_rank_cols();
  const char* yb = static_cast<const char*>(t->yscale.p);
  if (mode == 3 && pl.ff.on) {  // both seeds in one pass over Y
    Plan::Chunk& c = pl.chunks[0];
    double* sc = c.scales->d();
    // scales, right B tiles and the KRl^T image straight from the sorted factors
    ctx->launches += cpdgpu::launch_kr_fused_operands(pl.spec(pl.p + 1, pl.N, c.r0), pl.Kp, pl.spec(1, pl.p, c.r0),
                                                      pl.Jp, c.Rc, sc, sc + 2 * RPc, c.KRr16->p, pl.ff.krl_img.p, pl.ff.img_on ? 1 : 0,
                                                      s);
    cpdgpu::Seed32FParams q{};
    q.kr_tiles = static_cast<const unsigned char*>(c.KRr16->p);
    q.krl_img = pl.ff.krl_img.p;
    q.scale_y = reinterpret_cast<const float*>(yb);
    q.inv_scale_y = reinterpret_cast<const double*>(yb + 8);
    q.inv_scale_kr = sc + 2 * RPc;
    q.rpart = pl.Rpart.d();
    q.lpart = static_cast<float*>(pl.ff.lpart32.p);
    q.nRT = pl.ff.nRT;
    q.nC = pl.ff.nC;
    q.units = pl.ff.U;
    q.P = pl.ff.P;
    q.slots = pl.ff.slots;
    q.window = pl.ff.window;
    q.band_tiles = pl.ff.band;
    static const char* m64_env = std::getenv("CPDGPU_F32_LEFT_M64");
    q.left_m64 = m64_env ? (std::atoi(m64_env) != 0 ? 1 : 0) : 1;
    static const char* knob_env = std::getenv("CPDGPU_F32F_KNOBS");
    q.knobs = knob_env ? std::atoi(knob_env) : 0;
    if (pl.ff.img_on && pl.ff.lred) {  // one band slot, summed in L2 by the drains
      q.knobs |= 512;
      CK(cudaMemsetAsync(pl.ff.lpart32.p, 0, static_cast<size_t>(pl.ff.nC) * 64 * 64 * sizeof(float), s));
    }
    q.fault = ctx->fault_dev;
    q.stall = force_stall();
    q.watchdog = watchdog_on(q.stall);
    static const bool trace = std::getenv("CPDGPU_SEED_TRACE") != nullptr;
    DevBuf tb;
    if (trace && pl.ff.img_on) {
      tb.ensure(static_cast<size_t>(q.P) * 16 * 8 * 8);
      CK(cudaMemsetAsync(tb.p, 0, tb.bytes, s));
      q.trace = static_cast<unsigned long long*>(tb.p);
    }
    if (ctx->timing) CK(cudaEventRecord(seed_event(ctx), s));
    ctx->launches += pl.ff.img_on ? cpdgpu::launch_seed_f32i(q, &pl.ff.imap, s)
                                  : cpdgpu::launch_seed_f32f(q, &pl.ymap_r, s);
    if (q.trace) {
      std::vector<unsigned long long> h(static_cast<size_t>(q.P) * 128);
      CK(cudaMemcpyAsync(h.data(), tb.p, tb.bytes, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      double a[16][8] = {};
      for (int c = 0; c < q.P; ++c)
        for (int w = 0; w < 16; ++w)
          for (int k = 0; k < 8; ++k) a[w][k] += static_cast<double>(h[(static_cast<size_t>(c) * 16 + w) * 8 + k]) / q.P;
      std::fprintf(stderr, "[f32i trace] avg cycles per CTA (%.0f tiles): mma total %.0f wait full %.0f lempty %.0f "
                   "kfull %.0f rempty %.0f kl_full %.0f issue %.0f | left mma total %.0f wait full %.0f lempty %.0f "
                   "kl_full %.0f issue %.0f | producer total %.0f wait empty %.0f | drain0 "
                   "total %.0f rfull %.0f lfull %.0f | drain8 rfull %.0f lfull %.0f\n", a[13][7], a[13][6], a[13][0], a[13][1],
                   a[13][2], a[13][3], a[13][4], a[13][5], a[15][6], a[15][0], a[15][1], a[15][4], a[15][5], a[12][6],
                   a[12][0], a[0][6], a[0][0], a[0][1], a[8][0], a[8][1]);
    }
    if (ctx->timing) CK(cudaEventRecord(seed_event(ctx), s));
    return;
  }
  for (auto& c : pl.chunks) {
    double* sc = c.scales->d();
    ctx->launches += cpdgpu::launch_kr_scale(pl.spec(pl.p + 1, pl.N, c.r0), pl.spec(1, pl.p, c.r0), c.Rc, sc,
                                             sc + 2 * RPc, s);
    if (mode & 1)
      ctx->launches += cpdgpu::launch_kr_split(c.KRr->d(), pl.Kp, RPc, sc, c.KRr16->p, s);
    if (mode & 2)
      ctx->launches += cpdgpu::launch_kr_split(c.KRl->d(), pl.Jp, RPc, sc + RPc, c.KRl16->p, s);
    for (int side = 0; side < 2; ++side) {
      if (!(mode & (1 << side))) continue;
      const Plan::F32Pass& f = side ? pl.fl : pl.fr;
      cpdgpu::Seed32Params q{};
      q.kr_tiles = static_cast<const unsigned char*>(side ? c.KRl16->p : c.KRr16->p);
      q.scale_y = reinterpret_cast<const float*>(yb);
      q.inv_scale_y = reinterpret_cast<const double*>(yb + 8);
      q.inv_scale_kr = sc + 2 * RPc + side * RPc;
      q.part = (side ? pl.Lpart.d() + c.lpart_off : pl.Rpart.d() + c.rpart_off);
      q.nK = f.nK;
      q.units = f.U;
      q.P = f.P;
      q.slots = f.slots;
      static const int chunk_env = std::getenv("CPDGPU_F32_CHUNK") ? std::atoi(std::getenv("CPDGPU_F32_CHUNK")) : 8;
      static const int dbg_env = std::getenv("CPDGPU_F32_DEBUG") ? std::atoi(std::getenv("CPDGPU_F32_DEBUG")) : 0;
      q.chunk = chunk_env > 0 ? chunk_env : 8;
      q.debug = dbg_env;
      static const bool trace = std::getenv("CPDGPU_SEED_TRACE") != nullptr;
      DevBuf tb;
      if (trace) {
        tb.ensure(static_cast<size_t>(q.P) * 10 * 8 * 8);
        CK(cudaMemsetAsync(tb.p, 0, tb.bytes, s));
        q.trace = static_cast<unsigned long long*>(tb.p);
      }
      if (ctx->timing) CK(cudaEventRecord(seed_event(ctx), s));
      ctx->launches += cpdgpu::launch_seed_f32(q, side ? &pl.ymap_l : &pl.ymap_r, side, s);
      if (ctx->timing) CK(cudaEventRecord(seed_event(ctx), s));
      if (trace) {
        std::vector<unsigned long long> h(static_cast<size_t>(q.P) * 80);
        CK(cudaMemcpyAsync(h.data(), tb.p, tb.bytes, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        double a[10][8] = {};
        for (int c = 0; c < q.P; ++c)
          for (int w = 0; w < 10; ++w)
            for (int k = 0; k < 8; ++k) a[w][k] += static_cast<double>(h[(static_cast<size_t>(c) * 10 + w) * 8 + k]) / q.P;
        std::fprintf(stderr, "[f32 trace side %d] avg cycles per CTA: split w0 full %.0f cempty %.0f accfull %.0f split %.0f "
                     "drain %.0f total %.0f | producer empty %.0f total %.0f | mma cfull %.0f kfull %.0f accempty %.0f "
                     "total %.0f\n", side, a[0][0], a[0][1], a[0][2], a[0][4], a[0][5], a[0][3], a[8][0], a[8][3],
                     a[9][1], a[9][2], a[9][0], a[9][3]);
      }
    }
  }
  CK(cudaGetLastError());
}

// Both fp64 seeds in one pass on the int8 tensor cores: Khatri-Rao digit images
// of both sides (one launch, from the sorted factors), then the fused pass.
void run_seeds_i8(cpdgpu_ctx* ctx, Plan& pl) {
  cudaStream_t s = ctx->stream;
  Plan::I8& g = pl.i8;
  Plan::Chunk& c = pl.chunks[0];
  const double* ys = pl.tensor->yscale8.d();
  // the device re-checks the call's error budget with 1 % slack over the host guard
  // (rounding of the two sums never trips it for factors the host passed)
  ctx->launches += cpdgpu::launch_kr_digits(pl.spec(pl.p + 1, pl.N, c.r0), pl.Kp, pl.spec(1, pl.p, c.r0), pl.Jp, c.Rc,
                                            g.N, g.NL, ys, g.img_r.p, g.w_r.d(), g.img_l.p, g.w_l.d(),
                                            pl.tensor->numel, kI8ErrorBudget * 1.01, ctx->fault_dev, s);
  ctx->i8_last_key = std::make_tuple(pl.tensor->id, pl.R, pl.raw_frame ? pl.p : 0);
  cpdgpu::SeedI8Params q{};
  q.J = pl.Jp;
  q.K = pl.Kp;
  q.R = c.Rc;
  q.RP = c.NT * 8;
  q.N = g.N;
  q.NL = g.NL;
  q.nRB = g.nRB;
  q.nCT = g.nCT;
  q.T = g.T;
  q.P = g.P;
  q.slots = g.slots;
  q.img_r = static_cast<const unsigned char*>(g.img_r.p);
  q.img_l = static_cast<const unsigned char*>(g.img_l.p);
  q.w_r = g.w_r.d();
  q.w_l = g.w_l.d();
  q.yscale = ys;
  q.Rpart = pl.Rpart.d() + c.rpart_off;
  static const bool dbg = std::getenv("CPDGPU_I8_DEBUG") != nullptr;
  static DevBuf progress;
  if (dbg) {
    progress.ensure(static_cast<size_t>(g.P) * 16 * sizeof(unsigned));
    CK(cudaMemsetAsync(progress.p, 0, progress.bytes, s));
  }
  q.progress = dbg ? static_cast<unsigned*>(progress.p) : nullptr;
  static const int knobs = std::getenv("CPDGPU_I8_KNOBS") ? std::atoi(std::getenv("CPDGPU_I8_KNOBS")) : 0;
  q.knobs = knobs;
  q.fault = ctx->fault_dev;
  q.stall = force_stall();
  q.watchdog = watchdog_on(q.stall);
  q.Lpart = g.nRB == 1 ? pl.Ls.d() + static_cast<int64_t>(c.r0) * pl.Kp : pl.Lpart.d() + c.lpart_off;
  q.lred = g.lred ? 1 : 0;  // slot 0 zeroed by this gradient's prologue
  // CPDGPU_I8_RHALF=1 (read when the gradient's launches are recorded): the right product as two
  // M = 64 row halves, the first issued while the tile is still being split.  Exact like the
  // default, but measured 1-4 % slower at c2 / c3: it removes the split's wait for the planes and
  // doubles the right product's MMAs, and the pass is then bound by the tensor pipe's operand reads
  // (profiles/r02_i8_rhalf.txt), so it stays opt-in.
  const char* rhalf_env = std::getenv("CPDGPU_I8_RHALF");
  q.rhalf = rhalf_env && std::atoi(rhalf_env) != 0 ? 1 : 0;
  static const bool trace = std::getenv("CPDGPU_SEED_TRACE") != nullptr;
  DevBuf tb;
  if (trace) {
    tb.ensure(static_cast<size_t>(g.P) * 14 * 6 * 8);
    CK(cudaMemsetAsync(tb.p, 0, tb.bytes, s));
    q.trace = static_cast<unsigned long long*>(tb.p);
  }
  if (ctx->timing) CK(cudaEventRecord(seed_event(ctx), s));
  ctx->launches += cpdgpu::launch_seed_i8(q, &g.ymap, s);
  if (ctx->timing) CK(cudaEventRecord(seed_event(ctx), s));
  if (trace) {
    std::vector<unsigned long long> h(static_cast<size_t>(g.P) * 14 * 6);
    CK(cudaMemcpyAsync(h.data(), tb.p, tb.bytes, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    double a[14][6] = {};
    for (int c = 0; c < g.P; ++c)
      for (int w = 0; w < 14; ++w)
        for (int i = 0; i < 6; ++i) a[w][i] += static_cast<double>(h[(static_cast<size_t>(c) * 14 + w) * 6 + i]) / g.P;
    std::fprintf(stderr, "[i8 trace] avg per CTA (%.1f tiles): split w0 raw_full %.0f dig_empty %.0f total %.0f | "
                 "drain w8 accR %.0f accL %.0f total %.0f | mma dig_full %.0f rb_full %.0f accR_empty %.0f "
                 "lb/accL %.0f total %.0f | producer total %.0f\n", a[0][5], a[0][0], a[0][1], a[0][4], a[8][0],
                 a[8][1], a[8][4], a[13][0], a[13][1], a[13][2], a[13][3], a[13][4], a[12][4]);
  }
  CK(cudaGetLastError());
}

// While an int8 gradient is recorded, the seed partials' consumers (reductions,
// fused first level) see the int8 geometry: row blocks of 128, its slot table.
struct I8Geometry {
  Plan& pl;
  bool on;
  explicit I8Geometry(Plan& p) : pl(p), on(p.i8.on) {
    if (on) swap();
  }
  ~I8Geometry() {
    if (on) swap();
  }
  void swap() {
    Plan::Chunk& c = pl.chunks[0];
    std::swap(c.sp.TI, pl.i8.TI_s);
    std::swap(c.sp.nRB, pl.i8.nRB_s);
    std::swap(pl.slot_tab.p, pl.i8.tab.p);
    std::swap(pl.slot_tab.bytes, pl.i8.tab.bytes);
    std::swap(pl.slot_tab_ptr_len, pl.i8.tab_len);
    std::swap(pl.slot_tab_max, pl.i8.tab_max);
    std::swap(pl.lpart_direct, pl.i8.lpart_direct);
  }
};

void run_seeds(cpdgpu_ctx* ctx, Plan& pl, int mode) {
  if (pl.f32) {
    run_seeds_f32(ctx, pl, mode, pl.tensor);
    return;
  }
  cudaStream_t s = ctx->stream;
  static const bool trace = std::getenv("CPDGPU_SEED_TRACE") != nullptr;
  for (auto& c : pl.chunks) {
    if (ctx->timing) CK(cudaEventRecord(seed_event(ctx), s));
    DevBuf tb;
    if (trace) {
      tb.ensure(static_cast<size_t>(c.sp.P) * 9 * 8 * 8);
      CK(cudaMemsetAsync(tb.p, 0, tb.bytes, s));
      c.sp.trace = static_cast<unsigned long long*>(tb.p);
    }
    c.sp.tl = ctx->tl_ptr();
    c.sp.tl_slot = c.sp.tl ? ctx->tl_slot() : 0;
    if (mode == 2 && pl.use_lc) {
      cpdgpu::SeedParams q = c.sp;
      q.TI = static_cast<int>(pl.lc_TJ);
      q.nRB = pl.lc_nCB;
      q.nCT = pl.lc_nRT;
      q.T = pl.lc_U;
      q.P = pl.lc_P;
      q.slots = pl.lc_slots;
      q.stages = 3;
      q.Rpart = pl.LCpart.d() + c.lc_off;
      ctx->launches += cpdgpu::launch_seed_left_cols(q, &pl.ymapL, &c.kmapL, c.NT, s);
    } else {
      ctx->launches += cpdgpu::launch_seed_f64(c.sp, &pl.tmap, &c.kmap, c.NT, mode, s);
    }
    if (ctx->timing) CK(cudaEventRecord(seed_event(ctx), s));
    if (trace) {
      std::vector<unsigned long long> h(static_cast<size_t>(c.sp.P) * 72);
      CK(cudaMemcpyAsync(h.data(), tb.p, tb.bytes, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      c.sp.trace = nullptr;
      double w[9] = {0}, tot[9] = {0}, mx = 0;
      unsigned long long g0 = ~0ull;
      for (int cta = 0; cta < c.sp.P; ++cta) g0 = std::min(g0, h[static_cast<size_t>(cta) * 72 + 1]);
      double pdl[9] = {0}, end[9] = {0}, endmax = 0, entmax = 0;
      for (int cta = 0; cta < c.sp.P; ++cta)
        for (int wp = 0; wp < 9; ++wp) {
          const unsigned long long* e = &h[(static_cast<size_t>(cta) * 9 + wp) * 8];
          w[wp] += e[0];
          tot[wp] += e[2];
          mx = std::max(mx, static_cast<double>(e[2]));
          pdl[wp] += static_cast<double>(e[4] - g0);
          end[wp] += static_cast<double>(e[6] - g0);
          endmax = std::max(endmax, static_cast<double>(e[6] - g0));
          entmax = std::max(entmax, static_cast<double>(e[1] - g0));
        }
      std::fprintf(stderr, "[seed trace mode %d] per-warp avg cycles (wait/total): ", mode);
      for (int wp = 0; wp < 9; ++wp) std::fprintf(stderr, "w%d %.0f/%.0f  ", wp, w[wp] / c.sp.P, tot[wp] / c.sp.P);
      std::fprintf(stderr, "max warp total %.0f\n", mx);
      if (std::getenv("CPDGPU_SEED_TRACE_CTAS")) {  // per-CTA end (max over warps), tiles, first tile
        for (int cta = 0; cta < c.sp.P; ++cta) {
          unsigned long long e = 0;
          for (int wp = 0; wp < 9; ++wp) e = std::max(e, h[(static_cast<size_t>(cta) * 9 + wp) * 8 + 6]);
          const long long t0 = static_cast<long long>(cta) * c.sp.T / c.sp.P;
          std::fprintf(stderr, "cta %d end %.0f tiles %llu t0 %lld rb0 %lld ct0 %lld\n", cta, static_cast<double>(e - g0),
                       h[(static_cast<size_t>(cta) * 9) * 8 + 3], t0, t0 / c.sp.nCT, t0 % c.sp.nCT);
        }
      }
      std::fprintf(stderr, "[seed trace mode %d] ns from first CTA entry: last entry %.0f, pdl return w0 %.0f w8 %.0f, "
                   "end avg w0 %.0f w4 %.0f, last end %.0f\n", mode, entmax, pdl[0] / c.sp.P, pdl[8] / c.sp.P,
                   end[0] / c.sp.P, end[4] / c.sp.P, endmax);
    }
  }
  CK(cudaGetLastError());
}

// ---- prologue and recursion-tail steps -----------------------------------------

// Khatri-Rao spec over sorted modes lo..hi whose factors live at base (packed
// in the caller's mode order when orig, in the sorted order otherwise).
KRSpec spec_over(const Plan& pl, const double* base, bool orig, int lo, int hi, int r0) {
  KRSpec s{};
  s.n = lo > hi ? 0 : hi - lo + 1;
  for (int k = 0; k < s.n; ++k) {
    const int j = lo - 1 + k;
    const int64_t off = orig ? pl.off_orig[pl.perm[j] - 1] : pl.off_sorted[j];
    s.dims[k] = pl.sd[j];
    s.A[k] = base + off + pl.sd[j] * r0;
  }
  return s;
}

// Khatri-Rao rows for the chunks' K1 launches: kr_mask 1 = KR(p+1..N) rows
// (right product), 2 = KR(1..p) rows (left product).
void add_kr_jobs(const Plan& pl, cpdgpu::Prologue& pr, const double* base, bool orig, int kr_mask) {
  for (const auto& c : pl.chunks) {
    if (kr_mask & 1) {
      cpdgpu::KRJob& k = pr.kr[pr.nkr++];
      k.spec = spec_over(pl, base, orig, pl.p + 1, pl.N, c.r0);
      k.L = pl.Kp;
      k.R = c.Rc;
      k.NT = c.NT;
      k.LDK = c.sp.LDK;
      k.out = c.KRr->d();
    }
    if (kr_mask & 2) {
      cpdgpu::KRJob& k = pr.kr[pr.nkr++];
      k.spec = spec_over(pl, base, orig, 1, pl.p, c.r0);
      k.L = pl.Jp;
      k.R = c.Rc;
      k.NT = c.NT;
      k.LDK = c.sp.LDK;
      k.out = c.KRl->d();
    }
  }
}

// Gradient prologue: sorted factors <- fin (caller order), output table <- gout
// (caller order, gout_base + off_orig), Khatri-Rao rows read straight from fin.
cpdgpu::Prologue grad_prologue(const Plan& pl, const double* fin, double* gout_base, int kr_mask) {
  cpdgpu::Prologue pr{};
  pr.N = pl.N;
  pr.fin = fin;
  pr.Fs = pl.Fs.d();
  for (int j = 0; j < pl.N; ++j) {
    pr.src_off[j] = pl.off_orig[pl.perm[j] - 1];
    pr.dst_off[j] = pl.off_sorted[j];
    pr.len[j] = pl.sd[j] * pl.R;
  }
  for (int m = 0; m < pl.N; ++m) pr.gout[m] = gout_base ? gout_base + pl.off_orig[m] : nullptr;
  add_kr_jobs(pl, pr, fin, true, kr_mask);
  return pr;
}

// Khatri-Rao rows only, from the sorted device factors (ALS / hook sweeps).
void launch_kr_from_fs(cpdgpu_ctx* ctx, Plan& pl, int kr_mask) {
  cpdgpu::Prologue pr{};
  pr.N = 0;
  pr.Fs = nullptr;
  add_kr_jobs(pl, pr, pl.Fs.d(), false, kr_mask);
  ctx->launches += cpdgpu::launch_prologue(pr, static_cast<double**>(pl.gtab.p), ctx->num_sms, ctx->stream);
}

void set_gtab(cpdgpu_ctx* ctx, Plan& pl, double* gout_base) {
  cpdgpu::Prologue pr{};
  pr.N = pl.N;
  pr.Fs = nullptr;
  for (int m = 0; m < pl.N; ++m) pr.gout[m] = gout_base + pl.off_orig[m];
  ctx->launches += cpdgpu::launch_prologue(pr, static_cast<double**>(pl.gtab.p), ctx->num_sms, ctx->stream);
}

cpdgpu::TailOp op_base(int type, int R) {
  cpdgpu::TailOp o{};
  o.type = type;
  o.R = R;
  o.out_slot = -1;
  return o;
}

// Seed-partial reductions for the given seed mode.
void add_reduce_ops(const Plan& pl, cpdgpu::TailStep& st, int mode) {
  if (pl.f32 && mode == 3 && pl.ff.on) {  // fused pass: right slots per row tile, left fp32 per band
    const Plan::Chunk& c = pl.chunks[0];
    const Plan::F32Fused& ff = pl.ff;
    cpdgpu::TailOp o = op_base(cpdgpu::kOpReduceRight, c.Rc);
    o.Z = pl.Rpart.d();
    o.B = ff.tab_max >= 16 ? 1 : 0;
    o.M = pl.Jp;
    o.RP = cpdgpu::seed_f32_rank_cols();
    o.TI = 128;
    o.rb_ptr = static_cast<const int*>(ff.tab.p);
    o.slot_list = static_cast<const int*>(ff.tab.p) + ff.tab_len;
    o.out = pl.Rs.d();
    o.ldo = pl.Jp;
    st.op[st.n++] = o;
    return;  // the left partials: launch_reduce_left32 right after the seed
  }
  if (pl.f32) {  // both sides: per-CTA fp64 partial blocks [slot][64][128]
    for (const auto& c : pl.chunks)
      for (int side = 0; side < 2; ++side) {
        if (!(mode & (1 << side))) continue;
        const Plan::F32Pass& f = side ? pl.fl : pl.fr;
        cpdgpu::TailOp o = op_base(cpdgpu::kOpReduceRight, c.Rc);
        o.Z = side ? pl.Lpart.d() + c.lpart_off : pl.Rpart.d() + c.rpart_off;
        o.B = f.tab_max >= 16 ? 1 : 0;
        o.M = side ? pl.Kp : pl.Jp;
        o.RP = cpdgpu::seed_f32_rank_cols();
        o.TI = 128;
        o.rb_ptr = static_cast<const int*>(f.tab.p);
        o.slot_list = static_cast<const int*>(f.tab.p) + f.tab_len;
        o.out = (side ? pl.Ls.d() : pl.Rs.d()) + static_cast<int64_t>(c.r0) * o.M;
        o.ldo = o.M;
        st.op[st.n++] = o;
      }
    return;
  }
  for (const auto& c : pl.chunks) {
    if (mode & 1) {
      cpdgpu::TailOp o = op_base(cpdgpu::kOpReduceRight, c.Rc);
      o.Z = pl.Rpart.d() + c.rpart_off;
      o.B = pl.slot_tab_max >= 16 ? 1 : 0;  // many slots per row: lanes over slots
      o.M = pl.Jp;
      o.RP = c.NT * 8;
      o.TI = c.sp.TI;
      o.rb_ptr = static_cast<const int*>(pl.slot_tab.p);
      o.slot_list = static_cast<const int*>(pl.slot_tab.p) + pl.slot_tab_ptr_len;
      o.out = pl.Rs.d() + static_cast<int64_t>(c.r0) * pl.Jp;
      o.ldo = pl.Jp;
      st.op[st.n++] = o;
    }
    if (mode == 2 && pl.use_lc) {  // column-block partial slots [slot][RP][TJ]
      cpdgpu::TailOp o = op_base(cpdgpu::kOpReduceRight, c.Rc);
      o.Z = pl.LCpart.d() + c.lc_off;
      o.B = pl.lc_tab_max >= 16 ? 1 : 0;
      o.M = pl.Kp;
      o.RP = c.NT * 8;
      o.TI = static_cast<int>(pl.lc_TJ);
      o.rb_ptr = static_cast<const int*>(pl.lc_tab.p);
      o.slot_list = static_cast<const int*>(pl.lc_tab.p) + pl.lc_tab_len;
      o.out = pl.Ls.d() + static_cast<int64_t>(c.r0) * pl.Kp;
      o.ldo = pl.Kp;
      st.op[st.n++] = o;
    } else if ((mode & 2) && !pl.lpart_direct) {
      cpdgpu::TailOp o = op_base(cpdgpu::kOpReduceLeft, c.Rc);
      o.Z = pl.Lpart.d() + c.lpart_off;
      o.M = pl.Kp;
      o.B = pl.i8.on && pl.i8.lred ? 1 : c.sp.nRB;
      o.out = pl.Ls.d() + static_cast<int64_t>(c.r0) * pl.Kp;
      o.ldo = pl.Kp;
      st.op[st.n++] = o;
    }
  }
}

// Right phase at sorted mode j (mttkrp.cpp:165-193), reading R^(j) at cur:
//   extraction  G(j)[b, r] = sum_a R^(j)[a + J_{j-1} b, r] KR(1..j-1)[a, r]   (Eq 3.12)
//   recursion   R^(j-1)[a, r] = sum_b R^(j)[a + J_{j-1} b, r] A_j[b, r]      (Eq 3.20)
void add_right_extract(const Plan& pl, cpdgpu::TailStep& st, int j, const double* cur) {
  cpdgpu::TailOp o = op_base(cpdgpu::kOpContractA, static_cast<int>(pl.R));
  o.Z = cur;
  o.ldz = pl.Jp;
  o.M = pl.J[j - 1];
  o.B = pl.sd[j - 1];
  o.kr = spec_over(pl, pl.Fs.d(), false, 1, j - 1, 0);
  o.out_slot = pl.perm[j - 1] - 1;
  o.ldo = pl.sd[j - 1];
  st.op[st.n++] = o;
}
void add_right_recurse(const Plan& pl, cpdgpu::TailStep& st, int j, const double* cur, double* nxt) {
  cpdgpu::TailOp o = op_base(cpdgpu::kOpContractB, static_cast<int>(pl.R));
  o.Z = cur;
  o.ldz = pl.Jp;
  o.M = pl.J[j - 1];
  o.B = pl.sd[j - 1];
  o.kr = spec_over(pl, pl.Fs.d(), false, j, j, 0);
  o.out = nxt;
  o.ldo = pl.Jp;
  st.op[st.n++] = o;
}
// Left phase at sorted mode j (mttkrp.cpp:212-241), reading L^(j) at cur:
//   extraction  G(j)[b, r] = sum_c L^(j)[b + I_j c, r] KR(j+1..N)[c, r]      (Eq 3.16)
//   recursion   L^(j+1)[c, r] = sum_b L^(j)[b + I_j c, r] A_j[b, r]          (Eq 3.22)
void add_left_extract(const Plan& pl, cpdgpu::TailStep& st, int j, const double* cur) {
  cpdgpu::TailOp o = op_base(cpdgpu::kOpContractB, static_cast<int>(pl.R));
  o.Z = cur;
  o.ldz = pl.Kp;
  o.M = pl.sd[j - 1];
  o.B = pl.K(j);
  o.kr = spec_over(pl, pl.Fs.d(), false, j + 1, pl.N, 0);
  o.out_slot = pl.perm[j - 1] - 1;
  o.ldo = pl.sd[j - 1];
  st.op[st.n++] = o;
}
void add_left_recurse(const Plan& pl, cpdgpu::TailStep& st, int j, const double* cur, double* nxt) {
  cpdgpu::TailOp o = op_base(cpdgpu::kOpContractA, static_cast<int>(pl.R));
  o.Z = cur;
  o.ldz = pl.Kp;
  o.M = pl.sd[j - 1];
  o.B = pl.K(j);
  o.kr = spec_over(pl, pl.Fs.d(), false, j, j, 0);
  o.out = nxt;
  o.ldo = pl.Kp;
  st.op[st.n++] = o;
}

// Point the seed-partial reduction of one side straight at its gradient slot
// (rows x R column-major): used when that seed already is R^(1) or L^(N).
void redirect_to_gradient(const Plan& pl, cpdgpu::TailStep& st, bool right) {
  const double* base = right ? pl.Rs.d() : pl.Ls.d();
  const int64_t rows = right ? pl.Jp : pl.Kp;
  const int m = right ? pl.perm[0] - 1 : pl.perm[pl.N - 1] - 1;
  for (int i = 0; i < st.n; ++i) {
    cpdgpu::TailOp& o = st.op[i];
    if (!o.out || o.out < base || o.out >= base + rows * pl.R) continue;
    o.out_off = o.out - base;  // r0 * rows for the chunk
    o.out = nullptr;
    o.out_slot = m;
    o.ldo = rows;
  }
}

void launch_step(cpdgpu_ctx* ctx, Plan& pl, const cpdgpu::TailStep& st0) {
  cpdgpu::TailStep st = st0;
  st.tl = ctx->tl_ptr();
  if (st.tl) st.tl_slot = ctx->tl_slot();
  ctx->launches += cpdgpu::launch_tail_step(st, static_cast<double* const*>(pl.gtab.p), ctx->num_sms, ctx->stream);
}

// CPDGPU_TIMELINE: reset the stamps before a call, print them after it.
void timeline_reset(cpdgpu_ctx* ctx) {
  if (!ctx->tl_on) return;
  static std::vector<unsigned long long> init = [] {
    std::vector<unsigned long long> v(64 * 3, ~0ull);
    for (int i = 0; i < 64; ++i) v[3 * i + 2] = 0;
    return v;
  }();
  CK(cudaMemcpyAsync(ctx->tl_ptr(), init.data(), init.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice,
                     ctx->stream));
  ctx->tl_next = 1;  // slot 0: prologue
}
void timeline_print(cpdgpu_ctx* ctx, const char* what) {
  if (!ctx->tl_on) return;
  std::vector<unsigned long long> h(64 * 3);
  CK(cudaMemcpyAsync(h.data(), ctx->tl_ptr(), h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                     ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  const double t0 = static_cast<double>(h[0]);
  std::fprintf(stderr, "[timeline %s] us from prologue entry (entry/wait/exit):", what);
  for (int i = 0; i < 64; ++i) {  // graph replays keep the slots of the capture
    if (h[3 * i + 2] == 0) continue;
    std::fprintf(stderr, "  #%d %.1f/%.1f/%.1f", i, (h[3 * i] - t0) * 1e-3, (h[3 * i + 1] - t0) * 1e-3,
                 (h[3 * i + 2] - t0) * 1e-3);
  }
  std::fprintf(stderr, "\n");
}

// Whole hook-free gradient after the prologue: fused seeds, reductions, then
// the right and left phases advancing together, one launch per level.
// Fused first level (L0Side, kernels.h) for the sides whose level-0 step holds an
// extraction and a recursion over the seed: the right side when p >= 2, the left
// when p + 1 < N.  fp64, one rank chunk, per-row slot sums (not lane-parallel).
// Returns the number of sides set up; the caller drops their reductions and
// level-0 ops.  Disabled by CPDGPU_NO_L0.
int build_l0(cpdgpu_ctx* ctx, Plan& pl, cpdgpu::L0Step& l0, bool& fuse_r, bool& fuse_l) {
  static const bool disabled = std::getenv("CPDGPU_NO_L0") != nullptr;
  fuse_r = fuse_l = false;
  // fp32: the fused pass only (right slots [slot][64 r][128 i] like the int8 pass's;
  // its left side reads Ls, which reduce_left32 has summed from the band partials)
  const bool f32f = pl.f32 && pl.ff.on && pl.p + 1 <= pl.N;
  static const char* l0f_env = std::getenv("CPDGPU_F32_L0");
  if (disabled || (pl.f32 && (!f32f || (l0f_env && std::atoi(l0f_env) == 0))) || pl.chunks.size() != 1 ||
      (f32f ? pl.ff.tab_max : pl.slot_tab_max) >= 16)
    return 0;
  const Plan::Chunk& c = pl.chunks[0];
  const int R = static_cast<int>(pl.R);
  fuse_r = pl.p >= 2 && pl.J[pl.p - 1] <= cpdgpu::kL0MaxRows;
  fuse_l = pl.p + 1 < pl.N && pl.sd[pl.p] <= cpdgpu::kL0MaxRows;
  const int nsides = (fuse_r ? 1 : 0) + (fuse_l ? 1 : 0);
  if (nsides == 0) return 0;
  // chunks per (side, r): at least two CTAs per SM, and about 1024 seed rows per CTA
  // (long reductions like c3's 38416 rows per column gain from more loads in flight)
  int64_t rows_max = 0;
  if (fuse_r) rows_max = std::max<int64_t>(rows_max, pl.Jp);
  if (fuse_l) rows_max = std::max<int64_t>(rows_max, pl.Kp);
  static const char* rows_env = std::getenv("CPDGPU_L0_ROWS");  // A/B knob: seed rows per CTA
  const int64_t per_cta = rows_env && std::atoi(rows_env) > 0 ? std::atoi(rows_env) : 1024;
  const int target = static_cast<int>(std::max<int64_t>((2 * ctx->num_sms + R * nsides - 1) / (R * nsides),
                                                        cpdgpu::ceil_div(rows_max, per_cta)));
  auto chunks = [&](cpdgpu::L0Side& sd) {
    int64_t nq = std::min<int64_t>(target, sd.B);
    int64_t bq = cpdgpu::ceil_div(sd.B, nq);
    if (bq * sd.M > cpdgpu::kL0MaxRows) bq = std::max<int64_t>(1, cpdgpu::kL0MaxRows / sd.M);
    sd.bq = static_cast<int>(bq);
    sd.nq = static_cast<int>(cpdgpu::ceil_div(sd.B, bq));
  };
  l0 = cpdgpu::L0Step{};
  l0.R = R;
  size_t scratch = 0;
  if (fuse_r) {  // right: opA extraction G(p), opB recursion R^(p-1) (G(1) when p == 2)
    cpdgpu::L0Side& sd = l0.side[l0.nsides++];
    const int j = pl.p;
    sd.zsrc = 1;
    sd.Z = pl.Rpart.d() + c.rpart_off;
    if (f32f) {
      sd.Z = pl.Rpart.d();
      sd.RP = cpdgpu::seed_f32_rank_cols();
      sd.TI = 128;
      sd.rb_ptr = static_cast<const int*>(pl.ff.tab.p);
      sd.slot_list = static_cast<const int*>(pl.ff.tab.p) + pl.ff.tab_len;
    } else {
      sd.RP = c.NT * 8;
      sd.TI = c.sp.TI;
      sd.rb_ptr = static_cast<const int*>(pl.slot_tab.p);
      sd.slot_list = static_cast<const int*>(pl.slot_tab.p) + pl.slot_tab_ptr_len;
    }
    sd.M = pl.J[j - 1];
    sd.B = pl.sd[j - 1];
    sd.krA = spec_over(pl, pl.Fs.d(), false, 1, j - 1, 0);
    sd.krB = spec_over(pl, pl.Fs.d(), false, j, j, 0);
    sd.outA = nullptr;
    sd.slotA = pl.perm[j - 1] - 1;
    sd.ldoA = pl.sd[j - 1];
    if (j == 2) {
      sd.outB = nullptr;
      sd.slotB = pl.perm[0] - 1;
      sd.ldoB = pl.sd[0];
    } else {
      sd.outB = pl.Rtmp.d();
      sd.ldoB = pl.Jp;
    }
    chunks(sd);
    scratch += static_cast<size_t>(R) * sd.nq * sd.M;
  }
  if (fuse_l) {  // left: opA recursion L^(p+2) (G(N) when p + 2 == N), opB extraction G(p+1)
    cpdgpu::L0Side& sd = l0.side[l0.nsides++];
    const int j = pl.p + 1;
    if (pl.lpart_direct || f32f) {
      sd.zsrc = 0;
      sd.Z = pl.Ls.d();
      sd.ldz = pl.Kp;
    } else {
      sd.zsrc = 2;
      sd.Z = pl.Lpart.d() + c.lpart_off;
      sd.pcount = pl.i8.on && pl.i8.lred ? 1 : static_cast<int>(c.sp.nRB);
      sd.pK = pl.Kp;
      sd.ldz = static_cast<int64_t>(R) * pl.Kp;
    }
    sd.M = pl.sd[j - 1];
    sd.B = pl.K(j);
    sd.krA = spec_over(pl, pl.Fs.d(), false, j, j, 0);
    sd.krB = spec_over(pl, pl.Fs.d(), false, j + 1, pl.N, 0);
    if (j + 1 == pl.N) {
      sd.outA = nullptr;
      sd.slotA = pl.perm[pl.N - 1] - 1;
      sd.ldoA = pl.sd[pl.N - 1];
    } else {
      sd.outA = pl.Ltmp.d();
      sd.ldoA = pl.Kp;
    }
    sd.outB = nullptr;
    sd.slotB = pl.perm[j - 1] - 1;
    sd.ldoB = pl.sd[j - 1];
    chunks(sd);
    scratch += static_cast<size_t>(R) * sd.nq * sd.M;
  }
  if (pl.l0_scratch.bytes < scratch * sizeof(double)) pl.l0_scratch.ensure(scratch * sizeof(double));
  if (pl.l0_tickets.bytes < 2 * static_cast<size_t>(R) * sizeof(unsigned)) {
    pl.l0_tickets.ensure(2 * static_cast<size_t>(R) * sizeof(unsigned));
    CK(cudaMemsetAsync(pl.l0_tickets.p, 0, pl.l0_tickets.bytes, ctx->stream));
  }
  size_t off = 0;
  for (int i = 0; i < l0.nsides; ++i) {
    cpdgpu::L0Side& sd = l0.side[i];
    sd.scratch = pl.l0_scratch.d() + off;
    off += static_cast<size_t>(R) * sd.nq * sd.M;
    sd.tickets = static_cast<unsigned*>(pl.l0_tickets.p) + i * R;
  }
  return l0.nsides;
}

void gradient_body(cpdgpu_ctx* ctx, Plan& pl) {
  const bool left = pl.p + 1 <= pl.N;
  I8Geometry geometry(pl);
  ctx->last_seed_path = pl.f32 ? ((left && pl.ff.on) ? (pl.ff.img_on ? 4 : 3) : 2) : (pl.i8.on ? 1 : 0);
  if (pl.i8.on)
    run_seeds_i8(ctx, pl);
  else
    run_seeds(ctx, pl, left ? 3 : 1);
  cpdgpu::TailStep st{};
  add_reduce_ops(pl, st, left ? 3 : 1);
  // The extractions G(1) = R^(1) and G(N) = L^(N) are copies (empty Khatri-Rao
  // products): the step producing R^(1) / L^(N) writes the gradient directly.
  const bool g1_direct = pl.p == 1;  // the right seed is R^(1)
  if (g1_direct) redirect_to_gradient(pl, st, /*right=*/true);
  const bool gN_direct = left && pl.p + 1 == pl.N && !pl.lpart_direct;  // the left seed is L^(N)
  if (gN_direct) redirect_to_gradient(pl, st, /*right=*/false);
  if (pl.f32 && left && pl.ff.on) {  // fused fp32 seed: its fp32 left partials, summed over the bands
    const Plan::Chunk& c = pl.chunks[0];
    const int RPc = cpdgpu::seed_f32_rank_cols();
    ctx->launches += cpdgpu::launch_reduce_left32(
        static_cast<const float*>(pl.ff.lpart32.p), pl.ff.img_on && pl.ff.lred ? 1 : pl.ff.nB, pl.ff.nC, pl.Kp, c.Rc,
        reinterpret_cast<const double*>(static_cast<const char*>(pl.tensor->yscale.p) + 8), c.scales->d() + 3 * RPc,
        gN_direct ? nullptr : pl.Ls.d(), static_cast<double* const*>(pl.gtab.p), gN_direct ? pl.perm[pl.N - 1] - 1 : -1,
        pl.Kp, pl.ff.img_on ? 1 : 0, ctx->stream);
  }
  cpdgpu::L0Step l0{};
  bool fuse_r = false, fuse_l = false;
  const int nl0 = build_l0(ctx, pl, l0, fuse_r, fuse_l);
  if (nl0 > 0) {  // the fused sides' reductions go; the rest of the step stays
    cpdgpu::TailStep keep{};
    for (int i = 0; i < st.n; ++i) {
      const bool right = st.op[i].type == cpdgpu::kOpReduceRight;
      if (!(right ? fuse_r : fuse_l)) keep.op[keep.n++] = st.op[i];
    }
    st = keep;
  }
  launch_step(ctx, pl, st);
  if (nl0 > 0) {
    l0.tl = ctx->tl_ptr();
    if (l0.tl) l0.tl_slot = ctx->tl_slot();
    ctx->launches += cpdgpu::launch_l0_step(l0, static_cast<double* const*>(pl.gtab.p), ctx->stream);
  }
  double* rc = pl.Rs.d();
  double* rn = pl.Rtmp.d();
  double* lc = pl.Ls.d();
  double* ln = pl.Ltmp.d();
  const int levels = std::max(pl.p, pl.N - pl.p);
  for (int lv = 0; lv < levels; ++lv) {
    cpdgpu::TailStep s{};
    const int jr = pl.p - lv;      // right phase mode at this level
    const int jl = pl.p + 1 + lv;  // left phase mode at this level
    if (jr >= 2 && lv == 0 && fuse_r) {
      // done by the fused first level (R^(p-1) in Rtmp, or G(1))
    } else if (jr >= 2) {
      add_right_extract(pl, s, jr, rc);
      add_right_recurse(pl, s, jr, rc, rn);
      if (jr == 2) {  // R^(1) is G(1)
        cpdgpu::TailOp& o = s.op[s.n - 1];
        o.out = nullptr;
        o.out_slot = pl.perm[0] - 1;
        o.ldo = pl.sd[0];
      }
    } else if (jr == 1 && !g1_direct && pl.p >= 2) {
      // already written by the previous level's recursion
    } else if (jr == 1 && !g1_direct) {
      add_right_extract(pl, s, jr, rc);
    }
    if (jl <= pl.N && lv == 0 && fuse_l) {
      // done by the fused first level (L^(p+2) in Ltmp, or G(N))
    } else if (jl <= pl.N) {
      if (jl < pl.N) {
        add_left_extract(pl, s, jl, lc);
        add_left_recurse(pl, s, jl, lc, ln);
        if (jl + 1 == pl.N) {  // L^(N) is G(N)
          cpdgpu::TailOp& o = s.op[s.n - 1];
          o.out = nullptr;
          o.out_slot = pl.perm[pl.N - 1] - 1;
          o.ldo = pl.sd[pl.N - 1];
        }
      } else if (!gN_direct && jl == pl.p + 1) {
        add_left_extract(pl, s, jl, lc);  // the left seed itself is L^(N) (lpart_direct)
      }
    }
    if (s.n > 0) launch_step(ctx, pl, s);
    if (jr >= 2) std::swap(rc, rn);
    if (jl < pl.N) std::swap(lc, ln);
  }
  CK(cudaGetLastError());
}

// Gauss-Seidel sweep body shared by ALS and the generic hook: separate right /
// left seed passes; after(j) runs once G(j) is out and may replace A_j before
// the recursion consumes it (mttkrp.cpp:137-144, 174, 203, 222).
using ModeCallback = std::function<void(int j)>;

void sweep_body(cpdgpu_ctx* ctx, Plan& pl, const ModeCallback& after) {
  launch_kr_from_fs(ctx, pl, 1);
  run_seeds(ctx, pl, 1);
  {
    cpdgpu::TailStep st{};
    add_reduce_ops(pl, st, 1);
    launch_step(ctx, pl, st);
  }
  double* rc = pl.Rs.d();
  double* rn = pl.Rtmp.d();
  for (int j = pl.p; j >= 1; --j) {
    cpdgpu::TailStep st{};
    add_right_extract(pl, st, j, rc);
    launch_step(ctx, pl, st);
    after(j);
    if (j >= 2) {
      cpdgpu::TailStep sr{};
      add_right_recurse(pl, sr, j, rc, rn);
      launch_step(ctx, pl, sr);
      std::swap(rc, rn);
    }
  }
  if (pl.p + 1 <= pl.N) {
    launch_kr_from_fs(ctx, pl, 2);
    run_seeds(ctx, pl, 2);
    if (!pl.lpart_direct || pl.use_lc) {
      cpdgpu::TailStep st{};
      add_reduce_ops(pl, st, 2);
      launch_step(ctx, pl, st);
    }
    double* lc = pl.Ls.d();
    double* ln = pl.Ltmp.d();
    for (int j = pl.p + 1; j <= pl.N; ++j) {
      cpdgpu::TailStep st{};
      add_left_extract(pl, st, j, lc);
      launch_step(ctx, pl, st);
      after(j);
      if (j < pl.N) {
        cpdgpu::TailStep sl{};
        add_left_recurse(pl, sl, j, lc, ln);
        launch_step(ctx, pl, sl);
        std::swap(lc, ln);
      }
    }
  }
  CK(cudaGetLastError());
}

// Graph of the hook-free gradient (prologue + body), captured once per plan;
// each call patches the prologue node (input factors, output pointers).
void run_gradient(cpdgpu_ctx* ctx, Plan& pl, const double* fin, double* gout_base) {
  const bool left = pl.p + 1 <= pl.N;
  // the int8 seed builds its Khatri-Rao digits from the sorted factors itself, and
  // the fused fp32 pass its fp16 operands (launch_kr_fused_operands): no fp64 rows
  const bool own_kr = pl.i8.on || (pl.f32 && left && pl.ff.on);
  cpdgpu::Prologue pr = grad_prologue(pl, fin, gout_base, own_kr ? 0 : (left ? 3 : 1));
  pr.tl = ctx->tl_ptr();
  if (pl.i8.on && pl.i8.lred) {  // the int8 seed adds its left partials into this slot
    pr.zero = pl.Lpart.d() + pl.chunks[0].lpart_off;
    pr.zero_n = pl.chunks[0].Rc * pl.Kp;
  }
  timeline_reset(ctx);
  struct PrintAtExit {
    cpdgpu_ctx* c;
    ~PrintAtExit() {
      try {
        timeline_print(c, "gradient");
      } catch (...) {
      }
    }
  } print_at_exit{ctx};
  const bool use_graph = ctx->graphs && !ctx->timing && std::getenv("CPDGPU_SEED_TRACE") == nullptr;
  if (!use_graph) {
    ctx->launches += cpdgpu::launch_prologue(pr, static_cast<double**>(pl.gtab.p), ctx->num_sms, ctx->stream);
    gradient_body(ctx, pl);
    return;
  }
  if (!pl.grad_exec) {
    if (!pl.grad_warm) {  // first call eager: configures kernel attributes outside capture
      ctx->launches += cpdgpu::launch_prologue(pr, static_cast<double**>(pl.gtab.p), ctx->num_sms, ctx->stream);
      gradient_body(ctx, pl);
      pl.grad_warm = true;
      return;
    }
    const uint64_t before = ctx->launches;
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    cpdgpu::launch_prologue(pr, static_cast<double**>(pl.gtab.p), ctx->num_sms, ctx->stream);
    gradient_body(ctx, pl);
    CK(cudaStreamEndCapture(ctx->stream, &g));
    pl.grad_graph_launches = ctx->launches - before + 1;
    ctx->launches = before;
    size_t n = 0;
    CK(cudaGraphGetNodes(g, nullptr, &n));
    std::vector<cudaGraphNode_t> nodes(n);
    CK(cudaGraphGetNodes(g, nodes.data(), &n));
    pl.prologue_node = nullptr;
    for (auto nd : nodes) {
      cudaGraphNodeType ty;
      CK(cudaGraphNodeGetType(nd, &ty));
      if (ty != cudaGraphNodeTypeKernel) continue;
      cudaKernelNodeParams kp{};
      CK(cudaGraphKernelNodeGetParams(nd, &kp));
      if (kp.func == cpdgpu::prologue_kernel_fn()) pl.prologue_node = nd;
    }
    if (!pl.prologue_node) fail(CPDGPU_CUDA_ERROR, "graph capture: prologue node not found");
    CK(cudaGraphInstantiate(&pl.grad_exec, g, 0));
    pl.grad_graph = g;
  }
  // patch the prologue's arguments, then replay
  cudaKernelNodeParams kp{};
  dim3 grid, block;
  cpdgpu::prologue_geometry(pr, ctx->num_sms, &grid, &block);
  void* gt = pl.gtab.p;
  void* args[] = {const_cast<cpdgpu::Prologue*>(&pr), &gt};
  kp.func = const_cast<void*>(cpdgpu::prologue_kernel_fn());
  kp.gridDim = grid;
  kp.blockDim = block;
  kp.sharedMemBytes = 0;
  kp.kernelParams = args;
  kp.extra = nullptr;
  CK(cudaGraphExecKernelNodeSetParams(pl.grad_exec, pl.prologue_node, &kp));
  CK(cudaGraphLaunch(pl.grad_exec, ctx->stream));
  ctx->launches += pl.grad_graph_launches;
}

// Direct mode-n MTTKRP (Algorithm 1's cost model: one pass over Y per mode)
// with the gradient's own machinery in the sorted frame: sorted mode j <= p* takes
// the right seed at p* and the right recursions down to j (extraction at j);
// j > p* takes the left seed (column-block pass) and the left recursions up to j.
// One seed pass plus small recursions per call, for any aspect ratio.
void direct_body(cpdgpu_ctx* ctx, Plan& pl, const double* fin, double* gout_base, int n) {
  int j = 1;
  while (pl.perm[j - 1] != n) ++j;  // sorted position of caller mode n
  const bool right = j <= pl.p;
  ctx->launches += cpdgpu::launch_prologue(grad_prologue(pl, fin, gout_base, right ? 1 : 2),
                                           static_cast<double**>(pl.gtab.p), ctx->num_sms, ctx->stream);
  run_seeds(ctx, pl, right ? 1 : 2);
  {
    cpdgpu::TailStep st{};
    add_reduce_ops(pl, st, right ? 1 : 2);
    if (st.n > 0) launch_step(ctx, pl, st);
  }
  if (right) {
    double* rc = pl.Rs.d();
    double* rn = pl.Rtmp.d();
    for (int k = pl.p; k > j; --k) {
      cpdgpu::TailStep s{};
      add_right_recurse(pl, s, k, rc, rn);
      launch_step(ctx, pl, s);
      std::swap(rc, rn);
    }
    cpdgpu::TailStep s{};
    add_right_extract(pl, s, j, rc);
    launch_step(ctx, pl, s);
  } else {
    double* lc = pl.Ls.d();
    double* ln = pl.Ltmp.d();
    for (int k = pl.p + 1; k < j; ++k) {
      cpdgpu::TailStep s{};
      add_left_recurse(pl, s, k, lc, ln);
      launch_step(ctx, pl, s);
      std::swap(lc, ln);
    }
    cpdgpu::TailStep s{};
    add_left_extract(pl, s, j, lc);
    launch_step(ctx, pl, s);
  }
  CK(cudaGetLastError());
}

// mttkrp_direct's multiplication charge (mttkrp.cpp:29-54, kron.cpp:85-93):
// R (J_N + sum_{k=2}^{n-1} J_k + sum_{k=n+1}^{N} J_k / I_n), caller's mode order.
uint64_t direct_count(const std::vector<int64_t>& dims, int64_t R, int n) {
  const int N = static_cast<int>(dims.size());
  std::vector<uint64_t> J(static_cast<size_t>(N) + 1, 1);
  for (int k = 1; k <= N; ++k) J[k] = J[k - 1] * static_cast<uint64_t>(dims[k - 1]);
  uint64_t s = J[N];
  for (int k = 2; k <= n - 1; ++k) s += J[k];
  for (int k = n + 1; k <= N; ++k) s += J[k] / static_cast<uint64_t>(dims[n - 1]);
  return static_cast<uint64_t>(R) * s;
}

Plan& direct_plan(cpdgpu_ctx* ctx, cpdgpu_tensor* y, int64_t R) {
  ensure_sorted(ctx, y);
  Plan& pl = *get_plan(ctx, y, R, 0);
  bind_seed_inputs(ctx, pl, y);
  return pl;
}

void upload_host_factors(cpdgpu_ctx* ctx, Plan& pl, cpdgpu_tensor* t, const double* const* factors) {
  for (int m = 0; m < pl.N; ++m)
    std::memcpy(pl.hF.d() + pl.off_orig[m], factors[m],
                static_cast<size_t>(t->dims[m] * pl.R) * sizeof(double));
  CK(cudaMemcpyAsync(pl.Forig.d(), pl.hF.d(), static_cast<size_t>(pl.total_factor) * sizeof(double),
                     cudaMemcpyHostToDevice, ctx->stream));
}

// Sorted device factors <- caller-order device buffer (ALS / hook entry).
void gather_factors(cpdgpu_ctx* ctx, Plan& pl, const double* src_orig) {
  int64_t so[kMaxModes], dof[kMaxModes], len[kMaxModes];
  for (int j = 0; j < pl.N; ++j) {
    so[j] = pl.off_orig[pl.perm[j] - 1];
    dof[j] = pl.off_sorted[j];
    len[j] = pl.sd[j] * pl.R;
  }
  ctx->launches += cpdgpu::launch_gather_blocks(src_orig, pl.Fs.d(), pl.N, so, dof, len, ctx->stream);
}

void scatter_factors(cpdgpu_ctx* ctx, Plan& pl, double* dst_orig) {
  int64_t so[kMaxModes], dof[kMaxModes], len[kMaxModes];
  for (int j = 0; j < pl.N; ++j) {  // caller block m <- sorted block j with perm[j] = m + 1
    const int m = pl.perm[j] - 1;
    so[m] = pl.off_sorted[j];
    dof[m] = pl.off_orig[m];
    len[m] = pl.sd[j] * pl.R;
  }
  ctx->launches += cpdgpu::launch_gather_blocks(pl.Fs.d(), dst_orig, pl.N, so, dof, len, ctx->stream);
}

void validate_common(cpdgpu_ctx* ctx, cpdgpu_tensor* y, int64_t R, const char* who) {
  if (!ctx || !y) fail(CPDGPU_ARGUMENT_ERROR, "%s: null context or tensor", who);
  if (y->dims.size() < 2) fail(CPDGPU_ARGUMENT_ERROR, "%s: need an order-2 or higher tensor", who);
  if (R < 1) fail(CPDGPU_ARGUMENT_ERROR, "%s: rank must be positive", who);
  use_device(ctx);
  ctx->seed_used = 0;
}

void compute_norm2(cpdgpu_ctx* ctx, cpdgpu_tensor* t) {
  if (t->norm2 >= 0.0) return;
  ctx->scratch.ensure(2048 * sizeof(double));
  DevBuf out;
  out.ensure(sizeof(double));
  ctx->launches += cpdgpu::launch_norm2(t->data, static_cast<int>(t->elem()), t->numel,
                                        ctx->scratch.d(), out.d(), ctx->stream);
  double v = 0.0;
  CK(cudaMemcpyAsync(&v, out.d(), sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  t->norm2 = v;
}

cpdgpu_tensor* new_tensor(cpdgpu_ctx* ctx, cpdgpu_dtype dtype, int N, const int64_t* dims) {
  if (N < 1 || N > kMaxModes) fail(CPDGPU_ARGUMENT_ERROR, "tensor: order %d outside 1..%d", N, kMaxModes);
  if (dtype != CPDGPU_F64 && dtype != CPDGPU_F32) fail(CPDGPU_ARGUMENT_ERROR, "tensor: unknown dtype");
  auto t = std::make_unique<cpdgpu_tensor>();
  t->ctx = ctx;
  t->dtype = dtype;
  t->dims.assign(dims, dims + N);
  t->numel = prefix(t->dims).back();
  t->perm = sort_perm(t->dims);
  t->identity = true;
  for (int j = 0; j < N; ++j) t->identity &= (t->perm[j] == j + 1);
  t->id = ctx->next_id++;
  return t.release();
}

// Drop cached plans of a tensor (its id is never reused).
void forget_tensor(cpdgpu_ctx* ctx, uint64_t id) {
  for (auto it = ctx->plans.begin(); it != ctx->plans.end();) {
    if (std::get<0>(it->first) == id) it = ctx->plans.erase(it);
    else ++it;
  }
}

void init_grams(cpdgpu_ctx* ctx, Plan& pl) {
  const int R = static_cast<int>(pl.R);
  for (int j = 1; j <= pl.N; ++j)
    ctx->launches += cpdgpu::launch_gram(pl.factor(j), pl.sd[j - 1], R,
                                         pl.grams.d() + static_cast<int64_t>(j - 1) * R * R, ctx->stream);
}

// One fast ALS sweep on the device (als.cpp:69-78): right seed pass, modes
// p..1, left seed pass with the updated factors, modes p+1..N.  G(n) lands in
// Gorig (through the output table set by prepare_als).
void als_sweep_device(cpdgpu_ctx* ctx, Plan& pl, double rtol) {
  const int R = static_cast<int>(pl.R);
  sweep_body(ctx, pl, [&](int j) {
    double* G = pl.Gorig.d() + pl.off_orig[pl.perm[j - 1] - 1];
    ctx->launches += cpdgpu::launch_als_update(G, pl.sd[j - 1], R, pl.grams.d(), pl.N, j - 1, rtol,
                                               pl.factor(j), pl.grams.d() + static_cast<int64_t>(j - 1) * R * R,
                                               static_cast<int*>(pl.status.p), ctx->stream);
  });
}

// cost after a sweep: last visited mode L (fast_update_order) gives <Y, Yhat>
void als_cost(cpdgpu_ctx* ctx, Plan& pl, double* cost_slot, int L = 0) {
  if (L == 0) L = pl.p + 1 <= pl.N ? pl.N : 1;
  ctx->launches += cpdgpu::launch_als_cost(pl.factor(L), pl.Gorig.d() + pl.off_orig[pl.perm[L - 1] - 1],
                                           pl.sd[L - 1], static_cast<int>(pl.R), pl.grams.d(), pl.N, pl.norm.d(),
                                           cost_slot, ctx->stream);
}

// Sweep through a CUDA graph captured once per plan (fixed device buffers).
void als_sweep_graph(cpdgpu_ctx* ctx, Plan& pl, double rtol) {
  if (!ctx->graphs || ctx->timing) {
    als_sweep_device(ctx, pl, rtol);
    return;
  }
  if (pl.als_exec && pl.als_rtol != rtol) {
    cudaGraphExecDestroy(pl.als_exec);
    pl.als_exec = nullptr;
  }
  if (!pl.als_exec) {
    if (!pl.als_warm) {
      als_sweep_device(ctx, pl, rtol);
      pl.als_warm = true;
      return;
    }
    const uint64_t before = ctx->launches;
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    als_sweep_device(ctx, pl, rtol);
    CK(cudaStreamEndCapture(ctx->stream, &g));
    pl.als_graph_launches = ctx->launches - before;
    ctx->launches = before;
    CK(cudaGraphInstantiate(&pl.als_exec, g, 0));
    CK(cudaGraphDestroy(g));
    pl.als_rtol = rtol;
  }
  CK(cudaGraphLaunch(pl.als_exec, ctx->stream));
  ctx->launches += pl.als_graph_launches;
}

void download_factors(cpdgpu_ctx* ctx, Plan& pl, cpdgpu_tensor* t, double* const* factors) {
  scatter_factors(ctx, pl, pl.Forig.d());
  CK(cudaMemcpyAsync(pl.hF.d(), pl.Forig.d(), static_cast<size_t>(pl.total_factor) * sizeof(double),
                     cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  for (int m = 0; m < pl.N; ++m)
    std::memcpy(factors[m], pl.hF.d() + pl.off_orig[m],
                static_cast<size_t>(t->dims[m] * pl.R) * sizeof(double));
}

void check_status(cpdgpu_ctx* ctx, Plan& pl) {
  int st = 0;
  CK(cudaMemcpyAsync(&st, pl.status.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (st == 4) fail(CPDGPU_NUMERIC_ERROR, "als_update_mode: non-finite gradient input");
}

// ---- the other gradient consumers on the device (als.cpp:58-101) -----------------

// Direct MTTKRP of caller mode n from the live sorted factors (Fs): the sweeps'
// form of direct_body (no factor gather).
void direct_body_fs(cpdgpu_ctx* ctx, Plan& pl, int n) {
  int j = 1;
  while (pl.perm[j - 1] != n) ++j;
  const bool right = j <= pl.p;
  launch_kr_from_fs(ctx, pl, right ? 1 : 2);
  run_seeds(ctx, pl, right ? 1 : 2);
  {
    cpdgpu::TailStep st{};
    add_reduce_ops(pl, st, right ? 1 : 2);
    if (st.n > 0) launch_step(ctx, pl, st);
  }
  cpdgpu::TailStep s{};
  if (right) {
    double* rc = pl.Rs.d();
    double* rn = pl.Rtmp.d();
    for (int k = pl.p; k > j; --k) {
      cpdgpu::TailStep r{};
      add_right_recurse(pl, r, k, rc, rn);
      launch_step(ctx, pl, r);
      std::swap(rc, rn);
    }
    add_right_extract(pl, s, j, rc);
  } else {
    double* lc = pl.Ls.d();
    double* ln = pl.Ltmp.d();
    for (int k = pl.p + 1; k < j; ++k) {
      cpdgpu::TailStep r{};
      add_left_recurse(pl, r, k, lc, ln);
      launch_step(ctx, pl, r);
      std::swap(lc, ln);
    }
    add_left_extract(pl, s, j, lc);
  }
  launch_step(ctx, pl, s);
}

int sorted_pos(const Plan& pl, int n) {
  int j = 1;
  while (pl.perm[j - 1] != n) ++j;
  return j;
}

// mu_sweep (als.cpp:80-91) through the Gauss-Seidel sweep.
void mu_sweep_device(cpdgpu_ctx* ctx, Plan& pl, double eps) {
  const int R = static_cast<int>(pl.R);
  sweep_body(ctx, pl, [&](int j) {
    double* G = pl.Gorig.d() + pl.off_orig[pl.perm[j - 1] - 1];
    ctx->launches += cpdgpu::launch_mu_update(G, pl.sd[j - 1], R, pl.grams.d(), pl.N, j - 1, eps, pl.factor(j),
                                              pl.grams.d() + static_cast<int64_t>(j - 1) * R * R, ctx->stream);
  });
}

// gd_step (als.cpp:93-101): every mode's gradient at the pre-step factors, the
// simultaneous step, then fresh Grams.
void gd_step_device(cpdgpu_ctx* ctx, Plan& pl, double eta) {
  const int R = static_cast<int>(pl.R);
  launch_kr_from_fs(ctx, pl, pl.p + 1 <= pl.N ? 3 : 1);
  gradient_body(ctx, pl);
  for (int j = 1; j <= pl.N; ++j)
    ctx->launches += cpdgpu::launch_gd_update(pl.Gorig.d() + pl.off_orig[pl.perm[j - 1] - 1], pl.sd[j - 1], R,
                                              pl.grams.d(), pl.N, j - 1, eta, pl.factor(j), ctx->stream);
  init_grams(ctx, pl);
}

// als_sweep_direct (als.cpp:58-67): direct MTTKRP + update per caller mode of order.
void direct_sweep_device(cpdgpu_ctx* ctx, Plan& pl, const std::vector<int>& order, double rtol) {
  const int R = static_cast<int>(pl.R);
  for (int n : order) {
    direct_body_fs(ctx, pl, n);
    const int j = sorted_pos(pl, n);
    ctx->launches += cpdgpu::launch_als_update(pl.Gorig.d() + pl.off_orig[n - 1], pl.sd[j - 1], R, pl.grams.d(),
                                               pl.N, j - 1, rtol, pl.factor(j),
                                               pl.grams.d() + static_cast<int64_t>(j - 1) * R * R,
                                               static_cast<int*>(pl.status.p), ctx->stream);
  }
}

// cost after an iteration of `algo` (Gram identity, kruskal.cpp:58-77): Gauss-
// Seidel sweeps reuse the last visited mode's gradient; gd needs one fresh
// direct MTTKRP (of sorted mode 1) at the stepped factors.
void algo_cost(cpdgpu_ctx* ctx, Plan& pl, int algo, const std::vector<int>& order, double* slot) {
  if (algo == 0) {
    als_cost(ctx, pl, slot, sorted_pos(pl, order.back()));
  } else if (algo == 3) {
    direct_body_fs(ctx, pl, pl.perm[0]);
    als_cost(ctx, pl, slot, 1);
  } else {
    als_cost(ctx, pl, slot);
  }
}

void check_nonneg_inputs(cpdgpu_ctx* ctx, Plan& pl, cpdgpu_tensor* y, const double* const* factors) {
  for (size_t m = 0; m < y->dims.size(); ++m)
    for (int64_t q = 0; q < y->dims[m] * pl.R; ++q)
      if (factors[m][q] < 0.0) fail(CPDGPU_DOMAIN_ERROR, "mu_sweep: factors have negative entries");
  DevBuf flag;
  flag.ensure(sizeof(int));
  CK(cudaMemsetAsync(flag.p, 0, sizeof(int), ctx->stream));
  ctx->launches += cpdgpu::launch_nonneg_check(y->data, static_cast<int>(y->elem()), y->numel,
                                               static_cast<int*>(flag.p), ctx->stream);
  int bad = 0;
  CK(cudaMemcpyAsync(&bad, flag.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (bad) fail(CPDGPU_DOMAIN_ERROR, "mu_sweep: tensor has negative entries");
}

void prepare_als(cpdgpu_ctx* ctx, Plan& pl, cpdgpu_tensor* y) {
  compute_norm2(ctx, y);
  CK(cudaMemcpyAsync(pl.norm.d(), &y->norm2, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemsetAsync(pl.status.p, 0, sizeof(int), ctx->stream));
  gather_factors(ctx, pl, pl.Forig.d());
  set_gtab(ctx, pl, pl.Gorig.d());
  init_grams(ctx, pl);
}

}  // namespace

// ---- C-ABI ---------------------------------------------------------------------

extern "C" {

int cpdgpu_create(cpdgpu_ctx** out, int device) {
  if (!out) return CPDGPU_ARGUMENT_ERROR;
  *out = nullptr;
  auto ctx = std::make_unique<cpdgpu_ctx>();
  const int st = guarded(nullptr, [&] {
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) fail(CPDGPU_ARGUMENT_ERROR, "device %d outside 0..%d", device, n - 1);
    ctx->device = device;
    CK(cudaSetDevice(device));
    CK(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device));
    int major = 0, minor = 0;
    CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    CK(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
    if (major != 10 || minor != 0)
      fail(CPDGPU_CUDA_ERROR, "device %d is sm_%d%d; this library is built for sm_100a (B200) only",
           device, major, minor);
    CK(cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking));
    ctx->stream = ctx->own;
    int* fh = nullptr;
    CK(cudaHostAlloc(reinterpret_cast<void**>(&fh), sizeof(int), cudaHostAllocMapped));
    *fh = 0;
    ctx->fault_host = fh;
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->fault_dev), fh, 0));
    int* gh = nullptr;
    CK(cudaHostAlloc(reinterpret_cast<void**>(&gh), sizeof(int), cudaHostAllocMapped));
    *gh = 0;
    ctx->guard_host = gh;
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->guard_dev), gh, 0));
  });
  if (st != CPDGPU_OK) return st;
  *out = ctx.release();
  return CPDGPU_OK;
}

int cpdgpu_destroy(cpdgpu_ctx* ctx) {
  if (!ctx) return CPDGPU_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  ctx->plans.clear();
  if (ctx->own) cudaStreamDestroy(ctx->own);
  delete ctx;
  return CPDGPU_OK;
}

const char* cpdgpu_last_error(const cpdgpu_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int cpdgpu_device_workspace(cpdgpu_ctx* ctx, int64_t* current_bytes, int64_t* peak_bytes) {
  if (!ctx) return CPDGPU_ARGUMENT_ERROR;
  if (current_bytes) *current_bytes = static_cast<int64_t>(g_ws_cur.load());
  if (peak_bytes) *peak_bytes = static_cast<int64_t>(g_ws_peak.load());
  return CPDGPU_OK;
}

int cpdgpu_set_stream(cpdgpu_ctx* ctx, void* stream) {
  if (!ctx) return CPDGPU_ARGUMENT_ERROR;
  ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own;
  return CPDGPU_OK;
}

int cpdgpu_synchronize(cpdgpu_ctx* ctx) {
  return guarded(ctx, [&] {
    use_device(ctx);
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

int cpdgpu_set_graphs(cpdgpu_ctx* ctx, int enabled) {
  if (!ctx) return CPDGPU_ARGUMENT_ERROR;
  ctx->graphs = enabled != 0;
  return CPDGPU_OK;
}

int cpdgpu_set_deterministic(cpdgpu_ctx* ctx, int enabled) {
  if (!ctx) return CPDGPU_ARGUMENT_ERROR;
  ctx->deterministic = enabled != 0;
  return CPDGPU_OK;
}

uint64_t cpdgpu_launch_count(const cpdgpu_ctx* ctx) { return ctx ? ctx->launches : 0; }
int cpdgpu_last_seed_path(const cpdgpu_ctx* ctx) { return ctx ? ctx->last_seed_path : -1; }

int cpdgpu_set_timing(cpdgpu_ctx* ctx, int enabled) {
  if (!ctx) return CPDGPU_ARGUMENT_ERROR;
  ctx->timing = enabled != 0;
  return CPDGPU_OK;
}

int cpdgpu_last_seed_ms(cpdgpu_ctx* ctx, double* ms) {
  return guarded(ctx, [&] {
    if (!ms) fail(CPDGPU_ARGUMENT_ERROR, "last_seed_ms: null argument");
    use_device(ctx);
    double tot = 0.0;
    for (size_t i = 0; i + 1 < ctx->seed_used; i += 2) {
      CK(cudaEventSynchronize(ctx->seed_events[i + 1]));
      float f = 0.f;
      CK(cudaEventElapsedTime(&f, ctx->seed_events[i], ctx->seed_events[i + 1]));
      tot += f;
    }
    *ms = tot;
  });
}

}  // extern "C"

// ---- host -> device copies of Y ---------------------------------------------------
// A caller of the reference holds Y in pageable memory (DenseTensor's std::vector,
// dense_tensor.hpp:15-47).  cudaMemcpy from pageable memory is staged by the driver
// on one thread; here large pageable sources go through the library's own pinned
// staging buffers, filled by a few host threads (one stream and two 8 MB slots
// each), so the copy runs near the PCIe rate instead of one core's memcpy rate.
// Pinned / registered sources and small copies take the plain cudaMemcpyAsync.
// CPDGPU_STAGED_UPLOAD=0 turns the staging off; CPDGPU_UPLOAD_THREADS sets the threads.
struct HostStager {
  static constexpr size_t kChunk = size_t(8) << 20;
  int device = 0, W = 0;
  std::vector<void*> pin;            // [W][2]
  std::vector<cudaStream_t> st;      // [W]
  std::vector<cudaEvent_t> ev;       // [W][2]
  explicit HostStager(int dev) : device(dev) {
    const char* e = std::getenv("CPDGPU_UPLOAD_THREADS");
    int w = e ? std::atoi(e) : static_cast<int>(std::thread::hardware_concurrency() / 2);
    W = std::max(1, std::min(w, 8));
    pin.assign(static_cast<size_t>(2 * W), nullptr);
    st.assign(static_cast<size_t>(W), nullptr);
    ev.assign(static_cast<size_t>(2 * W), nullptr);
    for (int i = 0; i < 2 * W; ++i) {
      if (cudaHostAlloc(&pin[i], kChunk, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        pin[i] = nullptr;
        W = 0;  // no pinned memory to be had: the plain copy
        return;
      }
      CK(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    }
    for (int i = 0; i < W; ++i) CK(cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking));
  }
  ~HostStager() {
    cudaSetDevice(device);
    for (auto s : st) if (s) cudaStreamDestroy(s);
    for (auto e : ev) if (e) cudaEventDestroy(e);
    for (auto p : pin) if (p) cudaFreeHost(p);
  }
  // dst (device) <- src (pageable host); returns when the bytes are on the device
  void copy(void* dst, const void* src, size_t bytes) {
    const size_t nchunk = (bytes + kChunk - 1) / kChunk;
    std::atomic<int> err{0};
    auto work = [&](int w) {
      if (cudaSetDevice(device) != cudaSuccess) { err = 1; return; }
      int use = 0;
      for (size_t c = static_cast<size_t>(w); c < nchunk && !err; c += static_cast<size_t>(W), ++use) {
        const int slot = 2 * w + (use & 1);
        const size_t off = c * kChunk, n = std::min(kChunk, bytes - off);
        if (use >= 2 && cudaEventSynchronize(ev[slot]) != cudaSuccess) { err = 1; return; }
        std::memcpy(pin[slot], static_cast<const char*>(src) + off, n);
        if (cudaMemcpyAsync(static_cast<char*>(dst) + off, pin[slot], n, cudaMemcpyHostToDevice, st[w]) != cudaSuccess ||
            cudaEventRecord(ev[slot], st[w]) != cudaSuccess) { err = 1; return; }
      }
      if (cudaStreamSynchronize(st[w]) != cudaSuccess) err = 1;
    };
    std::vector<std::thread> th;
    for (int w = 1; w < W; ++w) th.emplace_back(work, w);
    work(0);
    for (auto& t : th) t.join();
    if (err) {
      const cudaError_t e = cudaGetLastError();
      fail(CPDGPU_CUDA_ERROR, "staged upload failed: %s", cudaGetErrorString(e));
    }
  }
};

namespace {
bool host_is_pageable(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

// Y's bytes to the device, ordered after the work already on the context stream;
// `sync`: return only when they have landed (pageable sources always do)
void upload_bytes(cpdgpu_ctx* ctx, void* dst, const void* host, size_t bytes, bool sync) {
  const char* staged_env = std::getenv("CPDGPU_STAGED_UPLOAD");  // per call: tests and bench compare both
  const bool staged_on = !(staged_env && staged_env[0] == '0');
  if (staged_on && bytes >= (size_t(32) << 20) && host_is_pageable(host)) {
    if (!ctx->stager) ctx->stager = std::make_shared<HostStager>(ctx->device);
    if (ctx->stager->W > 0) {
      CK(cudaStreamSynchronize(ctx->stream));  // earlier readers of dst are done
      ctx->stager->copy(dst, host, bytes);
      return;
    }
  }
  CK(cudaMemcpyAsync(dst, host, bytes, cudaMemcpyHostToDevice, ctx->stream));
  if (sync) CK(cudaStreamSynchronize(ctx->stream));
}
}  // namespace

extern "C" {

int cpdgpu_tensor_update(cpdgpu_ctx* ctx, cpdgpu_tensor* t, const void* host) {
  return guarded(ctx, [&] {
    if (!ctx || !t || !host) fail(CPDGPU_ARGUMENT_ERROR, "tensor_update: null argument");
    use_device(ctx);
    upload_bytes(ctx, t->data, host, static_cast<size_t>(t->numel) * t->elem(), /*sync=*/false);
    t->norm2 = -1.0;
    ++t->version;
    if (!t->identity && t->sorted_ready) {  // refresh the sorted copy lazily
      cudaFree(t->sorted);
      ws_add(-static_cast<long long>(t->numel * static_cast<int64_t>(t->elem())));
      t->sorted = nullptr;
      t->sorted_ready = false;
    }
  });
}

int cpdgpu_tensor_upload(cpdgpu_ctx* ctx, const void* host, cpdgpu_dtype dtype, int N,
                         const int64_t* dims, cpdgpu_tensor** out) {
  return guarded(ctx, [&] {
    if (!ctx || !out || !dims) fail(CPDGPU_ARGUMENT_ERROR, "tensor_upload: null argument");
    use_device(ctx);
    std::unique_ptr<cpdgpu_tensor> t(new_tensor(ctx, dtype, N, dims));
    const size_t bytes = static_cast<size_t>(t->numel) * t->elem();
    CK(cudaMalloc(&t->data, bytes));
    t->owned = true;
    if (host) upload_bytes(ctx, t->data, host, bytes, /*sync=*/true);
    else CK(cudaMemsetAsync(t->data, 0, bytes, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    *out = t.release();
  });
}

int cpdgpu_tensor_wrap_device(cpdgpu_ctx* ctx, void* device_ptr, cpdgpu_dtype dtype, int N,
                              const int64_t* dims, cpdgpu_tensor** out) {
  return guarded(ctx, [&] {
    if (!ctx || !out || !dims || !device_ptr) fail(CPDGPU_ARGUMENT_ERROR, "tensor_wrap_device: null argument");
    use_device(ctx);
    std::unique_ptr<cpdgpu_tensor> t(new_tensor(ctx, dtype, N, dims));
    t->data = device_ptr;
    t->owned = false;
    *out = t.release();
  });
}

int cpdgpu_tensor_generate(cpdgpu_ctx* ctx, cpdgpu_dtype dtype, int N, const int64_t* dims,
                           cpdgpu_dist dist, uint64_t seed, int64_t offset, cpdgpu_tensor** out) {
  return guarded(ctx, [&] {
    if (!ctx || !out || !dims) fail(CPDGPU_ARGUMENT_ERROR, "tensor_generate: null argument");
    if (dist != CPDGPU_DIST_NORMAL && dist != CPDGPU_DIST_UNIFORM_PM1)
      fail(CPDGPU_ARGUMENT_ERROR, "tensor_generate: unknown distribution");
    use_device(ctx);
    std::unique_ptr<cpdgpu_tensor> t(new_tensor(ctx, dtype, N, dims));
    CK(cudaMalloc(&t->data, static_cast<size_t>(t->numel) * t->elem()));
    t->owned = true;
    ctx->launches += cpdgpu::launch_generate(t->data, static_cast<int>(t->elem()), t->numel,
                                             static_cast<int>(dist), seed, offset, ctx->stream);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(ctx->stream));
    *out = t.release();
  });
}

int cpdgpu_tensor_axpby_kruskal(cpdgpu_ctx* ctx, cpdgpu_tensor* t, double alpha, double beta,
                                const double* const* factors, int64_t R) {
  return guarded(ctx, [&] {
    if (!ctx || !t || !factors) fail(CPDGPU_ARGUMENT_ERROR, "tensor_axpby_kruskal: null argument");
    if (R < 1) fail(CPDGPU_ARGUMENT_ERROR, "tensor_axpby_kruskal: rank must be positive");
    use_device(ctx);
    const int N = static_cast<int>(t->dims.size());
    int64_t total = 0;
    for (int m = 0; m < N; ++m) total += t->dims[m] * R;
    DevBuf F;
    F.ensure(static_cast<size_t>(total) * sizeof(double));
    KRSpec all{};
    all.n = N;
    int64_t off = 0;
    for (int m = 0; m < N; ++m) {
      CK(cudaMemcpyAsync(F.d() + off, factors[m], static_cast<size_t>(t->dims[m] * R) * sizeof(double),
                         cudaMemcpyHostToDevice, ctx->stream));
      all.dims[m] = t->dims[m];
      all.A[m] = F.d() + off;
      off += t->dims[m] * R;
    }
    ctx->launches += cpdgpu::launch_axpby_kruskal(t->data, static_cast<int>(t->elem()), N, t->dims.data(),
                                                  all, static_cast<int>(R), alpha, beta, ctx->stream);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(ctx->stream));
    t->norm2 = -1.0;
    ++t->version;
    t->sorted_ready = t->identity ? t->sorted_ready : false;
    if (!t->identity && t->sorted) {
      cudaFree(t->sorted);
      ws_add(-static_cast<long long>(t->numel * static_cast<int64_t>(t->elem())));
      t->sorted = nullptr;
    }
  });
}

int cpdgpu_tensor_download(cpdgpu_ctx* ctx, const cpdgpu_tensor* t, void* host) {
  return guarded(ctx, [&] {
    if (!ctx || !t || !host) fail(CPDGPU_ARGUMENT_ERROR, "tensor_download: null argument");
    use_device(ctx);
    CK(cudaMemcpyAsync(host, t->data, static_cast<size_t>(t->numel) * t->elem(), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

int cpdgpu_tensor_norm2(cpdgpu_ctx* ctx, cpdgpu_tensor* t, double* out) {
  return guarded(ctx, [&] {
    if (!ctx || !t || !out) fail(CPDGPU_ARGUMENT_ERROR, "tensor_norm2: null argument");
    use_device(ctx);
    compute_norm2(ctx, t);
    *out = t->norm2;
  });
}

int cpdgpu_tensor_device_ptr(const cpdgpu_tensor* t, void** device_ptr) {
  if (!t || !device_ptr) return CPDGPU_ARGUMENT_ERROR;
  *device_ptr = t->data;
  return CPDGPU_OK;
}

int cpdgpu_tensor_free(cpdgpu_tensor* t) {
  if (!t) return CPDGPU_OK;
  if (t->ctx) {
    cudaSetDevice(t->ctx->device);
    cudaStreamSynchronize(t->ctx->stream);
    forget_tensor(t->ctx, t->id);
  }
  delete t;
  return CPDGPU_OK;
}

// ---- TDNB files (io.cpp:162-216): binary tensor ingest straight to the device ------

namespace {
struct FileCloser {
  FILE* f;
  ~FileCloser() {
    if (f) std::fclose(f);
  }
};
struct PinnedBuf {
  void* p = nullptr;
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
};
}  // namespace

int cpdgpu_tensor_load_tdnb(cpdgpu_ctx* ctx, const char* path, int64_t slab_lo, int64_t slab_hi,
                            cpdgpu_tensor** out) {
  return guarded(ctx, [&] {
    if (!ctx || !path || !out) fail(CPDGPU_ARGUMENT_ERROR, "load_tdnb: null argument");
    *out = nullptr;
    use_device(ctx);
    FileCloser fc{std::fopen(path, "rb")};
    if (!fc.f) fail(CPDGPU_PARSE_ERROR, "%s: cannot open", path);
    std::fseek(fc.f, 0, SEEK_END);
    const int64_t size = static_cast<int64_t>(std::ftell(fc.f));
    std::fseek(fc.f, 0, SEEK_SET);
    char magic[4] = {0, 0, 0, 0};
    if (size < 4 || std::fread(magic, 1, 4, fc.f) != 4 || std::memcmp(magic, "TDNB", 4) != 0)
      fail(CPDGPU_PARSE_ERROR, "%s: bad magic at byte 0", path);
    auto u32 = [&](int64_t at, const char* what) {
      unsigned char b[4];
      if (at + 4 > size || std::fread(b, 1, 4, fc.f) != 4) fail(CPDGPU_PARSE_ERROR, "%s: truncated %s at byte %lld", path, what, (long long)at);
      return static_cast<uint32_t>(b[0]) | (static_cast<uint32_t>(b[1]) << 8) | (static_cast<uint32_t>(b[2]) << 16) |
             (static_cast<uint32_t>(b[3]) << 24);
    };
    const uint32_t n = u32(4, "order");
    if (n < 1 || n > 64) fail(CPDGPU_PARSE_ERROR, "%s: implausible order at byte 4", path);
    if (n > static_cast<uint32_t>(kMaxModes)) fail(CPDGPU_ARGUMENT_ERROR, "%s: order %u above %d", path, n, kMaxModes);
    std::vector<int64_t> dims(n);
    for (uint32_t k = 0; k < n; ++k) {
      const int64_t at = 8 + 4 * static_cast<int64_t>(k);
      const uint32_t d = u32(at, "dimension");
      if (d < 1) fail(CPDGPU_PARSE_ERROR, "%s: nonpositive dimension at byte %lld", path, (long long)at);
      dims[k] = d;
    }
    const int64_t head = 8 + 4 * static_cast<int64_t>(n);
    const int64_t numel = prefix(dims).back();
    const int64_t want = head + 8 * numel;
    if (size < want) {  // the first value that is not complete
      const int64_t at = head + 8 * ((size - head) / 8);
      fail(CPDGPU_PARSE_ERROR, "%s: truncated value at byte %lld", path, (long long)at);
    }
    if (size > want) fail(CPDGPU_PARSE_ERROR, "%s: trailing data at byte %lld", path, (long long)want);
    // slab of the last mode
    const int64_t last = dims[n - 1];
    int64_t lo = 0, hi = last;
    if (slab_hi > slab_lo) {
      if (slab_lo < 0 || slab_hi > last)
        fail(CPDGPU_INDEX_ERROR, "%s: slab [%lld, %lld) outside the last mode 0..%lld", path, (long long)slab_lo,
             (long long)slab_hi, (long long)last);
      lo = slab_lo;
      hi = slab_hi;
    }
    const int64_t plane = numel / last;
    std::vector<int64_t> ld = dims;
    ld[n - 1] = hi - lo;
    std::unique_ptr<cpdgpu_tensor> t(new_tensor(ctx, CPDGPU_F64, static_cast<int>(n), ld.data()));
    const size_t bytes = static_cast<size_t>(t->numel) * 8;
    CK(cudaMalloc(&t->data, bytes));
    t->owned = true;
    // file -> pinned (double-buffered) -> device; the host reads chunk i + 1 while chunk i copies
    const size_t chunk = std::min<size_t>(bytes, size_t(64) << 20);
    PinnedBuf pb[2];
    cudaEvent_t done[2];
    for (int b = 0; b < 2; ++b) {
      CK(cudaHostAlloc(&pb[b].p, std::max<size_t>(chunk, 8), cudaHostAllocDefault));
      CK(cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming));
    }
    std::fseek(fc.f, static_cast<long>(head + 8 * lo * plane), SEEK_SET);
    size_t at = 0;
    int b = 0;
    bool used[2] = {false, false};
    while (at < bytes) {
      const size_t len = std::min(chunk, bytes - at);
      if (used[b]) CK(cudaEventSynchronize(done[b]));
      if (std::fread(pb[b].p, 1, len, fc.f) != len)
        fail(CPDGPU_PARSE_ERROR, "%s: read failed at byte %lld", path, (long long)(head + 8 * lo * plane + at));
      CK(cudaMemcpyAsync(static_cast<char*>(t->data) + at, pb[b].p, len, cudaMemcpyHostToDevice, ctx->stream));
      CK(cudaEventRecord(done[b], ctx->stream));
      used[b] = true;
      at += len;
      b ^= 1;
    }
    CK(cudaStreamSynchronize(ctx->stream));
    for (int k = 0; k < 2; ++k) cudaEventDestroy(done[k]);
    t->sorted = t->identity ? t->data : nullptr;
    t->sorted_ready = t->identity;
    *out = t.release();
  });
}

int cpdgpu_tensor_save_tdnb(cpdgpu_ctx* ctx, const cpdgpu_tensor* t, const char* path) {
  return guarded(ctx, [&] {
    if (!ctx || !t || !path) fail(CPDGPU_ARGUMENT_ERROR, "save_tdnb: null argument");
    use_device(ctx);
    for (int64_t d : t->dims)
      if (d > 0xFFFFFFFFll) fail(CPDGPU_ARGUMENT_ERROR, "%s: dimension too large for binary format", path);
    FileCloser fc{std::fopen(path, "wb")};
    if (!fc.f) fail(CPDGPU_ARGUMENT_ERROR, "%s: cannot open for writing", path);
    std::vector<unsigned char> head;
    head.insert(head.end(), {'T', 'D', 'N', 'B'});
    auto put32 = [&](uint32_t v) {
      for (int k = 0; k < 4; ++k) head.push_back(static_cast<unsigned char>(v >> (8 * k)));
    };
    put32(static_cast<uint32_t>(t->dims.size()));
    for (int64_t d : t->dims) put32(static_cast<uint32_t>(d));
    if (std::fwrite(head.data(), 1, head.size(), fc.f) != head.size()) fail(CPDGPU_ARGUMENT_ERROR, "%s: write failed", path);
    const size_t chunk_el = size_t(8) << 20;  // elements per chunk
    PinnedBuf pb, wide;
    CK(cudaHostAlloc(&pb.p, chunk_el * t->elem(), cudaHostAllocDefault));
    if (t->dtype == CPDGPU_F32) CK(cudaHostAlloc(&wide.p, chunk_el * 8, cudaHostAllocDefault));
    for (int64_t at = 0; at < t->numel; at += static_cast<int64_t>(chunk_el)) {
      const size_t n = static_cast<size_t>(std::min<int64_t>(static_cast<int64_t>(chunk_el), t->numel - at));
      CK(cudaMemcpyAsync(pb.p, static_cast<const char*>(t->data) + at * t->elem(), n * t->elem(),
                         cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      const void* src = pb.p;
      if (t->dtype == CPDGPU_F32) {  // exact widening to the file's f64
        const float* f = static_cast<const float*>(pb.p);
        double* w = static_cast<double*>(wide.p);
        for (size_t k = 0; k < n; ++k) w[k] = static_cast<double>(f[k]);
        src = wide.p;
      }
      if (std::fwrite(src, 8, n, fc.f) != n) fail(CPDGPU_ARGUMENT_ERROR, "%s: write failed", path);
    }
  });
}

// Uniform01 (rng.hpp:9-26): std::mt19937_64 seeded with the splitmix of the seed,
// 53-bit doubles in [0, 1); the reference's generate_problem / random_init draws.
int cpdgpu_uniform01_fill(uint64_t seed, int64_t n, double* out) {
  return guarded(nullptr, [&] {
    if (n > 0 && !out) fail(CPDGPU_ARGUMENT_ERROR, "uniform01_fill: null output");
    uint64_t x = seed + 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    std::mt19937_64 eng(x ^ (x >> 31));
    for (int64_t i = 0; i < n; ++i) out[i] = static_cast<double>(eng() >> 11) * 0x1.0p-53;
  });
}

// cost(y, model) (kruskal.cpp:58-77) on the device by the Gram identity:
// |Y|^2 - 2 <Y, Yhat> + 1^T (hadamard of the Grams) 1, <Y, Yhat> = sum A_n .* M_n
// with one direct MTTKRP (sorted mode 1, the cheapest side).
int cpdgpu_cost(cpdgpu_ctx* ctx, cpdgpu_tensor* y, int64_t R, const double* const* factors, double* out) {
  return guarded(ctx, [&] {
    validate_common(ctx, y, R, "cost");
    if (!factors || !out) fail(CPDGPU_ARGUMENT_ERROR, "cost: null argument");
    if (R > 64) fail(CPDGPU_ARGUMENT_ERROR, "cost: rank above the device limit 64");
    ensure_sorted(ctx, y);
    Plan& pl = *get_plan(ctx, y, R, 0);
    bind_seed_inputs(ctx, pl, y);
    upload_host_factors(ctx, pl, y, factors);
    prepare_als(ctx, pl, y);
    pl.costs.ensure(sizeof(double));
    direct_body_fs(ctx, pl, pl.perm[0]);
    als_cost(ctx, pl, pl.costs.d(), 1);
    CK(cudaMemcpyAsync(out, pl.costs.d(), sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

int cpdgpu_select_pivot(int N, const int64_t* dims, int* pivot) {
  return guarded(nullptr, [&] {
    if (!dims || !pivot || N < 0) fail(CPDGPU_ARGUMENT_ERROR, "select_pivot: null argument");
    *pivot = select_pivot(std::vector<int64_t>(dims, dims + N));
  });
}

int cpdgpu_sort_modes(int N, const int64_t* dims, int* perm, int* inverse) {
  return guarded(nullptr, [&] {
    if (!dims || !perm || N < 1) fail(CPDGPU_ARGUMENT_ERROR, "sort_modes: bad argument");
    const auto p = sort_perm(std::vector<int64_t>(dims, dims + N));
    for (int j = 0; j < N; ++j) {
      perm[j] = p[j];
      if (inverse) inverse[p[j] - 1] = j + 1;
    }
  });
}

int cpdgpu_fast_update_order(int N, const int64_t* dims, int* order) {
  return guarded(nullptr, [&] {
    if (!dims || !order) fail(CPDGPU_ARGUMENT_ERROR, "fast_update_order: null argument");
    if (N < 2) fail(CPDGPU_ARGUMENT_ERROR, "fast_update_order: need an order-2 or higher shape");
    const std::vector<int64_t> d(dims, dims + N);
    const auto perm = sort_perm(d);
    std::vector<int64_t> sd(N);
    for (int j = 0; j < N; ++j) sd[j] = d[perm[j] - 1];
    const int p = select_pivot(sd);
    int at = 0;
    for (int j = p; j >= 1; --j) order[at++] = perm[j - 1];
    for (int j = p + 1; j <= N; ++j) order[at++] = perm[j - 1];
  });
}

int cpdgpu_reference_workspace(int N, const int64_t* dims, int64_t R, int64_t* out) {
  return guarded(nullptr, [&] {
    if (!dims || !out || N < 2 || R < 1) fail(CPDGPU_ARGUMENT_ERROR, "reference_workspace: bad argument");
    const std::vector<int64_t> d(dims, dims + N);
    if (!ascending(d)) fail(CPDGPU_ARGUMENT_ERROR, "reference_workspace: dims must be ascending");
    *out = reference_peak_workspace(d, select_pivot(d), R);
  });
}

// predicted_mult_count (mttkrp.cpp:255-290), restated over J_k = prod_{m<=k} I_m.
int cpdgpu_predicted_mult_count(int N, const int64_t* dims, int64_t R, int n, int variant, uint64_t* out) {
  return guarded(nullptr, [&] {
    if (!dims || !out || N < 1) fail(CPDGPU_ARGUMENT_ERROR, "predicted_mult_count: null argument");
    if (n < 1 || n > N) fail(CPDGPU_INDEX_ERROR, "predicted_mult_count: mode %d outside 1..%d", n, N);
    if (R < 1) fail(CPDGPU_ARGUMENT_ERROR, "predicted_mult_count: rank must be positive");
    const std::vector<int64_t> d(dims, dims + N);
    if (!ascending(d)) fail(CPDGPU_ARGUMENT_ERROR, "predicted_mult_count: dims must be ascending");
    if (variant < 0 || variant > 2) fail(CPDGPU_ARGUMENT_ERROR, "predicted_mult_count: unknown variant %d", variant);
    const auto J = prefix(d);
    auto sumj = [&](int lo, int hi, int64_t div) {
      uint64_t t = 0;
      for (int k = std::max(lo, 0); k <= hi; ++k) t += static_cast<uint64_t>(J[k] / div);
      return t;
    };
    auto K = [&](int m) { return static_cast<uint64_t>(J[N] / J[m]); };
    const uint64_t uR = static_cast<uint64_t>(R), JN = static_cast<uint64_t>(J[N]);
    if (variant == 0) {  // unfold + multiply, plus the Kronecker build-up
      *out = uR * (JN + sumj(2, n - 1, 1) + sumj(n + 1, N, d[n - 1]));
      return;
    }
    const int p = select_pivot(d);
    if (n == p || n == p + 1) {
      const uint64_t pivot_term = std::min<uint64_t>(static_cast<uint64_t>(J[n]), K(n - 1));
      *out = uR * (sumj(2, n - 1, 1) + pivot_term + sumj(n + 2, N, J[n]) + JN);
    } else if (n < p) {
      *out = uR * sumj(2, n + 1, 1);
    } else {  // n > p + 1: `fast` keeps the trailing J_k raw, `fast_derived` divides by J_n
      *out = uR * (K(n - 2) + K(n - 1) + (variant == 1 ? sumj(n + 2, N, 1) : sumj(n + 2, N, J[n])));
    }
  });
}

uint64_t cpdgpu_fast_count_realized(int N, const int64_t* dims, int64_t R, int n) {
  try {
    if (!dims || N < 2 || R < 1 || n < 1 || n > N) return 0;
    const std::vector<int64_t> d(dims, dims + N);
    if (!ascending(d)) return 0;
    return count_realized(d, R, n);
  } catch (...) {
    return 0;
  }
}

int cpdgpu_cp_gradient_all(cpdgpu_ctx* ctx, cpdgpu_tensor* y, int64_t R, const double* const* factors,
                           double* const* gradients, uint64_t* mults_per_mode, int64_t* peak_workspace) {
  return guarded(ctx, [&] {
    validate_common(ctx, y, R, "cp_gradient_all");
    if (!factors || !gradients) fail(CPDGPU_ARGUMENT_ERROR, "cp_gradient_all: null factor or gradient list");
    ensure_sorted(ctx, y);
    Plan& pl = *get_plan(ctx, y, R, 0);
    bind_seed_inputs(ctx, pl, y, true);
    if (pl.i8.tensor_ok) i8_apply_factor_guard(pl, i8_factors_ok_host(pl, factors, true, i8_factor_limit(y)));
    upload_host_factors(ctx, pl, y, factors);
    run_gradient(ctx, pl, pl.Forig.d(), pl.Gorig.d());
    CK(cudaMemcpyAsync(pl.hG.d(), pl.Gorig.d(), static_cast<size_t>(pl.total_factor) * sizeof(double),
                       cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (int m = 0; m < pl.N; ++m)
      std::memcpy(gradients[m], pl.hG.d() + pl.off_orig[m],
                  static_cast<size_t>(y->dims[m] * R) * sizeof(double));
    if (mults_per_mode)
      for (int j = 1; j <= pl.N; ++j) mults_per_mode[pl.perm[j - 1] - 1] = count_realized(pl.sd, R, j);
    if (peak_workspace) *peak_workspace = reference_peak_workspace(pl.sd, pl.p, R);
  });
}

int cpdgpu_cp_gradient_all_hook(cpdgpu_ctx* ctx, cpdgpu_tensor* y, int64_t R, double* const* factors,
                                double* const* gradients, cpdgpu_mode_hook hook, void* user,
                                int64_t* peak_workspace) {
  return guarded(ctx, [&] {
    validate_common(ctx, y, R, "cp_gradient_all");
    if (!factors || !gradients) fail(CPDGPU_ARGUMENT_ERROR, "cp_gradient_all: null factor or gradient list");
    ensure_sorted(ctx, y);
    Plan& pl = *get_plan(ctx, y, R, 0);
    bind_seed_inputs(ctx, pl, y);
    upload_host_factors(ctx, pl, y, factors);
    gather_factors(ctx, pl, pl.Forig.d());
    set_gtab(ctx, pl, pl.Gorig.d());
    // emit (mttkrp.cpp:134-145): gradient out, counter charge, hook, re-read factor
    auto emit = [&](int j) {
      const int orig = pl.perm[j - 1];
      const int64_t rows = pl.sd[j - 1];
      const size_t bytes = static_cast<size_t>(rows * R) * sizeof(double);
      CK(cudaMemcpyAsync(gradients[orig - 1], pl.Gorig.d() + pl.off_orig[orig - 1], bytes, cudaMemcpyDeviceToHost,
                         ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      if (hook) {
        const int st = hook(user, orig, gradients[orig - 1], rows, R, count_realized(pl.sd, R, j));
        if (st != 0) fail(st, "cp_gradient_all: hook for mode %d failed", orig);
        CK(cudaMemcpyAsync(pl.factor(j), factors[orig - 1], bytes, cudaMemcpyHostToDevice, ctx->stream));
      }
    };
    // The left seed must see factors the hook replaced on the right side
    // (mttkrp.cpp:143, 203): two seed passes, as in the ALS sweep.
    sweep_body(ctx, pl, emit);
    CK(cudaStreamSynchronize(ctx->stream));
    if (peak_workspace) *peak_workspace = reference_peak_workspace(pl.sd, pl.p, R);
  });
}

int cpdgpu_cp_gradient_all_device(cpdgpu_ctx* ctx, cpdgpu_tensor* y, int64_t R, const double* factors_dev,
                                  double* gradients_dev, int pivot) {
  return guarded(ctx, [&] {
    validate_common(ctx, y, R, "cp_gradient_all");
    if (!factors_dev || !gradients_dev) fail(CPDGPU_ARGUMENT_ERROR, "cp_gradient_all: null device buffer");
    if (pivot < 0 || pivot > static_cast<int>(y->dims.size()))
      fail(CPDGPU_ARGUMENT_ERROR, "cp_gradient_all: pivot %d outside 0..%zu", pivot, y->dims.size());
    if (pivot == 0) ensure_sorted(ctx, y);
    Plan& pl = *get_plan(ctx, y, R, pivot);
    bind_seed_inputs(ctx, pl, y, true);
    i8_device_guard(ctx, pl, factors_dev, y);
    run_gradient(ctx, pl, factors_dev, gradients_dev);
    CK(cudaGetLastError());
  });
}

int cpdgpu_mttkrp_direct(cpdgpu_ctx* ctx, cpdgpu_tensor* y, int64_t R, const double* const* factors, int n,
                         double* out, uint64_t* mults) {
  return guarded(ctx, [&] {
    validate_common(ctx, y, R, "mttkrp_direct");
    const int N = static_cast<int>(y->dims.size());
    if (n < 1 || n > N) fail(CPDGPU_INDEX_ERROR, "mttkrp_direct: mode %d outside 1..%d", n, N);
    if (!factors || !out) fail(CPDGPU_ARGUMENT_ERROR, "mttkrp_direct: null factor list or output");
    Plan& pl = direct_plan(ctx, y, R);
    upload_host_factors(ctx, pl, y, factors);
    direct_body(ctx, pl, pl.Forig.d(), pl.Gorig.d(), n);
    CK(cudaMemcpyAsync(out, pl.Gorig.d() + pl.off_orig[n - 1], static_cast<size_t>(y->dims[n - 1] * R) * sizeof(double),
                       cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (mults) *mults = direct_count(y->dims, R, n);
  });
}

int cpdgpu_mttkrp_direct_device(cpdgpu_ctx* ctx, cpdgpu_tensor* y, int64_t R, const double* factors_dev, int n,
                                double* gradients_dev) {
  return guarded(ctx, [&] {
    validate_common(ctx, y, R, "mttkrp_direct");
    const int N = static_cast<int>(y->dims.size());
    if (n < 1 || n > N) fail(CPDGPU_INDEX_ERROR, "mttkrp_direct: mode %d outside 1..%d", n, N);
    if (!factors_dev || !gradients_dev) fail(CPDGPU_ARGUMENT_ERROR, "mttkrp_direct: null device buffer");
    Plan& pl = direct_plan(ctx, y, R);
    direct_body(ctx, pl, factors_dev, gradients_dev, n);
  });
}

int cpdgpu_als_sweep_direct(cpdgpu_ctx* ctx, cpdgpu_tensor* y, int64_t R, double* const* factors, const int* order,
                            int norder, double pinv_rtol, uint64_t* mults) {
  return guarded(ctx, [&] {
    validate_common(ctx, y, R, "als_sweep_direct");
    const int N = static_cast<int>(y->dims.size());
    if (!factors || (norder > 0 && !order)) fail(CPDGPU_ARGUMENT_ERROR, "als_sweep_direct: null argument");
    if (pinv_rtol < 0.0) fail(CPDGPU_ARGUMENT_ERROR, "pinv_psd: rtol must be nonnegative");
    if (R > 64) fail(CPDGPU_ARGUMENT_ERROR, "als_sweep_direct: rank above the device ALS limit 64");
    uint64_t total = 0;
    std::vector<double> m;
    for (int i = 0; i < norder; ++i) {  // als.cpp:58-67: each update sees the previous ones
      const int n = order[i];
      if (n < 1 || n > N) fail(CPDGPU_INDEX_ERROR, "als_sweep_direct: mode %d outside 1..%d", n, N);
      m.resize(static_cast<size_t>(y->dims[n - 1] * R));
      uint64_t c = 0;
      int st = cpdgpu_mttkrp_direct(ctx, y, R, factors, n, m.data(), &c);
      if (st != CPDGPU_OK) fail(st, "%s", ctx->err.c_str());
      total += c;
      st = cpdgpu_als_update_mode(ctx, N, y->dims.data(), R, m.data(), factors, n, pinv_rtol, factors[n - 1]);
      if (st != CPDGPU_OK) fail(st, "%s", ctx->err.c_str());
    }
    if (mults) *mults = total;
  });
}

int cpdgpu_mu_sweep(cpdgpu_ctx* ctx, cpdgpu_tensor* y, int64_t R, double* const* factors, double eps,
                    uint64_t* mults) {
  return guarded(ctx, [&] {
    validate_common(ctx, y, R, "mu_sweep");
    if (!factors) fail(CPDGPU_ARGUMENT_ERROR, "mu_sweep: null factor list");
    if (eps < 0.0) fail(CPDGPU_ARGUMENT_ERROR, "mu_sweep: eps must be nonnegative");
    if (R > 64) fail(CPDGPU_ARGUMENT_ERROR, "mu_sweep: rank above the device limit 64");
    ensure_sorted(ctx, y);
    Plan& pl = *get_plan(ctx, y, R, 0);
    bind_seed_inputs(ctx, pl, y);
    check_nonneg_inputs(ctx, pl, y, factors);
    upload_host_factors(ctx, pl, y, factors);
    prepare_als(ctx, pl, y);
    mu_sweep_device(ctx, pl, eps);
    CK(cudaStreamSynchronize(ctx->stream));
    download_factors(ctx, pl, y, factors);
    if (mults) {
      *mults = 0;
      for (int j = 1; j <= pl.N; ++j) *mults += count_realized(pl.sd, R, j);
    }
  });
}

int cpdgpu_gd_step(cpdgpu_ctx* ctx, cpdgpu_tensor* y, int64_t R, double* const* factors, double eta,
                   uint64_t* mults) {
  return guarded(ctx, [&] {
    validate_common(ctx, y, R, "gd_step");
    if (!factors) fail(CPDGPU_ARGUMENT_ERROR, "gd_step: null factor list");
    if (!(eta >= 0.0)) fail(CPDGPU_ARGUMENT_ERROR, "gd_step: eta must be nonnegative");
    if (R > 64) fail(CPDGPU_ARGUMENT_ERROR, "gd_step: rank above the device limit 64");
    ensure_sorted(ctx, y);
    Plan& pl = *get_plan(ctx, y, R, 0);
    bind_seed_inputs(ctx, pl, y);
    upload_host_factors(ctx, pl, y, factors);
    prepare_als(ctx, pl, y);
    gd_step_device(ctx, pl, eta);
    CK(cudaStreamSynchronize(ctx->stream));
    download_factors(ctx, pl, y, factors);
    if (mults) {
      *mults = 0;
      for (int j = 1; j <= pl.N; ++j) *mults += count_realized(pl.sd, R, j);
    }
  });
}

int cpdgpu_run_algo(cpdgpu_ctx* ctx, cpdgpu_tensor* y, int64_t R, double* const* factors, int algo,
                    int order_pivot, int max_iters, double tol, double pinv_rtol, double mu_eps, double gd_eta,
                    double* cost_trace, double* rel_trace, double* sec_trace, uint64_t* mults_trace,
                    int* iters_run) {
  if (algo == 1)
    return cpdgpu_als_run(ctx, y, R, factors, max_iters, tol, pinv_rtol, cost_trace, rel_trace, sec_trace,
                          mults_trace, iters_run);
  return guarded(ctx, [&] {
    validate_common(ctx, y, R, "run");
    if (algo < 0 || algo > 3) fail(CPDGPU_ARGUMENT_ERROR, "run: unknown algorithm %d", algo);
    if (max_iters < 1) fail(CPDGPU_ARGUMENT_ERROR, "run: max_iters must be at least 1");
    if (tol < 0.0 || pinv_rtol < 0.0 || mu_eps < 0.0) fail(CPDGPU_ARGUMENT_ERROR, "run: tolerances must be nonnegative");
    if (algo == 3 && !(gd_eta >= 0.0)) fail(CPDGPU_ARGUMENT_ERROR, "gd_step: eta must be nonnegative");
    if (!factors || !cost_trace || !rel_trace || !iters_run) fail(CPDGPU_ARGUMENT_ERROR, "run: null argument");
    if (R > 64) fail(CPDGPU_ARGUMENT_ERROR, "run: rank above the device ALS limit 64");
    ensure_sorted(ctx, y);
    Plan& pl = *get_plan(ctx, y, R, 0);
    bind_seed_inputs(ctx, pl, y);
    if (algo == 2) check_nonneg_inputs(ctx, pl, y, factors);
    upload_host_factors(ctx, pl, y, factors);
    prepare_als(ctx, pl, y);
    pl.costs.ensure(static_cast<size_t>(max_iters) * sizeof(double));
    // als_direct visits caller modes 1..N or fast_update_order (als.cpp:168-170)
    std::vector<int> order(static_cast<size_t>(pl.N));
    std::iota(order.begin(), order.end(), 1);
    if (algo == 0 && order_pivot) {
      std::vector<int> o(static_cast<size_t>(pl.N));
      cpdgpu_fast_update_order(static_cast<int>(y->dims.size()), y->dims.data(), o.data());
      order = o;
    }
    uint64_t per_sweep = 0;
    if (algo == 0)
      for (int n : order) per_sweep += direct_count(y->dims, R, n);
    else
      for (int j = 1; j <= pl.N; ++j) per_sweep += count_realized(pl.sd, R, j);
    std::vector<cudaEvent_t> ev(2 * static_cast<size_t>(max_iters));
    for (auto& e : ev) CK(cudaEventCreate(&e));
    const double ynorm = std::sqrt(y->norm2);
    double prev = std::nan("");
    int done = 0;
    for (int it = 1; it <= max_iters; ++it) {
      CK(cudaEventRecord(ev[2 * (it - 1)], ctx->stream));
      if (algo == 0) direct_sweep_device(ctx, pl, order, pinv_rtol);
      else if (algo == 2) mu_sweep_device(ctx, pl, mu_eps);
      else gd_step_device(ctx, pl, gd_eta);
      CK(cudaEventRecord(ev[2 * (it - 1) + 1], ctx->stream));
      algo_cost(ctx, pl, algo, order, pl.costs.d() + (it - 1));
      ++done;
      if (tol > 0.0) {
        double d = 0.0;
        CK(cudaMemcpyAsync(&d, pl.costs.d() + (it - 1), sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        if (it > 1 && std::abs(d - prev) / std::max(prev, 1e-15) < tol) break;
        prev = d;
      }
    }
    CK(cudaStreamSynchronize(ctx->stream));
    check_status(ctx, pl);
    CK(cudaMemcpy(cost_trace, pl.costs.d(), static_cast<size_t>(done) * sizeof(double), cudaMemcpyDeviceToHost));
    for (int i = 0; i < done; ++i) {
      rel_trace[i] = ynorm > 0.0 ? std::sqrt(cost_trace[i]) / ynorm : std::sqrt(cost_trace[i]);
      if (sec_trace) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ev[2 * i], ev[2 * i + 1]));
        sec_trace[i] = ms * 1e-3;
      }
      if (mults_trace) mults_trace[i] = per_sweep * static_cast<uint64_t>(i + 1);
    }
    for (auto& e : ev) cudaEventDestroy(e);
    *iters_run = done;
    download_factors(ctx, pl, y, factors);
  });
}

int cpdgpu_pinv_psd(cpdgpu_ctx* ctx, int64_t R, const double* s, double rtol, double* out) {
  return guarded(ctx, [&] {
    if (!ctx || (R > 0 && (!s || !out))) fail(CPDGPU_ARGUMENT_ERROR, "pinv_psd: null argument");
    if (rtol < 0.0) fail(CPDGPU_ARGUMENT_ERROR, "pinv_psd: rtol must be nonnegative");
    if (R > 64) fail(CPDGPU_ARGUMENT_ERROR, "pinv_psd: rank %lld above the device limit 64", (long long)R);
    if (R == 0) return;
    use_device(ctx);
    DevBuf d;
    d.ensure(2 * static_cast<size_t>(R * R) * sizeof(double));
    CK(cudaMemcpyAsync(d.d(), s, static_cast<size_t>(R * R) * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    ctx->launches += cpdgpu::launch_pinv_psd(d.d(), static_cast<int>(R), rtol, d.d() + R * R, ctx->stream);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, d.d() + R * R, static_cast<size_t>(R * R) * sizeof(double), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

int cpdgpu_als_update_mode(cpdgpu_ctx* ctx, int N, const int64_t* dims, int64_t R, const double* m,
                           const double* const* factors, int n, double rtol, double* out) {
  return guarded(ctx, [&] {
    if (!ctx || !dims || !m || !factors || !out) fail(CPDGPU_ARGUMENT_ERROR, "als_update_mode: null argument");
    if (n < 1 || n > N) fail(CPDGPU_INDEX_ERROR, "als_update_mode: mode %d outside 1..%d", n, N);
    if (R < 1 || R > 64) fail(CPDGPU_ARGUMENT_ERROR, "als_update_mode: rank %lld outside 1..64", (long long)R);
    if (rtol < 0.0) fail(CPDGPU_ARGUMENT_ERROR, "pinv_psd: rtol must be nonnegative");
    use_device(ctx);
    int64_t total = 0;
    for (int k = 0; k < N; ++k) total += dims[k] * R;
    DevBuf F, G, grams, st;
    F.ensure(static_cast<size_t>(total) * sizeof(double));
    G.ensure(static_cast<size_t>(dims[n - 1] * R) * sizeof(double) * 2);
    grams.ensure(static_cast<size_t>(N + 1) * R * R * sizeof(double));
    st.ensure(sizeof(int));
    CK(cudaMemsetAsync(st.p, 0, sizeof(int), ctx->stream));
    int64_t off = 0;
    for (int k = 0; k < N; ++k) {
      CK(cudaMemcpyAsync(F.d() + off, factors[k], static_cast<size_t>(dims[k] * R) * sizeof(double),
                         cudaMemcpyHostToDevice, ctx->stream));
      ctx->launches += cpdgpu::launch_gram(F.d() + off, dims[k], static_cast<int>(R), grams.d() + k * R * R,
                                           ctx->stream);
      off += dims[k] * R;
    }
    const size_t gb = static_cast<size_t>(dims[n - 1] * R) * sizeof(double);
    CK(cudaMemcpyAsync(G.d(), m, gb, cudaMemcpyHostToDevice, ctx->stream));
    double* A = G.d() + dims[n - 1] * R;
    ctx->launches += cpdgpu::launch_als_update(G.d(), dims[n - 1], static_cast<int>(R), grams.d(), N, n - 1, rtol,
                                               A, grams.d() + N * R * R, static_cast<int*>(st.p), ctx->stream);
    CK(cudaGetLastError());
    int status = 0;
    CK(cudaMemcpyAsync(&status, st.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(out, A, gb, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (status == 4) fail(CPDGPU_NUMERIC_ERROR, "als_update_mode: non-finite gradient input");
  });
}

int cpdgpu_als_sweep(cpdgpu_ctx* ctx, cpdgpu_tensor* y, int64_t R, double* const* factors, double pinv_rtol,
                     double* cost_out, uint64_t* mults) {
  return guarded(ctx, [&] {
    validate_common(ctx, y, R, "als_sweep_fast");
    if (!factors) fail(CPDGPU_ARGUMENT_ERROR, "als_sweep_fast: null factor list");
    if (pinv_rtol < 0.0) fail(CPDGPU_ARGUMENT_ERROR, "pinv_psd: rtol must be nonnegative");
    if (R > 64) fail(CPDGPU_ARGUMENT_ERROR, "als_sweep_fast: rank above the device ALS limit 64");
    ensure_sorted(ctx, y);
    Plan& pl = *get_plan(ctx, y, R, 0);
    bind_seed_inputs(ctx, pl, y);
    upload_host_factors(ctx, pl, y, factors);
    prepare_als(ctx, pl, y);
    pl.costs.ensure(sizeof(double));
    als_sweep_graph(ctx, pl, pinv_rtol);
    als_cost(ctx, pl, pl.costs.d());
    check_status(ctx, pl);
    download_factors(ctx, pl, y, factors);
    if (cost_out) CK(cudaMemcpy(cost_out, pl.costs.d(), sizeof(double), cudaMemcpyDeviceToHost));
    if (mults) {
      uint64_t tot = 0;
      for (int j = 1; j <= pl.N; ++j) tot += count_realized(pl.sd, R, j);
      *mults = tot;
    }
  });
}

int cpdgpu_als_run(cpdgpu_ctx* ctx, cpdgpu_tensor* y, int64_t R, double* const* factors, int max_iters,
                   double tol, double pinv_rtol, double* cost_trace, double* rel_trace, double* sec_trace,
                   uint64_t* mults_trace, int* iters_run) {
  return guarded(ctx, [&] {
    validate_common(ctx, y, R, "run");
    if (max_iters < 1) fail(CPDGPU_ARGUMENT_ERROR, "run: max_iters must be at least 1");
    if (tol < 0.0 || pinv_rtol < 0.0) fail(CPDGPU_ARGUMENT_ERROR, "run: tolerances must be nonnegative");
    if (!factors || !cost_trace || !rel_trace || !iters_run) fail(CPDGPU_ARGUMENT_ERROR, "run: null argument");
    if (R > 64) fail(CPDGPU_ARGUMENT_ERROR, "run: rank above the device ALS limit 64");
    ensure_sorted(ctx, y);
    Plan& pl = *get_plan(ctx, y, R, 0);
    bind_seed_inputs(ctx, pl, y);
    upload_host_factors(ctx, pl, y, factors);
    prepare_als(ctx, pl, y);
    pl.costs.ensure(static_cast<size_t>(max_iters) * sizeof(double));
    uint64_t per_sweep = 0;
    for (int j = 1; j <= pl.N; ++j) per_sweep += count_realized(pl.sd, R, j);
    std::vector<cudaEvent_t> ev(2 * static_cast<size_t>(max_iters));
    for (auto& e : ev) CK(cudaEventCreate(&e));
    const double ynorm = std::sqrt(y->norm2);
    double prev = std::nan("");
    int done = 0;
    for (int it = 1; it <= max_iters; ++it) {
      CK(cudaEventRecord(ev[2 * (it - 1)], ctx->stream));
      als_sweep_graph(ctx, pl, pinv_rtol);
      CK(cudaEventRecord(ev[2 * (it - 1) + 1], ctx->stream));
      als_cost(ctx, pl, pl.costs.d() + (it - 1));
      ++done;
      if (tol > 0.0) {  // early stop needs the fit on the host every sweep
        double d = 0.0;
        CK(cudaMemcpyAsync(&d, pl.costs.d() + (it - 1), sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        if (it > 1 && std::abs(d - prev) / std::max(prev, 1e-15) < tol) break;
        prev = d;
      }
    }
    CK(cudaStreamSynchronize(ctx->stream));
    check_status(ctx, pl);
    CK(cudaMemcpy(cost_trace, pl.costs.d(), static_cast<size_t>(done) * sizeof(double), cudaMemcpyDeviceToHost));
    for (int i = 0; i < done; ++i) {
      rel_trace[i] = ynorm > 0.0 ? std::sqrt(cost_trace[i]) / ynorm : std::sqrt(cost_trace[i]);
      if (sec_trace) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ev[2 * i], ev[2 * i + 1]));
        sec_trace[i] = ms * 1e-3;
      }
      if (mults_trace) mults_trace[i] = per_sweep * static_cast<uint64_t>(i + 1);
    }
    for (auto& e : ev) cudaEventDestroy(e);
    *iters_run = done;
    download_factors(ctx, pl, y, factors);
  });
}

// ---- multi-GPU: last-mode slab sharding ---------------------------

int cpdgpu_comm_unique_id(unsigned char* id) {
  return guarded(nullptr, [&] {
    if (!id) fail(CPDGPU_ARGUMENT_ERROR, "comm_unique_id: null id");
    NcclApi& a = nccl_api();
    if (!a.ok) fail(CPDGPU_CUDA_ERROR, "comm_unique_id: %s", a.why.c_str());
    ncclUniqueId u;
    const ncclResult_t r = a.get_unique_id(&u);
    if (r != ncclSuccess) fail(CPDGPU_CUDA_ERROR, "ncclGetUniqueId: %s", a.error_string(r));
    std::memcpy(id, u.internal, CPDGPU_COMM_ID_BYTES);
  });
}

int cpdgpu_comm_init(cpdgpu_ctx* ctx, const unsigned char* id, int nranks, int rank) {
  return guarded(ctx, [&] {
    if (!ctx || !id) fail(CPDGPU_ARGUMENT_ERROR, "comm_init: null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks)
      fail(CPDGPU_ARGUMENT_ERROR, "comm_init: rank %d outside 0..%d", rank, nranks - 1);
    NcclApi& a = nccl_api();
    if (!a.ok) fail(CPDGPU_CUDA_ERROR, "comm_init: %s", a.why.c_str());
    use_device(ctx);
    auto c = std::make_unique<Comm>();
    c->nranks = nranks;
    c->rank = rank;
    ncclUniqueId u;
    std::memcpy(u.internal, id, CPDGPU_COMM_ID_BYTES);
    const ncclResult_t r = a.init_rank(&c->nccl, nranks, u, rank);
    if (r != ncclSuccess) fail(CPDGPU_CUDA_ERROR, "ncclCommInitRank: %s", a.error_string(r));
    ctx->comm = std::move(c);
  });
}

int cpdgpu_comm_init_host(cpdgpu_ctx* ctx, int nranks, int rank, cpdgpu_allreduce_fn fn, void* user) {
  return guarded(ctx, [&] {
    if (!ctx || !fn) fail(CPDGPU_ARGUMENT_ERROR, "comm_init_host: null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks)
      fail(CPDGPU_ARGUMENT_ERROR, "comm_init_host: rank %d outside 0..%d", rank, nranks - 1);
    auto c = std::make_unique<Comm>();
    c->nranks = nranks;
    c->rank = rank;
    c->host_fn = fn;
    c->user = user;
    ctx->comm = std::move(c);
  });
}

int cpdgpu_comm_destroy(cpdgpu_ctx* ctx) {
  return guarded(ctx, [&] {
    if (!ctx) fail(CPDGPU_ARGUMENT_ERROR, "comm_destroy: null context");
    if (ctx->comm) use_device(ctx);
    ctx->comm.reset();
  });
}

int cpdgpu_slab_bounds(int64_t extent, int nranks, int rank, int64_t* lo, int64_t* hi) {
  return guarded(nullptr, [&] {
    if (!lo || !hi || nranks < 1 || rank < 0 || rank >= nranks || extent < 0)
      fail(CPDGPU_ARGUMENT_ERROR, "slab_bounds: bad argument");
    const int64_t base = extent / nranks, extra = extent % nranks;
    *lo = rank * base + std::min<int64_t>(rank, extra);
    *hi = *lo + base + (rank < extra ? 1 : 0);
  });
}

}  // extern "C"

namespace {

struct ShardGeom {
  std::vector<int64_t> gdims;
  int N = 0, pivot = 0;
  int64_t lo = 0, hi = 0, partial = 0, total = 0;  // packed G(1..N-1) length, + I_N R
};

ShardGeom shard_geometry(cpdgpu_ctx* ctx, cpdgpu_tensor* slab, int N, const int64_t* global_dims, int64_t R,
                         const char* who) {
  if (!ctx || !slab || !global_dims) fail(CPDGPU_ARGUMENT_ERROR, "%s: null argument", who);
  if (!ctx->comm) fail(CPDGPU_ARGUMENT_ERROR, "%s: no communicator (cpdgpu_comm_init)", who);
  ShardGeom g;
  g.N = N;
  g.gdims.assign(global_dims, global_dims + N);
  validate_common(ctx, slab, R, who);
  if (N < 2 || static_cast<int>(slab->dims.size()) != N)
    fail(CPDGPU_SHAPE_ERROR, "%s: slab order %zu, global order %d", who, slab->dims.size(), N);
  for (int k = 0; k + 1 < N; ++k) {
    if (g.gdims[k] < 1 || (k > 0 && g.gdims[k] < g.gdims[k - 1]))
      fail(CPDGPU_ARGUMENT_ERROR, "%s: global dims must be positive and ascending (sort modes first)", who);
    if (slab->dims[k] != g.gdims[k])
      fail(CPDGPU_SHAPE_ERROR, "%s: slab mode %d has extent %lld, global %lld", who, k + 1,
           static_cast<long long>(slab->dims[k]), static_cast<long long>(g.gdims[k]));
  }
  if (g.gdims[N - 1] < g.gdims[N - 2])
    fail(CPDGPU_ARGUMENT_ERROR, "%s: global dims must be ascending (sort modes first)", who);
  const Comm& c = *ctx->comm;
  if (cpdgpu_slab_bounds(g.gdims[N - 1], c.nranks, c.rank, &g.lo, &g.hi) != CPDGPU_OK || g.hi - g.lo < 1)
    fail(CPDGPU_ARGUMENT_ERROR, "%s: last mode %lld has fewer slices than the %d ranks", who,
         static_cast<long long>(g.gdims[N - 1]), c.nranks);
  if (slab->dims[N - 1] != g.hi - g.lo)
    fail(CPDGPU_SHAPE_ERROR, "%s: rank %d holds slices [%lld, %lld) but its slab has %lld", who, c.rank,
         static_cast<long long>(g.lo), static_cast<long long>(g.hi), static_cast<long long>(slab->dims[N - 1]));
  g.pivot = select_pivot(g.gdims);
  if (g.pivot >= N) fail(CPDGPU_ARGUMENT_ERROR, "%s: the pivot is the last mode; nothing to shard", who);
  for (int k = 0; k + 1 < N; ++k) g.partial += g.gdims[k] * R;
  g.total = g.partial + g.gdims[N - 1] * R;
  return g;
}

// In-place sum of `count` device doubles across the communicator, ordered on the
// context stream (NCCL), or staged through host memory for the caller's collective.
void comm_allreduce(cpdgpu_ctx* ctx, double* dev, int64_t count, const char* who) {
  Comm& c = *ctx->comm;
  if (c.nranks == 1) return;
  if (c.nccl) {
    NcclApi& a = nccl_api();
    const ncclResult_t r =
        a.all_reduce(dev, dev, static_cast<size_t>(count), ncclFloat64, ncclSum, c.nccl, ctx->stream);
    if (r != ncclSuccess) fail(CPDGPU_CUDA_ERROR, "%s: ncclAllReduce: %s", who, a.error_string(r));
    return;
  }
  const size_t bytes = static_cast<size_t>(count) * sizeof(double);
  c.hbuf.ensure(bytes);
  CK(cudaMemcpyAsync(c.hbuf.p, dev, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  const int st = c.host_fn(c.user, c.hbuf.d(), count);
  if (st != 0) fail(st > 0 ? st : CPDGPU_CUDA_ERROR, "%s: host all-reduce failed (%d)", who, st);
  CK(cudaMemcpyAsync(dev, c.hbuf.p, bytes, cudaMemcpyHostToDevice, ctx->stream));
}

// local gradient of the slab at the global pivot, then ONE in-place all-reduce of
// [partial G(1..N-1) | G(N) rows placed at the slab's offset] into out_dev
void sharded_device(cpdgpu_ctx* ctx, cpdgpu_tensor* slab, const ShardGeom& g, int64_t R, const double* fdev,
                    double* out_dev) {
  Comm& c = *ctx->comm;
  const int64_t rows = g.hi - g.lo, IN = g.gdims[g.N - 1];
  c.lbuf.ensure(static_cast<size_t>(g.partial + rows * R) * sizeof(double));
  Plan& pl = *get_plan(ctx, slab, R, g.pivot);
  bind_seed_inputs(ctx, pl, slab, true);
  i8_device_guard(ctx, pl, fdev, slab);
  run_gradient(ctx, pl, fdev, c.lbuf.d());
  CK(cudaMemcpyAsync(out_dev, c.lbuf.d(), static_cast<size_t>(g.partial) * sizeof(double), cudaMemcpyDeviceToDevice,
                     ctx->stream));
  CK(cudaMemsetAsync(out_dev + g.partial, 0, static_cast<size_t>(IN * R) * sizeof(double), ctx->stream));
  CK(cudaMemcpy2DAsync(out_dev + g.partial + g.lo, static_cast<size_t>(IN) * sizeof(double), c.lbuf.d() + g.partial,
                       static_cast<size_t>(rows) * sizeof(double), static_cast<size_t>(rows) * sizeof(double),
                       static_cast<size_t>(R), cudaMemcpyDeviceToDevice, ctx->stream));
  comm_allreduce(ctx, out_dev, g.total, "cp_gradient_all_sharded");
}

// ---- sharded fast ALS (als.cpp:69-78 over last-mode slabs) ------------------------
// The sweep keeps its Gauss-Seidel order (the global frame: modes p*..1, then
// p*+1..N).  G(j), j < N, is a linear sum over slabs: one all-reduce of I_j x R
// before A_j's update, identical on every rank, which the recursion then
// consumes.  A_N's rows belong to the slab: the update is local and only its Gram
// (R x R) is summed.  The cost (kruskal.cpp:58-77) needs <Y, Yhat> over A_N's
// rows: one all-reduce of [A_N rows | G(N) rows] placed at the slab offset, which
// also hands every rank the whole updated A_N.

void sharded_als_prepare(cpdgpu_ctx* ctx, Plan& pl, cpdgpu_tensor* slab, const ShardGeom& g,
                         const double* const* factors) {
  const int64_t R = pl.R, rows = g.hi - g.lo;
  for (int m = 0; m + 1 < pl.N; ++m)
    std::memcpy(pl.hF.d() + pl.off_orig[m], factors[m], static_cast<size_t>(g.gdims[m] * R) * sizeof(double));
  for (int64_t r = 0; r < R; ++r)
    std::memcpy(pl.hF.d() + pl.off_orig[pl.N - 1] + r * rows, factors[pl.N - 1] + r * g.gdims[pl.N - 1] + g.lo,
                static_cast<size_t>(rows) * sizeof(double));
  CK(cudaMemcpyAsync(pl.Forig.d(), pl.hF.d(), static_cast<size_t>(pl.total_factor) * sizeof(double),
                     cudaMemcpyHostToDevice, ctx->stream));
  compute_norm2(ctx, slab);  // the slab's ||Y||^2, summed below
  CK(cudaMemcpyAsync(pl.norm.d(), &slab->norm2, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemsetAsync(pl.status.p, 0, sizeof(int), ctx->stream));
  gather_factors(ctx, pl, pl.Forig.d());
  set_gtab(ctx, pl, pl.Gorig.d());
  init_grams(ctx, pl);
  comm_allreduce(ctx, pl.norm.d(), 1, "als_sweep_sharded");
  comm_allreduce(ctx, pl.grams.d() + static_cast<int64_t>(pl.N - 1) * R * R, R * R, "als_sweep_sharded");
}

void sharded_als_sweep(cpdgpu_ctx* ctx, Plan& pl, const ShardGeom& g, double rtol, double* cost_slot) {
  Comm& c = *ctx->comm;
  const int R = static_cast<int>(pl.R);
  const int64_t rows = g.hi - g.lo, IN = g.gdims[pl.N - 1];
  sweep_body(ctx, pl, [&](int j) {
    double* G = pl.Gorig.d() + pl.off_orig[j - 1];  // global frame: sorted j is caller j
    double* gram = pl.grams.d() + static_cast<int64_t>(j - 1) * R * R;
    if (j < pl.N) comm_allreduce(ctx, G, pl.sd[j - 1] * R, "als_sweep_sharded");
    ctx->launches += cpdgpu::launch_als_update(G, pl.sd[j - 1], R, pl.grams.d(), pl.N, j - 1, rtol, pl.factor(j),
                                               gram, static_cast<int*>(pl.status.p), ctx->stream);
    if (j == pl.N) comm_allreduce(ctx, gram, static_cast<int64_t>(R) * R, "als_sweep_sharded");
  });
  // [A_N | G(N)] at the slab offset, zeros elsewhere, summed: whole A_N and G(N)
  c.xbuf.ensure(static_cast<size_t>(2 * IN * R) * sizeof(double));
  double* x = c.xbuf.d();
  CK(cudaMemsetAsync(x, 0, static_cast<size_t>(2 * IN * R) * sizeof(double), ctx->stream));
  const size_t pitch = static_cast<size_t>(IN) * sizeof(double), w = static_cast<size_t>(rows) * sizeof(double);
  CK(cudaMemcpy2DAsync(x + g.lo, pitch, pl.factor(pl.N), w, w, static_cast<size_t>(R), cudaMemcpyDeviceToDevice,
                       ctx->stream));
  CK(cudaMemcpy2DAsync(x + IN * R + g.lo, pitch, pl.Gorig.d() + pl.off_orig[pl.N - 1], w, w, static_cast<size_t>(R),
                       cudaMemcpyDeviceToDevice, ctx->stream));
  comm_allreduce(ctx, x, 2 * IN * R, "als_sweep_sharded");
  if (cost_slot)
    ctx->launches += cpdgpu::launch_als_cost(x, x + IN * R, IN, R, pl.grams.d(), pl.N, pl.norm.d(), cost_slot,
                                             ctx->stream);
}

// Every rank reports the same outcome: a NumericError (status 4, or the int8
// budget fault) on any rank fails the call on all of them.
void sharded_agree(cpdgpu_ctx* ctx, Plan& pl) {
  int st = 0;
  CK(cudaMemcpyAsync(&st, pl.status.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  const int fault = *ctx->fault_host;
  Comm& c = *ctx->comm;
  c.lbuf.ensure(2 * sizeof(double));
  const double flags[2] = {st == 4 ? 1.0 : 0.0, fault != 0 ? 1.0 : 0.0};
  CK(cudaMemcpyAsync(c.lbuf.p, flags, sizeof(flags), cudaMemcpyHostToDevice, ctx->stream));
  comm_allreduce(ctx, c.lbuf.d(), 2, "als_sweep_sharded");
  double any[2] = {0.0, 0.0};
  CK(cudaMemcpyAsync(any, c.lbuf.p, sizeof(any), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (fault) return;  // guarded() reports this rank's own fault
  if (st == 4) fail(CPDGPU_NUMERIC_ERROR, "als_update_mode: non-finite gradient input");
  if (any[0] > 0.0) fail(CPDGPU_NUMERIC_ERROR, "als_sweep_sharded: non-finite gradient input on another rank");
  if (any[1] > 0.0)
    fail(CPDGPU_NUMERIC_ERROR, "als_sweep_sharded: another rank's seed pass failed its check; this sweep is invalid");
}

void sharded_als_download(cpdgpu_ctx* ctx, Plan& pl, const ShardGeom& g, double* const* factors) {
  Comm& c = *ctx->comm;
  const int64_t R = pl.R, IN = g.gdims[pl.N - 1];
  scatter_factors(ctx, pl, pl.Forig.d());
  CK(cudaMemcpyAsync(pl.hF.d(), pl.Forig.d(), static_cast<size_t>(pl.total_factor) * sizeof(double),
                     cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(factors[pl.N - 1], c.xbuf.d(), static_cast<size_t>(IN * R) * sizeof(double),
                     cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  for (int m = 0; m + 1 < pl.N; ++m)
    std::memcpy(factors[m], pl.hF.d() + pl.off_orig[m], static_cast<size_t>(g.gdims[m] * R) * sizeof(double));
}

}  // namespace

extern "C" {

int cpdgpu_cp_gradient_all_sharded_device(cpdgpu_ctx* ctx, cpdgpu_tensor* slab, int N, const int64_t* global_dims,
                                          int64_t R, const double* factors_dev, double* out_dev) {
  return guarded(ctx, [&] {
    const ShardGeom g = shard_geometry(ctx, slab, N, global_dims, R, "cp_gradient_all_sharded");
    if (!factors_dev || !out_dev) fail(CPDGPU_ARGUMENT_ERROR, "cp_gradient_all_sharded: null device buffer");
    sharded_device(ctx, slab, g, R, factors_dev, out_dev);
    CK(cudaGetLastError());
  });
}

int cpdgpu_cp_gradient_all_sharded(cpdgpu_ctx* ctx, cpdgpu_tensor* slab, int N, const int64_t* global_dims,
                                   int64_t R, const double* const* factors, double* const* gradients,
                                   uint64_t* mults) {
  return guarded(ctx, [&] {
    const ShardGeom g = shard_geometry(ctx, slab, N, global_dims, R, "cp_gradient_all_sharded");
    if (!factors || !gradients) fail(CPDGPU_ARGUMENT_ERROR, "cp_gradient_all_sharded: null factor or gradient list");
    Comm& c = *ctx->comm;
    const int64_t rows = g.hi - g.lo;
    // the slab's packed factors: modes 1..N-1 whole, rows [lo, hi) of mode N
    std::vector<double> hf(static_cast<size_t>(g.partial + rows * R));
    for (int64_t m = 0, at = 0; m + 1 < N; ++m) {
      std::memcpy(hf.data() + at, factors[m], static_cast<size_t>(g.gdims[m] * R) * sizeof(double));
      at += g.gdims[m] * R;
    }
    for (int64_t r = 0; r < R; ++r)
      std::memcpy(hf.data() + g.partial + r * rows, factors[N - 1] + r * g.gdims[N - 1] + g.lo,
                  static_cast<size_t>(rows) * sizeof(double));
    c.fbuf.ensure(hf.size() * sizeof(double));
    c.xbuf.ensure(static_cast<size_t>(g.total) * sizeof(double));
    CK(cudaMemcpyAsync(c.fbuf.p, hf.data(), hf.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    sharded_device(ctx, slab, g, R, c.fbuf.d(), c.xbuf.d());
    for (int64_t m = 0, at = 0; m < N; ++m) {
      CK(cudaMemcpyAsync(gradients[m], c.xbuf.d() + at, static_cast<size_t>(g.gdims[m] * R) * sizeof(double),
                         cudaMemcpyDeviceToHost, ctx->stream));
      at += g.gdims[m] * R;
    }
    CK(cudaStreamSynchronize(ctx->stream));
    if (mults)
      for (int m = 0; m < N; ++m) mults[m] = count_realized(g.gdims, R, m + 1);
  });
}

}  // extern "C"

namespace {

// max_iters sharded sweeps (run(), als.cpp:147-210, Algorithm::als_fast) with the
// per-sweep costs in pl.costs; returns the number of sweeps done
int sharded_als_loop(cpdgpu_ctx* ctx, cpdgpu_tensor* slab, const ShardGeom& g, int64_t R,
                     double* const* factors, int max_iters, double tol, double rtol, double* sec_trace) {
  if (R > 64) fail(CPDGPU_ARGUMENT_ERROR, "als_sweep_sharded: rank above the device ALS limit 64");
  if (rtol < 0.0 || tol < 0.0) fail(CPDGPU_ARGUMENT_ERROR, "als_sweep_sharded: tolerances must be nonnegative");
  if (!factors) fail(CPDGPU_ARGUMENT_ERROR, "als_sweep_sharded: null factor list");
  Plan& pl = *get_plan(ctx, slab, R, g.pivot);
  bind_seed_inputs(ctx, pl, slab);
  sharded_als_prepare(ctx, pl, slab, g, factors);
  if (pl.i8.tensor_ok) {
    std::vector<const double*> mf(pl.N);
    for (int m = 0; m < pl.N; ++m) mf[m] = pl.hF.d() + pl.off_orig[m];
    i8_apply_factor_guard(pl, i8_factors_ok_host(pl, mf.data(), true, i8_factor_limit(slab)));
  }
  pl.costs.ensure(static_cast<size_t>(max_iters) * sizeof(double));
  std::vector<cudaEvent_t> ev(sec_trace ? 2 * static_cast<size_t>(max_iters) : 0);
  for (auto& e : ev) CK(cudaEventCreate(&e));
  struct Free {
    std::vector<cudaEvent_t>& v;
    ~Free() {
      for (auto e : v) cudaEventDestroy(e);
    }
  } free_events{ev};
  double prev = std::nan("");
  int done = 0;
  for (int it = 1; it <= max_iters; ++it) {
    if (sec_trace) CK(cudaEventRecord(ev[2 * (it - 1)], ctx->stream));
    sharded_als_sweep(ctx, pl, g, rtol, pl.costs.d() + (it - 1));
    if (sec_trace) CK(cudaEventRecord(ev[2 * (it - 1) + 1], ctx->stream));
    ++done;
    if (tol > 0.0) {  // the cost is global, so every rank stops at the same sweep
      double d = 0.0;
      CK(cudaMemcpyAsync(&d, pl.costs.d() + (it - 1), sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      if (it > 1 && std::abs(d - prev) / std::max(prev, 1e-15) < tol) break;
      prev = d;
    }
  }
  sharded_agree(ctx, pl);
  for (int i = 0; sec_trace && i < done; ++i) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, ev[2 * i], ev[2 * i + 1]));
    sec_trace[i] = ms * 1e-3;
  }
  sharded_als_download(ctx, pl, g, factors);
  return done;
}

uint64_t als_sweep_count(const std::vector<int64_t>& dims, int64_t R) {
  uint64_t tot = 0;
  for (int j = 1; j <= static_cast<int>(dims.size()); ++j) tot += count_realized(dims, R, j);
  return tot;
}

}  // namespace

extern "C" {

int cpdgpu_als_sweep_sharded(cpdgpu_ctx* ctx, cpdgpu_tensor* slab, int N, const int64_t* global_dims, int64_t R,
                             double* const* factors, double pinv_rtol, double* cost_out, uint64_t* mults) {
  return guarded(ctx, [&] {
    const ShardGeom g = shard_geometry(ctx, slab, N, global_dims, R, "als_sweep_sharded");
    sharded_als_loop(ctx, slab, g, R, factors, 1, 0.0, pinv_rtol, nullptr);
    Plan& pl = *get_plan(ctx, slab, R, g.pivot);
    if (cost_out) CK(cudaMemcpy(cost_out, pl.costs.d(), sizeof(double), cudaMemcpyDeviceToHost));
    if (mults) *mults = als_sweep_count(g.gdims, R);
  });
}

int cpdgpu_als_run_sharded(cpdgpu_ctx* ctx, cpdgpu_tensor* slab, int N, const int64_t* global_dims, int64_t R,
                           double* const* factors, int max_iters, double tol, double pinv_rtol, double* cost_trace,
                           double* rel_trace, double* sec_trace, uint64_t* mults_trace, int* iters_run) {
  return guarded(ctx, [&] {
    const ShardGeom g = shard_geometry(ctx, slab, N, global_dims, R, "run_sharded");
    if (max_iters < 1) fail(CPDGPU_ARGUMENT_ERROR, "run_sharded: max_iters must be at least 1");
    if (!cost_trace || !rel_trace || !iters_run) fail(CPDGPU_ARGUMENT_ERROR, "run_sharded: null argument");
    const int done = sharded_als_loop(ctx, slab, g, R, factors, max_iters, tol, pinv_rtol, sec_trace);
    Plan& pl = *get_plan(ctx, slab, R, g.pivot);
    double ynorm2 = 0.0;
    CK(cudaMemcpy(&ynorm2, pl.norm.d(), sizeof(double), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(cost_trace, pl.costs.d(), static_cast<size_t>(done) * sizeof(double), cudaMemcpyDeviceToHost));
    const double ynorm = std::sqrt(ynorm2);
    const uint64_t per_sweep = als_sweep_count(g.gdims, R);
    for (int i = 0; i < done; ++i) {
      rel_trace[i] = ynorm > 0.0 ? std::sqrt(cost_trace[i]) / ynorm : std::sqrt(cost_trace[i]);
      if (mults_trace) mults_trace[i] = per_sweep * static_cast<uint64_t>(i + 1);
    }
    *iters_run = done;
  });
}

}  // extern "C"
