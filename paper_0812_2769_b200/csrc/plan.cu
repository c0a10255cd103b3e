// plan.cu — plan lifecycle and the non-solver entry points of the C-ABI:
// gsk_spmv / gsk_plan_spmv (SPEC sparse-core spmv; AC-3), gsk_dot (AC-5),
// gsk_plan_residual_norm, SELL copy-out, probes, diagnostics.
#include <csignal>
#include <cstring>
#include <execinfo.h>
#include <unistd.h>
#include <map>
#include <mutex>
#include <set>
#include <unordered_map>
#include <string>
#include <vector>
#include <chrono>
#include "internal.cuh"

namespace gsk {

// Debug aid (GSK_SEGV_TRACE=1): on SIGSEGV print the native backtrace to stderr, then
// hand the signal to the previous handler (Python's faulthandler prints its stacks).
static struct sigaction g_prev_segv;
static void segv_trace(int sig, siginfo_t* info, void* ctx) {
  void* frames[64];
  const int k = backtrace(frames, 64);
  const char msg[] = "gsk: SIGSEGV, native backtrace:\n";
  (void)!write(2, msg, sizeof msg - 1);
  backtrace_symbols_fd(frames, k, 2);
  sigaction(SIGSEGV, &g_prev_segv, nullptr);
  if (g_prev_segv.sa_flags & SA_SIGINFO) {
    if (g_prev_segv.sa_sigaction) g_prev_segv.sa_sigaction(sig, info, ctx);
  } else if (g_prev_segv.sa_handler != SIG_DFL && g_prev_segv.sa_handler != SIG_IGN) {
    g_prev_segv.sa_handler(sig);
  }
  raise(sig);
}
static int install_segv_trace() {
  const char* e = std::getenv("GSK_SEGV_TRACE");
  if (!e || e[0] != '1') return 0;
  struct sigaction sa {};
  sa.sa_sigaction = segv_trace;
  sa.sa_flags = SA_SIGINFO;
  sigemptyset(&sa.sa_mask);
  sigaction(SIGSEGV, &sa, &g_prev_segv);
  return 1;
}
static const int g_segv_installed = install_segv_trace();

static thread_local std::string t_err;
std::atomic<int64_t> g_launches{0};

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  t_err = buf;
}

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

Geometry make_geometry(int n) {
  Geometry g;
  g.n = n;
  return g;
}

bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("GSK_PDL");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

// rcd: a row-class plan (16 windows per CTA: its passes prefetch the CTA's whole row
// block at once; measured at C4 / C3 +1.5% over 8, 4 is -5%; the slot kernels are 1.4%
// slower at 16)
int spmv_wpc_max(bool rcd) {
  static int w = 0;
  if (!w) {
    const char* e = std::getenv("GSK_WPC");
    w = e ? std::atoi(e) : -1;
    if (w != 1 && w != 2 && w != 4 && w != 8 && w != 16) w = -1;
  }
  return w > 0 ? w : (rcd ? 16 : 8);
}

bool pass_alternate() {
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("GSK_ALT");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

// Test-only fault hook: GSK_FAULT=<rho0|omega0|nan>:<iteration> (BicgState).
void read_fault(int* kind, int* it) {
  *kind = GSK_FAULT_NONE;
  *it = 0;
  const char* e = std::getenv("GSK_FAULT");
  if (!e) return;
  const char* c = std::strchr(e, ':');
  if (!c) return;
  const std::string k(e, c - e);
  *kind = k == "rho0" ? GSK_FAULT_RHO0 : k == "omega0" ? GSK_FAULT_OMEGA0 : k == "nan" ? GSK_FAULT_NAN : GSK_FAULT_NONE;
  *it = std::atoi(c + 1);
}

bool short_slots_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("GSK_SHORT");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

int smem_carveout() {
  static int c = -3;
  if (c == -3) {
    const char* e = std::getenv("GSK_CARVEOUT");
    c = e ? std::atoi(e) : 25;
    if (c > 100) c = 100;
    if (c < -1) c = -1;
  }
  return c;
}

// Function attributes are per device: (device, key) pairs already configured.
static std::mutex g_attr_mu;
static std::set<std::pair<int, const void*>> g_attr_done;
static int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}
bool device_attr_done(const void* key) {
  std::lock_guard<std::mutex> lock(g_attr_mu);
  return g_attr_done.count({current_device(), key}) > 0;
}
void device_attr_mark(const void* key) {
  std::lock_guard<std::mutex> lock(g_attr_mu);
  g_attr_done.insert({current_device(), key});
}

// Workspace cache: device blocks released by a plan (after its stream
// drained) stay mapped, keyed by (device, size class), and serve the next plan that asks
// for the same class, so plans built and destroyed in a loop (bench.py's e2e step: SELL
// arrays, 7 Bi-CGSTAB vectors, the 31-vector GMRES basis — ~7 GB at C4) cost no
// cudaMalloc / cudaFree; a cudaFree of a GB-sized block synchronises the device and
// unmaps it (10-270 ms per plan at C4, profiles/r02_e2e_breakdown.txt).  Size classes:
// powers of two below 2 MB, multiples of 2 MB above.  The cache holds at most
// GSK_POOL_MB (default 32768) per device; GSK_POOL_MB=0 disables it; a failed
// cudaMalloc first returns the device's cached blocks and retries.
static std::mutex g_pool_mu;
static std::multimap<std::pair<int, size_t>, void*> g_pool_free;
static std::unordered_map<void*, std::pair<int, size_t>> g_pool_live;
static std::unordered_map<int, size_t> g_pool_bytes;  // cached (free) bytes per device
static size_t pool_cap() {
  static const size_t cap = [] {
    const char* e = std::getenv("GSK_POOL_MB");
    return (size_t)(e ? std::atoll(e) : 32768LL) << 20;
  }();
  return cap;
}
static size_t pool_class(size_t bytes) {
  if (bytes == 0) bytes = 1;
  if (bytes >= (2u << 20)) return (bytes + (2u << 20) - 1) & ~(size_t)((2u << 20) - 1);
  size_t c = 256;
  while (c < bytes) c <<= 1;
  return c;
}
static void pool_trim_locked(int dev) {
  for (auto it = g_pool_free.begin(); it != g_pool_free.end();) {
    if (it->first.first == dev) {
      cudaFree(it->second);
      it = g_pool_free.erase(it);
    } else {
      ++it;
    }
  }
  g_pool_bytes[dev] = 0;
}
cudaError_t pool_alloc(void** p, size_t bytes) {
  const int dev = current_device();
  const size_t cls = pool_class(bytes);
  std::lock_guard<std::mutex> lock(g_pool_mu);
  auto it = g_pool_free.find({dev, cls});
  if (it != g_pool_free.end()) {
    *p = it->second;
    g_pool_free.erase(it);
    g_pool_bytes[dev] -= cls;
    g_pool_live[*p] = {dev, cls};
    return cudaSuccess;
  }
  cudaError_t e = cudaMalloc(p, cls);
  if (e == cudaErrorMemoryAllocation && g_pool_bytes[dev] > 0) {
    cudaGetLastError();
    pool_trim_locked(dev);
    e = cudaMalloc(p, cls);
  }
  if (e == cudaSuccess) g_pool_live[*p] = {dev, cls};
  return e;
}
void pool_release(void* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lock(g_pool_mu);
  auto it = g_pool_live.find(p);
  if (it == g_pool_live.end()) {  // not a pool block
    cudaFree(p);
    return;
  }
  const auto key = it->second;
  g_pool_live.erase(it);
  if (g_pool_bytes[key.first] + key.second > pool_cap()) {
    cudaFree(p);
    return;
  }
  g_pool_free.insert({key, p});
  g_pool_bytes[key.first] += key.second;
}

// A plan's pinned host flags (16 ints) come from a process-wide free list and are never
// returned to the driver: cudaFreeHost was measured at 8-500 ms per plan now and then (it
// synchronises and unmaps; profiles/r02_e2e_breakdown.txt), the dominant cost of a plan's
// life cycle in a build / solve / destroy loop.
static std::mutex g_pin_mu;
static std::vector<int*> g_pin_free;
cudaError_t pinned_flags_alloc(int** p) {
  {
    std::lock_guard<std::mutex> lock(g_pin_mu);
    if (!g_pin_free.empty()) {
      *p = g_pin_free.back();
      g_pin_free.pop_back();
    } else {
      *p = nullptr;
    }
  }
  if (!*p) {
    const cudaError_t e = cudaMallocHost(p, sizeof(int) * 16);
    if (e != cudaSuccess) return e;
  }
  for (int q = 0; q < 16; ++q) (*p)[q] = 0;
  return cudaSuccess;
}
void pinned_flags_release(int* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lock(g_pin_mu);
  g_pin_free.push_back(p);
}

void set_pass_carveout(const void* kern) {
  const int pct = smem_carveout();
  if (pct < 0 || device_attr_done(kern)) return;
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
  cudaGetLastError();  // a refused hint is not an error of the pass
  device_attr_mark(kern);
}

int num_sms() {
  static std::mutex mu;
  static std::unordered_map<int, int> sms;
  const int dev = current_device();
  std::lock_guard<std::mutex> lock(mu);
  auto it = sms.find(dev);
  if (it != sms.end()) return it->second;
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  if (v <= 0) v = 148;
  sms[dev] = v;
  return v;
}

// Reduction scratch: CTA partials of one pass ([MAXD][pstride], pstride >= CTAs).
int alloc_reduction(gsk_plan* P, cudaStream_t s, bool async) {
  P->pstride = ((P->geo.n + TB - 1) / TB + 7) & ~7;  // multiple of 8: 16-byte aligned rows
  const size_t bytes = sizeof(double) * MAXD * (size_t)P->pstride;
  // (no stream-ordered allocation anywhere in the library: the default memory pool
  // returns its memory to the OS at the next synchronisation and maps it again at the next
  // cudaMallocAsync — measured as random 50-700 ms stalls in a plan build / destroy loop,
  // profiles/r02_e2e_breakdown.txt; everything comes from the workspace cache instead)
  (void)s;
  (void)async;
  GSK_CUDA(pool_alloc((void**)&P->part, bytes));
  return GSK_OK;
}

// ---- ops --------------------------------------------------------------------------
struct OpSpmv {
  static constexpr int D = 0;
  static constexpr int NV = 0;
  static constexpr bool kSpmv = true;
  const double* x;
  double* y;
  __device__ bool begin() { return true; }
  __device__ const double* vin(int) const { return nullptr; }
  __device__ const double* gathered() const { return x; }  // the one vector gather() reads
  __device__ double gather(int c) const { return __ldg(x + c); }
  __device__ void row(int i, double v, const double (&)[1], double (&)[1]) const { y[i] = v; }
};

struct OpDot {
  static constexpr int D = 1;
  static constexpr int NV = 2;
  static constexpr bool kSpmv = false;
  const double* a;
  const double* b;
  double* out;
  __device__ bool begin() { return true; }
  __device__ const double* vin(int k) const { return k == 0 ? a : b; }
  __device__ double gather(int) const { return 0.0; }
  __device__ void row(int, double, const double (&v)[NV], double (&c)[1]) const { c[0] = v[0] * v[1]; }
  __device__ void finish(const double (&s)[1], int lane) const {
    if (lane == 0) *out = s[0];
  }
};

// ||w o (b - A x)||^2
struct OpResNorm {
  static constexpr int D = 1;
  static constexpr int NV = 2;
  static constexpr bool kSpmv = true;
  const double* x;
  const double* b;
  const double* w;
  double* out;
  __device__ bool begin() { return true; }
  __device__ const double* vin(int k) const { return k == 0 ? b : w; }
  __device__ double gather(int c) const { return __ldg(x + c); }
  __device__ void row(int, double y, const double (&v)[NV], double (&c)[1]) const {
    const double r = v[0] - y;
    const double u = w ? v[1] * r : r;
    c[0] = u * u;
  }
  __device__ void finish(const double (&s)[1], int lane) const {
    if (lane == 0) *out = s[0];
  }
};

static int plan_alloc_common(gsk_plan* P) {
  P->geo = make_geometry(P->A.n);
  GSK_TRY(alloc_reduction(P, nullptr, false));
  GSK_CUDA(pool_alloc((void**)&P->scratch, sizeof(double) * 8));
  GSK_CUDA(cudaStreamCreateWithFlags(&P->st, cudaStreamNonBlocking));
  GSK_CUDA(pinned_flags_alloc(&P->h_flag));
  GSK_CUDA(cudaEventCreate(&P->t0));
  GSK_CUDA(cudaEventCreate(&P->t1));
  for (auto& k : P->pev)
    for (auto& e : k) {
      GSK_CUDA(cudaEventCreate(&e[0]));
      GSK_CUDA(cudaEventCreate(&e[1]));
    }
  for (auto& e : P->qev) GSK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  P->csr = CsrView{P->A.n, P->A.row_ptr, P->A.col_idx, P->A.values};
  return GSK_OK;
}

static int check_csr(const gsk_csr* A, const char* who) {
  if (!A || A->n < 1 || A->nnz < 0 || !A->row_ptr || (A->nnz > 0 && (!A->col_idx || !A->values))) {
    set_error("%s: invalid gsk_csr (n >= 1, nnz >= 0, non-null arrays required)", who);
    return GSK_E_INVALID;
  }
  return GSK_OK;
}

// Order work on the plan stream after the caller's stream (and vice versa at the end).
int join_in(gsk_plan* P, cudaStream_t caller) {
  cudaEvent_t e;
  GSK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  GSK_CUDA(cudaEventRecord(e, caller));
  GSK_CUDA(cudaStreamWaitEvent(P->st, e, 0));
  GSK_CUDA(cudaEventDestroy(e));
  return GSK_OK;
}
int join_out(gsk_plan* P, cudaStream_t caller) {
  cudaEvent_t e;
  GSK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  GSK_CUDA(cudaEventRecord(e, P->st));
  GSK_CUDA(cudaStreamWaitEvent(caller, e, 0));
  GSK_CUDA(cudaEventDestroy(e));
  return GSK_OK;
}

int end_capture(cudaStream_t s, int rc, cudaGraphExec_t* out, long long* kernels, const char* what) {
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(s, &g);
  if (rc < 0) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  if (e != cudaSuccess) {
    set_error("%s graph capture: %s", what, cudaGetErrorString(e));
    return GSK_E_CUDA;
  }
  size_t nn = 0;
  cudaGraphGetNodes(g, nullptr, &nn);
  std::vector<cudaGraphNode_t> nodes(nn);
  cudaGraphGetNodes(g, nodes.data(), &nn);
  long long k = 0;
  for (auto nd : nodes) {
    cudaGraphNodeType ty;
    if (cudaGraphNodeGetType(nd, &ty) == cudaSuccess && ty == cudaGraphNodeTypeKernel) ++k;
  }
  e = cudaGraphInstantiate(out, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) {
    set_error("%s graph instantiate: %s", what, cudaGetErrorString(e));
    return GSK_E_CUDA;
  }
  g_launches.fetch_sub(k);  // counted per replay instead
  *kernels = k;
  return GSK_OK;
}

int run_batches(gsk_plan* P, cudaGraphExec_t* graphs, long long maxb, long long kernels, const int* done_dev,
                const int* kinds, int nkinds) {
  NvtxRange nv("gsk:graph_batches");
  constexpr int NQ = gsk_plan::NQ;
  cudaStream_t s = P->st;
  // batches in flight: 3 for large systems (a late host check never idles the GPU);
  // 1 for small ones, where a queued batch that returns at once costs as much as a
  // real one
  const int depth = P->A.n >= (1 << 20) ? NQ : 1;
  long long launched = 0, checked = 0;
  auto launch = [&]() -> int {
    const int c = (int)(launched % NQ);
    GSK_CUDA(cudaGraphLaunch(graphs[c], s));
    g_launches.fetch_add(kernels);
    GSK_CUDA(cudaMemcpyAsync(P->h_flag + c, done_dev, sizeof(int), cudaMemcpyDeviceToHost, s));
    GSK_CUDA(cudaEventRecord(P->qev[c], s));
    ++launched;
    return GSK_OK;
  };
  while (launched < depth && launched < maxb) GSK_TRY(launch());
  for (;;) {
    const int c = (int)(checked % NQ);
    GSK_CUDA(cudaEventSynchronize(P->qev[c]));
    for (int q = 0; q < nkinds; ++q) {
      const int kind = kinds[q];
      float ms = 0;
      if (cudaEventElapsedTime(&ms, P->pev[kind][c][0], P->pev[kind][c][1]) == cudaSuccess) {
        P->probe_ms[kind] += ms;
        P->probe_n[kind] += 1;
      } else {
        (void)cudaGetLastError();  // probe not recorded in this graph (e.g. GMRES m = 1)
      }
    }
    const int done = P->h_flag[c];
    ++checked;
    if (done) break;
    if (launched < maxb)
      GSK_TRY(launch());
    else if (checked == launched)
      break;
  }
  // drain the batches still queued (they return at once: the done flag is set)
  GSK_CUDA(cudaStreamSynchronize(s));
  return GSK_OK;
}

int ensure_hist(gsk_plan* P, int maxit) {
  if (P->hist_cap >= maxit + 1) return GSK_OK;
  if (P->hist_d) {
    GSK_CUDA(cudaStreamSynchronize(P->st));  // no queued pass still writes it
    pool_release(P->hist_d);
  }
  P->hist_d = nullptr;
  GSK_CUDA(pool_alloc((void**)&P->hist_d, sizeof(double) * (size_t)(maxit + 1)));
  P->hist_cap = maxit + 1;
  return GSK_OK;
}

}  // namespace gsk

using namespace gsk;

extern "C" {

const char* gsk_last_error(void) { return t_err.c_str(); }
int64_t gsk_launch_count(void) { return g_launches.load(); }
int gsk_version(void) { return 1; }

int gsk_plan_create(const gsk_csr* A, const gsk_opts* opts, gsk_plan** plan, void* stream) {
  return plan_create_impl(A, opts, -1, plan, as_stream(stream));
}

}  // extern "C"

namespace gsk {
int plan_create_impl(const gsk_csr* A, const gsk_opts* opts, int sell_pad, gsk_plan** plan, cudaStream_t stream) {
  NvtxRange nv("gsk:plan_create");
  GSK_TRY(check_csr(A, "gsk_plan_create"));
  if (!plan) {
    set_error("gsk_plan_create: plan is NULL");
    return GSK_E_INVALID;
  }
  int fmt = opts ? opts->format : GSK_FMT_CSR;
  if (fmt != GSK_FMT_CSR && fmt != GSK_FMT_SELL) {
    set_error("gsk_plan_create: unknown format %d", fmt);
    return GSK_E_INVALID;
  }
  gsk_plan* P = new gsk_plan();
  P->A = *A;
  P->fmt = fmt;
  P->sell_pad = sell_pad;
  P->poll = opts ? opts->poll : 0;
  P->weights = opts ? opts->weights : nullptr;
  const int sched = opts ? opts->bicg_schedule : GSK_BICG_AUTO;
  if (sched < 0 || sched > 3) {
    delete P;
    set_error("gsk_plan_create: unknown bicg_schedule %d", sched);
    return GSK_E_INVALID;
  }
  // auto: the four-pass schedule (one kernel fewer, a second gather stream) where the
  // iteration is L2-resident and launch-bound (C2: 37.4k vs 35.2k it/s), else split
  // (C3 / C4 / C5: the extra gathers cost 7-23%; profiles/r02_experiments)
  const double ws = 12.0 * (double)A->nnz + 4.0 * (double)A->n + 64.0 * (double)A->n;
  P->bmode = sched == GSK_BICG_AUTO ? (ws <= 64e6 ? GSK_BICG_SPLIT4 : GSK_BICG_SPLIT) : sched;
  const int orth = opts ? opts->gmres_orth : GSK_ORTH_MGS;
  if (orth != GSK_ORTH_MGS && orth != GSK_ORTH_CGS2) {
    delete P;
    set_error("gsk_plan_create: unknown gmres_orth %d", orth);
    return GSK_E_INVALID;
  }
  P->orth = orth;
  P->sell_index = opts ? opts->sell_index : 0;
  P->wstop = (opts && opts->gmres_wstop) ? 1 : 0;
  P->engine = opts ? opts->engine : GSK_ENGINE_AUTO;
  if (P->engine < GSK_ENGINE_AUTO || P->engine > GSK_ENGINE_CLUSTER) {
    delete P;
    set_error("gsk_plan_create: unknown engine %d", opts->engine);
    return GSK_E_INVALID;
  }
  if (P->sell_index < 0 || P->sell_index > 3) {
    delete P;
    set_error("gsk_plan_create: unknown sell_index %d", opts->sell_index);
    return GSK_E_INVALID;
  }
  // GSK_TRACE_PLAN=1: host time of the phases of a plan build on stderr
  static const bool trace = std::getenv("GSK_TRACE_PLAN") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  const auto t0 = now();
  int rc = plan_alloc_common(P);
  const auto t1 = now();
  auto t2 = t1, t3 = t1;
  if (rc == GSK_OK && fmt == GSK_FMT_SELL) {
    cudaStream_t s = stream;
    rc = join_in(P, s);
    if (rc == GSK_OK) rc = sell_build(P, P->st);
    t2 = now();
    if (rc == GSK_OK && P->sell_index == 1) rc = sell_dict_build(P, P->st);
    if (rc == GSK_OK && P->sell_index == 2) rc = sellu_build(P, P->st);
    if (rc == GSK_OK && P->sell_index == 3) rc = rcd_build(P, P->st);
    if (rc == GSK_OK) rc = join_out(P, s);
    if (rc == GSK_OK && cudaStreamSynchronize(P->st) != cudaSuccess) rc = GSK_E_CUDA;
    t3 = now();
  }
  if (trace)
    std::fprintf(stderr, "[gsk] plan n=%d: alloc %.2f ms, SELL build %.2f ms, encodings %.2f ms\n", A->n, ms(t0, t1),
                 ms(t1, t2), ms(t2, t3));
  if (rc != GSK_OK) {
    gsk_plan_destroy(P);
    return rc;
  }
  *plan = P;
  return GSK_OK;
}
}  // namespace gsk

extern "C" {

int gsk_plan_refresh(gsk_plan* P, void* stream) {
  NvtxRange nv("gsk:plan_refresh");
  if (!P) return GSK_E_INVALID;
  if (P->shards) return shard_refresh(P, as_stream(stream));
  if (P->fmt != GSK_FMT_SELL) return GSK_OK;
  cudaStream_t s = as_stream(stream);
  GSK_TRY(join_in(P, s));
  GSK_TRY(sell_fill_values(P, P->st));
  GSK_TRY(join_out(P, s));
  GSK_CUDA(cudaStreamSynchronize(P->st));
  return GSK_OK;
}

void gsk_plan_destroy(gsk_plan* P) {
  if (!P) return;
  static const bool trace = std::getenv("GSK_TRACE_PLAN") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  const auto t0 = now();
  if (P->st) cudaStreamSynchronize(P->st);
  if (P->shards) shard_destroy(P->shards);
  const auto t1 = now();
  for (auto g : P->bgraph)
    if (g) cudaGraphExecDestroy(g);
  for (auto g : P->ggraph)
    if (g) cudaGraphExecDestroy(g);
  const auto t2 = now();
  void* bufs[] = {P->cptr, P->clen, P->scol, P->sval, P->roff, P->wid, P->part, P->scratch,
                  P->bvec, P->bstate, P->W, P->gstate, P->garr, P->hist_d, P->mpart, P->sidx, P->dptr, P->dict,
                  P->cpart, P->uptr, P->udel, P->umask, P->uval, P->kcls, P->kdict, P->ktab, P->kslots, P->drcd};
  for (void* b : bufs) pool_release(b);  // the plan stream drained above
  const auto t3 = now();
  pinned_flags_release(P->h_flag);
  const auto t4 = now();
  for (auto& k : P->pev)
    for (auto& e : k) {
      if (e[0]) cudaEventDestroy(e[0]);
      if (e[1]) cudaEventDestroy(e[1]);
    }
  for (auto e : P->qev)
    if (e) cudaEventDestroy(e);
  if (P->t0) cudaEventDestroy(P->t0);
  if (P->t1) cudaEventDestroy(P->t1);
  if (P->st) cudaStreamDestroy(P->st);
  const auto t5 = now();
  if (trace)
    std::fprintf(stderr, "[gsk] destroy: sync %.2f ms, graphs %.2f ms, buffers %.2f ms, pinned %.2f ms, events+stream %.2f ms\n",
                 ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4), ms(t4, t5));
  delete P;
}

int gsk_plan_spmv(gsk_plan* P, const double* x, double* y, void* stream) {
  if (P && P->shards && x && y) return shard_spmv(P, x, y, as_stream(stream));
  if (!P || !x || !y) {
    set_error("gsk_plan_spmv: NULL argument");
    return GSK_E_INVALID;
  }
  cudaStream_t s = as_stream(stream);
  OpSpmv op{x, y};
  if (run_pass(P, op, s) < 0) return GSK_E_CUDA;
  GSK_CUDA(cudaStreamSynchronize(s));
  return GSK_OK;
}

int gsk_spmv(const gsk_csr* A, const double* x, double* y, void* stream) {
  gsk_plan* P = nullptr;
  GSK_TRY(gsk_plan_create(A, nullptr, &P, stream));
  int rc = gsk_plan_spmv(P, x, y, stream);
  gsk_plan_destroy(P);
  return rc;
}

int gsk_plan_residual_norm(gsk_plan* P, const double* b, const double* x, const double* w,
                           double* result, void* stream) {
  if (P && P->shards) {
    set_error("gsk_plan_residual_norm: not available on a sharded plan (use the per-shard solvers)");
    return GSK_E_INVALID;
  }
  if (!P || !b || !x || !result) {
    set_error("gsk_plan_residual_norm: NULL argument");
    return GSK_E_INVALID;
  }
  cudaStream_t s = as_stream(stream);
  OpResNorm op{x, b, w, P->scratch};
  if (run_pass(P, op, s) < 0) return GSK_E_CUDA;
  double v = 0;
  GSK_CUDA(cudaMemcpyAsync(&v, P->scratch, sizeof(double), cudaMemcpyDeviceToHost, s));
  GSK_CUDA(cudaStreamSynchronize(s));
  *result = sqrt(v);
  return GSK_OK;
}

int gsk_dot(int64_t n, const double* a, const double* b, double* result, void* stream) {
  if (n < 1 || n > 0x7fffffff || !a || !b || !result) {
    set_error("gsk_dot: invalid arguments");
    return GSK_E_INVALID;
  }
  gsk_plan tmp;
  tmp.A.n = (int)n;
  tmp.geo = make_geometry((int)n);
  cudaStream_t s = as_stream(stream);
  GSK_TRY(alloc_reduction(&tmp, s, true));
  double* out = nullptr;
  GSK_CUDA(pool_alloc((void**)&out, sizeof(double)));
  OpDot op{a, b, out};
  int rc = run_pass(&tmp, op, s) < 0 ? GSK_E_CUDA : GSK_OK;
  double v = 0;
  if (rc == GSK_OK && cudaMemcpyAsync(&v, out, sizeof(double), cudaMemcpyDeviceToHost, s) != cudaSuccess)
    rc = GSK_E_CUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) rc = GSK_E_CUDA;
  pool_release(tmp.part);  // the stream drained above
  pool_release(out);
  *result = v;
  return rc;
}

int gsk_plan_sell_info(gsk_plan* P, int64_t* nchunks, int64_t* nslots) {
  if (P && P->shards) {
    set_error("gsk_plan_sell_info: not available on a sharded plan (use the per-shard solvers)");
    return GSK_E_INVALID;
  }
  if (!P || P->fmt != GSK_FMT_SELL) {
    set_error("gsk_plan_sell_info: plan is not SELL");
    return GSK_E_INVALID;
  }
  if (nchunks) *nchunks = P->nchunks;
  if (nslots) *nslots = P->nslots;
  return GSK_OK;
}

int gsk_plan_sell_copy(gsk_plan* P, int32_t* chunk_ptr, int32_t* chunk_len, int32_t* scol,
                       double* sval, uint8_t* roff, void* stream) {
  if (P && P->shards) {
    set_error("gsk_plan_sell_copy: not available on a sharded plan (use the per-shard solvers)");
    return GSK_E_INVALID;
  }
  if (!P || P->fmt != GSK_FMT_SELL) {
    set_error("gsk_plan_sell_copy: plan is not SELL");
    return GSK_E_INVALID;
  }
  cudaStream_t s = as_stream(stream);
  GSK_CUDA(cudaStreamSynchronize(P->st));
  if (chunk_ptr) GSK_CUDA(cudaMemcpyAsync(chunk_ptr, P->cptr, sizeof(int) * (P->nchunks + 1), cudaMemcpyDeviceToDevice, s));
  if (chunk_len) GSK_CUDA(cudaMemcpyAsync(chunk_len, P->clen, sizeof(int) * P->nchunks, cudaMemcpyDeviceToDevice, s));
  if (scol) GSK_CUDA(cudaMemcpyAsync(scol, P->scol, sizeof(int) * P->nslots, cudaMemcpyDeviceToDevice, s));
  if (sval) GSK_CUDA(cudaMemcpyAsync(sval, P->sval, sizeof(double) * P->nslots, cudaMemcpyDeviceToDevice, s));
  if (roff) GSK_CUDA(cudaMemcpyAsync(roff, P->roff, P->nchunks * SELL_C, cudaMemcpyDeviceToDevice, s));
  GSK_CUDA(cudaStreamSynchronize(s));
  return GSK_OK;
}

int gsk_plan_sell_dict(gsk_plan* P, int64_t* ndict, int32_t* dict_ptr, int32_t* dict, uint8_t* sidx,
                       void* stream) {
  if (P && P->shards) {
    set_error("gsk_plan_sell_dict: not available on a sharded plan (use the per-shard solvers)");
    return GSK_E_INVALID;
  }
  if (!P || P->fmt != GSK_FMT_SELL) {
    set_error("gsk_plan_sell_dict: plan is not SELL");
    return GSK_E_INVALID;
  }
  if (!P->dict) {
    if (ndict) *ndict = -1;
    return GSK_OK;
  }
  if (ndict) *ndict = P->ndict;
  cudaStream_t s = as_stream(stream);
  if (dict_ptr) GSK_CUDA(cudaMemcpyAsync(dict_ptr, P->dptr, sizeof(int) * (P->nchunks + 1), cudaMemcpyDeviceToDevice, s));
  if (dict) GSK_CUDA(cudaMemcpyAsync(dict, P->dict, sizeof(int) * P->ndict, cudaMemcpyDeviceToDevice, s));
  if (sidx) GSK_CUDA(cudaMemcpyAsync(sidx, P->sidx, P->nslots, cudaMemcpyDeviceToDevice, s));
  GSK_CUDA(cudaStreamSynchronize(s));
  return GSK_OK;
}

int gsk_plan_sell_uniform(gsk_plan* P, int64_t* nuslots, int32_t* uptr, int32_t* udel, uint32_t* umask,
                          double* uval, void* stream) {
  if (!P || P->shards || P->fmt != GSK_FMT_SELL) {
    set_error("gsk_plan_sell_uniform: plan is not an unsharded SELL plan");
    return GSK_E_INVALID;
  }
  if (!P->uptr) {
    if (nuslots) *nuslots = -1;
    return GSK_OK;
  }
  if (nuslots) *nuslots = P->nuslots;
  cudaStream_t s = as_stream(stream);
  const size_t nch = (size_t)P->nchunks;
  if (uptr) GSK_CUDA(cudaMemcpyAsync(uptr, P->uptr, sizeof(int) * (nch + 1), cudaMemcpyDeviceToDevice, s));
  if (udel) GSK_CUDA(cudaMemcpyAsync(udel, P->udel, sizeof(int) * nch * SELLU_MAXL, cudaMemcpyDeviceToDevice, s));
  if (umask) GSK_CUDA(cudaMemcpyAsync(umask, P->umask, sizeof(unsigned) * nch * SELLU_MAXL, cudaMemcpyDeviceToDevice, s));
  if (uval) GSK_CUDA(cudaMemcpyAsync(uval, P->uval, sizeof(double) * P->nuslots, cudaMemcpyDeviceToDevice, s));
  GSK_CUDA(cudaStreamSynchronize(s));
  return GSK_OK;
}

int gsk_plan_row_classes(gsk_plan* P, int64_t* ncls, uint16_t* cls, void* entries, void* stream) {
  if (P && P->shards && P->fmt == GSK_FMT_SELL && !cls && !entries) {  // count only
    if (ncls) *ncls = shard_row_classes(P);
    return GSK_OK;
  }
  if (!P || P->shards || P->fmt != GSK_FMT_SELL) {
    set_error("gsk_plan_row_classes: plan is not an unsharded SELL plan");
    return GSK_E_INVALID;
  }
  if (!P->sell.rcd) {
    if (ncls) *ncls = -1;
    return GSK_OK;
  }
  if (ncls) *ncls = P->ncls;
  cudaStream_t s = as_stream(stream);
  if (cls) GSK_CUDA(cudaMemcpyAsync(cls, P->kcls, sizeof(uint16_t) * (size_t)P->A.n, cudaMemcpyDeviceToDevice, s));
  if (entries)
    GSK_CUDA(cudaMemcpyAsync(entries, P->kdict, sizeof(RcdEntry) * (size_t)P->ncls, cudaMemcpyDeviceToDevice, s));
  GSK_CUDA(cudaStreamSynchronize(s));
  return GSK_OK;
}

int gsk_plan_class_slots(gsk_plan* P, int32_t* ns, int32_t* deltas, void* slots, void* stream) {
  if (!P || P->shards || P->fmt != GSK_FMT_SELL || !ns) {
    set_error("gsk_plan_class_slots: plan is not an unsharded SELL plan (or ns is NULL)");
    return GSK_E_INVALID;
  }
  const bool on = P->sell.rcd && P->hrcd.kslots;
  *ns = on ? P->hrcd.ns : -1;
  if (!on) return GSK_OK;
  if (deltas)
    for (int k = 0; k < RCD_MAXL; ++k) deltas[k] = P->hrcd.sdel[k];
  if (slots) {
    cudaStream_t s = as_stream(stream);
    GSK_CUDA(cudaMemcpyAsync(slots, P->kslots, sizeof(RcdSlots) * (size_t)P->ncls, cudaMemcpyDeviceToDevice, s));
    GSK_CUDA(cudaStreamSynchronize(s));
  }
  return GSK_OK;
}

int gsk_plan_probe(gsk_plan* P, int kind, double* avg_ms, int64_t* count) {
  if (!P || kind < 0 || kind >= gsk_plan::NPROBE) {
    set_error("gsk_plan_probe: bad arguments");
    return GSK_E_INVALID;
  }
  if (avg_ms) *avg_ms = P->probe_n[kind] ? P->probe_ms[kind] / P->probe_n[kind] : 0.0;
  if (count) *count = P->probe_n[kind];
  return GSK_OK;
}

}  // extern "C"
