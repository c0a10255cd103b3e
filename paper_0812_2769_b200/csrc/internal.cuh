// internal.cuh — host-side plumbing of libgsk: errors, launch accounting, geometry,
// the plan object and the device-resident solver states.
#pragma once
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <nvtx3/nvToolsExt.h>
#include "common.cuh"
#include "engine.cuh"
#include "gsk.h"

namespace gsk {

// NVTX range over one library call (header-only NVTX3: no cost unless a profiler
// injects itself), so nsys / ncu timelines show the solver phases by name.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};


void set_error(const char* fmt, ...);
extern std::atomic<int64_t> g_launches;

#define GSK_CUDA(call)                                                                      \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      ::gsk::set_error("%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
                       __LINE__);                                                           \
      return GSK_E_CUDA;                                                                    \
    }                                                                                       \
  } while (0)

#define GSK_LAUNCHED(k)                         \
  do {                                          \
    ::gsk::g_launches.fetch_add(k);             \
    cudaError_t e_ = cudaGetLastError();        \
    if (e_ != cudaSuccess) {                    \
      ::gsk::set_error("kernel launch: %s (%s:%d)", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return GSK_E_CUDA;                        \
    }                                           \
  } while (0)

#define GSK_TRY(x)              \
  do {                          \
    int rc_ = (x);              \
    if (rc_ != GSK_OK) return rc_; \
  } while (0)

struct Geometry {
  int n = 0;
};
Geometry make_geometry(int n);

// Device-resident Bi-CGSTAB state (scalars + control flags), DESIGN.md §5.
// fault_kind / fault_it: the test-only fault hook (GSK_FAULT=<kind>:<iteration>, read at
// solve start on unsharded plans; the oracle's orc_set_fault mirrors it): 1 forces
// rho = 0 at the end of that iteration, 2 forces omega = 0 in it, 3 writes NaN into r_0
// in its update (exercises the verdict paths identically on both sides).
struct BicgState {
  double rho, rho_prev, alpha, omega, beta, n0, n0u, tol;
  double true_rel, true_rel_w;
  int iter, maxit, done, status, halfstep, bd, hist_len, pad;
  int fault_kind, fault_it;
};
enum { GSK_FAULT_NONE = 0, GSK_FAULT_RHO0 = 1, GSK_FAULT_OMEGA0 = 2, GSK_FAULT_NAN = 3 };

// Device-resident GMRES(m) state; arrays H[(m+1)*m] (row-major), cs[m], sn[m],
// g[m+1], y[m], inv[m+2] (inv[j] = 1/||w_j||, basis slot j is stored unnormalised).
struct GmresState {
  double beta0, n0w, tol, true_rel, true_rel_w;
  double *H, *cs, *sn, *g, *y, *inv;
  double *c1, *c2;  // CGS2: the two classical projections of the current step
  int it, maxit, m, k, cycle_stop, final_, conv, diverged, skip_x, done, status, restarts,
      hist_len;
  int wstop;  // gsk_opts.gmres_wstop: stop on the weighted true residual at cycle ends
};

cudaStream_t as_stream(void* s);
struct ShardSet;  // row-block shards of a plan (shard.cu)
void shard_destroy(ShardSet* S);

}  // namespace gsk

struct gsk_plan {
  gsk_csr A{};
  int fmt = GSK_FMT_CSR;
  int poll = 0;
  int bmode = 2;  // Bi-CGSTAB schedule: 1 fused, 2 split
  int orth = 0;   // GMRES orthogonalisation: 0 MGS, 1 double classical Gram-Schmidt
  int wstop = 0;  // GMRES stops on the weighted true residual at cycle ends (gsk_opts.gmres_wstop)
  const double* weights = nullptr;
  gsk::Geometry geo;
  gsk::CsrView csr{};
  gsk::SellView sell{};
  // SELL storage (owned)
  int* cptr = nullptr;
  int* clen = nullptr;
  int* scol = nullptr;
  double* sval = nullptr;
  uint8_t* roff = nullptr;
  uint8_t* wid = nullptr;   // [nwindows] natural-order windows (sell.cu)
  int64_t nchunks = 0, nslots = 0;
  uint8_t* sidx = nullptr;  // column-index dictionary (SELL-D); null = plain int32 columns
  int* dptr = nullptr;
  int* dict = nullptr;
  int64_t ndict = 0;
  int* uptr = nullptr;      // SELL-U (sell_index 2): slot offsets, deltas, masks, values
  int* udel = nullptr;
  unsigned* umask = nullptr;
  double* uval = nullptr;
  int64_t nuslots = 0;
  uint16_t* kcls = nullptr;        // row-class dictionary (sell_index 3): class per row,
  gsk::RcdEntry* kdict = nullptr;  // class entries [RCD_MAXCLS]
  void* ktab = nullptr;            // build scratch: hash table + flags (sell.cu)
  gsk::RcdSlots* kslots = nullptr; // stencil slots of the classes [RCD_MAXCLS] (when they share one stencil)
  gsk::RcdView hrcd{};             // host copy of the row-class view in use (kcls null: not in use)
  gsk::RcdView* drcd = nullptr;    // its device copy (SellView::rcd)
  int64_t ncls = 0;                // classes in use (0: inapplicable, plain SELL passes)
  int sell_maxlen = 0;      // longest SELL chunk (slots per lane)
  int sell_index = 0;       // 0 plain int32 columns, 1 dictionary (SELL-D), 2 uniform (SELL-U),
                            // 3 row-class dictionary (RCD)
  int sell_pad = -1;        // padding column value (INT_MIN in shard plans)
  // reduction scratch
  double* part = nullptr;      // [MAXD][pstride] CTA partials of the current pass
  int pstride = 0;             // >= number of CTAs of any pass (ceil(n/256))
  double* scratch = nullptr;   // [n] (residual norms)
  cudaStream_t st = nullptr;
  int* h_flag = nullptr;       // pinned
  // Bi-CGSTAB workspace
  double* bvec = nullptr;      // 7 vectors: r, rhat, pa, pb, va, vb, t
  gsk::BicgState* bstate = nullptr;
  static constexpr int NQ = 3;  // graph copies = batches in flight (host checks lag)
  cudaGraphExec_t bgraph[NQ] = {};
  const double* bkey_b = nullptr;
  const double* bkey_x = nullptr;
  int bK = 0;
  long long bkernels = 0;  // kernel nodes per Bi-CGSTAB graph replay
  long long gkernels = 0;  // kernel nodes per GMRES cycle replay
  const double* bkey_h = nullptr;
  // GMRES workspace
  double* W = nullptr;         // (m+1) n
  int Wm = 0;
  gsk::GmresState* gstate = nullptr;
  double* garr = nullptr;      // H, cs, sn, g, y, inv
  cudaGraphExec_t ggraph[NQ] = {};
  const double* gkey_b = nullptr;
  const double* gkey_x = nullptr;
  int gkey_m = 0;
  const double* gkey_h = nullptr;
  int gkey_orth = -1;
  double* mpart = nullptr;     // [MDOT_MAX][pstride] partials of multi-dot passes
  double* cpart = nullptr;     // cooperative kernel partials [2][MAXD][256] + barrier words
  int engine = GSK_ENGINE_AUTO; // on-chip single-CTA solver / graph passes / cooperative
  // history (device)
  double* hist_d = nullptr;
  int hist_cap = 0;
  // kernel probes: per kind, events recorded around one launch per batch
  // kinds: 0 Bi-CGSTAB v = A p pass, 1 Bi-CGSTAB t = A s pass, 2 GMRES MGS pass,
  // 3 GMRES Arnoldi SpMV pass, 4 Bi-CGSTAB x / r update pass (S4 / P3);
  // [graph copy][start/stop]
  static constexpr int NPROBE = 5;
  cudaEvent_t pev[NPROBE][NQ][2] = {};
  cudaEvent_t qev[NQ] = {};
  double probe_ms[NPROBE] = {};
  int64_t probe_n[NPROBE] = {};
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  unsigned pass_seq = 0;  // passes launched (captured): parity = CTA order of the next
  gsk::ShardSet* shards = nullptr;  // non-null: a row-block sharded plan (shard.cu)
};

namespace gsk {
// Launch one fused pass over the plan's rows: Op::kSpmv selects an SpMV pass in the
// plan's format (CSR or SELL) or a pure vector pass.
int num_sms();
bool pdl_enabled();  // GSK_PDL=0 in the environment disables programmatic launches
int spmv_wpc_max(bool rcd = false);
bool pass_alternate();  // alternate the CTA order of consecutive passes (GSK_ALT=0: off)  // windows per CTA of SpMV passes (8; GSK_WPC overrides, pow2 <= 16)

// Kernel launch with the programmatic-stream-serialization attribute (PDL).
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Shared-memory carveout of the SELL pass kernels: 25% of the SM's 228 KB (57 KB), the rest
// of the unified L1/shared memory caches the x gather.  Measured at C4 (sweep 18-100%,
// the driver's choice, and the smallest carveout that keeps full occupancy): S1 0.330 ->
// 0.325 ms, S3 0.306 -> 0.302 ms although S1 then runs 3 instead of 4 CTAs per SM.
// GSK_CARVEOUT=<percent> overrides it, GSK_CARVEOUT=-1 leaves the driver's choice.
int smem_carveout();
void set_pass_carveout(const void* kern);
bool short_slots_enabled();  // GSK_SHORT=0 disables the <= 5-slot kernels
void read_fault(int* kind, int* it);  // GSK_FAULT test hook (BicgState)
// plan workspace cache (plan.cu): pool_alloc / pool_release instead of cudaMalloc /
// cudaFree for plan-owned buffers; release only what no queued work still uses
cudaError_t pinned_flags_alloc(int** p);  // a plan's pinned host flags (never freed: plan.cu)
void pinned_flags_release(int* p);
cudaError_t pool_alloc(void** p, size_t bytes);
void pool_release(void* p);
// per-device "function attributes already set" registry (keyed by any pointer)
bool device_attr_done(const void* key);
void device_attr_mark(const void* key);
template <typename... KArgs>
void pass_carveout(void (*kern)(KArgs...)) {
  set_pass_carveout(reinterpret_cast<const void*>(kern));
}

// Launch one pass kernel: an SpMV pass in the plan's format (CSR or SELL) or a vector
// pass; *ntiles_out receives its CTA count (= CTA partials per dot).  pe0/pe1: optional
// probe events recorded around the kernel (graph capture: external event nodes).
template <class Op>
int launch_pass(gsk_plan* P, const Op& op, cudaStream_t s, int* ntiles_out, cudaEvent_t pe0 = nullptr,
                cudaEvent_t pe1 = nullptr) {
  const int n = P->geo.n;
  const int sms = num_sms();
  int ntiles;
  const int rev = pass_alternate() ? (P->pass_seq++ & 1) : 0;
  if (pe0) GSK_CUDA(cudaEventRecordWithFlags(pe0, s, cudaEventRecordExternal));
  if constexpr (!Op::kSpmv) {
    // RPT rows per thread when that still leaves >= 2 CTAs per SM, else 2
    constexpr int R = VecRpt<Op::NV>::value;
    if ((long long)n >= 2LL * TB * R * sms) {
      ntiles = (n + TB * R - 1) / (TB * R);
      GSK_CUDA(launch_k(pass_kernel<0, R, Op>, ntiles, TB, 0, s, P->csr, P->sell, n, R, op, P->part, P->pstride, rev));
    } else {
      ntiles = (n + TB * 2 - 1) / (TB * 2);
      GSK_CUDA(launch_k(pass_kernel<0, 2, Op>, ntiles, TB, 0, s, P->csr, P->sell, n, 2, op, P->part, P->pstride, rev));
    }
  } else {
    const int windows = (n + TB - 1) / TB;
    // windows per CTA: as many as keep >= 3 CTAs per SM busy
    int wpc = spmv_wpc_max(P->fmt == GSK_FMT_SELL && P->sell.rcd != nullptr);
    while (wpc > 1 && (long long)windows < (long long)wpc * 3 * sms) wpc >>= 1;
    ntiles = (windows + wpc - 1) / wpc;
    // natural-order SELL plans (every window unsorted, sell.cu) run the NAT kernels
    const bool nat = P->sell.all_nat != 0;
    if (P->fmt == GSK_FMT_SELL && P->sell.rcd) {  // row-class dictionary (no slot data)
      auto k = !P->hrcd.kslots ? pass_kernel<5, 1, Op, true>
                               : P->hrcd.ns == 7 ? pass_kernel<6, 1, Op, true> : pass_kernel<7, 1, Op, true>;
      pass_carveout(k);
      GSK_CUDA(launch_k(k, ntiles, TB, 0, s, P->csr, P->sell, n, wpc, op, P->part, P->pstride, rev));
    } else if (P->fmt == GSK_FMT_SELL && P->sell.uptr) {
      auto k = nat ? pass_kernel<4, 1, Op, true> : pass_kernel<4, 1, Op, false>;
      pass_carveout(k);
      GSK_CUDA(launch_k(k, ntiles, TB, 0, s, P->csr, P->sell, n, wpc, op, P->part, P->pstride, rev));
    } else if (P->fmt == GSK_FMT_SELL && P->sell.dict) {
      auto k = nat ? pass_kernel<3, 1, Op, true> : pass_kernel<3, 1, Op, false>;
      pass_carveout(k);
      GSK_CUDA(launch_k(k, ntiles, TB, 0, s, P->csr, P->sell, n, wpc, op, P->part, P->pstride, rev));
    } else if (P->fmt == GSK_FMT_SELL) {
      // natural plans with chunks of <= 5 slots (2-D 5-point) run the short-slot kernels
      auto k = !nat ? pass_kernel<2, 1, Op, false>
                    : (P->sell_maxlen <= 5 && short_slots_enabled()) ? pass_kernel<2, 1, Op, true, 5>
                                                                       : pass_kernel<2, 1, Op, true>;
      pass_carveout(k);
      GSK_CUDA(launch_k(k, ntiles, TB, 0, s, P->csr, P->sell, n, wpc, op, P->part, P->pstride, rev));
    } else {  // CSR passes keep the driver's carveout (their 43 KB stage needs it)
      GSK_CUDA(launch_k(pass_kernel<1, 1, Op>, ntiles, TB, 0, s, P->csr, P->sell, n, wpc, op, P->part, P->pstride, rev));
    }
  }
  GSK_LAUNCHED(1);
  if (pe1) GSK_CUDA(cudaEventRecordWithFlags(pe1, s, cudaEventRecordExternal));
  *ntiles_out = ntiles;
  return GSK_OK;
}

// One pass and, when it reduces dot products, the single-CTA finish kernel.  Returns
// the number of kernels launched (or a negative error).
template <class Op>
int run_pass(gsk_plan* P, const Op& op, cudaStream_t s, cudaEvent_t pe0 = nullptr, cudaEvent_t pe1 = nullptr) {
  int ntiles = 0;
  GSK_TRY(launch_pass(P, op, s, &ntiles, pe0, pe1));
  if constexpr (Op::D > 0) {
    GSK_CUDA(launch_k(finish_kernel<Op>, 1, FIN_THREADS, 0, s, op, P->part, P->pstride, ntiles));
    GSK_LAUNCHED(1);
    return 2;
  }
  return 1;
}
// Launch a multi-dot pass (J dots per row) and its J-CTA finish.
template <class Op>
int run_mdot(gsk_plan* P, const Op& op, int J, cudaStream_t s, cudaEvent_t pe0 = nullptr,
             cudaEvent_t pe1 = nullptr) {
  const int n = P->geo.n;
  const int sms = num_sms();
  const int tiles = (n + MD_TILE - 1) / MD_TILE;
  int tpc = 8;  // tiles per CTA: as many as still leave >= 2 waves of CTAs
  while (tpc > 1 && (long long)tiles < (long long)tpc * MDOT_MINB * sms * 2) tpc >>= 1;
  const int ntiles = (tiles + tpc - 1) / tpc;
  const int rev = pass_alternate() ? (P->pass_seq++ & 1) : 0;
  if (pe0) GSK_CUDA(cudaEventRecordWithFlags(pe0, s, cudaEventRecordExternal));
  if constexpr (!Op::kSpmv)
    GSK_CUDA(launch_k(mdot_pass<0, Op>, ntiles, TB, 0, s, P->csr, P->sell, n, tpc, op, P->mpart, P->pstride, rev));
  else if (P->fmt == GSK_FMT_SELL)
    GSK_CUDA(launch_k(mdot_pass<2, Op>, ntiles, TB, 0, s, P->csr, P->sell, n, tpc, op, P->mpart, P->pstride, rev));
  else
    GSK_CUDA(launch_k(mdot_pass<1, Op>, ntiles, TB, 0, s, P->csr, P->sell, n, tpc, op, P->mpart, P->pstride, rev));
  GSK_LAUNCHED(1);
  if (pe1) GSK_CUDA(cudaEventRecordWithFlags(pe1, s, cudaEventRecordExternal));
  GSK_CUDA(launch_k(mdot_finish<Op>, J, FIN_THREADS, 0, s, op, P->mpart, P->pstride, ntiles));
  GSK_LAUNCHED(1);
  return 2;
}

int sell_build(gsk_plan* P, cudaStream_t s);
int sell_fill_values(gsk_plan* P, cudaStream_t s);
int sell_dict_build(gsk_plan* P, cudaStream_t s);
int sellu_build(gsk_plan* P, cudaStream_t s);
int rcd_build(gsk_plan* P, cudaStream_t s);  // also the refresh (the classes depend on the values)
int coop_bicgstab_run(gsk_plan* P, const double* b, double tol, int maxit, double* x, int* used);
// On-chip single-CTA solvers (small.cu) for n <= GSK_SMALL_NMAX: one launch runs the
// whole solve; the caller has set x = x0 and zeroed/initialised the state.
int small_bicgstab_run(gsk_plan* P, const double* b, double tol, int maxit, double* x);
int small_gmres_run(gsk_plan* P, const double* b, double* x, const GmresState& h);
#define GSK_CLUSTER_NMAX 65536        // rows the cluster solvers take (16 CTAs x 4096)
// where engine AUTO picks them (measured, profiles/r01_small_timing.json): Bi-CGSTAB
// up to 32768 rows (19.9 vs 24.0 us/it; 28.3 vs 24.6 at 40000), GMRES up to 65536
#define GSK_CLUSTER_AUTO_BICG 32768
#define GSK_CLUSTER_AUTO_GMRES 65536
#define GSK_COOP_AUTO_BICG 81920  // the cooperative Bi-CGSTAB above the cluster range
// On-chip solvers on one thread-block cluster (cluster.cu) for n <= 65536; *used = 0
// when the system does not fit (the caller then runs the graph path).
int cluster_bicgstab_run(gsk_plan* P, const double* b, double tol, int maxit, double* x, int* used);
int cluster_gmres_run(gsk_plan* P, const double* b, double* x, const GmresState& h, int* used);
int ensure_hist(gsk_plan* P, int maxit);
int bicgstab_report(gsk_plan* P, double* hist, gsk_report* rep, cudaStream_t caller);
int gmres_report(gsk_plan* P, double* hist, gsk_report* rep, cudaStream_t caller);
int plan_create_impl(const gsk_csr* A, const gsk_opts* opts, int sell_pad, gsk_plan** plan, cudaStream_t s);
int shard_bicgstab_run(gsk_plan* P, const double* b, const double* x0, double tol, int maxit, double* x,
                       double* hist, gsk_report* rep, cudaStream_t caller);
int shard_gmres_run(gsk_plan* P, const double* b, const double* x0, int m, double tol, int maxit, double* x,
                    double* hist, gsk_report* rep, cudaStream_t caller);
int shard_refresh(gsk_plan* P, cudaStream_t s);
int64_t shard_row_classes(gsk_plan* P);
int shard_spmv(gsk_plan* P, const double* x, double* y, cudaStream_t caller);
// End a stream capture begun by the caller: instantiate the graph, count its kernel
// nodes (returned in *kernels; launches made during capture are not counted).
int end_capture(cudaStream_t s, int rc, cudaGraphExec_t* out, long long* kernels, const char* what);

// A stream capture fails if another host thread makes a device-wide call meanwhile
// (e.g. cudaDeviceSynchronize invalidates every capture in progress on the device), so
// a failed capture is retried a few times before its error is returned.
template <class F>
int capture_retry(F&& capture) {
  int rc = GSK_OK;
  for (int attempt = 0; attempt < 8; ++attempt) {
    rc = capture();
    if (rc == GSK_OK) return rc;
    cudaGetLastError();  // the invalidation is not sticky; clear it before the next attempt
  }
  return rc;
}
int join_in(gsk_plan* P, cudaStream_t caller);
// Replay graphs[b % NQ] for batch b until the device flag *done_dev is set (checked on
// the host one batch behind, NQ batches in flight) or maxb batches ran; accumulates
// the probe events of the kinds listed.
int run_batches(gsk_plan* P, cudaGraphExec_t* graphs, long long maxb, long long kernels, const int* done_dev,
                const int* kinds, int nkinds);
int join_out(gsk_plan* P, cudaStream_t caller);
}  // namespace gsk
