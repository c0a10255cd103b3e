// internal.cuh — host-side plumbing of libgsk: errors, launch accounting, geometry,
// the plan object and the device-resident solver states.
#pragma once
#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include "common.cuh"
#include "stream.cuh"
#include "gsk.h"

namespace gsk {

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

struct Geometry {
  int n = 0;
};
Geometry make_geometry(int n);

// Device-resident Bi-CGSTAB state (scalars + control flags), DESIGN.md §5.
struct BicgState {
  double rho, rho_prev, alpha, omega, beta, n0, n0u, tol;
  double true_rel, true_rel_w;
  int iter, maxit, done, status, halfstep, bd, hist_len, pad;
};

// Device-resident GMRES(m) state; arrays H[(m+1)*m] (row-major), cs[m], sn[m],
// g[m+1], y[m], inv[m+2] (inv[j] = 1/||w_j||, basis slot j is stored unnormalised).
struct GmresState {
  double beta0, n0w, tol, true_rel, true_rel_w;
  double *H, *cs, *sn, *g, *y, *inv;
  int it, maxit, m, k, cycle_stop, final_, conv, diverged, skip_x, done, status, restarts,
      hist_len, pad;
};

cudaStream_t as_stream(void* s);

}  // namespace gsk

struct gsk_plan {
  gsk_csr A{};
  int fmt = GSK_FMT_CSR;
  int poll = 0;
  int bmode = 2;  // Bi-CGSTAB schedule: 1 fused, 2 split
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
  int64_t nchunks = 0, nslots = 0;
  // reduction scratch
  static constexpr int NSLOT = 16;  // reduction slots (one per pass kind)
  double* part = nullptr;      // [MAXD][256] CTA partials
  unsigned* tickets = nullptr; // [NSLOT]
  double* scratch = nullptr;   // [n] (residual norms)
  cudaStream_t st = nullptr;
  int* h_flag = nullptr;       // pinned
  // Bi-CGSTAB workspace
  double* bvec = nullptr;      // 7 vectors: r, rhat, pa, pb, va, vb, t
  gsk::BicgState* bstate = nullptr;
  cudaGraphExec_t bgraph[2] = {nullptr, nullptr};
  const double* bkey_b = nullptr;
  const double* bkey_x = nullptr;
  int bK = 0;
  const double* bkey_h = nullptr;
  // GMRES workspace
  double* W = nullptr;         // (m+1) n
  int Wm = 0;
  gsk::GmresState* gstate = nullptr;
  double* garr = nullptr;      // H, cs, sn, g, y, inv
  cudaGraphExec_t ggraph[2] = {nullptr, nullptr};
  const double* gkey_b = nullptr;
  const double* gkey_x = nullptr;
  int gkey_m = 0;
  const double* gkey_h = nullptr;
  // history (device)
  double* hist_d = nullptr;
  int hist_cap = 0;
  // kernel probes: per kind, events recorded around one launch per batch
  // kinds: 0 Bi-CGSTAB v = A p pass, 1 Bi-CGSTAB t = A s pass, 2 GMRES MGS pass,
  // 3 GMRES Arnoldi SpMV pass; [graph copy][start/stop]
  static constexpr int NPROBE = 4;
  cudaEvent_t pev[NPROBE][2][2] = {};
  double probe_ms[NPROBE] = {};
  int64_t probe_n[NPROBE] = {};
  cudaEvent_t t0 = nullptr, t1 = nullptr;
};

namespace gsk {
// Launch one fused pass over the plan's rows: Op::kSpmv selects an SpMV pass in the
// plan's format (CSR or SELL) or a pure vector pass.
int num_sms();

// Launch one pass of the streaming engine: an SpMV pass in the plan's format (CSR
// or SELL) or a vector pass; persistent grid of at most 2 CTAs per SM.
template <int FMT, class Op>
int launch_stream(gsk_plan* P, const Op& op, int slot, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    GSK_CUDA(cudaFuncSetAttribute(stream_pass<FMT, Op>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  st_dyn_smem()));
    attr = true;
  }
  const int n = P->geo.n;
  const int rows = FMT == 0 ? VecTile<Op::NV>::W * TB : TB;
  const int ntiles = (n + rows - 1) / rows;
  int tpc = 1;  // tiles per CTA: pow2 with at most 256 CTAs (aligned blocks of the tree)
  while ((ntiles + tpc - 1) / tpc > 256) tpc <<= 1;
  const int grid = (ntiles + tpc - 1) / tpc;
  Red red{P->part, P->tickets + slot, tpc, ntiles};
  stream_pass<FMT, Op><<<grid, ST_THREADS, st_dyn_smem(), s>>>(P->csr, P->sell, n, ntiles, op, red);
  GSK_LAUNCHED(1);
  return GSK_OK;
}

template <class Op>
int run_pass(gsk_plan* P, const Op& op, int slot, cudaStream_t s) {
  if constexpr (!Op::kSpmv) {
    return launch_stream<0>(P, op, slot, s);
  } else {
    if (P->fmt == GSK_FMT_SELL) return launch_stream<2>(P, op, slot, s);
    return launch_stream<1>(P, op, slot, s);
  }
}
#define GSK_TRY(x)              \
  do {                          \
    int rc_ = (x);              \
    if (rc_ != GSK_OK) return rc_; \
  } while (0)

int sell_build(gsk_plan* P, cudaStream_t s);
int sell_fill_values(gsk_plan* P, cudaStream_t s);
int ensure_hist(gsk_plan* P, int maxit);
int join_in(gsk_plan* P, cudaStream_t caller);
int join_out(gsk_plan* P, cudaStream_t caller);
}  // namespace gsk
