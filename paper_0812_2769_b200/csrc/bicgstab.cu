// bicgstab.cu — Bi-CGSTAB (van der Vorst 1992) as three
// fused device passes per iteration with device-resident scalars:
//
//   P1  p = r + beta (p_old - omega v_old)  recomputed at every gathered column,
//       v = A p,   sigma = <r^, v>          -> alpha = rho / sigma
//   P2  s = r - alpha v  recomputed at every gathered column,
//       t = A s,   <t,s>, <t,t>, ||s||_w^2  -> half-step exit or omega = <t,s>/<t,t>
//   P3  x += alpha p + omega s,  r = s - omega t,  <r^, r>, ||r||_w^2
//       -> history, stopping test, breakdown tests
//          (PAPER.md:315-321), rho, beta
//
// p and v are double-buffered (the pass that writes p_new/v_new still gathers
// p_old/v_old at neighbouring columns).  Recomputing p and s at the gather is the
// same operation on the same operands as the stored value, so results are
// bit-identical to the unfused algorithm (AC-6) while moving 2 B_A + 17 vectors
// per iteration instead of 2 B_A + 19.  The split schedule S0..S4 (below; the
// default, measured faster on B200) keeps plain SpMV gathers.  Each reducing pass is
// followed by a one-CTA finish kernel (canonical tree + scalar epilogue), so
// iterations run back to back from a captured CUDA graph (K iterations per replay)
// with one host check of the `done` flag per replay, NQ replays in flight.
#include <cmath>
#include <vector>
#include "bicg_ops.cuh"

namespace gsk {

static int batch_size(const gsk_plan* P) {
  int K = P->poll;
  if (K <= 0) {
    const long long n = P->A.n;
    K = (int)std::min<long long>(64, std::max<long long>(4, (1LL << 26) / n));  // ~4+ ms batches at C4
  }
  return (K + 1) & ~1;  // even: p/v buffer parity repeats per replay
}

static int capture_bicg(gsk_plan* P, double* x, int K, int copy, cudaGraphExec_t* out) {
  const int n = P->A.n;
  double* V = P->bvec;
  double *r = V, *rh = V + (size_t)n, *pa = V + 2 * (size_t)n, *pb = V + 3 * (size_t)n,
         *va = V + 4 * (size_t)n, *vb = V + 5 * (size_t)n, *t = V + 6 * (size_t)n;
  const double* w = P->weights;
  cudaStream_t s = P->st;
  GSK_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  int rc = 0;
  auto ev = [&](int kind, int edge, int k) { return k == 0 ? P->pev[kind][copy][edge] : nullptr; };
  for (int k = 0; k < K && rc >= 0; ++k) {
    if (P->bmode == 1) {  // fused 3-pass schedule
      double *po = (k & 1) ? pb : pa, *vo = (k & 1) ? vb : va;
      double *pn = (k & 1) ? pa : pb, *vn = (k & 1) ? va : vb;
      OpP1<> p1{r, po, vo, rh, pn, vn, P->bstate, 0, 0};
      OpP2<> p2{r, vn, w, t, P->hist_d, P->bstate, 0};
      OpP3 p3{vn, pn, t, rh, w, x, r, P->hist_d, P->bstate, 0, 0, 0};
      rc = run_pass(P, p1, s, ev(0, 0, k), ev(0, 1, k));
      if (rc >= 0) rc = run_pass(P, p2, s, ev(1, 0, k), ev(1, 1, k));
      if (rc >= 0) rc = run_pass(P, p3, s, ev(4, 0, k), ev(4, 1, k));
    } else if (P->bmode == 3) {  // four-pass schedule: q / p alternate between pa and vb
      double *qs = (k & 1) ? vb : pa, *pd = (k & 1) ? pa : vb;
      double *v = va, *sv = pb;
      OpS1q<> s1{qs, r, rh, pd, v, P->bstate, 0.0};
      OpS2 s2{r, v, w, sv, P->hist_d, P->bstate, 0};
      OpS3<> s3{sv, t, P->bstate};
      OpS4q s4{sv, t, rh, w, v, pd, x, r, P->hist_d, P->bstate, 0, 0, 0, 0};
      rc = run_pass(P, s1, s, ev(0, 0, k), ev(0, 1, k));
      if (rc >= 0) rc = run_pass(P, s2, s);
      if (rc >= 0) rc = run_pass(P, s3, s, ev(1, 0, k), ev(1, 1, k));
      if (rc >= 0) rc = run_pass(P, s4, s, ev(4, 0, k), ev(4, 1, k));
    } else {  // split 5-pass schedule: p = pa, v = va, s = pb
      double *p = pa, *v = va, *sv = pb;
      OpS0 s0{r, v, p, P->bstate, 0, 0};
      OpS1<> s1{p, rh, v, P->bstate};
      OpS2 s2{r, v, w, sv, P->hist_d, P->bstate, 0};
      OpS3<> s3{sv, t, P->bstate};
      OpS4 s4{sv, p, t, rh, w, x, r, P->hist_d, P->bstate, 0, 0, 0};
      rc = run_pass(P, s0, s);
      if (rc >= 0) rc = run_pass(P, s1, s, ev(0, 0, k), ev(0, 1, k));
      if (rc >= 0) rc = run_pass(P, s2, s);
      if (rc >= 0) rc = run_pass(P, s3, s, ev(1, 0, k), ev(1, 1, k));
      if (rc >= 0) rc = run_pass(P, s4, s, ev(4, 0, k), ev(4, 1, k));
    }
  }
  return end_capture(s, rc, out, &P->bkernels, "bicgstab");
}

// Copy the device state and history out into the report (after t1 was recorded).
int bicgstab_report(gsk_plan* P, double* hist, gsk_report* rep, cudaStream_t caller) {
  cudaStream_t s = P->st;
  BicgState hs{};
  GSK_CUDA(cudaMemcpyAsync(&hs, P->bstate, sizeof hs, cudaMemcpyDeviceToHost, s));
  GSK_CUDA(cudaStreamSynchronize(s));
  std::vector<double> H(hs.hist_len);
  GSK_CUDA(cudaMemcpy(H.data(), P->hist_d, sizeof(double) * hs.hist_len, cudaMemcpyDeviceToHost));
  if (hist) std::copy(H.begin(), H.end(), hist);
  float ms = 0;
  GSK_CUDA(cudaEventElapsedTime(&ms, P->t0, P->t1));
  rep->status = hs.status;
  rep->iterations = hs.hist_len - 1;
  rep->restarts = 0;
  rep->history_len = hs.hist_len;
  rep->breakdown_at = hs.bd;
  rep->pad_ = 0;
  rep->relres = H.back();
  rep->true_relres = hs.true_rel;
  rep->true_relres_w = hs.true_rel_w;
  double best = H[0];
  for (double v : H) best = std::min(best, v);
  rep->best_relres = best;
  rep->solve_ms = ms;
  GSK_TRY(join_out(P, caller));
  return GSK_OK;
}

static int bicgstab_run(gsk_plan* P, const double* b, const double* x0, double tol, int maxit,
                        double* x, double* hist, gsk_report* rep, cudaStream_t caller) {
  if (!b || !x || !rep || !(tol > 0) || maxit < 1) {
    set_error("bicgstab: invalid arguments (b, x, rep non-null; tol > 0; maxit >= 1)");
    return GSK_E_INVALID;
  }
  if (P->shards) return shard_bicgstab_run(P, b, x0, tol, maxit, x, hist, rep, caller);
  const int n = P->A.n;
  if (!P->bvec) GSK_CUDA(pool_alloc((void**)&P->bvec, sizeof(double) * 7 * (size_t)n));
  if (!P->bstate) GSK_CUDA(pool_alloc((void**)&P->bstate, sizeof(BicgState)));
  GSK_TRY(ensure_hist(P, maxit));
  // small systems: one launch runs the whole iteration loop — on one SM with the
  // vectors in shared memory (small.cu; by default for n <= 2048, where
  // it is measured faster: 6.7 vs 31 us per iteration at n = 1024), on one cluster or
  // on a cooperative grid.  Same operators, bit-identical results.
  const bool small = (P->engine == GSK_ENGINE_AUTO && n <= 2048) ||
                     (P->engine == GSK_ENGINE_SMALL && n <= GSK_SMALL_NMAX);
  // one thread-block cluster (cluster.cu) above that, up to 16384 rows: 12-15 vs 25-27
  // us per iteration on the graph passes
  const bool clus = !small && ((P->engine == GSK_ENGINE_AUTO && n <= GSK_CLUSTER_AUTO_BICG) ||
                               (P->engine == GSK_ENGINE_CLUSTER && n <= GSK_CLUSTER_NMAX));
  // a persistent cooperative grid (coop.cu) above that, up to 81920 rows: 20.7-24.1 vs
  // 22.9-26.9 us per iteration on the graph passes (profiles/r02v_coop.json); even at
  // ~90000 rows, slower beyond
  const bool coop = !small && !clus && ((P->engine == GSK_ENGINE_AUTO && n <= GSK_COOP_AUTO_BICG) ||
                                        P->engine == GSK_ENGINE_COOP);
  if (small || clus || coop) {
    cudaStream_t s = P->st;
    GSK_TRY(join_in(P, caller));
    GSK_CUDA(cudaEventRecord(P->t0, s));
    if (x0) {
      if (x0 != x) GSK_CUDA(cudaMemcpyAsync(x, x0, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    } else {
      GSK_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, s));
    }
    int used = 1, rc;
    if (small)
      rc = small_bicgstab_run(P, b, tol, maxit, x);
    else if (clus)
      rc = cluster_bicgstab_run(P, b, tol, maxit, x, &used);
    else
      rc = coop_bicgstab_run(P, b, tol, maxit, x, &used);
    if (rc != GSK_OK) {  // e.g. a cluster that cannot be scheduled (MIG, partitioned GPU)
      if (P->engine != GSK_ENGINE_AUTO) return rc;
      cudaGetLastError();  // AUTO: the graph passes below instead
      used = 0;
    }
    if (used) {
      GSK_CUDA(cudaEventRecord(P->t1, s));
      return bicgstab_report(P, hist, rep, caller);
    }
    GSK_CUDA(cudaStreamSynchronize(s));  // nothing pending on the plan stream before the capture
  }
  const int K = batch_size(P);
  if (!P->bgraph[0] || P->bkey_b != b || P->bkey_x != x || P->bK != K || P->bkey_h != P->hist_d) {
    for (auto& g : P->bgraph)
      if (g) {
        cudaGraphExecDestroy(g);
        g = nullptr;
      }
    for (int c = 0; c < gsk_plan::NQ; ++c) GSK_TRY(capture_retry([&] { return capture_bicg(P, x, K, c, &P->bgraph[c]); }));
    P->bkey_b = b;
    P->bkey_x = x;
    P->bK = K;
    P->bkey_h = P->hist_d;
  }
  cudaStream_t s = P->st;
  GSK_TRY(join_in(P, caller));
  GSK_CUDA(cudaEventRecord(P->t0, s));
  if (x0) {
    if (x0 != x) GSK_CUDA(cudaMemcpyAsync(x, x0, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  } else {
    GSK_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, s));
  }
  BicgState h{};
  h.tol = tol;
  h.maxit = maxit;
  read_fault(&h.fault_kind, &h.fault_it);  // test-only hook (graph passes, unsharded)
  GSK_CUDA(cudaMemcpyAsync(P->bstate, &h, sizeof h, cudaMemcpyHostToDevice, s));
  double* V = P->bvec;
  OpInit<> init{x, b, P->weights, V, V + (size_t)n, V + 2 * (size_t)n, V + 4 * (size_t)n, P->hist_d, P->bstate};
  if (run_pass(P, init, s) < 0) return GSK_E_CUDA;
  // batches of K iterations; the next batch is queued before the flag of the
  // previous one is read, so the GPU never idles on the host check
  const long long maxb = (maxit + K - 1) / K + 1;
  const int kinds[3] = {0, 1, 4};
  GSK_TRY(run_batches(P, P->bgraph, maxb, P->bkernels, &P->bstate->done, kinds, 3));
  OpFinal<> fin{x, b, P->weights, P->bstate};
  if (run_pass(P, fin, s) < 0) return GSK_E_CUDA;
  GSK_CUDA(cudaEventRecord(P->t1, s));
  return bicgstab_report(P, hist, rep, caller);
}

}  // namespace gsk

using namespace gsk;

extern "C" int gsk_bicgstab_solve_plan(gsk_plan* plan, const double* b, const double* x0, double tol,
                                       int maxit, double* x, double* hist, gsk_report* rep, void* stream) {
  NvtxRange nv("gsk:bicgstab");
  if (!plan) {
    set_error("gsk_bicgstab_solve_plan: plan is NULL");
    return GSK_E_INVALID;
  }
  return bicgstab_run(plan, b, x0, tol, maxit, x, hist, rep, as_stream(stream));
}

extern "C" int gsk_bicgstab_solve(const gsk_csr* A, const double* b, const double* x0, double tol,
                                  int maxit, double* x, double* hist, gsk_report* rep, void* stream) {
  gsk_plan* P = nullptr;
  GSK_TRY(gsk_plan_create(A, nullptr, &P, stream));
  int rc = bicgstab_run(P, b, x0, tol, maxit, x, hist, rep, as_stream(stream));
  gsk_plan_destroy(P);
  return rc;
}
