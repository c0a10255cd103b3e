// gmres.cu — restarted GMRES(m) (Saad & Schultz 1986) with
// modified Gram-Schmidt Arnoldi (BASELINE north star; reading B9) and the Givens
// least-squares update in one warp (arithmetic AC-7).
//
// Arnoldi step j (1-based) is j+1 fused passes over the rows:
//   S_j      w = A v_j                       h_1j = <w, v_1>
//   M_{i,j}  w = w - h_ij v_i   (i < j)      h_{i+1,j} = <w, v_{i+1}>
//   L_j      w = w - h_jj v_j                ||w||^2 -> h_{j+1,j}; rotations, g,
//                                            history; back substitution at cycle end
// The basis is stored unnormalised (w_j) with inv_j = 1/h_{j,j-1}; every use
// recomputes v_j = RN(w_j * inv_j), the same operation as explicit normalisation, so
// it is bit-identical while saving a read and a write per step.
// A cycle is one captured CUDA graph: the steps, then X (x += sum_k y_k v_k) and R
// (r = b - A x -> next v_1, restart, or the final true residual).  Passes after a
// cycle-ending step return at once (device flag), so the host checks once per cycle.
#include <cmath>
#include <vector>
#include <cstring>
#include "gmres_ops.cuh"

namespace gsk {

static int capture_cycle(gsk_plan* P, const double* b, double* x, int m, int copy, cudaGraphExec_t* out) {
  const size_t n = (size_t)P->A.n;
  cudaStream_t s = P->st;
  GmresState* st = P->gstate;
  auto slot = [&](int j) { return P->W + (size_t)(j - 1) * n; };
  GSK_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  int rc = 0;
  for (int j = 1; j <= m && rc >= 0 && P->orth == 1; ++j) {
    OpCgsS<> sp{slot(j), slot(j + 1), st, j, 0};
    OpCgsA a{};
    a.W = P->W, a.n = n, a.Wn = slot(j + 1), a.st = st, a.j = j;
    OpCgsB bp{};
    bp.W = P->W, bp.n = n, bp.Wn = slot(j + 1), bp.st = st, bp.j = j;
    OpCgsC c{};
    c.W = P->W, c.n = n, c.Wn = slot(j + 1), c.st = st, c.j = j, c.hist = P->hist_d;
    rc = j == 1 ? run_pass(P, sp, s, P->pev[3][copy][0], P->pev[3][copy][1]) : run_pass(P, sp, s);
    if (rc >= 0) rc = run_mdot(P, a, j, s);
    if (rc >= 0) rc = j == 2 ? run_mdot(P, bp, j, s, P->pev[2][copy][0], P->pev[2][copy][1]) : run_mdot(P, bp, j, s);
    if (rc >= 0) rc = run_mdot(P, c, 1, s);
  }
  // GSK_ARNOLDI=fused: S_j and h_1j in one SpMV pass with a dot (OpArnoldi; the same
  // leaves and tree as OpCgsS + OpH1, so the same bits) — an experiment for
  // natural-order SELL plans, whose dot passes need no per-window barrier
  static const bool fused_env = [] {
    const char* e = std::getenv("GSK_ARNOLDI");
    return e && std::strcmp(e, "fused") == 0;
  }();
  const bool fused = fused_env && P->fmt == GSK_FMT_SELL && P->sell.all_nat;
  for (int j = 1; j <= m && rc >= 0 && P->orth == 0; ++j) {
    if (fused) {
      OpArnoldi<> a{slot(j), slot(1), slot(j + 1), st, j, 0, 0};
      rc = j == 1 ? run_pass(P, a, s, P->pev[3][copy][0], P->pev[3][copy][1]) : run_pass(P, a, s);
    } else {
      // S_j as a plain SpMV pass (w = A v_j) + the h_1j dot pass (OpH1)
      OpCgsS<> a{slot(j), slot(j + 1), st, j, 0};
      rc = j == 1 ? run_pass(P, a, s, P->pev[3][copy][0], P->pev[3][copy][1]) : run_pass(P, a, s);
      if (rc >= 0) rc = run_pass(P, OpH1{slot(j + 1), slot(1), st, j, 0}, s);
    }
    for (int i = 1; i < j && rc >= 0; ++i) {
      OpMgs mg{slot(i), slot(i + 1), slot(j + 1), st, i, j, 0, 0, 0};
      rc = (j == 2 && i == 1) ? run_pass(P, mg, s, P->pev[2][copy][0], P->pev[2][copy][1]) : run_pass(P, mg, s);
    }
    if (rc >= 0) {
      OpLast l{slot(j), slot(j + 1), P->hist_d, st, j, 0, 0};
      rc = run_pass(P, l, s);
    }
  }
  if (rc >= 0) {
    OpXupd<> xu{P->W, x, st, n, 0, nullptr, nullptr};
    rc = run_pass(P, xu, s);
  }
  if (rc >= 0) {
    OpGResid<> r{x, b, P->weights, slot(1), P->hist_d, st, 0};
    rc = run_pass(P, r, s);
  }
  return end_capture(s, rc, out, &P->gkernels, "gmres");
}

// Copy the device state and history out into the report (after t1 was recorded).
int gmres_report(gsk_plan* P, double* hist, gsk_report* rep, cudaStream_t caller) {
  cudaStream_t s = P->st;
  GmresState hs{};
  GSK_CUDA(cudaMemcpyAsync(&hs, P->gstate, sizeof hs, cudaMemcpyDeviceToHost, s));
  GSK_CUDA(cudaStreamSynchronize(s));
  std::vector<double> H(hs.hist_len);
  GSK_CUDA(cudaMemcpy(H.data(), P->hist_d, sizeof(double) * hs.hist_len, cudaMemcpyDeviceToHost));
  if (hist) std::copy(H.begin(), H.end(), hist);
  float ms = 0;
  GSK_CUDA(cudaEventElapsedTime(&ms, P->t0, P->t1));
  rep->status = hs.status;
  rep->iterations = hs.it;
  rep->restarts = hs.restarts;
  rep->history_len = hs.hist_len;
  rep->breakdown_at = 0;
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

static int gmres_run(gsk_plan* P, const double* b, const double* x0, int m, double tol, int maxit,
                     double* x, double* hist, gsk_report* rep, cudaStream_t caller) {
  if (!b || !x || !rep || !(tol > 0) || maxit < 1 || m < 1 || m > MAX_M) {
    set_error("gmres: invalid arguments (b, x, rep non-null; tol > 0; maxit >= 1; 1 <= m <= %d)", MAX_M);
    return GSK_E_INVALID;
  }
  if (P->shards) return shard_gmres_run(P, b, x0, m, tol, maxit, x, hist, rep, caller);
  const size_t n = (size_t)P->A.n;
  if (P->Wm < m) {
    if (P->W) {
      GSK_CUDA(cudaStreamSynchronize(P->st));  // no queued pass still reads it
      pool_release(P->W);
    }
    P->W = nullptr;
    cudaError_t e = pool_alloc((void**)&P->W, sizeof(double) * (size_t)(m + 1) * n);
    if (e != cudaSuccess) {
      set_error("gmres: cannot allocate the (m+1) x n basis: %s", cudaGetErrorString(e));
      P->Wm = 0;
      return GSK_E_NOMEM;
    }
    P->Wm = m;
    for (auto& g : P->ggraph)
      if (g) {
        cudaGraphExecDestroy(g);
        g = nullptr;
      }
  }
  if (P->orth == 1 && m > MDOT_MAX) {
    set_error("gmres: double classical Gram-Schmidt supports m <= %d", MDOT_MAX);
    return GSK_E_INVALID;
  }
  if (P->orth == 1 && !P->mpart)
    GSK_CUDA(pool_alloc((void**)&P->mpart, sizeof(double) * MDOT_MAX * (size_t)P->pstride));
  if (!P->gstate) GSK_CUDA(pool_alloc((void**)&P->gstate, sizeof(GmresState)));
  if (!P->garr) GSK_CUDA(pool_alloc((void**)&P->garr, sizeof(double) * (size_t)((MAX_M + 1) * MAX_M + 7 * MAX_M + 8)));
  GSK_TRY(ensure_hist(P, maxit));
  // small systems: the whole solve in one launch on one SM (small.cu), MGS only
  // (default for n <= 1024), or on one thread-block cluster (cluster.cu) up to 65536
  // rows and m <= 40 (2-2.4x faster than the graph passes there)
  const bool small = ((P->engine == GSK_ENGINE_AUTO && n <= 1024) || (P->engine == GSK_ENGINE_SMALL && n <= GSK_SMALL_NMAX)) &&
                     P->orth == 0;
  const bool clus = !small && P->orth == 0 && m <= 40 &&
                    ((P->engine == GSK_ENGINE_AUTO && n <= GSK_CLUSTER_AUTO_GMRES) ||
                     (P->engine == GSK_ENGINE_CLUSTER && n <= GSK_CLUSTER_NMAX));
  // the graph passes' captured cycles (for these b, x, m, history and orthogonalisation)
  auto ensure_graphs = [&]() -> int {
    if (P->ggraph[0] && P->gkey_b == b && P->gkey_x == x && P->gkey_m == m && P->gkey_h == P->hist_d &&
        P->gkey_orth == P->orth)
      return GSK_OK;
    for (auto& g : P->ggraph)
      if (g) {
        cudaGraphExecDestroy(g);
        g = nullptr;
      }
    for (int c = 0; c < gsk_plan::NQ; ++c) GSK_TRY(capture_retry([&] { return capture_cycle(P, b, x, m, c, &P->ggraph[c]); }));
    P->gkey_b = b;
    P->gkey_x = x;
    P->gkey_m = m;
    P->gkey_h = P->hist_d;
    P->gkey_orth = P->orth;
    return GSK_OK;
  };
  if (!small && !clus) GSK_TRY(ensure_graphs());
  cudaStream_t s = P->st;
  GSK_TRY(join_in(P, caller));
  GSK_CUDA(cudaEventRecord(P->t0, s));
  if (x0) {
    if (x0 != x) GSK_CUDA(cudaMemcpyAsync(x, x0, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  } else {
    GSK_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, s));
  }
  GmresState h{};
  double* A = P->garr;
  h.H = A;
  h.cs = A + (MAX_M + 1) * MAX_M;
  h.sn = h.cs + MAX_M;
  h.g = h.sn + MAX_M;
  h.y = h.g + MAX_M + 1;
  h.inv = h.y + MAX_M;
  h.c1 = h.inv + MAX_M + 2;
  h.c2 = h.c1 + MAX_M;
  h.tol = tol;
  h.maxit = maxit;
  h.m = m;
  h.wstop = P->wstop;
  GSK_CUDA(cudaMemsetAsync(P->garr, 0, sizeof(double) * (size_t)((MAX_M + 1) * MAX_M + 7 * MAX_M + 8), s));
  GSK_CUDA(cudaMemcpyAsync(P->gstate, &h, sizeof h, cudaMemcpyHostToDevice, s));
  int cused = 0;
  if (clus) {
    const int rc = cluster_gmres_run(P, b, x, h, &cused);
    if (rc != GSK_OK) {  // e.g. a cluster that cannot be scheduled (MIG, partitioned GPU)
      if (P->engine != GSK_ENGINE_AUTO) return rc;
      cudaGetLastError();  // AUTO: the graph passes below instead
      cused = 0;
    }
  }
  if (small) {
    GSK_TRY(small_gmres_run(P, b, x, h));
  } else if (cused) {
  } else {
    if (clus) {  // the cluster engine declined: capture now (nothing pending on the plan stream)
      GSK_CUDA(cudaStreamSynchronize(s));
      GSK_TRY(ensure_graphs());
    }
    OpGResid<> init{x, b, P->weights, P->W, P->hist_d, P->gstate, 1};
    if (run_pass(P, init, s) < 0) return GSK_E_CUDA;
    const long long maxc = (long long)maxit + 2;
    const int kinds[2] = {2, 3};
    GSK_TRY(run_batches(P, P->ggraph, maxc, P->gkernels, &P->gstate->done, kinds, 2));
  }
  GSK_CUDA(cudaEventRecord(P->t1, s));
  return gmres_report(P, hist, rep, caller);
}

}  // namespace gsk

using namespace gsk;

extern "C" int gsk_gmres_solve_plan(gsk_plan* plan, const double* b, const double* x0, int m, double tol,
                                    int maxit, double* x, double* hist, gsk_report* rep, void* stream) {
  NvtxRange nv("gsk:gmres");
  if (!plan) {
    set_error("gsk_gmres_solve_plan: plan is NULL");
    return GSK_E_INVALID;
  }
  return gmres_run(plan, b, x0, m, tol, maxit, x, hist, rep, as_stream(stream));
}

extern "C" int gsk_gmres_solve(const gsk_csr* A, const double* b, const double* x0, int m, double tol,
                               int maxit, double* x, double* hist, gsk_report* rep, void* stream) {
  gsk_plan* P = nullptr;
  GSK_TRY(gsk_plan_create(A, nullptr, &P, stream));
  int rc = gmres_run(P, b, x0, m, tol, maxit, x, hist, rep, as_stream(stream));
  gsk_plan_destroy(P);
  return rc;
}
