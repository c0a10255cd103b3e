// oracle/oracle.cpp — the parity ORACLE.  TEST INFRASTRUCTURE ONLY.
//
// Plain, slow, obviously-correct fp64 CPU implementation of what the hot path
// computes.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load it.  It shares no code, header or constant with
// the CUDA path (paper_0812_2769_b200/csrc); the two meet only in the seeded
// inputs from workloads/.
//
// Paper: Gordon & Gordon, "Geometric scaling: a simple preconditioner for certain
// linear systems with discontinuous coefficients" (arXiv 0812.2769).
//   GS(p)      PAPER.md:92-97 and Eq. (2)
//   L_p norm   PAPER.md:193-196 (|.| applied, reading G1)
//   solvers    PAPER.md:100-102, 232-235 (restarted GMRES, Bi-CGSTAB)
//   stopping   PAPER.md:299-321 (relative residual < eps, breakdown)
//   u0 = 0
// The paper is silent on summation order, FMA use and the Givens / back-solve
// details; the arithmetic contract AC-1..AC-7 of DESIGN.md §4 fixes them and is
// followed here literally:
//   AC-2 no contraction: built with -ffp-contract=off; every fma is std::fma.
//   AC-3 SpMV row: acc = +0; for k ascending: acc = fma(val[k], x[col[k]], acc).
//   AC-5 dot: q_i = RN(a_i*b_i), zero-padded to L = 2^ceil(log2 n), pairwise
//        tree T(2k) = T(first k) + T(last k), result T + 0.0.
//
// Build: g++ -O2 -mfma -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC.
// OpenMP only splits loops whose iterations are independent (rows, elements, the
// pairs of one tree level), so results do not depend on the thread count.
//
// Parity status per function (pins live in tests/test_oracle*.py):
//   orc_dot, orc_spmv, orc_gs_scale, orc_bicgstab, orc_gmres, orc_sell_build: pinned.
#include <cstdint>
#include <cmath>
#include <cstring>
#include <vector>
#include <algorithm>
#include <numeric>
#include <omp.h>

extern "C" {

// Report (mirrors the fields of the C-ABI report by name; independent definition).
struct orc_report {
  int32_t status;        // 0 converged, 1 maxit, 2 breakdown, 3 diverged
  int32_t iterations;
  int32_t restarts;
  int32_t history_len;
  int32_t breakdown_at;
  int32_t pad_;
  double relres;         // last history value
  double true_relres;    // ||b-Ax|| / ||b-Ax0|| (unweighted, solved frame)
  double true_relres_w;  // same with stopping-frame weights (== true_relres if none)
  double best_relres;    // min over the history
};

int orc_num_threads() { return omp_get_max_threads(); }

// ---- AC-5: canonical pairwise tree --------------------------------------------------
static double tree_sum(std::vector<double>& q, int64_t n) {
  int64_t L = 1;
  while (L < n) L <<= 1;
  q.resize(L, 0.0);
  for (int64_t i = n; i < L; ++i) q[i] = 0.0;
  // one tree level at a time: out[i] = in[2i] + in[2i+1] (separate buffers, so
  // splitting a level across threads cannot change any value)
  static thread_local std::vector<double> nxt;
  nxt.resize(L / 2 > 0 ? L / 2 : 1);
  double* in = q.data();
  double* out = nxt.data();
  for (int64_t len = L; len > 1; len >>= 1) {
    #pragma omp parallel for schedule(static) if (len > 65536)
    for (int64_t i = 0; i < len / 2; ++i) out[i] = in[2 * i] + in[2 * i + 1];
    std::copy(out, out + len / 2, in);
  }
  return q[0] + 0.0;
}

// products buffer reused across calls (allocation only; no arithmetic involved)
static std::vector<double>& leaves(int64_t n) {
  static thread_local std::vector<double> q;
  q.assign(n > 0 ? n : 1, 0.0);
  return q;
}

// <a, b> under AC-5.
double orc_dot(int64_t n, const double* a, const double* b) {
  std::vector<double>& q = leaves(n);
  double* qp = q.data();
  #pragma omp parallel for schedule(static) if (n > 65536)
  for (int64_t i = 0; i < n; ++i) qp[i] = a[i] * b[i];
  return tree_sum(q, n);
}

// sum_i (w_i a_i)^2 under AC-5 (w null: plain <a,a>).
double orc_wnorm2(int64_t n, const double* a, const double* w) {
  std::vector<double>& q = leaves(n);
  double* qp = q.data();
  #pragma omp parallel for schedule(static) if (n > 65536)
  for (int64_t i = 0; i < n; ++i) {
    double u = w ? w[i] * a[i] : a[i];
    qp[i] = u * u;
  }
  return tree_sum(q, n);
}

// ---- SpMV, AC-3 (SPEC sparse-core spmv; y = A x) -----------------------------------
void orc_spmv(int64_t n, const int32_t* rp, const int32_t* ci, const double* v,
              const double* x, double* y) {
  #pragma omp parallel for schedule(static) if (n > 65536)
  for (int64_t i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int32_t k = rp[i]; k < rp[i + 1]; ++k) acc = std::fma(v[k], x[ci[k]], acc);
    y[i] = acc;
  }
}

// ---- GS(p): Eq. (2), PAPER.md:207-214 ------------------------------------------------
// d_i = 1/||a_i||_p ; (DA)_ij = a_ij * d_i ; (Db)_i = b_i * d_i   (reading G2: multiply
// by D as written).  AC-4 norm: p=2 acc = fma(a,a,acc), sqrt; p=1 acc += |a|;
// p>=3 |a|^p by repeated multiplication, root pow(acc, 1/p).
// Returns 0, -1 (p<1), or -2 (zero row; *bad_row = smallest such row).  Outputs may
// alias inputs.  b / b_out / d_out may be null.
int orc_gs_scale(int64_t n, const int32_t* rp, const double* val, const double* b, int p,
                 double* val_out, double* b_out, double* d_out, int32_t* bad_row) {
  if (p < 1) return -1;
  std::vector<double> d(n);
  int64_t bad = -1;
  for (int64_t i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int32_t k = rp[i]; k < rp[i + 1]; ++k) {
      double a = std::fabs(val[k]);
      if (p == 1) acc = acc + a;
      else if (p == 2) acc = std::fma(val[k], val[k], acc);
      else {
        double t = a;
        for (int e = 1; e < p; ++e) t = t * a;
        acc = acc + t;
      }
    }
    double nrm = (p == 1) ? acc : (p == 2 ? std::sqrt(acc) : std::pow(acc, 1.0 / p));
    if (nrm == 0.0) { if (bad < 0) bad = i; d[i] = 0.0; continue; }
    d[i] = 1.0 / nrm;
  }
  if (bad >= 0) { if (bad_row) *bad_row = (int32_t)bad; return -2; }
  for (int64_t i = 0; i < n; ++i) {
    for (int32_t k = rp[i]; k < rp[i + 1]; ++k) val_out[k] = val[k] * d[i];
    if (b && b_out) b_out[i] = b[i] * d[i];
    if (d_out) d_out[i] = d[i];
  }
  return 0;
}

// ---- two-sided scaling D^(1/2) A D^(1/2) y = D^(1/2) b, x = D^(1/2) y --------------
// PAPER.md:245-251 (the variant the authors also tried).  D = diag(1/||a_i||_p) as in
// Eq. (2); reading S1: s_i = sqrt(d_i), a'_ij = (a_ij * s_i) * s_j
// (left factor first), b'_i = b_i * s_i, and x_i = s_i * y_i.
int orc_gs_scale_sym(int64_t n, const int32_t* rp, const int32_t* ci, const double* val,
                     const double* b, int p, double* val_out, double* b_out, double* s_out,
                     int32_t* bad_row) {
  std::vector<double> d(n);
  int rc = orc_gs_scale(n, rp, val, nullptr, p, std::vector<double>(rp[n]).data(), nullptr,
                        d.data(), bad_row);
  if (rc != 0) return rc;
  std::vector<double> sq(n);
  for (int64_t i = 0; i < n; ++i) sq[i] = std::sqrt(d[i]);
  for (int64_t i = 0; i < n; ++i) {
    for (int32_t k = rp[i]; k < rp[i + 1]; ++k) val_out[k] = (val[k] * sq[i]) * sq[ci[k]];
    if (b && b_out) b_out[i] = b[i] * sq[i];
    if (s_out) s_out[i] = sq[i];
  }
  return 0;
}

void orc_unscale(int64_t n, const double* s, const double* y, double* x) {
  for (int64_t i = 0; i < n; ++i) x[i] = s[i] * y[i];
}

// ---- SELL-C-sigma layout (BASELINE.json configs[3]) -------------------------------
// Windows of sigma consecutive rows; inside a window rows are stably sorted by
// descending length (ties keep row order) — unless the rows in their natural order
// need no more padded slots than sorted (reading L1: the sort only exists to
// cut padding), in which case the window keeps the natural order; chunks of C rows;
// chunk_len = longest row of the chunk; slot (k, lane) of chunk c at
// chunk_ptr[c] + k*C + lane, holding the row's k-th CSR entry (CSR order kept) or
// col -1 / val 0 as padding; roff[c*C + lane] = in-window offset of the row (uint8,
// sigma <= 256).
int64_t orc_sell_size(int64_t n, const int32_t* rp, int C, int sigma) {
  int64_t nch = (n + C - 1) / C, tot = 0;
  for (int64_t w = 0; w * sigma < n; ++w) {
    int64_t r0 = w * sigma, r1 = std::min<int64_t>(n, r0 + sigma);
    std::vector<int32_t> len;
    for (int64_t r = r0; r < r1; ++r) len.push_back(rp[r + 1] - rp[r]);
    std::stable_sort(len.begin(), len.end(), [](int32_t a, int32_t b) { return a > b; });
    for (size_t s = 0; s < len.size(); s += C) tot += (int64_t)len[s] * C;
  }
  (void)nch;
  return tot;
}

int orc_sell_build(int64_t n, const int32_t* rp, const int32_t* ci, const double* v, int C,
                   int sigma, int32_t* chunk_ptr, int32_t* chunk_len, int32_t* scol,
                   double* sval, uint8_t* roff) {
  if (C <= 0 || sigma <= 0 || sigma % C != 0 || sigma > 256) return -1;
  int64_t nch = (n + C - 1) / C;
  chunk_ptr[0] = 0;
  for (int64_t w = 0; w * sigma < n; ++w) {
    int64_t r0 = w * sigma, r1 = std::min<int64_t>(n, r0 + sigma), cnt = r1 - r0;
    std::vector<int32_t> order(cnt), sorted(cnt);
    std::iota(order.begin(), order.end(), 0);
    std::iota(sorted.begin(), sorted.end(), 0);
    std::stable_sort(sorted.begin(), sorted.end(), [&](int32_t a, int32_t b) {
      return (rp[r0 + a + 1] - rp[r0 + a]) > (rp[r0 + b + 1] - rp[r0 + b]);
    });
    auto slots = [&](const std::vector<int32_t>& ord) {  // padded slots of the window / C
      int64_t tot = 0;
      for (int64_t s0 = 0; s0 < cnt; s0 += C) {
        int32_t L = 0;
        for (int64_t s = s0; s < std::min<int64_t>(cnt, s0 + C); ++s)
          L = std::max(L, rp[r0 + ord[s] + 1] - rp[r0 + ord[s]]);
        tot += L;
      }
      return tot;
    };
    if (slots(order) > slots(sorted)) order = sorted;
    int64_t c0 = r0 / C, c1 = (r1 + C - 1) / C;
    for (int64_t c = c0; c < c1; ++c) {
      int64_t s0 = c * C - r0;  // first position of the chunk in this window
      int32_t L = 0;
      for (int64_t s = s0; s < std::min<int64_t>(cnt, s0 + C); ++s)
        L = std::max(L, rp[r0 + order[s] + 1] - rp[r0 + order[s]]);
      chunk_len[c] = L;
      chunk_ptr[c + 1] = chunk_ptr[c] + L * C;
      for (int lane = 0; lane < C; ++lane) {
        int64_t s = s0 + lane;
        bool real = s < cnt;
        int64_t row = real ? r0 + order[s] : -1;
        roff[c * C + lane] = (uint8_t)(real ? order[s] : s);
        int32_t len = real ? rp[row + 1] - rp[row] : 0;
        for (int32_t k = 0; k < L; ++k) {
          int64_t slot = (int64_t)chunk_ptr[c] + (int64_t)k * C + lane;
          if (k < len) { scol[slot] = ci[rp[row] + k]; sval[slot] = v[rp[row] + k]; }
          else { scol[slot] = -1; sval[slot] = 0.0; }
        }
      }
    }
  }
  (void)nch;
  return 0;
}

// ---- SELL column-index dictionary (storage format of the GPU path) ----
// Per chunk c: D_c = ascending distinct deltas (col - row) over the chunk's real slots;
// idx[slot] = position of the slot's delta in D_c, 255 for padding.  Valid only when
// every |D_c| <= 32 (returns 0), else returns 1 (format not applicable).
int64_t orc_sell_dict_size(int64_t n, int C, int sigma, const int32_t* chunk_ptr, const int32_t* scol,
                           const uint8_t* roff) {
  int64_t nch = (n + C - 1) / C, tot = 0;
  for (int64_t c = 0; c < nch; ++c) {
    std::vector<int32_t> d;
    int64_t w0 = (c * C) / sigma * sigma;
    int32_t L = (chunk_ptr[c + 1] - chunk_ptr[c]) / C;
    for (int lane = 0; lane < C; ++lane) {
      int64_t row = w0 + roff[c * C + lane];
      for (int32_t k = 0; k < L; ++k) {
        int32_t col = scol[chunk_ptr[c] + (int64_t)k * C + lane];
        if (col >= 0) d.push_back((int32_t)(col - row));
      }
    }
    std::sort(d.begin(), d.end());
    d.erase(std::unique(d.begin(), d.end()), d.end());
    if (d.size() > 32) return -1;
    tot += (int64_t)d.size();
  }
  return tot;
}

int orc_sell_dict(int64_t n, int C, int sigma, const int32_t* chunk_ptr, const int32_t* scol,
                  const uint8_t* roff, int32_t* dict_ptr, int32_t* dict, uint8_t* sidx) {
  int64_t nch = (n + C - 1) / C;
  dict_ptr[0] = 0;
  for (int64_t c = 0; c < nch; ++c) {
    std::vector<int32_t> d;
    int64_t w0 = (c * C) / sigma * sigma;
    int32_t L = (chunk_ptr[c + 1] - chunk_ptr[c]) / C;
    for (int lane = 0; lane < C; ++lane) {
      int64_t row = w0 + roff[c * C + lane];
      for (int32_t k = 0; k < L; ++k) {
        int32_t col = scol[chunk_ptr[c] + (int64_t)k * C + lane];
        if (col >= 0) d.push_back((int32_t)(col - row));
      }
    }
    std::sort(d.begin(), d.end());
    d.erase(std::unique(d.begin(), d.end()), d.end());
    if (d.size() > 32) return 1;
    for (size_t u = 0; u < d.size(); ++u) dict[dict_ptr[c] + u] = d[u];
    dict_ptr[c + 1] = dict_ptr[c] + (int32_t)d.size();
    for (int lane = 0; lane < C; ++lane) {
      int64_t row = w0 + roff[c * C + lane];
      for (int32_t k = 0; k < L; ++k) {
        int64_t slot = chunk_ptr[c] + (int64_t)k * C + lane;
        int32_t col = scol[slot];
        if (col < 0) { sidx[slot] = 255; continue; }
        int32_t delta = (int32_t)(col - row);
        sidx[slot] = (uint8_t)(std::lower_bound(d.begin(), d.end(), delta) - d.begin());
      }
    }
  }
  return 0;
}

// ---- SELL-U: chunk-uniform column offsets (storage format of the GPU path)
// For chunk c of a SELL layout (rows given by roff): U_c = the ascending distinct deltas
// col - row over the chunk's rows (at most maxu; else the encoding is inapplicable and
// -1 is returned); slot k of lane l (at uptr[c] + k*C + lane) holds row l's entry at
// column row + U_c[k], or 0.0 with bit l of umask[c*maxu + k] clear.  Sizes: return
// the slot total (call with null outputs first), uptr [nch+1], udel/umask [nch*maxu].
int64_t orc_sell_uniform(int64_t n, int C, int sigma, int maxu, const uint8_t* roff, const int32_t* rp,
                         const int32_t* ci, const double* v, int32_t* uptr, int32_t* udel, uint32_t* umask,
                         double* uval) {
  const int64_t nch = (n + C - 1) / C;
  int64_t tot = 0;
  if (uptr) uptr[0] = 0;
  for (int64_t c = 0; c < nch; ++c) {
    const int64_t w0 = (c * C) / sigma * sigma;
    std::vector<int64_t> U;  // ascending distinct deltas of the chunk
    for (int lane = 0; lane < C; ++lane) {
      const int64_t row = w0 + roff[c * C + lane];
      if (row >= n) continue;
      for (int32_t q = rp[row]; q < rp[row + 1]; ++q) U.push_back((int64_t)ci[q] - row);
    }
    std::sort(U.begin(), U.end());
    U.erase(std::unique(U.begin(), U.end()), U.end());
    if ((int64_t)U.size() > maxu) return -1;
    if (uptr) {
      uptr[c + 1] = (int32_t)(uptr[c] + (int64_t)U.size() * C);
      for (int k = 0; k < maxu; ++k) {
        udel[c * maxu + k] = k < (int)U.size() ? (int32_t)U[k] : 0;
        umask[c * maxu + k] = 0u;
      }
      for (int lane = 0; lane < C; ++lane) {
        const int64_t row = w0 + roff[c * C + lane];
        for (size_t k = 0; k < U.size(); ++k) {
          double a = 0.0;
          bool has = false;
          if (row < n)
            for (int32_t q = rp[row]; q < rp[row + 1]; ++q)
              if ((int64_t)ci[q] - row == U[k]) { a = v[q]; has = true; }
          uval[uptr[c] + (int64_t)k * C + lane] = a;
          if (has) umask[c * maxu + k] |= 1u << lane;
        }
      }
    }
    tot += (int64_t)U.size() * C;
  }
  return tot;
}

// ---- Row-class dictionary (storage format of the GPU path; DESIGN.md §5 "RCD") ----------
// The paper's test problems have piecewise-constant coefficients (PAPER.md:269-294,
// 328-347, 878-895): whole regions of the grid share one stencil row, before and after
// GS(p).  Two rows are of the same class when they have the same length, the same
// deltas col - row and bit-identical values, entry by entry in CSR order.  Classes are
// numbered by first occurrence in ascending row order; class k's entry holds its length,
// deltas and values (unused places 0).  Inapplicable (-1) when some row has more than
// maxlen entries or there are more than maxcls classes.  Outputs (nullable to only
// count): cls [n], dlen [maxcls], ddel / dval [maxcls * maxlen].  Returns the class count.
int64_t orc_row_classes(int64_t n, const int32_t* rp, const int32_t* ci, const double* v, int maxlen,
                        int maxcls, uint16_t* cls, int32_t* dlen, int32_t* ddel, double* dval) {
  std::vector<int64_t> rep;  // first row of every class, in order of appearance
  for (int64_t i = 0; i < n; ++i) {
    const int32_t a = rp[i], len = rp[i + 1] - a;
    if (len > maxlen) return -1;
    int64_t k = 0;
    for (; k < (int64_t)rep.size(); ++k) {  // plain linear search over the classes so far
      const int64_t r = rep[k];
      if (rp[r + 1] - rp[r] != len) continue;
      bool same = true;
      for (int32_t q = 0; q < len && same; ++q) {
        same = ((int64_t)ci[a + q] - i == (int64_t)ci[rp[r] + q] - r) &&
               std::memcmp(&v[a + q], &v[rp[r] + q], sizeof(double)) == 0;
      }
      if (same) break;
    }
    if (k == (int64_t)rep.size()) {
      if ((int64_t)rep.size() == maxcls) return -1;
      rep.push_back(i);
    }
    if (cls) cls[i] = (uint16_t)k;
  }
  if (dlen) {
    for (int64_t k = 0; k < (int64_t)rep.size(); ++k) {
      const int64_t r = rep[k];
      const int32_t len = rp[r + 1] - rp[r];
      dlen[k] = len;
      for (int q = 0; q < maxlen; ++q) {
        ddel[k * maxlen + q] = q < len ? (int32_t)((int64_t)ci[rp[r] + q] - r) : 0;
        dval[k * maxlen + q] = q < len ? v[rp[r] + q] : 0.0;
      }
    }
  }
  return (int64_t)rep.size();
}

// ---- Bi-CGSTAB (van der Vorst 1992, cited PAPER.md:102) ----------------------------
// DESIGN.md §4 algorithm B, arithmetic AC-6; stopping PAPER.md:302-307 (reading B1/B2:
// strict <, frame weights w optional); breakdown exact-zero tests (PAPER.md:315-321,
// reading B5); ||s|| half-step exit (B4); iterations = completed iterations (B6).
// hist[maxit+1] (nullable).  x0 nullable (= 0).  Returns 0 or -1 (bad args).
// Test-only fault hook, mirrored by the GPU's GSK_FAULT: kind 1 forces
// rho = 0 at the end of iteration g_fault_it, 2 forces omega = 0 in it, 3 writes NaN into
// r_0 in its update — so the breakdown and divergence verdicts can be reached on any
// system, identically on both sides.  Not part of the method.
static int g_fault_kind = 0, g_fault_it = 0;
void orc_set_fault(int kind, int it) {
  g_fault_kind = kind;
  g_fault_it = it;
}

int orc_bicgstab(int64_t n, const int32_t* rp, const int32_t* ci, const double* v,
                 const double* b, const double* x0, const double* w, double tol, int maxit,
                 double* x, double* hist, orc_report* rep) {
  if (n < 1 || maxit < 1 || !(tol > 0)) return -1;
  std::vector<double> r(n), rh(n), p(n, 0.0), vv(n, 0.0), s(n), t(n), ax(n);
  for (int64_t i = 0; i < n; ++i) x[i] = x0 ? x0[i] : 0.0;
  orc_spmv(n, rp, ci, v, x, ax.data());
  for (int64_t i = 0; i < n; ++i) { r[i] = b[i] - ax[i]; rh[i] = r[i]; }
  const double n0 = std::sqrt(orc_wnorm2(n, r.data(), w));
  const double n0u = std::sqrt(orc_wnorm2(n, r.data(), nullptr));
  std::memset(rep, 0, sizeof(*rep));
  std::vector<double> H;  // history
  H.push_back(n0 == 0.0 ? 0.0 : 1.0);
  int status = 1, iters = 0, bd = 0;
  if (n0 == 0.0) {
    status = 0;
  } else {
    double rho_prev = 1.0, alpha = 1.0, omega = 1.0;
    double rho = orc_dot(n, rh.data(), r.data());
    for (int i = 1; i <= maxit; ++i) {
      if (rho == 0.0) { status = 2; bd = i; break; }
      double beta = (rho / rho_prev) * (alpha / omega);
      for (int64_t k = 0; k < n; ++k) p[k] = std::fma(beta, std::fma(-omega, vv[k], p[k]), r[k]);
      orc_spmv(n, rp, ci, v, p.data(), vv.data());
      double sigma = orc_dot(n, rh.data(), vv.data());
      if (sigma == 0.0) { status = 2; bd = i; break; }
      alpha = rho / sigma;
      for (int64_t k = 0; k < n; ++k) s[k] = std::fma(-alpha, vv[k], r[k]);
      double sn = std::sqrt(orc_wnorm2(n, s.data(), w)) / n0;
      if (sn < tol) {
        for (int64_t k = 0; k < n; ++k) x[k] = std::fma(alpha, p[k], x[k]);
        H.push_back(sn); iters = i; status = 0;
        break;
      }
      orc_spmv(n, rp, ci, v, s.data(), t.data());
      double tt = orc_dot(n, t.data(), t.data());
      if (tt == 0.0) { status = 2; bd = i; break; }
      double ts = orc_dot(n, t.data(), s.data());
      omega = ts / tt;
      if (g_fault_kind == 2 && i == g_fault_it) omega = 0.0;
      for (int64_t k = 0; k < n; ++k) {
        x[k] = std::fma(omega, s[k], std::fma(alpha, p[k], x[k]));
        r[k] = std::fma(-omega, t[k], s[k]);
      }
      if (g_fault_kind == 3 && i == g_fault_it) r[0] = std::nan("");
      rho_prev = rho;
      double rn = std::sqrt(orc_wnorm2(n, r.data(), w)) / n0;
      H.push_back(rn); iters = i;
      if (!std::isfinite(rn)) { status = 3; break; }
      if (rn < tol) { status = 0; break; }
      if (omega == 0.0) { status = 2; bd = i; break; }
      if (i == maxit) { status = 1; break; }
      rho = orc_dot(n, rh.data(), r.data());
      if (g_fault_kind == 1 && i == g_fault_it) rho = 0.0;
    }
  }
  // final true residual (one extra SpMV), PAPER.md:672-677 / SPEC true_relres
  orc_spmv(n, rp, ci, v, x, ax.data());
  for (int64_t i = 0; i < n; ++i) r[i] = b[i] - ax[i];
  double tn = std::sqrt(orc_wnorm2(n, r.data(), nullptr));
  double tw = std::sqrt(orc_wnorm2(n, r.data(), w));
  rep->status = status;
  rep->iterations = iters;
  rep->restarts = 0;
  rep->history_len = (int32_t)H.size();
  rep->breakdown_at = bd;
  rep->relres = H.back();
  rep->true_relres = n0u == 0.0 ? 0.0 : tn / n0u;
  rep->true_relres_w = n0 == 0.0 ? 0.0 : tw / n0;
  rep->best_relres = *std::min_element(H.begin(), H.end());
  if (hist) std::memcpy(hist, H.data(), sizeof(double) * H.size());
  return 0;
}

// ---- restarted GMRES(m) (Saad & Schultz 1986, cited PAPER.md:101) ------------------
// DESIGN.md §4 algorithm G, arithmetic AC-7: modified Gram-Schmidt (reading B9),
// Givens rotations, column-oriented back substitution, x += sum_k y_k v_k (k
// ascending).  Iterations count inner Arnoldi steps (B6).  hist[it] is the
// least-squares residual estimate |g_{j+1}|/||r0||.  w (nullable) only enters the
// reported true_relres_w.
// orth: 0 = modified Gram-Schmidt (north star), 1 = double classical Gram-Schmidt as
// in AZTEC: h = V^T w; w -= V h; h' = V^T w; w -= V h';
// H(:,j) = h + h' (each update an FMA chain over i ascending).
int orc_gmres_orth(int64_t n, const int32_t* rp, const int32_t* ci, const double* v,
                   const double* b, const double* x0, const double* w, int m, double tol, int maxit,
                   int orth, double* x, double* hist, orc_report* rep);
int orc_gmres_wstop(int64_t n, const int32_t* rp, const int32_t* ci, const double* v,
                    const double* b, const double* x0, const double* w, int m, double tol, int maxit,
                    int orth, int wstop, double* x, double* hist, orc_report* rep);

int orc_gmres(int64_t n, const int32_t* rp, const int32_t* ci, const double* v,
              const double* b, const double* x0, const double* w, int m, double tol, int maxit,
              double* x, double* hist, orc_report* rep) {
  return orc_gmres_orth(n, rp, ci, v, b, x0, w, m, tol, maxit, 0, x, hist, rep);
}

int orc_gmres_orth(int64_t n, const int32_t* rp, const int32_t* ci, const double* v,
                   const double* b, const double* x0, const double* w, int m, double tol, int maxit,
                   int orth, double* x, double* hist, orc_report* rep) {
  return orc_gmres_wstop(n, rp, ci, v, b, x0, w, m, tol, maxit, orth, 0, x, hist, rep);
}

// wstop = 1 (reading B2w): the paper measured the relative residual "always"
// on the GS(2)-scaled system.  GMRES's per-step residual is the
// least-squares estimate, which exists only in the frame of the system solved, so with
// frame weights w the stopping test moves to where a residual vector exists: the estimate
// no longer stops the run, and at the end of every cycle (after x += V y and r = b - A x,
// which the restart computes anyway) the run is CONVERGED when ||w o r|| / ||w o r_0|| <
// tol.  The history keeps the per-step estimates.  wstop = 0: the estimate stops (B1/B2).
int orc_gmres_wstop(int64_t n, const int32_t* rp, const int32_t* ci, const double* v,
                    const double* b, const double* x0, const double* w, int m, double tol, int maxit,
                    int orth, int wstop, double* x, double* hist, orc_report* rep) {
  if (orth != 0 && orth != 1) return -1;
  if (n < 1 || maxit < 1 || m < 1 || !(tol > 0)) return -1;
  std::vector<double> r(n), ax(n), wv(n);
  std::vector<std::vector<double>> V(m + 1, std::vector<double>(n));
  std::vector<double> Hm((size_t)(m + 1) * m, 0.0), cs(m), sn(m), g(m + 1), y(m);
  auto h = [&](int i, int j) -> double& { return Hm[(size_t)i * m + j]; };  // 0-based
  for (int64_t i = 0; i < n; ++i) x[i] = x0 ? x0[i] : 0.0;
  orc_spmv(n, rp, ci, v, x, ax.data());
  for (int64_t i = 0; i < n; ++i) r[i] = b[i] - ax[i];
  const double beta0 = std::sqrt(orc_dot(n, r.data(), r.data()));
  const double n0w = std::sqrt(orc_wnorm2(n, r.data(), w));
  std::memset(rep, 0, sizeof(*rep));
  std::vector<double> H;
  H.push_back(beta0 == 0.0 ? 0.0 : 1.0);
  int status = 1, it = 0, restarts = 0;
  if (beta0 == 0.0) status = 0;
  bool done = (beta0 == 0.0);
  while (!done) {
    double beta = std::sqrt(orc_dot(n, r.data(), r.data()));
    double inv = 1.0 / beta;
    for (int64_t i = 0; i < n; ++i) V[0][i] = r[i] * inv;
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    int k = 0;
    bool stop_conv = false, stop_div = false;
    for (int j = 0; j < m; ++j) {  // Arnoldi step j+1
      ++it;
      orc_spmv(n, rp, ci, v, V[j].data(), wv.data());
      if (orth == 0) {
        for (int i = 0; i <= j; ++i) {  // modified Gram-Schmidt
          h(i, j) = orc_dot(n, wv.data(), V[i].data());
          for (int64_t q = 0; q < n; ++q) wv[q] = std::fma(-h(i, j), V[i][q], wv[q]);
        }
      } else {
        std::vector<double> c1(j + 1), c2(j + 1);
        for (int i = 0; i <= j; ++i) c1[i] = orc_dot(n, wv.data(), V[i].data());
        for (int64_t q = 0; q < n; ++q)
          for (int i = 0; i <= j; ++i) wv[q] = std::fma(-c1[i], V[i][q], wv[q]);
        for (int i = 0; i <= j; ++i) c2[i] = orc_dot(n, wv.data(), V[i].data());
        for (int64_t q = 0; q < n; ++q)
          for (int i = 0; i <= j; ++i) wv[q] = std::fma(-c2[i], V[i][q], wv[q]);
        for (int i = 0; i <= j; ++i) h(i, j) = c1[i] + c2[i];
      }
      double hn = std::sqrt(orc_dot(n, wv.data(), wv.data()));
      h(j + 1, j) = hn;
      for (int i = 0; i < j; ++i) {  // previous rotations on column j
        double a = h(i, j), bb = h(i + 1, j);
        h(i, j) = std::fma(cs[i], a, sn[i] * bb);
        h(i + 1, j) = std::fma(-sn[i], a, cs[i] * bb);
      }
      double a = h(j, j), bb = h(j + 1, j);
      double delta = std::sqrt(std::fma(a, a, bb * bb));
      cs[j] = a / delta;
      sn[j] = bb / delta;
      h(j, j) = delta;
      h(j + 1, j) = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      double rel = std::fabs(g[j + 1]) / beta0;
      H.push_back(rel);
      k = j + 1;
      if (!std::isfinite(rel)) { stop_div = true; break; }
      if (rel < tol && !wstop) { stop_conv = true; break; }
      if (hn == 0.0 || it == maxit) break;
      double invh = 1.0 / hn;
      for (int64_t q = 0; q < n; ++q) V[j + 1][q] = wv[q] * invh;
    }
    if (stop_div) { status = 3; break; }
    // column-oriented back substitution R y = g (R = upper k x k of H)
    std::vector<double> acc(g.begin(), g.begin() + k);
    for (int kk = k - 1; kk >= 0; --kk) {
      y[kk] = acc[kk] / h(kk, kk);
      for (int l = 0; l < kk; ++l) acc[l] = std::fma(-h(l, kk), y[kk], acc[l]);
    }
    for (int kk = 0; kk < k; ++kk)
      for (int64_t q = 0; q < n; ++q) x[q] = std::fma(y[kk], V[kk][q], x[q]);
    orc_spmv(n, rp, ci, v, x, ax.data());
    for (int64_t i = 0; i < n; ++i) r[i] = b[i] - ax[i];
    bool fin = true;
    for (int kk = 0; kk < k; ++kk) fin = fin && std::isfinite(y[kk]);
    if (!fin) { status = 3; break; }
    if (wstop) {  // the weighted true residual of the cycle's end
      const double twc = std::sqrt(orc_wnorm2(n, r.data(), w));
      const double relw = n0w == 0.0 ? 0.0 : twc / n0w;
      if (!std::isfinite(relw)) { status = 3; break; }
      if (relw < tol) stop_conv = true;
    }
    if (stop_conv) { status = 0; break; }
    if (it >= maxit) { status = 1; break; }
    ++restarts;
  }
  double tn = std::sqrt(orc_dot(n, r.data(), r.data()));
  double tw = std::sqrt(orc_wnorm2(n, r.data(), w));
  rep->status = status;
  rep->iterations = it;
  rep->restarts = restarts;
  rep->history_len = (int32_t)H.size();
  rep->breakdown_at = 0;
  rep->relres = H.back();
  rep->true_relres = beta0 == 0.0 ? 0.0 : tn / beta0;
  rep->true_relres_w = n0w == 0.0 ? 0.0 : tw / n0w;
  rep->best_relres = *std::min_element(H.begin(), H.end());
  if (hist) std::memcpy(hist, H.data(), sizeof(double) * H.size());
  return 0;
}

}  // extern "C"
