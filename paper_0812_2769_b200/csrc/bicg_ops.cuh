// bicg_ops.cuh — the Bi-CGSTAB pass operators (row epilogues + scalar epilogues),
// shared by the graph-replayed passes (bicgstab.cu) and the cooperative small-system
// kernel (coop.cu).  Arithmetic: AC-6.
#pragma once
#include "internal.cuh"

namespace gsk {

// Every op names its own-row operands (vin(k); the engine stages them through
// shared memory with TMA and hands the values to row() as v[k]).
template <class L = LdNC>
struct OpInit {  // r = b - A x; r^ = r; p_old = v_old = 0
  static constexpr int D = 2;
  static constexpr int NV = 2;
  static constexpr bool kSpmv = true;
  const double* x;
  const double* b;
  const double* w;
  double *r, *rh, *pa, *va, *hist;
  BicgState* st;
  __device__ bool begin() { return true; }
  __device__ const double* vin(int k) const { return k == 0 ? b : w; }
  __device__ double gather(int c) const { return L::ld(x + c); }
  __device__ void row(int i, double y, const double (&v)[NV], double (&c)[2]) const {
    const double ri = v[0] - y;
    r[i] = ri;
    rh[i] = ri;
    pa[i] = 0.0;
    va[i] = 0.0;
    const double u = w ? v[1] * ri : ri;
    c[0] = u * u;
    c[1] = ri * ri;
  }
  __device__ void finish(const double (&s)[2], int lane) const {
    if (lane) return;
    const double n0 = sqrt(s[0]);
    st->n0 = n0;
    st->n0u = sqrt(s[1]);
    hist[0] = n0 == 0.0 ? 0.0 : 1.0;
    st->hist_len = 1;
    st->iter = 1;
    st->rho_prev = 1.0;
    st->alpha = 1.0;
    st->omega = 1.0;
    st->status = GSK_MAXIT;
    st->bd = 0;
    st->halfstep = 0;
    st->done = 0;
    if (n0 == 0.0) {
      st->status = GSK_CONVERGED;
      st->done = 1;
      return;
    }
    const double rho = s[1];  // <r^, r> = <r, r>: the same leaves in the same tree
    st->rho = rho;
    if (rho == 0.0) {
      st->status = GSK_BREAKDOWN;
      st->bd = 1;
      st->done = 1;
      return;
    }
    st->beta = (rho / st->rho_prev) * (st->alpha / st->omega);
  }
};

// ---- fused schedule (3 passes; p and s recomputed at the gather) ---------------------
template <class L = LdNC>
struct OpP1 {
  static constexpr int kSellMinBlocks = 3;  // see SellTuning (engine.cuh)
  static constexpr int D = 1;
  static constexpr int NV = 4;
  static constexpr bool kSpmv = true;
  const double *r, *po, *vo, *rh;
  double *pn, *vn;
  BicgState* st;
  double beta, momega;
  __device__ bool begin() {
    if (st->done) return false;
    beta = st->beta;
    momega = -st->omega;
    return true;
  }
  __device__ const double* vin(int k) const { return k == 0 ? vo : k == 1 ? po : k == 2 ? r : rh; }
  __device__ double gather(int c) const {
    return __fma_rn(beta, __fma_rn(momega, L::ld(vo + c), L::ld(po + c)), L::ld(r + c));
  }
  __device__ void row(int i, double y, const double (&v)[NV], double (&c)[1]) const {
    pn[i] = __fma_rn(beta, __fma_rn(momega, v[0], v[1]), v[2]);
    vn[i] = y;
    c[0] = v[3] * y;
  }
  __device__ void finish(const double (&s)[1], int lane) const {
    if (lane) return;
    const double sigma = s[0];
    if (sigma == 0.0) {
      st->status = GSK_BREAKDOWN;
      st->bd = st->iter;
      st->done = 1;
      return;
    }
    st->alpha = st->rho / sigma;
  }
};

// half-step exit test shared by both schedules: ||s||_w / ||r0||_w < tol
__device__ __forceinline__ bool halfstep_exit(BicgState* st, double* hist, double ss) {
  const int i = st->iter;
  const double sn = sqrt(ss) / st->n0;
  if (sn < st->tol) {  // reading B4: x += alpha p in the update pass
    hist[i] = sn;
    st->hist_len = i + 1;
    st->status = GSK_CONVERGED;
    st->halfstep = 1;
    st->done = 1;
    return true;
  }
  return false;
}

__device__ __forceinline__ void set_omega(BicgState* st, double ts, double tt) {
  if (tt == 0.0) {
    st->status = GSK_BREAKDOWN;
    st->bd = st->iter;
    st->done = 1;
    return;
  }
  st->omega = (st->fault_kind == GSK_FAULT_OMEGA0 && st->fault_it == st->iter) ? 0.0 : ts / tt;
}

template <class L = LdNC>
struct OpP2 {
  static constexpr int kSellMinBlocks = 3;  // see SellTuning (engine.cuh)
  static constexpr int D = 3;
  static constexpr int NV = 3;
  static constexpr bool kSpmv = true;
  const double *r, *vn, *w;
  double *t, *hist;
  BicgState* st;
  double malpha;
  __device__ bool begin() {
    if (st->done) return false;
    malpha = -st->alpha;
    return true;
  }
  __device__ const double* vin(int k) const { return k == 0 ? vn : k == 1 ? r : w; }
  __device__ double gather(int c) const { return __fma_rn(malpha, L::ld(vn + c), L::ld(r + c)); }
  __device__ void row(int i, double y, const double (&v)[NV], double (&c)[3]) const {
    const double s = __fma_rn(malpha, v[0], v[1]);
    t[i] = y;
    c[0] = y * s;
    c[1] = y * y;
    const double u = w ? v[2] * s : s;
    c[2] = u * u;
  }
  __device__ void finish(const double (&s)[3], int lane) const {
    if (lane) return;
    if (halfstep_exit(st, hist, s[2])) return;
    set_omega(st, s[0], s[1]);
  }
};

// x, r update + <r^, r>, ||r||_w^2 -> history, stopping and breakdown tests
__device__ __forceinline__ void update_finish(BicgState* st, double* hist, int half, double alpha,
                                              double omega, const double (&s)[2]) {
  if (half) {
    st->halfstep = 0;
    return;
  }
  const int i = st->iter;
  const double rho_prev = st->rho;
  st->rho_prev = rho_prev;
  const double rn = sqrt(s[1]) / st->n0;
  hist[i] = rn;
  st->hist_len = i + 1;
  if (!isfinite(rn)) {
    st->status = GSK_DIVERGED;
    st->done = 1;
  } else if (rn < st->tol) {
    st->status = GSK_CONVERGED;
    st->done = 1;
  } else if (omega == 0.0) {
    st->status = GSK_BREAKDOWN;
    st->bd = i;
    st->done = 1;
  } else if (i == st->maxit) {
    st->status = GSK_MAXIT;
    st->done = 1;
  } else {
    const double rho = (st->fault_kind == GSK_FAULT_RHO0 && st->fault_it == i) ? 0.0 : s[0];
    st->rho = rho;
    if (rho == 0.0) {
      st->status = GSK_BREAKDOWN;
      st->bd = i + 1;
      st->done = 1;
    } else {
      st->beta = (rho / rho_prev) * (alpha / omega);
      st->iter = i + 1;
    }
  }
}

struct OpP3 {
  static constexpr int D = 2;
  static constexpr int NV = 7;
  static constexpr bool kSpmv = false;
  const double *vn, *pn, *t, *rh, *w;
  double *x, *r, *hist;
  BicgState* st;
  double alpha, omega;
  int half, nan0;
  __device__ bool begin() {
    half = st->halfstep;
    if (st->done && !half) return false;
    alpha = st->alpha;
    omega = st->omega;
    nan0 = st->fault_kind == GSK_FAULT_NAN && st->fault_it == st->iter;
    return true;
  }
  __device__ const double* vin(int k) const {
    return k == 0 ? x : k == 1 ? pn : k == 2 ? (half ? nullptr : vn) : k == 3 ? (half ? nullptr : r)
         : k == 4 ? (half ? nullptr : t) : k == 5 ? (half ? nullptr : rh) : (half ? nullptr : w);
  }
  __device__ double gather(int) const { return 0.0; }
  __device__ void row(int i, double, const double (&v)[NV], double (&c)[2]) const {
    if (half) {
      st_cold(x + i, __fma_rn(alpha, v[1], v[0]));
      c[0] = 0.0;
      c[1] = 0.0;
      return;
    }
    const double s = __fma_rn(-alpha, v[2], v[3]);
    st_cold(x + i, __fma_rn(omega, s, __fma_rn(alpha, v[1], v[0])));
    const double rr = (nan0 && i == 0) ? __longlong_as_double(0x7ff8000000000000ll) : __fma_rn(-omega, v[4], s);
    r[i] = rr;
    c[0] = v[5] * rr;
    const double u = w ? v[6] * rr : rr;
    c[1] = u * u;
  }
  __device__ void finish(const double (&s)[2], int lane) const {
    if (lane == 0) update_finish(st, hist, half, alpha, omega, s);
  }
};

// ---- split schedule (5 passes, plain SpMV gathers) -------------------
// S0  p = r + beta (p - omega v)                       (vector pass)
// S1  v = A p, sigma = <r^, v>                          -> alpha
// S2  s = r - alpha v, ||s||_w^2                        -> half-step exit
// S3  t = A s, <t,s>, <t,t>                             -> omega
// S4  x += alpha p + omega s, r = s - omega t, <r^,r>, ||r||_w^2
struct OpS0 {
  static constexpr int D = 0;
  static constexpr int NV = 3;
  static constexpr unsigned kEvict = 0b101u;  // S1 reads p only: v, r evict-first
  static constexpr bool kSpmv = false;
  const double *r, *v;
  double* p;
  BicgState* st;
  double beta, momega;
  __device__ bool begin() {
    if (st->done) return false;
    beta = st->beta;
    momega = -st->omega;
    return true;
  }
  __device__ const double* vin(int k) const { return k == 0 ? v : k == 1 ? p : r; }
  __device__ double gather(int) const { return 0.0; }
  __device__ void row(int i, double, const double (&x)[NV], double (&)[1]) const {
    p[i] = __fma_rn(beta, __fma_rn(momega, x[0], x[1]), x[2]);
  }
};

template <class L = LdNC>
struct OpS1 {
  static constexpr int D = 1;
  static constexpr int NV = 1;
  static constexpr unsigned kEvict = 0b1u;  // S2 does not read r^
  static constexpr bool kSpmv = true;
  const double *p, *rh;
  double* v;
  BicgState* st;
  __device__ bool begin() { return !st->done; }
  __device__ const double* vin(int) const { return rh; }
  __device__ const double* gathered() const { return p; }  // the one vector gather() reads
  __device__ double gather(int c) const { return L::ld(p + c); }
  __device__ void row(int i, double y, const double (&x)[NV], double (&c)[1]) const {
    v[i] = y;
    c[0] = x[0] * y;
  }
  __device__ void finish(const double (&s)[1], int lane) const {
    if (lane) return;
    const double sigma = s[0];
    if (sigma == 0.0) {
      st->status = GSK_BREAKDOWN;
      st->bd = st->iter;
      st->done = 1;
      return;
    }
    st->alpha = st->rho / sigma;
  }
};

// ---- four-pass schedule (bicg_schedule 3): S0 folded into its neighbours ------------
// S4q = S4 + q = p - omega v stored over p (own rows, in place); S1q gathers q and r and
// forms p = r + beta q at every gathered column (the same two FMAs as S0, in the same
// order: AC-6), writes p for its own rows into the other p buffer, then v = A p and
// <r^, v>.  Same bytes per iteration as the split schedule, one kernel fewer, a second
// gather stream in the SpMV pass.
template <class L = LdNC>
struct OpS1q {
  static constexpr int D = 1;
  static constexpr int NV = 3;
  static constexpr bool kSpmv = true;
  const double *q, *r, *rh;
  double *p, *v;
  BicgState* st;
  double beta;
  __device__ bool begin() {
    if (st->done) return false;
    beta = st->beta;
    return true;
  }
  __device__ const double* vin(int k) const { return k == 0 ? rh : k == 1 ? q : r; }
  __device__ double gather(int c) const { return __fma_rn(beta, L::ld(q + c), L::ld(r + c)); }
  __device__ void row(int i, double y, const double (&x)[NV], double (&c)[1]) const {
    p[i] = __fma_rn(beta, x[1], x[2]);
    v[i] = y;
    c[0] = x[0] * y;
  }
  __device__ void finish(const double (&s)[1], int lane) const {
    if (lane) return;
    const double sigma = s[0];
    if (sigma == 0.0) {
      st->status = GSK_BREAKDOWN;
      st->bd = st->iter;
      st->done = 1;
      return;
    }
    st->alpha = st->rho / sigma;
  }
};

struct OpS2 {
  static constexpr int D = 1;
  static constexpr int NV = 3;
  static constexpr unsigned kEvict = 0b111u;  // S3 reads only s
  static constexpr bool kSpmv = false;
  const double *r, *v, *w;
  double *s_, *hist;
  BicgState* st;
  double malpha;
  __device__ bool begin() {
    if (st->done) return false;
    malpha = -st->alpha;
    return true;
  }
  __device__ const double* vin(int k) const { return k == 0 ? v : k == 1 ? r : w; }
  __device__ double gather(int) const { return 0.0; }
  __device__ void row(int i, double, const double (&x)[NV], double (&c)[1]) const {
    const double s = __fma_rn(malpha, x[0], x[1]);
    s_[i] = s;
    const double u = w ? x[2] * s : s;
    c[0] = u * u;
  }
  __device__ void finish(const double (&s)[1], int lane) const {
    if (lane == 0) halfstep_exit(st, hist, s[0]);
  }
};

template <class L = LdNC>
struct OpS3 {
  static constexpr int D = 2;
  static constexpr int NV = 1;
  static constexpr bool kSpmv = true;
  const double* s_;
  double* t;
  BicgState* st;
  __device__ bool begin() { return !st->done; }
  __device__ const double* vin(int) const { return s_; }
  __device__ const double* gathered() const { return s_; }  // the one vector gather() reads
  __device__ double gather(int c) const { return L::ld(s_ + c); }
  __device__ void row(int i, double y, const double (&x)[NV], double (&c)[2]) const {
    t[i] = y;
    c[0] = y * x[0];
    c[1] = y * y;
  }
  __device__ void finish(const double (&s)[2], int lane) const {
    if (lane == 0) set_omega(st, s[0], s[1]);
  }
};

struct OpS4 {
  static constexpr int D = 2;
  static constexpr int NV = 6;
  static constexpr unsigned kEvict = 0b111101u;  // S0 reads r, p, v: only p kept
  static constexpr bool kSpmv = false;
  const double *s_, *p, *t, *rh, *w;
  double *x, *r, *hist;
  BicgState* st;
  double alpha, omega;
  int half, nan0;
  __device__ bool begin() {
    half = st->halfstep;
    if (st->done && !half) return false;
    alpha = st->alpha;
    omega = st->omega;
    nan0 = st->fault_kind == GSK_FAULT_NAN && st->fault_it == st->iter;
    return true;
  }
  __device__ const double* vin(int k) const {
    return k == 0 ? x : k == 1 ? p : k == 2 ? (half ? nullptr : s_) : k == 3 ? (half ? nullptr : t)
         : k == 4 ? (half ? nullptr : rh) : (half ? nullptr : w);
  }
  __device__ double gather(int) const { return 0.0; }
  __device__ void row(int i, double, const double (&v)[NV], double (&c)[2]) const {
    if (half) {
      st_cold(x + i, __fma_rn(alpha, v[1], v[0]));
      c[0] = 0.0;
      c[1] = 0.0;
      return;
    }
    const double s = v[2];
    st_cold(x + i, __fma_rn(omega, s, __fma_rn(alpha, v[1], v[0])));
    const double rr = (nan0 && i == 0) ? __longlong_as_double(0x7ff8000000000000ll) : __fma_rn(-omega, v[3], s);
    r[i] = rr;
    c[0] = v[4] * rr;
    const double u = w ? v[5] * rr : rr;
    c[1] = u * u;
  }
  __device__ void finish(const double (&s)[2], int lane) const {
    if (lane == 0) update_finish(st, hist, half, alpha, omega, s);
  }
};

// S4 of the four-pass schedule: also q = p - omega v over p (the next S1q's gather)
struct OpS4q {
  static constexpr int D = 2;
  static constexpr int NV = 7;
  static constexpr bool kSpmv = false;
  const double *s_, *t, *rh, *w, *v;
  double *p, *x, *r, *hist;
  BicgState* st;
  double alpha, omega;
  int half, nan0;
  __device__ bool begin() {
    half = st->halfstep;
    if (st->done && !half) return false;
    alpha = st->alpha;
    omega = st->omega;
    nan0 = st->fault_kind == GSK_FAULT_NAN && st->fault_it == st->iter;
    return true;
  }
  __device__ const double* vin(int k) const {
    return k == 0 ? x : k == 1 ? p : k == 2 ? (half ? nullptr : s_) : k == 3 ? (half ? nullptr : t)
         : k == 4 ? (half ? nullptr : rh) : k == 5 ? (half ? nullptr : w) : (half ? nullptr : v);
  }
  __device__ double gather(int) const { return 0.0; }
  __device__ void row(int i, double, const double (&u)[NV], double (&c)[2]) const {
    if (half) {
      st_cold(x + i, __fma_rn(alpha, u[1], u[0]));
      c[0] = 0.0;
      c[1] = 0.0;
      return;
    }
    const double s = u[2];
    st_cold(x + i, __fma_rn(omega, s, __fma_rn(alpha, u[1], u[0])));
    const double rr = (nan0 && i == 0) ? __longlong_as_double(0x7ff8000000000000ll) : __fma_rn(-omega, u[3], s);
    r[i] = rr;
    p[i] = __fma_rn(-omega, u[6], u[1]);  // q for the next S1q (p is not read again)
    c[0] = u[4] * rr;
    const double uw = w ? u[5] * rr : rr;
    c[1] = uw * uw;
  }
  __device__ void finish(const double (&s)[2], int lane) const {
    if (lane == 0) update_finish(st, hist, half, alpha, omega, s);
  }
};

template <class L = LdNC>
struct OpFinal {  // true residual ||b - A x|| (unweighted and weighted)
  static constexpr int D = 2;
  static constexpr int NV = 2;
  static constexpr bool kSpmv = true;
  const double *x, *b, *w;
  BicgState* st;
  __device__ bool begin() { return true; }
  __device__ const double* vin(int k) const { return k == 0 ? b : w; }
  __device__ double gather(int c) const { return L::ld(x + c); }
  __device__ void row(int i, double y, const double (&v)[NV], double (&c)[2]) const {
    const double ri = v[0] - y;
    c[0] = ri * ri;
    const double u = w ? v[1] * ri : ri;
    c[1] = u * u;
  }
  __device__ void finish(const double (&s)[2], int lane) const {
    if (lane) return;
    st->true_rel = st->n0u == 0.0 ? 0.0 : sqrt(s[0]) / st->n0u;
    st->true_rel_w = st->n0 == 0.0 ? 0.0 : sqrt(s[1]) / st->n0;
  }
};

}  // namespace gsk
