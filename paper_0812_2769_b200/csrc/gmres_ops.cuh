// gmres_ops.cuh — the GMRES(m) pass operators (row epilogues + scalar epilogues) and
// the single-warp Givens / back-substitution step, shared by the graph-replayed
// passes (gmres.cu) and the on-chip single-CTA solver (small.cu).  Arithmetic:
// AC-7.
#pragma once
#include "internal.cuh"

namespace gsk {

constexpr int MAX_M = 128;

// r = b - A x stored as basis slot 1; ||r||^2 and ||w o r||^2.
template <class L = LdNC>
struct OpGResid {
  static constexpr int D = 2;
  static constexpr int NV = 2;
  static constexpr bool kSpmv = true;
  const double *x, *b, *w;
  double* W1;
  double* hist;
  GmresState* st;
  int init;
  __device__ bool begin() { return !st->done; }
  __device__ const double* vin(int k) const { return k == 0 ? b : w; }
  __device__ double gather(int c) const { return L::ld(x + c); }
  __device__ void row(int i, double y, const double (&v)[NV], double (&c)[2]) const {
    const double ri = v[0] - y;
    W1[i] = ri;
    c[0] = ri * ri;
    const double u = w ? v[1] * ri : ri;
    c[1] = u * u;
  }
  __device__ void finish(const double (&s)[2], int lane) const {
    if (lane) return;
    const double beta = sqrt(s[0]);
    if (init) {
      st->beta0 = beta;
      st->n0w = sqrt(s[1]);
      hist[0] = beta == 0.0 ? 0.0 : 1.0;
      st->hist_len = 1;
      st->it = 0;
      st->restarts = 0;
      if (beta == 0.0) {
        st->status = GSK_CONVERGED;
        st->true_rel = 0.0;
        st->true_rel_w = 0.0;
        st->done = 1;
        return;
      }
    } else if (st->final_) {
      const double relw = st->n0w == 0.0 ? 0.0 : sqrt(s[1]) / st->n0w;
      int conv = st->conv, div = st->diverged;
      if (st->wstop && !div) {  // reading B2w: the weighted true residual decides
        div = !isfinite(relw);
        conv = relw < st->tol;
      }
      st->status = div ? GSK_DIVERGED : (conv ? GSK_CONVERGED : GSK_MAXIT);
      st->true_rel = beta / st->beta0;
      st->true_rel_w = relw;
      st->done = 1;
      return;
    } else {
      if (st->wstop) {  // a cycle's end: CONVERGED when ||w o r|| / ||w o r_0|| < tol (B2w)
        const double relw = st->n0w == 0.0 ? 0.0 : sqrt(s[1]) / st->n0w;
        if (!isfinite(relw) || relw < st->tol) {
          st->status = isfinite(relw) ? GSK_CONVERGED : GSK_DIVERGED;
          st->true_rel = beta / st->beta0;
          st->true_rel_w = relw;
          st->done = 1;
          return;
        }
      }
      st->restarts += 1;
    }
    st->inv[1] = 1.0 / beta;
    st->g[0] = beta;
    for (int q = 1; q <= st->m; ++q) st->g[q] = 0.0;
    st->k = 0;
    st->cycle_stop = 0;
  }
};

// S_j: w = A v_j into slot j+1; h_1j = <w, v_1>
template <class L = LdNC>
struct OpArnoldi {
  static constexpr int kSellMinBlocks = 3;  // see SellTuning (engine.cuh)
  static constexpr int D = 1;
  static constexpr int NV = 1;
  static constexpr bool kSpmv = true;
  const double *Wj, *W1;
  double* Wn;
  GmresState* st;
  int j;
  double invj, inv1;
  __device__ bool begin() {
    if (st->done || st->cycle_stop) return false;
    invj = st->inv[j];
    inv1 = st->inv[1];
    return true;
  }
  __device__ const double* vin(int) const { return W1; }
  __device__ double gather(int c) const { return L::ld(Wj + c) * invj; }
  __device__ void row(int i, double y, const double (&v)[NV], double (&c)[1]) const {
    Wn[i] = y;
    c[0] = y * (v[0] * inv1);
  }
  __device__ void finish(const double (&s)[1], int lane) const {
    if (lane == 0) st->H[0 * st->m + (j - 1)] = s[0];
  }
};

// h_1j = <w, v_1> as its own vector pass after a plain SpMV pass w = A v_j (OpCgsS):
// the same leaves w_i * RN(w1_i * inv_1) in the same canonical tree as OpArnoldi, but
// the SpMV runs at plain-SpMV speed (0.28 vs 0.36 ms at C4) and the dot streams two
// vectors.
struct OpH1 {
  static constexpr int D = 1;
  static constexpr int NV = 2;
  static constexpr bool kSpmv = false;
  const double *Wn, *W1;
  GmresState* st;
  int j;
  double inv1;
  __device__ bool begin() {
    if (st->done || st->cycle_stop) return false;
    inv1 = st->inv[1];
    return true;
  }
  __device__ const double* vin(int k) const { return k == 0 ? Wn : W1; }
  __device__ double gather(int) const { return 0.0; }
  __device__ void row(int, double, const double (&v)[NV], double (&c)[1]) const { c[0] = v[0] * (v[1] * inv1); }
  __device__ void finish(const double (&s)[1], int lane) const {
    if (lane == 0) st->H[0 * st->m + (j - 1)] = s[0];
  }
};

// M_{i,j}: w -= h_ij v_i; h_{i+1,j} = <w, v_{i+1}>
struct OpMgs {
  static constexpr int D = 1;
  static constexpr int NV = 3;
  static constexpr unsigned kEvict = 0b001u;  // the next pass reads w and v_{i+1}, not v_i
  static constexpr bool kSpmv = false;
  const double *Wi, *Wi1;
  double* Wn;
  GmresState* st;
  int i, j;
  double mh, invi, invi1;
  __device__ bool begin() {
    if (st->done || st->cycle_stop) return false;
    mh = -st->H[(i - 1) * st->m + (j - 1)];
    invi = st->inv[i];
    invi1 = st->inv[i + 1];
    return true;
  }
  __device__ const double* vin(int k) const { return k == 0 ? Wi : k == 1 ? Wn : Wi1; }
  __device__ double gather(int) const { return 0.0; }
  __device__ void row(int q, double, const double (&v)[NV], double (&c)[1]) const {
    const double w = __fma_rn(mh, v[0] * invi, v[1]);
    Wn[q] = w;
    c[0] = w * (v[2] * invi1);
  }
  __device__ void finish(const double (&s)[1], int lane) const {
    if (lane == 0) st->H[i * st->m + (j - 1)] = s[0];
  }
};

// End of Arnoldi step j (1-based; warp 0 of the finishing CTA): h_{j+1,j} = sqrt(hn2),
// the previous Givens rotations on column j, the new rotation, g, the history entry,
// the stopping tests and, when the cycle ends, the column-oriented
// back substitution R y = g in one warp (AC-7).
static __device__ void arnoldi_finish(GmresState* S, double* hist, int j, double hn2, int lane, int cgs2) {
  const int m = S->m, col = j - 1;
  double* H = S->H;
  __shared__ int need_bs;
  if (lane == 0) {
    const double hn = sqrt(hn2);
    if (cgs2)  // H(:, j) = h + h' of the two classical projections
      for (int i = 0; i < j; ++i) H[i * m + col] = S->c1[i] + S->c2[i];
    H[j * m + col] = hn;
    for (int i = 0; i < col; ++i) {  // previous rotations on column j
      const double a = H[i * m + col], b = H[(i + 1) * m + col];
      H[i * m + col] = __fma_rn(S->cs[i], a, S->sn[i] * b);
      H[(i + 1) * m + col] = __fma_rn(-S->sn[i], a, S->cs[i] * b);
    }
    const double a = H[col * m + col], b = H[j * m + col];
    const double delta = sqrt(__fma_rn(a, a, b * b));
    const double cj = a / delta, sj = b / delta;
    S->cs[col] = cj;
    S->sn[col] = sj;
    H[col * m + col] = delta;
    H[j * m + col] = 0.0;
    const double gj = S->g[col];
    S->g[col + 1] = -sj * gj;
    S->g[col] = cj * gj;
    const double rel = fabs(S->g[col + 1]) / S->beta0;
    const int it = S->it + 1;
    S->it = it;
    hist[it] = rel;
    S->hist_len = it + 1;
    S->k = j;
    int stop = 0;
    if (!isfinite(rel)) {
      S->diverged = 1;
      S->skip_x = 1;
      S->final_ = 1;
      stop = 1;
    } else if (rel < S->tol && !S->wstop) {  // (wstop: the estimate does not stop the run)
      S->conv = 1;
      S->final_ = 1;
      stop = 1;
    } else if (hn == 0.0 || it == S->maxit) {
      if (it == S->maxit) S->final_ = 1;
      stop = 1;
    } else {
      S->inv[j + 1] = 1.0 / hn;
    }
    S->cycle_stop = stop;
    need_bs = (stop && !S->skip_x) || (j == m);
  }
  __syncwarp();
  if (need_bs) {
    // column-oriented back substitution R y = g (AC-7), lanes own rows
    const int k = j;
    double acc[MAX_M / 32];
#pragma unroll
    for (int q = 0; q < MAX_M / 32; ++q) {
      const int l = lane + 32 * q;
      acc[q] = l < k ? S->g[l] : 0.0;
    }
    bool fin = true;
    for (int kk = k - 1; kk >= 0; --kk) {
      const int owner = kk & 31, qo = kk >> 5;
      double mine = 0.0;
#pragma unroll
      for (int q = 0; q < MAX_M / 32; ++q)
        if (q == qo) mine = acc[q];
      const double ykk = __shfl_sync(0xffffffffu, mine, owner) / H[kk * m + kk];
      fin = fin && isfinite(ykk);
      if (lane == 0) S->y[kk] = ykk;
#pragma unroll
      for (int q = 0; q < MAX_M / 32; ++q) {
        const int l = lane + 32 * q;
        if (l < kk) acc[q] = __fma_rn(-H[l * m + kk], ykk, acc[q]);
      }
    }
    if (lane == 0 && !fin) {
      S->diverged = 1;
      S->final_ = 1;
    }
  }
}

// L_j: w -= h_jj v_j; ||w||^2 -> Givens update, history, stopping, back-solve.
struct OpLast {
  static constexpr int D = 1;
  static constexpr int NV = 2;
  static constexpr unsigned kEvict = 0b01u;  // S_{j+1} gathers w only
  static constexpr bool kSpmv = false;
  const double* Wj;
  double* Wn;
  double* hist;
  GmresState* st;
  int j;
  double mh, invj;
  __device__ bool begin() {
    if (st->done || st->cycle_stop) return false;
    mh = -st->H[(j - 1) * st->m + (j - 1)];
    invj = st->inv[j];
    return true;
  }
  __device__ const double* vin(int k) const { return k == 0 ? Wj : Wn; }
  __device__ double gather(int) const { return 0.0; }
  __device__ void row(int q, double, const double (&v)[NV], double (&c)[1]) const {
    const double w = __fma_rn(mh, v[0] * invj, v[1]);
    Wn[q] = w;
    c[0] = w * w;
  }
  __device__ void finish(const double (&s)[1], int lane) const { arnoldi_finish(st, hist, j, s[0], lane, 0); }
};

// ---- double classical Gram-Schmidt (AZTEC's orthogonalisation) ----
// Step j = four passes: S  w = A v_j (SpMV pass);  A  c1_d = <w, v_d>;
// B  w -= sum_d c1_d v_d, c2_d = <w, v_d>;  C  w -= sum_d c2_d v_d, ||w||^2 ->
// H(:, j) = c1 + c2, Givens.  A, B, C are tile passes (mdot_pass: 8 consecutive rows
// per thread, 16-byte loads).  Each update is an FMA chain over d ascending (oracle
// orc_gmres_orth, orth = 1); v_d = RN(w_d * inv_d) as everywhere (AC-7).
#ifndef GSK_CGS_UNROLL
#define GSK_CGS_UNROLL 1
#endif
constexpr int kCgsUnroll = GSK_CGS_UNROLL;
struct CgsBase {
  const double* W;
  size_t n;
  double* Wn;
  GmresState* st;
  int j;
  int nd;
  const double* inv;
  __device__ bool live() const { return !(st->done || st->cycle_stop); }
  __device__ void basis8(int i0, int cnt, int d, double (&v)[8]) const {
    ld8(W + d * n + i0, cnt, v);
    const double s = inv[d + 1];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = v[k] * s;
  }
  // w -= sum_d c_d v_d over d < j (8 rows' chains interleaved); returns w (0 past cnt)
  __device__ void update8(int i0, int cnt, const double* c, double (&u)[8]) const {
    double w[8];
    ld8(Wn + i0, cnt, w);
#pragma unroll kCgsUnroll
    for (int d = 0; d < j; ++d) {
      double v[8];
      basis8(i0, cnt, d, v);
      const double mc = -c[d];
#pragma unroll
      for (int k = 0; k < 8; ++k) w[k] = __fma_rn(mc, v[k], w[k]);
    }
    st8(Wn + i0, cnt, w);
#pragma unroll
    for (int k = 0; k < 8; ++k) u[k] = k < cnt ? w[k] : 0.0;
  }
};

template <class L = LdNC>
struct OpCgsS {  // S: w = A v_j (no reduction)
  static constexpr int D = 0;
  static constexpr int NV = 0;
  static constexpr bool kSpmv = true;
  const double* Wj;
  double* Wn;
  GmresState* st;
  int j;
  double invj;
  __device__ bool begin() {
    if (st->done || st->cycle_stop) return false;
    invj = st->inv[j];
    return true;
  }
  __device__ const double* vin(int) const { return nullptr; }
  __device__ const double* gathered() const { return Wj; }  // gather(c) = gxform(Wj[c])
  __device__ double gxform(double v) const { return v * invj; }
  __device__ double gather(int c) const { return gxform(L::ld(Wj + c)); }
  __device__ void row(int i, double y, const double (&)[1], double (&)[1]) const { Wn[i] = y; }
};

struct OpCgsA : CgsBase {  // A: c1 = V^T w
  static constexpr bool kSpmv = false;
  __device__ bool begin() {
    if (!live()) return false;
    inv = st->inv;
    nd = j;
    return true;
  }
  __device__ double gather(int) const { return 0.0; }
  __device__ void value8(int i0, int cnt, const double (&)[8], double (&u)[8]) const {
    ld8(Wn + i0, cnt, u);
#pragma unroll
    for (int k = 0; k < 8; ++k) u[k] = k < cnt ? u[k] : 0.0;
  }
  __device__ void operand8(int i0, int cnt, int d, const double (&)[8], double (&v)[8]) const {
    basis8(i0, cnt, d, v);
  }
  __device__ void store(int d, double v) const { st->c1[d] = v; }
};

struct OpCgsB : CgsBase {  // B: w -= V c1, c2 = V^T w
  static constexpr bool kSpmv = false;
  __device__ bool begin() {
    if (!live()) return false;
    inv = st->inv;
    nd = j;
    return true;
  }
  __device__ double gather(int) const { return 0.0; }
  __device__ void value8(int i0, int cnt, const double (&)[8], double (&u)[8]) const { update8(i0, cnt, st->c1, u); }
  __device__ void operand8(int i0, int cnt, int d, const double (&)[8], double (&v)[8]) const {
    basis8(i0, cnt, d, v);
  }
  __device__ void store(int d, double v) const { st->c2[d] = v; }
};

struct OpCgsC : CgsBase {  // C: w -= V c2, ||w||^2 -> Givens etc. (warp finish)
  static constexpr bool kSpmv = false;
  static constexpr bool kWarpFinish = true;
  double* hist;
  __device__ bool begin() {
    if (!live()) return false;
    inv = st->inv;
    nd = 1;
    return true;
  }
  __device__ double gather(int) const { return 0.0; }
  __device__ void value8(int i0, int cnt, const double (&)[8], double (&u)[8]) const { update8(i0, cnt, st->c2, u); }
  __device__ void operand8(int, int, int, const double (&u)[8], double (&v)[8]) const {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = u[k];
  }
  __device__ void finish_warp(double hn2, int lane) const { arnoldi_finish(st, hist, j, hn2, lane, 1); }
};

// X: x += sum_{k=1..K} y_k v_k (k ascending)
template <class L = LdNC>
struct OpXupd {
  static constexpr int D = 0;
  static constexpr int NV = 1;
  static constexpr bool kSpmv = false;
  const double* W;
  double* x;
  GmresState* st;
  size_t n;
  int K;
  const double *y, *inv;
  __device__ bool begin() {
    if (st->done || st->skip_x) return false;
    K = st->k;
    y = st->y;
    inv = st->inv;
    return true;
  }
  __device__ const double* vin(int) const { return x; }
  __device__ double gather(int) const { return 0.0; }
  __device__ void row(int q, double, const double (&v)[NV], double (&)[1]) const {
    double xv = v[0];
    for (int k0 = 0; k0 < K; k0 += 8) {  // batches of 8 basis loads in flight, chain in k order
      double wv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) wv[u] = k0 + u < K ? L::ld(W + (size_t)(k0 + u) * n + q) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (k0 + u < K) xv = __fma_rn(L::ld(y + k0 + u), wv[u] * L::ld(inv + k0 + u + 1), xv);
    }
    x[q] = xv;
  }
};

}  // namespace gsk
