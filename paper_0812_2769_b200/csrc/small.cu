// small.cu — on-chip single-CTA solvers for small systems (SURVEY §8(a) a11 "K-SMALL";
// DESIGN.md §5).
//
// Below a few thousand rows every graph-replayed pass is pure latency (launch, grid
// drain, finish kernel: ~4 us whatever n is).  Here ONE 1024-thread CTA runs the whole
// solve: thread t owns rows t, t + 1024, ... (n <= GSK_SMALL_NMAX = 4096, four rows per
// thread at most); a pass is a loop over those rows, a reduction is warp butterflies +
// one warp over the window partials, and the passes are separated by __syncthreads
// instead of kernel boundaries.  Bi-CGSTAB keeps its six work vectors in shared memory
// (48 n bytes <= 192 KB); GMRES keeps its basis in global memory (L1/L2 resident) with
// plain coherent loads.  The operators are the graph path's (bicg_ops.cuh,
// gmres_ops.cuh) with the coherent load policy, and the reduction is the canonical
// tree (AC-5), so every result is bit-identical to the graph path and the oracle.
#include "bicg_ops.cuh"
#include "gmres_ops.cuh"

namespace gsk {

constexpr int SMALL_T = 1024;                  // threads of the one CTA
constexpr int SMALL_WS = GSK_SMALL_NMAX / 32;  // warp sums per dot product (128)
constexpr int SMALL_B = 4;                     // row entries loaded ahead of the FMA chain

// One pass of Op over all rows.  Window w (rows [256 w, 256 w + 256)) is warps
// 8 (w mod 4) .. +7 of slab w / 4, so each warp sum is the canonical subtree of its 32
// rows; warp 0 then builds each window's 8-warp tree (lane = window) and the butterfly
// over the windows (absent windows enter as +0 leaves, AC-5), adds + 0.0 and runs the
// Op's scalar epilogue.  Starts and ends with the state consistent across the CTA.
// (Measured: one row per thread beats 4 consecutive rows per thread on 256 threads —
// the pass is latency-bound, not shuffle-bound.)
template <class Op>
__device__ __forceinline__ void small_pass(const CsrView& A, int n, Op op, double* wsum) {
  constexpr int D = Op::D;
  constexpr int DD = D > 0 ? D : 1;
  constexpr int NVA = Op::NV > 0 ? Op::NV : 1;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int slabs = (n + SMALL_T - 1) / SMALL_T;
  const bool run = op.begin();  // reads the shared state: identical in every thread
  if (run) {
#pragma unroll 1
    for (int k = 0; k < slabs; ++k) {
      const int i = k * SMALL_T + t;
      double cc[DD];
#pragma unroll
      for (int d = 0; d < DD; ++d) cc[d] = 0.0;
      if (i < n) {
        double y = 0.0;
        if constexpr (Op::kSpmv) {  // SMALL_B entries' loads in flight, then their FMAs (AC-3)
          const int e = __ldg(A.rp + i + 1);
          for (int q0 = __ldg(A.rp + i); q0 < e; q0 += SMALL_B) {
            double av[SMALL_B];
            int cv[SMALL_B];
#pragma unroll
            for (int u = 0; u < SMALL_B; ++u)
              if (q0 + u < e) {
                av[u] = __ldg(A.v + q0 + u);
                cv[u] = __ldg(A.ci + q0 + u);
              }
#pragma unroll
            for (int u = 0; u < SMALL_B; ++u)
              if (q0 + u < e) y = __fma_rn(av[u], op.gather(cv[u]), y);
          }
        }
        double v[NVA];
#pragma unroll
        for (int kk = 0; kk < Op::NV; ++kk) {
          const double* src = op.vin(kk);
          v[kk] = src ? src[i] : 0.0;
        }
        op.row(i, y, v, cc);
      }
      if constexpr (D > 0) {
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
#pragma unroll
          for (int d = 0; d < D; ++d) cc[d] = cc[d] + __shfl_xor_sync(0xffffffffu, cc[d], off);
        }
        if (lane == 0) {
#pragma unroll
          for (int d = 0; d < D; ++d) wsum[d * SMALL_WS + k * 32 + warp] = cc[d];
        }
      }
    }
  }
  __syncthreads();
  if constexpr (D > 0) {
    if (run && warp == 0) {
      const int nwin = slabs * (SMALL_T / TB);
      double q[D];
#pragma unroll
      for (int d = 0; d < D; ++d) {
        double u = 0.0;
        if (lane < nwin) {
          const double* a = wsum + d * SMALL_WS + lane * 8;
          u = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
        }
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) u = u + __shfl_xor_sync(0xffffffffu, u, off);
        q[d] = u + 0.0;  // AC-5
      }
      op.finish(q, lane);
    }
    __syncthreads();
  }
}

// ---- Bi-CGSTAB: the split schedule S0..S4 (bicgstab.cu), vectors in shared memory ----
struct SmallBicgArgs {
  CsrView csr;
  int n;
  const double *b, *w;
  double *x, *hist;
  BicgState* st_out;
  double tol;
  int maxit;
};

__global__ void __launch_bounds__(SMALL_T, 1) small_bicgstab(SmallBicgArgs a) {
  extern __shared__ double vec[];  // r, r^, p, v, s, t
  __shared__ BicgState st;
  __shared__ double wsum[MAXD * SMALL_WS];
  const int n = a.n;
  double *r = vec, *rh = vec + n, *p = vec + 2 * n, *v = vec + 3 * n, *s = vec + 4 * n, *t = vec + 5 * n;
  if (threadIdx.x == 0) {
    st = BicgState{};
    st.tol = a.tol;
    st.maxit = a.maxit;
  }
  __syncthreads();
  small_pass(a.csr, n, OpInit<LdPlain>{a.x, a.b, a.w, r, rh, p, v, a.hist, &st}, wsum);
  while (!(st.done && !st.halfstep)) {
    small_pass(a.csr, n, OpS0{r, v, p, &st, 0, 0}, wsum);
    small_pass(a.csr, n, OpS1<LdPlain>{p, rh, v, &st}, wsum);
    small_pass(a.csr, n, OpS2{r, v, a.w, s, a.hist, &st, 0}, wsum);
    small_pass(a.csr, n, OpS3<LdPlain>{s, t, &st}, wsum);
    small_pass(a.csr, n, OpS4{s, p, t, rh, a.w, a.x, r, a.hist, &st, 0, 0, 0}, wsum);
  }
  small_pass(a.csr, n, OpFinal<LdPlain>{a.x, a.b, a.w, &st}, wsum);
  if (threadIdx.x == 0) *a.st_out = st;
}

int small_bicgstab_run(gsk_plan* P, const double* b, double tol, int maxit, double* x) {
  const int n = P->A.n;
  static const char attr_key = 0;  // function attributes are per device
  if (!device_attr_done(&attr_key)) {
    GSK_CUDA(cudaFuncSetAttribute(small_bicgstab, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(6 * sizeof(double) * GSK_SMALL_NMAX)));
    device_attr_mark(&attr_key);
  }
  SmallBicgArgs a{P->csr, n, b, P->weights, x, P->hist_d, P->bstate, tol, maxit};
  small_bicgstab<<<1, SMALL_T, 6 * sizeof(double) * (size_t)n, P->st>>>(a);
  GSK_LAUNCHED(1);
  return GSK_OK;
}

// ---- GMRES(m) with MGS: the cycle of gmres.cu (S_j, M_ij, L_j, X, R) in one CTA -------
struct SmallGmresArgs {
  CsrView csr;
  int n;
  const double *b, *w;
  double *x, *W, *hist;
  GmresState h;  // initial state (arrays in global memory, zeroed by the host)
  GmresState* st_out;
};

__global__ void __launch_bounds__(SMALL_T, 1) small_gmres(SmallGmresArgs a) {
  __shared__ GmresState st;
  __shared__ double wsum[MAXD * SMALL_WS];
  const int n = a.n;
  if (threadIdx.x == 0) st = a.h;
  __syncthreads();
  auto slot = [&](int j) { return a.W + (size_t)(j - 1) * n; };
  small_pass(a.csr, n, OpGResid<LdPlain>{a.x, a.b, a.w, a.W, a.hist, &st, 1}, wsum);
  const int m = st.m;
  const long long maxc = (long long)st.maxit + 2;  // as the host loop of gmres.cu
  for (long long c = 0; c < maxc && !st.done; ++c) {
    for (int j = 1; j <= m && !st.done && !st.cycle_stop; ++j) {
      small_pass(a.csr, n, OpArnoldi<LdPlain>{slot(j), slot(1), slot(j + 1), &st, j, 0, 0}, wsum);
      for (int i = 1; i < j; ++i) small_pass(a.csr, n, OpMgs{slot(i), slot(i + 1), slot(j + 1), &st, i, j, 0, 0, 0}, wsum);
      small_pass(a.csr, n, OpLast{slot(j), slot(j + 1), a.hist, &st, j, 0, 0}, wsum);
    }
    small_pass(a.csr, n, OpXupd<LdPlain>{a.W, a.x, &st, (size_t)n, 0, nullptr, nullptr}, wsum);
    small_pass(a.csr, n, OpGResid<LdPlain>{a.x, a.b, a.w, a.W, a.hist, &st, 0}, wsum);
  }
  if (threadIdx.x == 0) *a.st_out = st;
}

int small_gmres_run(gsk_plan* P, const double* b, double* x, const GmresState& h) {
  SmallGmresArgs a{P->csr, P->A.n, b, P->weights, x, P->W, P->hist_d, h, P->gstate};
  small_gmres<<<1, SMALL_T, 0, P->st>>>(a);
  GSK_LAUNCHED(1);
  return GSK_OK;
}

}  // namespace gsk
