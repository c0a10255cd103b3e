// coop.cu — cooperative single-launch Bi-CGSTAB for small and medium systems
// (SURVEY §8(a) a11 "K-SMALL").
//
// Below ~2M rows every pass of the graph-replayed solver is latency-bound (a pass +
// finish pair costs ~5 us of launch and tail regardless of n).  Here ONE cooperative
// launch runs the whole iteration loop: CTA b owns the aligned windows
// [b*wpc, (b+1)*wpc) (wpc a power of two, <= 256 CTAs, all co-resident — the
// cooperative launch fails rather than oversubscribe), the five passes of the split
// schedule are separated by grid barriers, and after each reducing pass EVERY CTA
// reduces the <= 256 CTA partials with the same canonical tree and runs the same
// scalar epilogue on its own shared-memory copy of the state — so all CTAs take
// identical decisions without another barrier.  Operators and arithmetic are the ones
// of the graph path (bicg_ops.cuh), hence the results are bit-identical to it and to
// the oracle.
#include "bicg_ops.cuh"

namespace gsk {

// Grid barrier over the co-resident grid: arrival counter + generation word, release
// / acquire ordering, tight acquire-load polling (bounded: a broken invariant traps
// instead of hanging the GPU).  A one-CTA grid needs only __syncthreads.
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void grid_barrier(unsigned* count, unsigned* gen) {
  __syncthreads();
  if (gridDim.x == 1) return;
  if (threadIdx.x == 0) {
    const unsigned g = ld_acquire(gen);
    __threadfence();
    if (atomicAdd(count, 1u) == gridDim.x - 1) {
      *count = 0u;
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(gen), "r"(g + 1) : "memory");
    } else {
      unsigned spin = 0;
      while (ld_acquire(gen) == g)
        if (++spin > (1u << 30)) __trap();
    }
  }
  __syncthreads();
}

// Canonical tree over the 256 values held by a CTA (thread t holds leaf t); the
// result is valid in warp 0.
template <int D>
__device__ __forceinline__ void block_tree_256(double (&v)[D], double* sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
#pragma unroll
    for (int d = 0; d < D; ++d) v[d] = v[d] + __shfl_xor_sync(0xffffffffu, v[d], off);
  }
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int d = 0; d < D; ++d) sm[d * 8 + warp] = v[d];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      double u = lane < 8 ? sm[d * 8 + lane] : 0.0;
      u = u + __shfl_xor_sync(0xffffffffu, u, 1);
      u = u + __shfl_xor_sync(0xffffffffu, u, 2);
      u = u + __shfl_xor_sync(0xffffffffu, u, 4);
      v[d] = u;
    }
  }
}

struct CoopArgs {
  CsrView csr;
  SellView sell;
  int fmt;  // 1 CSR, 2 SELL
  int n, wpc;
  const double *b, *w;
  double *x, *r, *rh, *p, *v, *s, *t, *hist;
  double* part;  // [2][MAXD][256]: CTA partials, double-buffered by reducing pass
  unsigned* bar;  // [2] count, generation
  BicgState* st_out;
  double tol;
  int maxit;
};

// One pass over the CTA's windows: SpMV (FMT 1/2) or vector rows, the Op's row
// epilogue, the CTA partial; then barrier, tree over the CTA partials, op.finish.
template <int FMT, class Op>
__device__ __forceinline__ void coop_pass(const CoopArgs& a, Op op, double* sy, double* wp, double* red, int& par) {
  constexpr int D = Op::D;
  constexpr int DD = D > 0 ? D : 1;
  constexpr int NVA = Op::NV > 0 ? Op::NV : 1;
  const int t = threadIdx.x, warp = t >> 5;
  const bool run = op.begin();  // identical in every CTA (same state copy values)
  if (run) {
    const int rb = blockIdx.x * a.wpc * TB;
    for (int w = 0; w < a.wpc; ++w) {
      const int r0 = rb + w * TB;
      double cc[DD];
#pragma unroll
      for (int d = 0; d < DD; ++d) cc[d] = 0.0;
      if (r0 < a.n) {
        const int i = r0 + t;
        double y = 0.0;
        if constexpr (FMT == 1) {
          if (i < a.n)
            for (int k = a.csr.rp[i]; k < a.csr.rp[i + 1]; ++k) y = __fma_rn(a.csr.v[k], op.gather(a.csr.ci[k]), y);
        } else if constexpr (FMT == 2) {
          y = sell_window<0>(a.sell, r0, [&](int col) { return op.gather(col); }, sy + (w & 1) * TB);
        }
        if (i < a.n) {
          double v[NVA];
#pragma unroll
          for (int k = 0; k < Op::NV; ++k) {  // coherent (L2) loads: written in this launch
            const double* src = op.vin(k);
            v[k] = src ? __ldcg(src + i) : 0.0;
          }
          op.row(i, y, v, cc);
        }
      }
      if constexpr (D > 0) warp_leaves<D>(cc, wp, w);
    }
    if constexpr (D > 0) {
      __syncthreads();
      if (warp == 0) cta_partial<D>(wp, a.wpc, a.part + par * MAXD * 256, 256, blockIdx.x);
    }
  }
  grid_barrier(a.bar, a.bar + 1);  // pass results (vectors, partials) visible grid-wide
  if constexpr (D > 0) {
    if (run) {
      const double* pp = a.part + par * MAXD * 256;
      double q[D];
#pragma unroll
      for (int d = 0; d < D; ++d) q[d] = t < (int)gridDim.x ? __ldcg(pp + d * 256 + t) : 0.0;
      block_tree_256<D>(q, red);
#pragma unroll
      for (int d = 0; d < D; ++d) q[d] = q[d] + 0.0;  // AC-5
      if (warp == 0) op.finish(q, t);
    }
    // the next reducing pass writes the other partial buffer; this one is rewritten
    // only after the next pass's barrier, i.e. after every CTA has read it
    par ^= 1;
    __syncthreads();  // the state copy is read by the next pass
  }
}

template <int FMT>
__global__ void __launch_bounds__(TB) coop_bicgstab(CoopArgs a) {
  __shared__ BicgState st;
  __shared__ double sy[2 * TB];
  __shared__ double wp[8 * MAXD * 8];
  __shared__ double red[MAXD * 8];
  if (threadIdx.x == 0) {
    st = BicgState{};
    st.tol = a.tol;
    st.maxit = a.maxit;
  }
  __syncthreads();
  int par = 0;
  OpInit<LdCG> init{a.x, a.b, a.w, a.r, a.rh, a.p, a.v, a.hist, &st};
  coop_pass<FMT>(a, init, sy, wp, red, par);
  OpS0 s0{a.r, a.v, a.p, &st, 0, 0};
  OpS1<LdCG> s1{a.p, a.rh, a.v, &st};
  OpS2 s2{a.r, a.v, a.w, a.s, a.hist, &st, 0};
  OpS3<LdCG> s3{a.s, a.t, &st};
  OpS4 s4{a.s, a.p, a.t, a.rh, a.w, a.x, a.r, a.hist, &st, 0, 0, 0};
  for (;;) {
    if (st.done && !st.halfstep) break;
    coop_pass<0>(a, s0, sy, wp, red, par);
    coop_pass<FMT>(a, s1, sy, wp, red, par);
    coop_pass<0>(a, s2, sy, wp, red, par);
    coop_pass<FMT>(a, s3, sy, wp, red, par);
    coop_pass<0>(a, s4, sy, wp, red, par);
  }
  OpFinal<LdCG> fin{a.x, a.b, a.w, &st};
  coop_pass<FMT>(a, fin, sy, wp, red, par);
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.st_out = st;
}

// Host side: returns GSK_OK with *used = 0 when the system does not fit the
// cooperative grid (the caller then runs the graph path).
int coop_bicgstab_run(gsk_plan* P, const double* b, double tol, int maxit, double* x, int* used) {
  *used = 0;
  const int n = P->A.n;
  const int windows = (n + TB - 1) / TB;
  int wpc = 1;
  while ((windows + wpc - 1) / wpc > 256) wpc <<= 1;
  if (wpc > 8) return GSK_OK;  // > 2^19 rows: the graph path streams better
  const int G = (windows + wpc - 1) / wpc;
  const int fmt = P->fmt == GSK_FMT_SELL ? 2 : 1;
  void (*kern)(CoopArgs) = fmt == 2 ? coop_bicgstab<2> : coop_bicgstab<1>;
  int per_sm = 0;
  GSK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TB, 0));
  if ((long long)per_sm * num_sms() < G) return GSK_OK;
  if (!P->cpart) GSK_CUDA(cudaMalloc(&P->cpart, sizeof(double) * 2 * MAXD * 256 + sizeof(unsigned) * 4));
  unsigned* bar = reinterpret_cast<unsigned*>(P->cpart + 2 * MAXD * 256);
  GSK_CUDA(cudaMemsetAsync(bar, 0, sizeof(unsigned) * 2, P->st));
  double* V = P->bvec;
  const size_t nn = (size_t)n;
  CoopArgs a{P->csr, P->sell, fmt, n, wpc, b, P->weights, x, V, V + nn, V + 2 * nn, V + 4 * nn, V + 3 * nn,
             V + 6 * nn, P->hist_d, P->cpart, bar, P->bstate, tol, maxit};
  void* args[] = {&a};
  GSK_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), G, TB, args, 0, P->st));
  GSK_LAUNCHED(1);
  *used = 1;
  return GSK_OK;
}

}  // namespace gsk
