// coop.cu — persistent cooperative Bi-CGSTAB for mid-size systems
// (SURVEY §8(a) a11 "K-SMALL").
//
// Between the one-cluster solver (<= 32768 rows) and the bandwidth-bound sizes, every
// pass of the graph-replayed solver is latency-bound: a pass + finish pair costs a few
// microseconds of launch, drain and tail regardless of n.  Here ONE cooperative launch
// runs the whole iteration loop: CTA b owns the aligned windows [b*wpc, (b+1)*wpc) (wpc
// a power of two <= 16, all CTAs co-resident — the cooperative launch fails rather than
// oversubscribe), the four passes of the four-pass schedule (S1q, S2, S3, S4q: the
// operators of bicg_ops.cuh) follow each other separated by ONE exchange each:
//
//   publish   every CTA writes its partials, then (thread 0, after the CTA barrier and
//             a gpu-scope fence) stores the pass epoch into its own flag word with
//             release semantics — no atomics, no shared counter to serialise on;
//   reduce    CTA 0 polls every flag (relaxed loads, up to four per thread, all in
//             flight; then an acquire fence), reduces the G partials with the
//             canonical tree (AC-5: up to 4 consecutive partials per thread, then the
//             256-leaf block tree), stores the D sums and releases its broadcast word;
//   finish    every other CTA acquires the broadcast word (one poller per CTA: no
//             G x G flag traffic on one L2 slice), reads the D sums and runs the op's
//             scalar epilogue on its own shared-memory copy of the state, so all CTAs
//             take identical decisions without another exchange.
//
// Partials and sums are double-buffered by reducing pass (a CTA can be at most one pass ahead
// of the slowest: it cannot pass the next exchange before the slowest has published
// it, which that CTA does only after reading this pass's partials).  Vectors written in
// the launch are read through L2 (__ldcg), never the non-coherent read-only path.
// Arithmetic and operators are those of the graph path, hence bit-identical results.
#include "bicg_ops.cuh"

namespace gsk {

constexpr int COOP_GMAX = 1024;  // CTAs of the cooperative grid (at most)
constexpr int COOP_WPC_MAX = 16; // windows per CTA (cta_partial's WMAX)

__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Publish this CTA's pass results under epoch e and wait until every CTA has published
// e: every thread polls up to four flags with relaxed loads (all in flight together),
// the CTA repeats until all are current, then an acquire fence orders the reads that
// follow (bounded: a broken invariant traps instead of hanging the GPU).
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
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
  int n, wpc, lpt;  // lpt: CTA partials per finish thread (1, 2 or 4; G <= 256 lpt)
  const double *b, *w;
  double *x, *r, *rh, *pa, *pb, *va, *vb, *t, *hist;
  double* part;     // [2][MAXD][COOP_GMAX]: CTA partials, double-buffered by reducing pass
  double* res;      // [2][MAXD]: the reduced values, written by CTA 0
  unsigned* flags;  // [COOP_GMAX] per-CTA epoch words (zeroed before the launch)
  unsigned* bcast;  // CTA 0's epoch word: res of that pass is valid
  BicgState* st_out;
  double tol;
  int maxit, fault_kind, fault_it;
};

struct CoopSmem {
  BicgState st;
  double sy[2 * TB];
  double wp[COOP_WPC_MAX * MAXD * 8];
  double red[MAXD * 8];
};

// One pass over the CTA's windows: SpMV (FMT 1 CSR, 2 SELL; NAT: natural-order SELL
// windows, MAXL slots per lane in registers) or vector rows, the op's row epilogue, the
// CTA partial; then the exchange, the tree over the CTA partials and op.finish.
template <int FMT, bool NAT, int MAXL, class Op>
__device__ __forceinline__ void coop_pass(const CoopArgs& a, Op op, CoopSmem& sm, unsigned& epoch, int& par) {
  constexpr int D = Op::D;
  constexpr int DD = D > 0 ? D : 1;
  constexpr int NVA = Op::NV > 0 ? Op::NV : 1;
  const int t = threadIdx.x, warp = t >> 5;
  if (!op.begin()) return;  // identical in every CTA (same state values): no exchange
  const int rb = blockIdx.x * a.wpc * TB;
  for (int w = 0; w < a.wpc; ++w) {
    const int r0 = rb + w * TB;
    double cc[DD];
#pragma unroll
    for (int d = 0; d < DD; ++d) cc[d] = 0.0;
    if (r0 < a.n) {  // uniform over the CTA
      const int i = r0 + t;
      double y = 0.0;
      auto g = [&](int col) { return op.gather(col); };
      if constexpr (Op::kSpmv && FMT == 1) {
        if (i < a.n)
          for (int k = __ldg(a.csr.rp + i), e = __ldg(a.csr.rp + i + 1); k < e; ++k)
            y = __fma_rn(__ldg(a.csr.v + k), g(__ldg(a.csr.ci + k)), y);
      } else if constexpr (Op::kSpmv && NAT) {
        y = sell_window_nat<0, MAXL>(a.sell, r0, g);
      } else if constexpr (Op::kSpmv) {
        y = sell_window<0>(a.sell, r0, g, sm.sy + (w & 1) * TB);
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
    if constexpr (D > 0) warp_leaves<D>(cc, sm.wp, w);
  }
  double* pp = a.part + par * MAXD * COOP_GMAX;
  double* rr = a.res + par * MAXD;
  if constexpr (D > 0) {
    __syncthreads();
    if (warp == 0) cta_partial<D>(sm.wp, a.wpc, pp, COOP_GMAX, blockIdx.x);
  }
  __syncthreads();  // every thread's vector and partial stores precede the release
  const unsigned e = ++epoch;
  const int G = gridDim.x;
  double q[DD];
  if (blockIdx.x == 0) {  // the reducer: acquire every CTA's flag, reduce, broadcast
    unsigned spin = 0;
    for (;;) {
      bool ok = true;
#pragma unroll
      for (int k = 0; k < COOP_GMAX / TB; ++k) {
        const int j = t + k * TB;
        if (j >= 1 && j < G) ok &= (int)(ld_relaxed(a.flags + j) - e) >= 0;
      }
      if (__syncthreads_and(ok)) break;
      if (++spin > (1u << 26)) __trap();
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    if constexpr (D > 0) {
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const double* src = pp + d * COOP_GMAX;
        if (a.lpt == 1) {
          q[d] = t < G ? __ldcg(src + t) : 0.0;
        } else if (a.lpt == 2) {
          const int j = 2 * t;
          const double u0 = j < G ? __ldcg(src + j) : 0.0, u1 = j + 1 < G ? __ldcg(src + j + 1) : 0.0;
          q[d] = u0 + u1;
        } else {
          const int j = 4 * t;
          const double u0 = j < G ? __ldcg(src + j) : 0.0, u1 = j + 1 < G ? __ldcg(src + j + 1) : 0.0;
          const double u2 = j + 2 < G ? __ldcg(src + j + 2) : 0.0, u3 = j + 3 < G ? __ldcg(src + j + 3) : 0.0;
          q[d] = (u0 + u1) + (u2 + u3);
        }
      }
      double qq[D];
#pragma unroll
      for (int d = 0; d < D; ++d) qq[d] = q[d];
      block_tree_256<D>(qq, sm.red);
#pragma unroll
      for (int d = 0; d < D; ++d) q[d] = qq[d];
      if (t < D) {
#pragma unroll
        for (int d = 0; d < D; ++d)
          if (t == d) rr[d] = qq[d];
      }
    }
    __syncthreads();
    if (t == 0 && G > 1) {
      __threadfence();
      st_release(a.bcast, e);
    }
  } else {  // publish, then wait for the reducer's broadcast
    if (t == 0) {
      __threadfence();
      st_release(a.flags + blockIdx.x, e);
      unsigned spin = 0;
      while ((int)(ld_acquire(a.bcast) - e) < 0)
        if (++spin > (1u << 28)) __trap();
    }
    __syncthreads();
    if constexpr (D > 0) {
      if (warp == 0) {
#pragma unroll
        for (int d = 0; d < D; ++d) q[d] = __ldcg(rr + d);
      }
    }
  }
  if constexpr (D > 0) {
#pragma unroll
    for (int d = 0; d < D; ++d) q[d] = q[d] + 0.0;  // AC-5
    double qf[D];
#pragma unroll
    for (int d = 0; d < D; ++d) qf[d] = q[d];
    if (warp == 0) op.finish(qf, t);
    // the next reducing pass writes the other partial / result buffer; this one is
    // rewritten only after the next pass's exchange, i.e. after every CTA has read it
    par ^= 1;
    __syncthreads();  // the state copy is read by the next pass
  }
}

template <int FMT, bool NAT, int MAXL, int MINB>
__global__ void __launch_bounds__(TB, MINB) coop_bicgstab(CoopArgs a) {
  __shared__ CoopSmem sm;
  if (threadIdx.x == 0) {
    sm.st = BicgState{};
    sm.st.tol = a.tol;
    sm.st.maxit = a.maxit;
    sm.st.fault_kind = a.fault_kind;
    sm.st.fault_it = a.fault_it;
  }
  __syncthreads();
  int par = 0;
  unsigned epoch = 0;
  BicgState* st = &sm.st;
  OpInit<LdCG> init{a.x, a.b, a.w, a.r, a.rh, a.pa, a.va, a.hist, st};
  coop_pass<FMT, NAT, MAXL>(a, init, sm, epoch, par);
  double *v = a.va, *sv = a.pb;
  for (int k = 0;; ++k) {
    if (sm.st.done && !sm.st.halfstep) break;
    // four-pass schedule (bicgstab.cu, bicg_schedule 3): q / p alternate between pa and vb
    double *qs = (k & 1) ? a.vb : a.pa, *pd = (k & 1) ? a.pa : a.vb;
    OpS1q<LdCG> s1{qs, a.r, a.rh, pd, v, st, 0.0};
    OpS2 s2{a.r, v, a.w, sv, a.hist, st, 0};
    OpS3<LdCG> s3{sv, a.t, st};
    OpS4q s4{sv, a.t, a.rh, a.w, v, pd, a.x, a.r, a.hist, st, 0, 0, 0, 0};
    coop_pass<FMT, NAT, MAXL>(a, s1, sm, epoch, par);
    coop_pass<0, false, 8>(a, s2, sm, epoch, par);
    coop_pass<FMT, NAT, MAXL>(a, s3, sm, epoch, par);
    coop_pass<0, false, 8>(a, s4, sm, epoch, par);
  }
  OpFinal<LdCG> fin{a.x, a.b, a.w, st};
  coop_pass<FMT, NAT, MAXL>(a, fin, sm, epoch, par);
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.st_out = sm.st;
}

template <int MINB>
static void (*coop_kernel(bool sell, bool nat, bool shortl))(CoopArgs) {
  return !sell ? coop_bicgstab<1, false, 8, MINB>
       : !nat  ? coop_bicgstab<2, false, 8, MINB>
       : shortl ? coop_bicgstab<2, true, 5, MINB> : coop_bicgstab<2, true, 8, MINB>;
}

// Windows per CTA: the smallest power of two (<= 16) whose grid fits the co-resident
// CTAs (GSK_COOP_G caps the grid below that, for tuning) and COOP_GMAX.
static int coop_max_grid() {
  const char* e = getenv("GSK_COOP_G");
  const int g = e ? atoi(e) : 0;
  return g > 0 ? std::min(g, COOP_GMAX) : COOP_GMAX;
}

// Host side: returns GSK_OK with *used = 0 when the system does not fit the
// cooperative grid or the plan's format (SELL-D / SELL-U) is not supported here (the
// caller then runs the graph path).
int coop_bicgstab_run(gsk_plan* P, const double* b, double tol, int maxit, double* x, int* used) {
  *used = 0;
  const int n = P->A.n;
  if (P->fmt == GSK_FMT_SELL && (P->sell.dict || P->sell.uptr)) return GSK_OK;
  const bool sell = P->fmt == GSK_FMT_SELL;
  const bool nat = sell && P->sell.all_nat != 0;
  const bool shortl = nat && P->sell_maxlen <= 5;
  // register budget (CTAs per SM): GSK_COOP_MINB = 2, 3 or 4 (default 2: 3 and 4 spill
  // and run 10-60% slower, profiles/r02u_coop_m*.json)
  const char* mb = getenv("GSK_COOP_MINB");
  const int minb = mb ? atoi(mb) : 2;
  void (*kern)(CoopArgs) = minb == 2 ? coop_kernel<2>(sell, nat, shortl)
                         : minb == 4 ? coop_kernel<4>(sell, nat, shortl) : coop_kernel<3>(sell, nat, shortl);
  int per_sm = 0;
  GSK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TB, 0));
  const long long resident = (long long)per_sm * num_sms();
  const int gmax = (int)std::min<long long>(resident, coop_max_grid());
  const int windows = (n + TB - 1) / TB;
  int wpc = 1;
  while ((windows + wpc - 1) / wpc > gmax && wpc < COOP_WPC_MAX) wpc <<= 1;
  const int G = (windows + wpc - 1) / wpc;
  if (G > gmax || G < 1) return GSK_OK;  // too large: the graph path streams better
  const int lpt = G <= 256 ? 1 : G <= 512 ? 2 : 4;
  // [2][MAXD][COOP_GMAX] partials, [2][MAXD] results, then COOP_GMAX flags + the broadcast word
  const size_t pdoubles = 2 * MAXD * COOP_GMAX + 2 * MAXD;
  if (!P->cpart) GSK_CUDA(pool_alloc((void**)&P->cpart, sizeof(double) * pdoubles + sizeof(unsigned) * (COOP_GMAX + 32)));
  unsigned* flags = reinterpret_cast<unsigned*>(P->cpart + pdoubles);
  GSK_CUDA(cudaMemsetAsync(flags, 0, sizeof(unsigned) * (COOP_GMAX + 32), P->st));
  double* V = P->bvec;
  const size_t nn = (size_t)n;
  CoopArgs a{};
  a.csr = P->csr;
  a.sell = P->sell;
  a.n = n;
  a.wpc = wpc;
  a.lpt = lpt;
  a.b = b;
  a.w = P->weights;
  a.x = x;
  a.r = V;
  a.rh = V + nn;
  a.pa = V + 2 * nn;
  a.pb = V + 3 * nn;
  a.va = V + 4 * nn;
  a.vb = V + 5 * nn;
  a.t = V + 6 * nn;
  a.hist = P->hist_d;
  a.part = P->cpart;
  a.res = P->cpart + 2 * MAXD * COOP_GMAX;
  a.flags = flags;
  a.bcast = flags + COOP_GMAX;
  a.st_out = P->bstate;
  a.tol = tol;
  a.maxit = maxit;
  read_fault(&a.fault_kind, &a.fault_it);
  void* args[] = {&a};
  GSK_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), G, TB, args, 0, P->st));
  GSK_LAUNCHED(1);
  *used = 1;
  return GSK_OK;
}

}  // namespace gsk
