// cluster.cu — on-chip solvers on one thread-block cluster: the
// single-CTA solvers of small.cu spread over CS <= 16 CTAs of a cluster, for systems
// of up to 16 x 4096 rows (the paper's Problem 1 at 128 x 128 is 16384 rows).
//
// CTA c of the cluster owns the aligned row block [c B, (c+1) B) (B a power of two,
// <= 4096), rows c B + 1024 k + t for thread t.  Bi-CGSTAB keeps its six vectors in the
// CTAs' shared memory (each CTA its block; SpMV gathers of another CTA's rows go
// through distributed shared memory), GMRES its basis in global memory (L2; gathers of
// rows written by other CTAs bypass L1).  A pass: the rows, a warp
// butterfly per 32 rows and the CTA's tree over its warps (a canonical subtree, the
// block being aligned), the CTA value parked in shared memory, ONE cluster barrier
// (hardware, release/acquire at cluster scope: vectors and CTA values visible), then
// every CTA reads the CS CTA values through distributed shared memory, joins them
// with the top of the same tree (+ 0.0, AC-5) and runs the operator's scalar epilogue
// on its own shared-memory copy of the state — every CTA takes the same decisions
// without another barrier.  Operators are the graph path's (bicg_ops.cuh,
// gmres_ops.cuh): results are bit-identical to it and to the oracle.  GMRES keeps
// its small dense arrays (H, Givens, g, y, 1/norms) per CTA in shared memory, so the
// replicated epilogues never race on global memory.
#include <cooperative_groups.h>
#include "bicg_ops.cuh"
#include "gmres_ops.cuh"

namespace cg = cooperative_groups;

namespace gsk {

constexpr int CL_T = 1024;      // threads per CTA = max rows per CTA
constexpr int CL_MAX = 16;      // CTAs per cluster (non-portable size)
constexpr int CL_NMAX = 4 * CL_T * CL_MAX;  // 65536 rows
constexpr int CL_MMAX = 40;     // GMRES restart length with its arrays in shared memory

constexpr int CL_RPT = 4;       // rows per thread at most (CTA blocks of <= 4096 rows)

struct ClusterRed {
  double wsum[MAXD][CL_RPT * 32];  // warp sums of the CTA's block, in row order
  double cpart[2][MAXD];           // this CTA's block value, double-buffered by reducing pass
};

template <class Op, class = void>
struct Gathers : std::false_type {};
template <class Op>
struct Gathers<Op, std::void_t<decltype(std::declval<Op>().gathered())>> : std::true_type {};
// gather(c) = gxform(gathered()[c]) for ops that transform the gathered value
template <class Op, class = void>
struct GXform {
  __device__ static double apply(const Op&, double v) { return v; }
};
template <class Op>
struct GXform<Op, std::void_t<decltype(std::declval<Op>().gxform(0.0))>> {
  __device__ static double apply(const Op& op, double v) { return op.gxform(v); }
};

// DSM: the vectors live in the CTAs' shared memory (each CTA its own block, addressed
// through a base pointer offset by -r0 so that operators index them by global row);
// an operator's gathered vector is then read from the owning CTA's shared memory —
// local, or through distributed shared memory for rows of another CTA.
template <bool DSM = false, class Op>
__device__ __forceinline__ void cluster_pass(const CsrView& A, int n, int r0, int B, Op op, ClusterRed& R,
                                             int& par) {
  constexpr int D = Op::D;
  constexpr int DD = D > 0 ? D : 1;
  constexpr int NVA = Op::NV > 0 ? Op::NV : 1;
  cg::cluster_group cluster = cg::this_cluster();
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int slabs = (B + CL_T - 1) / CL_T;
  const bool run = op.begin();  // the shared state copy: identical in every CTA
  if (run) {
#pragma unroll 1
    for (int k = 0; k < slabs; ++k) {  // rows r0 + 1024 k + t (warp sums in row order)
      const int i = r0 + k * CL_T + t;
      double cc[DD];
#pragma unroll
      for (int d = 0; d < DD; ++d) cc[d] = 0.0;
      if (k * CL_T + t < B && i < n) {
        double y = 0.0;
        if constexpr (Op::kSpmv && DSM && Gathers<Op>::value) {  // AC-3 chain, DSMEM gathers
          const double* gb = op.gathered() + r0;  // this CTA's block of the gathered vector
          const unsigned me = cluster.block_rank();
          const int lgB = __ffs(B) - 1;
          const int e = __ldg(A.rp + i + 1);
          for (int q = __ldg(A.rp + i); q < e; ++q) {
            const int c = __ldg(A.ci + q);
            const unsigned owner = (unsigned)c >> lgB;
            const int off = c - (int)(owner << lgB);
            const double xc = GXform<Op>::apply(op, owner == me ? gb[off] : cluster.map_shared_rank(gb, owner)[off]);
            y = __fma_rn(__ldg(A.v + q), xc, y);
          }
        } else if constexpr (Op::kSpmv) {  // AC-3 chain in CSR order
          const int e = __ldg(A.rp + i + 1);
          for (int q = __ldg(A.rp + i); q < e; ++q) y = __fma_rn(__ldg(A.v + q), op.gather(__ldg(A.ci + q)), y);
        }
        double v[NVA];
#pragma unroll
        for (int kk = 0; kk < Op::NV; ++kk) {
          const double* src = op.vin(kk);
          v[kk] = src ? src[i] : 0.0;  // own rows: written by this thread only
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
          for (int d = 0; d < D; ++d) R.wsum[d][k * 32 + warp] = cc[d];
        }
      }
    }
  }
  if constexpr (D > 0) {
    __syncthreads();
    if (run && warp == 0) {
      // the block's tree over its B/32 warp sums: lane l joins sums 4l..4l+3 (an
      // aligned subtree), then a butterfly over the lanes
      const int nw = B >= 32 ? B / 32 : 1;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        double a4[CL_RPT];
#pragma unroll
        for (int q = 0; q < CL_RPT; ++q) a4[q] = CL_RPT * lane + q < nw ? R.wsum[d][CL_RPT * lane + q] : 0.0;
        double u = (a4[0] + a4[1]) + (a4[2] + a4[3]);
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) u = u + __shfl_xor_sync(0xffffffffu, u, off);
        if (lane == 0) R.cpart[par][d] = u;
      }
    }
  }
  cluster.sync();  // the pass's vectors and the CTA values, cluster-wide
  if constexpr (D > 0) {
    if (run && warp == 0) {
      const int cs = (int)cluster.num_blocks();
      double q[D];
#pragma unroll
      for (int d = 0; d < D; ++d) {
        double u = lane < cs ? *cluster.map_shared_rank(&R.cpart[par][d], lane) : 0.0;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) u = u + __shfl_xor_sync(0xffffffffu, u, off);
        q[d] = u + 0.0;  // AC-5
      }
      op.finish(q, lane);
    }
    // the next reducing pass writes the other buffer; this one is rewritten only after
    // the next pass's cluster barrier, i.e. after every CTA has read it
    par ^= 1;
    __syncthreads();
  }
}

// ---- Bi-CGSTAB: split schedule, vectors in the cluster's shared memory ---------------------
struct ClusterBicgArgs {
  CsrView csr;
  int n, B;
  const double *b, *w;
  double *x, *hist;
  BicgState* st_out;
  double tol;
  int maxit;
};

__global__ void __launch_bounds__(CL_T, 1) cluster_bicgstab(ClusterBicgArgs a) {
  extern __shared__ double vec[];  // this CTA's rows of r, r^, p, v, s, t (B each)
  __shared__ BicgState st;
  __shared__ ClusterRed R;
  const int n = a.n, B = a.B, r0 = (int)cg::this_cluster().block_rank() * B;
  // base pointers offset by -r0: operators index the vectors by global row
  double *r = vec - r0, *rh = vec + B - r0, *p = vec + 2 * B - r0, *v = vec + 3 * B - r0, *s = vec + 4 * B - r0,
         *t = vec + 5 * B - r0;
  if (threadIdx.x == 0) {
    st = BicgState{};
    st.tol = a.tol;
    st.maxit = a.maxit;
  }
  __syncthreads();
  int par = 0;
  cluster_pass<true>(a.csr, n, r0, B, OpInit<LdCG>{a.x, a.b, a.w, r, rh, p, v, a.hist, &st}, R, par);
  while (!(st.done && !st.halfstep)) {
    cluster_pass<true>(a.csr, n, r0, B, OpS0{r, v, p, &st, 0, 0}, R, par);
    cluster_pass<true>(a.csr, n, r0, B, OpS1<LdPlain>{p, rh, v, &st}, R, par);
    cluster_pass<true>(a.csr, n, r0, B, OpS2{r, v, a.w, s, a.hist, &st, 0}, R, par);
    cluster_pass<true>(a.csr, n, r0, B, OpS3<LdPlain>{s, t, &st}, R, par);
    cluster_pass<true>(a.csr, n, r0, B, OpS4{s, p, t, rh, a.w, a.x, r, a.hist, &st, 0, 0, 0}, R, par);
  }
  cluster_pass<true>(a.csr, n, r0, B, OpFinal<LdCG>{a.x, a.b, a.w, &st}, R, par);
  if (cg::this_cluster().block_rank() == 0 && threadIdx.x == 0) *a.st_out = st;
  cg::this_cluster().sync();  // no CTA exits while another may still read its shared memory
}

// Cluster geometry for n rows: CS CTAs (power of two, <= 16) of B rows (power of two,
// <= 4096, up to four rows per thread); 0 if n is too large.
// As many CTAs as give each at least 256 rows (measured: 256-row blocks beat 1024-row
// blocks at n = 4096 by 10-35%).
static int cluster_geometry(int n, int* B) {
  if (n > CL_NMAX) return 0;
  int cs = 1;
  while (cs * 256 < n && cs < CL_MAX) cs <<= 1;
  int b = 32;
  while (b * cs < n) b <<= 1;
  *B = b;
  return cs;
}

static cudaError_t launch_cluster(const void* kern, int cs, void** args, cudaStream_t s, size_t smem = 0) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs);
  cfg.blockDim = dim3(CL_T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, kern, args);
}

int cluster_bicgstab_run(gsk_plan* P, const double* b, double tol, int maxit, double* x, int* used) {
  *used = 0;
  const int n = P->A.n;
  int B = 0;
  const int cs = cluster_geometry(n, &B);
  if (!cs) return GSK_OK;
  static const char attr_key = 0;  // function attributes are per device
  if (!device_attr_done(&attr_key)) {
    GSK_CUDA(cudaFuncSetAttribute(cluster_bicgstab, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    GSK_CUDA(cudaFuncSetAttribute(cluster_bicgstab, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(6 * sizeof(double) * CL_RPT * CL_T)));
    device_attr_mark(&attr_key);
  }
  ClusterBicgArgs a{P->csr, n, B, b, P->weights, x, P->hist_d, P->bstate, tol, maxit};
  void* args[] = {&a};
  GSK_CUDA(launch_cluster(reinterpret_cast<const void*>(cluster_bicgstab), cs, args, P->st, 6 * sizeof(double) * B));
  GSK_LAUNCHED(1);
  *used = 1;
  return GSK_OK;
}

// ---- GMRES(m) with MGS: the cycle of gmres.cu on the cluster ------------------------------
struct ClusterGmresArgs {
  CsrView csr;
  int n, B;
  const double *b, *w;
  double *x, *W, *hist;
  GmresState h;  // initial scalars (the arrays are replaced by shared-memory copies)
  GmresState* st_out;
};

template <bool SMEMW>
__global__ void __launch_bounds__(CL_T, 1) cluster_gmres(ClusterGmresArgs a) {
  extern __shared__ double wsm[];  // SMEMW: this CTA's rows of the m+1 basis vectors
  __shared__ GmresState st;
  __shared__ ClusterRed R;
  constexpr int M = CL_MMAX;
  constexpr int NARR = (M + 1) * M + 7 * M + 8;
  __shared__ double arr[NARR];
  const int n = a.n, r0 = (int)cg::this_cluster().block_rank() * a.B;
  const int m = a.h.m;
  for (int k = threadIdx.x; k < NARR; k += blockDim.x) arr[k] = 0.0;
  if (threadIdx.x == 0) {
    st = a.h;
    st.H = arr;  // (m+1) x m row-major with stride m, as in gmres.cu
    st.cs = arr + (M + 1) * M;
    st.sn = st.cs + M;
    st.g = st.sn + M;
    st.y = st.g + M + 1;
    st.inv = st.y + M;
    st.c1 = st.inv + M + 2;
    st.c2 = st.c1 + M;
  }
  __syncthreads();
  // basis slot j: global (stride n) or this CTA's shared block (stride B, base -r0)
  double* const W0 = SMEMW ? wsm - r0 : a.W;
  const size_t ws = SMEMW ? (size_t)a.B : (size_t)n;
  auto slot = [&](int j) { return W0 + (size_t)(j - 1) * ws; };
  int par = 0;
  cluster_pass<SMEMW>(a.csr, n, r0, a.B, OpGResid<LdCG>{a.x, a.b, a.w, slot(1), a.hist, &st, 1}, R, par);
  const long long maxc = (long long)st.maxit + 2;
  for (long long c = 0; c < maxc && !st.done; ++c) {
    for (int j = 1; j <= m && !st.done && !st.cycle_stop; ++j) {
      cluster_pass<SMEMW>(a.csr, n, r0, a.B, OpCgsS<LdCG>{slot(j), slot(j + 1), &st, j, 0}, R, par);
      cluster_pass<SMEMW>(a.csr, n, r0, a.B, OpH1{slot(j + 1), slot(1), &st, j, 0}, R, par);
      for (int i = 1; i < j; ++i)
        cluster_pass<SMEMW>(a.csr, n, r0, a.B, OpMgs{slot(i), slot(i + 1), slot(j + 1), &st, i, j, 0, 0, 0}, R, par);
      cluster_pass<SMEMW>(a.csr, n, r0, a.B, OpLast{slot(j), slot(j + 1), a.hist, &st, j, 0, 0}, R, par);
    }
    cluster_pass<SMEMW>(a.csr, n, r0, a.B, OpXupd<LdPlain>{W0, a.x, &st, ws, 0, nullptr, nullptr}, R, par);
    cluster_pass<SMEMW>(a.csr, n, r0, a.B, OpGResid<LdCG>{a.x, a.b, a.w, slot(1), a.hist, &st, 0}, R, par);
  }
  if (cg::this_cluster().block_rank() == 0) {
    if (threadIdx.x == 0) {  // scalars only (the report reads no arrays)
      GmresState o = st;
      o.H = a.h.H;
      o.cs = a.h.cs;
      o.sn = a.h.sn;
      o.g = a.h.g;
      o.y = a.h.y;
      o.inv = a.h.inv;
      o.c1 = a.h.c1;
      o.c2 = a.h.c2;
      *a.st_out = o;
    }
  }
  cg::this_cluster().sync();  // no CTA exits while another may still read its shared memory
}

int cluster_gmres_run(gsk_plan* P, const double* b, double* x, const GmresState& h, int* used) {
  *used = 0;
  const int n = P->A.n;
  int B = 0;
  const int cs = cluster_geometry(n, &B);
  if (!cs || h.m > CL_MMAX) return GSK_OK;
  constexpr size_t kWsm = 196 * 1024;  // basis in shared memory when it fits
  const size_t wbytes = sizeof(double) * (size_t)(h.m + 1) * B;
  const bool smemw = wbytes <= kWsm;
  static const char attr_key = 0;  // function attributes are per device
  if (!device_attr_done(&attr_key)) {
    GSK_CUDA(cudaFuncSetAttribute(cluster_gmres<false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    GSK_CUDA(cudaFuncSetAttribute(cluster_gmres<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    GSK_CUDA(cudaFuncSetAttribute(cluster_gmres<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kWsm));
    device_attr_mark(&attr_key);
  }
  ClusterGmresArgs a{P->csr, n, B, b, P->weights, x, P->W, P->hist_d, h, P->gstate};
  void* args[] = {&a};
  if (smemw)
    GSK_CUDA(launch_cluster(reinterpret_cast<const void*>(cluster_gmres<true>), cs, args, P->st, wbytes));
  else
    GSK_CUDA(launch_cluster(reinterpret_cast<const void*>(cluster_gmres<false>), cs, args, P->st));
  GSK_LAUNCHED(1);
  *used = 1;
  return GSK_OK;
}

}  // namespace gsk
