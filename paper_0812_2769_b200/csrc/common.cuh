// common.cuh — shared device machinery of libgsk (sm_100a).
//
// Everything here is memory-bound fp64: no tensor cores (nothing is a dense
// contraction).  The pieces:
//   * views of the two matrix formats (CSR, SELL-C-sigma with C=32, sigma=256);
//   * the row-tile engine: a CTA of 256 threads owns 256 consecutive rows; it runs
//     the SpMV of its rows (CSR rows staged through shared memory with coalesced
//     loads, or one SELL window = 8 chunks of 32 rows) and an epilogue in canonical
//     row order (thread t <-> row r0 + t);
//   * the canonical pairwise-tree reduction of the arithmetic contract (AC-5,
//     DESIGN.md §4): warp butterflies xor 1..16 are exactly the tree over 32
//     consecutive leaves, a fixed tree joins warps; the last CTA of each group of
//     256 tiles (atomic ticket) reduces the group, the last group reduces the groups
//     and runs the scalar epilogue on the device (no host round trip per iteration).
// Kernels are compiled with --fmad=false; every FMA is an explicit __fma_rn (AC-2).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gsk {

constexpr int TB = 256;         // threads per CTA = rows per sub-tile = SELL sigma
constexpr int SELL_C = 32;      // SELL chunk height (one warp)
constexpr int SELL_SIGMA = 256; // SELL sorting window
constexpr int CSR_CAP = 2048;   // entries of a 256-row CSR sub-tile staged in smem
constexpr int MAXD = 3;         // max dot products fused into one pass

struct CsrView {
  int n;
  const int* __restrict__ rp;
  const int* __restrict__ ci;
  const double* __restrict__ v;
};

struct SellView {
  int n;
  int nchunks;
  const int* __restrict__ cptr;     // [nchunks+1] slot offsets
  const int* __restrict__ scol;     // [nslots], -1 = padding
  const double* __restrict__ sval;  // [nslots]
  const uint8_t* __restrict__ roff; // [nchunks*32] in-window row offset
};

// Reduction bookkeeping of one fused pass.  Tile = 256 rows = one CTA; group = 256
// consecutive tiles (65536 rows).  The last CTA of a group (ticket) reduces the
// group's tile partials; the last group reduces the group partials and runs the
// scalar epilogue.  Every level is an aligned power-of-two block of the canonical
// tree, so the result is the contract's T(q) (+0.0).
struct Red {
  double* part;       // [D][ntiles] tile partials
  double* gpart;      // [D][ngroups] group partials
  unsigned* gticket;  // [ngroups] arrivals per group (self-resetting)
  unsigned* ticket;   // arrivals of groups (self-resetting)
  int ntiles;
  int ngroups;
  int gnp2;           // ngroups rounded up to a power of two
};

// Tile geometry of a launch.
struct Tiles {
  int n;
};

__device__ __forceinline__ double ldcs(const double* p) { return __ldcs(p); }
__device__ __forceinline__ int ldcs(const int* p) { return __ldcs(p); }

// ---------------------------------------------------------------------------------
// Canonical tree over the 256 values held by a CTA (thread t holds leaf t).
// Returns the tree value in every lane of warp 0 (valid in thread 0).
template <int D>
__device__ __forceinline__ void block_tree(double (&v)[D], double* sm /*[D*8]*/) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
#pragma unroll
    for (int d = 0; d < D; ++d) v[d] = v[d] + __shfl_xor_sync(0xffffffffu, v[d], off);
  }
  __syncthreads();  // sm may still be read by a previous call
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

// Tree over cnt partials p[d*stride + i] padded with +0 to np2 (pow2), computed by
// the whole CTA.  np2 <= 256: one leaf per thread.  Otherwise warp w owns the
// contiguous segment [w*seg, (w+1)*seg), walks it 32 leaves at a time (butterfly =
// tree of 32) and lane 0 joins the 32-leaf trees with a binary counter, which for a
// pow2 count is exactly the tree; a tree of 8 joins the warps.
template <int D>
__device__ void array_tree(const double* p, int stride, int cnt, int np2, double (&v)[D], double* sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (np2 <= TB) {
#pragma unroll
    for (int d = 0; d < D; ++d) v[d] = threadIdx.x < cnt ? __ldcg(p + (size_t)d * stride + threadIdx.x) : 0.0;
    block_tree<D>(v, sm);
    return;
  }
  const int seg = np2 / 8;
  double stk[D][20];
  int lvl[20];
  int sp = 0;
  for (int q = 0; q < seg; q += 32) {
    const int idx = warp * seg + q + lane;
    double u[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      u[d] = idx < cnt ? __ldcg(p + (size_t)d * stride + idx) : 0.0;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) u[d] = u[d] + __shfl_xor_sync(0xffffffffu, u[d], off);
    }
    if (lane == 0) {
#pragma unroll
      for (int d = 0; d < D; ++d) stk[d][sp] = u[d];
      lvl[sp] = 0;
      ++sp;
      while (sp >= 2 && lvl[sp - 1] == lvl[sp - 2]) {
#pragma unroll
        for (int d = 0; d < D; ++d) stk[d][sp - 2] = stk[d][sp - 2] + stk[d][sp - 1];
        lvl[sp - 2] += 1;
        --sp;
      }
    }
  }
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int d = 0; d < D; ++d) sm[d * 8 + warp] = stk[d][0];
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

// ---------------------------------------------------------------------------------
// One CSR sub-tile: returns y_{r0+t} = sum_k val_k G(col_k) (AC-3 chain) for thread t.
struct CsrStage {
  double v[CSR_CAP];
  int c[CSR_CAP];
};

template <class G>
__device__ __forceinline__ double csr_subtile(const CsrView& A, int r0, const G& g, CsrStage& st) {
  const int t = threadIdx.x, r = r0 + t;
  const int rend = min(r0 + TB, A.n);
  const int s0 = A.rp[r0], s1 = A.rp[rend];
  const int cnt = s1 - s0;
  double acc = 0.0;
  if (cnt <= CSR_CAP) {
    for (int k = t; k < cnt; k += TB) {
      st.v[k] = ldcs(A.v + s0 + k);
      st.c[k] = ldcs(A.ci + s0 + k);
    }
    __syncthreads();
    if (r < A.n) {
      const int a = A.rp[r] - s0, b = A.rp[r + 1] - s0;
      for (int k = a; k < b; ++k) acc = __fma_rn(st.v[k], g(st.c[k]), acc);
    }
    __syncthreads();
  } else if (r < A.n) {
    for (int k = A.rp[r]; k < A.rp[r + 1]; ++k) acc = __fma_rn(ldcs(A.v + k), g(ldcs(A.ci + k)), acc);
  }
  return acc;
}

// One SELL window (8 chunks of 32 rows = 256 rows starting at r0, r0 % 256 == 0):
// lane l of warp w computes the row in slot l of chunk r0/32 + w, the result is
// scattered to sy[] at the row's in-window offset and read back in canonical order.
template <class G>
__device__ __forceinline__ double sell_subtile(const SellView& A, int r0, const G& g, double* sy) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int c = (r0 >> 5) + warp;
  if (c < A.nchunks) {
    const int rl = A.roff[c * SELL_C + lane];
    const int p0 = A.cptr[c], L = (A.cptr[c + 1] - p0) >> 5;
    const int base = p0 + lane;
    double acc = 0.0;
    if (L <= 8) {
      int cols[8];
      double vals[8], xs[8];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k < L) { cols[k] = ldcs(A.scol + base + k * SELL_C); vals[k] = ldcs(A.sval + base + k * SELL_C); }
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k < L && cols[k] >= 0) xs[k] = g(cols[k]);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k < L && cols[k] >= 0) acc = __fma_rn(vals[k], xs[k], acc);
    } else {
      for (int k = 0; k < L; ++k) {
        const int col = ldcs(A.scol + base + k * SELL_C);
        if (col >= 0) acc = __fma_rn(ldcs(A.sval + base + k * SELL_C), g(col), acc);
      }
    }
    sy[rl] = acc;
  }
  __syncthreads();
  const double y = sy[t];
  __syncthreads();
  return y;
}

// ---------------------------------------------------------------------------------
// The fused pass: CTA b owns rows [256 b, 256 b + 256).  Op provides:
//   static constexpr int D;                       number of fused dot products
//   bool begin();                                 load device scalars; false = uniform early exit
//   double gather(int col) const;                 x_col as seen by the SpMV
//   void row(int i, double y, double (&c)[D]);    canonical-order row epilogue
//   void finish(const double (&s)[D], int lane);  scalar epilogue (warp 0 of the last CTA)
// FMT: 0 = no SpMV (vector pass), 1 = CSR, 2 = SELL.
template <int FMT>
struct Smem;
template <>
struct Smem<0> {
  double wres[8 * 2 * 8];  // [window][d][warp], D <= 2 for vector passes
  double red[MAXD * 8];
  int last;
};
template <>
struct Smem<1> {
  CsrStage csr;
  double red[MAXD * 8];
  int last;
};
template <>
struct Smem<2> {
  double sy[TB];
  double red[MAXD * 8];
  int last;
};

// Register budget: SELL keeps 8 slots of (col, val, x) in flight per lane; 64
// registers allow 4 CTAs (1024 threads) per SM.  CSR / vector passes fit 32-40.
template <int FMT>
struct Occ {
  static constexpr int kMinBlocks = FMT == 2 ? 3 : 4;
};

// Thread 0 holds the tile partial tp[D].  Tile partials -> group partials (last CTA
// of each group of 256 tiles) -> scalars (last group) -> op.finish on warp 0.
template <int D, class Op>
__device__ __forceinline__ void tickets_and_finish(const Op& op, const double (&tp)[D], const Red& red,
                                                   double* smred, int& smlast) {
  const int tile = blockIdx.x, g = tile >> 8;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int d = 0; d < D; ++d) red.part[(size_t)d * red.ntiles + tile] = tp[d];
    __threadfence();
    const int gsize = min(TB, red.ntiles - (g << 8));
    smlast = (atomicAdd(red.gticket + g, 1u) == (unsigned)(gsize - 1));
  }
  __syncthreads();
  if (!smlast) return;
  __threadfence();
  double gv[D];
  array_tree<D>(red.part + ((size_t)g << 8), red.ntiles, min(TB, red.ntiles - (g << 8)), TB, gv, smred);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int d = 0; d < D; ++d) red.gpart[(size_t)d * red.ngroups + g] = gv[d];
    red.gticket[g] = 0u;
    __threadfence();
    smlast = (atomicAdd(red.ticket, 1u) == (unsigned)(red.ngroups - 1));
  }
  __syncthreads();
  if (!smlast) return;
  __threadfence();
  double sums[D];
  array_tree<D>(red.gpart, red.ngroups, red.ngroups, red.gnp2, sums, smred);
#pragma unroll
  for (int d = 0; d < D; ++d) sums[d] = sums[d] + 0.0;  // AC-5: T + 0.0 (pad-size independent)
  if (threadIdx.x < 32) op.finish(sums, threadIdx.x);
  if (threadIdx.x == 0) *red.ticket = 0u;
}

// Tree over SUB (pow2) values, registers, compile-time unrolled.
template <int SUB, int D>
__device__ __forceinline__ void reg_tree(double (&v)[SUB][D]) {
#pragma unroll
  for (int len = SUB; len > 1; len >>= 1) {
#pragma unroll
    for (int q = 0; q < len / 2; ++q) {
#pragma unroll
      for (int d = 0; d < D; ++d) v[q][d] = v[2 * q][d] + v[2 * q + 1][d];
    }
  }
}

// SpMV passes: a CTA owns SUB_S consecutive 256-row windows (processed in turn);
// vector passes: SUB_V windows, thread t owning rows r0 + t + 256 s of every window,
// all rows' loads in flight together.
constexpr int SUB_S = 4;
constexpr int SUB_V = 8;

template <int FMT, class Op>
__global__ void __launch_bounds__(TB, Occ<FMT>::kMinBlocks)
    fused_pass(CsrView csr, SellView sell, Tiles tl, Op op, Red red) {
  if (!op.begin()) return;
  constexpr int D = Op::D;
  constexpr int DD = D > 0 ? D : 1;
  __shared__ Smem<FMT> sm;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if constexpr (FMT == 0) {
    const int r0 = blockIdx.x * (TB * SUB_V);
    double cc[SUB_V][DD];
#pragma unroll
    for (int s = 0; s < SUB_V; ++s) {
#pragma unroll
      for (int d = 0; d < DD; ++d) cc[s][d] = 0.0;
      const int i = r0 + s * TB + threadIdx.x;
      if (i < tl.n) op.row(i, 0.0, cc[s]);
    }
    if constexpr (D > 0) {
      // leaf t of window s sits in thread t: butterflies = trees of 32 leaves
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
#pragma unroll
        for (int s = 0; s < SUB_V; ++s) {
#pragma unroll
          for (int d = 0; d < D; ++d) cc[s][d] = cc[s][d] + __shfl_xor_sync(0xffffffffu, cc[s][d], off);
        }
      }
      if (lane == 0) {
#pragma unroll
        for (int s = 0; s < SUB_V; ++s) {
#pragma unroll
          for (int d = 0; d < D; ++d) sm.wres[(s * D + d) * 8 + warp] = cc[s][d];
        }
      }
      __syncthreads();
      double tp[D];
      if (warp == 0) {
#pragma unroll
        for (int s = 0; s < SUB_V; ++s) {
#pragma unroll
          for (int d = 0; d < D; ++d) {
            double u = lane < 8 ? sm.wres[(s * D + d) * 8 + lane] : 0.0;
            u = u + __shfl_xor_sync(0xffffffffu, u, 1);
            u = u + __shfl_xor_sync(0xffffffffu, u, 2);
            u = u + __shfl_xor_sync(0xffffffffu, u, 4);
            cc[s][d] = u;
          }
        }
        reg_tree<SUB_V, DD>(cc);
      }
#pragma unroll
      for (int d = 0; d < D; ++d) tp[d] = cc[0][d];
      tickets_and_finish<D>(op, tp, red, sm.red, sm.last);
    }
  } else {
    const int rb = blockIdx.x * (TB * SUB_S);
    double wp[SUB_S][DD];
#pragma unroll
    for (int s = 0; s < SUB_S; ++s) {
      const int r0 = rb + s * TB;
#pragma unroll
      for (int d = 0; d < DD; ++d) wp[s][d] = 0.0;
      if (r0 < tl.n) {  // uniform over the CTA
        double y = 0.0;
        if constexpr (FMT == 1) y = csr_subtile(csr, r0, [&](int col) { return op.gather(col); }, sm.csr);
        if constexpr (FMT == 2) y = sell_subtile(sell, r0, [&](int col) { return op.gather(col); }, sm.sy);
        const int i = r0 + threadIdx.x;
        double cc[DD];
#pragma unroll
        for (int d = 0; d < DD; ++d) cc[d] = 0.0;
        if (i < tl.n) op.row(i, y, cc);
        if constexpr (D > 0) {
          block_tree<D>(cc, sm.red);
#pragma unroll
          for (int d = 0; d < D; ++d) wp[s][d] = cc[d];
        }
      }
    }
    if constexpr (D > 0) {
      reg_tree<SUB_S, DD>(wp);
      double tp[D];
#pragma unroll
      for (int d = 0; d < D; ++d) tp[d] = wp[0][d];
      tickets_and_finish<D>(op, tp, red, sm.red, sm.last);
    }
  }
}

}  // namespace gsk
