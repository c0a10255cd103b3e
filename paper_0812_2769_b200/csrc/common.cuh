// common.cuh — shared device machinery of libgsk (sm_100a).
//
// Everything here is memory-bound fp64: no tensor cores (nothing is a dense
// contraction).  The pieces:
//   * views of the two matrix formats (CSR, SELL-C-sigma with C=32, sigma=256);
//   * the row-tile engine: a CTA of 256 threads owns `sub` consecutive sub-tiles of
//     256 rows; each sub-tile is one SpMV pass (CSR rows staged through shared
//     memory with coalesced loads, or one SELL window = 8 chunks of 32 rows) and an
//     epilogue in canonical row order (thread t <-> row r0 + t);
//   * the canonical pairwise-tree reduction of the arithmetic contract (AC-5,
//     DESIGN.md §4): warp butterflies xor 1..16 are exactly the tree over 32
//     consecutive leaves, a fixed tree joins warps, sub-tiles and tiles, and the
//     last CTA to finish (atomic ticket) reduces the per-tile partials and runs the
//     scalar epilogue on the device (no host round trip per iteration).
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
constexpr int MAX_SUB = 64;     // max sub-tiles per CTA

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

// Reduction bookkeeping of one fused pass: per-tile partials of D dot products,
// laid out [d][ntiles], an arrival ticket, and the pow2 tile count.
struct Red {
  double* part;
  unsigned* ticket;
  int ntiles;
  int np2;
};

// Tile geometry of a launch.
struct Tiles {
  int n;
  int sub;  // sub-tiles (of 256 rows) per CTA, power of two
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

// In-place tree over len (pow2) values in shared memory, single thread.
__device__ __forceinline__ double serial_tree(double* a, int len) {
  for (int l = len; l > 1; l >>= 1)
    for (int i = 0; i < l / 2; ++i) a[i] = a[2 * i] + a[2 * i + 1];
  return a[0];
}

// Tree over the per-tile partials p[0..np2) (entries >= ntiles are +0), computed by
// the whole CTA.  Warp w owns the contiguous segment [w*seg, (w+1)*seg); it walks
// the segment 32 leaves at a time (butterfly = tree of 32) and lane 0 joins the
// 32-leaf trees with a binary counter, which for a pow2 count is exactly the tree.
template <int D>
__device__ void grid_tree(const Red& red, double (&out)[D], double* sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double v[D];
  if (red.np2 <= TB) {
#pragma unroll
    for (int d = 0; d < D; ++d)
      v[d] = threadIdx.x < red.ntiles ? __ldcg(red.part + (size_t)d * red.ntiles + threadIdx.x) : 0.0;
    block_tree<D>(v, sm);
  } else {
    const int seg = red.np2 / 8;
    double stk[D][16];
    int lvl[16];
    int sp = 0;
    for (int q = 0; q < seg; q += 32) {
      const int idx = warp * seg + q + lane;
      double u[D];
#pragma unroll
      for (int d = 0; d < D; ++d) {
        u[d] = idx < red.ntiles ? __ldcg(red.part + (size_t)d * red.ntiles + idx) : 0.0;
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
#pragma unroll
  for (int d = 0; d < D; ++d) out[d] = v[d] + 0.0;  // AC-5: T + 0.0 (pad-size independent)
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
// The fused pass.  Op provides:
//   static constexpr int D;                       number of fused dot products
//   bool begin();                                 load device scalars; false = uniform early exit
//   double gather(int col) const;                 x_col as seen by the SpMV
//   void row(int i, double y, double (&c)[D]);    canonical-order row epilogue
//   void finish(const double (&s)[D], int lane);  scalar epilogue (warp 0 of last CTA)
// Fmt: 0 = no SpMV (vector pass), 1 = CSR, 2 = SELL.
struct Smem {
  union {
    CsrStage csr;
    double sy[TB];
  } u;
  double red[MAXD * 8];
  double subp[MAXD * MAX_SUB];
  int last;
};

template <int FMT, class Op>
__global__ void __launch_bounds__(TB) fused_pass(CsrView csr, SellView sell, Tiles tl, Op op, Red red) {
  if (!op.begin()) return;
  constexpr int D = Op::D;
  __shared__ Smem sm;
  const int tile = blockIdx.x;
  for (int s = 0; s < tl.sub; ++s) {
    const int r0 = (tile * tl.sub + s) * TB;
    if (r0 < tl.n) {
      double y = 0.0;
      if constexpr (FMT == 1) y = csr_subtile(csr, r0, [&](int col) { return op.gather(col); }, sm.u.csr);
      if constexpr (FMT == 2) y = sell_subtile(sell, r0, [&](int col) { return op.gather(col); }, sm.u.sy);
      const int i = r0 + threadIdx.x;
      if constexpr (D > 0) {
        double cc[D];
#pragma unroll
        for (int d = 0; d < D; ++d) cc[d] = 0.0;
        if (i < tl.n) op.row(i, y, cc);
        block_tree<D>(cc, sm.red);
        if (threadIdx.x == 0) {
#pragma unroll
          for (int d = 0; d < D; ++d) sm.subp[d * MAX_SUB + s] = cc[d];
        }
      } else {
        double cc[1];
        if (i < tl.n) op.row(i, y, cc);
      }
    } else if constexpr (D > 0) {
      if (threadIdx.x == 0) {
#pragma unroll
        for (int d = 0; d < D; ++d) sm.subp[d * MAX_SUB + s] = 0.0;
      }
    }
  }
  if constexpr (D > 0) {
    if (threadIdx.x == 0) {
#pragma unroll
      for (int d = 0; d < D; ++d) red.part[(size_t)d * red.ntiles + tile] = serial_tree(sm.subp + d * MAX_SUB, tl.sub);
      __threadfence();
      sm.last = (atomicAdd(red.ticket, 1u) == gridDim.x - 1);
    }
    __syncthreads();
    if (!sm.last) return;
    __threadfence();
    double sums[D];
    grid_tree<D>(red, sums, sm.red);
    if (threadIdx.x < 32) op.finish(sums, threadIdx.x);
    if (threadIdx.x == 0) *red.ticket = 0u;
  }
}

}  // namespace gsk
