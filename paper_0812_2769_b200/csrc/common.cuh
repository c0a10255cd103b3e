// common.cuh — shared definitions of libgsk (sm_100a): matrix views, reduction
// bookkeeping and small helpers.  The pass engine itself is engine.cuh.
// Everything is memory-bound fp64 (no tensor cores: nothing is a dense
// contraction).  Kernels are compiled with --fmad=false; every FMA is an explicit
// __fma_rn (arithmetic contract AC-2).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gsk {

constexpr int TB = 256;         // threads per CTA = rows per sub-tile = SELL sigma
constexpr int SELL_C = 32;      // SELL chunk height (one warp)
constexpr int SELL_SIGMA = 256; // SELL sorting window
constexpr int SELLU_MAXL = 8;   // SELL-U: distinct column deltas per chunk (at most)
constexpr int RCD_MAXL = 8;      // row-class dictionary: entries per row (at most)
constexpr int RCD_MAXCLS = 4096; // ... and classes per plan (at most)
constexpr int CSR_CAP = 1792;   // entries of a 256-row CSR window staged in smem (7 per row)
constexpr int MAXD = 3;         // max dot products fused into one pass

struct CsrView {
  int n;
  const int* __restrict__ rp;
  const int* __restrict__ ci;
  const double* __restrict__ v;
};

// One row class (sell.cu, DESIGN.md §5 "RCD"): the entries shared by every row of the
// class, in CSR order — values and deltas col - row (unused places 0) — one 128-byte line.
// The deltas are packed in 8-byte words with the length, {len, d0} {d1, d2} {d3, d4}
// {d5, d6} {d7, 0}: a pass reads the line with warp-uniform 8-byte loads (one L1 wavefront
// each; a 16-byte load costs four), four of them for the deltas of rows of <= 7 entries.
struct __align__(128) RcdEntry {
  double v[RCD_MAXL];
  int2 ld[5];  // ld[0] = {len, d0}, ld[k] = {d(2k-1), d(2k)}, ld[4] = {d7, 0}
  int pad_[6];
};

// Stencil slots of a row-class plan (sell.cu): when the deltas of ALL classes form one
// symmetric set {-s_k .. -s_1, -1, 0, 1, s_1 .. s_k} (a 5- or 7-point stencil on a
// structured grid), a class is a presence mask and one value per delta of that set, in
// ascending delta (= CSR) order; the deltas themselves are plan constants.
struct __align__(128) RcdSlots {
  double v[RCD_MAXL];
  unsigned mask;  // bit k: the class has an entry at delta sdel[k]
  unsigned pad_[15];
};

// Row-class data of a plan (device-resident; SellView::rcd points at it when the plan's
// passes read the classes): the class of every row, the class lines and, when all
// classes share one stencil, the slots and the plan's deltas.
struct RcdView {
  const uint16_t* __restrict__ kcls;   // [n]
  const RcdEntry* __restrict__ kdict;  // [<= RCD_MAXCLS]
  const RcdSlots* __restrict__ kslots; // [<= RCD_MAXCLS] (null: the deltas differ between classes)
  int sdel[RCD_MAXL];                  // the plan's ascending deltas (ns of them: 5 or 7)
  int ns;
  int sroll;  // 1: sdel[ns/2 + 2] == 256, the same thread's row of the next window
};

// NOTE: exactly 128 bytes.  With a larger SellView nvcc 12.9 generates different (less
// unrolled) code for every SELL pass kernel — the plain SpMV went from 0.264 to 0.312 ms
// at C4 when two pointers were added here — so optional encodings hang off one pointer.
struct SellView {
  int n;
  int nchunks;
  int pad;  // column value of padding slots: -1, or INT_MIN in a shard plan, whose
            // remapped columns may be negative (left halo)
  int all_nat;  // every window keeps its natural row order (sell.cu; 0: use roff)
  int l2pf;  // > 0: a pass prefetches the matrix data of the window l2pf ahead into L2
  const int* __restrict__ cptr;     // [nchunks+1] slot offsets
  const int* __restrict__ scol;     // [nslots], pad = padding
  const double* __restrict__ sval;  // [nslots]
  const uint8_t* __restrict__ roff; // [nchunks*32] in-window row offset
  // optional column-index dictionary (null: scol is used): per slot a uint8 index into
  // the chunk's ascending distinct deltas col - row (255 = padding)
  const uint8_t* __restrict__ sidx;  // [nslots]
  const int* __restrict__ dptr;      // [nchunks+1]
  const int* __restrict__ dict;      // [ndict]
  // windows kept in natural row order (sell.cu): wid[w] = 1 when lane l of warp k of
  // window w holds row 32 k + l
  const uint8_t* __restrict__ wid;  // [nwindows]
  // optional chunk-uniform column offsets (SELL-U, sell.cu; null: not built): per chunk
  // SELLU_MAXL deltas col - row and lane masks, slot offsets and values of that layout
  const int* __restrict__ uptr;        // [nchunks+1]
  const int* __restrict__ udel;        // [nchunks * SELLU_MAXL]
  const unsigned* __restrict__ umask;  // [nchunks * SELLU_MAXL]
  const double* __restrict__ uval;     // [nuslots]
  // optional row-class dictionary (RCD, sell.cu; null: not built or inapplicable): the
  // passes then read no slot data
  const RcdView* __restrict__ rcd;
};
static_assert(sizeof(SellView) == 128, "SellView must stay 128 bytes (see the note above)");

// Programmatic dependent launch (PDL): every pass / finish kernel waits for the
// previous kernel's completion (and memory) at entry, then lets the next kernel of the
// stream begin launching, so launch latency overlaps the tail of the previous grid.
// Both are no-ops when the kernel was launched without the PDL attribute.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Gather-load policy of the ops that gather a vector at neighbouring columns.  The
// graph passes read vectors written by an EARLIER kernel: the read-only path is valid.
// A kernel that writes and re-reads its vectors (coop.cu across CTAs, small.cu in one
// CTA) must use a coherent load instead.
struct LdNC {
  static __device__ __forceinline__ double ld(const double* p) { return __ldg(p); }
};
struct LdCG {  // L2 (coherent across SMs after the grid barrier's release/acquire)
  static __device__ __forceinline__ double ld(const double* p) { return __ldcg(p); }
};
struct LdPlain {  // generic load: shared or global memory, coherent within a CTA
  static __device__ __forceinline__ double ld(const double* p) { return *p; }
};

// 8-byte asynchronous global -> shared copy (LDGSTS): no register round trip, so all
// of a thread's loads can be in flight at once; completion via cp_async_wait<N>.
__device__ __forceinline__ void cp_async8(double* smem, const double* g) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async4(int* smem, const int* g) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(g) : "memory");
}
// TMA bulk prefetch of [p, p + bytes) into L2 (cp.async.bulk.prefetch.L2): one thread,
// no registers, nothing to wait for.  The range is shrunk to 16-byte boundaries inside
// it (the start of every array here is 256-byte aligned).
__device__ __forceinline__ void prefetch_l2(const void* p, size_t bytes) {
  const uintptr_t a = (reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15);
  const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes) & ~uintptr_t(15);
  if (e > a)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((unsigned)(e - a)) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Store of a result no pass reads soon (x in Bi-CGSTAB S4): evict-first in L2.
__device__ __forceinline__ void st_cold(double* p, double v) {
#ifndef GSK_NO_EVICT
  __stcs(p, v);
#else
  *p = v;
#endif
}

__device__ __forceinline__ double ldcs(const double* p) { return __ldcs(p); }
__device__ __forceinline__ int ldcs(const int* p) { return __ldcs(p); }

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

}  // namespace gsk
