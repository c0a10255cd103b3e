// engine.cuh — the row-pass engine of libgsk (sm_100a).
//
// Every hot pass of the solvers is `pass_kernel<FMT, Op>` followed, when it reduces
// dot products, by `finish_kernel<Op>`:
//
//   pass_kernel   CTA of 256 threads owning `wpc` consecutive 256-row windows.
//                 SpMV passes (FMT 1 CSR, 2 SELL) compute y for each window (CSR rows
//                 staged through shared memory with coalesced loads; SELL chunks of
//                 32 rows, one per warp, scattered back to canonical row order), then
//                 the Op's row epilogue runs in canonical order (thread t <-> row t of
//                 the window) and yields the dot-product leaves.  Vector passes
//                 (FMT 0) give each thread one row of each window, all loads in
//                 flight together.  Warp trees of 32 leaves: per window in SpMV
//                 passes (two dots share the first level), one reduce-scatter over
//                 all of a thread's leaves in vector passes; warp 0 finishes the trees
//                 of 8 warps and the tree over the CTA's windows, and writes ONE
//                 partial per CTA.  No fences, no atomics: the CTA ends as soon as its
//                 stores are issued.  SpMV passes prefetch the next window's own-row
//                 operands into shared memory with cp.async.  Row-class plans (FMT 5:
//                 class lines; 6 / 7: stencil slots of 7 / 5 deltas; sell.cu) read a
//                 uint16 class id per row instead of the slot data: thread t finishes
//                 row r0 + t of every window, +-1 entries come from the adjacent lanes,
//                 +-256 ones from the thread's own rows of the neighbouring windows, and
//                 thread 0 bulk-prefetches the CTA's whole row block into L2.
//   finish_kernel one CTA of 1024 threads reduces the CTA partials with the same
//                 canonical tree (AC-5) and runs the Op's scalar
//                 epilogue (alpha, omega, Givens, stopping tests, ...) on the device.
//   mdot_pass     the CGS2 tile engine (thread = 8 consecutive rows), further below;
//                 finish_local/global_kernel: the shard-split finish (shard.cu).
//
// Shared-memory scatter buffers and CSR stages are double-buffered by window parity,
// so a window costs one __syncthreads.  Kernels are compiled with --fmad=false; every
// FMA is an explicit __fma_rn (AC-2).
#pragma once
#include <type_traits>
#include "common.cuh"

namespace gsk {

constexpr int FIN_THREADS = 1024;
constexpr int FIN_LEAVES = 8;                          // partials per finish thread (fixed)
constexpr int FIN_ROUND = FIN_THREADS * FIN_LEAVES;    // 8192 partials per round

struct CsrStage {
  double v[CSR_CAP];
  int c[CSR_CAP];
};

template <int FMT>
struct PassSmem;
template <>
struct PassSmem<0> {
  double wp[16 * MAXD * 8];  // [window][d][warp]
};
constexpr int ASYNC_NV = 2;  // own-row operands prefetched with cp.async (SpMV passes)
template <>
struct PassSmem<1> {
  CsrStage st[2];
  double wp[16 * MAXD * 8];
};
template <>
struct PassSmem<2> {
  double sy[2][TB];
  double wp[16 * MAXD * 8];
  double vin[2][ASYNC_NV][TB];
};
template <>
struct PassSmem<3> : PassSmem<2> {};
// SELL passes sized to the Op: cp.async slots only for the operands it prefetches (the
// 25% carveout then holds 4 CTAs of a one-operand pass instead of 3)
// (natural-order kernels never scatter: no sy buffer, 4 KB less per CTA)
template <int NVS, bool NAT = false>
struct PassSmemSell {
  double sy[2][NAT ? 1 : TB];
  double wp[16 * MAXD * 8];
  double vin[2][NVS][TB];
};
template <bool NAT>
struct PassSmemSell<0, NAT> {
  double sy[2][NAT ? 1 : TB];
  double wp[16 * MAXD * 8];
  double vin[2][1][1];
};
struct PassSmemDirect {  // direct passes use no shared memory
  double wp[1];
};

// Register budget per pass kind (CTAs per SM): SELL keeps 8 slots (col, val, x) in
// flight per lane, vector passes RPT rows of NV operands; CSR is bounded by its
// double-buffered 43 KB stage.
// Rows per thread of a vector pass with NV own-row operands (all loads in flight).
template <int NV>
struct VecRpt {
  static constexpr int value = NV <= 3 ? 8 : 4;
};

// SELL register budget per Op: 64 registers (4 CTAs/SM) unless the Op declares
// kSellMinBlocks = 3; only then are its own-row operands loaded before the SpMV
// (prefetching them at 64 registers spills).  Measured at C4: plain SpMV and the
// Bi-CGSTAB passes are fastest at 4 CTAs/SM, the GMRES Arnoldi pass at 3.
template <class Op, class = void>
struct SellTuning {
  static constexpr int minb = 4;
};
template <class Op>
struct SellTuning<Op, std::void_t<decltype(Op::kSellMinBlocks)>> {
  static constexpr int minb = Op::kSellMinBlocks;
};

#ifndef GSK_SELLD_DOT_MINB
#define GSK_SELLD_DOT_MINB 4
#endif
#ifndef GSK_SELL_DIRECT
#define GSK_SELL_DIRECT 1
#endif
constexpr bool SELL_DIRECT = GSK_SELL_DIRECT;

// column-index encoding of a SELL pass format: FMT 2 int32, 3 SELL-D, 4 SELL-U, 5 RCD
// (row-class dictionary: no slot data at all), 6 / 7 RCD with stencil slots (7 / 5 deltas)
template <int FMT>
struct SellIdx {
  static constexpr int value = FMT == 3 ? 1 : FMT == 4 ? 2 : FMT >= 5 ? 3 : 0;
};

#ifndef GSK_RCD_MINB
#define GSK_RCD_MINB 4
#endif
#ifndef GSK_SHORT_MINB
#define GSK_SHORT_MINB 5
#endif
template <int FMT, class Op, int MAXL = 8>
struct PassOcc {
  // SELL passes without dot products run "direct": each lane finishes
  // the row of its own SELL slot (operands, output) with no per-window barrier.
  // (Measured with dots too, leaves parked by row in shared memory and reduced once
  // per CTA: bit-exact, but S1 unchanged and S3 slower — 80 registers to not spill.)
  static constexpr bool kDirect = SELL_DIRECT && FMT >= 2 && Op::D == 0;
  static constexpr int kMinBlocks = FMT >= 5 ? GSK_RCD_MINB
                                  : FMT == 1 ? 4
                                  : FMT == 3 ? (Op::D > 0 && SellTuning<Op>::minb == 4 ? GSK_SELLD_DOT_MINB
                                                                                       : SellTuning<Op>::minb)
                                  : (FMT == 2 || FMT == 4)
                                      ? (MAXL <= 5 && SellTuning<Op>::minb == 4 ? GSK_SHORT_MINB : SellTuning<Op>::minb)
                                      : 3;
  static constexpr bool kPrefetch = FMT == 1 || (FMT >= 2 && SellTuning<Op>::minb < 4);
  // otherwise (SELL at 4 CTAs/SM, no registers to spare) up to ASYNC_NV own-row
  // operands of window w+1 are copied into shared memory with cp.async during window w
  static constexpr bool kAsync = !kPrefetch && FMT >= 2 && Op::NV >= 1 && Op::NV <= ASYNC_NV;
};

// y for row r0 + t of a CSR window (AC-3 chain), staged through st.
template <class G>
__device__ __forceinline__ double csr_window(const CsrView& A, int r0, const G& g, CsrStage& st) {
  const int t = threadIdx.x, r = r0 + t;
  const int rend = min(r0 + TB, A.n);
  const int s0 = A.rp[r0], s1 = A.rp[rend];
  const int cnt = s1 - s0;
  double acc = 0.0;
  if (cnt <= CSR_CAP) {  // uniform over the CTA
    for (int k = t; k < cnt; k += TB) {
      st.v[k] = __ldcs(A.v + s0 + k);
      st.c[k] = __ldcs(A.ci + s0 + k);
    }
    __syncthreads();
    if (r < A.n) {
      const int a = A.rp[r] - s0, b = A.rp[r + 1] - s0;
      for (int k = a; k < b; ++k) acc = __fma_rn(st.v[k], g(st.c[k]), acc);
    }
  } else if (r < A.n) {
    for (int k = A.rp[r]; k < A.rp[r + 1]; ++k) acc = __fma_rn(__ldcs(A.v + k), g(__ldcs(A.ci + k)), acc);
  }
  return acc;
}

// Row-class (RCD) SpMV of row `row` of class `cls` (row >= n: 0): the class line is read
// with warp-uniform 8-byte loads (nearly every lane of a warp has the same class: one L1
// wavefront per load), then all gathers, then the AC-3 chain in CSR order.
// Measured at C4 and not kept (profiles/r02_experiments): two or four windows in flight
// per thread (-10% / -35%: the pass is bound by the L1 data pipe, ncu lsu wavefronts
// 80-86%, not by latency); the class line kept in registers across windows with a warp
// vote (-20%) and the +-1 neighbours taken from the adjacent lanes by shuffle (wavefronts
// -35%, but 3.4x the instructions: issue-bound, -45%).
template <class G>
__device__ __forceinline__ double rcd_row(const RcdView& A, int n, int row, int cls, const G& g) {
  const RcdEntry* e = A.kdict + cls;
  const int2 q0 = __ldg(&e->ld[0]);
  const int L = row < n ? q0.x : 0;
  int ds[RCD_MAXL];
  double xs[RCD_MAXL];
  ds[0] = q0.y;
#pragma unroll
  for (int h = 1; h < 4; ++h) {
    const int2 q = __ldg(&e->ld[h]);
    ds[2 * h - 1] = q.x;
    ds[2 * h] = q.y;
  }
  ds[7] = L > 7 ? __ldg(&e->ld[4]).x : 0;
#pragma unroll
  for (int k = 0; k < RCD_MAXL; ++k)
    if (k < L) xs[k] = g(row + ds[k]);
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < RCD_MAXL; ++k)
    if (k < L) acc = __fma_rn(__ldg(&e->v[k]), xs[k], acc);
  return acc;
}

// Ops that gather one vector expose it (gathered()): the row-class passes prefetch it.
template <class Op, class = void>
struct OpGathers : std::false_type {};
template <class Op>
struct OpGathers<Op, std::void_t<decltype(std::declval<const Op&>().gathered())>> : std::true_type {};

#ifndef GSK_RCD_PF
#define GSK_RCD_PF 1
#endif
#ifndef GSK_RCD_LB
#define GSK_RCD_LB 1
#endif
#ifndef GSK_RCD_EXP
#define GSK_RCD_EXP 0  // timing probes of the stencil-slot row code (1, 2: wrong results; never in a build)
#endif
constexpr int RCD_LB = GSK_RCD_LB;  // windows whose dot-product leaves are reduced together (1, 2, 4)

// Row-class SpMV with stencil slots (RcdSlots: every class's deltas come from the plan's
// symmetric set sdel[0..NS), centre C = NS / 2 with sdel[C] = 0, sdel[C -+ 1] = -+1): no
// delta loads, and the gathers that neighbouring threads already hold come from registers
// instead of the L1 data pipe —
//   * delta -+1: the adjacent lane's own-row value g(row -+ 1) by shuffle (lanes 0 / 31
//     load theirs);
//   * with roll (sdel[C + 2] == 256 = the window height: a grid line is one window): the
//     entry at delta -+256 is this thread's own-row value of the previous / next window,
//     kept from / loaded for the neighbouring window (xlo / xhi valid when has_lo / has_hi).
// The values are the same loads of the same memory, the chain is ascending delta = CSR
// order (AC-3): bit-identical to every other format.
template <int NS, class G>
__device__ __forceinline__ double rcd_row_slots(const RcdView& A, int n, int row, int cls, const G& g, double own,
                                                bool has_lo, double xlo, bool has_hi, double xhi) {
  constexpr int C = NS / 2;
  const int lane = threadIdx.x & 31;
  const RcdSlots* e = A.kslots + cls;
  const unsigned mask = row < n ? __ldg(&e->mask) : 0u;
  auto bit = [&](int k) { return ((mask >> k) & 1u) != 0u; };
  double xs[NS];
  const double up = __shfl_up_sync(0xffffffffu, own, 1);
  const double dn = __shfl_down_sync(0xffffffffu, own, 1);
  xs[C] = own;
  xs[C - 1] = lane > 0 ? up : (bit(C - 1) ? g(row - 1) : 0.0);
  xs[C + 1] = lane < 31 ? dn : (bit(C + 1) ? g(row + 1) : 0.0);
  xs[C - 2] = has_lo ? xlo : (bit(C - 2) ? g(row + A.sdel[C - 2]) : 0.0);
  xs[C + 2] = has_hi ? xhi : (bit(C + 2) ? g(row + A.sdel[C + 2]) : 0.0);
  if constexpr (NS == 7) {
#if GSK_RCD_EXP == 1  // timing probe only (wrong results): no far-plane gathers
    xs[0] = own;
    xs[6] = own;
#else
    xs[0] = bit(0) ? g(row + A.sdel[0]) : 0.0;
    xs[6] = bit(6) ? g(row + A.sdel[6]) : 0.0;
#endif
  }
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < NS; ++k) {
#if GSK_RCD_EXP == 2  // timing probe only (wrong results): no class-value loads
    const double a = 1.0 + k;
#else
    const double a = __ldg(&e->v[k]);
#endif
    if (bit(k)) acc = __fma_rn(a, xs[k], acc);
  }
  return acc;
}

// SELL window core: lane l of warp w computes slot l of chunk r0/32 + w and hands the
// row's y with its in-window offset to sink(rl, y).  NAT: the window keeps its natural
// row order (sell.cu), so the slot's row is r0 + t and roff is not read.
// IDX: 0 int32 column per slot, 1 SELL-D (uint8 index into the chunk's delta
// dictionary), 2 SELL-U (chunk-uniform deltas: slot k of every lane at delta udel[k],
// lane masks mark padding; no per-slot column data at all).
template <int IDX, bool NAT = false, int MAXL = 8, class G, class S, class Pre>
__device__ __forceinline__ void sell_window_sink(const SellView& A, int r0, const G& g, const S& sink,
                                                 const Pre& pre) {
  constexpr bool DICT = IDX == 1;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int c = (r0 >> 5) + warp;
  if (c < A.nchunks) {
    const int rl = NAT ? (t & (TB - 1)) : A.roff[c * SELL_C + lane];
    pre(rl);
    if constexpr (IDX == 3) {  // RCD (row r0 + t)
      static_assert(NAT || IDX != 3, "row-class passes finish row r0 + t");
      const int row = r0 + rl;
      const RcdView R = *A.rcd;
      sink(rl, rcd_row(R, A.n, row, row < A.n ? (int)__ldg(R.kcls + row) : 0, g));
      return;
    }
    if constexpr (IDX == 2) {
      const int p0 = A.uptr[c], L = (A.uptr[c + 1] - p0) >> 5;  // <= SELLU_MAXL
      // lane k < L holds delta k and its lane mask (two 32-byte loads per chunk)
      const int dv = lane < SELLU_MAXL ? __ldg(A.udel + (size_t)c * SELLU_MAXL + lane) : 0;
      const unsigned mv = lane < SELLU_MAXL ? __ldg(A.umask + (size_t)c * SELLU_MAXL + lane) : 0u;
      const int row = r0 + rl;
      const double* vb = A.uval + p0 + lane;
      double vals[SELLU_MAXL], xs[SELLU_MAXL];
      unsigned ok = 0u;
#pragma unroll
      for (int k = 0; k < SELLU_MAXL; ++k)  // the slot values first (one streaming stream)
        if (k < L) vals[k] = __ldcs(vb + k * SELL_C);
#pragma unroll
      for (int k = 0; k < SELLU_MAXL; ++k)
        if (k < L) {
          const int d = __shfl_sync(0xffffffffu, dv, k);
          const unsigned m = __shfl_sync(0xffffffffu, mv, k);
          if ((m >> lane) & 1u) {
            ok |= 1u << k;
            xs[k] = g(row + d);
          }
        }
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < SELLU_MAXL; ++k)
        if (k < L && ((ok >> k) & 1u)) acc = __fma_rn(vals[k], xs[k], acc);
      sink(rl, acc);
      return;
    }
    const int p0 = A.cptr[c], L = (A.cptr[c + 1] - p0) >> 5;
    const int base = p0 + lane;
    double acc = 0.0;
    if (DICT && L <= 8) {
      // SELL-D: col = row + dict_c[idx] (1-byte index per slot instead of 4)
      const int d0 = A.dptr[c], U = A.dptr[c + 1] - d0;
      const int dv = lane < U ? __ldg(A.dict + d0 + lane) : 0;
      const int row = r0 + rl;
      int cols[8];
      double vals[8], xs[8];
#pragma unroll
      for (int k = 0; k < 8; ++k)  // all slot loads first (shuffles would serialise them)
        if (k < L) {
          cols[k] = __ldcs(A.sidx + base + k * SELL_C);
          vals[k] = __ldcs(A.sval + base + k * SELL_C);
        }
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k < L) {
          const int delta = __shfl_sync(0xffffffffu, dv, cols[k] & 31);
          cols[k] = cols[k] == 255 ? A.pad : row + delta;
        }
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k < L && cols[k] != A.pad) xs[k] = g(cols[k]);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k < L && cols[k] != A.pad) acc = __fma_rn(vals[k], xs[k], acc);
    } else if (L <= MAXL) {  // MAXL: the slot arrays kept in registers (8; 5 for 2-D plans)
      int cols[MAXL];
      double vals[MAXL], xs[MAXL];
#pragma unroll
      for (int k = 0; k < MAXL; ++k)
        if (k < L) {
          cols[k] = __ldcs(A.scol + base + k * SELL_C);
          vals[k] = __ldcs(A.sval + base + k * SELL_C);
        }
#pragma unroll
      for (int k = 0; k < MAXL; ++k)
        if (k < L && cols[k] != A.pad) xs[k] = g(cols[k]);
#pragma unroll
      for (int k = 0; k < MAXL; ++k)
        if (k < L && cols[k] != A.pad) acc = __fma_rn(vals[k], xs[k], acc);
    } else {
      for (int k = 0; k < L; ++k) {  // long chunks: plain int32 columns (kept in every plan)
        const int col = __ldcs(A.scol + base + k * SELL_C);
        if (col != A.pad) acc = __fma_rn(__ldcs(A.sval + base + k * SELL_C), g(col), acc);
      }
    }
    sink(rl, acc);
  }
}

// L2 prefetch (TMA bulk, thread 0 of the CTA) of the matrix data of the window starting
// at row r0: the slot values and the column data of its chunks in the pass's encoding.
// It gives the window's streaming loads an L2 latency instead of a DRAM one without
// holding registers.
template <int IDX>
__device__ __forceinline__ void sell_prefetch_window(const SellView& A, int r0) {
  const int c0 = r0 >> 5;
  if (c0 >= A.nchunks) return;
  if constexpr (IDX == 3) {  // the window's class ids (512 bytes)
    prefetch_l2(A.rcd->kcls + r0, sizeof(uint16_t) * (size_t)min(TB, A.n - r0));
    return;
  }
  const int c1 = min(c0 + TB / SELL_C, A.nchunks);
  const int* ptr = IDX == 2 ? A.uptr : A.cptr;
  const int s0 = ptr[c0], s1 = ptr[c1];
  const double* vals = IDX == 2 ? A.uval : A.sval;
  prefetch_l2(vals + s0, sizeof(double) * (size_t)(s1 - s0));
  if constexpr (IDX == 0) prefetch_l2(A.scol + s0, sizeof(int) * (size_t)(s1 - s0));
  if constexpr (IDX == 1) prefetch_l2(A.sidx + s0, (size_t)(s1 - s0));
  if constexpr (IDX == 2) {
    prefetch_l2(A.udel + (size_t)c0 * SELLU_MAXL, sizeof(int) * SELLU_MAXL * (size_t)(c1 - c0));
    prefetch_l2(A.umask + (size_t)c0 * SELLU_MAXL, sizeof(unsigned) * SELLU_MAXL * (size_t)(c1 - c0));
  }
}

// ... scattering y to sy at its in-window offset (no barrier).
template <int IDX, class G>
__device__ __forceinline__ void sell_window_store(const SellView& A, int r0, const G& g, double* sy) {
  sell_window_sink<IDX>(A, r0, g, [&](int rl, double y) { sy[rl] = y; }, [](int) {});
}

// y for row r0 + t of a SELL window (scatter through sy, one barrier).
template <int IDX, class G>
__device__ __forceinline__ double sell_window(const SellView& A, int r0, const G& g, double* sy) {
  sell_window_store<IDX>(A, r0, g, sy);
  __syncthreads();
  return sy[threadIdx.x];
}

// ... of a natural-order window: thread t computes row r0 + t itself (no scatter, no
// barrier; 0 beyond the last chunk).
template <int IDX, int MAXL = 8, class G>
__device__ __forceinline__ double sell_window_nat(const SellView& A, int r0, const G& g) {
  double y = 0.0;
  sell_window_sink<IDX, true, MAXL>(A, r0, g, [&](int, double v) { y = v; }, [](int) {});
  return y;
}


// Op::kEvict (optional): bit k set = own-row operand vin(k) is not read by the NEXT
// pass, so the register-path load of it is evict-first (ld.global.cs) and
// leaves L2 to the vectors the next pass reads (pass order).
#ifndef GSK_NO_EVICT
template <class Op, class = void>
struct OpEvict {
  static constexpr unsigned value = 0;
};
template <class Op>
struct OpEvict<Op, std::void_t<decltype(Op::kEvict)>> {
  static constexpr unsigned value = Op::kEvict;
};
#else
template <class Op>
struct OpEvict {
  static constexpr unsigned value = 0;
};
#endif

// Own-row operands of the Op for row i.
template <class Op>
__device__ __forceinline__ void load_vin(const Op& op, int i, double (&v)[Op::NV > 0 ? Op::NV : 1]) {
#pragma unroll
  for (int k = 0; k < Op::NV; ++k) {
    const double* src = op.vin(k);
    v[k] = src ? (((OpEvict<Op>::value >> k) & 1u) ? __ldcs(src + i) : __ldg(src + i)) : 0.0;
  }
}

// Warp butterflies of one window's leaves (= trees of 32 leaves); lane 0 records the
// warp's value.  Two dots share the first level: even lanes keep dot 0, odd lanes dot
// 1 (each lane adds its partner's value of the dot it keeps: the same pairs (2i, 2i+1)
// and IEEE addition commutes), so a pair costs 6 shuffles instead of 10.
template <int D>
__device__ __forceinline__ void warp_leaves(double (&c)[D], double* wp, int w) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if constexpr (D == 2) {
    const bool odd = lane & 1;
    const double give = odd ? c[0] : c[1];
    const double keep = odd ? c[1] : c[0];
    double u = keep + __shfl_xor_sync(0xffffffffu, give, 1);
#pragma unroll
    for (int off = 2; off < 32; off <<= 1) u = u + __shfl_xor_sync(0xffffffffu, u, off);
    if (lane < 2) wp[(w * MAXD + lane) * 8 + warp] = u;
  } else {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
#pragma unroll
      for (int d = 0; d < D; ++d) c[d] = c[d] + __shfl_xor_sync(0xffffffffu, c[d], off);
    }
    if (lane == 0) {
#pragma unroll
      for (int d = 0; d < D; ++d) wp[(w * MAXD + d) * 8 + warp] = c[d];
    }
  }
}

// The same warp trees for all RPT x D leaves of a vector pass at once, as a
// reduce-scatter: at level l (partner lane ^ 2^l) every lane keeps half of its
// remaining values and adds its partner's copies of them (the canonical pairs, IEEE
// addition commutes), so K = RPT * D values cost K/2 + K/4 + ... + 1 shuffles, then the
// remaining levels one each, instead of 5 K.  Afterwards lane l (l < K) holds value
// bitreverse(l) of the K (window-major, dot-minor), which it records.
template <int RPT, int D>
__device__ __forceinline__ void warp_leaves_multi(double (&c)[RPT][D], double* wp) {
  constexpr int K0 = RPT * D;
  constexpr int K = K0 <= 1 ? 1 : K0 <= 2 ? 2 : K0 <= 4 ? 4 : K0 <= 8 ? 8 : K0 <= 16 ? 16 : 32;
  static_assert(K0 <= 32, "at most 32 leaves per lane");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double v[K];
#pragma unroll
  for (int q = 0; q < K; ++q) v[q] = q < K0 ? c[q / D][q % D] : 0.0;
  int off = 1;
#pragma unroll
  for (int len = K; len > 1; len >>= 1, off <<= 1) {
    const bool hi = lane & off;
#pragma unroll
    for (int q = 0; q < len / 2; ++q) {
      const double send = hi ? v[q] : v[q + len / 2];
      const double keep = hi ? v[q + len / 2] : v[q];
      v[q] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  double u = v[0];
#pragma unroll
  for (; off < 32; off <<= 1) u = u + __shfl_xor_sync(0xffffffffu, u, off);
  if (lane < K) {
    int idx = 0;  // the value this lane kept: bit l of the lane selects the upper half at level l
#pragma unroll
    for (int b = 0, h = K / 2; h >= 1; ++b, h >>= 1)
      if (lane & (1 << b)) idx += h;
    if (idx < K0) wp[((idx / D) * MAXD + idx % D) * 8 + warp] = u;
  }
}

// Warp 0, after a __syncthreads: lane w builds window w's tree over its 8 warp values,
// a butterfly over lanes 0..WMAX-1 joins the windows pairwise, lane 0 writes the CTA
// partial.  Windows beyond nw (pow2 <= WMAX) enter as +0 leaves: x + 0 = x, and the
// final + 0.0 of AC-5 canonicalises a zero's sign.
constexpr int WMAX = 16;  // windows per CTA (SpMV passes, GSK_WPC)
template <int D>
__device__ __forceinline__ void cta_partial(const double* wp, int nw, double* part, int stride, int slot) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    double u = 0.0;
    if (lane < nw) {
      const double* v = wp + (lane * MAXD + d) * 8;
      u = ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
    }
#pragma unroll
    for (int off = 1; off < WMAX; off <<= 1) u = u + __shfl_xor_sync(0xffffffffu, u, off);
    if (lane == 0) part[(size_t)d * stride + slot] = u;
  }
}

// FMT 0: vector pass, RPT windows (rows r0 + 256 w + t) per CTA, all loads in flight.
// FMT 1/2/3/4: SpMV pass over wpc windows (CSR, SELL, SELL-D, SELL-U); FMT 5/6/7: over the
// plan's row classes (class lines / stencil slots of 7 / 5 deltas).
// NAT (SELL only): every window of the plan keeps its natural row order (sell.cu), so
// thread t computes row r0 + t itself — no roff, no scatter, no per-window barrier.
// A compile-time choice: one code path per kernel keeps the 64-register budget.
// MAXL (plain SELL): slots per lane kept in registers; 5 for plans whose chunks are all
// at most 5 long (the 2-D 5-point systems), which frees registers for more CTAs per SM.
template <int FMT, int RPT, class Op, bool NAT = false, int MAXL = 8>
__global__ void __launch_bounds__(TB, PassOcc<FMT, Op, MAXL>::kMinBlocks)
    pass_kernel(CsrView csr, SellView sell, int n, int wpc, Op op, double* part, int stride, int rev) {
  pdl_enter();
  if (!op.begin()) return;
  // rev: CTAs take their row blocks in descending order (the tile's partial keeps its
  // slot, so the reduction tree is unchanged).  Consecutive passes alternate the
  // direction, so a pass starts on the rows whose vectors the previous pass touched
  // last, which are still in L2.
  const int bx = rev ? (int)gridDim.x - 1 - (int)blockIdx.x : (int)blockIdx.x;
  constexpr int D = Op::D;
  constexpr int DD = D > 0 ? D : 1;
  constexpr int NVA = Op::NV > 0 ? Op::NV : 1;
  constexpr bool kDirect = PassOcc<FMT, Op>::kDirect;
  using Smem = std::conditional_t<
      (FMT >= 5), PassSmemSell<0, true>,
      std::conditional_t<
      kDirect, PassSmemDirect,
      std::conditional_t<(FMT >= 2), PassSmemSell<(PassOcc<FMT, Op>::kAsync ? Op::NV : 0), NAT>, PassSmem<FMT>>>>;
  __shared__ __align__(16) Smem sm;
  const int t = threadIdx.x, warp = t >> 5;
  if constexpr (FMT >= 5) {
    // RCD: thread t finishes row r0 + t of every window; own-row operands in registers;
    // the class id of the next window is loaded while this one computes.  FMT 6 / 7: the
    // plan's classes share one 7- / 5-delta stencil (rcd_row_slots).
    constexpr int NS = FMT == 6 ? 7 : FMT == 7 ? 5 : 0;
    const int rb = bx * wpc * TB;
    const RcdView R = *sell.rcd;  // (device-resident: SellView itself must stay 128 bytes)
    // A thread has one row in flight, so its loads that miss L2 (its own rows of the
    // streamed vectors, the class ids, the far plane first touched by this CTA) would each
    // cost a DRAM latency per window: thread 0 asks for all of them at once — TMA bulk L2
    // prefetches of the CTA's whole row block (no registers, nothing to wait for)
    if (GSK_RCD_PF && t == 0 && rb < n) {
      const int rows = min(wpc * TB, n - rb);
      prefetch_l2(R.kcls + rb, sizeof(uint16_t) * (size_t)rows);
#pragma unroll
      for (int k = 0; k < Op::NV; ++k)
        if (op.vin(k)) prefetch_l2(op.vin(k) + rb, sizeof(double) * (size_t)rows);
      if constexpr (OpGathers<Op>::value) {
        const double* gx = op.gathered();
        prefetch_l2(gx + rb, sizeof(double) * (size_t)rows);
        if constexpr (NS > 0) {
          const int far = R.sdel[NS - 1];  // the outermost deltas -+far: one of the two
          // planes is first touched by this CTA (which one depends on the pass direction)
          if (rb + far < n) prefetch_l2(gx + rb + far, sizeof(double) * (size_t)min(rows, n - rb - far));
          if (rb - far >= 0) prefetch_l2(gx + rb - far, sizeof(double) * (size_t)rows);
        }
      }
    }
    int kn = rb + t < n ? (int)__ldg(R.kcls + rb + t) : 0;
    auto g = [&](int col) { return op.gather(col); };
    const bool roll = NS > 0 && R.sroll != 0;
    double own_prev = 0.0, own_cur = 0.0, own_next = 0.0;
    // one window: y of row r0 + t, the Op's row epilogue, the dot-product leaves in cc
    auto window = [&](int w, double (&cc)[DD]) {
      const int r0 = rb + w * TB;
#pragma unroll
      for (int d = 0; d < DD; ++d) cc[d] = 0.0;
      if (r0 < n) {  // uniform over the CTA
        const int i = r0 + t;
        const int kc = kn;
        double v[NVA];
        if (i < n) load_vin(op, i, v);
        kn = (w + 1 < wpc && i + TB < n) ? (int)__ldg(R.kcls + i + TB) : 0;
        double y;
        if constexpr (NS > 0) {
          const bool more = w + 1 < wpc && i + TB < n;  // this thread's row of the next window
          if (!roll || w == 0) own_cur = i < n ? g(i) : 0.0;
          if (roll) own_next = more ? g(i + TB) : 0.0;
          y = rcd_row_slots<NS>(R, n, i, kc, g, own_cur, roll && w > 0, own_prev, roll && more, own_next);
          own_prev = own_cur;
          own_cur = own_next;
        } else {
          y = rcd_row(R, n, i, kc, g);
        }
        if (i < n) op.row(i, y, v, cc);
      }
    };
    if (D > 0 && RCD_LB > 1 && wpc >= RCD_LB) {
      // the leaves of RCD_LB windows are reduced together: one reduce-scatter (K/2 + K/4 +
      // ... shuffles instead of 5 per value) and one dependent chain per RCD_LB windows
      for (int w0 = 0; w0 < wpc; w0 += RCD_LB) {
        double cb[RCD_LB][DD];
#pragma unroll
        for (int j = 0; j < RCD_LB; ++j) window(w0 + j, cb[j]);
        if constexpr (D > 0) warp_leaves_multi<RCD_LB, DD>(cb, sm.wp + (size_t)w0 * MAXD * 8);
      }
    } else {
      for (int w = 0; w < wpc; ++w) {
        double cc[DD];
        window(w, cc);
        if constexpr (D > 0) warp_leaves<D>(cc, sm.wp, w);
      }
    }
    if constexpr (D > 0) {
      __syncthreads();
      if (warp == 0) cta_partial<D>(sm.wp, wpc, part, stride, bx);
    }
  } else if constexpr (kDirect) {
    const int rb = bx * wpc * TB;
    if (sell.l2pf && wpc >= 4 && threadIdx.x == 0)
      for (int q = 1; q <= sell.l2pf && q < wpc; ++q) sell_prefetch_window<SellIdx<FMT>::value>(sell, rb + q * TB);
    for (int w = 0; w < wpc; ++w) {
      const int r0 = rb + w * TB;
      if (r0 >= n) break;  // uniform over the CTA
      if (sell.l2pf && wpc >= 4 && threadIdx.x == 0 && w + sell.l2pf + 1 < wpc)
        sell_prefetch_window<SellIdx<FMT>::value>(sell, r0 + (sell.l2pf + 1) * TB);
      auto g = [&](int col) { return op.gather(col); };
      double v[NVA];
      auto sink = [&](int rl, double y) {
        double cc[1];
        if (r0 + rl < n) op.row(r0 + rl, y, v, cc);
      };
      auto pre = [&](int rl) {  // own-row operands in flight during the row's SpMV
        if (r0 + rl < n) load_vin(op, r0 + rl, v);
      };
      sell_window_sink<SellIdx<FMT>::value, NAT, MAXL>(sell, r0, g, sink, pre);
    }
  } else if constexpr (FMT == 0) {
    const int r0 = bx * (TB * RPT);
    double v[RPT][NVA];
#pragma unroll
    for (int w = 0; w < RPT; ++w) {
      const int i = r0 + w * TB + t;
      if (i < n) load_vin(op, i, v[w]);
    }
    double cc[RPT][DD];
#pragma unroll
    for (int w = 0; w < RPT; ++w) {
      const int i = r0 + w * TB + t;
#pragma unroll
      for (int d = 0; d < DD; ++d) cc[w][d] = 0.0;
      if (i < n) op.row(i, 0.0, v[w], cc[w]);
    }
    if constexpr (D > 0) {
      warp_leaves_multi<RPT, D>(cc, sm.wp);
      __syncthreads();
      if (warp == 0) cta_partial<D>(sm.wp, RPT, part, stride, bx);
    }
  } else {
    const int rb = bx * wpc * TB;
    constexpr bool kPre = PassOcc<FMT, Op>::kPrefetch;
    constexpr bool kAsync = PassOcc<FMT, Op>::kAsync;
    // own-row operands of window w -> sm.vin[w & 1] (one commit group per window; each
    // thread copies and later reads only its own slots, so no barrier is involved)
    auto issue = [&](int w) {
      if constexpr (kAsync) {
        const int i = rb + w * TB + t;
        if (w < wpc && i < n) {
#pragma unroll
          for (int k = 0; k < Op::NV; ++k) {
            const double* src = op.vin(k);
            if (src) cp_async8(&sm.vin[w & 1][k][t], src + i);
          }
        }
        cp_async_commit();
      }
    };
    issue(0);
    if constexpr (FMT >= 2) {
      if (sell.l2pf && wpc >= 4 && threadIdx.x == 0)
        for (int q = 1; q <= sell.l2pf && q < wpc; ++q) sell_prefetch_window<SellIdx<FMT>::value>(sell, rb + q * TB);
    }
    for (int w = 0; w < wpc; ++w) {
      const int r0 = rb + w * TB;
      if constexpr (FMT >= 2) {
        if (sell.l2pf && wpc >= 4 && threadIdx.x == 0 && w + sell.l2pf + 1 < wpc && r0 < n)
          sell_prefetch_window<SellIdx<FMT>::value>(sell, r0 + (sell.l2pf + 1) * TB);
      }
      double cc[DD];
#pragma unroll
      for (int d = 0; d < DD; ++d) cc[d] = 0.0;
      issue(w + 1);
      if (r0 < n) {  // uniform over the CTA
        auto g = [&](int col) { return op.gather(col); };
        const int i = r0 + t;
        double v[NVA];
        if (kPre && i < n) load_vin(op, i, v);  // own-row operands in flight during the SpMV
        double y;
        if constexpr (FMT == 1) y = csr_window(csr, r0, g, sm.st[w & 1]);
        else if constexpr (NAT) y = sell_window_nat<SellIdx<FMT>::value, MAXL>(sell, r0, g);
        else y = sell_window<SellIdx<FMT>::value>(sell, r0, g, sm.sy[w & 1]);
        if constexpr (kAsync) {
          cp_async_wait<1>();  // all groups but window w+1's are complete
#pragma unroll
          for (int k = 0; k < Op::NV; ++k) v[k] = (i < n && op.vin(k)) ? sm.vin[w & 1][k][t] : 0.0;
        } else if (!kPre && i < n) {
          load_vin(op, i, v);
        }
        if (i < n) op.row(i, y, v, cc);
      }
      if constexpr (D > 0) warp_leaves<D>(cc, sm.wp, w);
    }
    if constexpr (D > 0) {
      __syncthreads();
      if (warp == 0) cta_partial<D>(sm.wp, wpc, part, stride, bx);
    }
  }
}

// One CTA: canonical tree over ntiles CTA partials, + 0.0, then the Op's scalar
// epilogue on warp 0.  The partials are zero-padded to a multiple of 8192 (trailing
// +0 leaves never change a tree value beyond the sign of a zero, which the final
// + 0.0 canonicalises): thread t owns leaves [8t, 8t+8) of each 8192-leaf round
// (four 16-byte loads), a register tree of 8, warp butterflies, a tree of 32
// warps, and a binary counter joins the rounds in order.  Skipped exactly when the
// pass was skipped (op.begin() reads the same device flags; only finish kernels
// change them).
// Canonical tree of D dot products over ntiles CTA partials (+ 0.0), valid in warp 0
// (every lane).  Body of the finish kernels; blockDim = FIN_THREADS.
// One round of LV partials per thread over the canonical tree (no round loop):
// thread t's LV leaves, a register tree, warp butterflies, the tree of 32 warps.
template <int D, int LV>
__device__ __forceinline__ void fin_one_round(const double* part, int stride, int ntiles, double (&s)[D]) {
  __shared__ double wsr[D][32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int base = t * LV;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    double l[LV];
    if (base + LV <= ntiles) {
      const double2* q = reinterpret_cast<const double2*>(part + (size_t)d * stride + base);
#pragma unroll
      for (int h = 0; h < LV / 2; ++h) {
        const double2 x = q[h];
        l[2 * h] = x.x;
        l[2 * h + 1] = x.y;
      }
    } else {
#pragma unroll
      for (int q = 0; q < LV; ++q) l[q] = base + q < ntiles ? part[(size_t)d * stride + base + q] : 0.0;
    }
#pragma unroll
    for (int len = LV; len > 1; len >>= 1) {
#pragma unroll
      for (int q = 0; q < len / 2; ++q) l[q] = l[2 * q] + l[2 * q + 1];
    }
    double u = l[0];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) u = u + __shfl_xor_sync(0xffffffffu, u, off);
    if (lane == 0) wsr[d][warp] = u;
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      double x = wsr[d][lane];
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) x = x + __shfl_xor_sync(0xffffffffu, x, off);
      s[d] = x + 0.0;
    }
  }
}

template <int D>
__device__ __forceinline__ void fin_tree(const double* part, int stride, int ntiles, double (&s)[D]) {
  // up to 16384 partials (vector passes with 4 rows per thread at C4): one round of
  // 16 leaves per thread instead of two rounds joined by the binary counter
  if (ntiles > FIN_ROUND && ntiles <= 2 * FIN_ROUND) {
    fin_one_round<D, 2 * FIN_LEAVES>(part, stride, ntiles, s);
    return;
  }
  __shared__ double ws[D][32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  double stk[D][12];
  int lvl[12];
  int sp = 0;
  const int rounds = (ntiles + FIN_ROUND - 1) / FIN_ROUND;
  int rp2 = 1;  // rounds padded to a power of two (zero rounds contribute +0)
  while (rp2 < rounds) rp2 <<= 1;
  for (int r = 0; r < rp2; ++r) {
    double u[D];
    const int base = r * FIN_ROUND + t * FIN_LEAVES;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      double l[FIN_LEAVES];
      if (base + FIN_LEAVES <= ntiles) {
        const double2* q = reinterpret_cast<const double2*>(part + (size_t)d * stride + base);
#pragma unroll
        for (int h = 0; h < FIN_LEAVES / 2; ++h) {
          const double2 x = q[h];
          l[2 * h] = x.x;
          l[2 * h + 1] = x.y;
        }
      } else {
#pragma unroll
        for (int q = 0; q < FIN_LEAVES; ++q) l[q] = base + q < ntiles ? part[(size_t)d * stride + base + q] : 0.0;
      }
      u[d] = ((l[0] + l[1]) + (l[2] + l[3])) + ((l[4] + l[5]) + (l[6] + l[7]));
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) u[d] = u[d] + __shfl_xor_sync(0xffffffffu, u[d], off);
    }
    __syncthreads();
    if (lane == 0) {
#pragma unroll
      for (int d = 0; d < D; ++d) ws[d][warp] = u[d];
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
      for (int d = 0; d < D; ++d) {
        double x = ws[d][lane];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) x = x + __shfl_xor_sync(0xffffffffu, x, off);
        u[d] = x;
      }
      if (rp2 == 1) {
#pragma unroll
        for (int d = 0; d < D; ++d) stk[d][0] = u[d];
      } else if (lane == 0) {
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
  }
  if (warp == 0) {
#pragma unroll
    for (int d = 0; d < D; ++d) s[d] = __shfl_sync(0xffffffffu, stk[d][0], 0) + 0.0;
  }
}

template <class Op>
__global__ void __launch_bounds__(FIN_THREADS) finish_kernel(Op op, const double* part, int stride,
                                                             int ntiles) {
  pdl_enter();
  if (!op.begin()) return;
  double s[Op::D];
  fin_tree<Op::D>(part, stride, ntiles, s);
  if (threadIdx.x < 32) op.finish(s, threadIdx.x);
}

// Row-block shards: each shard's finish writes its canonical subtree
// values (the shard's rows are an aligned power-of-two block of the global tree) ...
template <class Op>
__global__ void __launch_bounds__(FIN_THREADS) finish_local_kernel(Op op, const double* part, int stride,
                                                                   int ntiles, double* out) {
  pdl_enter();
  if (!op.begin()) return;
  double s[Op::D];
  fin_tree<Op::D>(part, stride, ntiles, s);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int d = 0; d < Op::D; ++d) out[d] = s[d];
  }
}

// ... and one warp joins the P shard values (gath[r * MAXD + d], P a power of two <= 32)
// with the top levels of the same tree, + 0.0, then runs the Op's scalar epilogue.
template <class Op>
__global__ void __launch_bounds__(32) finish_global_kernel(Op op, const double* gath, int P) {
  pdl_enter();
  if (!op.begin()) return;
  const int lane = threadIdx.x;
  double s[Op::D];
#pragma unroll
  for (int d = 0; d < Op::D; ++d) {
    double u = lane < P ? gath[lane * MAXD + d] : 0.0;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) u = u + __shfl_xor_sync(0xffffffffu, u, off);
    s[d] = u + 0.0;
  }
  op.finish(s, lane);
}

// Device-initiated shard reductions (shard.cu, gsk_shard_opts.peer_reduce).  Every
// process owns one buffer, [2][P][MAXD] doubles (epoch parity, shard, dot), then P
// uint64 epoch flags, then P uint64 epoch counters (its own shards'), and holds
// pointers to every process's buffer (CUDA IPC mappings; its own for local shards).
__host__ __device__ __forceinline__ unsigned long long* peer_flags(double* buf, int P) {
  return reinterpret_cast<unsigned long long*>(buf + 2 * (size_t)P * MAXD);
}
// ... each shard's finish stores its subtree values into every buffer's slot for this
// epoch's parity, then releases its flag (system scope) with the epoch number ...
template <class Op>
__global__ void __launch_bounds__(FIN_THREADS) finish_peer_local_kernel(Op op, const double* part, int stride,
                                                                        int ntiles, double* const* peers, int P,
                                                                        int me, unsigned long long* ep) {
  pdl_enter();
  if (!op.begin()) return;
  double s[Op::D];
  fin_tree<Op::D>(part, stride, ntiles, s);
  if (threadIdx.x == 0) {
    const unsigned long long e = *ep + 1;
    *ep = e;
    const int par = (int)(e & 1ull);
    for (int q = 0; q < P; ++q) {
      volatile double* g = peers[q] + ((size_t)par * P + me) * MAXD;
#pragma unroll
      for (int d = 0; d < Op::D; ++d) g[d] = s[d];
    }
    __threadfence_system();
    for (int q = 0; q < P; ++q) {
      unsigned long long* f = peer_flags(peers[q], P) + me;
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(e) : "memory");
    }
  }
}
// ... and one warp acquires the P flags of the epoch (lane q spins on flag q), reads the
// P values, joins them with the top of the canonical tree (+ 0.0) and runs the epilogue.
// Epochs advance identically on every process (the same reductions in the same order),
// and a value slot is rewritten two epochs later, after its reader has passed.
template <class Op>
__global__ void __launch_bounds__(32) finish_peer_global_kernel(Op op, double* own, int P,
                                                                const unsigned long long* ep) {
  pdl_enter();
  if (!op.begin()) return;
  const int lane = threadIdx.x;
  const unsigned long long e = *ep;
  const int par = (int)(e & 1ull);
  if (lane < P) {
    const unsigned long long* f = peer_flags(own, P) + lane;
    for (;;) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
      if (v >= e) break;
      __nanosleep(32);
    }
  }
  __syncwarp();
  const volatile double* g = own + ((size_t)par * P + (lane < P ? lane : 0)) * MAXD;
  double s[Op::D];
#pragma unroll
  for (int d = 0; d < Op::D; ++d) {
    double u = lane < P ? g[d] : 0.0;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) u = u + __shfl_xor_sync(0xffffffffu, u, off);
    s[d] = u + 0.0;
  }
  op.finish(s, lane);
}

// ---------------------------------------------------------------------------------
// Multi-dot passes (GMRES with double classical Gram-Schmidt): J
// dot products per row, J known at launch (<= MDOT_MAX).  A CTA owns tpc tiles of
// 2048 rows; in a tile thread t owns the 8 CONSECUTIVE rows 8t .. 8t+7, so each dot's
// 8 leaves of a thread are a canonical subtree reduced in registers, the warp
// butterfly extends it to 256 rows and warps' values (parked in smem) to 2048 — one
// butterfly per dot per 2048 rows instead of per 256, and every operand access is a
// 64-byte contiguous run per thread (16-byte loads).  SpMV ops scatter the SELL
// windows of the tile through smem first.  Op provides
//   bool begin(); int nd; double gather(int) (SpMV ops);
//   void value8(int i0, int cnt, const double (&y)[8], double (&u)[8])  rows i0.. (+cnt valid):
//        stores the rows' new w, returns u = w (0 for invalid rows)
//   void operand8(int i0, int cnt, int d, u, double (&v)[8])  -> operand d at rows i0..i0+7
//   void store(int d, double value)  or, with kWarpFinish, finish_warp(value, lane)
// The per-dot finish is mdot_finish<Op> with J CTAs.
constexpr int MDOT_MAX = 64;
#ifndef GSK_MDOT_MINB
#define GSK_MDOT_MINB 5
#endif
#ifndef GSK_MDOT_G
#define GSK_MDOT_G 1
#endif
constexpr int MDOT_MINB = GSK_MDOT_MINB;  // CTAs per SM (register budget)
constexpr int MDOT_G = GSK_MDOT_G;        // dots whose operand loads are in flight together
constexpr int MD_R = 8;                   // consecutive rows per thread
constexpr int MD_TILE = TB * MD_R;        // rows per tile (2048)

// 8 consecutive doubles at p (cnt of them valid): four 16-byte loads when possible.
__device__ __forceinline__ void ld8(const double* p, int cnt, double (&v)[8]) {
  if (cnt == 8 && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
    const double2* q = reinterpret_cast<const double2*>(p);
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const double2 x = __ldg(q + h);
      v[2 * h] = x.x;
      v[2 * h + 1] = x.y;
    }
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = k < cnt ? __ldg(p + k) : 0.0;
  }
}
__device__ __forceinline__ void st8(double* p, int cnt, const double (&v)[8]) {
  if (cnt == 8 && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
    double2* q = reinterpret_cast<double2*>(p);
#pragma unroll
    for (int h = 0; h < 4; ++h) q[h] = make_double2(v[2 * h], v[2 * h + 1]);
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (k < cnt) p[k] = v[k];
  }
}
__device__ __forceinline__ double tree8(const double (&a)[8]) {
  return ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
}

struct MdotSmem {
  double sy[MD_TILE];        // SpMV results of the tile in row order
  double wp[MDOT_MAX * 8];   // [dot][warp]
  double tp[8 * MDOT_MAX];   // [tile][dot]
};

template <int FMT, class Op>
__global__ void __launch_bounds__(TB, MDOT_MINB)
    mdot_pass(CsrView csr, SellView sell, int n, int tpc, Op op, double* part, int stride, int rev) {
  pdl_enter();
  if (!op.begin()) return;
  __shared__ __align__(16) MdotSmem sm;
  const int bx = rev ? (int)gridDim.x - 1 - (int)blockIdx.x : (int)blockIdx.x;  // as pass_kernel
  const int J = op.nd;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  for (int tl = 0; tl < tpc; ++tl) {
    const int r0 = (bx * tpc + tl) * MD_TILE;
    if (r0 >= n) {  // uniform: an all-padding tile
      for (int d = t; d < J; d += TB) sm.tp[tl * MDOT_MAX + d] = 0.0;
      continue;
    }
    const int i0 = r0 + MD_R * t;
    const int cnt = max(0, min(MD_R, n - i0));
    double y[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) y[k] = 0.0;
    if constexpr (Op::kSpmv) {
      auto g = [&](int col) { return op.gather(col); };
      if constexpr (FMT == 2) {
        for (int w = 0; w < MD_R; ++w)
          if (r0 + w * TB < n) sell_window_store<0>(sell, r0 + w * TB, g, sm.sy + w * TB);
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 8; ++k) y[k] = sm.sy[MD_R * t + k];
      } else {  // CSR (stencils: short rows), AC-3 chain per row
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (k < cnt) {
            const int i = i0 + k;
            double acc = 0.0;
            for (int q = csr.rp[i]; q < csr.rp[i + 1]; ++q) acc = __fma_rn(__ldcs(csr.v + q), g(__ldcs(csr.ci + q)), acc);
            y[k] = acc;
          }
      }
    }
    double u[8];
    op.value8(i0, cnt, y, u);
    for (int d0 = 0; d0 < J; d0 += MDOT_G) {
      double q[MDOT_G];
      double v[MDOT_G][8];
#pragma unroll
      for (int e = 0; e < MDOT_G; ++e)  // MDOT_G operand runs in flight
        if (d0 + e < J) op.operand8(i0, cnt, d0 + e, u, v[e]);
#pragma unroll
      for (int e = 0; e < MDOT_G; ++e) {
        double pr[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) pr[k] = u[k] * v[e][k];
        q[e] = d0 + e < J ? tree8(pr) : 0.0;
      }
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
#pragma unroll
        for (int e = 0; e < MDOT_G; ++e)
          if (d0 + e < J) q[e] = q[e] + __shfl_xor_sync(0xffffffffu, q[e], off);  // J uniform
      }
      if (lane == 0) {
#pragma unroll
        for (int e = 0; e < MDOT_G; ++e)
          if (d0 + e < J) sm.wp[(d0 + e) * 8 + warp] = q[e];
      }
    }
    __syncthreads();
    for (int d = t; d < J; d += TB) {
      double a[8];
#pragma unroll
      for (int w = 0; w < 8; ++w) a[w] = sm.wp[d * 8 + w];
      sm.tp[tl * MDOT_MAX + d] = tree8(a);
    }
    __syncthreads();  // sy / wp are rewritten by the next tile
  }
  for (int d = t; d < J; d += TB) {
    double a[8];
#pragma unroll
    for (int w = 0; w < 8; ++w) a[w] = w < tpc ? sm.tp[w * MDOT_MAX + d] : 0.0;
    part[(size_t)d * stride + bx] = tree8(a);
  }
}

// Tree of one CTA over ntiles partials p[0..ntiles) (as finish_kernel), result in warp 0.
__device__ __forceinline__ double cta_tree(const double* p, int ntiles) {
  __shared__ double ws[32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  double stk[12];
  int lvl[12];
  int sp = 0;
  const int rounds = (ntiles + FIN_ROUND - 1) / FIN_ROUND;
  int rp2 = 1;
  while (rp2 < rounds) rp2 <<= 1;
  double res = 0.0;
  for (int r = 0; r < rp2; ++r) {
    const int base = r * FIN_ROUND + t * FIN_LEAVES;
    double l[FIN_LEAVES];
#pragma unroll
    for (int q = 0; q < FIN_LEAVES; ++q) l[q] = base + q < ntiles ? p[base + q] : 0.0;
    double u = ((l[0] + l[1]) + (l[2] + l[3])) + ((l[4] + l[5]) + (l[6] + l[7]));
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) u = u + __shfl_xor_sync(0xffffffffu, u, off);
    __syncthreads();
    if (lane == 0) ws[warp] = u;
    __syncthreads();
    if (warp == 0) {
      double x = ws[lane];
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) x = x + __shfl_xor_sync(0xffffffffu, x, off);
      if (rp2 == 1) {
        res = x;
      } else if (lane == 0) {
        stk[sp] = x;
        lvl[sp] = 0;
        ++sp;
        while (sp >= 2 && lvl[sp - 1] == lvl[sp - 2]) {
          stk[sp - 2] = stk[sp - 2] + stk[sp - 1];
          lvl[sp - 2] += 1;
          --sp;
        }
      }
    }
  }
  if (warp == 0 && rp2 > 1) res = __shfl_sync(0xffffffffu, lane == 0 ? stk[0] : 0.0, 0);
  return res + 0.0;  // AC-5
}

template <class Op, class = void>
struct MdotWarpFinish : std::false_type {};
template <class Op>
struct MdotWarpFinish<Op, std::void_t<decltype(Op::kWarpFinish)>> : std::true_type {};

// Dot d = blockIdx.x of a multi-dot pass: canonical tree over the CTA partials, then
// op.store(d, value) by thread 0 (or the Op's warp-wide epilogue).
template <class Op>
__global__ void __launch_bounds__(FIN_THREADS) mdot_finish(Op op, const double* part, int stride, int ntiles) {
  pdl_enter();
  if (!op.begin()) return;
  const double v = cta_tree(part + (size_t)blockIdx.x * stride, ntiles);
  if constexpr (MdotWarpFinish<Op>::value) {
    if (threadIdx.x < 32) op.finish_warp(v, threadIdx.x);  // valid in warp 0
  } else if (threadIdx.x == 0) {
    op.store(blockIdx.x, v);
  }
}

}  // namespace gsk
