// stream.cuh — the persistent, TMA-pipelined row-tile engine (sm_100a).
//
// Every hot pass of the solvers (SpMV passes and vector passes) streams its
// matrix slots and own-row vectors through shared memory with 1-D bulk TMA copies
// (cp.async.bulk ... mbarrier::complete_tx) issued by one producer warp, while 8
// consumer warps (256 threads, thread t <-> row t of a 256-row window) compute:
//
//   producer (warp 8, lane 0)            consumers (warps 0..7)
//   for tile in my tiles:                for tile in my tiles:
//     wait empty[s]                        wait full[s]
//     meta[s] = ranges / flags             y = SpMV rows from stage s (gathers: global/L2)
//     expect_tx(full[s], bytes)            own-row operands from stage s
//     bulk copies -> stage s               release stage s (arrive empty[s])
//                                          canonical tree of the tile -> tickets -> finish
//
// CTAs are persistent: CTA b owns the contiguous tiles [b*tpc, (b+1)*tpc), tpc a
// power of two, at most 256 CTAs (<= 2 per SM), so CTA launch cost is paid once, the
// next tiles' bytes are in flight while a tile is reduced, and the CTA's partial is
// an aligned block of the canonical tree (one ticket per CTA, not per tile).  Streams that do
// not fit a stage (rows too long, unaligned tails) fall back to direct global loads
// for that tile; results are identical either way (same operands, same order).
// The reduction is the canonical tree of AC-5 exactly as in
// common.cuh, with consumer-only named barriers.
#pragma once
#include "common.cuh"

namespace gsk {

constexpr int ST_CW = 8;                  // consumer warps
constexpr int ST_THREADS = 32 * (ST_CW + 1);
constexpr int ST_NST = 3;                 // pipeline depth
constexpr int ST_STAGE = 32768;           // bytes per stage
constexpr int ST_SLOTS = 2048;            // SELL slots / CSR entries staged per window
constexpr int ST_MAXNV = 8;               // own-row vectors per pass

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// Bounded wait: a protocol bug traps (kernel error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t ok = 0;
  for (uint32_t spin = 0;; ++spin) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    if (ok) return;
    if (spin > (1u << 26)) __trap();
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// Canonical tree over the 256 consumer threads (named barrier version of block_tree).
template <int D>
__device__ __forceinline__ void cblock_tree(double (&v)[D], double* sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
#pragma unroll
    for (int d = 0; d < D; ++d) v[d] = v[d] + __shfl_xor_sync(0xffffffffu, v[d], off);
  }
  consumer_sync();
  if (lane == 0) {
#pragma unroll
    for (int d = 0; d < D; ++d) sm[d * 8 + warp] = v[d];
  }
  consumer_sync();
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

// Per-stage metadata written by the producer before it arrives on full[s].
struct StageMeta {
  int mat;    // matrix streams staged (SpMV passes)
  int vmask;  // bit k: own-row vector k staged
  int base;   // CSR: first staged entry; SELL: chunk_ptr of the window's first chunk
  int cp[9];  // SELL: chunk_ptr of the window's chunks
};

struct StSmem {
  uint64_t full[ST_NST];
  uint64_t empty[ST_NST];
  StageMeta meta[ST_NST];
  double sy[TB];
  double red[MAXD * 8];
  double wres[2][8 * 2 * 8];  // [tile parity][window*D + d][warp]
  int last;
};

// Rows per tile of a vector pass with NV staged vectors: largest pow2 number of
// 256-row windows (<= 8) whose NV vectors fit one stage.
template <int NV>
struct VecTile {
  static constexpr int raw = NV > 0 ? ST_STAGE / (NV * 8 * TB) : 8;
  static constexpr int W = raw >= 8 ? 8 : raw >= 4 ? 4 : raw >= 2 ? 2 : 1;
};

// Stage layout (bytes): SELL [sval 2048*8][scol 2048*4][roff 256][vec k: 256*8];
// CSR [val 2056*8][col 2056*4][vec k: 256*8]; vector pass [vec k: rows*8].
template <int FMT>
struct Layout {
  static constexpr int SCOL = FMT == 2 ? ST_SLOTS * 8 : (ST_SLOTS + 8) * 8;
  static constexpr int ROFF = ST_SLOTS * 12;
  static constexpr int VEC = FMT == 2 ? ST_SLOTS * 12 + 256 : FMT == 1 ? (ST_SLOTS + 8) * 12 : 0;
  static constexpr int NVCAP = FMT == 0 ? ST_MAXNV : (ST_STAGE - VEC) / (TB * 8);
};
static_assert(Layout<2>::NVCAP >= 3 && Layout<1>::NVCAP >= 3, "stage too small");
static_assert(8 * 2 * 8 >= 3 * 8, "wres holds SpMV passes with D <= 3");

// Binary counter over the CTA's tile partials, fed in tile order by thread 0: for a
// pow2 number of pushes it yields exactly the pairwise tree of the CTA's range.
template <int D>
struct TileCounter {
  double stk[D][16];
  int lvl[16];
  int sp = 0;
  __device__ __forceinline__ void push(const double (&v)[D]) {
#pragma unroll
    for (int d = 0; d < D; ++d) stk[d][sp] = v[d];
    lvl[sp] = 0;
    ++sp;
    while (sp >= 2 && lvl[sp - 1] == lvl[sp - 2]) {
#pragma unroll
      for (int d = 0; d < D; ++d) stk[d][sp - 2] = stk[d][sp - 2] + stk[d][sp - 1];
      lvl[sp - 2] += 1;
      --sp;
    }
  }
};

// After the CTA's last tile: publish its partial, take a ticket; the last CTA reduces
// the (<= 256) CTA partials with the canonical tree and runs op.finish on warp 0.
template <int D, class Op>
__device__ __forceinline__ void cta_finish(const Op& op, const double (&cp)[D], const Red& red, StSmem& sm) {
  if (threadIdx.x == 0) {
#pragma unroll
    for (int d = 0; d < D; ++d) red.part[d * 256 + blockIdx.x] = cp[d];
    __threadfence();
    sm.last = (atomicAdd(red.ticket, 1u) == gridDim.x - 1);
  }
  consumer_sync();
  if (!sm.last) return;
  __threadfence();
  double v[D];
#pragma unroll
  for (int d = 0; d < D; ++d) v[d] = threadIdx.x < gridDim.x ? __ldcg(red.part + d * 256 + threadIdx.x) : 0.0;
  cblock_tree<D>(v, sm.red);
#pragma unroll
  for (int d = 0; d < D; ++d) v[d] = v[d] + 0.0;  // AC-5: T + 0.0 (pad-size independent)
  if (threadIdx.x < 32) op.finish(v, threadIdx.x);
  if (threadIdx.x == 0) *red.ticket = 0u;
}

// FMT: 0 vector pass, 1 CSR SpMV, 2 SELL SpMV.  Tiles: SpMV = one 256-row window;
// vector pass = VecTile<NV>::W windows.  Op additionally provides
//   static constexpr int NV;  const double* vin(int k) const;   (own-row operands)
//   void row(int i, double y, const double (&v)[NV], double (&c)[D]);
template <int FMT, class Op>
__global__ void __launch_bounds__(ST_THREADS, 2)
    stream_pass(CsrView csr, SellView sell, int n, int ntiles, Op op, Red red) {
  if (!op.begin()) return;
  constexpr int D = Op::D;
  constexpr int DD = D > 0 ? D : 1;
  constexpr int NV = Op::NV;
  constexpr int NVA = NV > 0 ? NV : 1;
  constexpr int W = FMT == 0 ? VecTile<NV>::W : 1;
  constexpr int ROWS = W * TB;
  constexpr int NVCAP = Layout<FMT>::NVCAP;
  extern __shared__ __align__(128) uint8_t dyn[];
  __shared__ StSmem sm;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST_NST; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], ST_CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int t_begin = blockIdx.x * red.tpc;
  const int t_end = min(t_begin + red.tpc, ntiles);
  // ------------------------------------------------------------- producer warp
  if (warp == ST_CW) {
    if (lane != 0) return;
    int it = 0;
    for (int tile = t_begin; tile < t_end; ++tile, ++it) {
      const int s = it % ST_NST;
      const uint32_t ph = (it / ST_NST) & 1;
      mbar_wait(&sm.empty[s], ph ^ 1);
      uint8_t* stage = dyn + (size_t)s * ST_STAGE;
      StageMeta& M = sm.meta[s];
      const int r0 = tile * ROWS;
      const int rows = min(ROWS, n - r0);
      uint32_t bytes = 0;
      int mat = 0, vmask = 0;
      int c0 = 0, nch = 0, slots = 0, a = 0, e = 0;
      if constexpr (FMT == 2) {
        c0 = r0 >> 5;
        nch = min(8, sell.nchunks - c0);
        for (int q = 0; q <= nch; ++q) M.cp[q] = sell.cptr[c0 + q];
        M.base = M.cp[0];
        slots = M.cp[nch] - M.cp[0];
        if (slots <= ST_SLOTS) {
          mat = 1;
          bytes += slots * 12 + nch * 32;
        }
      } else if constexpr (FMT == 1) {
        const int s0 = csr.rp[r0], s1 = csr.rp[r0 + rows];
        a = s0 & ~3;
        e = (s1 + 3) & ~3;
        M.base = a;
        if (e - a <= ST_SLOTS + 8 && e <= csr.rp[n]) {
          mat = 1;
          bytes += (e - a) * 12;
        }
      }
#pragma unroll
      for (int k = 0; k < NV && k < NVCAP; ++k) {
        const double* src = op.vin(k);
        if (src && ((rows * 8) & 15) == 0 && ((reinterpret_cast<uintptr_t>(src + r0) & 15) == 0)) {
          vmask |= 1 << k;
          bytes += rows * 8;
        }
      }
      M.mat = mat;
      M.vmask = vmask;
      mbar_expect_tx(&sm.full[s], bytes);  // the stage's single arrival (+ its bytes)
      if constexpr (FMT == 2) {
        if (mat && slots > 0) {
          bulk_g2s(stage, sell.sval + M.base, slots * 8, &sm.full[s]);
          bulk_g2s(stage + Layout<2>::SCOL, sell.scol + M.base, slots * 4, &sm.full[s]);
        }
        if (mat) bulk_g2s(stage + Layout<2>::ROFF, sell.roff + (size_t)c0 * 32, nch * 32, &sm.full[s]);
      } else if constexpr (FMT == 1) {
        if (mat && e > a) {
          bulk_g2s(stage, csr.v + a, (e - a) * 8, &sm.full[s]);
          bulk_g2s(stage + Layout<1>::SCOL, csr.ci + a, (e - a) * 4, &sm.full[s]);
        }
      }
#pragma unroll
      for (int k = 0; k < NV && k < NVCAP; ++k)
        if (vmask & (1 << k))
          bulk_g2s(stage + Layout<FMT>::VEC + (size_t)k * ROWS * 8, op.vin(k) + r0, rows * 8, &sm.full[s]);
    }
    return;
  }

  // ------------------------------------------------------------- consumer warps
  const int t = threadIdx.x;
  int it = 0;
  TileCounter<DD> ctr;
  for (int tile = t_begin; tile < t_end; ++tile, ++it) {
    const int s = it % ST_NST;
    const uint32_t ph = (it / ST_NST) & 1;
    mbar_wait(&sm.full[s], ph);
    const uint8_t* stage = dyn + (size_t)s * ST_STAGE;
    const StageMeta& M = sm.meta[s];
    const double* vst = reinterpret_cast<const double*>(stage + Layout<FMT>::VEC);
    const int r0 = tile * ROWS;
    double cc[W][DD];
    if constexpr (FMT == 0) {
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const int i = r0 + w * TB + t;
#pragma unroll
        for (int d = 0; d < DD; ++d) cc[w][d] = 0.0;
        if (i < n) {
          double v[NVA];
#pragma unroll
          for (int k = 0; k < NV; ++k) {
            const double* src = op.vin(k);
            v[k] = (k < NVCAP && (M.vmask >> k) & 1) ? vst[(size_t)k * ROWS + w * TB + t]
                                                     : (src ? __ldg(src + i) : 0.0);
          }
          op.row(i, 0.0, v, cc[w]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[s]);
    } else {
      const int i = r0 + t;
      auto g = [&](int col) { return op.gather(col); };
      double y = 0.0;
      if constexpr (FMT == 2) {
        const int c = (r0 >> 5) + warp;
        if (c < sell.nchunks) {
          const double* sv = reinterpret_cast<const double*>(stage);
          const int* sc = reinterpret_cast<const int*>(stage + Layout<2>::SCOL);
          const uint8_t* ro = stage + Layout<2>::ROFF;
          const int p0 = M.cp[warp], L = (M.cp[warp + 1] - p0) >> 5;
          double acc = 0.0;
          int rl;
          if (M.mat) {
            rl = ro[warp * 32 + lane];
            const int off = p0 - M.base + lane;
            if (L <= 8) {
              int cols[8];
              double vals[8], xs[8];
#pragma unroll
              for (int k = 0; k < 8; ++k)
                if (k < L) { cols[k] = sc[off + k * 32]; vals[k] = sv[off + k * 32]; }
#pragma unroll
              for (int k = 0; k < 8; ++k)
                if (k < L && cols[k] >= 0) xs[k] = g(cols[k]);
#pragma unroll
              for (int k = 0; k < 8; ++k)
                if (k < L && cols[k] >= 0) acc = __fma_rn(vals[k], xs[k], acc);
            } else {
              for (int k = 0; k < L; ++k) {
                const int col = sc[off + k * 32];
                if (col >= 0) acc = __fma_rn(sv[off + k * 32], g(col), acc);
              }
            }
          } else {
            rl = sell.roff[c * 32 + lane];
            const int base = p0 + lane;
            for (int k = 0; k < L; ++k) {
              const int col = __ldcs(sell.scol + base + k * 32);
              if (col >= 0) acc = __fma_rn(__ldcs(sell.sval + base + k * 32), g(col), acc);
            }
          }
          sm.sy[rl] = acc;
        }
        consumer_sync();
        y = sm.sy[t];
      } else {  // CSR
        if (i < n) {
          const int a = csr.rp[i], b = csr.rp[i + 1];
          if (M.mat) {
            const double* sv = reinterpret_cast<const double*>(stage);
            const int* sc = reinterpret_cast<const int*>(stage + Layout<1>::SCOL);
            for (int k = a - M.base; k < b - M.base; ++k) y = __fma_rn(sv[k], g(sc[k]), y);
          } else {
            for (int k = a; k < b; ++k) y = __fma_rn(__ldcs(csr.v + k), g(__ldcs(csr.ci + k)), y);
          }
        }
      }
#pragma unroll
      for (int d = 0; d < DD; ++d) cc[0][d] = 0.0;
      if (i < n) {
        double v[NVA];
#pragma unroll
        for (int k = 0; k < NV; ++k) {
          const double* src = op.vin(k);
          v[k] = (k < NVCAP && (M.vmask >> k) & 1) ? vst[(size_t)k * TB + t] : (src ? __ldg(src + i) : 0.0);
        }
        op.row(i, y, v, cc[0]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[s]);
      if constexpr (FMT == 2) consumer_sync();  // sy is rewritten by the next tile
    }
    if constexpr (D > 0) {
      // leaf t of window w sits in thread t: butterflies are trees of 32 leaves
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
#pragma unroll
        for (int w = 0; w < W; ++w) {
#pragma unroll
          for (int d = 0; d < D; ++d) cc[w][d] = cc[w][d] + __shfl_xor_sync(0xffffffffu, cc[w][d], off);
        }
      }
      if (lane == 0) {
#pragma unroll
        for (int w = 0; w < W; ++w) {
#pragma unroll
          for (int d = 0; d < D; ++d) sm.wres[it & 1][(w * D + d) * 8 + warp] = cc[w][d];
        }
      }
      consumer_sync();
      double tp[DD];
      if (warp == 0) {
#pragma unroll
        for (int w = 0; w < W; ++w) {
#pragma unroll
          for (int d = 0; d < D; ++d) {
            double u = lane < 8 ? sm.wres[it & 1][(w * D + d) * 8 + lane] : 0.0;
            u = u + __shfl_xor_sync(0xffffffffu, u, 1);
            u = u + __shfl_xor_sync(0xffffffffu, u, 2);
            u = u + __shfl_xor_sync(0xffffffffu, u, 4);
            cc[w][d] = u;
          }
        }
        reg_tree<W, DD>(cc);
        if (lane == 0) {
#pragma unroll
          for (int d = 0; d < DD; ++d) tp[d] = cc[0][d];
          ctr.push(tp);
        }
      }
    }
  }
  if constexpr (D > 0) {
    // pad the CTA's range to tpc tiles with zero partials (tree shape of AC-5)
    double cp[DD];
    if (threadIdx.x == 0) {
      double z[DD];
#pragma unroll
      for (int d = 0; d < DD; ++d) z[d] = 0.0;
      for (int k = t_end - t_begin; k < red.tpc; ++k) ctr.push(z);
#pragma unroll
      for (int d = 0; d < DD; ++d) cp[d] = ctr.stk[d][0];
    }
    cta_finish<D>(op, cp, red, sm);
  }
}

inline int st_dyn_smem() { return ST_NST * ST_STAGE; }

}  // namespace gsk
