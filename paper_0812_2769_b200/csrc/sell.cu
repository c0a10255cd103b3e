// sell.cu — CSR -> SELL-C-sigma (C = 32, sigma = 256) on the device (BASELINE.json
// configs[3]; DESIGN.md §5/§6).  Integer work, bit-exact with the oracle's layout:
//   1. per sigma-window: stable rank of rows by descending length (ties by row id) —
//      unless the window's rows in natural order need no more padded slots than
//      sorted (reading L1: the sort exists to cut padding), in which
//      case they keep their natural order and the window is marked "natural" (wid);
//      roff[slot] = in-window row offset; chunk_len = longest row of a chunk;
//   2. chunk_ptr = exclusive scan of 32 * chunk_len (3 launches, 64-bit; a layout of
//      2^31 slots or more is rejected);
//   3. fill: slot (k, lane) of chunk c at chunk_ptr[c] + 32 k + lane, CSR order kept,
//      padding col = -1, val = 0 (predicated off in the SpMV, AC-3).
// In a natural window lane l of warp w holds row 32 w + l, so a pass finishes its rows
// in row order without the shared-memory scatter and its barrier (engine.cuh).
#include <algorithm>
#include <climits>
#include <cstring>
#include <vector>
#include "internal.cuh"

namespace gsk {

__global__ void __launch_bounds__(TB) sell_rank_kernel(int n, int nchunks, const int* __restrict__ rp,
                                                       uint8_t* roff, int* clen, uint8_t* wid) {
  __shared__ int len[TB];
  __shared__ int slen[TB];
  __shared__ int cmax[2][TB / SELL_C];
  const int w = blockIdx.x, t = threadIdx.x, r = w * TB + t;
  len[t] = r < n ? rp[r + 1] - rp[r] : 0;
  __syncthreads();
  const int li = len[t];
  int rank = 0;
  for (int j = 0; j < TB; ++j) {
    const int lj = len[j];
    rank += (lj > li) || (lj == li && j < t);
  }
  slen[rank] = li;
  // longest row of each chunk in natural order (rows beyond n have length 0)
  const int nat = __reduce_max_sync(0xffffffffu, li);
  if ((t & 31) == 0) cmax[0][t >> 5] = nat;
  __syncthreads();
  if ((t & 31) == 0) cmax[1][t >> 5] = slen[t];  // sorted: the chunk's first row
  __syncthreads();
  int snat = 0, ssrt = 0;  // padded slots / 32 of the window, natural vs sorted
#pragma unroll
  for (int k = 0; k < TB / SELL_C; ++k) {
    snat += cmax[0][k];
    ssrt += cmax[1][k];
  }
  const bool natural = snat <= ssrt;
  const int slot = natural ? t : rank;
  const int c = w * (TB / SELL_C) + (slot >> 5);
  if (c < nchunks) roff[(size_t)w * TB + slot] = (uint8_t)t;
  if (t == 0) wid[w] = natural ? 1 : 0;
  if ((t & 31) == 0) {
    const int cc = w * (TB / SELL_C) + (t >> 5);
    if (cc < nchunks) clen[cc] = cmax[natural ? 0 : 1][t >> 5];
  }
}

// exclusive scan of mult*clen into cptr[0..nchunks] in three launches (integer work,
// order-free): per-block sums of SCAN_B chunks, one CTA scans the block sums, each
// block scans its chunks from its offset.
constexpr int SCAN_T = 1024;
constexpr int SCAN_B = 4 * SCAN_T;  // chunks per block

__device__ __forceinline__ long long block_excl_scan(long long v, long long* sh, long long* total) {
  const int t = threadIdx.x;
  sh[t] = v;
  __syncthreads();
  for (int off = 1; off < SCAN_T; off <<= 1) {
    const long long u = t >= off ? sh[t - off] : 0;
    __syncthreads();
    sh[t] += u;
    __syncthreads();
  }
  const long long incl = sh[t];
  if (total) *total = sh[SCAN_T - 1];
  __syncthreads();
  return incl - v;
}

__global__ void __launch_bounds__(SCAN_T) sell_scan_sums(int nchunks, const int* __restrict__ clen, long long* bsum,
                                                       int mult) {
  __shared__ long long sh[SCAN_T];
  const int b0 = blockIdx.x * SCAN_B, t = threadIdx.x;
  long long v = 0;
  for (int k = 0; k < SCAN_B / SCAN_T; ++k) {
    const int c = b0 + k * SCAN_T + t;
    if (c < nchunks) v += (long long)clen[c] * mult;
  }
  long long tot = 0;
  block_excl_scan(v, sh, &tot);
  if (t == 0) bsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(SCAN_T) sell_scan_offsets(int nblocks, long long* bsum) {
  __shared__ long long sh[SCAN_T];
  long long carry = 0;
  for (int base = 0; base < nblocks; base += SCAN_T) {
    const int i = base + threadIdx.x;
    const long long v = i < nblocks ? bsum[i] : 0;
    long long tot = 0;
    const long long ex = block_excl_scan(v, sh, &tot);
    if (i < nblocks) bsum[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) bsum[nblocks] = carry;  // the grand total (checked on the host)
}

__global__ void __launch_bounds__(SCAN_T) sell_scan_final(int nchunks, const int* __restrict__ clen,
                                                        const long long* __restrict__ boff, int* cptr, int mult) {
  __shared__ long long sh[SCAN_T];
  const int b0 = blockIdx.x * SCAN_B, t = threadIdx.x;
  constexpr int PER = SCAN_B / SCAN_T;  // thread t owns chunks b0 + PER t .. + PER-1
  long long loc[PER];
  long long v = 0;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int c = b0 + PER * t + k;
    loc[k] = c < nchunks ? (long long)clen[c] * mult : 0;
    v += loc[k];
  }
  long long run = boff[blockIdx.x] + block_excl_scan(v, sh, nullptr);
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int c = b0 + PER * t + k;
    if (c < nchunks) cptr[c] = (int)run;
    run += loc[k];
    if (c == nchunks - 1) cptr[nchunks] = (int)run;
  }
}

// *total (nullable) receives the 64-bit sum; cptr is int32, so a sum of 2^31 or more
// is GSK_E_INVALID (the wrapped offsets are never used).
static int sell_scan(int nchunks, const int* clen, int* cptr, int mult, cudaStream_t s, long long* total) {
  const int nb = (nchunks + SCAN_B - 1) / SCAN_B;
  long long* bsum = nullptr;
  GSK_CUDA(pool_alloc((void**)&bsum, sizeof(long long) * (nb + 1)));  // (not cudaMallocAsync: plan.cu)
  sell_scan_sums<<<nb, SCAN_T, 0, s>>>(nchunks, clen, bsum, mult);
  sell_scan_offsets<<<1, SCAN_T, 0, s>>>(nb, bsum);
  sell_scan_final<<<nb, SCAN_T, 0, s>>>(nchunks, clen, bsum, cptr, mult);
  GSK_LAUNCHED(3);
  long long tot = 0;
  GSK_CUDA(cudaMemcpyAsync(&tot, bsum + nb, sizeof tot, cudaMemcpyDeviceToHost, s));
  GSK_CUDA(cudaStreamSynchronize(s));
  pool_release(bsum);
  if (total) *total = tot;
  if (tot > INT_MAX) {
    set_error("SELL layout: %lld slots do not fit int32 offsets (limit 2^31 - 1)", tot);
    return GSK_E_INVALID;
  }
  return GSK_OK;
}

__global__ void __launch_bounds__(TB) sell_fill_kernel(int n, int nchunks, const int* __restrict__ rp,
                                                       const int* __restrict__ ci, const double* __restrict__ v,
                                                       const int* __restrict__ cptr, const uint8_t* __restrict__ roff,
                                                       int* scol, double* sval, bool values_only, int pad) {
  const int w = blockIdx.x, t = threadIdx.x, lane = t & 31;
  const int c = w * (TB / SELL_C) + (t >> 5);
  if (c >= nchunks) return;
  const int row = w * TB + roff[(size_t)c * SELL_C + lane];
  const int p0 = cptr[c], L = (cptr[c + 1] - p0) / SELL_C;
  const int a = row < n ? rp[row] : 0;
  const int len = row < n ? rp[row + 1] - a : 0;
  for (int k = 0; k < L; ++k) {
    const size_t slot = (size_t)p0 + (size_t)k * SELL_C + lane;
    if (k < len) {
      if (!values_only) scol[slot] = ci[a + k];
      sval[slot] = v[a + k];
    } else {
      if (!values_only) scol[slot] = pad;
      sval[slot] = 0.0;
    }
  }
}

int sell_build(gsk_plan* P, cudaStream_t s) {
  const int n = P->A.n;
  const int nwin = (n + TB - 1) / TB;
  P->nchunks = (n + SELL_C - 1) / SELL_C;
  GSK_CUDA(pool_alloc((void**)&P->clen, sizeof(int) * P->nchunks));
  GSK_CUDA(pool_alloc((void**)&P->cptr, sizeof(int) * (P->nchunks + 1)));
  GSK_CUDA(pool_alloc((void**)&P->roff, (size_t)P->nchunks * SELL_C));
  GSK_CUDA(pool_alloc((void**)&P->wid, (size_t)nwin));
  sell_rank_kernel<<<nwin, TB, 0, s>>>(n, (int)P->nchunks, P->A.row_ptr, P->roff, P->clen, P->wid);
  GSK_LAUNCHED(1);
  long long tot = 0;
  GSK_TRY(sell_scan((int)P->nchunks, P->clen, P->cptr, SELL_C, s, &tot));
  P->nslots = tot;
  // every window natural? (then the passes run the NAT kernels) and the longest chunk
  // (<= 5: the short-slot kernels)
  int all_nat = 1, maxlen = 0;
  {
    std::vector<uint8_t> h(nwin);
    std::vector<int> cl(P->nchunks);
    GSK_CUDA(cudaMemcpyAsync(h.data(), P->wid, nwin, cudaMemcpyDeviceToHost, s));
    GSK_CUDA(cudaMemcpyAsync(cl.data(), P->clen, sizeof(int) * P->nchunks, cudaMemcpyDeviceToHost, s));
    GSK_CUDA(cudaStreamSynchronize(s));
    for (uint8_t f : h) all_nat &= f;
    for (int v : cl) maxlen = std::max(maxlen, v);
  }
  P->sell_maxlen = maxlen;
  GSK_CUDA(pool_alloc((void**)&P->scol, sizeof(int) * (size_t)(tot > 0 ? tot : 1)));
  GSK_CUDA(pool_alloc((void**)&P->sval, sizeof(double) * (size_t)(tot > 0 ? tot : 1)));
  sell_fill_kernel<<<nwin, TB, 0, s>>>(n, (int)P->nchunks, P->A.row_ptr, P->A.col_idx, P->A.values,
                                       P->cptr, P->roff, P->scol, P->sval, false, P->sell_pad);
  GSK_LAUNCHED(1);
  P->sell = SellView{};
  P->sell.n = n;
  P->sell.nchunks = (int)P->nchunks;
  P->sell.pad = P->sell_pad;
  P->sell.all_nat = all_nat;
  P->sell.cptr = P->cptr;
  P->sell.scol = P->scol;
  P->sell.sval = P->sval;
  P->sell.roff = P->roff;
  P->sell.wid = P->wid;
  // L2 prefetch lead in windows (engine.cuh): 1 when the slot data is far larger than
  // L2 (C4: SpMV 0.274 -> 0.266 ms, S3 0.283 -> 0.275 ms), else 0 — with a matrix of
  // 1.5-2x L2 (C3, C5) it cost 3-6% (profiles/r02_experiments); passes with fewer than
  // 4 windows per CTA skip it too.  GSK_L2PF overrides (2 was slower at C4).
  static const int l2pf_env = [] {
    const char* e = std::getenv("GSK_L2PF");
    return e ? std::atoi(e) : -1;
  }();
  P->sell.l2pf = l2pf_env >= 0 ? l2pf_env : (12.0 * (double)tot > 512e6 ? 1 : 0);
  return GSK_OK;
}

// ---- column-index dictionary ("SELL-D") ---------------------------------
// One warp per chunk.  The chunk's distinct deltas col - row (real slots only) are
// extracted in ascending order by repeated warp minima; a chunk with more than 32
// deltas makes the format inapplicable (*fail = 1).  Pass 0 counts, pass 1 writes the
// dictionary and the per-slot uint8 index (255 = padding).
__global__ void __launch_bounds__(TB) sell_dict_kernel(int nchunks, const int* __restrict__ cptr,
                                                       const int* __restrict__ scol, const uint8_t* __restrict__ roff,
                                                       int* ucount, const int* __restrict__ dptr, int* dict,
                                                       uint8_t* sidx, int* fail, int pass, int pad) {
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * (TB / 32) + (threadIdx.x >> 5);
  if (c >= nchunks) return;
  const long long row = (long long)(c * SELL_C) / SELL_SIGMA * SELL_SIGMA + roff[c * SELL_C + lane];
  const int p0 = cptr[c], L = (cptr[c + 1] - p0) / SELL_C;
  long long last = LLONG_MIN;
  int U = 0;
  int dv = 0;  // lane u < U holds dictionary entry u
  for (;;) {
    long long mine = LLONG_MAX;
    for (int k = 0; k < L; ++k) {
      const int col = scol[p0 + k * SELL_C + lane];
      if (col != pad) {
        const long long d = (long long)col - row;
        if (d > last && d < mine) mine = d;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const long long o = __shfl_xor_sync(0xffffffffu, mine, off);
      mine = o < mine ? o : mine;
    }
    if (mine == LLONG_MAX) break;
    if (U < 32 && lane == U) dv = (int)mine;
    ++U;
    last = mine;
    if (U > 32) break;
  }
  if (pass == 0) {
    if (lane == 0) {
      ucount[c] = U;
      if (U > 32) atomicExch(fail, 1);
    }
    return;
  }
  if (lane < U) dict[dptr[c] + lane] = dv;
  for (int k = 0; k < L; ++k) {
    const int slot = p0 + k * SELL_C + lane;
    const int col = scol[slot];
    const int d = (int)((long long)col - row);
    int pos = 0;
    for (int u = 0; u < U; ++u) pos += __shfl_sync(0xffffffffu, dv, u) < d;  // lower bound
    sidx[slot] = col != pad ? (uint8_t)pos : (uint8_t)255;
  }
}

int sell_dict_build(gsk_plan* P, cudaStream_t s) {
  const int nch = (int)P->nchunks;
  const int grid = (nch + TB / 32 - 1) / (TB / 32);
  int* ucount = nullptr;
  int* fail = nullptr;
  GSK_CUDA(cudaMalloc(&ucount, sizeof(int) * (nch + 1)));
  GSK_CUDA(cudaMalloc(&fail, sizeof(int)));
  GSK_CUDA(cudaMemsetAsync(fail, 0, sizeof(int), s));
  GSK_CUDA(pool_alloc((void**)&P->dptr, sizeof(int) * (nch + 1)));
  sell_dict_kernel<<<grid, TB, 0, s>>>(nch, P->cptr, P->scol, P->roff, ucount, nullptr, nullptr, nullptr, fail, 0, P->sell_pad);
  GSK_LAUNCHED(1);
  int hfail = 0;
  GSK_CUDA(cudaMemcpyAsync(&hfail, fail, sizeof(int), cudaMemcpyDeviceToHost, s));
  GSK_CUDA(cudaStreamSynchronize(s));
  if (hfail) {  // some chunk has > 32 distinct deltas: keep plain int32 columns
    cudaFree(ucount);
    cudaFree(fail);
    pool_release(P->dptr);  // the stream was synchronised above
    P->dptr = nullptr;
    return GSK_OK;
  }
  GSK_TRY(sell_scan(nch, ucount, P->dptr, 1, s, nullptr));
  int tot = 0;
  GSK_CUDA(cudaMemcpyAsync(&tot, P->dptr + nch, sizeof(int), cudaMemcpyDeviceToHost, s));
  GSK_CUDA(cudaStreamSynchronize(s));
  P->ndict = tot;
  GSK_CUDA(pool_alloc((void**)&P->dict, sizeof(int) * (size_t)(tot > 0 ? tot : 1)));
  GSK_CUDA(pool_alloc((void**)&P->sidx, (size_t)(P->nslots > 0 ? P->nslots : 1)));
  sell_dict_kernel<<<grid, TB, 0, s>>>(nch, P->cptr, P->scol, P->roff, ucount, P->dptr, P->dict, P->sidx, fail, 1, P->sell_pad);
  GSK_LAUNCHED(1);
  GSK_CUDA(cudaStreamSynchronize(s));
  cudaFree(ucount);
  cudaFree(fail);
  P->sell.sidx = P->sidx;
  P->sell.dptr = P->dptr;
  P->sell.dict = P->dict;
  return GSK_OK;
}

int sellu_fill_values(gsk_plan* P, cudaStream_t s);

int sell_fill_values(gsk_plan* P, cudaStream_t s) {
  if (P->uval) GSK_TRY(sellu_fill_values(P, s));
  if (P->sell_index == 3) GSK_TRY(rcd_build(P, s));  // the classes depend on the values
  const int n = P->A.n;
  const int nwin = (n + TB - 1) / TB;
  sell_fill_kernel<<<nwin, TB, 0, s>>>(n, (int)P->nchunks, P->A.row_ptr, P->A.col_idx, P->A.values,
                                       P->cptr, P->roff, P->scol, P->sval, true, P->sell_pad);
  GSK_LAUNCHED(1);
  return GSK_OK;
}

}  // namespace gsk

namespace gsk {

// ---- chunk-uniform column offsets ("SELL-U") ---------------------------
// A chunk is stored with one slot per distinct delta col - row of its rows (ascending,
// <= SELLU_MAXL): slot k of lane l holds row l's entry at column row + udel[c][k], or
// padding (bit l of umask[c][k] clear).  The deltas and masks are per chunk, so the
// column index costs 8 bytes per 32 slots instead of 4 bytes per slot, and the gather
// addresses need no per-slot load.  Each row's entries stay in ascending column order
// (ascending deltas), so the SpMV chain is AC-3's.  On the stencil systems a chunk has
// exactly as many deltas as its longest row: the same slots as SELL-C-sigma.
__global__ void __launch_bounds__(TB) sellu_meta_kernel(int n, int nchunks, const int* __restrict__ rp,
                                                        const int* __restrict__ ci, const uint8_t* __restrict__ roff,
                                                        int* ucnt, int* udel, unsigned* umask, int* fail) {
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * (TB / 32) + (threadIdx.x >> 5);
  if (c >= nchunks) return;
  const long long row = (long long)(c * SELL_C) / SELL_SIGMA * SELL_SIGMA + roff[c * SELL_C + lane];
  const bool real = row < n;
  const int a = real ? rp[row] : 0, e = real ? rp[row + 1] : 0;
  long long last = LLONG_MIN;
  int U = 0, dv = 0;
  unsigned mv = 0u;
  for (;;) {
    long long mine = LLONG_MAX;
    for (int q = a; q < e; ++q) {
      const long long d = (long long)ci[q] - row;
      if (d > last && d < mine) mine = d;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const long long o = __shfl_xor_sync(0xffffffffu, mine, off);
      mine = o < mine ? o : mine;
    }
    if (mine == LLONG_MAX) break;
    bool has = false;
    for (int q = a; q < e; ++q) has |= ((long long)ci[q] - row == mine);
    const unsigned m = __ballot_sync(0xffffffffu, has);
    if (lane == U) {
      dv = (int)mine;
      mv = m;
    }
    ++U;
    last = mine;
    if (U > SELLU_MAXL) break;
  }
  if (lane == 0) {
    ucnt[c] = U;
    if (U > SELLU_MAXL) atomicExch(fail, 1);
  }
  if (lane < SELLU_MAXL) {
    udel[(size_t)c * SELLU_MAXL + lane] = lane < U ? dv : 0;
    umask[(size_t)c * SELLU_MAXL + lane] = lane < U ? mv : 0u;
  }
}

// values of a SELL-U layout (at plan creation and after every rescaling): the row's
// entries (ascending columns) merged with the chunk's ascending deltas
__global__ void __launch_bounds__(TB) sellu_fill_kernel(int n, int nchunks, const int* __restrict__ rp,
                                                        const int* __restrict__ ci, const double* __restrict__ v,
                                                        const uint8_t* __restrict__ roff, const int* __restrict__ uptr,
                                                        const int* __restrict__ udel, double* uval) {
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * (TB / 32) + (threadIdx.x >> 5);
  if (c >= nchunks) return;
  const long long row = (long long)(c * SELL_C) / SELL_SIGMA * SELL_SIGMA + roff[c * SELL_C + lane];
  const bool real = row < n;
  int q = real ? rp[row] : 0;
  const int e = real ? rp[row + 1] : 0;
  const int p0 = uptr[c], U = (uptr[c + 1] - p0) / SELL_C;
  for (int k = 0; k < U; ++k) {
    const long long d = udel[(size_t)c * SELLU_MAXL + k];
    double val = 0.0;
    if (q < e && (long long)ci[q] - row == d) val = v[q++];
    uval[(size_t)p0 + (size_t)k * SELL_C + lane] = val;
  }
}

int sellu_fill_values(gsk_plan* P, cudaStream_t s) {
  const int nch = (int)P->nchunks;
  const int grid = (nch + TB / 32 - 1) / (TB / 32);
  sellu_fill_kernel<<<grid, TB, 0, s>>>(P->A.n, nch, P->A.row_ptr, P->A.col_idx, P->A.values, P->roff, P->uptr,
                                        P->udel, P->uval);
  GSK_LAUNCHED(1);
  return GSK_OK;
}

int sellu_build(gsk_plan* P, cudaStream_t s) {
  const int nch = (int)P->nchunks;
  const int grid = (nch + TB / 32 - 1) / (TB / 32);
  int* ucnt = nullptr;
  int* fail = nullptr;
  GSK_CUDA(cudaMalloc(&ucnt, sizeof(int) * (nch + 1)));
  GSK_CUDA(cudaMalloc(&fail, sizeof(int)));
  GSK_CUDA(cudaMemsetAsync(fail, 0, sizeof(int), s));
  GSK_CUDA(pool_alloc((void**)&P->udel, sizeof(int) * (size_t)nch * SELLU_MAXL));
  GSK_CUDA(pool_alloc((void**)&P->umask, sizeof(unsigned) * (size_t)nch * SELLU_MAXL));
  sellu_meta_kernel<<<grid, TB, 0, s>>>(P->A.n, nch, P->A.row_ptr, P->A.col_idx, P->roff, ucnt, P->udel, P->umask,
                                        fail);
  GSK_LAUNCHED(1);
  int hfail = 0;
  GSK_CUDA(cudaMemcpyAsync(&hfail, fail, sizeof(int), cudaMemcpyDeviceToHost, s));
  GSK_CUDA(cudaStreamSynchronize(s));
  long long tot = 0;
  int rc = GSK_OK;
  if (!hfail) {
    GSK_CUDA(pool_alloc((void**)&P->uptr, sizeof(int) * (nch + 1)));
    rc = sell_scan(nch, ucnt, P->uptr, SELL_C, s, &tot);
  }
  cudaFree(ucnt);
  cudaFree(fail);
  // inapplicable (a chunk with more than SELLU_MAXL deltas, or int32 offsets would
  // overflow): the plan keeps plain int32 columns
  if (hfail || rc != GSK_OK) {
    for (void* b : {(void*)P->udel, (void*)P->umask, (void*)P->uptr})
      pool_release(b);  // cudaFree(ucnt) above synchronised the device
    P->udel = nullptr;
    P->umask = nullptr;
    P->uptr = nullptr;
    return GSK_OK;
  }
  P->nuslots = tot;
  GSK_CUDA(pool_alloc((void**)&P->uval, sizeof(double) * (size_t)(tot > 0 ? tot : 1)));
  GSK_TRY(sellu_fill_values(P, s));
  GSK_CUDA(cudaStreamSynchronize(s));
  P->sell.uptr = P->uptr;
  P->sell.udel = P->udel;
  P->sell.umask = P->umask;
  P->sell.uval = P->uval;
  return GSK_OK;
}

}  // namespace gsk

namespace gsk {

// ---- row-class dictionary ("RCD") ---------------------------------------
// The paper's problems have piecewise-constant coefficients: whole
// regions share one stencil row, before and after GS(p).  Rows with the same length,
// deltas col - row and bit-identical values (CSR order) form a class; a pass then reads
// a 2-byte class id per row and the class's 128-byte entry (L1-resident) instead of 12
// bytes per nonzero — the same FMA chain on the same operands (AC-3), so bit-identical
// results.  Classes are numbered by first occurrence (the oracle's orc_row_classes).
//   1. hash every row (64-bit) into an open-addressing table keyed by the hash, keeping
//      the smallest row of each key;
//   2. host: used slots sorted by that row -> class ids (a 256 KB round trip);
//   3. every row looks its slot up, is compared entry by entry with the class's first row
//      (a hash collision makes the format inapplicable rather than wrong) and stores its
//      id; a class's first row writes the dictionary entry.
// Inapplicable (the plan keeps its plain SELL passes): a row longer than RCD_MAXL, more
// than RCD_MAXCLS classes, a collision.
constexpr int RCD_HT = 4 * RCD_MAXCLS;  // table slots (power of two)
struct RcdSlot {
  unsigned long long key;  // 0 = empty
  int row;                 // smallest row with this key
  int id;                  // class id (step 2)
};

__device__ __forceinline__ unsigned long long rcd_mix(unsigned long long h, unsigned long long x) {
  h = (h ^ x) * 0xff51afd7ed558ccdull;
  return h ^ (h >> 32);
}
// kmask: all ones, or fewer bits under the test hook GSK_RCD_HASH_BITS (forces different
// rows onto one key, which the entry-by-entry comparison of step 3 must catch)
__device__ __forceinline__ unsigned long long rcd_key(int i, const int* __restrict__ rp, const int* __restrict__ ci,
                                                      const double* __restrict__ v, unsigned long long kmask) {
  const int a = rp[i], len = rp[i + 1] - a;
  unsigned long long h = rcd_mix(0x9e3779b97f4a7c15ull, (unsigned long long)len);
  for (int q = 0; q < len; ++q) {
    h = rcd_mix(h, (unsigned long long)(long long)(ci[a + q] - i));
    h = rcd_mix(h, (unsigned long long)__double_as_longlong(v[a + q]));
  }
  h &= kmask;
  return h ? h : 1ull;
}

__global__ void rcd_init_kernel(RcdSlot* tab, int* flags) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < RCD_HT) tab[t] = RcdSlot{0ull, INT_MAX, -1};
  if (t < 2) flags[t] = 0;  // [0] fail, [1] classes
}

__global__ void __launch_bounds__(TB) rcd_hash_kernel(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                                      const double* __restrict__ v, RcdSlot* tab, int* flags,
                                                      unsigned long long kmask) {
  const int i = blockIdx.x * TB + threadIdx.x;
  if (i >= n) return;
  if (rp[i + 1] - rp[i] > RCD_MAXL) {
    flags[0] = 1;
    return;
  }
  const unsigned long long key = rcd_key(i, rp, ci, v, kmask);
  int slot = (int)(key & (RCD_HT - 1));
  for (int probe = 0; probe < RCD_HT; ++probe, slot = (slot + 1) & (RCD_HT - 1)) {
    // a plain look first: almost every row finds its class already there
    unsigned long long cur = *(volatile unsigned long long*)&tab[slot].key;
    if (cur == 0ull) {
      cur = atomicCAS(&tab[slot].key, 0ull, key);
      if (cur == 0ull) {
        cur = key;
        if (atomicAdd(&flags[1], 1) >= RCD_MAXCLS) flags[0] = 1;
      }
    }
    if (cur == key) {
      if (*(volatile int*)&tab[slot].row > i) atomicMin(&tab[slot].row, i);
      return;
    }
    if (*(volatile int*)&flags[0]) return;  // already inapplicable
  }
  flags[0] = 1;  // table full
}

__global__ void __launch_bounds__(TB) rcd_assign_kernel(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                                        const double* __restrict__ v, const RcdSlot* __restrict__ tab,
                                                        uint16_t* kcls, RcdEntry* kdict, int* flags,
                                                        unsigned long long kmask) {
  const int i = blockIdx.x * TB + threadIdx.x;
  if (i >= n) return;
  const unsigned long long key = rcd_key(i, rp, ci, v, kmask);
  int slot = (int)(key & (RCD_HT - 1));
  while (tab[slot].key != key) slot = (slot + 1) & (RCD_HT - 1);  // present (step 1)
  const int rep = tab[slot].row, id = tab[slot].id;
  const int a = rp[i], len = rp[i + 1] - a, ra = rp[rep];
  bool same = rp[rep + 1] - ra == len;
  for (int q = 0; q < len && same; ++q)
    same = (ci[a + q] - i == ci[ra + q] - rep) &&
           __double_as_longlong(v[a + q]) == __double_as_longlong(v[ra + q]);
  if (!same) flags[0] = 2;  // two different rows with one hash
  kcls[i] = (uint16_t)id;
  if (i == rep) {
    RcdEntry e;
    int dd[RCD_MAXL + 2];
    for (int q = 0; q < RCD_MAXL; ++q) {
      e.v[q] = q < len ? v[a + q] : 0.0;
      dd[q + 1] = q < len ? ci[a + q] - i : 0;
    }
    dd[0] = len;
    dd[RCD_MAXL + 1] = 0;
    for (int q = 0; q < 5; ++q) e.ld[q] = make_int2(dd[2 * q], dd[2 * q + 1]);
    for (int q = 0; q < 6; ++q) e.pad_[q] = 0;
    kdict[id] = e;
  }
}

int rcd_build(gsk_plan* P, cudaStream_t s) {
  const int n = P->A.n;
  static_assert(sizeof(RcdEntry) == 128 && sizeof(RcdSlot) == 16, "RCD layouts");
  const bool had = P->sell.rcd != nullptr;
  if (!P->kcls) {
    GSK_CUDA(pool_alloc((void**)&P->drcd, sizeof(RcdView)));
    GSK_CUDA(pool_alloc((void**)&P->kcls, sizeof(uint16_t) * (size_t)n));
    GSK_CUDA(pool_alloc((void**)&P->kdict, sizeof(RcdEntry) * RCD_MAXCLS));
    GSK_CUDA(pool_alloc((void**)&P->ktab, sizeof(RcdSlot) * RCD_HT + 2 * sizeof(int)));
  }
  RcdSlot* tab = reinterpret_cast<RcdSlot*>(P->ktab);
  int* flags = reinterpret_cast<int*>(tab + RCD_HT);
  const int grid = (n + TB - 1) / TB;
  static const unsigned long long kmask = [] {  // test hook: hash keys of GSK_RCD_HASH_BITS bits
    const char* e = std::getenv("GSK_RCD_HASH_BITS");
    const int bits = e ? std::atoi(e) : 64;
    return bits > 0 && bits < 64 ? (1ull << bits) - 1 : ~0ull;
  }();
  rcd_init_kernel<<<(RCD_HT + TB - 1) / TB, TB, 0, s>>>(tab, flags);
  rcd_hash_kernel<<<grid, TB, 0, s>>>(n, P->A.row_ptr, P->A.col_idx, P->A.values, tab, flags, kmask);
  GSK_LAUNCHED(2);
  std::vector<RcdSlot> h(RCD_HT);
  int hf[2] = {0, 0};
  GSK_CUDA(cudaMemcpyAsync(hf, flags, sizeof hf, cudaMemcpyDeviceToHost, s));
  GSK_CUDA(cudaStreamSynchronize(s));
  bool ok = hf[0] == 0 && hf[1] <= RCD_MAXCLS;
  int ncls = 0;
  if (ok) {
    GSK_CUDA(cudaMemcpyAsync(h.data(), tab, sizeof(RcdSlot) * RCD_HT, cudaMemcpyDeviceToHost, s));
    GSK_CUDA(cudaStreamSynchronize(s));
    std::vector<std::pair<int, int>> used;  // (first row, slot)
    for (int q = 0; q < RCD_HT; ++q)
      if (h[q].key) used.emplace_back(h[q].row, q);
    std::sort(used.begin(), used.end());
    ncls = (int)used.size();
    for (int k = 0; k < ncls; ++k) h[used[k].second].id = k;
    GSK_CUDA(cudaMemcpyAsync(tab, h.data(), sizeof(RcdSlot) * RCD_HT, cudaMemcpyHostToDevice, s));
    rcd_assign_kernel<<<grid, TB, 0, s>>>(n, P->A.row_ptr, P->A.col_idx, P->A.values, tab, P->kcls, P->kdict, flags,
                                          kmask);
    GSK_LAUNCHED(1);
    GSK_CUDA(cudaMemcpyAsync(hf, flags, sizeof hf, cudaMemcpyDeviceToHost, s));
    GSK_CUDA(cudaStreamSynchronize(s));
    ok = hf[0] == 0;
  }
  P->ncls = ok ? ncls : 0;
  const int had_ns = (had && P->hrcd.kslots) ? P->hrcd.ns : 0;
  P->hrcd = RcdView{};
  P->hrcd.kcls = ok ? P->kcls : nullptr;
  P->hrcd.kdict = ok ? P->kdict : nullptr;
  // stencil slots (engine.cuh rcd_row_slots): the classes' deltas taken together are one
  // symmetric set {.., -1, 0, 1, ..} of 5 or 7 — then a class becomes a presence mask and
  // one value per delta of that set (host work on <= 4096 class lines)
  static const bool slots_on = [] {
    const char* e = std::getenv("GSK_RCD_SLOTS");
    return !e || std::atoi(e) != 0;
  }();
  if (ok && slots_on) {
    std::vector<RcdEntry> ent(ncls);
    GSK_CUDA(cudaMemcpyAsync(ent.data(), P->kdict, sizeof(RcdEntry) * ncls, cudaMemcpyDeviceToHost, s));
    GSK_CUDA(cudaStreamSynchronize(s));
    auto delta = [](const RcdEntry& e, int q) { return q == 0 ? e.ld[0].y : (q & 1) ? e.ld[(q + 1) / 2].x : e.ld[q / 2].y; };
    std::vector<int> U;
    for (const RcdEntry& e : ent)
      for (int q = 0; q < e.ld[0].x; ++q) U.push_back(delta(e, q));
    std::sort(U.begin(), U.end());
    U.erase(std::unique(U.begin(), U.end()), U.end());
    const int ns = (int)U.size(), c = ns / 2;
    bool sym = (ns == 5 || ns == 7) && U[c] == 0 && U[c - 1] == -1 && U[c + 1] == 1;
    for (int k = 0; sym && k < ns; ++k) sym = U[k] == -U[ns - 1 - k];
    if (sym) {
      std::vector<RcdSlots> sl(ncls);
      for (int k = 0; k < ncls; ++k) {
        RcdSlots& o = sl[k];
        std::memset(&o, 0, sizeof o);
        for (int q = 0; q < ent[k].ld[0].x; ++q) {
          const int pos = (int)(std::lower_bound(U.begin(), U.end(), delta(ent[k], q)) - U.begin());
          o.v[pos] = ent[k].v[q];
          o.mask |= 1u << pos;
        }
      }
      if (!P->kslots) GSK_CUDA(pool_alloc((void**)&P->kslots, sizeof(RcdSlots) * RCD_MAXCLS));
      GSK_CUDA(cudaMemcpyAsync(P->kslots, sl.data(), sizeof(RcdSlots) * ncls, cudaMemcpyHostToDevice, s));
      GSK_CUDA(cudaStreamSynchronize(s));  // sl is a local
      P->hrcd.kslots = P->kslots;
      P->hrcd.ns = ns;
      for (int k = 0; k < RCD_MAXL; ++k) P->hrcd.sdel[k] = k < ns ? U[k] : 0;
      P->hrcd.sroll = U[c + 2] == TB ? 1 : 0;
    }
  }
  if (ok) {
    GSK_CUDA(cudaMemcpyAsync(P->drcd, &P->hrcd, sizeof(RcdView), cudaMemcpyHostToDevice, s));
    GSK_CUDA(cudaStreamSynchronize(s));
  }
  P->sell.rcd = ok ? P->drcd : nullptr;
  if (ok != had || had_ns != P->hrcd.ns) {  // captured graphs hold the other kernels: capture again
    P->bkey_b = nullptr;
    P->gkey_b = nullptr;
  }
  return GSK_OK;
}

}  // namespace gsk
