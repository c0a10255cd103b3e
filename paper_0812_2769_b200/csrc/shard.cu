// shard.cu — row-block sharding of a plan.
//
// P shards own contiguous row blocks [r B, min((r+1) B, n)), B = 2^ceil(log2 n) / P, so
// every block is an aligned power-of-two subtree of the canonical reduction tree (AC-5).
// A shard is a plain sub-plan over its rows: CSR with rebased row pointers and columns
// relative to the shard's first row (negative = left halo, >= n_r = right halo; the
// SELL padding marker is INT_MIN there), its own SELL layout and reduction scratch.
// Its vectors are stored with halo margins, [hl | own rows | hr], and the operators get
// own-row base pointers, so gathers at negative / large local columns read the halo.
//
// Per solver pass: (1) halo exchange of the vector the SpMV gathers — device copies
// between shards held by this process, ncclSend/ncclRecv between processes; (2) the
// pass kernel of every local shard; (3) for dot products: each shard's finish writes
// its subtree values to gath[r], the values are all-gathered (ncclAllGather) when the
// shards live in several processes, and one warp joins the P values with the top of
// the tree and runs the operator's scalar epilogue — on every process, identically.
// The operators, passes and scalar epilogues are those of the unsharded solvers, so a
// sharded solve is bit-identical to the unsharded one and to the oracle.
#include <dlfcn.h>
#include <nccl.h>
#include <climits>
#include <cstring>
#include <vector>
#include "bicg_ops.cuh"
#include "gmres_ops.cuh"

namespace gsk {

// ---- NCCL, resolved from the process's libnccl.so.2 at run time -------------------------
struct NcclApi {
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclAllGather) allGather = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
};

static const NcclApi* nccl() {
  static NcclApi api;
  static int state = 0;  // 0 untried, 1 loaded, -1 unavailable
  if (state == 0) {
    state = -1;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
      api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(h, "ncclCommInitRank"));
      api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(h, "ncclCommDestroy"));
      api.allGather = reinterpret_cast<decltype(api.allGather)>(dlsym(h, "ncclAllGather"));
      api.send = reinterpret_cast<decltype(api.send)>(dlsym(h, "ncclSend"));
      api.recv = reinterpret_cast<decltype(api.recv)>(dlsym(h, "ncclRecv"));
      api.groupStart = reinterpret_cast<decltype(api.groupStart)>(dlsym(h, "ncclGroupStart"));
      api.groupEnd = reinterpret_cast<decltype(api.groupEnd)>(dlsym(h, "ncclGroupEnd"));
      api.errorString = reinterpret_cast<decltype(api.errorString)>(dlsym(h, "ncclGetErrorString"));
      if (api.getUniqueId && api.commInitRank && api.commDestroy && api.allGather && api.send && api.recv &&
          api.groupStart && api.groupEnd && api.errorString)
        state = 1;
    }
  }
  return state == 1 ? &api : nullptr;
}

#define GSK_NCCL(call)                                                                   \
  do {                                                                                   \
    ncclResult_t r_ = (call);                                                            \
    if (r_ != ncclSuccess) {                                                             \
      ::gsk::set_error("%s failed: %s", #call, ::gsk::nccl()->errorString(r_));          \
      return GSK_E_CUDA;                                                                 \
    }                                                                                    \
  } while (0)

// ---- layout ---------------------------------------------------------------------------
static int shard_rows(int64_t n, int P, int r, int64_t* lo, int64_t* hi) {
  if (n < 1 || P < 1 || P > 32 || (P & (P - 1)) || r < 0 || r >= P) {
    set_error("shard layout: need n >= 1, P a power of two in [1, 32], 0 <= r < P");
    return GSK_E_INVALID;
  }
  int64_t N = 1;
  while (N < n) N <<= 1;
  const int64_t B = N / P;
  if (B < 1 || (int64_t)(P - 1) * B >= n) {
    set_error("shard layout: %d shards of %lld rows leave the last shard of n = %lld empty", P, (long long)B,
              (long long)n);
    return GSK_E_INVALID;
  }
  *lo = (int64_t)r * B;
  *hi = std::min<int64_t>(n, (int64_t)(r + 1) * B);
  return GSK_OK;
}

struct Shard {
  gsk_plan* sub = nullptr;  // plan over the shard's rows (local CSR, SELL, scratch)
  int64_t lo = 0, hi = 0;
  int n = 0, hl = 0, hr = 0;
  size_t pitch = 0;         // vector pitch: hl + n + hr
  int* rp = nullptr;        // owned local CSR arrays
  int* ci = nullptr;
  double* bvec = nullptr;   // Bi-CGSTAB: r, r^, p, v, s, t, x (7 pitches)
  double* W = nullptr;      // GMRES basis: (Wm + 1) pitches
  int Wm = 0;
  double* gx = nullptr;     // GMRES x (1 pitch)
  double* own(double* base, int k) const { return base + (size_t)k * pitch + hl; }
};

struct ShardSet {
  int P = 1, first = 0, count = 1;
  ncclComm_t comm = nullptr;
  std::vector<int64_t> lo, hi;   // all shards
  std::vector<int> hl, hr;       // all shards
  std::vector<Shard> sh;         // this process's shards
  double* gath = nullptr;        // [P][MAXD] shard values of the current reduction
  int* mm = nullptr;             // halo scan scratch
  int64_t rows0 = 0;             // first row held by this process
  // device-initiated reductions (peer_reduce): this process's buffer (values, flags,
  // epoch counters; engine.cuh), the P buffer pointers on the device, the IPC mappings
  bool peer = false;
  double* pbuf = nullptr;
  double** dpeers = nullptr;
  std::vector<void*> opened;
  // device-initiated halos (peer mode): each shard's mailbox as seen from this process
  // (its own, or a neighbour's through the IPC mapping of that process's buffer)
  std::vector<char*> box;
  double* ebuf = nullptr;       // emulation (all shards here): the mailboxes
};

// Halo mailbox of shard q (peer mode): [2][hl_q] doubles received from
// the left neighbour, [2][hr_q] from the right (by epoch parity), then four uint64 —
// the epochs released by the left / right neighbour, this shard's halo epoch, and its
// push ticket counter.
static size_t box_bytes(int hl, int hr) { return ((16 * ((size_t)hl + hr) + 32) + 255) & ~size_t(255); }
static size_t red_bytes(int P) {
  return ((sizeof(double) * 2 * (size_t)P * MAXD + 2 * sizeof(unsigned long long) * (size_t)P) + 255) & ~size_t(255);
}

struct BoxView {
  double* left;   // [2][hl]
  double* right;  // [2][hr]
  unsigned long long* flags;  // [0] from left, [1] from right, [2] halo epoch, [3] ticket
  int hl, hr;
};
static BoxView box_view(char* b, int hl, int hr) {
  BoxView v{};
  if (!b) return v;
  v.left = reinterpret_cast<double*>(b);
  v.right = v.left + 2 * (size_t)hl;
  v.flags = reinterpret_cast<unsigned long long*>(v.right + 2 * (size_t)hr);
  v.hl = hl;
  v.hr = hr;
  return v;
}

// push: shard r's boundary rows into its neighbours' mailboxes (peer stores over
// NVLink); the last CTA (a ticket per launch) releases the neighbours' flags with the
// new epoch and records it in r's own mailbox
__global__ void __launch_bounds__(256) halo_push_kernel(const double* v, int n, BoxView me, BoxView lnb, int to_left,
                                                        BoxView rnb, int to_right) {
  pdl_enter();
  const unsigned long long e = me.flags[2] + 1;
  const int par = (int)(e & 1ull);
  const int tot = to_left + to_right;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += gridDim.x * blockDim.x) {
    if (i < to_left) lnb.right[(size_t)par * lnb.hr + i] = v[i];
    else rnb.left[(size_t)par * rnb.hl + (i - to_left)] = v[n - to_right + (i - to_left)];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long t = atomicAdd(me.flags + 3, 1ull);
    if (t == e * gridDim.x - 1) {  // every CTA's stores are fenced: release them
      __threadfence_system();
      if (to_left) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(lnb.flags + 1), "l"(e) : "memory");
      if (to_right) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(rnb.flags + 0), "l"(e) : "memory");
      me.flags[2] = e;
    }
  }
}

// pull: wait for the neighbours' epoch, copy the mailboxes into the vector's margins
__global__ void __launch_bounds__(256) halo_pull_kernel(double* v, int n, BoxView me) {
  pdl_enter();
  const unsigned long long e = me.flags[2];
  const int par = (int)(e & 1ull);
  if (threadIdx.x == 0) {
    for (int k = 0; k < 2; ++k) {
      if ((k == 0 && !me.hl) || (k == 1 && !me.hr)) continue;
      for (;;) {
        unsigned long long f;
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(f) : "l"(me.flags + k) : "memory");
        if (f >= e) break;
        __nanosleep(32);
      }
    }
  }
  __syncthreads();
  const int tot = me.hl + me.hr;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += gridDim.x * blockDim.x) {
    if (i < me.hl) v[i - me.hl] = __ldcv(me.left + (size_t)par * me.hl + i);
    else v[n + (i - me.hl)] = __ldcv(me.right + (size_t)par * me.hr + (i - me.hl));
  }
}

void shard_destroy(ShardSet* S) {
  if (!S) return;
  for (auto& s : S->sh) {
    if (s.sub) gsk_plan_destroy(s.sub);
    // (the workspace cache, as a plan's buffers: the parent plan's stream was drained by
    // gsk_plan_destroy before this is called)
    for (void* b : {(void*)s.rp, (void*)s.ci, (void*)s.bvec, (void*)s.W, (void*)s.gx}) pool_release(b);
  }
  if (S->gath) cudaFree(S->gath);
  if (S->mm) cudaFree(S->mm);
  for (void* p : S->opened) cudaIpcCloseMemHandle(p);
  if (S->dpeers) cudaFree(S->dpeers);
  if (S->pbuf) cudaFree(S->pbuf);
  if (S->ebuf) cudaFree(S->ebuf);
  delete S;
}

// min / max column over the entries [k0, k1) (integer atomics: order-independent)
__global__ void col_minmax_kernel(const int* __restrict__ ci, int64_t k0, int64_t k1, int* mm) {
  int lo = INT_MAX, hi = INT_MIN;
  for (int64_t k = k0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < k1; k += (int64_t)gridDim.x * blockDim.x) {
    const int c = ci[k];
    lo = min(lo, c);
    hi = max(hi, c);
  }
  for (int off = 16; off > 0; off >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, off));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, off));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(mm, lo);
    atomicMax(mm + 1, hi);
  }
}

__global__ void shard_rp_kernel(const int* __restrict__ rp, int64_t lo, int n, int* rpl) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= n) rpl[i] = rp[lo + i] - rp[lo];
}

__global__ void shard_ci_kernel(const int* __restrict__ ci, int64_t k0, int64_t nnz, int lo, int* cil) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nnz) cil[k] = ci[k0 + k] - lo;
}

// Halo copies between shards on one device: segment blockIdx.x, strided over blockIdx.y.
struct HaloSeg {
  double* dst;
  const double* src;
  int n;
};
struct HaloList {
  HaloSeg s[64];
  int count;
};
__global__ void __launch_bounds__(256) halo_kernel(HaloList L) {
  pdl_enter();
  const HaloSeg g = L.s[blockIdx.x];
  for (int i = blockIdx.y * blockDim.x + threadIdx.x; i < g.n; i += gridDim.y * blockDim.x) g.dst[i] = g.src[i];
}

// Exchange the halo of one vector; base(i) = own-row base of local shard i.
template <class Base>
static int shard_halo(gsk_plan* P, Base base, cudaStream_t s) {
  ShardSet* S = P->shards;
  if (S->peer && S->P > 1) {  // device-initiated: pushes into the neighbours' mailboxes, then pulls
    constexpr int kHaloCtas = 16;
    for (int i = 0; i < S->count; ++i) {
      const int r = S->first + i;
      const Shard& d = S->sh[i];
      const BoxView me = box_view(S->box[r], S->hl[r], S->hr[r]);
      const BoxView l = r > 0 ? box_view(S->box[r - 1], S->hl[r - 1], S->hr[r - 1]) : BoxView{};
      const BoxView rr = r + 1 < S->P ? box_view(S->box[r + 1], S->hl[r + 1], S->hr[r + 1]) : BoxView{};
      GSK_CUDA(launch_k(halo_push_kernel, kHaloCtas, 256, 0, s, (const double*)base(i), d.n, me, l,
                        r > 0 ? S->hr[r - 1] : 0, rr, r + 1 < S->P ? S->hl[r + 1] : 0));
      GSK_LAUNCHED(1);
    }
    for (int i = 0; i < S->count; ++i) {
      const int r = S->first + i;
      GSK_CUDA(launch_k(halo_pull_kernel, kHaloCtas, 256, 0, s, base(i), S->sh[i].n,
                        box_view(S->box[r], S->hl[r], S->hr[r])));
      GSK_LAUNCHED(1);
    }
    return GSK_OK;
  }
  if (!S->comm) {  // every shard on this GPU: device copies
    if (S->P == 1) return GSK_OK;
    HaloList L{};
    int c = 0;
    for (int i = 0; i < S->count; ++i) {
      const Shard& d = S->sh[i];
      if (i > 0 && d.hl) L.s[c++] = HaloSeg{base(i) - d.hl, base(i - 1) + S->sh[i - 1].n - d.hl, d.hl};
      if (i + 1 < S->count && d.hr) L.s[c++] = HaloSeg{base(i) + d.n, base(i + 1), d.hr};
    }
    L.count = c;
    if (c) {
      GSK_CUDA(launch_k(halo_kernel, dim3(c, 32), 256, 0, s, L));
      GSK_LAUNCHED(1);
    }
    return GSK_OK;
  }
  // one shard per process: pairwise send / receive with the neighbours
  const NcclApi* api = nccl();
  const int r = S->first;
  const Shard& d = S->sh[0];
  double* v = base(0);
  GSK_NCCL(api->groupStart());
  if (r > 0) {
    if (d.hl) GSK_NCCL(api->recv(v - d.hl, d.hl, ncclDouble, r - 1, S->comm, s));
    if (S->hr[r - 1]) GSK_NCCL(api->send(v, S->hr[r - 1], ncclDouble, r - 1, S->comm, s));
  }
  if (r + 1 < S->P) {
    if (d.hr) GSK_NCCL(api->recv(v + d.n, d.hr, ncclDouble, r + 1, S->comm, s));
    if (S->hl[r + 1]) GSK_NCCL(api->send(v + d.n - S->hl[r + 1], S->hl[r + 1], ncclDouble, r + 1, S->comm, s));
  }
  GSK_NCCL(api->groupEnd());
  return GSK_OK;
}

// One pass on every local shard; with dot products, per-shard finishes, the gather of
// the P shard values and the global finish.  mk(i) builds the operator of shard i.
template <class MakeOp>
static int shard_pass(gsk_plan* P, MakeOp mk, cudaStream_t s, cudaEvent_t pe0 = nullptr, cudaEvent_t pe1 = nullptr) {
  using Op = decltype(mk(0));
  ShardSet* S = P->shards;
  for (int i = 0; i < S->count; ++i) {
    gsk_plan* Q = S->sh[i].sub;
    const Op op = mk(i);
    int nt = 0;
    GSK_TRY(launch_pass(Q, op, s, &nt, i == 0 ? pe0 : nullptr, i == 0 ? pe1 : nullptr));
    if constexpr (Op::D > 0) {
      if (S->peer)  // values stored into every process's buffer + a released epoch flag
        GSK_CUDA(launch_k(finish_peer_local_kernel<Op>, 1, FIN_THREADS, 0, s, op, (const double*)Q->part,
                          Q->pstride, nt, (double* const*)S->dpeers, S->P, S->first + i,
                          peer_flags(S->pbuf, S->P) + S->P + (S->first + i)));
      else
        GSK_CUDA(launch_k(finish_local_kernel<Op>, 1, FIN_THREADS, 0, s, op, (const double*)Q->part, Q->pstride,
                          nt, S->gath + (size_t)(S->first + i) * MAXD));
      GSK_LAUNCHED(1);
    }
  }
  if constexpr (Op::D > 0) {
    if (S->peer) {
      GSK_CUDA(launch_k(finish_peer_global_kernel<Op>, 1, 32, 0, s, mk(0), S->pbuf, S->P,
                        (const unsigned long long*)(peer_flags(S->pbuf, S->P) + S->P + S->first)));
    } else {
      if (S->comm)
        GSK_NCCL(nccl()->allGather(S->gath + (size_t)S->first * MAXD, S->gath, MAXD, ncclDouble, S->comm, s));
      GSK_CUDA(launch_k(finish_global_kernel<Op>, 1, 32, 0, s, mk(0), (const double*)S->gath, S->P));
    }
    GSK_LAUNCHED(1);
  }
  return GSK_OK;
}

// x (user, this process's rows) <-> the shards' halo-margined copies
static int shard_x_in(gsk_plan* P, const double* x0, double* (*xbase)(Shard&), cudaStream_t s) {
  ShardSet* S = P->shards;
  for (auto& d : S->sh) {
    double* xi = xbase(d);
    if (x0)
      GSK_CUDA(cudaMemcpyAsync(xi, x0 + (d.lo - S->rows0), sizeof(double) * d.n, cudaMemcpyDeviceToDevice, s));
    else
      GSK_CUDA(cudaMemsetAsync(xi, 0, sizeof(double) * d.n, s));
  }
  return GSK_OK;
}
static int shard_x_out(gsk_plan* P, double* x, double* (*xbase)(Shard&), cudaStream_t s) {
  ShardSet* S = P->shards;
  for (auto& d : S->sh)
    GSK_CUDA(cudaMemcpyAsync(x + (d.lo - S->rows0), xbase(d), sizeof(double) * d.n, cudaMemcpyDeviceToDevice, s));
  return GSK_OK;
}

// ---- Bi-CGSTAB (split schedule S0..S4, bicgstab.cu) -------------------------------------
static double* bicg_x(Shard& d) { return d.own(d.bvec, 6); }

static int shard_capture_bicg(gsk_plan* P, int K, int copy, cudaGraphExec_t* out) {
  ShardSet* S = P->shards;
  cudaStream_t s = P->st;
  BicgState* st = P->bstate;
  auto V = [&](int i, int k) { return S->sh[i].own(S->sh[i].bvec, k); };  // 0 r 1 r^ 2 p 3 v 4 s 5 t 6 x
  auto W = [&](int i) { return P->weights ? P->weights + (S->sh[i].lo - S->rows0) : nullptr; };
  GSK_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  int rc = GSK_OK;
  auto ev = [&](int kind, int edge, int k) { return k == 0 ? P->pev[kind][copy][edge] : nullptr; };
  for (int k = 0; k < K && rc == GSK_OK; ++k) {
    rc = shard_pass(P, [&](int i) { return OpS0{V(i, 0), V(i, 3), V(i, 2), st, 0, 0}; }, s);
    if (rc == GSK_OK) rc = shard_halo(P, [&](int i) { return V(i, 2); }, s);
    if (rc == GSK_OK)
      rc = shard_pass(P, [&](int i) { return OpS1<>{V(i, 2), V(i, 1), V(i, 3), st}; }, s, ev(0, 0, k), ev(0, 1, k));
    if (rc == GSK_OK)
      rc = shard_pass(P, [&](int i) { return OpS2{V(i, 0), V(i, 3), W(i), V(i, 4), P->hist_d, st, 0}; }, s);
    if (rc == GSK_OK) rc = shard_halo(P, [&](int i) { return V(i, 4); }, s);
    if (rc == GSK_OK)
      rc = shard_pass(P, [&](int i) { return OpS3<>{V(i, 4), V(i, 5), st}; }, s, ev(1, 0, k), ev(1, 1, k));
    if (rc == GSK_OK)
      rc = shard_pass(P, [&](int i) {
        return OpS4{V(i, 4), V(i, 2), V(i, 5), V(i, 1), W(i), V(i, 6), V(i, 0), P->hist_d, st, 0, 0, 0};
      }, s);
  }
  return end_capture(s, rc, out, &P->bkernels, "sharded bicgstab");
}

int shard_bicgstab_run(gsk_plan* P, const double* b, const double* x0, double tol, int maxit, double* x,
                       double* hist, gsk_report* rep, cudaStream_t caller) {
  ShardSet* S = P->shards;
  for (auto& d : S->sh)
    if (!d.bvec) GSK_CUDA(pool_alloc((void**)&d.bvec, sizeof(double) * 7 * d.pitch));
  if (!P->bstate) GSK_CUDA(pool_alloc((void**)&P->bstate, sizeof(BicgState)));
  GSK_TRY(ensure_hist(P, maxit));
  int K = P->poll;
  if (K <= 0) K = (int)std::min<long long>(64, std::max<long long>(4, (1LL << 26) / P->A.n));
  K = (K + 1) & ~1;
  if (!P->bgraph[0] || P->bkey_b != b || P->bK != K || P->bkey_h != P->hist_d) {
    for (auto& g : P->bgraph)
      if (g) {
        cudaGraphExecDestroy(g);
        g = nullptr;
      }
    for (int c = 0; c < gsk_plan::NQ; ++c) GSK_TRY(capture_retry([&] { return shard_capture_bicg(P, K, c, &P->bgraph[c]); }));
    P->bkey_b = b;
    P->bK = K;
    P->bkey_h = P->hist_d;
  }
  cudaStream_t s = P->st;
  GSK_TRY(join_in(P, caller));
  GSK_CUDA(cudaEventRecord(P->t0, s));
  GSK_TRY(shard_x_in(P, x0, bicg_x, s));
  BicgState h{};
  h.tol = tol;
  h.maxit = maxit;
  GSK_CUDA(cudaMemcpyAsync(P->bstate, &h, sizeof h, cudaMemcpyHostToDevice, s));
  auto V = [&](int i, int k) { return S->sh[i].own(S->sh[i].bvec, k); };
  auto Bv = [&](int i) { return b + (S->sh[i].lo - S->rows0); };
  auto W = [&](int i) { return P->weights ? P->weights + (S->sh[i].lo - S->rows0) : nullptr; };
  GSK_TRY(shard_halo(P, [&](int i) { return V(i, 6); }, s));
  GSK_TRY(shard_pass(P, [&](int i) {
    return OpInit<>{V(i, 6), Bv(i), W(i), V(i, 0), V(i, 1), V(i, 2), V(i, 3), P->hist_d, P->bstate};
  }, s));
  const long long maxb = (maxit + K - 1) / K + 1;
  const int kinds[2] = {0, 1};
  GSK_TRY(run_batches(P, P->bgraph, maxb, P->bkernels, &P->bstate->done, kinds, 2));
  GSK_TRY(shard_halo(P, [&](int i) { return V(i, 6); }, s));
  GSK_TRY(shard_pass(P, [&](int i) { return OpFinal<>{V(i, 6), Bv(i), W(i), P->bstate}; }, s));
  GSK_TRY(shard_x_out(P, x, bicg_x, s));
  GSK_CUDA(cudaEventRecord(P->t1, s));
  return bicgstab_report(P, hist, rep, caller);
}

// ---- GMRES(m) with MGS (gmres.cu), one cycle per captured graph ------------------------
static double* gmres_x(Shard& d) { return d.gx + d.hl; }

static int shard_capture_cycle(gsk_plan* P, const double* b, int m, int copy, cudaGraphExec_t* out) {
  ShardSet* S = P->shards;
  cudaStream_t s = P->st;
  GmresState* st = P->gstate;
  auto slot = [&](int i, int j) { return S->sh[i].own(S->sh[i].W, j - 1); };
  auto Bv = [&](int i) { return b + (S->sh[i].lo - S->rows0); };
  auto Wt = [&](int i) { return P->weights ? P->weights + (S->sh[i].lo - S->rows0) : nullptr; };
  GSK_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  int rc = GSK_OK;
  for (int j = 1; j <= m && rc == GSK_OK; ++j) {
    rc = shard_halo(P, [&](int i) { return slot(i, j); }, s);
    if (rc == GSK_OK) {
      auto mk = [&](int i) { return OpCgsS<>{slot(i, j), slot(i, j + 1), st, j, 0}; };
      rc = j == 1 ? shard_pass(P, mk, s, P->pev[3][copy][0], P->pev[3][copy][1]) : shard_pass(P, mk, s);
      if (rc == GSK_OK) rc = shard_pass(P, [&](int i) { return OpH1{slot(i, j + 1), slot(i, 1), st, j, 0}; }, s);
    }
    for (int q = 1; q < j && rc == GSK_OK; ++q) {
      auto mk = [&](int i) { return OpMgs{slot(i, q), slot(i, q + 1), slot(i, j + 1), st, q, j, 0, 0, 0}; };
      rc = (j == 2 && q == 1) ? shard_pass(P, mk, s, P->pev[2][copy][0], P->pev[2][copy][1]) : shard_pass(P, mk, s);
    }
    if (rc == GSK_OK)
      rc = shard_pass(P, [&](int i) { return OpLast{slot(i, j), slot(i, j + 1), P->hist_d, st, j, 0, 0}; }, s);
  }
  if (rc == GSK_OK)
    rc = shard_pass(P, [&](int i) {
      return OpXupd<>{slot(i, 1), gmres_x(S->sh[i]), st, S->sh[i].pitch, 0, nullptr, nullptr};
    }, s);
  if (rc == GSK_OK) rc = shard_halo(P, [&](int i) { return gmres_x(S->sh[i]); }, s);
  if (rc == GSK_OK)
    rc = shard_pass(P, [&](int i) {
      return OpGResid<>{gmres_x(S->sh[i]), Bv(i), Wt(i), slot(i, 1), P->hist_d, st, 0};
    }, s);
  return end_capture(s, rc, out, &P->gkernels, "sharded gmres");
}

int shard_gmres_run(gsk_plan* P, const double* b, const double* x0, int m, double tol, int maxit, double* x,
                    double* hist, gsk_report* rep, cudaStream_t caller) {
  ShardSet* S = P->shards;
  if (P->orth != GSK_ORTH_MGS) {
    set_error("gmres: sharded plans use modified Gram-Schmidt (gmres_orth = GSK_ORTH_MGS)");
    return GSK_E_INVALID;
  }
  for (auto& d : S->sh) {
    if (d.Wm < m) {
      if (d.W) {
        GSK_CUDA(cudaStreamSynchronize(P->st));  // no queued pass still uses it
        pool_release(d.W);
      }
      d.W = nullptr;
      cudaError_t e = pool_alloc((void**)&d.W, sizeof(double) * (size_t)(m + 1) * d.pitch);
      if (e != cudaSuccess) {
        set_error("gmres: cannot allocate a shard's (m+1) x n basis: %s", cudaGetErrorString(e));
        d.Wm = 0;
        return GSK_E_NOMEM;
      }
      d.Wm = m;
      for (auto& g : P->ggraph)
        if (g) {
          cudaGraphExecDestroy(g);
          g = nullptr;
        }
    }
    if (!d.gx) GSK_CUDA(pool_alloc((void**)&d.gx, sizeof(double) * d.pitch));
  }
  const size_t garr = (size_t)((MAX_M + 1) * MAX_M + 7 * MAX_M + 8);
  if (!P->gstate) GSK_CUDA(pool_alloc((void**)&P->gstate, sizeof(GmresState)));
  if (!P->garr) GSK_CUDA(pool_alloc((void**)&P->garr, sizeof(double) * garr));
  GSK_TRY(ensure_hist(P, maxit));
  if (!P->ggraph[0] || P->gkey_b != b || P->gkey_m != m || P->gkey_h != P->hist_d) {
    for (auto& g : P->ggraph)
      if (g) {
        cudaGraphExecDestroy(g);
        g = nullptr;
      }
    for (int c = 0; c < gsk_plan::NQ; ++c) GSK_TRY(capture_retry([&] { return shard_capture_cycle(P, b, m, c, &P->ggraph[c]); }));
    P->gkey_b = b;
    P->gkey_m = m;
    P->gkey_h = P->hist_d;
  }
  cudaStream_t s = P->st;
  GSK_TRY(join_in(P, caller));
  GSK_CUDA(cudaEventRecord(P->t0, s));
  GSK_TRY(shard_x_in(P, x0, gmres_x, s));
  GmresState h{};
  double* A = P->garr;
  h.H = A;
  h.cs = A + (MAX_M + 1) * MAX_M;
  h.sn = h.cs + MAX_M;
  h.g = h.sn + MAX_M;
  h.y = h.g + MAX_M + 1;
  h.inv = h.y + MAX_M;
  h.c1 = h.inv + MAX_M + 2;
  h.c2 = h.c1 + MAX_M;
  h.tol = tol;
  h.maxit = maxit;
  h.m = m;
  h.wstop = P->wstop;
  GSK_CUDA(cudaMemsetAsync(P->garr, 0, sizeof(double) * garr, s));
  GSK_CUDA(cudaMemcpyAsync(P->gstate, &h, sizeof h, cudaMemcpyHostToDevice, s));
  auto Bv = [&](int i) { return b + (S->sh[i].lo - S->rows0); };
  auto Wt = [&](int i) { return P->weights ? P->weights + (S->sh[i].lo - S->rows0) : nullptr; };
  GSK_TRY(shard_halo(P, [&](int i) { return gmres_x(S->sh[i]); }, s));
  GSK_TRY(shard_pass(P, [&](int i) {
    return OpGResid<>{gmres_x(S->sh[i]), Bv(i), Wt(i), S->sh[i].own(S->sh[i].W, 0), P->hist_d, P->gstate, 1};
  }, s));
  const int kinds[2] = {2, 3};
  GSK_TRY(run_batches(P, P->ggraph, (long long)maxit + 2, P->gkernels, &P->gstate->done, kinds, 2));
  GSK_TRY(shard_x_out(P, x, gmres_x, s));
  GSK_CUDA(cudaEventRecord(P->t1, s));
  return gmres_report(P, hist, rep, caller);
}

// ---- y = A x on this process's rows (halo-exchanged x) -----------------------------------
struct OpShardSpmv {
  static constexpr int D = 0;
  static constexpr int NV = 0;
  static constexpr bool kSpmv = true;
  const double* x;
  double* y;
  __device__ bool begin() { return true; }
  __device__ const double* vin(int) const { return nullptr; }
  __device__ double gather(int c) const { return __ldg(x + c); }
  __device__ void row(int i, double v, const double (&)[1], double (&)[1]) const { y[i] = v; }
};

int shard_spmv(gsk_plan* P, const double* x, double* y, cudaStream_t caller) {
  ShardSet* S = P->shards;
  for (auto& d : S->sh)
    if (!d.bvec) GSK_CUDA(pool_alloc((void**)&d.bvec, sizeof(double) * 7 * d.pitch));
  cudaStream_t s = P->st;
  GSK_TRY(join_in(P, caller));
  GSK_TRY(shard_x_in(P, x, bicg_x, s));
  GSK_TRY(shard_halo(P, [&](int i) { return bicg_x(S->sh[i]); }, s));
  GSK_TRY(shard_pass(P, [&](int i) { return OpShardSpmv{bicg_x(S->sh[i]), y + (S->sh[i].lo - S->rows0)}; }, s));
  GSK_TRY(join_out(P, caller));
  GSK_CUDA(cudaStreamSynchronize(caller));
  return GSK_OK;
}

// classes of this process's shard plans: the largest count, or -1 if one runs plain SELL
int64_t shard_row_classes(gsk_plan* P) {
  int64_t k = 0;
  for (auto& d : P->shards->sh) {
    if (!d.sub->sell.rcd) return -1;
    k = std::max<int64_t>(k, d.sub->ncls);
  }
  return k;
}

int shard_refresh(gsk_plan* P, cudaStream_t caller) {
  for (auto& d : P->shards->sh) GSK_TRY(gsk_plan_refresh(d.sub, caller));
  return GSK_OK;
}

}  // namespace gsk

using namespace gsk;

extern "C" {

int gsk_shard_rows(int64_t n, int32_t nshards, int32_t r, int64_t* lo, int64_t* hi) {
  if (!lo || !hi) {
    set_error("gsk_shard_rows: NULL output");
    return GSK_E_INVALID;
  }
  return shard_rows(n, nshards, r, lo, hi);
}

int gsk_shard_halo_host(int64_t n, const int32_t* row_ptr, const int32_t* col, int32_t nshards, int32_t r,
                        int32_t* hl, int32_t* hr) {
  if (!row_ptr || !col || !hl || !hr) {
    set_error("gsk_shard_halo_host: NULL argument");
    return GSK_E_INVALID;
  }
  int64_t lo, hi;
  GSK_TRY(shard_rows(n, nshards, r, &lo, &hi));
  int64_t cmin = lo, cmax = hi - 1;
  for (int64_t k = row_ptr[lo]; k < row_ptr[hi]; ++k) {
    cmin = std::min<int64_t>(cmin, col[k]);
    cmax = std::max<int64_t>(cmax, col[k]);
  }
  *hl = (int32_t)(lo - cmin);
  *hr = (int32_t)(cmax - (hi - 1));
  int64_t plo, phi, nlo, nhi;
  if (r > 0) {
    shard_rows(n, nshards, r - 1, &plo, &phi);
    if (*hl > phi - plo) {
      set_error("gsk_shard_halo_host: shard %d reads beyond shard %d (halo %d rows)", r, r - 1, *hl);
      return GSK_E_INVALID;
    }
  }
  if (r + 1 < nshards) {
    shard_rows(n, nshards, r + 1, &nlo, &nhi);
    if (*hr > nhi - nlo) {
      set_error("gsk_shard_halo_host: shard %d reads beyond shard %d (halo %d rows)", r, r + 1, *hr);
      return GSK_E_INVALID;
    }
  }
  return GSK_OK;
}

int gsk_nccl_unique_id(char* id) {
  const NcclApi* api = nccl();
  if (!api || !id) {
    set_error("gsk_nccl_unique_id: libnccl.so.2 not loadable or NULL id");
    return GSK_E_INVALID;
  }
  ncclUniqueId u;
  GSK_NCCL(api->getUniqueId(&u));
  std::memcpy(id, u.internal, sizeof u.internal);
  return GSK_OK;
}

int gsk_nccl_comm_create(const char* id, int32_t nranks, int32_t rank, void** comm) {
  const NcclApi* api = nccl();
  if (!api || !id || !comm || nranks < 1 || rank < 0 || rank >= nranks) {
    set_error("gsk_nccl_comm_create: libnccl.so.2 not loadable or bad arguments");
    return GSK_E_INVALID;
  }
  ncclUniqueId u;
  std::memcpy(u.internal, id, sizeof u.internal);
  ncclComm_t c = nullptr;
  GSK_NCCL(api->commInitRank(&c, nranks, u, rank));
  *comm = c;
  return GSK_OK;
}

int gsk_nccl_comm_destroy(void* comm) {
  const NcclApi* api = nccl();
  if (!api || !comm) return GSK_E_INVALID;
  GSK_NCCL(api->commDestroy(reinterpret_cast<ncclComm_t>(comm)));
  return GSK_OK;
}

int gsk_plan_create_sharded(const gsk_csr* A, const gsk_opts* opts, const gsk_shard_opts* so, gsk_plan** plan,
                            void* stream) {
  NvtxRange nv("gsk:plan_create_sharded");
  if (!A || !so || !plan || A->n < 1 || !A->row_ptr || (A->nnz > 0 && (!A->col_idx || !A->values))) {
    set_error("gsk_plan_create_sharded: invalid arguments");
    return GSK_E_INVALID;
  }
  const int P = so->nshards;
  int64_t lo0, hi0;
  GSK_TRY(shard_rows(A->n, P, 0, &lo0, &hi0));
  // one process holding every shard (no communicator), or one shard per process over
  // NCCL (P = 1 with a communicator runs the NCCL code path on a single GPU)
  const bool local = !so->nccl_comm && so->count == P && so->first == 0;
  const bool remote = so->nccl_comm && so->count == 1 && so->first >= 0 && so->first < P;
  if (!local && !remote) {
    set_error("gsk_plan_create_sharded: need count == nshards without a communicator (all shards on this GPU) "
              "or count == 1 with an NCCL communicator");
    return GSK_E_INVALID;
  }
  const bool linput = so->local_input != 0;
  if (linput && !remote) {
    set_error("gsk_plan_create_sharded: local_input needs count == 1 and an NCCL communicator");
    return GSK_E_INVALID;
  }
  if (remote && !nccl()) {
    set_error("gsk_plan_create_sharded: libnccl.so.2 is not loadable");
    return GSK_E_INVALID;
  }
  cudaStream_t s = as_stream(stream);
  // the parent plan: stream, events, states, graphs, history (CSR view of the whole
  // matrix, never used for passes)
  gsk_opts po = opts ? *opts : gsk_opts{};
  const int fmt = po.format;
  po.format = GSK_FMT_CSR;
  gsk_plan* Pp = nullptr;
  GSK_TRY(plan_create_impl(A, &po, -1, &Pp, s));
  Pp->fmt = fmt;
  ShardSet* S = new ShardSet();
  Pp->shards = S;
  S->P = P;
  S->first = so->first;
  S->count = so->count;
  S->comm = reinterpret_cast<ncclComm_t>(so->nccl_comm);
  S->lo.resize(P);
  S->hi.resize(P);
  S->hl.assign(P, 0);
  S->hr.assign(P, 0);
  auto fail = [&](int rc) {
    gsk_plan_destroy(Pp);
    return rc;
  };
  if (cudaMalloc(&S->mm, sizeof(int) * 2) != cudaSuccess || cudaMalloc(&S->gath, sizeof(double) * P * MAXD) != cudaSuccess) {
    set_error("gsk_plan_create_sharded: allocation failed");
    return fail(GSK_E_NOMEM);
  }
  if (cudaMemsetAsync(S->gath, 0, sizeof(double) * P * MAXD, s) != cudaSuccess) return fail(GSK_E_CUDA);
  // entries [k0, k1) of shard r in A's arrays (local input: this process's rows only)
  auto entry_range = [&](int r, int* k01) -> int {
    const int64_t a = linput ? 0 : S->lo[r], b = linput ? S->hi[r] - S->lo[r] : S->hi[r];
    if (cudaMemcpyAsync(&k01[0], A->row_ptr + a, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaMemcpyAsync(&k01[1], A->row_ptr + b, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      return GSK_E_CUDA;
    return GSK_OK;
  };
  for (int r = 0; r < P; ++r) shard_rows(A->n, P, r, &S->lo[r], &S->hi[r]);
  // halo widths of every shard: from the global matrix (every process computes all of
  // them), or — local input — each process its own, all-gathered
  for (int r = 0; r < P; ++r) {
    if (linput && r != so->first) continue;
    int k01[2];
    if (entry_range(r, k01) != GSK_OK) return fail(GSK_E_CUDA);
    const int init[2] = {INT_MAX, INT_MIN};
    int mm[2] = {INT_MAX, INT_MIN};
    if (k01[1] > k01[0]) {
      if (cudaMemcpyAsync(S->mm, init, sizeof init, cudaMemcpyHostToDevice, s) != cudaSuccess) return fail(GSK_E_CUDA);
      col_minmax_kernel<<<num_sms() * 4, 256, 0, s>>>(A->col_idx, k01[0], k01[1], S->mm);
      if (cudaMemcpyAsync(mm, S->mm, sizeof mm, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
          cudaStreamSynchronize(s) != cudaSuccess)
        return fail(GSK_E_CUDA);
    }
    S->hl[r] = mm[0] < S->lo[r] ? (int)(S->lo[r] - mm[0]) : 0;
    S->hr[r] = mm[1] > S->hi[r] - 1 ? (int)(mm[1] - (S->hi[r] - 1)) : 0;
  }
  if (linput && P > 1) {  // every process's (hl, hr), all-gathered
    int* hh = nullptr;
    if (cudaMalloc(&hh, sizeof(int) * 2 * P) != cudaSuccess) return fail(GSK_E_NOMEM);
    const int mine[2] = {S->hl[so->first], S->hr[so->first]};
    std::vector<int> all(2 * P);
    int rc = GSK_OK;
    if (cudaMemcpyAsync(hh + 2 * so->first, mine, sizeof mine, cudaMemcpyHostToDevice, s) != cudaSuccess) rc = GSK_E_CUDA;
    if (rc == GSK_OK && nccl()->allGather(hh + 2 * so->first, hh, 2, ncclInt32, S->comm, s) != ncclSuccess) {
      set_error("gsk_plan_create_sharded: ncclAllGather of the halo widths failed");
      rc = GSK_E_CUDA;
    }
    if (rc == GSK_OK && (cudaMemcpyAsync(all.data(), hh, sizeof(int) * 2 * P, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
                         cudaStreamSynchronize(s) != cudaSuccess))
      rc = GSK_E_CUDA;
    cudaFree(hh);
    if (rc != GSK_OK) return fail(rc);
    for (int r = 0; r < P; ++r) {
      S->hl[r] = all[2 * r];
      S->hr[r] = all[2 * r + 1];
    }
  }
  for (int r = 0; r < P; ++r) {
    if ((r > 0 && S->hl[r] > S->hi[r - 1] - S->lo[r - 1]) || (r + 1 < P && S->hr[r] > S->hi[r + 1] - S->lo[r + 1]) ||
        (r == 0 && S->hl[r]) || (r + 1 == P && S->hr[r])) {
      set_error("gsk_plan_create_sharded: shard %d reads rows beyond its neighbouring shards (halo %d / %d rows); "
                "only banded systems can be sharded", r, S->hl[r], S->hr[r]);
      return fail(GSK_E_INVALID);
    }
  }
  S->rows0 = S->lo[S->first];
  if (so->peer_reduce) {  // device-initiated reductions and halos: buffers, IPC mappings
    S->peer = true;
    // reduction area, then (one shard per process) this shard's halo mailbox
    const size_t rb = red_bytes(P);
    const size_t bytes = rb + (remote ? box_bytes(S->hl[so->first], S->hr[so->first]) : 0);
    if (cudaMalloc(&S->pbuf, bytes) != cudaSuccess || cudaMalloc(&S->dpeers, sizeof(double*) * P) != cudaSuccess) {
      set_error("gsk_plan_create_sharded: allocation of the peer-reduction buffers failed");
      return fail(GSK_E_NOMEM);
    }
    if (cudaMemsetAsync(S->pbuf, 0, bytes, s) != cudaSuccess) return fail(GSK_E_CUDA);
    S->box.assign(P, nullptr);
    if (remote) {
      S->box[so->first] = reinterpret_cast<char*>(S->pbuf) + rb;
    } else {  // all shards here: one mailbox each
      std::vector<size_t> off(P + 1, 0);
      for (int q = 0; q < P; ++q) off[q + 1] = off[q] + box_bytes(S->hl[q], S->hr[q]);
      if (cudaMalloc(&S->ebuf, off[P]) != cudaSuccess) return fail(GSK_E_NOMEM);
      if (cudaMemsetAsync(S->ebuf, 0, off[P], s) != cudaSuccess) return fail(GSK_E_CUDA);
      for (int q = 0; q < P; ++q) S->box[q] = reinterpret_cast<char*>(S->ebuf) + off[q];
    }
    std::vector<double*> ptrs(P, S->pbuf);  // one process: every shard's buffer is this one
    if (remote && P > 1) {
      cudaIpcMemHandle_t mine;
      if (cudaIpcGetMemHandle(&mine, S->pbuf) != cudaSuccess) {
        set_error("gsk_plan_create_sharded: cudaIpcGetMemHandle failed");
        return fail(GSK_E_CUDA);
      }
      char* dh = nullptr;
      const size_t hb = sizeof(cudaIpcMemHandle_t);
      std::vector<cudaIpcMemHandle_t> all(P);
      int rc = cudaMalloc(&dh, hb * P) == cudaSuccess ? GSK_OK : GSK_E_NOMEM;
      if (rc == GSK_OK && cudaMemcpyAsync(dh + hb * so->first, &mine, hb, cudaMemcpyHostToDevice, s) != cudaSuccess)
        rc = GSK_E_CUDA;
      if (rc == GSK_OK && nccl()->allGather(dh + hb * so->first, dh, hb, ncclChar, S->comm, s) != ncclSuccess) {
        set_error("gsk_plan_create_sharded: ncclAllGather of the IPC handles failed");
        rc = GSK_E_CUDA;
      }
      if (rc == GSK_OK && (cudaMemcpyAsync(all.data(), dh, hb * P, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
                           cudaStreamSynchronize(s) != cudaSuccess))
        rc = GSK_E_CUDA;
      if (dh) cudaFree(dh);
      if (rc != GSK_OK) return fail(rc);
      for (int q = 0; q < P; ++q) {
        if (q == so->first) continue;
        void* p = nullptr;
        if (cudaIpcOpenMemHandle(&p, all[q], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
          set_error("gsk_plan_create_sharded: cudaIpcOpenMemHandle of rank %d's buffer failed", q);
          return fail(GSK_E_CUDA);
        }
        S->opened.push_back(p);
        ptrs[q] = static_cast<double*>(p);
        if (q == so->first - 1 || q == so->first + 1) S->box[q] = static_cast<char*>(p) + rb;  // neighbours' mailboxes
      }
    }
    if (cudaMemcpyAsync(S->dpeers, ptrs.data(), sizeof(double*) * P, cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      return fail(GSK_E_CUDA);
  }
  // this process's shards: local CSR arrays and sub-plans
  S->sh.resize(S->count);
  gsk_opts so2 = opts ? *opts : gsk_opts{};
  so2.weights = nullptr;
  for (int i = 0; i < S->count; ++i) {
    const int r = S->first + i;
    Shard& d = S->sh[i];
    d.lo = S->lo[r];
    d.hi = S->hi[r];
    d.n = (int)(d.hi - d.lo);
    d.hl = S->hl[r];
    d.hr = S->hr[r];
    d.pitch = (size_t)d.hl + d.n + d.hr;
    int k01[2];
    if (entry_range(r, k01) != GSK_OK) return fail(GSK_E_CUDA);
    const int64_t nnz = k01[1] - k01[0];
    if (pool_alloc((void**)&d.rp, sizeof(int) * (d.n + 1)) != cudaSuccess ||
        pool_alloc((void**)&d.ci, sizeof(int) * (nnz > 0 ? nnz : 1)) != cudaSuccess) {
      set_error("gsk_plan_create_sharded: allocation failed");
      return fail(GSK_E_NOMEM);
    }
    shard_rp_kernel<<<(d.n + 256) / 256, 256, 0, s>>>(A->row_ptr, linput ? 0 : d.lo, d.n, d.rp);
    if (nnz > 0) shard_ci_kernel<<<(unsigned)((nnz + 255) / 256), 256, 0, s>>>(A->col_idx, k01[0], nnz, (int)d.lo, d.ci);
    if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess) {
      set_error("gsk_plan_create_sharded: shard CSR kernels failed");
      return fail(GSK_E_CUDA);
    }
    gsk_csr L{d.n, (int32_t)nnz, d.rp, d.ci, A->values + k01[0]};
    int rc = plan_create_impl(&L, &so2, INT_MIN, &d.sub, s);
    if (rc != GSK_OK) return fail(rc);
  }
  *plan = Pp;
  return GSK_OK;
}

}  // extern "C"
