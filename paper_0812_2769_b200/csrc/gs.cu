// gs.cu — GS(p): divide each row of A and its entry of b by the row's L_p norm.
//   PAPER.md:92-97 (definition), Eq. (2) PAPER.md:207-214 (DAx = Db, D = diag(1/||a_i||_p)).
// One pass over the nnz: a CTA owns 256 consecutive rows; their value segment is
// staged into shared memory with coalesced loads, each thread reduces its own row
// segment in ascending column order (AC-4: p=2 fma chain + sqrt, p=1 running sum of
// |a|, p>=3 repeated products + pow), the segment is rescaled in shared memory and
// written back coalesced.  Bytes: 16 nnz + 4(n+1) + 24 n (read a, write a, r/w b, d).
#include <mutex>
#include "internal.cuh"

namespace gsk {

__device__ __forceinline__ double row_norm_term(double a, int p) {
  const double m = fabs(a);
  double t = m;
  for (int e = 1; e < p; ++e) t = t * m;
  return t;
}

// norms_only: write s_i = sqrt(1/||a_i||_p) to dout and nothing else (two-sided
// scaling, first pass).
// PP: 1, 2 (specialised) or 0 (any p >= 3, passed in p)
template <int PP>
__global__ void __launch_bounds__(TB, 8) gs_kernel(int n, const int* __restrict__ rp,
                                                const double* vin, double* vout,
                                                const double* b, double* bout, double* dout,
                                                int p, int* bad, int norms_only) {
  __shared__ double sv[CSR_CAP];
  const int r0 = blockIdx.x * TB, t = threadIdx.x, r = r0 + t;
  const int rend = min(r0 + TB, n);
  const int s0 = __ldg(rp + r0), s1 = __ldg(rp + rend), cnt = s1 - s0;
  const bool staged = cnt <= CSR_CAP;
  if (staged) {
    for (int k = t; k < cnt; k += TB) cp_async8(sv + k, vin + s0 + k);
    cp_async_commit();
  }
  // own-row operands while the segment is in flight
  int a0 = 0, a1 = 0;
  double bi = 0.0;
  if (r < n) {
    a0 = __ldg(rp + r);
    a1 = __ldg(rp + r + 1);
    if (b && bout && !norms_only) bi = __ldcs(b + r);
  }
  if (staged) {
    cp_async_wait<0>();
    __syncthreads();
  }
  double d = 0.0;
  if (r < n) {
    const double* seg = staged ? sv + (a0 - s0) : vin + a0;
    const int len = a1 - a0;
    double acc = 0.0;
    double nrm;
    if constexpr (PP == 2) {
      for (int k = 0; k < len; ++k) acc = __fma_rn(seg[k], seg[k], acc);
      nrm = sqrt(acc);
    } else if constexpr (PP == 1) {
      for (int k = 0; k < len; ++k) acc = acc + fabs(seg[k]);
      nrm = acc;
    } else {
      for (int k = 0; k < len; ++k) acc = acc + row_norm_term(seg[k], p);
      nrm = pow(acc, 1.0 / p);
    }
    if (nrm == 0.0) {
      atomicMin(bad, r);
    } else {
      d = 1.0 / nrm;
    }
    if (norms_only) {
      dout[r] = sqrt(d);
    } else if (staged) {
      double* sg = sv + (a0 - s0);
      for (int k = 0; k < len; ++k) sg[k] = sg[k] * d;
    } else {
      for (int k = 0; k < len; ++k) vout[a0 + k] = vin[a0 + k] * d;
    }
    if (!norms_only) {
      if (b && bout) __stcs(bout + r, bi * d);
      if (dout) __stcs(dout + r, d);
    }
  }
  if (staged && !norms_only) {
    __syncthreads();
    for (int k = t; k < cnt; k += TB) __stcs(vout + s0 + k, sv[k]);
  }
}

// a'_ij = (a_ij * s_i) * s_j, b'_i = b_i * s_i (reading S1)

// Staged like gs_kernel: the 256-row window's values and columns arrive in shared
// memory with cp.async, each thread scales its row there (the column factor is a
// gather of s), and the window is written back coalesced.
__global__ void __launch_bounds__(TB) sym_scale_kernel(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                                       const double* vin, double* vout, const double* b,
                                                       double* bout, const double* __restrict__ sv) {
  __shared__ double sval[CSR_CAP];
  __shared__ int scol[CSR_CAP];
  const int r0 = blockIdx.x * TB, t = threadIdx.x, r = r0 + t;
  const int rend = min(r0 + TB, n);
  const int s0 = __ldg(rp + r0), s1 = __ldg(rp + rend), cnt = s1 - s0;
  const bool staged = cnt <= CSR_CAP;
  if (staged) {
    for (int k = t; k < cnt; k += TB) {
      cp_async8(sval + k, vin + s0 + k);
      cp_async4(scol + k, ci + s0 + k);
    }
    cp_async_commit();
  }
  int a0 = 0, a1 = 0;
  double si = 0.0, bi = 0.0;
  if (r < n) {
    a0 = __ldg(rp + r);
    a1 = __ldg(rp + r + 1);
    si = sv[r];
    if (b && bout) bi = __ldcs(b + r);
  }
  if (staged) {
    cp_async_wait<0>();
    __syncthreads();
  }
  if (r < n) {
    if (staged) {
      for (int k = a0 - s0; k < a1 - s0; ++k) sval[k] = (sval[k] * si) * __ldg(sv + scol[k]);
    } else {
      for (int k = a0; k < a1; ++k) vout[k] = (vin[k] * si) * __ldg(sv + ci[k]);
    }
    if (b && bout) __stcs(bout + r, bi * si);
  }
  if (staged) {
    __syncthreads();
    for (int k = t; k < cnt; k += TB) __stcs(vout + s0 + k, sval[k]);
  }
}

__global__ void unscale_kernel(int64_t n, const double* s, const double* y, double* x) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = s[i] * y[i];
}

static int launch_gs(int grid, cudaStream_t s, int n, const int* rp, const double* vin, double* vout,
                     const double* b, double* bout, double* dout, int p, int* bad, int norms_only) {
  if (p == 2)
    gs_kernel<2><<<grid, TB, 0, s>>>(n, rp, vin, vout, b, bout, dout, p, bad, norms_only);
  else if (p == 1)
    gs_kernel<1><<<grid, TB, 0, s>>>(n, rp, vin, vout, b, bout, dout, p, bad, norms_only);
  else
    gs_kernel<0><<<grid, TB, 0, s>>>(n, rp, vin, vout, b, bout, dout, p, bad, norms_only);
  return GSK_OK;
}

// One device word per GPU for the zero-row flag (avoids a stream-ordered allocation per
// call).  Calls hold that device's mutex from the reset to the read-back, so concurrent
// callers on different streams / host threads never share a flag; calls on different
// devices do not wait for each other.
constexpr int kMaxDevices = 64;
static std::mutex g_flag_mu[kMaxDevices];
static int current_dev() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}
static int* zero_row_flag(int dev, int* err) {
  static int* flag[kMaxDevices] = {};
  if (dev < 0 || dev >= kMaxDevices || (!flag[dev] && cudaMalloc(&flag[dev], sizeof(int)) != cudaSuccess)) {
    *err = 1;
    return nullptr;
  }
  return flag[dev];
}

}  // namespace gsk

using namespace gsk;

extern "C" int gsk_gs_scale_sym(const gsk_csr* A, const double* b, int p, double* values_out,
                                double* b_out, double* s_out, int32_t* bad_row, void* stream) {
  NvtxRange nv("gsk:gs_scale_sym");
  if (!A || A->n < 1 || A->nnz < 0 || !A->row_ptr || !s_out ||
      (A->nnz > 0 && (!A->values || !values_out || !A->col_idx))) {
    set_error("gsk_gs_scale_sym: invalid arguments");
    return GSK_E_INVALID;
  }
  if (p < 1) {
    set_error("gsk_gs_scale_sym: p must be >= 1 (got %d)", p);
    return GSK_E_INVALID;
  }
  if (values_out == A->values || (b_out && b_out == b)) {
    set_error("gsk_gs_scale_sym: outputs must not alias inputs (column scaling reads other rows)");
    return GSK_E_INVALID;
  }
  cudaStream_t s = as_stream(stream);
  const int dev = current_dev();
  if (dev < 0 || dev >= kMaxDevices) {
    set_error("gs: device ordinal %d out of range", dev);
    return GSK_E_INVALID;
  }
  std::lock_guard<std::mutex> lock(g_flag_mu[dev]);
  int ferr = 0;
  int* dbad = zero_row_flag(dev, &ferr);
  if (ferr) {
    set_error("gs: cannot allocate the zero-row flag");
    return GSK_E_NOMEM;
  }
  const int big = 0x7f7f7f7f;  // > any row index; set by a byte memset (no host copy)
  GSK_CUDA(cudaMemsetAsync(dbad, 0x7f, sizeof(int), s));
  const int grid = (A->n + TB - 1) / TB;
  GSK_TRY(launch_gs(grid, s, A->n, A->row_ptr, A->values, nullptr, nullptr, nullptr, s_out, p, dbad, 1));
  GSK_LAUNCHED(1);
  int hbad = big;
  GSK_CUDA(cudaMemcpyAsync(&hbad, dbad, sizeof(int), cudaMemcpyDeviceToHost, s));
  GSK_CUDA(cudaStreamSynchronize(s));
  if (hbad != big) {
    if (bad_row) *bad_row = hbad;
    set_error("gsk_gs_scale_sym: row %d has zero L_%d norm", hbad, p);
    return GSK_E_ZERO_ROW;
  }
  sym_scale_kernel<<<grid, TB, 0, s>>>(A->n, A->row_ptr, A->col_idx, A->values, values_out, b, b_out, s_out);
  GSK_LAUNCHED(1);
  GSK_CUDA(cudaStreamSynchronize(s));
  return GSK_OK;
}

extern "C" int gsk_gs_unscale(int64_t n, const double* s_in, const double* y, double* x, void* stream) {
  if (n < 1 || !s_in || !y || !x) {
    set_error("gsk_gs_unscale: invalid arguments");
    return GSK_E_INVALID;
  }
  cudaStream_t s = as_stream(stream);
  unscale_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, s_in, y, x);
  GSK_LAUNCHED(1);
  GSK_CUDA(cudaStreamSynchronize(s));
  return GSK_OK;
}

extern "C" int gsk_gs_scale(const gsk_csr* A, const double* b, int p, double* values_out,
                            double* b_out, double* d_out, int32_t* bad_row, void* stream) {
  NvtxRange nv("gsk:gs_scale");
  if (!A || A->n < 1 || A->nnz < 0 || !A->row_ptr || (A->nnz > 0 && (!A->values || !values_out))) {
    set_error("gsk_gs_scale: invalid matrix");
    return GSK_E_INVALID;
  }
  if (p < 1) {
    set_error("gsk_gs_scale: p must be >= 1 (got %d)", p);
    return GSK_E_INVALID;
  }
  if ((b_out && !b)) {
    set_error("gsk_gs_scale: b_out given without b");
    return GSK_E_INVALID;
  }
  cudaStream_t s = as_stream(stream);
  const int dev = current_dev();
  if (dev < 0 || dev >= kMaxDevices) {
    set_error("gs: device ordinal %d out of range", dev);
    return GSK_E_INVALID;
  }
  std::lock_guard<std::mutex> lock(g_flag_mu[dev]);
  int ferr = 0;
  int* dbad = zero_row_flag(dev, &ferr);
  if (ferr) {
    set_error("gs: cannot allocate the zero-row flag");
    return GSK_E_NOMEM;
  }
  const int big = 0x7f7f7f7f;  // > any row index; set by a byte memset (no host copy)
  GSK_CUDA(cudaMemsetAsync(dbad, 0x7f, sizeof(int), s));
  const int grid = (A->n + TB - 1) / TB;
  GSK_TRY(launch_gs(grid, s, A->n, A->row_ptr, A->values, values_out, b, b_out, d_out, p, dbad, 0));
  GSK_LAUNCHED(1);
  int hbad = big;
  GSK_CUDA(cudaMemcpyAsync(&hbad, dbad, sizeof(int), cudaMemcpyDeviceToHost, s));
  GSK_CUDA(cudaStreamSynchronize(s));
  if (hbad != big) {
    if (bad_row) *bad_row = hbad;
    set_error("gsk_gs_scale: row %d has zero L_%d norm", hbad, p);
    return GSK_E_ZERO_ROW;
  }
  return GSK_OK;
}
