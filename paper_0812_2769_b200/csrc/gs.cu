// gs.cu — GS(p): divide each row of A and its entry of b by the row's L_p norm.
//   PAPER.md:92-97 (definition), Eq. (2) PAPER.md:207-214 (DAx = Db, D = diag(1/||a_i||_p)).
// One pass over the nnz: a CTA owns 256 consecutive rows; their value segment is
// staged into shared memory with coalesced loads, each thread reduces its own row
// segment in ascending column order (AC-4: p=2 fma chain + sqrt, p=1 running sum of
// |a|, p>=3 repeated products + pow), the segment is rescaled in shared memory and
// written back coalesced.  Bytes: 16 nnz + 4(n+1) + 24 n (read a, write a, r/w b, d).
#include "internal.cuh"

namespace gsk {

__device__ __forceinline__ double row_norm_term(double a, int p) {
  const double m = fabs(a);
  double t = m;
  for (int e = 1; e < p; ++e) t = t * m;
  return t;
}

__global__ void __launch_bounds__(TB) gs_kernel(int n, const int* __restrict__ rp,
                                                const double* vin, double* vout,
                                                const double* b, double* bout, double* dout,
                                                int p, int* bad) {
  __shared__ double sv[CSR_CAP];
  const int r0 = blockIdx.x * TB, t = threadIdx.x, r = r0 + t;
  const int rend = min(r0 + TB, n);
  const int s0 = rp[r0], s1 = rp[rend], cnt = s1 - s0;
  const bool staged = cnt <= CSR_CAP;
  if (staged) {
    for (int k = t; k < cnt; k += TB) sv[k] = __ldcs(vin + s0 + k);
    __syncthreads();
  }
  double d = 0.0;
  if (r < n) {
    const int a0 = rp[r], a1 = rp[r + 1];
    const double* seg = staged ? sv + (a0 - s0) : vin + a0;
    const int len = a1 - a0;
    double acc = 0.0;
    if (p == 2) {
      for (int k = 0; k < len; ++k) acc = __fma_rn(seg[k], seg[k], acc);
    } else if (p == 1) {
      for (int k = 0; k < len; ++k) acc = acc + fabs(seg[k]);
    } else {
      for (int k = 0; k < len; ++k) acc = acc + row_norm_term(seg[k], p);
    }
    const double nrm = (p == 1) ? acc : (p == 2 ? sqrt(acc) : pow(acc, 1.0 / p));
    if (nrm == 0.0) {
      atomicMin(bad, r);
    } else {
      d = 1.0 / nrm;
    }
    if (staged) {
      double* sg = sv + (a0 - s0);
      for (int k = 0; k < len; ++k) sg[k] = sg[k] * d;
    } else {
      for (int k = 0; k < len; ++k) vout[a0 + k] = vin[a0 + k] * d;
    }
    if (b && bout) bout[r] = b[r] * d;
    if (dout) dout[r] = d;
  }
  if (staged) {
    __syncthreads();
    for (int k = t; k < cnt; k += TB) __stcs(vout + s0 + k, sv[k]);
  }
}

}  // namespace gsk

using namespace gsk;

extern "C" int gsk_gs_scale(const gsk_csr* A, const double* b, int p, double* values_out,
                            double* b_out, double* d_out, int32_t* bad_row, void* stream) {
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
  int* dbad = nullptr;
  GSK_CUDA(cudaMallocAsync(&dbad, sizeof(int), s));
  const int big = 0x7fffffff;
  GSK_CUDA(cudaMemcpyAsync(dbad, &big, sizeof(int), cudaMemcpyHostToDevice, s));
  const int grid = (A->n + TB - 1) / TB;
  gs_kernel<<<grid, TB, 0, s>>>(A->n, A->row_ptr, A->values, values_out, b, b_out, d_out, p, dbad);
  GSK_LAUNCHED(1);
  int hbad = big;
  GSK_CUDA(cudaMemcpyAsync(&hbad, dbad, sizeof(int), cudaMemcpyDeviceToHost, s));
  GSK_CUDA(cudaFreeAsync(dbad, s));
  GSK_CUDA(cudaStreamSynchronize(s));
  if (hbad != big) {
    if (bad_row) *bad_row = hbad;
    set_error("gsk_gs_scale: row %d has zero L_%d norm", hbad, p);
    return GSK_E_ZERO_ROW;
  }
  return GSK_OK;
}
