// Stored-factor solves, one thread per (system, parity), evaluated in the
// reference's exact operation order (solvers.py:100-126 and 162-198):
// with EXACT factors from shen_factor.cu the results are bit-identical to
// chebchan.  y is staged in the output array (written by the forward sweep,
// read back and overwritten by x in the backward sweep), so each thread
// streams its column twice.  This is the reference-faithful path (and the
// one small batches use); the chunked fused solve is the fast path.
#include "shen_common.cuh"
#include "shen_kernels.h"

namespace shen {

// numpy complex / real division is Smith's algorithm, which for a real
// divisor reduces to multiplication by the correctly rounded reciprocal;
// real / real is a true division.
__device__ __forceinline__ cplx div_ref(cplx a, double d) {
  const double r = __drcp_rn(d);
  return {__dmul_rn(a.re, r), __dmul_rn(a.im, r)};
}
__device__ __forceinline__ double div_ref(double a, double d) { return __ddiv_rn(a, d); }

template <typename V>
__global__ void __launch_bounds__(256) helm_seq_kernel(HelmSeqArgs a) {
  using O = VOps<V>;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= 2 * a.batch) return;
  const int par = (int)(tid / a.batch);
  const int64_t j = tid - (int64_t)par * a.batch;
  const int64_t B = a.batch;
  const int n = (a.n_dir - par + 1) / 2;
  const V* rhs = static_cast<const V*>(a.rhs);
  V* out = static_cast<V*>(a.out);
  auto at = [&](int i) { return (int64_t)(par + 2 * i) * B + j; };
  const double* low = a.low[par];
  const double* d = a.d[par];
  const double* e = a.e[par];
  const double* t = a.t[par];
  V y = O::ld(rhs + at(0));
  O::st(out + at(0), y);
  for (int i = 1; i < n; ++i) {
    y = O::sub_sc(O::ld(rhs + at(i)), low[(int64_t)(i - 1) * B + j], y);
    O::st(out + at(i), y);
  }
  V x1 = div_ref(out[at(n - 1)], d[(int64_t)(n - 1) * B + j]);
  out[at(n - 1)] = x1;
  if (n > 1) {
    V x0 = div_ref(O::sub_sc(out[at(n - 2)], e[(int64_t)(n - 2) * B + j], x1), d[(int64_t)(n - 2) * B + j]);
    out[at(n - 2)] = x0;
    V x2 = x1;
    x1 = x0;
    V run = O::zero();
    for (int i = n - 3; i >= 0; --i) {
      run = O::add(run, x2);
      const int64_t r = (int64_t)i * B + j;
      V acc = O::sub_sc(O::sub_sc(out[at(i)], e[r], x1), t[r], run);
      V x = div_ref(acc, d[r]);
      out[at(i)] = x;
      x2 = x1;
      x1 = x;
    }
  }
}

template <typename V>
__global__ void __launch_bounds__(256) bih_seq_kernel(BihSeqArgs a) {
  using O = VOps<V>;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= 2 * a.batch) return;
  const int par = (int)(tid / a.batch);
  const int64_t j = tid - (int64_t)par * a.batch;
  const int64_t B = a.batch;
  const int n = (a.n_bih - par + 1) / 2;
  const V* rhs = static_cast<const V*>(a.rhs);
  V* out = static_cast<V*>(a.out);
  auto at = [&](int i) { return (int64_t)(par + 2 * i) * B + j; };
  const double *low2 = a.low2[par], *low4 = a.low4[par];
  const double *d = a.d[par], *e = a.e[par], *f = a.f[par], *av = a.a[par], *bv = a.b[par];
  // forward: y_i = rhs_i - low2[i-1] y_{i-1} - low4[i-2] y_{i-2}
  V y2 = O::zero(), y1 = O::ld(rhs + at(0));
  O::st(out + at(0), y1);
  if (n > 1) {
    V y = O::sub_sc(O::ld(rhs + at(1)), low2[j], y1);
    O::st(out + at(1), y);
    y2 = y1;
    y1 = y;
  }
  for (int i = 2; i < n; ++i) {
    V y = O::sub_sc(O::sub_sc(O::ld(rhs + at(i)), low2[(int64_t)(i - 1) * B + j], y1), low4[(int64_t)(i - 2) * B + j],
                    y2);
    O::st(out + at(i), y);
    y2 = y1;
    y1 = y;
  }
  // backward with the two running tail sums (Alg. 4)
  V x1 = O::zero(), x2 = O::zero(), x3 = O::zero();
  V sq = O::zero(), ss = O::zero();
  for (int i = n - 1; i >= 0; --i) {
    const int64_t r = (int64_t)i * B + j;
    const int k = par + 2 * i;
    V acc = out[at(i)];
    if (i + 1 < n) acc = O::sub_sc(acc, e[r], x1);
    if (i + 2 < n) acc = O::sub_sc(acc, f[r], x2);
    if (i + 3 < n) {
      sq = O::add(sq, O::scale(a.q[k + 6], x3));
      ss = O::add(ss, O::scale(a.s[k + 6], x3));
      V t = O::add(O::scale(av[r], sq), O::scale(bv[r], ss));
      acc = O::sub(acc, O::scale(a.xi0, t));
    }
    V x = div_ref(acc, d[r]);
    out[at(i)] = x;
    x3 = x2;
    x2 = x1;
    x1 = x;
  }
}

cudaError_t launch_helm_seq(const HelmSeqArgs& a, bool cplx_rhs, cudaStream_t st) {
  if (a.batch <= 0) return cudaSuccess;
  const unsigned blocks = (unsigned)((2 * a.batch + 255) / 256);
  if (cplx_rhs)
    helm_seq_kernel<cplx><<<blocks, 256, 0, st>>>(a);
  else
    helm_seq_kernel<double><<<blocks, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_bih_seq(const BihSeqArgs& a, bool cplx_rhs, cudaStream_t st) {
  if (a.batch <= 0) return cudaSuccess;
  const unsigned blocks = (unsigned)((2 * a.batch + 255) / 256);
  if (cplx_rhs)
    bih_seq_kernel<cplx><<<blocks, 256, 0, st>>>(a);
  else
    bih_seq_kernel<double><<<blocks, 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace shen
