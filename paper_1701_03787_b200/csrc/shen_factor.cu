// Factorisation kernels: one thread per (wavenumber system, parity), the row
// recurrence of the reference walked sequentially (solvers.py:201-241 and
// 271-355).  Lanes map to consecutive systems, so every warp touches the
// same row constants (broadcast loads) and writes coalesced 256-B rows.
//
// Outputs (any subset):
//   * full compressed factors (reference layout, EXACT mode) -- the lazy
//     HelmholtzLU.low/d/e/tail and BiharmonicLU.low2/.../b attributes;
//   * chunk checkpoints (FAST mode) -- the factor state entering every
//     chunk of R rows, consumed by the chunked solve;
//   * the first near-zero pivot row per parity (ZeroPivotError).
#include "shen_rows.cuh"
#include "shen_kernels.h"

namespace shen {

template <bool EXACT>
__global__ void __launch_bounds__(256) helm_factor_kernel(HelmFactorArgs a) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= 2 * a.batch) return;
  const int par = (int)(tid / a.batch);
  const int64_t j = tid - (int64_t)par * a.batch;
  const int n = (a.n_dir - par + 1) / 2;  // rows of this parity
  const int nsup = (a.n_dir - 2 - par + 1) / 2 > 0 ? (a.n_dir - 2 - par + 1) / 2 : 0;
  const double cb = __ldg(a.cb + j);
  const double sub = __dmul_rn(cb, -1.5707963267948966);  // cb * (-pi/2)
  const int64_t B = a.batch;
  const int R = a.chunk_rows > 0 ? a.chunk_rows : (1 << 30);
  HelmState s{0, 0, 0};
  HelmProj pj{0, 0, 0, 0, 0};
  double dl = 0.0, el = 0.0, tl = 0.0;  // ratios of the last row (fast mode)
  for (int i = 0; i < n; ++i) {
    const int k = par + 2 * i;
    HelmRow h = helm_row(a.ca, cb, sub, __ldg(a.sd + k), __ldg(a.st + k), __ldg(a.md + k), i < nsup);
    double low, d, e, t;
    if (EXACT) {
      low = helm_step_exact(s, h, sub, i == 0);
      d = s.d; e = s.e; t = s.t;
    } else {
      const int r = i % R;
      if (i == 0) hp_origin(pj);
      else if (r == 0) hp_start(pj, dl, el, tl);
      else if ((r & 7) == 0) hp_rescale(pj);
      low = hp_step(pj, h, sub, d, e, t);
      dl = d; el = e; tl = t;
    }
    note_pivot(a.pivot, par, i, d);
    if (a.low[par] != nullptr) {
      if (i > 0) a.low[par][(int64_t)(i - 1) * B + j] = low;
      a.d[par][(int64_t)i * B + j] = d;
      a.e[par][(int64_t)i * B + j] = e;
      a.t[par][(int64_t)i * B + j] = t;
    }
    if (a.ckpt != nullptr && (i + 1) % R == 0 && i + 1 < n) {
      const int c = (i + 1) / R;
      double* base = a.ckpt + ((int64_t)(c * 2 + par) * 3) * B + j;
      base[0] = d;
      base[B] = e;
      base[2 * B] = t;
    }
  }
}

template <bool EXACT>
__global__ void __launch_bounds__(256) bih_factor_kernel(BihFactorArgs a) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= 2 * a.batch) return;
  const int par = (int)(tid / a.batch);
  const int64_t j = tid - (int64_t)par * a.batch;
  const int n = (a.n_bih - par + 1) / 2;
  const double xi1 = __ldg(a.xi1 + j), xi2 = __ldg(a.xi2 + j);
  const int64_t B = a.batch;
  BihU u{0, 0, 0, 0, 0, 0}, u1{0, 0, 0, 0, 0, 0}, u2{0, 0, 0, 0, 0, 0};
  double c[B_NCOL];
  for (int i = 0; i < n; ++i) {
    const int k = par + 2 * i;
    load_bih_row(a.tab, k, c);
    double l2, l4;
    if (EXACT) {
      const BihBands h = bih_bands(a.xi0, xi1, xi2, c);
      bih_step_exact(u, u1, u2, h, c, a.xi0, i, l2, l4);
    } else {
      bih_fast_prescale(c, a.xi0);
      const BihBands h = bih_bands_fast(xi1, xi2, c);
      bih_step_fast(u, u1, u2, h, c, l2, l4);
    }
    note_pivot(a.pivot, par, i, u.d);
    if (a.d[par] != nullptr) {
      if (i >= 1) a.low2[par][(int64_t)(i - 1) * B + j] = l2;
      if (i >= 2) a.low4[par][(int64_t)(i - 2) * B + j] = l4;
      a.d[par][(int64_t)i * B + j] = u.d;
      a.e[par][(int64_t)i * B + j] = u.e;
      a.f[par][(int64_t)i * B + j] = u.f;
      a.a[par][(int64_t)i * B + j] = u.a;
      a.b[par][(int64_t)i * B + j] = u.b;
    }
    u2 = u1;
    u1 = u;
    if (a.ckpt != nullptr && a.chunk_rows > 0 && (i + 1) % a.chunk_rows == 0 && i + 1 < n) {
      const int cc = (i + 1) / a.chunk_rows;
      double* base = a.ckpt + ((int64_t)(cc * 2 + par) * 10) * B + j;
      base[0] = u1.d; base[B] = u1.e; base[2 * B] = u1.f; base[3 * B] = u1.a; base[4 * B] = u1.b;
      base[5 * B] = u2.d; base[6 * B] = u2.e; base[7 * B] = u2.f; base[8 * B] = u2.a; base[9 * B] = u2.b;
    }
  }
}

cudaError_t launch_helm_factor(const HelmFactorArgs& a, bool exact, cudaStream_t st) {
  if (a.batch <= 0) return cudaSuccess;
  const int threads = 256;
  const int64_t blocks = (2 * a.batch + threads - 1) / threads;
  if (exact)
    helm_factor_kernel<true><<<(unsigned)blocks, threads, 0, st>>>(a);
  else
    helm_factor_kernel<false><<<(unsigned)blocks, threads, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_bih_factor(const BihFactorArgs& a, bool exact, cudaStream_t st) {
  if (a.batch <= 0) return cudaSuccess;
  const int threads = 256;
  const int64_t blocks = (2 * a.batch + threads - 1) / threads;
  if (exact)
    bih_factor_kernel<true><<<(unsigned)blocks, threads, 0, st>>>(a);
  else
    bih_factor_kernel<false><<<(unsigned)blocks, threads, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace shen
