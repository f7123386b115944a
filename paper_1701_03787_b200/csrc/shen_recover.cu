// Divergence variable and horizontal-velocity recovery of the stepper
// (reference stepper.py:296-303), fused per line:
//
//   f_scal = D u                 D = deriv_bih_to_dir (banded, odd offsets)
//   f      = B_D^-1 f_scal       per-parity banded Cholesky (transforms.py:163-175)
//   v      = (1j m f + 1j n g) / z2'      w = (1j n f - 1j m g) / z2'
//   (z2' = z2, or 1 on the mean mode, which the stepper then overwrites)
//
// One thread per (line, parity): the forward Cholesky sweep consumes D u
// rows as they are formed and parks y in v's storage; the backward sweep
// reads it back, produces f row by row and writes v and w directly -- u and
// g are read once, v and w written once (plus the y round trip in L2/HBM).
// The reference materialises f_scal, f (LAPACK zpbtrs) and six temporaries.
#include <cuda_runtime.h>
#include <stdint.h>

#include "shen_kernels.h"

namespace shen {
namespace {

struct Z {
  double re, im;
};
__device__ __forceinline__ Z zld(const double2* p) {
  const double2 v = *p;
  return {v.x, v.y};
}
__device__ __forceinline__ Z zadd(Z a, Z b) { return {a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ Z zsub(Z a, Z b) { return {a.re - b.re, a.im - b.im}; }
__device__ __forceinline__ Z zscale(double c, Z v) { return {c * v.re, c * v.im}; }
__device__ __forceinline__ Z zmul(Z a, Z b) {
  return {__dsub_rn(__dmul_rn(a.re, b.re), __dmul_rn(a.im, b.im)), __dadd_rn(__dmul_rn(a.re, b.im), __dmul_rn(a.im, b.re))};
}

__global__ void recover_kernel(RecoverArgs a) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 2 * a.L) return;
  const int par = (int)(t / a.L);
  const int64_t l = t - (int64_t)par * a.L;
  const int64_t L = a.L;
  const int n = a.n_dir;
  const int m = (n - par + 1) / 2;
  const double* ab = a.fac + (int64_t)par * 2 * a.mmax;  // upper band storage, nband = 1
  auto U = [&](int i, int j) -> double { return __ldg(ab + (int64_t)(1 - (j - i)) * a.mmax + j); };
  const double2* u = static_cast<const double2*>(a.u) + l;
  auto Du = [&](int k) -> Z {  // (D u)[k], offsets in the reference's order
    Z v = {0.0, 0.0};
    for (int q = 0; q < a.d.n_off; ++q) {
      const int dk = a.d.off[q];
      const int k0 = dk < 0 ? -dk : 0, k1 = min(a.d.nr, a.d.nc - dk);
      if (k >= k0 && k < k1) {
        const double c = __ldg(a.d.diag + (int64_t)q * a.d.nr + k);
        const Z x = zld(u + (int64_t)(k + dk) * L);
        v = {__dadd_rn(v.re, __dmul_rn(c, x.re)), __dadd_rn(v.im, __dmul_rn(c, x.im))};
      }
    }
    return v;
  };
  double2* vout = static_cast<double2*>(a.v) + l;
  double2* wout = static_cast<double2*>(a.w) + l;
  const double2* g = static_cast<const double2*>(a.g) + l;
  // forward: U^T y = D u (y parked in v)
  Z y1 = {0.0, 0.0};
  for (int i = 0; i < m; ++i) {
    const int k = par + 2 * i;
    Z acc = Du(k);
    if (i >= 1) acc = zsub(acc, zscale(U(i - 1, i), y1));
    const Z y = zscale(1.0 / U(i, i), acc);
    vout[(int64_t)k * L] = make_double2(y.re, y.im);
    y1 = y;
  }
  // backward: U f = y, then v, w of the row
  const Z im_m = {__ldg(a.im_m_re + l), __ldg(a.im_m_im + l)}, im_n = {__ldg(a.im_n_re + l), __ldg(a.im_n_im + l)};
  const double sz = __ldg(a.safe_z2 + l);
  Z x1 = {0.0, 0.0};
  for (int i = m - 1; i >= 0; --i) {
    const int k = par + 2 * i;
    Z acc = zld(vout + (int64_t)k * L);
    if (i + 1 < m) acc = zsub(acc, zscale(U(i, i + 1), x1));
    const Z f = zscale(1.0 / U(i, i), acc);
    x1 = f;
    const Z gk = zld(g + (int64_t)k * L);
    const Z vn = zadd(zmul(im_m, f), zmul(im_n, gk));
    const Z wn = zsub(zmul(im_n, f), zmul(im_m, gk));
    vout[(int64_t)k * L] = make_double2(__ddiv_rn(vn.re, sz), __ddiv_rn(vn.im, sz));
    wout[(int64_t)k * L] = make_double2(__ddiv_rn(wn.re, sz), __ddiv_rn(wn.im, sz));
  }
}

}  // namespace

cudaError_t launch_recover(const RecoverArgs& a, cudaStream_t st) {
  if (a.L <= 0 || a.n_dir <= 0) return cudaSuccess;
  recover_kernel<<<(unsigned)((2 * a.L + 127) / 128), 128, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace shen
