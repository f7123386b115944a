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

// Same sweeps for the reference's fixed structure (deriv offsets -3, -1, 1),
// with every row a step reads arriving through a cp.async ring in shared
// memory issued kRecRing - 1 steps ahead: forward -- the one u row that
// enters the (k-3, k-1, k+1) window, plus the step's 3 + 2 operator / factor
// entries (per warp, one lane each, read as broadcasts); backward -- the
// parked y row and the g row, plus 2 factor entries.  (The per-line walk
// above waits a global latency inside every step: ~1.8 TB/s.)  Warps are
// single-parity (lines padded to a multiple of 32).  Same operations in the
// same order as recover_kernel, except that the four divisions by z2 per row
// are one reciprocal per line and four products (fp64 division is a ~30
// instruction sequence; ncu: the kernel was issue-bound on them) -- within
// an ulp, like LAPACK's own rounding differences (tests gate 1e-12).
#ifndef SHEN_REC_RING
#define SHEN_REC_RING 10
#endif
constexpr int kRecRing = SHEN_REC_RING;  // 16-32 B per step and thread: a deep ring keeps enough bytes in flight
constexpr int kRecThreads = 128;
constexpr int kRecTab = 5;

__device__ __forceinline__ void rcp16(void* dst, const void* src, bool pred) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(pred ? 16 : 0) : "memory");
}
__device__ __forceinline__ void rcp8(void* dst, const void* src, bool pred) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(pred ? 8 : 0) : "memory");
}
template <int N>
__device__ __forceinline__ void rwait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }
__device__ __forceinline__ void rcommit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }

__global__ void __launch_bounds__(kRecThreads) recover_ring_kernel(RecoverArgs a, int64_t Lp) {
  __shared__ __align__(16) double2 rows[kRecRing][2][kRecThreads];
  __shared__ __align__(16) double tabs[kRecRing][kRecThreads / 32][kRecTab];
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int par = t >= Lp ? 1 : 0;
  const int64_t l_raw = t - (int64_t)par * Lp;
  const bool live = l_raw < a.L && t < 2 * Lp;
  if (!__any_sync(0xffffffffu, live)) return;
  const int64_t l = live ? l_raw : 0;
  const int64_t L = a.L;
  const int n = a.n_dir, nr = a.d.nr, nc = a.d.nc;
  const int m = (n - par + 1) / 2;
  const double* ab = a.fac + (int64_t)par * 2 * a.mmax;  // upper band storage, nband = 1
  const double2* u = static_cast<const double2*>(a.u) + l;
  const double2* g = static_cast<const double2*>(a.g) + l;
  double2* vout = static_cast<double2*>(a.v) + l;
  double2* wout = static_cast<double2*>(a.w) + l;
  // ---------------- forward: U^T y = D u (y parked in v)
  // step i: row k = par + 2 i; u window rows k-3, k-1 carried, row k+1 from the ring
  auto fissue = [&](int i) {
    const int s = i % kRecRing, k = par + 2 * i, j = k + 1;
    const bool on = live && i < m && j < nc;
    rcp16(&rows[s][0][tid], u + (on ? (int64_t)j * L : 0), on);
    if (lane < kRecTab) {
      // lanes 0..2: deriv entries q at row k; 3: U(i-1, i); 4: U(i, i)
      const double* src = lane < 3 ? a.d.diag + (int64_t)lane * nr + k : ab + (lane == 3 ? 0 : a.mmax) + i;
      const bool ot = i < m && (lane < 3 ? k < nr : true);
      rcp8(&tabs[s][wid][lane], ot ? src : ab, ot);
    }
    rcommit();
  };
#pragma unroll
  for (int i = 0; i < kRecRing - 1; ++i) fissue(i);
  auto uval = [&](int j) -> Z { return (j >= 0 && j < nc) ? zld(u + (int64_t)j * L) : Z{0.0, 0.0}; };
  Z wm3 = uval(par - 3), wm1 = uval(par - 1);  // rows k-3, k-1
  Z y1 = {0.0, 0.0};
  for (int i = 0; i < m; ++i) {
    const int k = par + 2 * i;
    rwait<kRecRing - 2>();
    __syncwarp();
    const int s = i % kRecRing;
    const double* tv = tabs[s][wid];
    const Z wp1 = zld(&rows[s][0][tid]);
    // (D u)[k], offsets -3, -1, 1 in the reference's order
    Z acc = {0.0, 0.0};
    const Z xs[3] = {wm3, wm1, wp1};
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int dk = 2 * q - 3;
      const int k0 = dk < 0 ? -dk : 0, k1 = min(nr, nc - dk);
      if (k >= k0 && k < k1)
        acc = {__dadd_rn(acc.re, __dmul_rn(tv[q], xs[q].re)), __dadd_rn(acc.im, __dmul_rn(tv[q], xs[q].im))};
    }
    if (i >= 1) acc = zsub(acc, zscale(tv[3], y1));
    const Z y = zscale(1.0 / tv[4], acc);
    if (live) vout[(int64_t)k * L] = make_double2(y.re, y.im);
    y1 = y;
    wm3 = wm1;
    wm1 = wp1;
    fissue(i + kRecRing - 1);
  }
  rwait<0>();
  __syncwarp();
  // ---------------- backward: U f = y, then v, w of the row
  // step b: i = m - 1 - b, row k = par + 2 i: parked y and g rows, U(i, i+1), U(i, i)
  auto bissue = [&](int b) {
    const int s = b % kRecRing, i = m - 1 - b, k = par + 2 * i;
    const bool on = live && i >= 0;
    rcp16(&rows[s][0][tid], vout + (on ? (int64_t)k * L : 0), on);
    rcp16(&rows[s][1][tid], g + (on ? (int64_t)k * L : 0), on);
    if (lane < 2) {
      const bool ot = i >= 0 && (lane == 1 || i + 1 < m);
      rcp8(&tabs[s][wid][lane], ot ? ab + (lane == 0 ? i + 1 : a.mmax + i) : ab, ot);
    }
    rcommit();
  };
#pragma unroll
  for (int b = 0; b < kRecRing - 1; ++b) bissue(b);
  const Z im_m = {__ldg(a.im_m_re + l), __ldg(a.im_m_im + l)}, im_n = {__ldg(a.im_n_re + l), __ldg(a.im_n_im + l)};
  const double rsz = 1.0 / __ldg(a.safe_z2 + l);  // one division per line, not four per row
  Z x1 = {0.0, 0.0};
  for (int b = 0; b < m; ++b) {
    const int i = m - 1 - b, k = par + 2 * i;
    rwait<kRecRing - 2>();
    __syncwarp();
    const int s = b % kRecRing;
    const double* tv = tabs[s][wid];
    Z acc = zld(&rows[s][0][tid]);
    if (i + 1 < m) acc = zsub(acc, zscale(tv[0], x1));
    const Z f = zscale(1.0 / tv[1], acc);
    x1 = f;
    const Z gk = zld(&rows[s][1][tid]);
    const Z vn = zadd(zmul(im_m, f), zmul(im_n, gk));
    const Z wn = zsub(zmul(im_n, f), zmul(im_m, gk));
    if (live) {
      vout[(int64_t)k * L] = make_double2(vn.re * rsz, vn.im * rsz);
      wout[(int64_t)k * L] = make_double2(wn.re * rsz, wn.im * rsz);
    }
    bissue(b + kRecRing - 1);
  }
  rwait<0>();
}

}  // namespace

cudaError_t launch_recover(const RecoverArgs& a, cudaStream_t st) {
  if (a.L <= 0 || a.n_dir <= 0) return cudaSuccess;
  const bool fixed = a.d.n_off == 3 && a.d.off[0] == -3 && a.d.off[1] == -1 && a.d.off[2] == 1;
  if (fixed) {
    const int64_t Lp = (a.L + 31) / 32 * 32;  // single-parity warps
    recover_ring_kernel<<<(unsigned)((2 * Lp + kRecThreads - 1) / kRecThreads), kRecThreads, 0, st>>>(a, Lp);
  } else {
    recover_kernel<<<(unsigned)((2 * a.L + 127) / 128), 128, 0, st>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace shen
