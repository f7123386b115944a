// Pointwise pieces of the nonlinear term H = u x omega (reference
// stepper.py:148-185), SURVEY.md 8(f) rank 3.  The transforms around them are
// the wall-normal operator GEMMs and cuFFT (nonlinear.py).
//
//   shen_scale_lines: y[r, l] = c_l * x[r, l] (complex, products rounded separately):
//                     the 1j m / 1j n derivative factors and the dealiasing
//                     mask, one per Fourier line;
//   shen_cross:       om_y = du_dz - dw_dx, om_z = dv_dx - du_dy and
//                     h = (v om_z - w om_y, w om_x - u om_z, u om_y - v om_x)
//                     on the physical grid, in the reference's operation order
//                     (8 fields in, 3 out: one HBM pass);
//   shen_cross_paired: the same on fields held as symmetric / antisymmetric
//                     parts about the channel centre (x -> -x pairs the
//                     wall-normal points j and N-1-j): reads e, o of each
//                     field, forms the values at both points of a pair, and
//                     writes h's symmetric / antisymmetric parts -- so both
//                     wall-normal operators act on half the modes (GEMMs of
//                     half the flops) with no extra pass;
//   shen_pair_split / shen_pair_merge: the same pairing for the 3-D
//                     transforms (one elementwise pass on each side of the
//                     half-size operator GEMMs);
//   shen_scale_rows:  scale_lines with row strides (the even / odd
//                     coefficient rows of the paired forward operator are
//                     interleaved while the mask is applied).
#include <cuda_runtime.h>
#include <stdint.h>

#include "shen_kernels.h"

namespace shen {
namespace {

__global__ void scale_lines_kernel(int64_t rows, int64_t L, const double2* x,
                                   const double* __restrict__ cre, const double* __restrict__ cim,
                                   double2* y) {  // x may alias y
  const int64_t n = rows * L;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = i % L;
    const double ar = __ldg(cre + l), ai = __ldg(cim + l);
    const double2 b = x[i];
    y[i] = make_double2(__dsub_rn(__dmul_rn(ar, b.x), __dmul_rn(ai, b.y)),
                        __dadd_rn(__dmul_rn(ar, b.y), __dmul_rn(ai, b.x)));
  }
}

// fields: [u, v, w, om_x, dv_dx, dw_dx, du_dy, du_dz], each n points apart
__global__ void cross_kernel(int64_t n, const double* __restrict__ f, double* __restrict__ h) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double u = __ldg(f + i), v = __ldg(f + n + i), w = __ldg(f + 2 * n + i), om_x = __ldg(f + 3 * n + i);
    const double dv_dx = __ldg(f + 4 * n + i), dw_dx = __ldg(f + 5 * n + i);
    const double du_dy = __ldg(f + 6 * n + i), du_dz = __ldg(f + 7 * n + i);
    const double om_y = __dsub_rn(du_dz, dw_dx);
    const double om_z = __dsub_rn(dv_dx, du_dy);
    h[i] = __dsub_rn(__dmul_rn(v, om_z), __dmul_rn(w, om_y));
    h[n + i] = __dsub_rn(__dmul_rn(w, om_x), __dmul_rn(u, om_z));
    h[2 * n + i] = __dsub_rn(__dmul_rn(u, om_y), __dmul_rn(v, om_x));
  }
}

__device__ __forceinline__ void cross_point(const double (&f)[8], double& h0, double& h1, double& h2) {
  const double om_y = __dsub_rn(f[7], f[5]);
  const double om_z = __dsub_rn(f[4], f[6]);
  h0 = __dsub_rn(__dmul_rn(f[1], om_z), __dmul_rn(f[2], om_y));
  h1 = __dsub_rn(__dmul_rn(f[2], f[3]), __dmul_rn(f[0], om_z));
  h2 = __dsub_rn(__dmul_rn(f[0], om_y), __dmul_rn(f[1], f[3]));
}

// fields / h: [field][P + Q rows][M points]; rows 0..P-1 symmetric parts
// (point j, j < Q, pairs with N-1-j; row Q is the centre point when P > Q),
// rows P..P+Q-1 antisymmetric parts
__global__ void cross_paired_kernel(int64_t P, int64_t Q, int64_t M, const double* __restrict__ f,
                                    double* __restrict__ h) {
  const int64_t fs = (P + Q) * M, n = P * M;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const bool pair = i < Q * M;
    double top[8], bot[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double e = __ldg(f + q * fs + i);
      const double o = pair ? __ldg(f + q * fs + P * M + i) : 0.0;
      top[q] = __dadd_rn(e, o);
      bot[q] = __dsub_rn(e, o);
    }
    double t0, t1, t2;
    cross_point(top, t0, t1, t2);
    if (pair) {
      double b0, b1, b2;
      cross_point(bot, b0, b1, b2);
      h[i] = __dadd_rn(t0, b0);
      h[fs + i] = __dadd_rn(t1, b1);
      h[2 * fs + i] = __dadd_rn(t2, b2);
      h[P * M + i] = __dsub_rn(t0, b0);
      h[fs + P * M + i] = __dsub_rn(t1, b1);
      h[2 * fs + P * M + i] = __dsub_rn(t2, b2);
    } else {  // centre point: its own symmetric part
      h[i] = t0;
      h[fs + i] = t1;
      h[2 * fs + i] = t2;
    }
  }
}

__global__ void scale_rows_kernel(int64_t rows, int64_t L, const double2* x, int64_t xs, const double* __restrict__ cre,
                                  const double* __restrict__ cim, double2* y, int64_t ys) {
  const int64_t n = rows * L;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / L, l = i - r * L;
    const double ar = __ldg(cre + l), ai = __ldg(cim + l);
    const double2 b = x[r * xs + l];
    y[r * ys + l] = make_double2(__dsub_rn(__dmul_rn(ar, b.x), __dmul_rn(ai, b.y)),
                                 __dadd_rn(__dmul_rn(ar, b.y), __dmul_rn(ai, b.x)));
  }
}

// mirror pairing of wall-normal rows (real view, M doubles per row):
// split  y[j] = x[j] + x[N-1-j], y[Q] = x[Q] (centre), y[P+j] = x[j] - x[N-1-j]
// merge  x[j] = y[j] + y[P+j],  x[N-1-j] = y[j] - y[P+j],  x[Q] = y[Q]
// grid: x over the row's M/2 double2 columns, y = pair row j < P (no index division)
__global__ void pair_split_kernel(int64_t P, int64_t Q, int64_t M2, const double2* __restrict__ x,
                                  double2* __restrict__ y) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t j = blockIdx.y, N = P + Q;
  if (c >= M2) return;
  const double2 a = __ldg(x + j * M2 + c);
  if (j < Q) {
    const double2 b = __ldg(x + (N - 1 - j) * M2 + c);
    y[j * M2 + c] = make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
    y[(P + j) * M2 + c] = make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y));
  } else {
    y[j * M2 + c] = a;
  }
}
__global__ void pair_merge_kernel(int64_t P, int64_t Q, int64_t M2, const double2* __restrict__ y,
                                  double2* __restrict__ x) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t j = blockIdx.y, N = P + Q;
  if (c >= M2) return;
  const double2 e = __ldg(y + j * M2 + c);
  if (j < Q) {
    const double2 o = __ldg(y + (P + j) * M2 + c);
    x[j * M2 + c] = make_double2(__dadd_rn(e.x, o.x), __dadd_rn(e.y, o.y));
    x[(N - 1 - j) * M2 + c] = make_double2(__dsub_rn(e.x, o.x), __dsub_rn(e.y, o.y));
  } else {
    x[j * M2 + c] = e;
  }
}

unsigned grid_for(int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n + 255) / 256;
  return (unsigned)(want < (int64_t)sms * 16 ? want : (int64_t)sms * 16);
}

}  // namespace

cudaError_t launch_cross_paired(int64_t P, int64_t Q, int64_t M, const double* fields, double* h, cudaStream_t st) {
  if (P <= 0 || M <= 0) return cudaSuccess;
  cross_paired_kernel<<<grid_for(P * M), 256, 0, st>>>(P, Q, M, fields, h);
  return cudaGetLastError();
}

cudaError_t launch_pair(bool merge, int64_t P, int64_t Q, int64_t M, const double* src, double* dst,
                        cudaStream_t st) {
  if (P <= 0 || M <= 0) return cudaSuccess;
  if (M % 2 != 0 || P > 65535 || (reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) % 16 != 0)
    return cudaErrorInvalidValue;  // rows of complex values (double2-aligned)
  const int64_t M2 = M / 2;
  const dim3 grid((unsigned)((M2 + 255) / 256), (unsigned)P);
  if (merge)
    pair_merge_kernel<<<grid, 256, 0, st>>>(P, Q, M2, reinterpret_cast<const double2*>(src),
                                            reinterpret_cast<double2*>(dst));
  else
    pair_split_kernel<<<grid, 256, 0, st>>>(P, Q, M2, reinterpret_cast<const double2*>(src),
                                            reinterpret_cast<double2*>(dst));
  return cudaGetLastError();
}

cudaError_t launch_scale_rows(int64_t rows, int64_t L, const void* x, int64_t xs, const double* cre,
                              const double* cim, void* y, int64_t ys, cudaStream_t st) {
  if (rows <= 0 || L <= 0) return cudaSuccess;
  scale_rows_kernel<<<grid_for(rows * L), 256, 0, st>>>(rows, L, static_cast<const double2*>(x), xs, cre, cim,
                                                        static_cast<double2*>(y), ys);
  return cudaGetLastError();
}

cudaError_t launch_scale_lines(int64_t rows, int64_t L, const void* x, const double* cre, const double* cim, void* y,
                               cudaStream_t st) {
  if (rows <= 0 || L <= 0) return cudaSuccess;
  scale_lines_kernel<<<grid_for(rows * L), 256, 0, st>>>(rows, L, static_cast<const double2*>(x), cre, cim,
                                                         static_cast<double2*>(y));
  return cudaGetLastError();
}

cudaError_t launch_cross(int64_t n, const double* fields, double* h, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  cross_kernel<<<grid_for(n), 256, 0, st>>>(n, fields, h);
  return cudaGetLastError();
}

}  // namespace shen
