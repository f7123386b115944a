// Pointwise piece of the nonlinear term H = u x omega (reference
// stepper.py:148-185), SURVEY.md 8(f) rank 3.  The transforms around it are
// the fused wall-normal kernels (shen_wall.cu) and the plane FFT kernels
// (shen_plane_fft.cu), which also apply the per-line factors (1j m, 1j n, the
// dealiasing mask).
//
//   shen_cross:       om_y = du_dz - dw_dx, om_z = dv_dx - du_dy and
//                     h = (v om_z - w om_y, w om_x - u om_z, u om_y - v om_x)
//                     on the physical grid, in the reference's operation order
//                     (8 fields in, 3 out: one HBM pass).
#include <cuda_runtime.h>
#include <stdint.h>

#include "shen_kernels.h"

namespace shen {
namespace {

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

unsigned grid_for(int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n + 255) / 256;
  return (unsigned)(want < (int64_t)sms * 16 ? want : (int64_t)sms * 16);
}

}  // namespace

cudaError_t launch_cross(int64_t n, const double* fields, double* h, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  cross_kernel<<<grid_for(n), 256, 0, st>>>(n, fields, h);
  return cudaGetLastError();
}

}  // namespace shen
