// Wall-normal (axis 0) pieces of the Shen transforms, reference
// transforms.py:81-205.  Layout: arrays (rows, L) with the L = n_y*(n_z/2+1)
// Fourier lines contiguous, complex128; one thread per line walks the rows,
// so every row access of a warp is a coalesced 512-B piece.
//
// The DCTs along axis 0 go through an FFT of an extended sequence (cuFFT,
// called from the host layer) with these kernels doing everything around it:
//   Gauss  (DCT-II / DCT-III, N = n_x+1 points):
//     forward : symmetric extension e = [x_0..x_{N-1}, x_{N-1}..x_0] (2N rows),
//               Y = FFT_2N(e), DCT-II_k = w_k Y_k with w_k = exp(-i pi k / 2N);
//     inverse : Z_k = c_k conj(w_k) (k < N), Z_{2N-k} = c_k w_k, Z_N = 0,
//               sum_k c_k cos(pi k (2n+1)/2N) = (IFFT_2N^unnormalised(Z)_n + c_0) / 2.
//   Gauss-Lobatto (DCT-I, N = n_x+1 points):
//     even extension [x_0..x_{N-1}, x_{N-2}..x_1] (2 n_x rows), DCT-I = FFT.
// Post-processing fuses the Chebyshev scaling and the Shen stencil
// (transforms.py:81-110) and the inverse pre-processing fuses shen_expand
// (transforms.py:113-126).  mass_solve is the per-parity banded Cholesky
// solve (transforms.py:163-175) with the host's LAPACK factors.
#include <cuda_runtime.h>
#include <stdint.h>

#include "shen_common.cuh"

namespace shen {

struct c2 {
  double x, y;
};
__device__ __forceinline__ c2 ld2(const double2* p) {
  const double2 v = __ldg(p);
  return {v.x, v.y};
}
__device__ __forceinline__ void st2(double2* p, c2 v) { *p = make_double2(v.x, v.y); }
__device__ __forceinline__ c2 cmul(c2 a, c2 b) { return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x}; }
__device__ __forceinline__ c2 cadd(c2 a, c2 b) { return {a.x + b.x, a.y + b.y}; }
__device__ __forceinline__ c2 csub(c2 a, c2 b) { return {a.x - b.x, a.y - b.y}; }
__device__ __forceinline__ c2 cscale(double s, c2 a) { return {s * a.x, s * a.y}; }

// Every kernel is one thread per Fourier line (x) and a chunk of kRowChunk
// rows (y), so that small line counts still fill the machine.
constexpr int kRowChunk = 16;

// ---------------------------------------------------------------- extensions
// kind 0: Gauss forward symmetric extension (N -> 2N rows)
// kind 1: Gauss-Lobatto even extension (N -> 2N-2 rows)
__global__ void xf_extend_kernel(int kind, int N, int64_t L, const double2* __restrict__ x, double2* __restrict__ e) {
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= L) return;
  const int M = kind == 0 ? 2 * N : 2 * N - 2;
  const int m0 = blockIdx.y * kRowChunk, m1 = min(M, m0 + kRowChunk);
  for (int m = m0; m < m1; ++m) {
    int src;
    if (m < N) src = m;
    else src = kind == 0 ? 2 * N - 1 - m : 2 * N - 2 - m;
    e[(int64_t)m * L + l] = __ldg(x + (int64_t)src * L + l);
  }
}

// ---------------------------------------------------------------- forward post
// Y: FFT of the extension (rows 0..N-1 used).  w_k = scale * (Gauss: tw_k Y_k,
// GL: Y_k); then space 0: Chebyshev coefficients (2/pi, halved ends), 1:
// Dirichlet w_k - w_{k+2}, 2: biharmonic w_k - c2_k w_{k+2} + c4_k w_{k+4},
// 3: the raw scalar products w (chebyshev_scalar).
// tw: [N] complex twiddles exp(-i pi k/2N) (host precomputed).
__global__ void xf_fwd_post_kernel(int gl, int space, int N, int64_t L, double scale, const double2* __restrict__ tw,
                                   const double2* __restrict__ Y, double2* __restrict__ out) {
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= L) return;
  const int n_x = N - 1;
  auto w_at = [&](int k) -> c2 {
    c2 y = ld2(Y + (int64_t)k * L + l);
    if (!gl) y = cmul(ld2(tw + k), y);
    return cscale(scale, y);
  };
  const int k0 = blockIdx.y * kRowChunk;
  if (space == 0 || space == 3) {
    for (int k = k0; k < min(N, k0 + kRowChunk); ++k) {
      c2 v = w_at(k);
      if (space == 3) {
        st2(out + (int64_t)k * L + l, v);
        continue;
      }
      v = cscale(2.0 / 3.141592653589793, v);
      if (k == 0 || (gl && k == n_x)) v = cscale(0.5, v);
      st2(out + (int64_t)k * L + l, v);
    }
    return;
  }
  if (space == 1) {
    if (k0 >= n_x - 1) return;
    c2 wk = w_at(k0), wk1 = w_at(k0 + 1);
    for (int k = k0; k < min(n_x - 1, k0 + kRowChunk); ++k) {
      const c2 wk2 = w_at(k + 2);
      st2(out + (int64_t)k * L + l, csub(wk, wk2));
      wk = wk1;
      wk1 = wk2;
    }
    return;
  }
  if (k0 >= n_x - 3) return;
  c2 w0 = w_at(k0), w1 = w_at(k0 + 1), w2 = w_at(k0 + 2), w3 = w_at(k0 + 3);
  for (int k = k0; k < min(n_x - 3, k0 + kRowChunk); ++k) {
    const c2 w4 = w_at(k + 4);
    const double kk = (double)k;
    const double c2k = 2 * (kk + 2) / (kk + 3), c4k = (kk + 1) / (kk + 3);
    st2(out + (int64_t)k * L + l, cadd(csub(w0, cscale(c2k, w2)), cscale(c4k, w4)));
    w0 = w1; w1 = w2; w2 = w3; w3 = w4;
  }
}

// ---------------------------------------------------------------- inverse pre
// coefficients of `space` (n rows) -> Chebyshev coefficients c (N = n_x+1)
// (shen_expand) -> FFT input: Gauss Z (2N rows, twiddled), GL even extension
// (2N-2 rows), or (gl == 2) the expanded coefficients themselves (N rows).
// Also writes c_0 and c_{n_x} per line into cends[2][L] (may be NULL).
__global__ void xf_inv_pre_kernel(int gl, int space, int n, int N, int64_t L, const double2* __restrict__ tw,
                                  const double2* __restrict__ coef, double2* __restrict__ Z, double2* __restrict__ cends) {
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= L) return;
  auto a_at = [&](int k) -> c2 {
    if (k < 0 || k >= n) return {0.0, 0.0};
    return ld2(coef + (int64_t)k * L + l);
  };
  const int M = gl ? 2 * N - 2 : 2 * N;
  const int k0 = blockIdx.y * kRowChunk;
  for (int k = k0; k < min(N, k0 + kRowChunk); ++k) {
    c2 c = a_at(k);
    if (space == 1) {
      c = csub(c, a_at(k - 2));
    } else if (space == 2) {
      const double j2 = (double)(k - 2), j4 = (double)(k - 4);
      if (k >= 2 && k - 2 < n) c = csub(c, cscale(2 * (j2 + 2) / (j2 + 3), a_at(k - 2)));
      if (k >= 4 && k - 4 < n) c = cadd(c, cscale((j4 + 1) / (j4 + 3), a_at(k - 4)));
    }
    if (cends && k == 0) st2(cends + l, c);
    if (cends && k == N - 1) st2(cends + L + l, c);
    if (gl == 2) {  // plain shen_expand output (N rows)
      st2(Z + (int64_t)k * L + l, c);
    } else if (gl) {
      st2(Z + (int64_t)k * L + l, c);
      if (k > 0 && k < N - 1) st2(Z + (int64_t)(M - k) * L + l, c);
    } else {
      const c2 w = ld2(tw + k);
      st2(Z + (int64_t)k * L + l, cmul({w.x, -w.y}, c));
      if (k > 0) st2(Z + (int64_t)(M - k) * L + l, cmul(w, c));
    }
  }
  if (!gl && blockIdx.y == 0) st2(Z + (int64_t)N * L + l, {0.0, 0.0});
}

// ---------------------------------------------------------------- inverse post
// F: unnormalised inverse FFT (Gauss) / FFT (GL) of Z; lines out (N rows):
//   Gauss: (F_n + c_0)/2 ; GL: F_n/2 + c_0/2 + (-1)^n c_{n_x}/2
// (transforms.py:129-137)
__global__ void xf_inv_post_kernel(int gl, int N, int64_t L, const double2* __restrict__ F,
                                   const double2* __restrict__ cends, double2* __restrict__ out) {
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= L) return;
  const c2 c0 = ld2(cends + l), cN = ld2(cends + L + l);
  const int m0 = blockIdx.y * kRowChunk;
  for (int m = m0; m < min(N, m0 + kRowChunk); ++m) {
    c2 f = ld2(F + (int64_t)m * L + l);
    c2 v;
    if (!gl) {
      v = cscale(0.5, cadd(f, c0));
    } else {
      v = cadd(cscale(0.5, f), cscale(0.5, c0));
      v = (m & 1) ? csub(v, cscale(0.5, cN)) : cadd(v, cscale(0.5, cN));
    }
    st2(out + (int64_t)m * L + l, v);
  }
}

// ---------------------------------------------------------------- mass solve
// Per parity p, the banded SPD system U^T U x = s (upper Cholesky factor U of
// bandwidth nb = 1 or 2, LAPACK band storage rows (nb+1) x m per parity):
// forward U^T y = s, backward U x = y (zpbtrs).  fac layout: [2][nb+1][mmax].
// Per CTA: the rows' reciprocal pivots and off-diagonal factor entries of
// both parities are staged in shared memory once ([2][mmax + 1] each of
// 1/U_ii, U_{i-1,i}, U_{i-2,i}); one thread per (line, parity), a warp =
// 32 consecutive lines of one parity (coalesced 512-B row pieces); each sweep
// keeps the next kQ rows' loads in flight in a register queue (the loads are
// independent of the recurrence), so the sweep is bound by its FMA chain and
// HBM rather than by load latency.  Arithmetic: y = (s - u1 y1 - u2 y2) / U_ii
// and x = (y - U_{i,i+1} x1 - U_{i,i+2} x2) / U_ii with the division as a
// product by the reciprocal, as before.
constexpr int kMassQ = 4;

// (s and x may be the same array: the in-place solve of transforms._mass_pass)
__global__ void __launch_bounds__(256) xf_mass_kernel(int nband, int n, int mmax, int64_t L,
                                                      const double* __restrict__ fac, const double2* s, double2* x) {
  extern __shared__ double msm[];
  double* rdg = msm;                       // [2][mmax + 1] 1 / U_ii
  double* u1 = msm + 2 * (mmax + 1);       // [2][mmax + 1] U_{i-1,i} (0 for i = 0)
  double* u2 = msm + 4 * (mmax + 1);       // [2][mmax + 1] U_{i-2,i} (0 for i < 2 or nband = 1)
  for (int e = threadIdx.x; e < 2 * (mmax + 1); e += blockDim.x) {
    const int p = e / (mmax + 1), i = e - p * (mmax + 1);
    const int m = (n - p + 1) / 2;
    const double* ab = fac + (int64_t)p * (nband + 1) * mmax;
    double r = 0.0, a = 0.0, b = 0.0;
    if (i < m) {
      r = 1.0 / __ldg(ab + (int64_t)nband * mmax + i);
      if (i >= 1) a = __ldg(ab + (int64_t)(nband - 1) * mmax + i);
      if (nband == 2 && i >= 2) b = __ldg(ab + i);
    }
    rdg[e] = r;
    u1[e] = a;
    u2[e] = b;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nw = ((L + 31) / 32) * 2;  // warps of work: (32-line group, parity)
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (w >= nw) return;
  const int par = (int)(w & 1);
  const int64_t l = (w >> 1) * 32 + lane;
  if (l >= L) return;
  const int m = (n - par + 1) / 2;
  const double* R = rdg + par * (mmax + 1);
  const double* A = u1 + par * (mmax + 1);
  const double* Bq = u2 + par * (mmax + 1);
  const int64_t rs = 2 * L;
  const double2* sp = s + (int64_t)par * L + l;
  double2* xp = x + (int64_t)par * L + l;
  // forward U^T y = s
  c2 q[kMassQ];
#pragma unroll
  for (int k = 0; k < kMassQ; ++k) q[k] = k < m ? ld2(sp + k * rs) : c2{0.0, 0.0};
  c2 y1 = {0, 0}, y2 = {0, 0};
  for (int i0 = 0; i0 < m; i0 += kMassQ) {
#pragma unroll
    for (int k = 0; k < kMassQ; ++k) {
      const int i = i0 + k;
      if (i < m) {
        c2 acc = q[k];
        const int inext = i + kMassQ;
        q[k] = inext < m ? ld2(sp + inext * rs) : c2{0.0, 0.0};
        acc = csub(acc, cscale(A[i], y1));
        if (nband == 2) acc = csub(acc, cscale(Bq[i], y2));
        const c2 y = cscale(R[i], acc);
        st2(xp + i * rs, y);
        y2 = y1;
        y1 = y;
      }
    }
  }
  // backward U x = y (y read back from x, the queue refilled bottom-up)
#pragma unroll
  for (int k = 0; k < kMassQ; ++k) {
    const int i = m - 1 - k;
    q[k] = i >= 0 ? c2{xp[i * rs].x, xp[i * rs].y} : c2{0.0, 0.0};
  }
  c2 x1 = {0, 0}, x2 = {0, 0};
  for (int i0 = m - 1; i0 >= 0; i0 -= kMassQ) {
#pragma unroll
    for (int k = 0; k < kMassQ; ++k) {
      const int i = i0 - k;
      if (i >= 0) {
        c2 acc = q[k];
        const int inext = i - kMassQ;
        q[k] = inext >= 0 ? c2{xp[inext * rs].x, xp[inext * rs].y} : c2{0.0, 0.0};
        if (i + 1 < m) acc = csub(acc, cscale(A[i + 1], x1));
        if (nband == 2 && i + 2 < m) acc = csub(acc, cscale(Bq[i + 2], x2));
        const c2 v = cscale(R[i], acc);
        st2(xp + i * rs, v);
        x2 = x1;
        x1 = v;
      }
    }
  }
}

static unsigned blocks_for(int64_t n) { return (unsigned)((n + 255) / 256); }
static dim3 grid_for(int64_t L, int rows) { return dim3(blocks_for(L), (unsigned)((rows + kRowChunk - 1) / kRowChunk)); }

cudaError_t launch_xf_extend(int kind, int N, int64_t L, const void* x, void* e, cudaStream_t st) {
  if (L <= 0) return cudaSuccess;
  xf_extend_kernel<<<grid_for(L, kind == 0 ? 2 * N : 2 * N - 2), 256, 0, st>>>(kind, N, L, static_cast<const double2*>(x), static_cast<double2*>(e));
  return cudaGetLastError();
}
cudaError_t launch_xf_fwd_post(int gl, int space, int N, int64_t L, double scale, const void* tw, const void* Y,
                               void* out, cudaStream_t st) {
  if (L <= 0) return cudaSuccess;
  xf_fwd_post_kernel<<<grid_for(L, N), 256, 0, st>>>(gl, space, N, L, scale, static_cast<const double2*>(tw),
                                                    static_cast<const double2*>(Y), static_cast<double2*>(out));
  return cudaGetLastError();
}
cudaError_t launch_xf_inv_pre(int gl, int space, int n, int N, int64_t L, const void* tw, const void* coef, void* Z,
                              void* cends, cudaStream_t st) {
  if (L <= 0) return cudaSuccess;
  xf_inv_pre_kernel<<<grid_for(L, N), 256, 0, st>>>(gl, space, n, N, L, static_cast<const double2*>(tw),
                                                   static_cast<const double2*>(coef), static_cast<double2*>(Z),
                                                   static_cast<double2*>(cends));
  return cudaGetLastError();
}
cudaError_t launch_xf_inv_post(int gl, int N, int64_t L, const void* F, const void* cends, void* out, cudaStream_t st) {
  if (L <= 0) return cudaSuccess;
  xf_inv_post_kernel<<<grid_for(L, N), 256, 0, st>>>(gl, N, L, static_cast<const double2*>(F),
                                                    static_cast<const double2*>(cends), static_cast<double2*>(out));
  return cudaGetLastError();
}
cudaError_t launch_xf_mass(int nband, int n, int mmax, int64_t L, const double* fac, const void* s, void* x,
                           cudaStream_t st) {
  if (L <= 0) return cudaSuccess;
  const int64_t warps = ((L + 31) / 32) * 2;
  const size_t smem = (size_t)6 * (mmax + 1) * sizeof(double);
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(xf_mass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  xf_mass_kernel<<<(unsigned)((warps + 7) / 8), 256, smem, st>>>(nband, n, mmax, L, fac, static_cast<const double2*>(s),
                                                                 static_cast<double2*>(x));
  return cudaGetLastError();
}

}  // namespace shen
