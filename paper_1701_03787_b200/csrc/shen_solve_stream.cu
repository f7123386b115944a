// Streaming fused factor+solve: lanes = consecutive wavenumber systems.
//
// The RHS/solution layout is (n_modes, batch) with the batch contiguous, so
// a warp of 32 consecutive systems reads and writes whole 512-B row segments
// (and a CTA of W warps W*512 B) -- the access pattern HBM is fast at.  Each
// thread runs the reference's sequential sweeps for one (system, parity):
//
//   forward   rows 0..n-1: the compressed-LU row recurrence (fast-mode
//             arithmetic shared with the build kernel, restarting every R
//             rows exactly as the build does) and y_i = b_i - low_i y_{i-1};
//             y is staged in the output array (st.global with an L2
//             evict-last policy so it is still in L2 when read back);
//   backward  segments of R rows from the bottom: the segment's factors
//             are recomputed from the build's checkpoint into registers,
//             then the reference back-substitution overwrites y with x
//             (streaming store).
//
// There is no inter-thread coupling at all: results do not depend on the
// decomposition (no scans, no consistency correction).  The kernel is
// persistent with a bounded number of resident warps per SM so that the
// staged y of the systems in flight stays within L2.
#include <algorithm>

#include "shen_rows.cuh"
#include "shen_kernels.h"

namespace shen {

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_keep(double2* ptr, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(ptr), "d"(v.x), "d"(v.y), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_keep(double* ptr, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(ptr), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_keep(cplx* p, cplx v, uint64_t pol) {
  st_keep(reinterpret_cast<double2*>(p), make_double2(v.re, v.im), pol);
}

__device__ __forceinline__ cplx sfma(double s, cplx b, cplx a) { return {__fma_rn(s, b.re, a.re), __fma_rn(s, b.im, a.im)}; }
__device__ __forceinline__ double sfma(double s, double b, double a) { return __fma_rn(s, b, a); }
__device__ __forceinline__ cplx smul(double s, cplx b) { return {s * b.re, s * b.im}; }
__device__ __forceinline__ double smul(double s, double b) { return s * b; }
__device__ __forceinline__ cplx sadd(cplx a, cplx b) { return {a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ double sadd(double a, double b) { return a + b; }
__device__ __forceinline__ cplx ssub(cplx a, cplx b) { return {a.re - b.re, a.im - b.im}; }
__device__ __forceinline__ double ssub(double a, double b) { return a - b; }
template <typename V> __device__ __forceinline__ V szero();
template <> __device__ __forceinline__ double szero<double>() { return 0.0; }
template <> __device__ __forceinline__ cplx szero<cplx>() { return {0.0, 0.0}; }

// ======================================================================= Helmholtz
// smem: row table [n][4] (sd, st, md, has_sup) of this CTA's parity.
template <typename V, int R>
__global__ void __launch_bounds__(128) helm_stream_kernel(HelmChunkArgs a) {
  using O = VOps<V>;
  extern __shared__ __align__(16) double smem[];
  const int par = blockIdx.y;
  const int64_t B = a.batch;
  const int n = (a.n_dir - par + 1) / 2;
  const int nsup = (a.n_dir - 2 - par + 1) / 2 > 0 ? (a.n_dir - 2 - par + 1) / 2 : 0;
  const int nseg = (n + R - 1) / R;
  double4* tab = reinterpret_cast<double4*>(smem);
  for (int i = threadIdx.x; i < nseg * R; i += blockDim.x) {
    double4 v = make_double4(0.0, 0.0, 0.0, 0.0);
    if (i < n) {
      const int k = par + 2 * i;
      v = make_double4(__ldg(a.sd + k), __ldg(a.st + k), __ldg(a.md + k), i < nsup ? 1.0 : 0.0);
    }
    tab[i] = v;
  }
  __syncthreads();
  const V* rhs = static_cast<const V*>(a.rhs);
  V* out = static_cast<V*>(a.out);
  const uint64_t keep = policy_evict_last();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < B; j += stride) {
    const double cb = __ldg(a.cb + j);
    const double sub = __dmul_rn(cb, -1.5707963267948966);
    // ---------------- forward
    HelmProj pj;
    hp_origin(pj);
    V y = szero<V>();
    double dl = 0.0, el = 0.0, tl = 0.0;
    for (int s = 0; s < nseg; ++s) {
      if (s > 0) hp_start(pj, dl, el, tl);
      V b[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = s * R + r;
        b[r] = i < n ? O::ld_cs(rhs + (int64_t)(par + 2 * i) * B + j) : szero<V>();
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = s * R + r;
        const double4 tv = tab[i];
        const HelmRow row = helm_row(a.ca, cb, sub, tv.x, tv.y, tv.z, tv.w != 0.0);
        if (r > 0 && (r & 7) == 0) hp_rescale(pj);
        double d, e, t;
        const double low = hp_step(pj, row, sub, d, e, t);
        dl = d; el = e; tl = t;
        y = sfma(-low, y, b[r]);
        if (i < n) st_keep(out + (int64_t)(par + 2 * i) * B + j, y, keep);
      }
    }
    // ---------------- backward
    V x1 = szero<V>(), S = szero<V>();
    for (int s = nseg - 1; s >= 0; --s) {
      HelmProj q;
      if (s == 0) {
        hp_origin(q);
      } else {
        const double* ck = a.ckpt + ((int64_t)(s * 2 + par) * 3) * B + j;
        hp_start(q, __ldg(ck), __ldg(ck + B), __ldg(ck + 2 * B));
      }
      double rd_[R], e_[R], t_[R];
      V yv[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = s * R + r;
        yv[r] = i < n ? out[(int64_t)(par + 2 * i) * B + j] : szero<V>();
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = s * R + r;
        const double4 tv = tab[i];
        const HelmRow row = helm_row(a.ca, cb, sub, tv.x, tv.y, tv.z, tv.w != 0.0);
        if (r > 0 && (r & 7) == 0) hp_rescale(q);
        double d, e, t;
        hp_step(q, row, sub, d, e, t);
        const bool valid = i < n;
        rd_[r] = valid ? q.rd : 0.0;
        e_[r] = valid ? e : 0.0;
        t_[r] = valid ? t : 0.0;
      }
#pragma unroll
      for (int r = R - 1; r >= 0; --r) {
        const int i = s * R + r;
        const V acc = ssub(ssub(yv[r], smul(e_[r], x1)), smul(t_[r], S));
        const V x = smul(rd_[r], acc);
        S = sadd(x1, S);
        x1 = x;
        if (i < n) O::st_cs(out + (int64_t)(par + 2 * i) * B + j, x);
      }
    }
  }
}

// ======================================================================= biharmonic
template <typename V, int R>
__global__ void __launch_bounds__(128) bih_stream_kernel(BihChunkArgs a) {
  using O = VOps<V>;
  const int par = blockIdx.y;
  const int64_t B = a.batch;
  const int nb = a.n_bih;
  const int n = (nb - par + 1) / 2;
  const int nseg = (n + R - 1) / R;
  const V* rhs = static_cast<const V*>(a.rhs);
  V* out = static_cast<V*>(a.out);
  const double xi0 = a.xi0;
  const uint64_t keep = policy_evict_last();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < B; j += stride) {
    const double xi1 = __ldg(a.xi1 + j), xi2 = __ldg(a.xi2 + j);
    // ---------------- forward
    BihU u{0, 0, 0, 0, 0, 0}, u1{0, 0, 0, 0, 0, 0}, u2{0, 0, 0, 0, 0, 0};
    V y1 = szero<V>(), y2 = szero<V>();
    for (int s = 0; s < nseg; ++s) {
      V b[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = s * R + r;
        b[r] = i < n ? O::ld_cs(rhs + (int64_t)(par + 2 * i) * B + j) : szero<V>();
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = s * R + r;
        const int k = min(par + 2 * i, nb - 1);
        double c[B_NCOL];
#pragma unroll
        for (int q = 0; q < B_NCOL; ++q) c[q] = __ldg(a.tab + (int64_t)k * B_NCOL + q);
        const BihBands hb = bih_bands(xi0, xi1, xi2, c);
        double l2, l4;
        bih_step_fast(u, u1, u2, hb, c, xi0, l2, l4);
        u2 = u1;
        u1 = u;
        const V y = sfma(-l4, y2, sfma(-l2, y1, b[r]));
        y2 = y1;
        y1 = y;
        if (i < n) st_keep(out + (int64_t)(par + 2 * i) * B + j, y, keep);
      }
    }
    // ---------------- backward
    V x1 = szero<V>(), x2 = szero<V>(), sq = szero<V>(), sv = szero<V>();
    for (int s = nseg - 1; s >= 0; --s) {
      BihU w{0, 0, 0, 0, 0, 0}, w1{0, 0, 0, 0, 0, 0}, w2{0, 0, 0, 0, 0, 0};
      if (s > 0) {
        const double* ck = a.ckpt + ((int64_t)(s * 2 + par) * 10) * B + j;
        w1.d = __ldg(ck); w1.e = __ldg(ck + B); w1.f = __ldg(ck + 2 * B); w1.a = __ldg(ck + 3 * B);
        w1.b = __ldg(ck + 4 * B);
        w2.d = __ldg(ck + 5 * B); w2.e = __ldg(ck + 6 * B); w2.f = __ldg(ck + 7 * B); w2.a = __ldg(ck + 8 * B);
        w2.b = __ldg(ck + 9 * B);
        w1.rd = rcp_fast(w1.d);
        w2.rd = s * R >= 2 ? rcp_fast(w2.d) : 0.0;
      }
      double rd_[R], e_[R], f_[R], a_[R], b_[R], qn_[R], sn_[R];
      V yv[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = s * R + r;
        yv[r] = i < n ? out[(int64_t)(par + 2 * i) * B + j] : szero<V>();
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = s * R + r;
        const int k = min(par + 2 * i, nb - 1);
        double c[B_NCOL];
#pragma unroll
        for (int q = 0; q < B_NCOL; ++q) c[q] = __ldg(a.tab + (int64_t)k * B_NCOL + q);
        const BihBands hb = bih_bands(xi0, xi1, xi2, c);
        double l2, l4;
        bih_step_fast(w, w1, w2, hb, c, xi0, l2, l4);
        w2 = w1;
        w1 = w;
        const bool valid = i < n;
        rd_[r] = valid ? w.rd : 0.0;
        e_[r] = valid ? w.e : 0.0;
        f_[r] = valid ? w.f : 0.0;
        a_[r] = valid ? w.a : 0.0;
        b_[r] = valid ? w.b : 0.0;
        qn_[r] = valid ? c[B_Q4] : 0.0;
        sn_[r] = valid ? c[B_S4] : 0.0;
      }
#pragma unroll
      for (int r = R - 1; r >= 0; --r) {
        const int i = s * R + r;
        V acc = ssub(ssub(yv[r], smul(e_[r], x1)), smul(f_[r], x2));
        acc = ssub(acc, smul(xi0, sadd(smul(a_[r], sq), smul(b_[r], sv))));
        const V x = smul(rd_[r], acc);
        sq = sfma(qn_[r], x2, sq);
        sv = sfma(sn_[r], x2, sv);
        x2 = x1;
        x1 = x;
        if (i < n) O::st_cs(out + (int64_t)(par + 2 * i) * B + j, x);
      }
    }
  }
}

// ======================================================================= launchers
static int stream_blocks_per_parity(int warps_per_sm, int threads) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int total_warps = sms * warps_per_sm;
  return std::max(1, total_warps / (threads / 32) / 2);
}

template <typename V, int R>
static cudaError_t helm_stream_R(const HelmChunkArgs& a, int warps_per_sm, cudaStream_t st) {
  const int threads = 64;
  const int n0 = (a.n_dir + 1) / 2;
  const size_t smem = (size_t)((n0 + R - 1) / R) * R * sizeof(double4);
  cudaError_t err = cudaFuncSetAttribute(helm_stream_kernel<V, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  const int64_t want = (a.batch + threads - 1) / threads;
  dim3 grid((unsigned)std::min<int64_t>(want, stream_blocks_per_parity(warps_per_sm, threads)), 2);
  helm_stream_kernel<V, R><<<grid, threads, smem, st>>>(a);
  return cudaGetLastError();
}

template <typename V, int R>
static cudaError_t bih_stream_R(const BihChunkArgs& a, int warps_per_sm, cudaStream_t st) {
  const int threads = 64;
  const int64_t want = (a.batch + threads - 1) / threads;
  dim3 grid((unsigned)std::min<int64_t>(want, stream_blocks_per_parity(warps_per_sm, threads)), 2);
  bih_stream_kernel<V, R><<<grid, threads, 0, st>>>(a);
  return cudaGetLastError();
}

template <typename V>
static cudaError_t helm_stream_dispatch(const HelmChunkArgs& a, int w, cudaStream_t st) {
  switch (a.chunk_rows) {
    case 4: return helm_stream_R<V, 4>(a, w, st);
    case 8: return helm_stream_R<V, 8>(a, w, st);
    case 16: return helm_stream_R<V, 16>(a, w, st);
    default: return cudaErrorInvalidValue;
  }
}

template <typename V>
static cudaError_t bih_stream_dispatch(const BihChunkArgs& a, int w, cudaStream_t st) {
  switch (a.chunk_rows) {
    case 4: return bih_stream_R<V, 4>(a, w, st);
    case 8: return bih_stream_R<V, 8>(a, w, st);
    case 16: return bih_stream_R<V, 16>(a, w, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_helm_stream(const HelmChunkArgs& a, bool cplx_rhs, int warps_per_sm, cudaStream_t st) {
  if (a.batch <= 0) return cudaSuccess;
  return cplx_rhs ? helm_stream_dispatch<cplx>(a, warps_per_sm, st) : helm_stream_dispatch<double>(a, warps_per_sm, st);
}

cudaError_t launch_bih_stream(const BihChunkArgs& a, bool cplx_rhs, int warps_per_sm, cudaStream_t st) {
  if (a.batch <= 0) return cudaSuccess;
  return cplx_rhs ? bih_stream_dispatch<cplx>(a, warps_per_sm, st) : bih_stream_dispatch<double>(a, warps_per_sm, st);
}

}  // namespace shen
