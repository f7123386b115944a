// Streaming fused factor+solve: lanes = consecutive wavenumber systems.
//
// The RHS/solution layout is (n_modes, batch) with the batch contiguous, so
// a warp of 32 consecutive systems reads and writes whole 512-B row
// segments -- the access pattern HBM is fast at.  Each thread runs the
// reference's sequential sweeps for one (system, parity); there is no
// inter-thread coupling (no scans, no consistency correction):
//
//   forward   rows 0..n-1: the compressed-LU row recurrence (fast-mode
//             arithmetic shared with the build kernel, restarting every R
//             rows exactly as the build does) and y_i = b_i - low_i y_{i-1};
//   backward  segments of R rows from the bottom: the segment's factors are
//             recomputed from the build's checkpoint into registers, then the
//             reference back-substitution turns y into x.
//
// Where y lives between the sweeps decides the HBM traffic.  A CTA is two
// warps (parity 0 and parity 1 of the same 32 systems) and there is ONE
// persistent CTA per SM, so only 64 systems-parities per SM are in flight:
// the last `tail` rows of every y stay in shared memory (they are the first
// ones the backward sweep needs) and the rest is staged in the output array
// with an L2 evict-last policy -- at BASELINE config 4 that is ~58 MB over the
// whole chip, inside the 126 MB L2, so the y round trip costs L2 bandwidth,
// not HBM.  Latency is hidden by cp.async prefetch of the next segment (RHS
// rows in the forward, staged y in the backward) instead of by occupancy.
#include <algorithm>

#include "shen_rows.cuh"
#include "shen_kernels.h"

namespace shen {

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_keep(double* ptr, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(ptr), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_keep(cplx* p, cplx v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.re), "d"(v.im), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cpa(cplx* dst, const cplx* src, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  const int n = pred ? 16 : 0;  // src-size 0 -> zero fill, no global access
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cpa(double* dst, const double* src, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  const int n = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

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

constexpr int kStreamThreads = 64;  // 2 warps: parity 0, parity 1

// Shared-memory plan common to both operators (per CTA):
//   stage [kRing][R][64] V : cp.async ring (forward RHS / backward y)
//   tail  [T][64]    V : the last T = tail_segs*R rows of y of every thread
//   (Helmholtz only) table [2][nseg*R] double4
struct StreamPlan {
  int nseg[2];      // segments per parity
  int tail_segs;    // segments of y kept in shared memory
};

// segment s of parity `par` -> where its y lives: >= 0 -> tail segment index
__device__ __forceinline__ int tail_slot(int s, int nseg, int tail_segs) {
  const int first = nseg - tail_segs;
  return s >= first ? s - first : -1;
}

constexpr int kRing = 4;  // stage buffers; prefetch distance kRing - 1 segments

// cp.async the rows of segment s (parity rows s*R ...) of `src` into stage buffer b
template <typename V, int R>
__device__ __forceinline__ void stage_segment(V* stage, int b, const V* src, int s, int n, int par, int64_t B,
                                              int64_t jc, bool jv, int tid) {
  V* dst = stage + (size_t)b * R * kStreamThreads;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = s * R + r;
    cpa(dst + r * kStreamThreads + tid, src + (int64_t)(par + 2 * min(i, n - 1)) * B + jc, jv && i < n);
  }
}

// ======================================================================= Helmholtz
template <typename V, int R>
__global__ void __launch_bounds__(kStreamThreads, 1) helm_stream_kernel(HelmChunkArgs a, int tail_segs, int tab_rows) {
  using O = VOps<V>;
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x, lane = tid & 31, par = tid >> 5;
  const int64_t B = a.batch;
  const int n = (a.n_dir - par + 1) / 2;
  const int nseg = (n + R - 1) / R;
  const int tseg = min(tail_segs, nseg);
  V* stage = reinterpret_cast<V*>(smem);                        // [2][R][64]
  V* tail = stage + kRing * R * kStreamThreads;                 // [tail_segs*R][64]
  double4* tab = reinterpret_cast<double4*>(tail + (size_t)tail_segs * R * kStreamThreads);  // [2][tab_rows]
  for (int idx = tid; idx < 2 * tab_rows; idx += kStreamThreads) {
    const int p = idx / tab_rows, i = idx - p * tab_rows;
    const int np = (a.n_dir - p + 1) / 2;
    const int nsp = (a.n_dir - 2 - p + 1) / 2 > 0 ? (a.n_dir - 2 - p + 1) / 2 : 0;
    double4 v = make_double4(0.0, 0.0, 0.0, 0.0);
    if (i < np) {
      const int k = p + 2 * i;
      v = make_double4(__ldg(a.sd + k), __ldg(a.st + k), __ldg(a.md + k), i < nsp ? 1.0 : 0.0);
    }
    tab[idx] = v;
  }
  __syncthreads();
  const double4* mytab = tab + par * tab_rows;
  const V* rhs = static_cast<const V*>(a.rhs);
  V* out = static_cast<V*>(a.out);
  const uint64_t keep = policy_evict_last();
  const int64_t ngroups = (B + 31) / 32;
  auto rowp = [&](auto* base, int i, int64_t j) { return base + (int64_t)(par + 2 * i) * B + j; };

  for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
    const int64_t j = g * 32 + lane;
    const bool jv = j < B;
    const int64_t jc = jv ? j : B - 1;  // clamped (loads stay in bounds; results discarded)
    const double cb = __ldg(a.cb + jc);
    const double sub = __dmul_rn(cb, -1.5707963267948966);
    // ---------------- forward
#pragma unroll
    for (int u = 0; u < kRing - 1; ++u) {
      if (u < nseg) stage_segment<V, R>(stage, u, rhs, u, n, par, B, jc, jv, tid);
      cpa_commit();
    }
    HelmProj pj;
    hp_origin(pj);
    V y = szero<V>();
    double dl = 0.0, el = 0.0, tl = 0.0;
    for (int s = 0; s < nseg; ++s) {
      if (s + kRing - 1 < nseg) stage_segment<V, R>(stage, (s + kRing - 1) % kRing, rhs, s + kRing - 1, n, par, B, jc, jv, tid);
      cpa_commit();
      cpa_wait<kRing - 1>();
      const V* cur = stage + (size_t)(s % kRing) * R * kStreamThreads;
      if (s > 0) hp_start(pj, dl, el, tl);
      const int ts = tail_slot(s, nseg, tseg);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = s * R + r;
        const double4 tv = mytab[i];
        const HelmRow row = helm_row(a.ca, cb, sub, tv.x, tv.y, tv.z, tv.w != 0.0);
        if (r > 0 && (r & 7) == 0) hp_rescale(pj);
        double d, e, t;
        const double low = hp_step(pj, row, sub, d, e, t);
        dl = d; el = e; tl = t;
        y = sfma(-low, y, cur[r * kStreamThreads + tid]);
        if (ts >= 0)
          tail[(ts * R + r) * kStreamThreads + tid] = y;
        else if (jv && i < n)
          st_keep(rowp(out, i, j), y, keep);
      }
    }
    // ---------------- backward
    cpa_wait<0>();
    // staged (global) segments are consumed in the order first_tail-1, ..., 0
    const int first_tail = nseg - tseg;
#pragma unroll
    for (int u = 0; u < kRing - 1; ++u) {
      if (first_tail - 1 - u >= 0) stage_segment<V, R>(stage, u, out, first_tail - 1 - u, n, par, B, jc, jv, tid);
      cpa_commit();
    }
    V x1 = szero<V>(), S = szero<V>();
    for (int s = nseg - 1; s >= 0; --s) {
      const int ts = tail_slot(s, nseg, tseg);
      HelmProj q;
      if (s == 0) {
        hp_origin(q);
      } else {
        const double* ck = a.ckpt + ((int64_t)(s * 2 + par) * 3) * B + jc;
        hp_start(q, __ldg(ck), __ldg(ck + B), __ldg(ck + 2 * B));
      }
      double rd_[R], e_[R], t_[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = s * R + r;
        const double4 tv = mytab[i];
        const HelmRow row = helm_row(a.ca, cb, sub, tv.x, tv.y, tv.z, tv.w != 0.0);
        if (r > 0 && (r & 7) == 0) hp_rescale(q);
        double d, e, t;
        hp_step(q, row, sub, d, e, t);
        const bool valid = i < n;
        rd_[r] = valid ? q.rd : 0.0;
        e_[r] = valid ? e : 0.0;
        t_[r] = valid ? t : 0.0;
      }
      const V* ysrc;
      if (ts >= 0) {
        ysrc = tail + (size_t)ts * R * kStreamThreads;
      } else {
        const int u = first_tail - 1 - s;  // position in the staged sequence
        if (s - (kRing - 1) >= 0)
          stage_segment<V, R>(stage, (u + kRing - 1) % kRing, out, s - (kRing - 1), n, par, B, jc, jv, tid);
        cpa_commit();
        cpa_wait<kRing - 1>();
        ysrc = stage + (size_t)(u % kRing) * R * kStreamThreads;
      }
#pragma unroll
      for (int r = R - 1; r >= 0; --r) {
        const int i = s * R + r;
        const V yv = ysrc[r * kStreamThreads + tid];
        const V acc = ssub(ssub(yv, smul(e_[r], x1)), smul(t_[r], S));
        const V x = smul(rd_[r], acc);
        S = sadd(x1, S);
        x1 = x;
        if (jv && i < n) O::st_cs(rowp(out, i, j), x);
      }
    }
    cpa_wait<0>();
  }
}

// ======================================================================= biharmonic
template <typename V, int R>
__global__ void __launch_bounds__(kStreamThreads, 1) bih_stream_kernel(BihChunkArgs a, int tail_segs) {
  using O = VOps<V>;
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x, lane = tid & 31, par = tid >> 5;
  const int64_t B = a.batch;
  const int nb = a.n_bih;
  const int n = (nb - par + 1) / 2;
  const int nseg = (n + R - 1) / R;
  const int tseg = min(tail_segs, nseg);
  V* stage = reinterpret_cast<V*>(smem);
  V* tail = stage + kRing * R * kStreamThreads;
  const V* rhs = static_cast<const V*>(a.rhs);
  V* out = static_cast<V*>(a.out);
  const double xi0 = a.xi0;
  const uint64_t keep = policy_evict_last();
  const int64_t ngroups = (B + 31) / 32;
  auto rowp = [&](auto* base, int i, int64_t j) { return base + (int64_t)(par + 2 * i) * B + j; };

  for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
    const int64_t j = g * 32 + lane;
    const bool jv = j < B;
    const int64_t jc = jv ? j : B - 1;
    const double xi1 = __ldg(a.xi1 + jc), xi2 = __ldg(a.xi2 + jc);
    // ---------------- forward
#pragma unroll
    for (int q = 0; q < kRing - 1; ++q) {
      if (q < nseg) stage_segment<V, R>(stage, q, rhs, q, n, par, B, jc, jv, tid);
      cpa_commit();
    }
    BihU u{0, 0, 0, 0, 0, 0}, u1{0, 0, 0, 0, 0, 0}, u2{0, 0, 0, 0, 0, 0};
    V y1 = szero<V>(), y2 = szero<V>();
    for (int s = 0; s < nseg; ++s) {
      if (s + kRing - 1 < nseg) stage_segment<V, R>(stage, (s + kRing - 1) % kRing, rhs, s + kRing - 1, n, par, B, jc, jv, tid);
      cpa_commit();
      cpa_wait<kRing - 1>();
      const V* cur = stage + (size_t)(s % kRing) * R * kStreamThreads;
      const int ts = tail_slot(s, nseg, tseg);
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
        const V y = sfma(-l4, y2, sfma(-l2, y1, cur[r * kStreamThreads + tid]));
        y2 = y1;
        y1 = y;
        if (ts >= 0)
          tail[(ts * R + r) * kStreamThreads + tid] = y;
        else if (jv && i < n)
          st_keep(rowp(out, i, j), y, keep);
      }
    }
    // ---------------- backward
    cpa_wait<0>();
    const int first_tail = nseg - tseg;
#pragma unroll
    for (int q = 0; q < kRing - 1; ++q) {
      if (first_tail - 1 - q >= 0) stage_segment<V, R>(stage, q, out, first_tail - 1 - q, n, par, B, jc, jv, tid);
      cpa_commit();
    }
    V x1 = szero<V>(), x2 = szero<V>(), sq = szero<V>(), sv = szero<V>();
    for (int s = nseg - 1; s >= 0; --s) {
      const int ts = tail_slot(s, nseg, tseg);
      BihU w{0, 0, 0, 0, 0, 0}, w1{0, 0, 0, 0, 0, 0}, w2{0, 0, 0, 0, 0, 0};
      if (s > 0) {
        const double* ck = a.ckpt + ((int64_t)(s * 2 + par) * 10) * B + jc;
        w1.d = __ldg(ck); w1.e = __ldg(ck + B); w1.f = __ldg(ck + 2 * B); w1.a = __ldg(ck + 3 * B);
        w1.b = __ldg(ck + 4 * B);
        w2.d = __ldg(ck + 5 * B); w2.e = __ldg(ck + 6 * B); w2.f = __ldg(ck + 7 * B); w2.a = __ldg(ck + 8 * B);
        w2.b = __ldg(ck + 9 * B);
        w1.rd = rcp_fast(w1.d);
        w2.rd = s * R >= 2 ? rcp_fast(w2.d) : 0.0;
      }
      double rd_[R], e_[R], f_[R], a_[R], b_[R];
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
      }
      const V* ysrc;
      if (ts >= 0) {
        ysrc = tail + (size_t)ts * R * kStreamThreads;
      } else {
        const int u = first_tail - 1 - s;  // position in the staged sequence
        if (s - (kRing - 1) >= 0)
          stage_segment<V, R>(stage, (u + kRing - 1) % kRing, out, s - (kRing - 1), n, par, B, jc, jv, tid);
        cpa_commit();
        cpa_wait<kRing - 1>();
        ysrc = stage + (size_t)(u % kRing) * R * kStreamThreads;
      }
#pragma unroll
      for (int r = R - 1; r >= 0; --r) {
        const int i = s * R + r;
        const int k = min(par + 2 * i, nb - 1);
        const double qn = i < n ? __ldg(a.tab + (int64_t)k * B_NCOL + B_Q4) : 0.0;
        const double sn = i < n ? __ldg(a.tab + (int64_t)k * B_NCOL + B_S4) : 0.0;
        const V yv = ysrc[r * kStreamThreads + tid];
        V acc = ssub(ssub(yv, smul(e_[r], x1)), smul(f_[r], x2));
        acc = ssub(acc, smul(xi0, sadd(smul(a_[r], sq), smul(b_[r], sv))));
        const V x = smul(rd_[r], acc);
        sq = sfma(qn, x2, sq);
        sv = sfma(sn, x2, sv);
        x2 = x1;
        x1 = x;
        if (jv && i < n) O::st_cs(rowp(out, i, j), x);
      }
    }
    cpa_wait<0>();
  }
}

// ======================================================================= launchers
static int stream_ctas(int ctas_per_sm) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms * std::max(1, ctas_per_sm);
}

// shared memory for staging + tail; the tail takes what is left of `budget`
template <typename V, int R>
static int stream_tail_segs(int nseg_max, size_t fixed_bytes, size_t budget) {
  const size_t stage = (size_t)kRing * R * kStreamThreads * sizeof(V);
  const size_t per_seg = (size_t)R * kStreamThreads * sizeof(V);
  if (budget <= fixed_bytes + stage) return 0;
  const int t = (int)((budget - fixed_bytes - stage) / per_seg);
  return std::min(t, nseg_max);
}

template <typename V, int R>
static cudaError_t helm_stream_R(const HelmChunkArgs& a, int ctas_per_sm, cudaStream_t st) {
  const int n0 = (a.n_dir + 1) / 2;
  const int nseg0 = (n0 + R - 1) / R;
  const int tab_rows = nseg0 * R;
  const size_t tab_bytes = (size_t)2 * tab_rows * sizeof(double4);
  const size_t budget = (size_t)(220 * 1024) / std::max(1, ctas_per_sm);
  const int tail = stream_tail_segs<V, R>(nseg0, tab_bytes, budget);
  const size_t smem = (size_t)(kRing + tail) * R * kStreamThreads * sizeof(V) + tab_bytes;
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  cudaError_t err = cudaFuncSetAttribute(helm_stream_kernel<V, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  const int64_t groups = (a.batch + 31) / 32;
  const unsigned grid = (unsigned)std::min<int64_t>(groups, stream_ctas(ctas_per_sm));
  helm_stream_kernel<V, R><<<grid, kStreamThreads, smem, st>>>(a, tail, tab_rows);
  return cudaGetLastError();
}

template <typename V, int R>
static cudaError_t bih_stream_R(const BihChunkArgs& a, int ctas_per_sm, cudaStream_t st) {
  const int n0 = (a.n_bih + 1) / 2;
  const int nseg0 = (n0 + R - 1) / R;
  const size_t budget = (size_t)(200 * 1024) / std::max(1, ctas_per_sm);
  const int tail = stream_tail_segs<V, R>(nseg0, 0, budget);
  const size_t smem = (size_t)(kRing + tail) * R * kStreamThreads * sizeof(V);
  cudaError_t err = cudaFuncSetAttribute(bih_stream_kernel<V, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  const int64_t groups = (a.batch + 31) / 32;
  const unsigned grid = (unsigned)std::min<int64_t>(groups, stream_ctas(ctas_per_sm));
  bih_stream_kernel<V, R><<<grid, kStreamThreads, smem, st>>>(a, tail);
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

// `warps_per_sm` of the C ABI: resident CTAs per SM = warps_per_sm / 2
cudaError_t launch_helm_stream(const HelmChunkArgs& a, bool cplx_rhs, int warps_per_sm, cudaStream_t st) {
  if (a.batch <= 0) return cudaSuccess;
  const int ctas = std::max(1, warps_per_sm / 2);
  return cplx_rhs ? helm_stream_dispatch<cplx>(a, ctas, st) : helm_stream_dispatch<double>(a, ctas, st);
}

cudaError_t launch_bih_stream(const BihChunkArgs& a, bool cplx_rhs, int warps_per_sm, cudaStream_t st) {
  if (a.batch <= 0) return cudaSuccess;
  const int ctas = std::max(1, warps_per_sm / 2);
  return cplx_rhs ? bih_stream_dispatch<cplx>(a, ctas, st) : bih_stream_dispatch<double>(a, ctas, st);
}

}  // namespace shen
