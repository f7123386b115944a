// Structured matrix-vector products along the wall-normal axis (reference
// matrices.py:62-71 BandedMatrix.apply, :109-117 ConstantTailMatrix.apply,
// :145-152 Rank2TailMatrix.apply, :84-90 _parity_suffix_sum), batched over L
// lines (the (rows, L) layout of the solvers: lines contiguous, one thread
// per line, coalesced row accesses).
//
// The reference's evaluation order is kept exactly -- banded terms added to a
// zero row in offset order, only on each offset's valid row range; the tail
// term added last with the parity suffix sum accumulated bottom-up as
// s[j] = v[j] + s[j+2]; rank-2: diag * x, then + p sq, then + r ss -- so the
// results are bit-identical to the reference's (tests/test_apply_gpu.py).
// The suffix sums are carried in registers while each thread walks its
// line's rows from the bottom (x row j is folded into the running sum of its
// parity exactly when row j - tail_start is produced).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "shen_common.cuh"

namespace shen {
namespace {

constexpr int kMaxOff = 6;

struct ApplyArgs {
  int kind;  // 0 banded, 1 constant tail, 2 rank-2 tail
  int nr, nc;
  int64_t L;
  int n_off;
  int off[kMaxOff];
  const double* diag;  // [n_off][nr] (row-indexed; entries outside the valid range unused)
  const double* tail;  // [nr] (kind 1)
  int tail_start;      // kind 1
  const double* d;     // kind 2: diag, p, q, r, s [nr]
  const double* p;
  const double* q;
  const double* r;
  const double* s;
  int stage_lines;  // staged kernel: lines per block
};

template <typename V> struct A;
template <> struct A<double> {
  static __device__ __forceinline__ double zero() { return 0.0; }
  static __device__ __forceinline__ double ld(const double* p) { return __ldg(p); }
  static __device__ __forceinline__ double scale(double c, double v) { return __dmul_rn(c, v); }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
};
template <> struct A<cplx> {
  static __device__ __forceinline__ cplx zero() { return {0.0, 0.0}; }
  static __device__ __forceinline__ cplx ld(const cplx* p) {
    const double2 v = __ldg(reinterpret_cast<const double2*>(p));
    return {v.x, v.y};
  }
  // numpy casts the real factor to complex: (c + 0i)(a + bi); the 0 terms
  // leave c a, c b (signed zeros aside)
  static __device__ __forceinline__ cplx scale(double c, cplx v) { return {__dmul_rn(c, v.re), __dmul_rn(c, v.im)}; }
  static __device__ __forceinline__ cplx add(cplx a, cplx b) { return {__dadd_rn(a.re, b.re), __dadd_rn(a.im, b.im)}; }
};

template <bool SM>
__device__ __forceinline__ double ldt(const double* p) {
  if (SM) return *p;
  return __ldg(p);
}

// One line's walk (rows bottom-up).  X(j) reads x row j of this line; the
// table pointers in `a` point to global memory (SM = false) or to a shared
// copy (SM = true).
template <typename V, bool SM, typename FX>
__device__ __forceinline__ void apply_walk(const ApplyArgs& a, FX X, V* __restrict__ y, int64_t l) {
  using O = A<V>;
  const int64_t L = a.L;
  if (a.kind == 2) {
    // y = diag x; sq/ss = parity suffix sums of q x, s x; y[k] += p sq[k+2]; y[k] += r ss[k+2]
    const int n = a.nr;
    V sq[2] = {O::zero(), O::zero()}, ss[2] = {O::zero(), O::zero()};
    bool have[2] = {false, false};
    for (int k = n - 1; k >= 0; --k) {
      const int j = k + 2;  // fold x[j] into its parity's sums before row k uses them
      if (j < n) {
        const V xj = X(j);
        const V qx = O::scale(ldt<SM>(a.q + j), xj), sx = O::scale(ldt<SM>(a.s + j), xj);
        const int pj = j & 1;
        sq[pj] = have[pj] ? O::add(qx, sq[pj]) : qx;
        ss[pj] = have[pj] ? O::add(sx, ss[pj]) : sx;
        have[pj] = true;
      }
      V v = O::scale(ldt<SM>(a.d + k), X(k));
      if (k < n - 2) {
        v = O::add(v, O::scale(ldt<SM>(a.p + k), sq[k & 1]));
        v = O::add(v, O::scale(ldt<SM>(a.r + k), ss[k & 1]));
      }
      y[(int64_t)k * L + l] = v;
    }
    return;
  }
  V S[2] = {O::zero(), O::zero()};
  bool have[2] = {false, false};
  int next_j = a.nc - 1;  // next x row to fold into the suffix sums
  for (int k = a.nr - 1; k >= 0; --k) {
    V v = O::zero();
    for (int q = 0; q < a.n_off; ++q) {
      const int dk = a.off[q];
      const int k0 = dk < 0 ? -dk : 0, k1 = min(a.nr, a.nc - dk);
      if (k >= k0 && k < k1) v = O::add(v, O::scale(ldt<SM>(a.diag + (int64_t)q * a.nr + k), X(k + dk)));
    }
    if (a.kind == 1) {
      const int j = k + a.tail_start;
      if (j < a.nc) {
        // fold x rows from the bottom down to j (each once, in the
        // reference's s[j] = x[j] + s[j+2] order)
        for (; next_j >= j; --next_j) {
          const int pj = next_j & 1;
          S[pj] = have[pj] ? O::add(X(next_j), S[pj]) : X(next_j);
          have[pj] = true;
        }
        v = O::add(v, O::scale(ldt<SM>(a.tail + k), S[j & 1]));
      }
    }
    y[(int64_t)k * L + l] = v;
  }
}

template <typename V>
__global__ void apply_kernel(ApplyArgs a, const V* __restrict__ x, V* __restrict__ y) {
  using O = A<V>;
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= a.L) return;
  const int64_t L = a.L;
  apply_walk<V, false>(a, [&](int j) { return O::ld(x + (int64_t)j * L + l); }, y, l);
}

// Few lines (the stepper's mean-flow vectors, L = 1): one thread per line
// would wait a global-memory latency per row.  The block first stages its
// stage_lines (<= 8) lines of x and the row tables in shared memory (all
// threads, coalesced), then walks them from there -- same operations, same
// order.
constexpr int kStageThreads = 256;
constexpr int64_t kStagedMaxLines = 4096;  // below this the per-line walk is latency-bound

template <typename V>
__global__ void __launch_bounds__(kStageThreads) apply_staged_kernel(ApplyArgs a, const V* __restrict__ x,
                                                                     V* __restrict__ y) {
  extern __shared__ __align__(16) double sm[];
  const int LB = a.stage_lines;
  const int64_t l0 = (int64_t)blockIdx.x * LB;
  const int nl = (int)min((int64_t)LB, a.L - l0);
  V* xs = reinterpret_cast<V*>(sm);  // [nc][LB]
  double* ts = sm + (size_t)a.nc * LB * (sizeof(V) / sizeof(double));
  for (int idx = threadIdx.x; idx < a.nc * LB; idx += blockDim.x) {
    const int j = idx / LB, t = idx - j * LB;
    if (t < nl) xs[idx] = A<V>::ld(x + (int64_t)j * a.L + l0 + t);
  }
  // tables: the same pointers, rebased to the shared copy
  ApplyArgs b = a;
  auto stage = [&](const double* src, int count) -> const double* {
    double* dst = ts;
    for (int i = threadIdx.x; i < count; i += blockDim.x) dst[i] = __ldg(src + i);
    ts += count;
    return dst;
  };
  if (a.kind == 2) {
    b.d = stage(a.d, a.nr); b.p = stage(a.p, a.nr); b.q = stage(a.q, a.nr);
    b.r = stage(a.r, a.nr); b.s = stage(a.s, a.nr);
  } else {
    if (a.n_off > 0) b.diag = stage(a.diag, a.n_off * a.nr);
    if (a.kind == 1) b.tail = stage(a.tail, a.nr);
  }
  __syncthreads();
  const int t = threadIdx.x;
  if (t >= nl) return;
  apply_walk<V, true>(b, [&](int j) { return xs[j * LB + t]; }, y, l0 + t);
}

}  // namespace

cudaError_t launch_apply(int kind, int nr, int nc, int64_t L, int n_off, const int* offs, const double* diag,
                         const double* tail, int tail_start, const double* d, const double* p, const double* q,
                         const double* r, const double* s, const void* x, void* y, bool cplx_data, cudaStream_t st) {
  if (L <= 0 || nr <= 0) return cudaSuccess;
  if (n_off < 0 || n_off > kMaxOff) return cudaErrorInvalidValue;
  ApplyArgs a{};
  a.kind = kind; a.nr = nr; a.nc = nc; a.L = L; a.n_off = n_off;
  for (int i = 0; i < n_off; ++i) a.off[i] = offs[i];
  a.diag = diag; a.tail = tail; a.tail_start = tail_start;
  a.d = d; a.p = p; a.q = q; a.r = r; a.s = s;
  if (L < kStagedMaxLines) {
    const size_t tab = kind == 2 ? 5 * (size_t)nr : (size_t)(n_off + (kind == 1)) * nr;
    const size_t per_line = (size_t)nc * (cplx_data ? 16 : 8), budget = 48 * 1024;
    const int lines = tab * 8 + per_line <= budget ? (int)std::min<size_t>(8, (budget - tab * 8) / per_line) : 0;
    if (lines > 0) {
      a.stage_lines = lines;
      const size_t smem = per_line * lines + tab * 8;
      const unsigned blocks = (unsigned)((L + lines - 1) / lines);
      if (cplx_data)
        apply_staged_kernel<cplx><<<blocks, kStageThreads, smem, st>>>(a, static_cast<const cplx*>(x),
                                                                       static_cast<cplx*>(y));
      else
        apply_staged_kernel<double><<<blocks, kStageThreads, smem, st>>>(a, static_cast<const double*>(x),
                                                                         static_cast<double*>(y));
      return cudaGetLastError();
    }
  }
  const unsigned blocks = (unsigned)((L + 127) / 128);
  if (cplx_data)
    apply_kernel<cplx><<<blocks, 128, 0, st>>>(a, static_cast<const cplx*>(x), static_cast<cplx*>(y));
  else
    apply_kernel<double><<<blocks, 128, 0, st>>>(a, static_cast<const double*>(x), static_cast<double*>(y));
  return cudaGetLastError();
}

}  // namespace shen
