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

// row tables of one walk: global memory (SM = false) or a shared copy (SM = true)
struct Tabs {
  const double *diag, *tail, *d, *p, *q, *r, *s;
};

// One line's walk (rows bottom-up).  X(j) reads x row j of this line.  The
// sizes and offsets come from the kernel parameter `a` (constant bank; no
// local-memory copy), the tables from `t`.
template <typename V, bool SM, typename FX>
__device__ __forceinline__ void apply_walk(const ApplyArgs& a, const Tabs t, FX X, V* __restrict__ y, int64_t l) {
  using O = A<V>;
  const int64_t L = a.L;
  if (a.kind == 2) {
    // y = diag x; sq/ss = parity suffix sums of q x, s x; y[k] += p sq[k+2]; y[k] += r ss[k+2]
    const int n = a.nr;
    // suffix sums of the parity of row k (sq, ss) and of the other parity
    // (sq_o, ss_o), swapped every row: no dynamically indexed arrays (they
    // would live in local memory, on the dependency chain)
    V sq = O::zero(), ss = O::zero(), sq_o = O::zero(), ss_o = O::zero();
    bool have = false, have_o = false;
    for (int k = n - 1; k >= 0; --k) {
      const int j = k + 2;  // fold x[j] (same parity as k) into the sums before row k uses them
      if (j < n) {
        const V xj = X(j);
        const V qx = O::scale(ldt<SM>(t.q + j), xj), sx = O::scale(ldt<SM>(t.s + j), xj);
        sq = have ? O::add(qx, sq) : qx;
        ss = have ? O::add(sx, ss) : sx;
        have = true;
      }
      V v = O::scale(ldt<SM>(t.d + k), X(k));
      if (k < n - 2) {
        v = O::add(v, O::scale(ldt<SM>(t.p + k), sq));
        v = O::add(v, O::scale(ldt<SM>(t.r + k), ss));
      }
      y[(int64_t)k * L + l] = v;
      const V tq = sq, ts = ss;  // row k - 1 has the other parity
      const bool th = have;
      sq = sq_o; ss = ss_o; have = have_o;
      sq_o = tq; ss_o = ts; have_o = th;
    }
    return;
  }
  V S0 = O::zero(), S1 = O::zero();  // parity suffix sums (even / odd rows)
  bool have0 = false, have1 = false;
  int next_j = a.nc - 1;  // next x row to fold into the suffix sums
  for (int k = a.nr - 1; k >= 0; --k) {
    V v = O::zero();
#pragma unroll
    for (int q = 0; q < kMaxOff; ++q) {  // static indices: a stays in the parameter bank
      if (q >= a.n_off) break;
      const int dk = a.off[q];
      const int k0 = dk < 0 ? -dk : 0, k1 = min(a.nr, a.nc - dk);
      if (k >= k0 && k < k1) v = O::add(v, O::scale(ldt<SM>(t.diag + (int64_t)q * a.nr + k), X(k + dk)));
    }
    if (a.kind == 1) {
      const int j = k + a.tail_start;
      if (j < a.nc) {
        // fold x rows from the bottom down to j (each once, in the
        // reference's s[j] = x[j] + s[j+2] order)
        for (; next_j >= j; --next_j) {
          const V xj = X(next_j);
          if (next_j & 1) {
            S1 = have1 ? O::add(xj, S1) : xj;
            have1 = true;
          } else {
            S0 = have0 ? O::add(xj, S0) : xj;
            have0 = true;
          }
        }
        v = O::add(v, O::scale(ldt<SM>(t.tail + k), (j & 1) ? S1 : S0));
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
  const Tabs t{a.diag, a.tail, a.d, a.p, a.q, a.r, a.s};
  apply_walk<V, false>(a, t, [&](int j) { return O::ld(x + (int64_t)j * L + l); }, y, l);
}

// Many lines, parity-separable operator (every matrix of the set: all band
// offsets and the tail start of one parity, so rows of parity p read only x
// rows of parity (p + off) mod 2): one thread per (line, row parity) walks
// its rows bottom-up -- twice the threads, half the chain of apply_kernel --
// with the next rows' x loads issued ahead of the recurrence.  Each row gets
// the operations of apply_walk in the same order (banded terms in offset
// order onto zero, then the tail with its parity's suffix sum folded
// bottom-up), so the results stay bit-identical.
#ifndef SHEN_APPLY_PF
#define SHEN_APPLY_PF 6
#endif
constexpr int kApplyPf = SHEN_APPLY_PF;
template <typename V>
__global__ void __launch_bounds__(128) apply_par_kernel(ApplyArgs a, const V* __restrict__ x, V* __restrict__ y) {
  using O = A<V>;
  const int64_t L = a.L;
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);  // (32-line group, parity)
  const int par = (int)(w & 1);
  const int64_t l = (w >> 1) * 32 + (threadIdx.x & 31);
  if (l >= L) return;
  auto X = [&](int j) { return O::ld(x + (int64_t)j * L + l); };
  int k = a.nr - 1;
  if ((k & 1) != par) --k;
  if (a.kind == 2) {
    // y = d x; sq/ss: suffix sums of q x, s x over rows of parity par from k + 2 down
    V sq = O::zero(), ss = O::zero();
    bool have = false;
    for (; k >= 0; k -= 2) {
      const int j = k + 2;
      if (j < a.nr) {
        const V xj = X(j);
        const V qx = O::scale(__ldg(a.q + j), xj), sx = O::scale(__ldg(a.s + j), xj);
        sq = have ? O::add(qx, sq) : qx;
        ss = have ? O::add(sx, ss) : sx;
        have = true;
      }
      V v = O::scale(__ldg(a.d + k), X(k));
      if (k < a.nr - 2) {
        v = O::add(v, O::scale(__ldg(a.p + k), sq));
        v = O::add(v, O::scale(__ldg(a.r + k), ss));
      }
      y[(int64_t)k * L + l] = v;
    }
    return;
  }
  V S = O::zero();
  bool have = false;
  int next_j = -1;  // next x row of the tail parity to fold
  if (a.kind == 1) {
    next_j = a.nc - 1;
    if ((next_j & 1) != ((par + a.tail_start) & 1)) --next_j;
  }
  // With ~450 threads per SM on the config-3 lines the walk is bound by load
  // latency x loads in flight: the lowest x row a later step needs (the only
  // new one, the others were read by earlier steps) is prefetched kApplyPf
  // steps ahead.
  int dmin = a.kind == 1 ? a.tail_start : 0;
  for (int q = 0; q < a.n_off; ++q) dmin = min(dmin, a.off[q]);
  for (; k >= 0; k -= 2) {
    {
      const int r = k - 2 * kApplyPf + dmin;
      if (r >= 0 && r < a.nc) asm volatile("prefetch.global.L1 [%0];" ::"l"(x + (int64_t)r * L + l));
    }
    V v = O::zero();
#pragma unroll
    for (int q = 0; q < kMaxOff; ++q) {
      if (q >= a.n_off) break;
      const int dk = a.off[q];
      const int k0 = dk < 0 ? -dk : 0, k1 = min(a.nr, a.nc - dk);
      if (k >= k0 && k < k1) v = O::add(v, O::scale(__ldg(a.diag + (int64_t)q * a.nr + k), X(k + dk)));
    }
    if (a.kind == 1) {
      const int j = k + a.tail_start;
      if (j < a.nc) {
        for (; next_j >= j; next_j -= 2) {
          const V xj = X(next_j);
          S = have ? O::add(xj, S) : xj;
          have = true;
        }
        v = O::add(v, O::scale(__ldg(a.tail + k), S));
      }
    }
    y[(int64_t)k * L + l] = v;
  }
}

// Few lines (the stepper's mean-flow vectors, L = 1): a per-line walk is one
// thread doing ~100 dependent instructions per row.  Here a block takes
// stage_lines lines: (1) x and the row tables are staged in shared memory,
// (2) one thread per (line, parity) runs only the parity suffix sums (one
// add per row on the chain) into shared memory, (3) all threads form the
// rows in parallel.  Every row gets the same operations in the same order
// as in apply_walk, so the results are bit-identical.
constexpr int kStageThreads = 256;
constexpr int64_t kStagedMaxLines = 4096;  // below this the per-line walk is latency-bound

template <typename V>
__global__ void __launch_bounds__(kStageThreads) apply_staged_kernel(ApplyArgs a, const V* __restrict__ x,
                                                                     V* __restrict__ y) {
  using O = A<V>;
  extern __shared__ __align__(16) double sm[];
  const int LB = a.stage_lines, nr = a.nr, nc = a.nc;
  const int64_t l0 = (int64_t)blockIdx.x * LB;
  const int nl = (int)min((int64_t)LB, a.L - l0);
  V* xs = reinterpret_cast<V*>(sm);                       // [nc][LB]
  V* s1 = xs + (size_t)nc * LB;                           // kind 1: S [nc][LB]; kind 2: sq [nr][LB]
  V* s2 = s1 + (size_t)(a.kind == 2 ? nr : 0) * LB;      // kind 2: ss [nr][LB]
  double* ts = reinterpret_cast<double*>(s2 + (size_t)(a.kind == 2 ? nr : a.kind == 1 ? nc : 0) * LB);
  for (int idx = threadIdx.x; idx < nc * LB; idx += blockDim.x) {
    const int j = idx / LB, t = idx - j * LB;
    if (t < nl) xs[idx] = O::ld(x + (int64_t)j * a.L + l0 + t);
  }
  Tabs tb{a.diag, a.tail, a.d, a.p, a.q, a.r, a.s};
  auto stage = [&](const double* src, int count) -> const double* {
    double* dst = ts;
    for (int i = threadIdx.x; i < count; i += blockDim.x) dst[i] = __ldg(src + i);
    ts += count;
    return dst;
  };
  if (a.kind == 2) {
    tb.d = stage(a.d, nr); tb.p = stage(a.p, nr); tb.q = stage(a.q, nr);
    tb.r = stage(a.r, nr); tb.s = stage(a.s, nr);
  } else {
    if (a.n_off > 0) tb.diag = stage(a.diag, a.n_off * nr);
    if (a.kind == 1) tb.tail = stage(a.tail, nr);
  }
  __syncthreads();
  // (2) parity suffix sums, s[j] = v[j] + s[j + 2] from the bottom
  if (threadIdx.x < 2 * nl && a.kind != 0) {
    const int t = threadIdx.x >> 1, par = threadIdx.x & 1;
    if (a.kind == 1) {
      int j = nc - 1;
      if ((j & 1) != par) --j;
      V S = O::zero();
      for (bool have = false; j >= a.tail_start && j >= 0; j -= 2, have = true) {
        const V xj = xs[j * LB + t];
        S = have ? O::add(xj, S) : xj;
        s1[j * LB + t] = S;
      }
    } else {
      int j = nr - 1;
      if ((j & 1) != par) --j;
      V sq = O::zero(), ss = O::zero();
      for (bool have = false; j >= 2; j -= 2, have = true) {
        const V xj = xs[j * LB + t];
        const V qx = O::scale(tb.q[j], xj), sx = O::scale(tb.s[j], xj);
        sq = have ? O::add(qx, sq) : qx;
        ss = have ? O::add(sx, ss) : sx;
        s1[j * LB + t] = sq;
        s2[j * LB + t] = ss;
      }
    }
  }
  __syncthreads();
  // (3) rows in parallel
  for (int idx = threadIdx.x; idx < nr * LB; idx += blockDim.x) {
    const int k = idx / LB, t = idx - k * LB;
    if (t >= nl) continue;
    auto X = [&](int j) { return xs[j * LB + t]; };
    V v;
    if (a.kind == 2) {
      v = O::scale(tb.d[k], X(k));
      if (k < nr - 2) {
        v = O::add(v, O::scale(tb.p[k], s1[(k + 2) * LB + t]));
        v = O::add(v, O::scale(tb.r[k], s2[(k + 2) * LB + t]));
      }
    } else {
      v = O::zero();
#pragma unroll
      for (int q = 0; q < kMaxOff; ++q) {
        if (q >= a.n_off) break;
        const int dk = a.off[q];
        const int k0 = dk < 0 ? -dk : 0, k1 = min(nr, nc - dk);
        if (k >= k0 && k < k1) v = O::add(v, O::scale(tb.diag[q * nr + k], X(k + dk)));
      }
      if (a.kind == 1) {
        const int j = k + a.tail_start;
        if (j < nc) v = O::add(v, O::scale(tb.tail[k], s1[j * LB + t]));
      }
    }
    y[(int64_t)k * a.L + l0 + t] = v;
  }
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
    const size_t vb = cplx_data ? 16 : 8;
    const size_t per_line = vb * ((size_t)nc + (kind == 2 ? 2 * (size_t)nr : kind == 1 ? (size_t)nc : 0));
    const size_t budget = 160 * 1024;  // opt-in above 48 KB
    const int lines = tab * 8 + per_line <= budget ? (int)std::min<size_t>(8, (budget - tab * 8) / per_line) : 0;
    if (lines > 0) {
      a.stage_lines = lines;
      const size_t smem = per_line * lines + tab * 8;
      const unsigned blocks = (unsigned)((L + lines - 1) / lines);
      if (smem > 48 * 1024) {
        cudaError_t e = cplx_data
            ? cudaFuncSetAttribute(apply_staged_kernel<cplx>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
            : cudaFuncSetAttribute(apply_staged_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
      }
      if (cplx_data)
        apply_staged_kernel<cplx><<<blocks, kStageThreads, smem, st>>>(a, static_cast<const cplx*>(x),
                                                                       static_cast<cplx*>(y));
      else
        apply_staged_kernel<double><<<blocks, kStageThreads, smem, st>>>(a, static_cast<const double*>(x),
                                                                         static_cast<double*>(y));
      return cudaGetLastError();
    }
  }
  bool separable = true;  // every band offset (and the tail start) of one parity
  for (int i = 0; i < n_off; ++i) separable = separable && (((offs[i] - offs[0]) & 1) == 0);
  if (kind == 1 && n_off > 0) separable = separable && (((tail_start - offs[0]) & 1) == 0);
  if (separable) {
    const int64_t warps = ((L + 31) / 32) * 2;
    const unsigned pb = (unsigned)((warps + 3) / 4);
    if (cplx_data)
      apply_par_kernel<cplx><<<pb, 128, 0, st>>>(a, static_cast<const cplx*>(x), static_cast<cplx*>(y));
    else
      apply_par_kernel<double><<<pb, 128, 0, st>>>(a, static_cast<const double*>(x), static_cast<double*>(y));
    return cudaGetLastError();
  }
  const unsigned blocks = (unsigned)((L + 127) / 128);
  if (cplx_data)
    apply_kernel<cplx><<<blocks, 128, 0, st>>>(a, static_cast<const cplx*>(x), static_cast<cplx*>(y));
  else
    apply_kernel<double><<<blocks, 128, 0, st>>>(a, static_cast<const double*>(x), static_cast<double*>(y));
  return cudaGetLastError();
}

}  // namespace shen
