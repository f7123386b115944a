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
// Where y lives between the sweeps decides the HBM traffic.  Keeping it
// (in L2 or HBM) needs one y round trip per unknown; at the concurrency
// needed to hide the recurrences' latency (8-12 warps per SM) the y of the
// systems in flight does not fit L2, so the backward sweep instead re-reads
// the RHS segment and recomputes y from a per-segment y checkpoint (per-CTA
// scratch).  Traffic per unknown: 2 RHS reads + 1 solution write + the
// factor checkpoints (3 doubles per 8 rows for Helmholtz, 10 for the
// biharmonic) -- DESIGN.md section 4.2 has the measured numbers.  Latency is
// hidden by a per-thread cp.async ring that prefetches segments continuously
// across both sweeps and across system groups.
//
// Kernels: helm_stream_kernel / bih_stream_kernel (one system per thread);
// bih_pair_kernel (default for channel grids: mirror pairs (m, n) / (-m, n)
// share one factor recurrence, y checkpoints of the first 16 segments parked
// in tensor memory).  Variants measured slower (Helmholtz mirror pairs, a
// bulk-tensor-fed pair kernel) were removed from the product; DESIGN.md
// section 4.2 has their numbers.
#include <algorithm>
#include <cstdlib>
#include <type_traits>


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
// streaming RHS rows with an L2 evict-first policy (the pair kernel's y
// checkpoints, evict-last, then keep more of L2)
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void cpa_ef(cplx* dst, const cplx* src, bool pred, uint64_t pol) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  const int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;\n" ::"r"(s), "l"(src), "r"(n), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cpa_ef(double* dst, const double* src, bool pred, uint64_t pol) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  const int n = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2, %3;\n" ::"r"(s), "l"(src), "r"(n), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cpa(double* dst, const double* src, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  const int n = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(src), "r"(n) : "memory");
}
// y checkpoints: written in the forward sweep, read once in the backward;
// kept in L2 (evict_last) so the small per-CTA scratch does not round-trip
// through HBM (SHEN_YCKPT_KEEP=0 disables the hint)
#ifndef SHEN_YCKPT_KEEP
#define SHEN_YCKPT_KEEP 1
#endif
template <typename V>
__device__ __forceinline__ void ystore(V* p, V v) {
  if (SHEN_YCKPT_KEEP) st_keep(p, v, policy_evict_last());
  else *p = v;
}
// After its single read in the backward sweep a y checkpoint is dead: drop
// its L2 line without a write-back (discard.global.L2 acts as a weak write of
// an indeterminate value, ordered after this thread's read of the same
// address and before its next store there).  One lane per 128-B line.
#ifndef SHEN_YCKPT_DISCARD
#define SHEN_YCKPT_DISCARD 1
#endif
template <typename V>
__device__ __forceinline__ void ydiscard(const V* p, int lane) {
  constexpr int kPer = 128 / (int)sizeof(V);
  if (!SHEN_YCKPT_DISCARD) return;
  // the line also holds the checkpoints the other lanes of the warp read by
  // their own loads: order those reads before the discard explicitly
  __syncwarp(__activemask());
  if ((lane & (kPer - 1)) == 0 && ((reinterpret_cast<uintptr_t>(p) & 127) == 0))
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
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


// ---------------------------------------------------------------- tensor memory
// The biharmonic pair kernel parks the y checkpoints of its first segments
// (the longest-lived ones: written first in the forward sweep, read last in
// the backward) in TMEM instead of the L2-resident scratch.  Warp w owns lanes
// 32 (w % 4) .. +31 (the 32x32b shape: thread = lane) and a column range
// picked by w / 4.
#ifndef SHEN_PAIR_TMEM_SEGS
#define SHEN_PAIR_TMEM_SEGS 16
#endif
__device__ __forceinline__ void tmem_alloc512(uint32_t* slot) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(slot))
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc512(uint32_t base) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(base) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_st8(uint32_t a, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(a), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t a, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(a)
               : "memory");
}
__device__ __forceinline__ void tpack(double x, uint32_t* w) {
  w[0] = (uint32_t)__double2loint(x);
  w[1] = (uint32_t)__double2hiint(x);
}
__device__ __forceinline__ double tunpack(const uint32_t* w) { return __hiloint2double((int)w[1], (int)w[0]); }
__device__ __forceinline__ void tpack(cplx x, uint32_t* w) {
  tpack(x.re, w);
  tpack(x.im, w + 2);
}
template <typename V>
__device__ __forceinline__ V tunpackv(const uint32_t* w);
template <>
__device__ __forceinline__ double tunpackv<double>(const uint32_t* w) { return tunpack(w); }
template <>
__device__ __forceinline__ cplx tunpackv<cplx>(const uint32_t* w) { return {tunpack(w), tunpack(w + 2)}; }
// four values (y1, y2, z1, z2) of one checkpoint: 8 (real) or 16 (complex) columns
template <typename V>
__device__ __forceinline__ void tmem_put4(uint32_t a, V v0, V v1, V v2, V v3) {
  constexpr int W = sizeof(V) / 4;
  uint32_t w[4 * W];
  tpack(v0, w);
  tpack(v1, w + W);
  tpack(v2, w + 2 * W);
  tpack(v3, w + 3 * W);
  tmem_st8(a, w);
  if (W == 4) tmem_st8(a + 8, w + 8);
}
template <typename V>
__device__ __forceinline__ void tmem_get4(uint32_t a, V& v0, V& v1, V& v2, V& v3) {
  constexpr int W = sizeof(V) / 4;
  uint32_t w[4 * W];
  tmem_ld8(a, w);
  if (W == 4) tmem_ld8(a + 8, w + 8);
  tmem_wait_ld();
  v0 = tunpackv<V>(w);
  v1 = tunpackv<V>(w + W);
  v2 = tunpackv<V>(w + 2 * W);
  v3 = tunpackv<V>(w + 3 * W);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int kSG = 4;                    // 32-system groups per CTA (128 consecutive systems)
constexpr int kStreamThreads = 64 * kSG;  // warp w: parity w & 1, system group w >> 1

template <typename V>
__device__ __forceinline__ V* rowp_out(V* base, int par, int i, int64_t B, int64_t j) {
  return base + (int64_t)(par + 2 * i) * B + j;
}

constexpr int kRing = 3;  // stage buffers; prefetch distance kRing - 1 segments

// ---------------------------------------------------------------- per-thread segment stream
// Each thread streams its own column through a kRing-deep shared-memory ring
// with cp.async (16 B per row and thread; a warp covers whole 512-B row
// pieces).  The sequence of segments a thread consumes is continuous across
// the forward sweep (segments 0..nseg-1), the backward sweep (nseg-1..0) and
// consecutive system groups, so the prefetch distance never drains.
struct SegRef {
  int64_t g;
  int s;
};
// issue-side cursor over that sequence (no 64-bit division per segment)
struct SegIt {
  int64_t g;
  int k;  // position within the group's 2 nseg segments
  __device__ __forceinline__ SegRef ref(int nseg) const { return {g, k < nseg ? k : 2 * nseg - 1 - k}; }
  __device__ __forceinline__ void next(int nseg, int64_t gstride) {
    if (++k == 2 * nseg) {
      k = 0;
      g += gstride;
    }
  }
};


template <typename V, int R, int SG>
__device__ __forceinline__ void seg_issue(V* slot, const V* rhs, SegRef ref, int n, int par, int64_t B,
                                          int64_t ngroups, int64_t jb, int64_t je, int sgi, int lane,
                                          uint64_t pol = 0) {
  if (ref.g < ngroups) {
    const int64_t j = jb + ref.g * (32 * SG) + sgi * 32 + lane;
    const bool jv = j < je;
    const int64_t jc = jv ? j : je - 1;
    const V* p = rhs + (int64_t)(par + 2 * ref.s * R) * B + jc;
    const int64_t step = 2 * B;
    const int rows = min(R, n - ref.s * R);
    // walk the rows with pointer increments; rows past the end re-use the
    // last valid address with a zero-fill (src-size 0) copy
    if (jv && rows == R) {  // every segment but the last: no per-row predicates
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (pol) cpa_ef(slot + r * 32, p, true, pol);
        else cpa(slot + r * 32, p, true);
        p += step;
      }
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (pol) cpa_ef(slot + r * 32, p, jv && r < rows, pol);
        else cpa(slot + r * 32, p, jv && r < rows);
        if (r + 1 < rows) p += step;
      }
    }
  }
  cpa_commit();
}

// ======================================================================= Helmholtz
// v5: recompute-y streaming solve, per-thread cp.async ring, row constants
// read through the L1 (warp-uniform broadcast loads).  CTA = 2 warps
// (parity 0 / 1 of the same 32 systems).  HBM traffic per unknown: 2 RHS
// reads + 1 solution write (+ ~3 B of checkpoints).
template <typename V, int R, int RING, int SG>
__global__ void __launch_bounds__(64 * SG, 1) helm_stream_kernel(HelmChunkArgs a, V* ychk, int tab_rows) {
  constexpr int kT = 64 * SG;
  using O = VOps<V>;
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, par = warp & 1, sgi = warp >> 1;
  const int64_t B = a.batch;
  const int n = (a.n_dir - par + 1) / 2;
  const int nseg = (n + R - 1) / R;
  V* ring = reinterpret_cast<V*>(smem) + (size_t)warp * RING * R * 32 + lane;  // this thread's column
  const V* rhs = static_cast<const V*>(a.rhs);
  V* out = static_cast<V*>(a.out);
  // row constants (sd, st, md, has_sup) of both parities in shared memory,
  // loaded once per persistent CTA
  double4* tab = reinterpret_cast<double4*>(smem + (size_t)kT / 32 * RING * R * 32 * VOps<V>::ndouble);
  for (int idx = tid; idx < 2 * tab_rows; idx += kT) {
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
  const int64_t jb = a.jb, je = a.je < 0 ? B : a.je;
  const int64_t ngroups = (je - jb + 32 * SG - 1) / (32 * SG);
  const int64_t g0 = blockIdx.x, gstride = gridDim.x;
  if (g0 >= ngroups) return;
  const int64_t nq = ((ngroups - g0 + gstride - 1) / gstride) * 2 * nseg;
  int64_t qi = 0;
  int islot = 0, cslot = 0;  // ring slots being issued / consumed (no 64-bit modulo)
  SegIt it{g0, 0};
  for (; qi < RING - 1; ++qi) {
    if (qi < nq) seg_issue<V, R, SG>(ring + islot * R * 32, rhs, it.ref(nseg), n, par, B, ngroups, jb, je, sgi, lane);
    else cpa_commit();
    it.next(nseg, gstride);
    islot = islot + 1 == RING ? 0 : islot + 1;
  }
  auto consume = [&]() -> const V* {
    if (qi < nq) seg_issue<V, R, SG>(ring + islot * R * 32, rhs, it.ref(nseg), n, par, B, ngroups, jb, je, sgi, lane);
    else cpa_commit();
    it.next(nseg, gstride);
    ++qi;
    islot = islot + 1 == RING ? 0 : islot + 1;
    cpa_wait<RING - 1>();
    const V* p = ring + cslot * R * 32;
    cslot = cslot + 1 == RING ? 0 : cslot + 1;
    return p;
  };

  for (int64_t g = g0; g < ngroups; g += gstride) {
    const int64_t j = jb + g * (32 * SG) + sgi * 32 + lane;
    const bool jv = j < je;
    const int64_t jc = jv ? j : je - 1;
    const double cb = __ldg(a.cb + jc);
    const double sub = __dmul_rn(cb, -1.5707963267948966);
    V* outj = out + (int64_t)par * B + j;
    // y checkpoints: per-CTA scratch, [segment][thread] (only the group in flight)
    V* ychkj = ychk + (int64_t)blockIdx.x * (int64_t)(((a.n_dir + 1) / 2 + R - 1) / R) * kT + tid;
    const double* ckj = a.ckpt + (int64_t)par * 3 * B + jc;
    // ---------------- forward: y at segment ends only
    HelmProj pj;
    hp_origin(pj);
    V y = szero<V>();
    double dl = 0.0, el = 0.0, tl = 0.0;
    for (int s = 0; s < nseg; ++s) {
      const V* cur = consume();
      if (s > 0) hp_start(pj, dl, el, tl);
      const bool full = (s + 1) * R <= n;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = s * R + r;
        const double4 tv = mytab[i];
        const HelmRow row = helm_row(a.ca, cb, sub, tv.x, tv.y, tv.z, tv.w != 0.0);
        if (r > 0 && (r & 7) == 0) hp_rescale(pj);
        double d, e, t;
        const double low = hp_step(pj, row, sub, d, e, t);
        dl = d; el = e; tl = t;
        const V b = (full || i < n) ? cur[r * 32] : szero<V>();
        y = sfma(-low, y, b);
      }
      if (s + 1 < nseg) ystore(ychkj + s * kT, y);
    }
    // ---------------- backward: re-stream each segment (bottom first)
    V x1 = szero<V>(), S = szero<V>();
    // scalars of the next (lower) segment, loaded one segment ahead
    double ckd = 1.0, cke = 0.0, ckt = 0.0;
    V ckyv = szero<V>();
    if (nseg - 1 > 0) {
      const double* ck = ckj + (int64_t)6 * (nseg - 1) * B;
      ckd = __ldg(ck); cke = __ldg(ck + B); ckt = __ldg(ck + 2 * B);
      ckyv = ychkj[(nseg - 2) * kT];
    }
    for (int s = nseg - 1; s >= 0; --s) {
      HelmProj q;
      V yy = szero<V>();
      if (s == 0) {
        hp_origin(q);
      } else {
        hp_start(q, ckd, cke, ckt);
        yy = ckyv;
      }
      if (s > 0) ydiscard(ychkj + (s - 1) * kT, lane);
      if (s - 1 > 0) {
        const double* ck = ckj + (int64_t)6 * (s - 1) * B;
        ckd = __ldg(ck); cke = __ldg(ck + B); ckt = __ldg(ck + 2 * B);
        ckyv = ychkj[(s - 2) * kT];
      }
      const V* cur = consume();
      const bool full = (s + 1) * R <= n;
      double rd_[R], e_[R], t_[R];
      V y_[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = s * R + r;
        const double4 tv = mytab[i];
        const HelmRow row = helm_row(a.ca, cb, sub, tv.x, tv.y, tv.z, tv.w != 0.0);
        if (r > 0 && (r & 7) == 0) hp_rescale(q);
        double d, e, t;
        const double low = hp_step(q, row, sub, d, e, t);
        const bool valid = full || i < n;
        yy = sfma(-low, yy, valid ? cur[r * 32] : szero<V>());
        y_[r] = yy;
        rd_[r] = valid ? q.rd : 0.0;
        e_[r] = valid ? e : 0.0;
        t_[r] = valid ? t : 0.0;
      }
#pragma unroll
      for (int r = R - 1; r >= 0; --r) {
        const V acc = ssub(ssub(y_[r], smul(e_[r], x1)), smul(t_[r], S));
        const V x = smul(rd_[r], acc);
        S = sadd(x1, S);
        x1 = x;
        if (jv && (full || s * R + r < n)) O::st_cs(outj + (int64_t)2 * (s * R + r) * B, x);
      }
    }
  }
  cpa_wait<0>();
}

// ======================================================================= biharmonic
// PP: one parity per CTA (even CTAs parity 0, odd parity 1) with a one-parity
// row table -- half the shared memory, used when the both-parity table does
// not fit (n_x >= ~1800).
template <typename V, int R, bool SMEM_TAB, int RING, int SG, bool PP>
__global__ void __launch_bounds__(64 * SG, 1) bih_stream_kernel(BihChunkArgs a, V* ychk) {
  constexpr int kT = 64 * SG;
  constexpr int SGE = PP ? 2 * SG : SG;  // 32-system groups per CTA work item
  using O = VOps<V>;
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int par = PP ? (int)(blockIdx.x & 1) : (warp & 1), sgi = PP ? warp : (warp >> 1);
  const int64_t B = a.batch;
  const int nb = a.n_bih;
  const int n = (nb - par + 1) / 2;
  const int nseg = (n + R - 1) / R;
  V* ring = reinterpret_cast<V*>(smem) + (size_t)warp * RING * R * 32 + lane;
  // row-constant table: a compact shared-memory copy when it fits (loaded
  // once per persistent CTA), else the 18-column table through the read-only
  // path.  The compact rows keep the 13 per-mode values; the m-band and q/s
  // lookahead entries are read from rows k-2 / k-4 (4 virtual rows in front).
  double* stab = smem + (size_t)kT / 32 * RING * R * 32 * VOps<V>::ndouble;
  if (SMEM_TAB && PP) {
    // one parity: position i + 2 holds parity row i (mode par + 2 i); two virtual rows in front
    for (int q = tid; q < (n + 2) * BC_STRIDE; q += kT) {
      const int pos = q / BC_STRIDE, col = q - pos * BC_STRIDE, i = pos - 2;
      double v = 0.0;
      if (i >= 0 && col < BC_NCOL) {
        v = __ldg(a.tab + (int64_t)(par + 2 * i) * B_STRIDE + bc_src(col));
        if (col == BC_P || col == BC_R || col == BC_Q0 || col == BC_T2 || col == BC_T4)
          v = __dmul_rn(a.xi0, v);  // == bih_fast_prescale
      } else if (i == -1 && (col == BC_Q4 || col == BC_S4)) {
        v = __ldg(a.tab + (int64_t)par * B_STRIDE + (col == BC_Q4 ? B_Q2 : B_S2));
      }
      stab[q] = v;
    }
    __syncthreads();
  } else if (SMEM_TAB) {
    for (int q = tid; q < (nb + 4) * BC_STRIDE; q += kT) {
      const int kk = q / BC_STRIDE - 4, col = q - (kk + 4) * BC_STRIDE;
      double v = 0.0;
      if (kk >= 0 && col < BC_NCOL) {
        v = __ldg(a.tab + (int64_t)kk * B_STRIDE + bc_src(col));
        if (col == BC_P || col == BC_R || col == BC_Q0 || col == BC_T2 || col == BC_T4)
          v = __dmul_rn(a.xi0, v);  // == bih_fast_prescale
      }
      else if (kk >= -2 && (col == BC_Q4 || col == BC_S4))
        v = __ldg(a.tab + (int64_t)(kk + 2) * B_STRIDE + (col == BC_Q4 ? B_Q2 : B_S2));
      stab[q] = v;
    }
    __syncthreads();
  }
  const double* tab = a.tab;
  // table position of parity row i and the position step between rows k-2 and k
  auto tpos = [&](int i) { return PP ? i + 2 : par + 2 * i + 4; };
  constexpr int tstep = PP ? 1 : 2;
  auto row_consts = [&](int i, double* c) {  // parity row i (mode par + 2 i)
    if (SMEM_TAB) load_bih_row_compact(stab, tpos(i), tstep, c); else load_bih_row(tab, par + 2 * i, c);
  };
  auto q4s4 = [&](int i, double& q4, double& s4) {
    if (SMEM_TAB) {
      const double2 v = *reinterpret_cast<const double2*>(stab + (int64_t)tpos(i) * BC_STRIDE + BC_Q4);
      q4 = v.x; s4 = v.y;
    } else {
      const int k = par + 2 * i;
      q4 = tab[(int64_t)k * B_STRIDE + B_Q4];
      s4 = tab[(int64_t)k * B_STRIDE + B_S4];
    }
  };
  const V* rhs = static_cast<const V*>(a.rhs);
  V* out = static_cast<V*>(a.out);
  const double xi0 = a.xi0;
  const int64_t jb = a.jb, je = a.je < 0 ? B : a.je;
  const int64_t ngroups = (je - jb + 32 * SGE - 1) / (32 * SGE);
  const int64_t g0 = PP ? (blockIdx.x >> 1) : blockIdx.x;
  const int64_t gstride = PP ? ((gridDim.x + 1 - par) >> 1) : gridDim.x;
  if (g0 >= ngroups) return;
  const int64_t nq = ((ngroups - g0 + gstride - 1) / gstride) * 2 * nseg;
  int64_t qi = 0;
  int islot = 0, cslot = 0;  // ring slots being issued / consumed (no 64-bit modulo)
  SegIt it{g0, 0};
  for (; qi < RING - 1; ++qi) {
    if (qi < nq) seg_issue<V, R, SGE>(ring + islot * R * 32, rhs, it.ref(nseg), n, par, B, ngroups, jb, je, sgi, lane);
    else cpa_commit();
    it.next(nseg, gstride);
    islot = islot + 1 == RING ? 0 : islot + 1;
  }
  auto consume = [&]() -> V* {
    if (qi < nq) seg_issue<V, R, SGE>(ring + islot * R * 32, rhs, it.ref(nseg), n, par, B, ngroups, jb, je, sgi, lane);
    else cpa_commit();
    it.next(nseg, gstride);
    ++qi;
    islot = islot + 1 == RING ? 0 : islot + 1;
    cpa_wait<RING - 1>();
    V* p = ring + cslot * R * 32;
    cslot = cslot + 1 == RING ? 0 : cslot + 1;
    return p;
  };

  for (int64_t g = g0; g < ngroups; g += gstride) {
    const int64_t j = jb + g * (32 * SGE) + sgi * 32 + lane;
    const bool jv = j < je;
    const int64_t jc = jv ? j : je - 1;
    const double xi1 = __ldg(a.xi1 + jc), xi2 = __ldg(a.xi2 + jc);
    V* outj = out + (int64_t)par * B + j;
    V* ychkj = ychk + (int64_t)blockIdx.x * (int64_t)(((nb + 1) / 2 + R - 1) / R) * 2 * kT + tid;
    const double* ckj = a.ckpt + (int64_t)par * 10 * B + jc;
    // Segments are processed by generic lambdas instantiated twice: FULL
    // segments (all R rows valid -- every segment but possibly the last) run
    // without row masks or row-index clamps; the last one is masked.
    using Full = std::integral_constant<bool, true>;
    using Part = std::integral_constant<bool, false>;
    // ---------------- forward
    BihU u{0, 0, 0, 0, 0, 0}, u1{0, 0, 0, 0, 0, 0}, u2{0, 0, 0, 0, 0, 0};
    V y1 = szero<V>(), y2 = szero<V>();
    auto fwd_seg = [&](int s, auto full_tag) {
      constexpr bool FULL = decltype(full_tag)::value;
      constexpr bool CARRY = FULL && SMEM_TAB;  // k-2 / k-4 entries from registers
      const V* cur = consume();
      BihCarry cr;
      BihProd pr;
      if (CARRY) {
        bih_carry_init(stab, tpos(s * R), tstep, cr);
        bih_prod_init(xi2, cr, pr);
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = s * R + r;
        const int ic = FULL ? i : min(i, n - 1);
        double c[B_NCOL];
        double l2, l4;
        if (CARRY) {
          load_bih_row_carry(stab, tpos(ic), c, cr);
          bih_row_fast_carried(u, u1, u2, c, xi1, xi2, pr, r == 0, l2, l4);
        } else {
          row_consts(ic, c);
          if (!SMEM_TAB) bih_fast_prescale(c, xi0);  // the compact table is pre-scaled
          const BihBands hb = bih_bands_fast(xi1, xi2, c);
          bih_step_fast(u, u1, u2, hb, c, l2, l4);
        }
        u2 = u1;
        u1 = u;
        const V b = (FULL || i < n) ? cur[r * 32] : szero<V>();
        const V y = sfma(-l4, y2, sfma(-l2, y1, b));
        y2 = y1;
        y1 = y;
      }
    };
    const int nfull = n / R;  // segments with all R rows valid
    for (int s = 0; s < nseg; ++s) {
      if (s < nfull) fwd_seg(s, Full{}); else fwd_seg(s, Part{});
      if (s + 1 < nseg) {
        ystore(ychkj + (2 * s) * kT, y1);
        ystore(ychkj + (2 * s + 1) * kT, y2);
      }
    }
    // ---------------- backward
    // Checkpoint of the segment below the one being processed is prefetched
    // into registers (8-warp CTA); the 12-warp CTA has no registers to spare
    // and loads it at segment start.
    constexpr bool PF = (SG == 4);
    V x1 = szero<V>(), x2 = szero<V>(), sq = szero<V>(), sv = szero<V>();
    double ck[10];
    V cya = szero<V>(), cyb = szero<V>();
    auto load_ck = [&](int s) {
      const double* cp = ckj + (int64_t)20 * s * B;
#pragma unroll
      for (int q = 0; q < 10; ++q) ck[q] = __ldg(cp + q * B);
      cya = ychkj[(2 * (s - 1)) * kT];
      cyb = ychkj[(2 * (s - 1) + 1) * kT];
    };
    auto bwd_seg = [&](int s, auto full_tag) {
      constexpr bool FULL = decltype(full_tag)::value;
      BihU w{0, 0, 0, 0, 0, 0}, w1{0, 0, 0, 0, 0, 0}, w2{0, 0, 0, 0, 0, 0};
      V ya = szero<V>(), yb = szero<V>();
      if (s > 0) {  // factor state and y entering the segment
        if (!PF) load_ck(s);
        w1.d = ck[0]; w1.e = ck[1]; w1.f = ck[2]; w1.a = ck[3]; w1.b = ck[4];
        w2.d = ck[5]; w2.e = ck[6]; w2.f = ck[7]; w2.a = ck[8]; w2.b = ck[9];
        ya = cya;
        yb = cyb;
        ydiscard(ychkj + (2 * (s - 1)) * kT, lane);
        ydiscard(ychkj + (2 * (s - 1) + 1) * kT, lane);
        bih_set_rcp(w1);
        if (s * R >= 2) bih_set_rcp(w2);
        else bih_clear_rcp(w2);
      }
      if (PF && s - 1 > 0) load_ck(s - 1);
      V* cur = consume();
      constexpr bool CARRY = FULL && SMEM_TAB;
      BihCarry cr;
      BihProd pr;
      if (CARRY) {
        bih_carry_init(stab, tpos(s * R), tstep, cr);
        bih_prod_init(xi2, cr, pr);
      }
      // U-row entries pre-multiplied by 1/d (rows past n get 0, so x = 0 there):
      // x_i = y~_i - e~_i x_{i+1} - f~_i x_{i+2} - a~_i S_q - b~_i S_s
      double e_[R], f_[R], a_[R], b_[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = s * R + r;
        const int ic = FULL ? i : min(i, n - 1);
        double c[B_NCOL];
        double l2, l4;
        if (CARRY) {
          load_bih_row_carry(stab, tpos(ic), c, cr);
          bih_row_fast_carried(w, w1, w2, c, xi1, xi2, pr, r == 0, l2, l4);
        } else {
          row_consts(ic, c);
          if (!SMEM_TAB) bih_fast_prescale(c, xi0);
          const BihBands hb = bih_bands_fast(xi1, xi2, c);
          bih_step_fast(w, w1, w2, hb, c, l2, l4);
        }
        w2 = w1;
        w1 = w;
        const bool valid = FULL || i < n;
        const V y = sfma(-l4, yb, sfma(-l2, ya, valid ? cur[r * 32] : szero<V>()));
        yb = ya;
        ya = y;
        const double rd = valid ? w.rd : 0.0;
        cur[r * 32] = smul(rd, y);  // y~ replaces b in this thread's ring slot (frees R registers)
        e_[r] = rd * w.e;
        f_[r] = rd * w.f;
        a_[r] = rd * w.a;
        b_[r] = rd * w.b;
      }
      V* op = outj + (int64_t)2 * (s * R) * B;
#pragma unroll
      for (int r = R - 1; r >= 0; --r) {
        const int i = s * R + r;
        const bool valid = FULL || i < n;
        double qn, sn;
        q4s4(FULL ? i : min(i, n - 1), qn, sn);
        if (!valid) qn = sn = 0.0;
        V x = sfma(-e_[r], x1, cur[r * 32]);
        x = sfma(-f_[r], x2, x);
        x = sfma(-a_[r], sq, x);  // a~, b~ carry xi0
        x = sfma(-b_[r], sv, x);
        sq = sfma(qn, x2, sq);
        sv = sfma(sn, x2, sv);
        x2 = x1;
        x1 = x;
        if (jv && valid) O::st_cs(op + (int64_t)2 * r * B, x);
      }
    };
    if (PF && nseg - 1 > 0) load_ck(nseg - 1);
    for (int s = nseg - 1; s >= 0; --s) {
      if (s < nfull) bwd_seg(s, Full{}); else bwd_seg(s, Part{});
    }
  }
  cpa_wait<0>();
}

// ======================================================================= biharmonic, mirror pairs
// Systems (m, n) and (-m, n) of a channel grid have bitwise-identical z2, so
// the reference computes bitwise-identical factors for them.  One thread
// solves such a pair: the factor recurrence (bands, elimination, reciprocal
// -- ~2/3 of the biharmonic's fp64 work) and the row-table reads run once for
// two right-hand sides, and the factor checkpoints are read once for two.
// Every per-system operation is the one bih_stream_kernel performs, so the
// results are bit-identical to it.  Work items are pairs (P of them; an
// unpaired system is a pair of itself and is stored once); one parity per
// CTA with the one-parity compact table (the two RHS streams double the ring).
template <typename V, int R, int SG>
__global__ void __launch_bounds__(64 * SG, 1) bih_pair_kernel(BihChunkArgs a, V* ychk) {
  constexpr int kT = 64 * SG;
  constexpr int SGE = 2 * SG;  // 32-item groups per CTA work item (one parity per CTA)
  constexpr int RING = 2;
  using O = VOps<V>;
  extern __shared__ __align__(16) double smem_raw[];
  // ring rows 128-B aligned: the dynamic window is requested 128 B larger
  // (pointer arithmetic on the shared array itself, so the compiler keeps
  // the shared address space: LDS/STS, not generic loads)
  const uint32_t sbase = smem_u32(smem_raw);
  double* smem = smem_raw + ((((sbase + 127u) & ~127u) - sbase) >> 3);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int par = (int)(blockIdx.x & 1), sgi = warp;
  const int64_t B = a.batch;
  const int nb = a.n_bih;
  const int n = (nb - par + 1) / 2;
  const int nseg = (n + R - 1) / R;
  // ring slot: rows 0..R-1 of stream 0, then rows 0..R-1 of stream 1
  V* ring = reinterpret_cast<V*>(smem) + (size_t)warp * RING * 2 * R * 32 + lane;
  double* stab = smem + (size_t)kT / 32 * RING * 2 * R * 32 * VOps<V>::ndouble;
  // backward: the next segment's factor checkpoint (10 doubles) and y
  // checkpoints (4 values) land here by cp.async while the current segment
  // runs (registers have no room for a prefetch): ckd[q][kT], cky[q][kT]
  double* ckd = stab + (size_t)(n + 2) * BC_STRIDE;
  V* cky = reinterpret_cast<V*>(ckd + 10 * kT);
  for (int q = tid; q < (n + 2) * BC_STRIDE; q += kT) {
    const int pos = q / BC_STRIDE, col = q - pos * BC_STRIDE, i = pos - 2;
    double v = 0.0;
    if (i >= 0 && col < BC_NCOL) {
      v = __ldg(a.tab + (int64_t)(par + 2 * i) * B_STRIDE + bc_src(col));
      if (col == BC_P || col == BC_R || col == BC_Q0 || col == BC_T2 || col == BC_T4)
        v = __dmul_rn(a.xi0, v);  // == bih_fast_prescale
    } else if (i == -1 && (col == BC_Q4 || col == BC_S4)) {
      v = __ldg(a.tab + (int64_t)par * B_STRIDE + (col == BC_Q4 ? B_Q2 : B_S2));
    }
    stab[q] = v;
  }
  __syncthreads();
  auto tpos = [&](int i) { return i + 2; };
  constexpr int tstep = 1;
  auto q4s4 = [&](int i, double& q4, double& s4) {
    const double2 v = *reinterpret_cast<const double2*>(stab + (int64_t)tpos(i) * BC_STRIDE + BC_Q4);
    q4 = v.x; s4 = v.y;
  };
  const V* rhs = static_cast<const V*>(a.rhs);
  V* out = static_cast<V*>(a.out);
  const int64_t P = a.n_pairs;
  const int64_t* pa = a.pairs;
  const int64_t* pb = a.pairs + P;
  const int64_t ngroups = (P + 32 * SGE - 1) / (32 * SGE);
  const int64_t g0 = blockIdx.x >> 1;
  const int64_t gstride = (gridDim.x + 1 - par) >> 1;
  if (g0 >= ngroups) return;
  const int64_t nq = ((ngroups - g0 + gstride - 1) / gstride) * 2 * nseg;
  // TMEM for the y checkpoints of segments 0 .. KTM-1 (4 values each)
  constexpr int KTM = (SG == 4 && SHEN_PAIR_TMEM_SEGS > 0) ? SHEN_PAIR_TMEM_SEGS : 0;
  constexpr int TCOL = (int)sizeof(V);  // columns per checkpoint: 4 values x sizeof(V) / 4 B
  static_assert(KTM * TCOL <= 256, "two warps share a lane quadrant: 256 columns each");
  __shared__ uint32_t tmem_slot;
  uint32_t tbase = 0;
  if (KTM > 0) {
    if (warp == 0) tmem_alloc512(&tmem_slot);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    tbase = tmem_slot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(256 * (warp >> 2));
  }
  // per-thread segment stream over both systems of the thread's pair; the
  // pair's system indices are loaded once per group (a dependent global load
  // per segment issue was the kernel's largest stall)
  int64_t ig = -1, ija = 0, ijb = 0;
  auto issue = [&](V* slot, SegRef ref) {
    if (ref.g < ngroups) {
      const int64_t c = ref.g * (32 * SGE) + sgi * 32 + lane;
      const bool cv = c < P;
      if (ref.g != ig) {
        const int64_t cc = cv ? c : P - 1;
        ija = __ldg(pa + cc);
        ijb = __ldg(pb + cc);
        ig = ref.g;
      }
      const int64_t ja = ija, jb2 = ijb;
      const int rows = min(R, n - ref.s * R);
      const int64_t step = 2 * B;
      const V* p0 = rhs + (int64_t)(par + 2 * ref.s * R) * B + ja;
      const V* p1 = rhs + (int64_t)(par + 2 * ref.s * R) * B + jb2;
#ifndef SHEN_PAIR_EF
#define SHEN_PAIR_EF 0  // measured: evict-first RHS rows cost more DRAM reads (23.5 vs 22.6 ms)
#endif
      const uint64_t pol = policy_evict_first();
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const bool ok = cv && r < rows;
        if (SHEN_PAIR_EF) {
          cpa_ef(slot + r * 32, p0, ok, pol);
          cpa_ef(slot + (R + r) * 32, p1, ok, pol);
        } else {
          cpa(slot + r * 32, p0, ok);
          cpa(slot + (R + r) * 32, p1, ok);
        }
        if (r + 1 < rows) {
          p0 += step;
          p1 += step;
        }
      }
    }
    cpa_commit();
  };
  int64_t qi = 0;
  int islot = 0, cslot = 0;  // ring slots being issued / consumed (no 64-bit modulo)
  SegIt it{g0, 0};
  for (; qi < RING - 1; ++qi) {
    if (qi < nq) issue(ring + islot * 2 * R * 32, it.ref(nseg));
    else cpa_commit();
    it.next(nseg, gstride);
    islot = islot + 1 == RING ? 0 : islot + 1;
  }
  auto consume = [&]() -> V* {
    if (qi < nq) issue(ring + islot * 2 * R * 32, it.ref(nseg));
    else cpa_commit();
    it.next(nseg, gstride);
    ++qi;
    islot = islot + 1 == RING ? 0 : islot + 1;
    cpa_wait<RING - 1>();
    V* p = ring + cslot * 2 * R * 32;
    cslot = cslot + 1 == RING ? 0 : cslot + 1;
    return p;
  };

  for (int64_t g = g0; g < ngroups; g += gstride) {
    const int64_t c = g * (32 * SGE) + sgi * 32 + lane;
    const bool cv = c < P;
    const int64_t cc = cv ? c : P - 1;
    const int64_t ja = __ldg(pa + cc), jb2 = __ldg(pb + cc);
    const bool second = cv && jb2 != ja;  // store the second system (an unpaired one is stored once)
    const double xi1 = __ldg(a.xi1 + ja), xi2 = __ldg(a.xi2 + ja);
    V* outa = out + (int64_t)par * B + ja;
    V* outb = out + (int64_t)par * B + jb2;
    V* ychkj = ychk + (int64_t)blockIdx.x * (int64_t)(((nb + 1) / 2 + R - 1) / R) * 4 * kT + tid;
    const double* ckj = a.ckpt + (int64_t)par * 10 * B + ja;
    using Full = std::integral_constant<bool, true>;
    using Part = std::integral_constant<bool, false>;
    // ---------------- forward
    BihU u{0, 0, 0, 0, 0, 0}, u1{0, 0, 0, 0, 0, 0}, u2{0, 0, 0, 0, 0, 0};
    V y1 = szero<V>(), y2 = szero<V>(), z1 = szero<V>(), z2 = szero<V>();
    auto fwd_seg = [&](int s, auto full_tag) {
      constexpr bool FULL = decltype(full_tag)::value;
      const V* cur = consume();
      BihCarry cr;
      BihProd pr;
      if (FULL) {
        bih_carry_init(stab, tpos(s * R), tstep, cr);
        bih_prod_init(xi2, cr, pr);
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = s * R + r;
        const int ic = FULL ? i : min(i, n - 1);
        double cv_[B_NCOL];
        double l2, l4;
        if (FULL) {
          load_bih_row_carry(stab, tpos(ic), cv_, cr);
          bih_row_fast_carried(u, u1, u2, cv_, xi1, xi2, pr, r == 0, l2, l4);
        } else {
          load_bih_row_compact(stab, tpos(ic), tstep, cv_);
          const BihBands hb = bih_bands_fast(xi1, xi2, cv_);
          bih_step_fast(u, u1, u2, hb, cv_, l2, l4);
        }
        u2 = u1;
        u1 = u;
        const bool valid = FULL || i < n;
        const V b0 = valid ? cur[r * 32] : szero<V>();
        const V b1 = valid ? cur[(R + r) * 32] : szero<V>();
        const V y = sfma(-l4, y2, sfma(-l2, y1, b0));
        y2 = y1;
        y1 = y;
        const V z = sfma(-l4, z2, sfma(-l2, z1, b1));
        z2 = z1;
        z1 = z;
      }
    };
    const int nfull = n / R;
    for (int s = 0; s < nseg; ++s) {
      if (s < nfull) fwd_seg(s, Full{}); else fwd_seg(s, Part{});
      if (s + 1 < nseg) {
        if (s < KTM) {
          tmem_put4(tbase + s * TCOL, y1, y2, z1, z2);
        } else {
          ystore(ychkj + (4 * s) * kT, y1);
          ystore(ychkj + (4 * s + 1) * kT, y2);
          ystore(ychkj + (4 * s + 2) * kT, z1);
          ystore(ychkj + (4 * s + 3) * kT, z2);
        }
      }
    }
    if (KTM > 0) tmem_wait_st();
    // ---------------- backward
    V x1 = szero<V>(), x2 = szero<V>(), sq = szero<V>(), sv = szero<V>();
    V w1x = szero<V>(), w2x = szero<V>(), tq = szero<V>(), tv = szero<V>();
    // checkpoints entering segment s into ckd / cky (own commit group: the
    // next consume() waits for it -- its ring group is issued after this one)
    auto ck_issue = [&](int s) {
      if (s > 0) {
        const double* cp = ckj + (int64_t)20 * s * B;
#pragma unroll
        for (int q = 0; q < 10; ++q) cpa(ckd + q * kT + tid, cp + q * B, true);
        if (s - 1 >= KTM) {
          const V* yk = ychkj + (4 * (s - 1)) * kT;
#pragma unroll
          for (int q = 0; q < 4; ++q) cpa(cky + q * kT + tid, yk + q * kT, true);
        }
      }
      cpa_commit();
    };
    auto bwd_seg = [&](int s, auto full_tag) {
      constexpr bool FULL = decltype(full_tag)::value;
      BihU w{0, 0, 0, 0, 0, 0}, w1{0, 0, 0, 0, 0, 0}, w2{0, 0, 0, 0, 0, 0};
      V ya = szero<V>(), yb = szero<V>(), za = szero<V>(), zb = szero<V>();
      V* cur = consume();  // also completes ck_issue(s) (cp.async path)
      if (s > 0) {  // factor state and y entering the segment
        const double* c = ckd + tid;
        w1.d = c[0]; w1.e = c[kT]; w1.f = c[2 * kT]; w1.a = c[3 * kT]; w1.b = c[4 * kT];
        w2.d = c[5 * kT]; w2.e = c[6 * kT]; w2.f = c[7 * kT]; w2.a = c[8 * kT]; w2.b = c[9 * kT];
        if (s - 1 < KTM) {
          tmem_get4(tbase + (s - 1) * TCOL, ya, yb, za, zb);
        } else {
          const V* yv = cky + tid;
          ya = yv[0]; yb = yv[kT]; za = yv[2 * kT]; zb = yv[3 * kT];
          V* yk = ychkj + (4 * (s - 1)) * kT;
          ydiscard(yk, lane);
          ydiscard(yk + kT, lane);
          ydiscard(yk + 2 * kT, lane);
          ydiscard(yk + 3 * kT, lane);
        }
        bih_set_rcp(w1);
        if (s * R >= 2) bih_set_rcp(w2);
        else bih_clear_rcp(w2);
      }
      ck_issue(s - 1);  // the buffer is free again: next segment's checkpoints
      BihCarry cr;
      BihProd pr;
      if (FULL) {
        bih_carry_init(stab, tpos(s * R), tstep, cr);
        bih_prod_init(xi2, cr, pr);
      }
      double e_[R], f_[R], a_[R], b_[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = s * R + r;
        const int ic = FULL ? i : min(i, n - 1);
        double cv_[B_NCOL];
        double l2, l4;
        if (FULL) {
          load_bih_row_carry(stab, tpos(ic), cv_, cr);
          bih_row_fast_carried(w, w1, w2, cv_, xi1, xi2, pr, r == 0, l2, l4);
        } else {
          load_bih_row_compact(stab, tpos(ic), tstep, cv_);
          const BihBands hb = bih_bands_fast(xi1, xi2, cv_);
          bih_step_fast(w, w1, w2, hb, cv_, l2, l4);
        }
        w2 = w1;
        w1 = w;
        const bool valid = FULL || i < n;
        const V y = sfma(-l4, yb, sfma(-l2, ya, valid ? cur[r * 32] : szero<V>()));
        yb = ya;
        ya = y;
        const V z = sfma(-l4, zb, sfma(-l2, za, valid ? cur[(R + r) * 32] : szero<V>()));
        zb = za;
        za = z;
        const double rd = valid ? w.rd : 0.0;
        cur[r * 32] = smul(rd, y);
        cur[(R + r) * 32] = smul(rd, z);
        e_[r] = rd * w.e;
        f_[r] = rd * w.f;
        a_[r] = rd * w.a;
        b_[r] = rd * w.b;
      }
      V* opa = outa + (int64_t)2 * (s * R) * B;
      V* opb = outb + (int64_t)2 * (s * R) * B;
#pragma unroll
      for (int r = R - 1; r >= 0; --r) {
        const int i = s * R + r;
        const bool valid = FULL || i < n;
        double qn, sn;
        q4s4(FULL ? i : min(i, n - 1), qn, sn);
        if (!valid) qn = sn = 0.0;
        V x = sfma(-e_[r], x1, cur[r * 32]);
        x = sfma(-f_[r], x2, x);
        x = sfma(-a_[r], sq, x);
        x = sfma(-b_[r], sv, x);
        sq = sfma(qn, x2, sq);
        sv = sfma(sn, x2, sv);
        x2 = x1;
        x1 = x;
        V xb = sfma(-e_[r], w1x, cur[(R + r) * 32]);
        xb = sfma(-f_[r], w2x, xb);
        xb = sfma(-a_[r], tq, xb);
        xb = sfma(-b_[r], tv, xb);
        tq = sfma(qn, w2x, tq);
        tv = sfma(sn, w2x, tv);
        w2x = w1x;
        w1x = xb;
        if (cv && valid) O::st_cs(opa + (int64_t)2 * r * B, x);
        if (second && valid) O::st_cs(opb + (int64_t)2 * r * B, xb);
      }
    };
    ck_issue(nseg - 1);
    for (int s = nseg - 1; s >= 0; --s) {
      if (s < nfull) bwd_seg(s, Full{}); else bwd_seg(s, Part{});
    }
  }
  cpa_wait<0>();
  if (KTM > 0) {
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    if (warp == 0) tmem_dealloc512(tmem_slot);
  }
}

// ======================================================================= launchers
static int stream_ctas(int ctas_per_sm) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms * std::max(1, ctas_per_sm);
}

template <typename K>
static int resident_ctas(K kernel, size_t smem) {
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kStreamThreads, smem) != cudaSuccess) return 1;
  return std::max(1, occ);
}

template <typename V, int R, int SG, int RING>
static cudaError_t helm_stream_RR(const HelmChunkArgs& a, void* scratch, int ctas_per_sm, cudaStream_t st) {
  constexpr int kT = 64 * SG;
  const int n0 = (a.n_dir + 1) / 2;
  const int tab_rows = ((n0 + R - 1) / R) * R;
  const size_t smem = (size_t)RING * R * kT * sizeof(V) + (size_t)2 * tab_rows * sizeof(double4);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  auto kern = helm_stream_kernel<V, R, RING, SG>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  const int occ = std::min(8, ctas_per_sm > 0 ? std::min(ctas_per_sm, resident_ctas(kern, smem)) : resident_ctas(kern, smem));
  const int64_t nsys = (a.je < 0 ? a.batch : a.je) - a.jb;
  if (nsys <= 0) return cudaSuccess;
  const int64_t groups = (nsys + 32 * SG - 1) / (32 * SG);
  int64_t cap = stream_ctas(occ);
  if (a.max_ctas > 0) cap = std::min<int64_t>(cap, a.max_ctas);
  const unsigned grid = (unsigned)std::min<int64_t>(groups, cap);
  kern<<<grid, kT, smem, st>>>(a, static_cast<V*>(scratch), tab_rows);
  return cudaGetLastError();
}

template <typename V, int R, int SG>
static cudaError_t helm_stream_R(const HelmChunkArgs& a, void* scratch, int ctas_per_sm, cudaStream_t st) {
  // deepest ring that fits next to the row table (bytes in flight per SM)
  const int n0 = (a.n_dir + 1) / 2;
  const size_t tabb = (size_t)2 * (((n0 + R - 1) / R) * R) * sizeof(double4);
  if ((size_t)3 * R * 64 * SG * sizeof(V) + tabb <= 220 * 1024)
    return helm_stream_RR<V, R, SG, 3>(a, scratch, ctas_per_sm, st);
  return helm_stream_RR<V, R, SG, 2>(a, scratch, ctas_per_sm, st);
}

template <typename V, int R, bool SMEM_TAB, int RING, int SG, bool PP = false>
static cudaError_t bih_stream_launch(const BihChunkArgs& a, void* scratch, int ctas_per_sm, size_t smem,
                                     cudaStream_t st) {
  constexpr int kT = 64 * SG;
  constexpr int SGE = PP ? 2 * SG : SG;
  auto kern = bih_stream_kernel<V, R, SMEM_TAB, RING, SG, PP>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  const int occ = std::min(8, ctas_per_sm > 0 ? std::min(ctas_per_sm, resident_ctas(kern, smem)) : resident_ctas(kern, smem));
  const int64_t nsys = (a.je < 0 ? a.batch : a.je) - a.jb;
  if (nsys <= 0) return cudaSuccess;
  const int64_t groups = (PP ? 2 : 1) * ((nsys + 32 * SGE - 1) / (32 * SGE));  // PP: one item per parity
  int64_t cap = stream_ctas(occ);
  if (a.max_ctas > 0) cap = std::min<int64_t>(cap, a.max_ctas);
  if (PP) cap = std::max<int64_t>(cap, 2);  // the CTA's parity is blockIdx.x & 1: both must exist
  const unsigned grid = (unsigned)std::min<int64_t>(groups, cap);
  kern<<<grid, kT, smem, st>>>(a, static_cast<V*>(scratch));
  return cudaGetLastError();
}

template <typename V, int R, int SG>
static size_t bih_pair_smem(const BihChunkArgs& a) {
  constexpr int kT = 64 * SG;
  const size_t ring = (size_t)2 * 2 * R * kT * sizeof(V);
  const size_t tabp = (size_t)((a.n_bih + 1) / 2 + 2) * BC_STRIDE * sizeof(double);
  const size_t ckb = (size_t)kT * (10 * sizeof(double) + 4 * sizeof(V));
  return ring + tabp + ckb + 128;  // + alignment slack of the ring
}

template <typename V, int R, int SG>
static cudaError_t bih_pair_launch(const BihChunkArgs& a, void* scratch, cudaStream_t st) {
  constexpr int kT = 64 * SG;
  size_t smem = bih_pair_smem<V, R, SG>(a);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  // the 8-warp CTA allocates all 512 TMEM columns: request enough shared
  // memory that a second CTA can never be resident on the SM (it would spin
  // in tcgen05.alloc until the first one exits)
  if (SG == 4 && SHEN_PAIR_TMEM_SEGS > 0) smem = std::max(smem, (size_t)116 * 1024);
  auto kern = bih_pair_kernel<V, R, SG>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  if (a.n_pairs <= 0) return cudaSuccess;
  const int64_t groups = 2 * ((a.n_pairs + 32 * 2 * SG - 1) / (32 * 2 * SG));  // one item per parity
  int64_t cap = stream_ctas(1);
  if (a.max_ctas > 0) cap = std::min<int64_t>(cap, a.max_ctas);
  cap = std::max<int64_t>(cap, 2);  // the CTA's parity is blockIdx.x & 1: both must exist
  const unsigned grid = (unsigned)std::min<int64_t>(groups, cap);
  kern<<<grid, kT, smem, st>>>(a, static_cast<V*>(scratch));
  return cudaGetLastError();
}

template <typename V, int R, int SG>
static cudaError_t bih_stream_R(const BihChunkArgs& a, void* scratch, int ctas_per_sm, cudaStream_t st) {
  if (a.pairs != nullptr) {
    // the pair kernel needs two RHS rings plus the one-parity table in shared
    // memory; past n_x ~ 1150 it does not fit and the one-system kernel
    // solves every system (the pair table lists each exactly once)
    if (bih_pair_smem<V, R, 4>(a) <= 227 * 1024) return bih_pair_launch<V, R, 4>(a, scratch, st);
    // larger n_x (the one-parity table alone is ~115 KB at n_x = 2048): a
    // 4-warp pair CTA still fits (SHEN_PAIR_SMALL=0 falls through to the
    // one-system kernel)
    static const int small = getenv("SHEN_PAIR_SMALL") ? atoi(getenv("SHEN_PAIR_SMALL")) : 1;
    if (small && bih_pair_smem<V, R, 2>(a) <= 227 * 1024) return bih_pair_launch<V, R, 2>(a, scratch, st);
  }
  // the table in shared memory beats a deeper ring: the biharmonic rows are
  // slow enough that one segment of prefetch covers HBM latency
  // (a 3-deep ring measured slower at config 4: 29.5 vs 28.6 ms)
#ifndef SHEN_BIH_RING
#define SHEN_BIH_RING 2
#endif
  const size_t ring2 = (size_t)2 * R * 64 * SG * sizeof(V);
  const size_t ringb = (size_t)SHEN_BIH_RING * R * 64 * SG * sizeof(V);
  const size_t tabb = (size_t)(a.n_bih + 4) * BC_STRIDE * sizeof(double);
  static const bool force_pp = getenv("SHEN_BIH_PP") != nullptr && atoi(getenv("SHEN_BIH_PP")) != 0;
  if (!force_pp && ringb + tabb <= 220 * 1024)
    return bih_stream_launch<V, R, true, SHEN_BIH_RING, SG>(a, scratch, ctas_per_sm, ringb + tabb, st);
  const size_t tabp = (size_t)((a.n_bih + 1) / 2 + 2) * BC_STRIDE * sizeof(double);  // one parity
  if (ring2 + tabp <= 220 * 1024)
    return bih_stream_launch<V, R, true, 2, SG, true>(a, scratch, ctas_per_sm, ring2 + tabp, st);
  return bih_stream_launch<V, R, false, kRing, 4>(a, scratch, ctas_per_sm, (size_t)kRing * R * 256 * sizeof(V), st);
}

// CTA size (one persistent CTA per SM either way -- registers and shared
// memory): warps_per_sm 8 -> 4 system groups (8 warps), 12 -> 6 (12 warps),
// 0 -> the measured best at BASELINE config 4: 12 warps for Helmholtz
// (18.2 vs 19.8 ms), 8 for the biharmonic (28.6 vs 30.2 ms; its 8-warp CTA
// can afford to prefetch the segment checkpoints into registers).
template <typename V>
static cudaError_t helm_stream_dispatch(const HelmChunkArgs& a, void* sc, int w, cudaStream_t st) {
  if (a.chunk_rows != 8) return cudaErrorInvalidValue;  // the checkpoint spacing the kernels are built for
  return w == 8 ? helm_stream_R<V, 8, 4>(a, sc, 1, st) : helm_stream_R<V, 8, 6>(a, sc, 1, st);
}

template <typename V>
static cudaError_t bih_stream_dispatch(const BihChunkArgs& a, void* sc, int w, cudaStream_t st) {
  if (a.chunk_rows != 8) return cudaErrorInvalidValue;
  return w != 12 ? bih_stream_R<V, 8, 4>(a, sc, 1, st) : bih_stream_R<V, 8, 6>(a, sc, 1, st);
}

// per-CTA y-checkpoint scratch: grid is at most (#SMs x 8) CTAs
int64_t stream_scratch_bytes(int op, int n_modes, int chunk_rows, bool cplx_rhs) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    sms = 160;
  }
  const int64_t nseg0 = (((int64_t)n_modes + 1) / 2 + chunk_rows - 1) / chunk_rows;
  return (int64_t)sms * 8 * nseg0 * (op == 0 ? 1 : 2) * kStreamThreads * (cplx_rhs ? 16 : 8);
}

// warps_per_sm of the C ABI: 8 / 12 select the CTA size, 0 the per-operator default
cudaError_t launch_helm_stream(const HelmChunkArgs& a, void* scratch, bool cplx_rhs, int warps_per_sm,
                               cudaStream_t st) {
  if (a.batch <= 0) return cudaSuccess;
  // the bulk-copy ring moves 16-B aligned row pieces: real RHS needs an even batch
  if (!cplx_rhs && ((a.batch & 1) || (reinterpret_cast<uintptr_t>(a.rhs) & 15))) return cudaErrorInvalidValue;
  return cplx_rhs ? helm_stream_dispatch<cplx>(a, scratch, warps_per_sm, st)
                  : helm_stream_dispatch<double>(a, scratch, warps_per_sm, st);
}

cudaError_t launch_bih_stream(const BihChunkArgs& a, void* scratch, bool cplx_rhs, int warps_per_sm, cudaStream_t st) {
  if (a.batch <= 0) return cudaSuccess;
  if (!cplx_rhs && ((a.batch & 1) || (reinterpret_cast<uintptr_t>(a.rhs) & 15))) return cudaErrorInvalidValue;
  return cplx_rhs ? bih_stream_dispatch<cplx>(a, scratch, warps_per_sm, st)
                  : bih_stream_dispatch<double>(a, scratch, warps_per_sm, st);
}

}  // namespace shen
