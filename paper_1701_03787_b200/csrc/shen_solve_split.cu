// Chunk-split streaming Helmholtz solve: the RHS is read from HBM once (the
// second read comes from L2), the solution written once.
//
// The streaming solve (shen_solve_stream.cu) runs one thread per (system,
// parity) down and back up the whole column, so the data a thread re-reads
// in its backward sweep was fetched a full column earlier: at the 12 warps
// per SM the recurrences need, ~3 MB per SM is in flight and the re-read
// comes from HBM (51.8 B per unknown).  Here a CTA takes a group of 16
// consecutive systems and splits each (system, parity) column into 16
// chunks of K segments (8 rows each), one thread per chunk:
//
//   pass 1  chunk rows top-down from HBM: the factor recurrence from the
//           build's checkpoint at the chunk start (the fast arithmetic of
//           shen_rows.cuh, restarted at every segment exactly as the build
//           and the streaming solve do), y with zero entry (yh) and its
//           homogeneous response h, and the chunk's backward transfer map
//           sigma_top = P sigma_in + tau, sigma = (x_i, sum_{k > i} x_k),
//           accumulated in forward order (tau split into its yh and h parts);
//   scan    one thread per (system, parity) chains the 16 chunks: y entering
//           every chunk (forward), then the back-substitution state entering
//           every chunk from below (backward);
//   pass 2  chunk segments bottom-up, re-read from L2 (the group's 256 KB is
//           the whole working set of the SM): factors from the segment's
//           checkpoint, y = yh + h E recomputed, then the reference
//           back-substitution (solvers.py:118-125) writes x.
//
// tools/l2_reread.cu measured this access pattern: at 16 systems x 2
// parities x 16 chunks per SM the re-read hits L2 (DRAM reads 1.04x the
// RHS), at 32 systems 1.39x.  Complex RHS only; requires at most 4
// segments per chunk (n_x <= 1024) -- shen_helm_solve_split rejects other
// shapes and the Python layer falls back to the streaming solve.
// Replaces HelmholtzLU.solve (reference solvers.py:100-126).
#include <algorithm>

#include "shen_kernels.h"
#include "shen_rows.cuh"

namespace shen {
namespace {

constexpr int kR = 8;             // rows per segment (= build checkpoint spacing)
constexpr int kS = 16;            // systems per group
constexpr int kCH = 16;           // chunks per (system, parity)
constexpr int kT = kS * 2 * kCH;  // 512 threads
constexpr int kRing = 2;          // segment slots per thread
constexpr int kKM = 4;            // max segments per chunk
constexpr int kX = 13;            // exchange doubles per thread

__device__ __forceinline__ void cpa16(cplx* dst, const cplx* src, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  const int n = pred ? 16 : 0;  // src-size 0 -> zero fill, no global access
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cpa_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void cpa_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void st_cs(cplx* p, cplx v) {
  __stcs(reinterpret_cast<double2*>(p), make_double2(v.re, v.im));
}
__device__ __forceinline__ cplx cfma(double s, cplx b, cplx a) { return {__fma_rn(s, b.re, a.re), __fma_rn(s, b.im, a.im)}; }
__device__ __forceinline__ cplx cmul(double s, cplx b) { return {s * b.re, s * b.im}; }
__device__ __forceinline__ cplx cadd(cplx a, cplx b) { return {a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ cplx csub(cplx a, cplx b) { return {a.re - b.re, a.im - b.im}; }

// thread of (system s, parity p, chunk c): warp = 2 (c / 2) + p, lane = 16 (c % 2) + s
__device__ __forceinline__ int tid_of(int s, int p, int c) { return (2 * (c >> 1) + p) * 32 + 16 * (c & 1) + s; }

}  // namespace

__global__ void __launch_bounds__(kT, 1) helm_split_kernel(HelmChunkArgs a, int K, int tab_rows) {
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int s = lane & 15, par = warp & 1, c = 2 * (warp >> 1) + (lane >> 4);
  const int64_t B = a.batch;
  const int n = (a.n_dir - par + 1) / 2;
  const int nseg = (n + kR - 1) / kR;
  const int seg0 = c * K;
  const int nmine = max(0, min(nseg, seg0 + K) - seg0);
  cplx* ring = reinterpret_cast<cplx*>(smem);  // [slot][row][kT]
  double* X = smem + (size_t)kRing * kR * kT * 2;
  double4* tab = reinterpret_cast<double4*>(X + (size_t)kX * kT);
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
  const cplx* rhs = static_cast<const cplx*>(a.rhs);
  cplx* out = static_cast<cplx*>(a.out);
  const int64_t jb = a.jb, je = a.je < 0 ? B : a.je;
  const int64_t ngroups = (je - jb + kS - 1) / kS;
  const int64_t g0 = blockIdx.x, gstride = gridDim.x;
  if (g0 >= ngroups) return;

  // per-thread segment stream: per group pass 1 (seg0 .. seg0+nmine-1) then
  // pass 2 (the same segments bottom-up), continuous across groups
  int64_t ig = g0;
  int iq = 0;  // position within the group's 2 nmine segments
  int islot = 0, cslot = 0;
  auto issue = [&]() {
    if (nmine > 0 && ig < ngroups) {
      const int seg = iq < nmine ? seg0 + iq : seg0 + (2 * nmine - 1 - iq);
      const int64_t j = jb + ig * kS + s;
      const bool jv = j < je;
      const int64_t jc = jv ? j : je - 1;
      const int rows = min(kR, n - seg * kR);
      const cplx* p = rhs + (int64_t)(par + 2 * seg * kR) * B + jc;
      cplx* dst = ring + (size_t)islot * kR * kT + tid;
#pragma unroll
      for (int r = 0; r < kR; ++r) {
        cpa16(dst + r * kT, p, jv && r < rows);
        if (r + 1 < rows) p += 2 * B;
      }
      if (++iq == 2 * nmine) {
        iq = 0;
        ig += gstride;
      }
    }
    cpa_commit();
    islot ^= 1;
  };
  auto consume = [&]() -> const cplx* {
    issue();
    cpa_wait1();
    const cplx* p = ring + (size_t)cslot * kR * kT + tid;
    cslot ^= 1;
    return p;
  };
  issue();  // prefetch distance: one segment

  for (int64_t g = g0; g < ngroups; g += gstride) {
    const int64_t j = jb + g * kS + s;
    const bool jv = j < je;
    const int64_t jc = jv ? j : je - 1;
    const double cb = __ldg(a.cb + jc);
    const double sub = __dmul_rn(cb, -1.5707963267948966);
    const double* ckj = a.ckpt + (int64_t)par * 3 * B + jc;  // segment sg: + 6 sg B
    // ---------------- pass 1
    cplx yh = {0.0, 0.0};
    double hh = 1.0;
    double p00 = 1.0, p01 = 0.0, p10 = 0.0, p11 = 1.0;
    cplx ta = {0.0, 0.0}, tb = {0.0, 0.0};
    double ha = 0.0, hb = 0.0;
    cplx yck[kKM];
    double hck[kKM];
    if (nmine > 0) {
      HelmProj pj;
      double dl = 0.0, el = 0.0, tl = 0.0;
      if (seg0 == 0) {
        hp_origin(pj);
      } else {
        const double* ck = ckj + (int64_t)6 * seg0 * B;
        hp_start(pj, __ldg(ck), __ldg(ck + B), __ldg(ck + 2 * B));
      }
#pragma unroll
      for (int k = 0; k < kKM; ++k) {
        if (k < nmine) {
          yck[k] = yh;
          hck[k] = hh;
          const cplx* cur = consume();
          if (k > 0) hp_start(pj, dl, el, tl);
          const int sg = seg0 + k;
#pragma unroll
          for (int r = 0; r < kR; ++r) {
            const int i = sg * kR + r;
            const bool valid = i < n;
            const double4 tv = mytab[i];
            const HelmRow row = helm_row(a.ca, cb, sub, tv.x, tv.y, tv.z, tv.w != 0.0);
            double d, e, t;
            const double low = hp_step(pj, row, sub, d, e, t);
            dl = d; el = e; tl = t;
            if (valid) {
              const cplx b = cur[r * kT];
              yh = cfma(-low, yh, b);
              hh = -low * hh;
              const double rd = pj.rd, al = -rd * e, be = -rd * t;
              const cplx cy = cmul(rd, yh);
              const double ch = rd * hh;
              ta = cfma(p00, cy, ta);
              tb = cfma(p10, cy, tb);
              ha = fma(p00, ch, ha);
              hb = fma(p10, ch, hb);
              const double n00 = fma(p00, al, p01), n01 = fma(p00, be, p01);
              const double n10 = fma(p10, al, p11), n11 = fma(p10, be, p11);
              p00 = n00; p01 = n01; p10 = n10; p11 = n11;
            }
          }
        }
      }
    }
    X[0 * kT + tid] = hh;
    X[1 * kT + tid] = yh.re;
    X[2 * kT + tid] = yh.im;
    X[3 * kT + tid] = p00;
    X[4 * kT + tid] = p01;
    X[5 * kT + tid] = p10;
    X[6 * kT + tid] = p11;
    X[7 * kT + tid] = ta.re;
    X[8 * kT + tid] = ta.im;
    X[9 * kT + tid] = tb.re;
    X[10 * kT + tid] = tb.im;
    X[11 * kT + tid] = ha;
    X[12 * kT + tid] = hb;
    __syncthreads();
    // ---------------- scan: one thread per (system, parity)
    if (tid < 2 * kS) {
      const int s2 = tid & (kS - 1), p2 = tid >> 4;
      cplx E = {0.0, 0.0};  // y entering chunk 0 (never used: h = 0 from row 0 on)
      for (int cc = 0; cc < kCH; ++cc) {
        const int t = tid_of(s2, p2, cc);
        const double hc = X[0 * kT + t];
        const cplx yc = {X[1 * kT + t], X[2 * kT + t]};
        X[0 * kT + t] = E.re;
        X[1 * kT + t] = E.im;
        E = cfma(hc, E, yc);
      }
      cplx x1 = {0.0, 0.0}, S = {0.0, 0.0};  // state entering the last chunk from below
      for (int cc = kCH - 1; cc >= 0; --cc) {
        const int t = tid_of(s2, p2, cc);
        const cplx Ec = {X[0 * kT + t], X[1 * kT + t]};
        const double q00 = X[3 * kT + t], q01 = X[4 * kT + t], q10 = X[5 * kT + t], q11 = X[6 * kT + t];
        const cplx qa = {X[7 * kT + t], X[8 * kT + t]}, qb = {X[9 * kT + t], X[10 * kT + t]};
        const double qha = X[11 * kT + t], qhb = X[12 * kT + t];
        X[2 * kT + t] = x1.re;
        X[3 * kT + t] = x1.im;
        X[4 * kT + t] = S.re;
        X[5 * kT + t] = S.im;
        // sigma_top = P sigma_in + tau_yh + tau_h E
        const cplx nx = cfma(q00, x1, cfma(q01, S, cfma(qha, Ec, qa)));
        const cplx nS = cfma(q10, x1, cfma(q11, S, cfma(qhb, Ec, qb)));
        x1 = nx;
        S = nS;
      }
    }
    __syncthreads();
    const cplx E = {X[0 * kT + tid], X[1 * kT + tid]};
    cplx x1 = {X[2 * kT + tid], X[3 * kT + tid]}, S = {X[4 * kT + tid], X[5 * kT + tid]};
    __syncthreads();  // every thread has its entry state before the next group's pass 1 writes X
    // ---------------- pass 2: segments bottom-up
    cplx* outj = out + (int64_t)par * B + j;
    // the segment's factor checkpoint, loaded one segment ahead
    double ckd = 1.0, cke = 0.0, ckt = 0.0;
    if (nmine > 0 && seg0 + nmine - 1 > 0) {
      const double* ck = ckj + (int64_t)6 * (seg0 + nmine - 1) * B;
      ckd = __ldg(ck); cke = __ldg(ck + B); ckt = __ldg(ck + 2 * B);
    }
#pragma unroll
    for (int k = kKM - 1; k >= 0; --k) {
      if (k < nmine) {
        const int sg = seg0 + k;
        HelmProj q;
        if (sg == 0) hp_origin(q);
        else hp_start(q, ckd, cke, ckt);
        if (k > 0 && sg - 1 > 0) {
          const double* ck = ckj + (int64_t)6 * (sg - 1) * B;
          ckd = __ldg(ck); cke = __ldg(ck + B); ckt = __ldg(ck + 2 * B);
        }
        cplx y2 = yck[k];
        double h2 = hck[k];
        const cplx* cur = consume();
        double rd_[kR], e_[kR], t_[kR];
        cplx y_[kR];
#pragma unroll
        for (int r = 0; r < kR; ++r) {
          const int i = sg * kR + r;
          const bool valid = i < n;
          const double4 tv = mytab[i];
          const HelmRow row = helm_row(a.ca, cb, sub, tv.x, tv.y, tv.z, tv.w != 0.0);
          double d, e, t;
          const double low = hp_step(q, row, sub, d, e, t);
          const cplx b = valid ? cur[r * kT] : cplx{0.0, 0.0};
          y2 = cfma(-low, y2, b);
          h2 = -low * h2;
          y_[r] = valid ? cfma(h2, E, y2) : cplx{0.0, 0.0};
          rd_[r] = valid ? q.rd : 0.0;
          e_[r] = valid ? e : 0.0;
          t_[r] = valid ? t : 0.0;
        }
#pragma unroll
        for (int r = kR - 1; r >= 0; --r) {
          const cplx acc = csub(csub(y_[r], cmul(e_[r], x1)), cmul(t_[r], S));
          const cplx x = cmul(rd_[r], acc);
          S = cadd(x1, S);
          x1 = x;
          if (jv && sg * kR + r < n) st_cs(outj + (int64_t)2 * (sg * kR + r) * B, x);
        }
      }
    }
  }
  cpa_wait0();
}

size_t helm_split_smem(int n_dir) {
  const int n0 = (n_dir + 1) / 2;
  const int tab_rows = ((n0 + kR - 1) / kR) * kR;
  return (size_t)kRing * kR * kT * sizeof(cplx) + (size_t)kX * kT * sizeof(double) + (size_t)2 * tab_rows * sizeof(double4);
}

// complex RHS, checkpoints every 8 rows (shen_helm_factor chunk_rows = 8);
// returns cudaErrorNotSupported for shapes the kernel does not take
cudaError_t launch_helm_split(const HelmChunkArgs& a, cudaStream_t st) {
  if (a.batch <= 0) return cudaSuccess;
  if (a.chunk_rows != kR) return cudaErrorNotSupported;
  const int n0 = (a.n_dir + 1) / 2;
  const int nseg0 = (n0 + kR - 1) / kR;
  const int K = (nseg0 + kCH - 1) / kCH;
  if (K > kKM || nseg0 < 2) return cudaErrorNotSupported;
  if ((reinterpret_cast<uintptr_t>(a.rhs) | reinterpret_cast<uintptr_t>(a.out)) & 15) return cudaErrorInvalidValue;
  const size_t smem = helm_split_smem(a.n_dir);
  if (smem > 227 * 1024) return cudaErrorNotSupported;
  cudaError_t err = cudaFuncSetAttribute(helm_split_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  const int64_t je = a.je < 0 ? a.batch : a.je;
  if (je <= a.jb) return cudaSuccess;
  const int64_t groups = (je - a.jb + kS - 1) / kS;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t grid = std::min<int64_t>(groups, sms);
  if (a.max_ctas > 0) grid = std::min<int64_t>(grid, a.max_ctas);
  helm_split_kernel<<<(unsigned)grid, kT, smem, st>>>(a, K, ((n0 + kR - 1) / kR) * kR);
  return cudaGetLastError();
}

}  // namespace shen
