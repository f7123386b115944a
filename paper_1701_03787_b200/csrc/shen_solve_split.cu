// Chunk-split Helmholtz solve on mirror pairs: the RHS is read from HBM
// once (the backward sweep re-reads it from L2), the solution written once,
// and the factor recurrence runs once for the two systems (m, n), (-m, n) of
// a mirror pair (bitwise-identical z2, hence identical factors).
//
// A CTA takes one parity of a group of 16 pairs (16 consecutive kz columns of
// one (m, -m) row pair: 256-B row pieces per system) and splits the parity
// column into 16 chunks of up to 4 segments (8 rows each); thread = (pair,
// chunk), 256 threads:
//
//   pass 1  chunk rows top-down from HBM: the factor recurrence from the
//           build's checkpoint at the chunk start (the fast arithmetic of
//           shen_rows.cuh, restarted at every segment like the build and the
//           streaming solve), per system y with zero entry (yh), the shared
//           homogeneous response h, and the chunk's backward transfer map
//           sigma_top = P sigma_in + tau (sigma = (x_i, sum_{k > i} x_k)),
//           accumulated in forward order -- P and the h part of tau are
//           shared by the pair, the yh part is per system;
//   scan    one thread per (pair, system) chains the 16 chunks: y entering
//           every chunk, then the back-substitution state entering every
//           chunk from below;
//   pass 2  chunk segments bottom-up, re-read from L2 (the group's 256 KB is
//           the SM's working set): factors from the segment's checkpoint,
//           y = yh + h E, the reference back-substitution
//           (solvers.py:118-125) per system.
//
// The per-system operations are those of an unpaired chunk split; results
// agree with the streaming kernel to rounding (the chunk joins reassociate
// the recurrences).  Complex RHS, 8-row checkpoints, at most 4 segments per
// chunk (n_x <= 1024); other shapes are rejected (the caller falls back to
// the streaming kernel).  Replaces HelmholtzLU.solve (solvers.py:100-126).
#include <algorithm>

#include "shen_kernels.h"
#include "shen_rows.cuh"

namespace shen {
namespace {

constexpr int kR = 8;             // rows per segment (= build checkpoint spacing)
constexpr int kP = 16;            // pairs per group
constexpr int kCH = 16;           // chunks per parity column
constexpr int kT = kP * kCH;      // 256 threads
constexpr int kRing = 2;          // segment slots per thread (each: 2 systems x kR rows)
constexpr int kKM = 4;            // max segments per chunk
constexpr int kXs = 7;            // shared exchange doubles: h, P (4), h-part of tau (2)
constexpr int kXy = 6;            // per-system exchange doubles: yh (2), yh-part of tau (2 complex)

__device__ __forceinline__ void cpa16(cplx* dst, const cplx* src, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  const int n = pred ? 16 : 0;  // src-size 0 -> zero fill, no global access
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cpa_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void cpa_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void st_cs(cplx* p, cplx v) { __stcs(reinterpret_cast<double2*>(p), make_double2(v.re, v.im)); }
__device__ __forceinline__ cplx cfma(double s, cplx b, cplx a) { return {__fma_rn(s, b.re, a.re), __fma_rn(s, b.im, a.im)}; }
__device__ __forceinline__ cplx cmul(double s, cplx b) { return {s * b.re, s * b.im}; }
__device__ __forceinline__ cplx cadd(cplx a, cplx b) { return {a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ cplx csub(cplx a, cplx b) { return {a.re - b.re, a.im - b.im}; }

// thread of (pair s, chunk c): warp = c / 2, lane = 16 (c % 2) + s
__device__ __forceinline__ int tid_of(int s, int c) { return (c >> 1) * 32 + 16 * (c & 1) + s; }

}  // namespace

__global__ void __launch_bounds__(kT, 1) helm_split_pair_kernel(HelmChunkArgs a, int tab_rows) {
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int s = lane & 15, c = 2 * warp + (lane >> 4);
  const int64_t B = a.batch, P = a.n_pairs;
  const int64_t* pa = a.pairs;
  const int64_t* pb = a.pairs + P;
  cplx* ring = reinterpret_cast<cplx*>(smem);                      // [slot][sys][row][kT]
  double* XS = smem + (size_t)kRing * 2 * kR * kT * 2;              // [kXs][kT]
  double* XY = XS + (size_t)kXs * kT;                               // [2 sys][kXy][kT]
  double4* tab = reinterpret_cast<double4*>(XY + (size_t)2 * kXy * kT);  // [2][tab_rows]
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
  const int64_t ngroups = (P + kP - 1) / kP;
  const int64_t nitems = 2 * ngroups;  // (group, parity)
  const int64_t it0 = blockIdx.x, istride = gridDim.x;
  if (it0 >= nitems) return;
  const int nseg0 = ((a.n_dir + 1) / 2 + kR - 1) / kR;
  const int K = (nseg0 + kCH - 1) / kCH;

  // per-thread segment stream over the CTA's items: pass 1 (chunk segments
  // top-down), pass 2 (bottom-up), both systems of the pair per slot
  int64_t qi = it0;
  int iq = 0, islot = 0, cslot = 0;
  int64_t q_ig = -1, q_ja = 0, q_jb = 0;
  auto issue = [&]() {
    bool done = true;
    while (qi < nitems) {
      const int par = (int)(qi & 1);
      const int n = (a.n_dir - par + 1) / 2, nseg = (n + kR - 1) / kR;
      const int seg0 = c * K, nmine = max(0, min(nseg, seg0 + K) - seg0);
      if (nmine == 0) {  // this thread has no segments in this item
        qi += istride;
        iq = 0;
        continue;
      }
      const int64_t g = qi >> 1;
      const int64_t item = g * kP + s;
      const bool iv = item < P;
      if (g != q_ig) {
        const int64_t ic = iv ? item : P - 1;
        q_ja = __ldg(pa + ic);
        q_jb = __ldg(pb + ic);
        q_ig = g;
      }
      const int seg = iq < nmine ? seg0 + iq : seg0 + (2 * nmine - 1 - iq);
      const int rows = min(kR, n - seg * kR);
      const cplx* r0 = static_cast<const cplx*>(a.rhs) + (int64_t)(par + 2 * seg * kR) * B;
      const cplx* p0 = r0 + q_ja;
      const cplx* p1 = r0 + q_jb;
      cplx* dst = ring + (size_t)islot * 2 * kR * kT + tid;
#pragma unroll
      for (int r = 0; r < kR; ++r) {
        const bool ok = iv && r < rows;
        cpa16(dst + r * kT, p0, ok);
        cpa16(dst + (kR + r) * kT, p1, ok);
        if (r + 1 < rows) {
          p0 += 2 * B;
          p1 += 2 * B;
        }
      }
      if (++iq == 2 * nmine) {
        iq = 0;
        qi += istride;
      }
      done = false;
      break;
    }
    (void)done;
    cpa_commit();
    islot ^= 1;
  };
  auto consume = [&]() -> const cplx* {
    issue();
    cpa_wait1();
    const cplx* p = ring + (size_t)cslot * 2 * kR * kT + tid;
    cslot ^= 1;
    return p;
  };
  issue();  // prefetch distance: one segment

  for (int64_t itm = it0; itm < nitems; itm += istride) {
    const int par = (int)(itm & 1);
    const int64_t g = itm >> 1;
    const int n = (a.n_dir - par + 1) / 2;
    const int nseg = (n + kR - 1) / kR;
    const int seg0 = c * K;
    const int nmine = max(0, min(nseg, seg0 + K) - seg0);
    const int64_t item = g * kP + s;
    const bool iv = item < P;
    const int64_t ic = iv ? item : P - 1;
    const int64_t ja = __ldg(pa + ic), jb2 = __ldg(pb + ic);
    const bool second = iv && jb2 != ja;
    const double cb = __ldg(a.cb + ja);
    const double sub = __dmul_rn(cb, -1.5707963267948966);
    const double* ckj = a.ckpt + (int64_t)par * 3 * B + ja;  // segment sg: + 6 sg B
    const double4* mytab = tab + par * tab_rows;
    // ---------------- pass 1
    cplx yh0 = {0.0, 0.0}, yh1 = {0.0, 0.0};
    double hh = 1.0;
    double p00 = 1.0, p01 = 0.0, p10 = 0.0, p11 = 1.0;
    cplx ta0 = {0.0, 0.0}, tb0 = {0.0, 0.0}, ta1 = {0.0, 0.0}, tb1 = {0.0, 0.0};
    double ha = 0.0, hb = 0.0;
    cplx yck0[kKM], yck1[kKM];
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
          yck0[k] = yh0;
          yck1[k] = yh1;
          hck[k] = hh;
          const cplx* cur = consume();
          if (k > 0) hp_start(pj, dl, el, tl);
          const int sg = seg0 + k;
#pragma unroll
          for (int r = 0; r < kR; ++r) {
            const int i = sg * kR + r;
            const double4 tv = mytab[i];
            const HelmRow row = helm_row(a.ca, cb, sub, tv.x, tv.y, tv.z, tv.w != 0.0);
            double d, e, t;
            const double low = hp_step(pj, row, sub, d, e, t);
            dl = d; el = e; tl = t;
            if (i < n) {
              yh0 = cfma(-low, yh0, cur[r * kT]);
              yh1 = cfma(-low, yh1, cur[(kR + r) * kT]);
              hh = -low * hh;
              const double rd = pj.rd, al = -rd * e, be = -rd * t;
              const cplx cy0 = cmul(rd, yh0), cy1 = cmul(rd, yh1);
              const double ch = rd * hh;
              ta0 = cfma(p00, cy0, ta0);
              tb0 = cfma(p10, cy0, tb0);
              ta1 = cfma(p00, cy1, ta1);
              tb1 = cfma(p10, cy1, tb1);
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
    XS[0 * kT + tid] = hh;
    XS[1 * kT + tid] = p00;
    XS[2 * kT + tid] = p01;
    XS[3 * kT + tid] = p10;
    XS[4 * kT + tid] = p11;
    XS[5 * kT + tid] = ha;
    XS[6 * kT + tid] = hb;
    double* Y0 = XY;
    double* Y1 = XY + (size_t)kXy * kT;
    Y0[0 * kT + tid] = yh0.re; Y0[1 * kT + tid] = yh0.im;
    Y0[2 * kT + tid] = ta0.re; Y0[3 * kT + tid] = ta0.im; Y0[4 * kT + tid] = tb0.re; Y0[5 * kT + tid] = tb0.im;
    Y1[0 * kT + tid] = yh1.re; Y1[1 * kT + tid] = yh1.im;
    Y1[2 * kT + tid] = ta1.re; Y1[3 * kT + tid] = ta1.im; Y1[4 * kT + tid] = tb1.re; Y1[5 * kT + tid] = tb1.im;
    __syncthreads();
    // ---------------- scan: one thread per (pair, system)
    if (tid < 2 * kP) {
      const int s2 = tid & (kP - 1), sys = tid >> 4;
      double* Y = sys ? Y1 : Y0;
      cplx E = {0.0, 0.0};  // y entering chunk 0 (never used: h = 0 from row 0 on)
      for (int cc = 0; cc < kCH; ++cc) {
        const int t = tid_of(s2, cc);
        const double hc = XS[0 * kT + t];
        const cplx yc = {Y[0 * kT + t], Y[1 * kT + t]};
        Y[0 * kT + t] = E.re;  // E of chunk cc replaces its yh
        Y[1 * kT + t] = E.im;
        E = cfma(hc, E, yc);
      }
      cplx x1 = {0.0, 0.0}, S = {0.0, 0.0};  // state entering the last chunk from below
      for (int cc = kCH - 1; cc >= 0; --cc) {
        const int t = tid_of(s2, cc);
        const cplx Ec = {Y[0 * kT + t], Y[1 * kT + t]};
        const double q00 = XS[1 * kT + t], q01 = XS[2 * kT + t], q10 = XS[3 * kT + t], q11 = XS[4 * kT + t];
        const double qha = XS[5 * kT + t], qhb = XS[6 * kT + t];
        const cplx qa = {Y[2 * kT + t], Y[3 * kT + t]}, qb = {Y[4 * kT + t], Y[5 * kT + t]};
        Y[2 * kT + t] = x1.re;  // state entering chunk cc replaces its tau
        Y[3 * kT + t] = x1.im;
        Y[4 * kT + t] = S.re;
        Y[5 * kT + t] = S.im;
        // sigma_top = P sigma_in + tau_yh + tau_h E
        const cplx nx = cfma(q00, x1, cfma(q01, S, cfma(qha, Ec, qa)));
        const cplx nS = cfma(q10, x1, cfma(q11, S, cfma(qhb, Ec, qb)));
        x1 = nx;
        S = nS;
      }
    }
    __syncthreads();
    const cplx E0 = {Y0[0 * kT + tid], Y0[1 * kT + tid]}, E1 = {Y1[0 * kT + tid], Y1[1 * kT + tid]};
    cplx xa = {Y0[2 * kT + tid], Y0[3 * kT + tid]}, Sa = {Y0[4 * kT + tid], Y0[5 * kT + tid]};
    cplx xb = {Y1[2 * kT + tid], Y1[3 * kT + tid]}, Sb = {Y1[4 * kT + tid], Y1[5 * kT + tid]};
    __syncthreads();  // every thread has its entry state before the next item's pass 1 writes the exchange
    // ---------------- pass 2: segments bottom-up
    cplx* outa = static_cast<cplx*>(a.out) + (int64_t)par * B + ja;
    cplx* outb = static_cast<cplx*>(a.out) + (int64_t)par * B + jb2;
    double ckd = 1.0, cke = 0.0, ckt = 0.0;  // the segment's factor checkpoint, one segment ahead
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
        cplx ya = yck0[k], yb = yck1[k];
        double h2 = hck[k];
        const cplx* cur = consume();
        double rd_[kR], e_[kR], t_[kR];
        cplx ya_[kR], yb_[kR];
#pragma unroll
        for (int r = 0; r < kR; ++r) {
          const int i = sg * kR + r;
          const bool valid = i < n;
          const double4 tv = mytab[i];
          const HelmRow row = helm_row(a.ca, cb, sub, tv.x, tv.y, tv.z, tv.w != 0.0);
          double d, e, t;
          const double low = hp_step(q, row, sub, d, e, t);
          ya = cfma(-low, ya, valid ? cur[r * kT] : cplx{0.0, 0.0});
          yb = cfma(-low, yb, valid ? cur[(kR + r) * kT] : cplx{0.0, 0.0});
          h2 = -low * h2;
          ya_[r] = valid ? cfma(h2, E0, ya) : cplx{0.0, 0.0};
          yb_[r] = valid ? cfma(h2, E1, yb) : cplx{0.0, 0.0};
          rd_[r] = valid ? q.rd : 0.0;
          e_[r] = valid ? e : 0.0;
          t_[r] = valid ? t : 0.0;
        }
#pragma unroll
        for (int r = kR - 1; r >= 0; --r) {
          const int i = sg * kR + r;
          const cplx acca = csub(csub(ya_[r], cmul(e_[r], xa)), cmul(t_[r], Sa));
          const cplx accb = csub(csub(yb_[r], cmul(e_[r], xb)), cmul(t_[r], Sb));
          const cplx xna = cmul(rd_[r], acca), xnb = cmul(rd_[r], accb);
          Sa = cadd(xa, Sa);
          xa = xna;
          Sb = cadd(xb, Sb);
          xb = xnb;
          if (iv && i < n) st_cs(outa + (int64_t)2 * i * B, xna);
          if (second && i < n) st_cs(outb + (int64_t)2 * i * B, xnb);
        }
      }
    }
  }
  cpa_wait0();
}

size_t helm_split_pair_smem(int n_dir) {
  const int n0 = (n_dir + 1) / 2;
  const int tab_rows = ((n0 + kR - 1) / kR) * kR;
  return (size_t)kRing * 2 * kR * kT * sizeof(cplx) + (size_t)(kXs + 2 * kXy) * kT * sizeof(double) +
         (size_t)2 * tab_rows * sizeof(double4);
}

// complex RHS, checkpoints every 8 rows, mirror pairs in a.pairs / a.n_pairs;
// cudaErrorNotSupported for shapes the kernel does not take
cudaError_t launch_helm_split_pairs(const HelmChunkArgs& a, cudaStream_t st) {
  if (a.batch <= 0 || a.n_pairs <= 0) return cudaSuccess;
  if (a.chunk_rows != kR || a.pairs == nullptr) return cudaErrorNotSupported;
  const int n0 = (a.n_dir + 1) / 2;
  const int nseg0 = (n0 + kR - 1) / kR;
  const int K = (nseg0 + kCH - 1) / kCH;
  if (K > kKM || nseg0 < 2) return cudaErrorNotSupported;
  if ((reinterpret_cast<uintptr_t>(a.rhs) | reinterpret_cast<uintptr_t>(a.out)) & 15) return cudaErrorInvalidValue;
  const size_t smem = helm_split_pair_smem(a.n_dir);
  if (smem > 227 * 1024) return cudaErrorNotSupported;
  cudaError_t err = cudaFuncSetAttribute(helm_split_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  const int64_t items = 2 * ((a.n_pairs + kP - 1) / kP);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t grid = std::min<int64_t>(items, sms);
  if (a.max_ctas > 0) grid = std::min<int64_t>(grid, a.max_ctas);
  helm_split_pair_kernel<<<(unsigned)grid, kT, smem, st>>>(a, ((n0 + kR - 1) / kR) * kR);
  return cudaGetLastError();
}

}  // namespace shen
