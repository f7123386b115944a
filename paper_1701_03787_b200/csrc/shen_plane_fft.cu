// Periodic (y, z) plane transforms of the 3-D Shen transforms (reference
// transforms.py:181-205: numpy rfft2 / irfft2 over axes (1, 2) of the
// (n_x + 1, n_y, n_z) field), one HBM pass per direction.
//
// A plane of n_y x n_z = 256 x 256 doubles (512 KB; its half spectrum is
// 256 x 129 complex) does not fit one CTA's shared memory, so a
// thread-block cluster of 16 CTAs owns a plane and the y/z transpose goes
// through distributed shared memory instead of HBM.  CTA c holds the 16
// rows y = 16 j + c, i.e. one value of the low digit of y = 16 n1 + n2, so
// the 256-point y FFT (16 x 16 Cooley-Tukey) splits as
//
//   forward  z: two real rows per 256-point complex FFT (a + i b, split by
//            conjugate symmetry), rows loaded straight from HBM into registers;
//            y pass 1 (over n1 = j): local, every column, times W256^(c k1);
//            y pass 2 (over n2): CTA c takes k1 = c, reading the 16 CTAs'
//            pass-1 values of its k1 from distributed shared memory, and
//            writes the contiguous spectrum rows y' = c + 16 k2.
//   inverse  the same steps reversed: CTA c reads rows c + 16 k2, does the
//            pass over k2 and pushes each result to the CTA owning its n2;
//            the pass over k1 is local, then the z c2r of two rows per
//            complex FFT.  As numpy's irfft, the imaginary parts of the
//            z = 0 and z = n_z/2 coefficients are ignored.
//
// One cluster barrier per plane (plus one at the end / start that only
// guards shared-memory lifetime).  All arithmetic is fp64: radix-4 x 4
// register DFT16 butterflies and a W256^(a b) table (a, b < 16) laid out so
// both the per-lane and the per-CTA twiddle reads are conflict-free; results
// agree with pocketfft / cuFFT to rounding (~1e-16 relative).  Bytes per
// plane: 512 KB real + 516 KB complex, each once.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

#include "shen_kernels.h"

namespace shen {
namespace {

constexpr int kNY = 256, kNZ = 256, kNZH = kNZ / 2 + 1;
constexpr int kC = 16;                 // CTAs per plane (one non-portable cluster)
constexpr int kPair = 544;             // doubles per row pair in shared memory
constexpr int kSlot = 272;             // offset of the pair's second row (16 x 17 planar, padded)
constexpr int kThreads = 160;          // 128 for the z phase, 129 column tasks in the y phases
constexpr size_t kRegion = (size_t)8 * kPair * 8;  // 8 row pairs: 34816 B
constexpr size_t kSmem = 256 * 16 + kRegion;       // twiddle table + region

// W256^(a b) for a, b < 16, row a (host-computed, loaded to shared memory per CTA)
__device__ double2 g_tw[256];

// per-CTA phase timestamps (variant builds with -DSHEN_PF_TIMING only; tools/plane_fft_phases.py)
#ifdef SHEN_PF_TIMING
__device__ long long g_pf_ts[1 << 16][10];
#define PF_TS(k)                                                   \
  do {                                                             \
    if (threadIdx.x == 0 && blockIdx.x < (1 << 16)) {              \
      long long tnow;                                              \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));     \
      g_pf_ts[blockIdx.x][k] = tnow;                               \
      if ((k) == 0) {                                              \
        unsigned smid;                                             \
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));          \
        g_pf_ts[blockIdx.x][9] = smid;                             \
      }                                                            \
    }                                                              \
  } while (0)
#else
#define PF_TS(k) \
  do {           \
  } while (0)
#endif

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 w) {
  return make_double2(fma(a.x, w.x, -(a.y * w.y)), fma(a.x, w.y, a.y * w.x));
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 w) {  // a * conj(w)
  return make_double2(fma(a.x, w.x, a.y * w.y), fma(a.y, w.x, -(a.x * w.y)));
}

// exp(-+2 pi i J / 16) * a
template <int J, bool INV>
__device__ __forceinline__ double2 tw16(double2 a) {
  constexpr double C1 = 0.92387953251128675613, S1 = 0.38268343236508977173, R2 = 0.70710678118654752440;
  constexpr int j = J & 15;
  constexpr double sg = INV ? 1.0 : -1.0;  // sign of the sine
  if constexpr (j == 0) return a;
  else if constexpr (j == 4) return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
  else if constexpr (j == 8) return make_double2(-a.x, -a.y);
  else if constexpr (j == 2 || j == 6) {
    // (c + i sg s) with |c| = s = 1/sqrt 2
    constexpr double c = j == 2 ? R2 : -R2, s = sg * R2;
    return make_double2(c * a.x - s * a.y, c * a.y + s * a.x);
  } else {
    constexpr double c = j == 1 ? C1 : j == 3 ? S1 : -C1;   // j in {1, 3, 9}
    constexpr double s0 = j == 1 ? S1 : j == 3 ? C1 : -S1;  // sin(2 pi j / 16)
    constexpr double s = sg * s0;
    return make_double2(fma(c, a.x, -(s * a.y)), fma(c, a.y, s * a.x));
  }
}

template <bool INV>
__device__ __forceinline__ void dft4(double2& a0, double2& a1, double2& a2, double2& a3) {
  const double2 t0 = cadd(a0, a2), t1 = csub(a0, a2), t2 = cadd(a1, a3), t3 = csub(a1, a3);
  const double2 jt = INV ? make_double2(-t3.y, t3.x) : make_double2(t3.y, -t3.x);  // +-i t3
  a0 = cadd(t0, t2);
  a2 = csub(t0, t2);
  a1 = cadd(t1, jt);
  a3 = csub(t1, jt);
}

// in-register 16-point DFT, natural order in and out (n = 4 n1 + n2, k = k1 + 4 k2)
template <bool INV>
__device__ __forceinline__ void dft16(double2 (&v)[16]) {
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) dft4<INV>(v[n2], v[4 + n2], v[8 + n2], v[12 + n2]);
  // slot 4 k1 + n2 holds A[k1][n2]; twiddle by W16^(n2 k1)
  v[5] = tw16<1, INV>(v[5]);
  v[6] = tw16<2, INV>(v[6]);
  v[7] = tw16<3, INV>(v[7]);
  v[9] = tw16<2, INV>(v[9]);
  v[10] = tw16<4, INV>(v[10]);
  v[11] = tw16<6, INV>(v[11]);
  v[13] = tw16<3, INV>(v[13]);
  v[14] = tw16<6, INV>(v[14]);
  v[15] = tw16<9, INV>(v[15]);
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) dft4<INV>(v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]);
  double2 o[16];
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1)
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) o[k1 + 4 * k2] = v[4 * k1 + k2];
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = o[k];
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t cl_map(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ double2 ld_cl(uint32_t a) {
  double2 v;
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_cl(uint32_t a, double2 v) {
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// split cluster barrier: arrive (release) early, wait (acquire) late
__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ uint32_t cl_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cpa16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ double2 ld_nc2(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_cs2(double2* p, double2 v) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ void st_cs1(double* p, double v) {
  asm volatile("st.global.cs.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void cl_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ double ld_nc1(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ void load_tw(double2* tw) {
  for (int j = threadIdx.x; j < 256; j += blockDim.x) tw[j] = g_tw[j];
}

// XCH: the spectrum rows do not go to `out` but straight into the kx-row
// buffers of the ranks that own them (PlaneXch, peer memory over NVLink): the
// slab transform's all-to-all fused into the FFT's store.
template <bool XCH>
__global__ void __launch_bounds__(kThreads, 4)
    rfft2_256_kernel(const double* __restrict__ in, double2* __restrict__ out, const __grid_constant__ PlaneXch xc,
                     const double* __restrict__ fac) {
  extern __shared__ __align__(16) double sm[];
  double2* tw = reinterpret_cast<double2*>(sm);
  double* A = sm + 2 * 256;
  const int c = (int)cl_rank();
  const int64_t plane = blockIdx.x / kC;
  const int t = threadIdx.x;
  PF_TS(0);
  const int p = t >> 4, g = t & 15, lane = t & 31;
  double2 v[16];
  if (t < 128) {  // rows a = 16 (2p) + c, b = a + 16, straight into registers
    const double* ra = in + plane * (kNY * kNZ) + (int64_t)(32 * p + c) * kNZ + g;
#pragma unroll
    for (int n1 = 0; n1 < 16; ++n1) v[n1] = make_double2(ld_nc1(ra + 16 * n1), ld_nc1(ra + kC * kNZ + 16 * n1));
  }
  load_tw(tw);
  __syncthreads();
  PF_TS(1);
  double* pa = A + (p & 7) * kPair;
  // ---- z: rows a, b of pair p as one complex FFT, 16 threads per pair
  if (t < 128) {
    dft16<false>(v);
#pragma unroll
    for (int k1 = 1; k1 < 16; ++k1) v[k1] = cmul(v[k1], tw[16 * k1 + g]);
#pragma unroll
    for (int k1 = 0; k1 < 16; ++k1) {
      pa[17 * k1 + g] = v[k1].x;
      pa[kSlot + 17 * k1 + g] = v[k1].y;
    }
    __syncwarp();
#pragma unroll
    for (int n2 = 0; n2 < 16; ++n2) v[n2] = make_double2(pa[17 * g + n2], pa[kSlot + 17 * g + n2]);
    dft16<false>(v);  // v[k2] = Z[g + 16 k2]
    __syncwarp();
    const int partner = (lane & 16) | ((16 - g) & 15);
#pragma unroll
    for (int k2 = 0; k2 <= 8; ++k2) {
      // Z[256 - k]: lane 16 - g's Z[.. + 16 (15 - k2)], or (g = 0) this lane's Z[16 (16 - k2)]
      double mr = __shfl_sync(0xffffffffu, v[15 - k2].x, partner);
      double mi = __shfl_sync(0xffffffffu, v[15 - k2].y, partner);
      if (g == 0) {
        mr = v[(16 - k2) & 15].x;
        mi = v[(16 - k2) & 15].y;
      }
      const int k = g + 16 * k2;
      if (k <= kNZ / 2) {
        const double zr = v[k2].x, zi = v[k2].y;
        *reinterpret_cast<double2*>(pa + 2 * k) = make_double2(0.5 * (zr + mr), 0.5 * (zi - mi));
        *reinterpret_cast<double2*>(pa + kSlot + 2 * k) = make_double2(0.5 * (zi + mi), 0.5 * (mr - zr));
      }
    }
  }
  __syncthreads();
  PF_TS(2);
  // ---- y pass 1 (local): column z = t, row j = n1 at pair j >> 1, slot j & 1
  const int z = t;
  double* col = A + 2 * z;
  if (z < kNZH) {
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = *reinterpret_cast<const double2*>(col + (j >> 1) * kPair + (j & 1) * kSlot);
    dft16<false>(v);
#pragma unroll
    for (int k1 = 1; k1 < 16; ++k1) v[k1] = cmul(v[k1], tw[16 * c + k1]);
#pragma unroll
    for (int k1 = 0; k1 < 16; ++k1) *reinterpret_cast<double2*>(col + (k1 >> 1) * kPair + (k1 & 1) * kSlot) = v[k1];
  }
  cl_arrive();
  const uint32_t mine = smem_u32(col + (c >> 1) * kPair + (c & 1) * kSlot);  // this CTA's k1 = c
  cl_wait();
  PF_TS(3);
  // ---- y pass 2 over n2 = source CTA: X[c + 16 k2][z]
  if (z < kNZH) {
#pragma unroll
    for (int n2 = 0; n2 < 16; ++n2) v[n2] = ld_cl(cl_map(mine, (uint32_t)n2));
  }
  cl_arrive();  // remote reads done (shared memory may be released after the final wait)
  PF_TS(4);
  if (z < kNZH) {
    dft16<false>(v);
    if (fac != nullptr) {  // a real factor per (ky, kz) line, e.g. the dealiasing mask
#pragma unroll
      for (int k2 = 0; k2 < 16; ++k2) {
        const double f = __ldg(fac + (c + 16 * k2) * kNZH + z);
        v[k2] = make_double2(v[k2].x * f, v[k2].y * f);
      }
    }
    if (XCH) {
#pragma unroll
      for (int k2 = 0; k2 < 16; ++k2) {
        const int y = c + 16 * k2, q = xc.owner[y];
        double2* o = static_cast<double2*>(xc.base[q]) +
                     ((xc.plane0 + plane) * xc.rows[q] + xc.local_row[y]) * (int64_t)kNZH + z;
        *o = v[k2];  // the consumer reads it soon (and possibly over NVLink): no streaming hint
      }
    } else {
      double2* o = out + plane * (kNY * kNZH) + (int64_t)c * kNZH + z;
#pragma unroll
      for (int k2 = 0; k2 < 16; ++k2) st_cs2(o + (int64_t)(16 * k2) * kNZH, v[k2]);
    }
  }
  PF_TS(5);
  cl_wait();
  PF_TS(6);
}

// XCH: the spectrum rows are read from the kx-row buffers of their owners
// (the inverse slab transform's all-to-all fused into the FFT's load).
template <bool XCH>
__global__ void __launch_bounds__(kThreads, 4)
    irfft2_256_kernel(const double2* __restrict__ in, double* __restrict__ out, double scale,
                      const __grid_constant__ PlaneXch xc, const double* __restrict__ fac_re,
                      const double* __restrict__ fac_im) {
  extern __shared__ __align__(16) double sm[];
  double2* tw = reinterpret_cast<double2*>(sm);
  double* A = sm + 2 * 256;
  const int c = (int)cl_rank();
  const int64_t plane = blockIdx.x / kC;
  const int t = threadIdx.x;
  cl_arrive_relaxed();  // every CTA of the cluster has started before rows are pushed
  const int z = t;
  double2 v[16];
  // ---- y pass over k2 for k1 = c: rows c + 16 k2 of the spectrum
  if (z < kNZH) {
    if (XCH) {
#pragma unroll
      for (int k2 = 0; k2 < 16; ++k2) {
        const int y = c + 16 * k2, q = xc.owner[y];
        const double2* ip = static_cast<const double2*>(xc.base[q]) +
                            ((xc.plane0 + plane) * xc.rows[q] + xc.local_row[y]) * (int64_t)kNZH + z;
        v[k2] = *ip;  // plain load: peer memory written by another GPU's kernel before the host barrier
      }
    } else {
      const double2* ip = in + plane * (kNY * kNZH) + (int64_t)c * kNZH + z;
#pragma unroll
      for (int k2 = 0; k2 < 16; ++k2) v[k2] = ld_nc2(ip + (int64_t)(16 * k2) * kNZH);
    }
    if (fac_re != nullptr) {  // a complex factor per (ky, kz) line (i m, i n: the y / z derivatives)
#pragma unroll
      for (int k2 = 0; k2 < 16; ++k2) {
        const int e = (c + 16 * k2) * kNZH + z;
        const double fr = __ldg(fac_re + e), fi = __ldg(fac_im + e);
        v[k2] = make_double2(v[k2].x * fr - v[k2].y * fi, v[k2].x * fi + v[k2].y * fr);
      }
    }
  }
  load_tw(tw);
  __syncthreads();
  double* col = A + 2 * z;
  const uint32_t slot = smem_u32(col + (c >> 1) * kPair + (c & 1) * kSlot);  // k1 = c in every CTA
  if (z < kNZH) {
    dft16<true>(v);  // v[n2]
#pragma unroll
    for (int n2 = 1; n2 < 16; ++n2) v[n2] = cmulc(v[n2], tw[16 * n2 + c]);
  }
  cl_wait();
  if (z < kNZH) {
#pragma unroll
    for (int n2 = 0; n2 < 16; ++n2) st_cl(cl_map(slot, (uint32_t)n2), v[n2]);
  }
  cl_arrive();
  cl_wait();
  // ---- y pass over k1 (local): rows j = n1 of this CTA's n2 = c
  if (z < kNZH) {
#pragma unroll
    for (int k1 = 0; k1 < 16; ++k1) v[k1] = *reinterpret_cast<const double2*>(col + (k1 >> 1) * kPair + (k1 & 1) * kSlot);
    dft16<true>(v);
#pragma unroll
    for (int j = 0; j < 16; ++j) *reinterpret_cast<double2*>(col + (j >> 1) * kPair + (j & 1) * kSlot) = v[j];
  }
  __syncthreads();
  // ---- z c2r: rows a, b of pair p -> Z = X_a + i X_b (Hermitian-extended), one complex FFT
  if (t < 128) {
    const int p = t >> 4, g = t & 15;
    double* pa = A + p * kPair;
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2) {
      const int k = g + 16 * k2;
      const bool direct = k <= kNZ / 2;
      const int kk = direct ? k : kNZ - k;
      double2 a = *reinterpret_cast<const double2*>(pa + 2 * kk);
      double2 b = *reinterpret_cast<const double2*>(pa + kSlot + 2 * kk);
      if (kk == 0 || kk == kNZ / 2) a.y = b.y = 0.0;
      v[k2] = direct ? make_double2(a.x - b.y, a.y + b.x) : make_double2(a.x + b.y, b.x - a.y);
    }
    dft16<true>(v);  // v[n2]
#pragma unroll
    for (int n2 = 1; n2 < 16; ++n2) v[n2] = cmulc(v[n2], tw[16 * n2 + g]);
    __syncwarp();
#pragma unroll
    for (int n2 = 0; n2 < 16; ++n2) {
      pa[17 * n2 + g] = v[n2].x;
      pa[kSlot + 17 * n2 + g] = v[n2].y;
    }
    __syncwarp();
#pragma unroll
    for (int k1 = 0; k1 < 16; ++k1) v[k1] = make_double2(pa[17 * g + k1], pa[kSlot + 17 * g + k1]);
    dft16<true>(v);  // v[n1] = z[16 n1 + g]
    double* oa = out + plane * (kNY * kNZ) + (int64_t)(32 * p + c) * kNZ + g;  // row y = 16 (2p) + c
    double* ob = oa + kC * kNZ;                                                // row y = 16 (2p + 1) + c
#pragma unroll
    for (int n1 = 0; n1 < 16; ++n1) {
      st_cs1(oa + 16 * n1, scale * v[n1].x);
      st_cs1(ob + 16 * n1, scale * v[n1].y);
    }
  }
}

cudaError_t init_tw() {
  static bool done = false;
  if (done) return cudaSuccess;
  double2 h[256];
  for (int a = 0; a < 16; ++a)
    for (int b = 0; b < 16; ++b) {
      const int m = (a * b) & 255;  // exp(-2 pi i m / 256)
      h[16 * a + b] = make_double2(std::cos(M_PI * m / 128.0), -std::sin(M_PI * m / 128.0));
    }
  cudaError_t e = cudaMemcpyToSymbol(g_tw, h, sizeof(h));
  if (e == cudaSuccess) done = true;
  return e;
}

template <typename K, typename... Args>
cudaError_t launch_cluster(K kernel, int64_t planes, cudaStream_t st, Args... args) {
  cudaError_t e = init_tw();
  if (e != cudaSuccess) return e;
  // per kernel, not per instantiation of this template: kernels of one
  // signature (the <false> / <true> pairs) share K
  static const void* ready[8] = {};
  bool attr = false;
  int slot = 0;
  for (; slot < 8 && ready[slot] != nullptr; ++slot) attr = attr || ready[slot] == (const void*)kernel;
  if (!attr) {
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    if (slot < 8) ready[slot] = (const void*)kernel;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(planes * kC), 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kC;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

}  // namespace

bool plane_fft_supported(int n_y, int n_z) { return n_y == kNY && n_z == kNZ; }

cudaError_t launch_plane_rfft2(int64_t planes, int n_y, int n_z, const double* x, void* X, const double* fac,
                               cudaStream_t st) {
  if (planes <= 0) return cudaSuccess;
  if (!plane_fft_supported(n_y, n_z) || planes * kC > 0x7fffffffLL) return cudaErrorInvalidValue;
  return launch_cluster(rfft2_256_kernel<false>, planes, st, x, static_cast<double2*>(X), PlaneXch{}, fac);
}

cudaError_t launch_plane_rfft2_scatter(int64_t planes, int n_y, int n_z, const double* x, const PlaneXch& xc,
                                       cudaStream_t st) {
  if (planes <= 0) return cudaSuccess;
  if (!plane_fft_supported(n_y, n_z) || planes * kC > 0x7fffffffLL) return cudaErrorInvalidValue;
  return launch_cluster(rfft2_256_kernel<true>, planes, st, x, static_cast<double2*>(nullptr), xc,
                        static_cast<const double*>(nullptr));
}

cudaError_t launch_plane_irfft2_gather(int64_t planes, int n_y, int n_z, const PlaneXch& xc, double* x, double scale,
                                       cudaStream_t st) {
  if (planes <= 0) return cudaSuccess;
  if (!plane_fft_supported(n_y, n_z) || planes * kC > 0x7fffffffLL) return cudaErrorInvalidValue;
  return launch_cluster(irfft2_256_kernel<true>, planes, st, static_cast<const double2*>(nullptr), x, scale, xc,
                        static_cast<const double*>(nullptr), static_cast<const double*>(nullptr));
}

cudaError_t launch_plane_irfft2(int64_t planes, int n_y, int n_z, const void* X, double* x, double scale,
                                const double* fac_re, const double* fac_im, cudaStream_t st) {
  if (planes <= 0) return cudaSuccess;
  if (!plane_fft_supported(n_y, n_z) || planes * kC > 0x7fffffffLL) return cudaErrorInvalidValue;
  return launch_cluster(irfft2_256_kernel<false>, planes, st, static_cast<const double2*>(X), x, scale, PlaneXch{},
                        fac_re, fac_im);
}

}  // namespace shen

#ifdef SHEN_PF_TIMING
extern "C" int shen_pf_ts_read(void* host, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(host, shen::g_pf_ts, bytes);
}
#endif
