// Fused wall-normal Shen transforms: one kernel per direction does the
// whole axis-0 stage of the reference's 3-D transforms (transforms.py:81-205)
// on a tile of TL Fourier lines held in shared memory:
//
//   forward : DCT (scipy dct type 2 on Gauss points, type 1 on Gauss-Lobatto
//             points) -> Chebyshev scaling -> Shen stencil (shen_scalar,
//             transforms.py:81-110) -> per-parity banded Cholesky mass solve
//             with the reference's own LAPACK factors (transforms.py:143-175);
//   inverse : shen_expand (transforms.py:113-126) -> Chebyshev evaluation on
//             the points (transforms.py:129-137), times the 1/(n_y n_z) of
//             the following inverse periodic FFT.
//
// The DCTs run on chip as complex DFTs of one length-Ld sequence per line:
//   Gauss    Ld = N (Makhoul's reordering v_i = x_sigma(i), sigma = even
//            points ascending then odd points descending; the DCT-II is read
//            off V_k and V_{N-k}, and the DCT-III is the inverse map);
//   Lobatto  Ld = 2 n_x (the even extension; its DFT is the DCT-I).
// A length-Ld DFT is one of: a power-of-two FFT (Ld = M), Rader's algorithm
// for a prime Ld whose Ld - 1 = M is a power of two (N = 257 at config 3:
// a cyclic convolution of length 256), or Bluestein's chirp convolution on a
// power-of-two M >= 2 Ld - 1 otherwise.  The power-of-two FFT is a
// decimation-in-frequency pass sequence (radix 16 / 8 / 4 / 2 butterflies in
// registers, one pass per radix stage through shared memory) that leaves the
// spectrum in digit-reversed order; convolutions multiply there by the
// kernel's spectrum (host-built in the same order) and return to natural
// order by the mirrored decimation-in-time passes, the last forward and the
// first inverse pass fused in registers.  Tables (twiddles, Rader index
// maps, convolution kernels, chirps, stencil and Cholesky factors) are built
// on the host (paper_1701_03787_b200/wall.py).
//
// Layout: lines (rows, L) complex128, the L Fourier lines contiguous; the tile
// is rows x TL complex values (TL consecutive lines: 16 x 16 B = 256-B row
// pieces at TL = 16), shared-memory position p of line l at T[p * TL + l].
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "shen_common.cuh"
#include "shen_kernels.h"
#include "shen_tma.cuh"

namespace shen {
namespace {

using cd = double2;
constexpr int kWallThreads = 256;

// per-CTA phase timestamps (A/B variant builds with -DSHEN_WALL_TIMING only;
// tools/wall_phases.py reads them)
#ifdef SHEN_WALL_TIMING
__device__ long long g_wall_ts[1 << 16][6];
#define WALL_TS(k)                                                \
  do {                                                            \
    if (threadIdx.x == 0 && blockIdx.x < (1 << 16)) {             \
      g_wall_ts[blockIdx.x][k] = clock64();                       \
      if ((k) == 0) {                                             \
        unsigned smid;                                            \
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));         \
        g_wall_ts[blockIdx.x][5] = smid;                          \
      }                                                           \
    }                                                             \
  } while (0)
#else
#define WALL_TS(k) \
  do {             \
  } while (0)
#endif

__device__ __forceinline__ cd cadd(cd a, cd b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ cd csub(cd a, cd b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ cd cmul(cd a, cd b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ cd cmulc(cd a, cd b) {  // a * conj(b)
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ cd cscale(double s, cd a) { return make_double2(s * a.x, s * a.y); }
__device__ __forceinline__ cd cconj(cd a) { return make_double2(a.x, -a.y); }

// ------------------------------------------------------------------ register DFTs
// W16^e (forward sign e^{-2 pi i e / 16}, e < 8) applied to x; INV: conjugate
constexpr double kC1 = 0.92387953251128675613, kS1 = 0.38268343236508977173, kH = 0.70710678118654752440;
template <bool INV>
__device__ __forceinline__ cd w16(cd x, int e) {
  switch (e) {
    case 0: return x;
    case 4: return INV ? make_double2(-x.y, x.x) : make_double2(x.y, -x.x);
    case 2: return INV ? make_double2(kH * (x.x - x.y), kH * (x.x + x.y)) : make_double2(kH * (x.x + x.y), kH * (x.y - x.x));
    case 6: return INV ? make_double2(-kH * (x.x + x.y), kH * (x.x - x.y)) : make_double2(kH * (x.y - x.x), -kH * (x.x + x.y));
    default: {
      const double c = (e == 1) ? kC1 : (e == 3) ? kS1 : (e == 5) ? -kS1 : -kC1;
      const double s = (e == 1) ? kS1 : (e == 3) ? kC1 : (e == 5) ? kC1 : kS1;
      // forward: x * (c - i s); INV: x * (c + i s)
      return INV ? make_double2(fma(c, x.x, -s * x.y), fma(c, x.y, s * x.x))
                 : make_double2(fma(c, x.x, s * x.y), fma(c, x.y, -s * x.x));
    }
  }
}

template <int R>
__host__ __device__ constexpr int brev(int i) {
  int r = 0;
  for (int b = 1; b < R; b <<= 1) {
    r = (r << 1) | (i & 1);
    i >>= 1;
  }
  return r;
}

// in-register DFT of size R (natural order in and out); INV: conjugate kernel
template <int R, bool INV>
__device__ __forceinline__ void dft(cd* v) {
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int j = brev<R>(i);
    if (i < j) {
      const cd t = v[i];
      v[i] = v[j];
      v[j] = t;
    }
  }
#pragma unroll
  for (int s = 2; s <= R; s <<= 1) {
#pragma unroll
    for (int k = 0; k < s / 2; ++k) {
#pragma unroll
      for (int b = 0; b < R; b += s) {
        const cd t = w16<INV>(v[b + k + s / 2], k * (16 / s));
        const cd u = v[b + k];
        v[b + k] = cadd(u, t);
        v[b + k + s / 2] = csub(u, t);
      }
    }
  }
}

// W_M^{idx} from the table (forward sign); INV: conjugate
template <bool INV>
__device__ __forceinline__ cd twid(const cd* __restrict__ tw, int idx) {
  const cd w = __ldg(tw + idx);
  return INV ? cconj(w) : w;
}

struct Stage {
  int R, Ls;
};

// Compile-time plan shape: the DFT kind, radix sequence and lines per tile of
// the hot configurations (BASELINE config 3, n_x = 256: Gauss = Rader over
// 16 x 16, Lobatto = powers of two 16 x 8 x 4) are template constants, so
// every radix switch folds and the tile index math is constant shifts; any
// other plan runs the dynamic instantiation (WDyn) of the same code.
template <int K_, int S_, int R0_, int R1_, int R2_, int TLS_, bool PIPE_ = false>
struct WShape {
  static constexpr int K = K_, S = S_, R0 = R0_, R1 = R1_, R2 = R2_, TLS = TLS_;
  // PIPE: barriers span the 256 DFT threads only (named barrier 1), for a
  // kernel whose extra warps work on another tile meanwhile; a pipelined
  // forward kernel built on it (8 DFT warps + 1 mass-sweep warp, two tile
  // buffers, 1 CTA per SM) measured slower than two one-tile CTAs per SM
  // (190 vs 149 us at C3): the DFT passes need the second CTA's warps
  static constexpr bool PIPE = PIPE_;
};
using WDyn = WShape<-1, 0, 0, 0, 0, -1>;
// barrier of the threads that run the DFT passes (all of them, or warps 0-7
// of the pipelined kernel, whose ninth warp runs the mass sweeps meanwhile)
template <class SH>
__device__ __forceinline__ void wsync() {
  if (SH::PIPE) asm volatile("bar.sync 1, 256;" ::: "memory");
  else __syncthreads();
}
template <class SH>
__device__ __forceinline__ int sh_kind(const WallPlan& p) { return SH::K >= 0 ? SH::K : p.kind; }
template <class SH>
__device__ __forceinline__ int sh_nst(const WallPlan& p) { return SH::S > 0 ? SH::S : p.nstage; }
template <class SH>
__device__ __forceinline__ int sh_rad(const WallPlan& p, int s) {
  if (SH::S > 0) return s == 0 ? SH::R0 : s == 1 ? SH::R1 : s == 2 ? SH::R2 : 1;
  return p.radix[s];
}
template <class SH>
__device__ __forceinline__ int sh_M(const WallPlan& p) {
  return SH::S > 0 ? SH::R0 * (SH::S > 1 ? SH::R1 : 1) * (SH::S > 2 ? SH::R2 : 1) : p.M;
}
template <class SH>
__device__ __forceinline__ int sh_tls(const WallPlan& p) { return SH::TLS >= 0 ? SH::TLS : p.log2_lines; }

// one decimation-in-frequency pass (forward sign) in place: butterflies of
// radix R over sub-FFTs of size Ls (q = Ls / R apart), twiddle after
template <int R>
__device__ __forceinline__ void pass_dif(cd* T, int TLs, int M, int Ls, const cd* __restrict__ tw) {
  constexpr int lR = R == 16 ? 4 : R == 8 ? 3 : R == 4 ? 2 : 1;
  const int lLs = 31 - __clz(Ls), lM = 31 - __clz(M);
  const int lq = lLs - lR, q = 1 << lq, nb = M >> lR, TL = 1 << TLs, lts = lM - lLs;
  for (int w = threadIdx.x; w < nb * TL; w += kWallThreads) {
    const int l = w & (TL - 1), b = w >> TLs;
    const int blk = b >> lq, n1 = b & (q - 1), base = (blk << lLs) + n1;
    cd v[R];
#pragma unroll
    for (int j = 0; j < R; ++j) v[j] = T[((base + q * j) << TLs) + l];
    dft<R, false>(v);
    if (q > 1) {
#pragma unroll
      for (int k = 1; k < R; ++k) v[k] = cmul(v[k], twid<false>(tw, ((n1 * k) << lts) & (M - 1)));
    }
#pragma unroll
    for (int k = 0; k < R; ++k) T[((base + q * k) << TLs) + l] = v[k];
  }
}

// one decimation-in-time pass with the conjugate kernel (undoes pass_dif up to a factor R)
template <int R>
__device__ __forceinline__ void pass_dit_inv(cd* T, int TLs, int M, int Ls, const cd* __restrict__ tw) {
  constexpr int lR = R == 16 ? 4 : R == 8 ? 3 : R == 4 ? 2 : 1;
  const int lLs = 31 - __clz(Ls), lM = 31 - __clz(M);
  const int lq = lLs - lR, q = 1 << lq, nb = M >> lR, TL = 1 << TLs, lts = lM - lLs;
  for (int w = threadIdx.x; w < nb * TL; w += kWallThreads) {
    const int l = w & (TL - 1), b = w >> TLs;
    const int blk = b >> lq, n1 = b & (q - 1), base = (blk << lLs) + n1;
    cd v[R];
#pragma unroll
    for (int j = 0; j < R; ++j) v[j] = T[((base + q * j) << TLs) + l];
    if (q > 1) {
#pragma unroll
      for (int k = 1; k < R; ++k) v[k] = cmul(v[k], twid<true>(tw, ((n1 * k) << lts) & (M - 1)));
    }
    dft<R, true>(v);
#pragma unroll
    for (int k = 0; k < R; ++k) T[((base + q * k) << TLs) + l] = v[k];
  }
}

__device__ __forceinline__ void run_dif(int R, cd* T, int TLs, int M, int Ls, const cd* tw) {
  switch (R) {
    case 16: pass_dif<16>(T, TLs, M, Ls, tw); break;
    case 8: pass_dif<8>(T, TLs, M, Ls, tw); break;
    case 4: pass_dif<4>(T, TLs, M, Ls, tw); break;
    default: pass_dif<2>(T, TLs, M, Ls, tw); break;
  }
}
__device__ __forceinline__ void run_dit_inv(int R, cd* T, int TLs, int M, int Ls, const cd* tw) {
  switch (R) {
    case 16: pass_dit_inv<16>(T, TLs, M, Ls, tw); break;
    case 8: pass_dit_inv<8>(T, TLs, M, Ls, tw); break;
    case 4: pass_dit_inv<4>(T, TLs, M, Ls, tw); break;
    default: pass_dit_inv<2>(T, TLs, M, Ls, tw); break;
  }
}

// fused: last DIF pass (Ls = R, no twiddle), product with the convolution
// kernel (digit-reversed order), first inverse DIT pass (Ls = R)
template <int R>
__device__ __forceinline__ void pass_conv(cd* T, int TLs, int M, const cd* __restrict__ ker, cd* a0) {
  const int nb = M / R, TL = 1 << TLs;
  for (int w = threadIdx.x; w < nb * TL; w += kWallThreads) {
    const int l = w & (TL - 1), b = w >> TLs, base = b * R;  // R is a compile-time power of two
    cd v[R];
#pragma unroll
    for (int j = 0; j < R; ++j) v[j] = T[((base + j) << TLs) + l];
    dft<R, false>(v);
    if (b == 0 && a0 != nullptr) a0[l] = v[0];  // A(0): the DC term (Rader's X_0)
#pragma unroll
    for (int k = 0; k < R; ++k) v[k] = cmul(v[k], __ldg(ker + base + k));
    dft<R, true>(v);
#pragma unroll
    for (int k = 0; k < R; ++k) T[((base + k) << TLs) + l] = v[k];
  }
}
__device__ __forceinline__ void run_conv(int R, cd* T, int TLs, int M, const cd* ker, cd* a0) {
  switch (R) {
    case 16: pass_conv<16>(T, TLs, M, ker, a0); break;
    case 8: pass_conv<8>(T, TLs, M, ker, a0); break;
    case 4: pass_conv<4>(T, TLs, M, ker, a0); break;
    default: pass_conv<2>(T, TLs, M, ker, a0); break;
  }
}

// first DIF pass with a gather: position i of line l takes ld(i, l); every
// thread loads all of its butterflies' inputs before any thread stores
// (requires nb * TL <= threads), so the gather may read the rows it overwrites
template <class SH, int R, class LD>
__device__ __forceinline__ void pass_dif_gather(cd* T, int TLs, int M, const cd* __restrict__ tw, LD ld) {
  const int Ls = M, q = M / R, nb = M / R, TL = 1 << TLs, tstep = 1;
  const int w = threadIdx.x;
  const bool act = w < nb * TL;
  const int l = w & (TL - 1), n1 = w >> TLs;  // blk = 0
  cd v[R];
  if (act) {
#pragma unroll
    for (int j = 0; j < R; ++j) v[j] = ld(n1 + q * j, l);
  }
  wsync<SH>();
  if (act) {
    dft<R, false>(v);
    if (q > 1) {
#pragma unroll
      for (int k = 1; k < R; ++k) v[k] = cmul(v[k], twid<false>(tw, (n1 * k * tstep) & (M - 1)));
    }
#pragma unroll
    for (int k = 0; k < R; ++k) T[((n1 + q * k) << TLs) + l] = v[k];
  }
  (void)Ls;
}
// last inverse DIT pass (Ls = M) with a scatter: natural output index i of
// line l goes to st(i, l, value); loads all before any store (same condition)
template <class SH, int R, class ST>
__device__ __forceinline__ void pass_dit_inv_scatter(cd* T, int TLs, int M, const cd* __restrict__ tw, ST st) {
  const int q = M / R, nb = M / R, TL = 1 << TLs;
  const int w = threadIdx.x;
  const bool act = w < nb * TL;
  const int l = w & (TL - 1), n1 = w >> TLs;
  cd v[R];
  if (act) {
#pragma unroll
    for (int j = 0; j < R; ++j) v[j] = T[((n1 + q * j) << TLs) + l];
    if (q > 1) {
#pragma unroll
      for (int k = 1; k < R; ++k) v[k] = cmul(v[k], twid<true>(tw, (n1 * k) & (M - 1)));
    }
    dft<R, true>(v);
  }
  wsync<SH>();
  if (act) st(n1, q, l, v);  // outputs n1 + q k, k < R (v by reference: stays in registers)
}

template <class SH, class LD>
__device__ __forceinline__ void gather_first(int R, cd* T, int TLs, int M, const cd* tw, LD ld) {
  switch (R) {
    case 16: pass_dif_gather<SH, 16>(T, TLs, M, tw, ld); break;
    case 8: pass_dif_gather<SH, 8>(T, TLs, M, tw, ld); break;
    case 4: pass_dif_gather<SH, 4>(T, TLs, M, tw, ld); break;
    default: pass_dif_gather<SH, 2>(T, TLs, M, tw, ld); break;
  }
}
template <class SH, class ST>
__device__ __forceinline__ void scatter_last(int R, cd* T, int TLs, int M, const cd* tw, ST st) {
  switch (R) {
    case 16: pass_dit_inv_scatter<SH, 16>(T, TLs, M, tw, st); break;
    case 8: pass_dit_inv_scatter<SH, 8>(T, TLs, M, tw, st); break;
    case 4: pass_dit_inv_scatter<SH, 4>(T, TLs, M, tw, st); break;
    default: pass_dit_inv_scatter<SH, 2>(T, TLs, M, tw, st); break;
  }
}

// A length-M DFT of the gathered sequence: either the full forward FFT
// (digit-reversed result left in T) or, with a kernel, the cyclic
// convolution of the gathered sequence with it (natural order, handed to
// the scatter).  a0 receives the DC term of the forward FFT (Rader).
template <class SH, class LD, class ST>
__device__ __forceinline__ void wall_dft(const WallPlan& p, cd* T, int TLs, const cd* ker, cd* a0, LD ld,
                                         ST st) {
  const int M = sh_M<SH>(p), S = sh_nst<SH>(p);
  int Ls = M;
  gather_first<SH>(sh_rad<SH>(p, 0), T, TLs, M, p.tw, ld);
  wsync<SH>();
  if (ker == nullptr) {
    Ls /= sh_rad<SH>(p, 0);
#pragma unroll
    for (int s = 1; s < 4; ++s) {
      if (s >= S) break;
      run_dif(sh_rad<SH>(p, s), T, TLs, M, Ls, p.tw);
      Ls /= sh_rad<SH>(p, s);
      wsync<SH>();
    }
    return;
  }
  if (S == 1) {
    // a single radix stage: gather pass already did the forward DFT; multiply and invert in place
    const int TL = 1 << TLs;
    for (int w = threadIdx.x; w < M * TL; w += kWallThreads) {
      const int l = w & (TL - 1), i = w >> TLs;
      if (i == 0 && a0 != nullptr) a0[l] = T[l];
      T[(i << TLs) + l] = cmul(T[(i << TLs) + l], __ldg(ker + i));
    }
    wsync<SH>();
    scatter_last<SH>(sh_rad<SH>(p, 0), T, TLs, M, p.tw, st);
    wsync<SH>();
    return;
  }
  Ls /= sh_rad<SH>(p, 0);
#pragma unroll
  for (int s = 1; s < 3; ++s) {
    if (s >= S - 1) break;
    run_dif(sh_rad<SH>(p, s), T, TLs, M, Ls, p.tw);
    Ls /= sh_rad<SH>(p, s);
    wsync<SH>();
  }
  // S - 1 = 1..3: the last stage's convolution pass
  const int RL = S == 2 ? sh_rad<SH>(p, 1) : S == 3 ? sh_rad<SH>(p, 2) : sh_rad<SH>(p, 3);
  run_conv(RL, T, TLs, M, ker, a0);  // Ls == radix[S-1]
  wsync<SH>();
  Ls = RL;
#pragma unroll
  for (int s = 2; s >= 1; --s) {
    if (s > S - 2) continue;
    Ls *= sh_rad<SH>(p, s);
    run_dit_inv(sh_rad<SH>(p, s), T, TLs, M, Ls, p.tw);
    wsync<SH>();
  }
  scatter_last<SH>(sh_rad<SH>(p, 0), T, TLs, M, p.tw, st);
  wsync<SH>();
}

__device__ __forceinline__ int sigma(int i, int N) {  // Makhoul: v_i = x_sigma(i)
  const int h = (N + 1) >> 1;
  return i < h ? 2 * i : 2 * (N - 1 - i) + 1;
}

// ------------------------------------------------------------------ forward
// shared memory: tile T [rows_smem][TL] | side [2][TL] | mbarrier | (forward, mass) factors [2][3][mmax]
__device__ __forceinline__ unsigned char* wall_smem_base(unsigned char* raw) {
  return raw + ((1024u - (su32(raw) & 1023u)) & 1023u);  // TMA boxes land 128-B aligned
}

// the tile's rows [0, rows) arrive by 2-D TMA boxes of box rows (OOB rows and
// columns zero-filled)
__device__ __forceinline__ void wall_load(cd* T, uint64_t* bar, const CUtensorMap* tin, int rows, int box, int TL,
                                          int64_t l0) {
  if (threadIdx.x == 0) {
    mb_init(bar, 1);
    mb_fence_init();
  }
  __syncthreads();  // the barrier is initialised before anyone waits on it
  if (threadIdx.x == 0) {
    const int nbox = (rows + box - 1) / box;
    mb_expect(bar, (uint32_t)nbox * box * TL * sizeof(cd));
    for (int b = 0; b < nbox; ++b) tma_load_2d(T + (size_t)b * box * TL, tin, (int)(2 * l0), b * box, bar);
  }
}
__device__ __forceinline__ void wall_store(cd* T, const CUtensorMap* tout, int rows, int box, int TL, int64_t l0) {
  fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nbox = (rows + box - 1) / box;
    for (int b = 0; b < nbox; ++b) tma_store_2d(tout, (int)(2 * l0), b * box, T + (size_t)b * box * TL);
    bulk_commit();
    bulk_wait_read0();  // the CTA's shared memory must outlive the store's reads
  }
}

// DFT of a tile's lines and the Chebyshev scaling (everything of the
// forward kernel before the stencil / mass solve); the 256 DFT threads.
template <int KMAX, class SH>
__device__ __forceinline__ void fwd_dft_post(const WallPlan& p, cd* T, cd* side, int tid) {
  const int TLs = sh_tls<SH>(p), TL = 1 << TLs;
  const int kind = sh_kind<SH>(p), Mv = sh_M<SH>(p);
  const int N = p.N;
  const bool gauss = p.family == 0;
  // ---- DFT of the gathered sequence
  if (kind == 0) {  // power of two: Lobatto even extension z (Ld = M = 2 n_x)
    const int nx = N - 1;
    wall_dft<SH>(p, T, TLs, nullptr, nullptr,
             [&](int i, int l) { return T[((i <= nx ? i : Mv - i) << TLs) + l]; }, [](int, int, int, auto&) {});
  } else if (kind == 1) {  // Rader (Gauss, N prime, M = N - 1)
    if (tid < TL) side[tid] = T[tid];  // v_0 = x_0
    const double scl = p.scale;
    wall_dft<SH>(p, T, TLs, p.ker_f, side + TL,
             [&](int i, int l) { return T[(__ldg(p.gin_f + i) << TLs) + l]; },
             [&](int n1, int q, int l, auto& v) {
               // V_k = x_0 + conv_q at k = g^{-q}; its partner N - k is R/2
               // outputs later in the same butterfly (g^{(N-1)/2} = -1), so
               // the DCT-II post step (w_k, w_{N-k}) happens here in registers
               constexpr int R = sizeof(v) / sizeof(cd);
               const cd x0 = side[l];
#pragma unroll
               for (int kk = 0; kk < R / 2; ++kk) {
                 const int qa = n1 + q * kk, qb = qa + q * (R / 2);
                 const int ka = __ldg(p.gout + qa), kb = __ldg(p.gout + qb);
                 const cd Va = cadd(x0, v[kk]), Vb = cadd(x0, v[kk + R / 2]);
                 const cd mka = __ldg(p.mk + ka), mkb = __ldg(p.mk + kb);
                 const cd sa = cmul(mka, cadd(Va, cconj(Vb))), da = cmul(mka, csub(Va, cconj(Vb)));
                 const cd sb = cmul(mkb, cadd(Vb, cconj(Va))), db = cmul(mkb, csub(Vb, cconj(Va)));
                 T[(ka << TLs) + l] = make_double2(sa.x * scl, da.y * scl);
                 T[(kb << TLs) + l] = make_double2(sb.x * scl, db.y * scl);
               }
             });
    // w_0 = 2 V_0 (scaled), V_0 = x_0 + A(0)
    if (tid < TL) T[tid] = cscale(2.0 * scl, cadd(side[tid], side[TL + tid]));
    wsync<SH>();
  } else {  // Bluestein
    const int Ld = p.Ld, nx = N - 1;
    wall_dft<SH>(p, T, TLs, p.ker_f, nullptr,
             [&](int i, int l) {
               if (i >= Ld) return make_double2(0.0, 0.0);
               const int src = gauss ? sigma(i, N) : (i <= nx ? i : Ld - i);
               return cmul(T[(src << TLs) + l], __ldg(p.chirp_f + i));
             },
             [&](int n1, int q, int l, auto& v) {
               constexpr int R = sizeof(v) / sizeof(cd);
#pragma unroll
               for (int kk = 0; kk < R; ++kk) {
                 const int qq = n1 + q * kk;
                 if (qq < Ld) T[(qq << TLs) + l] = cmul(v[kk], __ldg(p.chirp_f + qq));
               }
             });
  }
  // ---- Chebyshev scalar products w_k (k < N), in place
  const double scl = p.scale;
  if (kind == 1) {
    // already w (fused into the last FFT pass)
  } else if (gauss) {
    // DCT-II from V_k and V_{N-k}: one thread owns both rows of a pair
    const int npair = N / 2 + 1;  // k = 0 .. N/2, partner (N - k) mod N
    for (int e = tid; e < npair * TL; e += kWallThreads) {
      const int k = e >> TLs, l = e & (TL - 1), k2 = k == 0 ? 0 : N - k;
      const cd a = T[(k << TLs) + l], b = T[(k2 << TLs) + l];
      const cd mk = __ldg(p.mk + k);
      const cd sa = cmul(mk, cadd(a, cconj(b))), da = cmul(mk, csub(a, cconj(b)));
      if (k2 != k) {
        const cd mk2 = __ldg(p.mk + k2);
        const cd sb = cmul(mk2, cadd(b, cconj(a))), db = cmul(mk2, csub(b, cconj(a)));
        T[(k2 << TLs) + l] = make_double2(sb.x * scl, db.y * scl);
      }
      T[(k << TLs) + l] = make_double2(sa.x * scl, da.y * scl);
    }
  } else if (kind == 0) {
    // DCT-I read in digit-reversed order: gather, then store
    cd wv[KMAX];
#pragma unroll
    for (int it = 0; it < KMAX; ++it) {
      const int e = tid + it * kWallThreads;
      if (e < N * TL) wv[it] = cscale(scl, T[(__ldg(p.pinv + (e >> TLs)) << TLs) + (e & (TL - 1))]);
    }
    wsync<SH>();
#pragma unroll
    for (int it = 0; it < KMAX; ++it) {
      const int e = tid + it * kWallThreads;
      if (e < N * TL) T[e] = wv[it];
    }
  } else {
    for (int e = tid; e < N * TL; e += kWallThreads) T[e] = cscale(scl, T[e]);
  }
}

// Stencil + U^T y = s + U x = y for the (line, parity, re | im) chain
// t < 4 TL of the tile (the mass-solve block of the forward kernel, see below).
// The factors are real, so the real and imaginary parts of a line are
// independent chains: they run on different warps (t >> (TLs + 1) = 0 | 1),
// which halves the fp64 issue per warp and row step.
__device__ __forceinline__ void fwd_mass_system(const WallPlan& p, cd* T, const double* mf, int TLs, int t) {
  const int TL = 1 << TLs, n = p.n_out, sp = p.space;
  const int l = t & (TL - 1), par = (t >> TLs) & 1, comp = t >> (TLs + 1);
  const int m = (n - par + 1) / 2;
  const double2* F = reinterpret_cast<const double2*>(mf) + (size_t)par * (p.mmax + 1) * 4;  // [m][4] double2
  double* col = reinterpret_cast<double*>(T + (par << TLs) + l) + comp;  // row par + 2 i at col[i * rs]
  const int rs = 2 << (TLs + 1);
  // Blocks of KB rows.  A block's w rows and coefficients are loaded while the
  // previous block's chain runs (before its stores: later rows, never
  // overwritten by them), the stencil parts t0 = a0 w_k - a2 w_{k+2} + a4 w_{k+4}
  // of a block are independent FMAs, and only y_i = (t0_i - f2 y_{i-2}) - f1 y_{i-1}
  // is serial: one FMA per row behind y_{i-1}.  (A row-at-a-time loop stalls
  // the warp on each row's own load -> FMA chain: ~55 cycles per row.)
  constexpr int KB = 4;
  const bool bih = sp == 2;
  double y1 = 0.0, y2 = 0.0;
  double q[KB + 2];
  double2 c0[KB], c1[KB], c2[KB];
  auto load_fwd = [&](int i0, double (&qq)[KB + 2], double2 (&a)[KB], double2 (&bb)[KB], double2 (&cc)[KB]) {
#pragma unroll
    for (int j = 0; j < KB + 2; ++j) qq[j] = col[min(i0 + j, m + 1) * rs];  // rows past m + 1 are never used
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      const int i = min(i0 + j, m);  // the table has mmax + 1 >= m + 1 rows
      a[j] = F[4 * i];
      bb[j] = F[4 * i + 1];
      cc[j] = F[4 * i + 2];
    }
  };
  load_fwd(0, q, c0, c1, c2);
  for (int i0 = 0; i0 < m; i0 += KB) {
    double t0[KB], f1[KB], f2[KB];
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      const double wc = bih ? q[j + 2] : 0.0;
      t0[j] = fma(c0[j].x, q[j], fma(-c0[j].y, q[j + 1], c1[j].x * wc));
      f1[j] = c1[j].y;
      f2[j] = c2[j].x;
    }
    load_fwd(i0 + KB, q, c0, c1, c2);  // next block (clamped past the end)
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      const double y = fma(-f1[j], y1, fma(-f2[j], y2, t0[j]));
      if (i0 + j < m) col[(i0 + j) * rs] = y;
      y2 = y1;
      y1 = y;
    }
  }
  // U x = y bottom-up: x_i = (a0 y_i - g2 x_{i+2}) - g1 x_{i+1}
  double x1 = 0.0, x2 = 0.0;
  double yy[KB];
  double2 d0[KB], d2[KB], d3[KB];
  auto load_bwd = [&](int i1, double (&v)[KB], double2 (&a)[KB], double2 (&cc)[KB], double2 (&dd)[KB]) {
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      const int i = max(i1 - j, 0);  // rows i1, i1 - 1, ...
      v[j] = col[i * rs];
      a[j] = F[4 * i];
      cc[j] = F[4 * i + 2];
      dd[j] = F[4 * i + 3];
    }
  };
  load_bwd(m - 1, yy, d0, d2, d3);
  for (int i1 = m - 1; i1 >= 0; i1 -= KB) {
    double s0[KB], g1[KB], g2[KB];
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      s0[j] = d0[j].x * yy[j];
      g1[j] = d2[j].y;
      g2[j] = d3[j].x;
    }
    load_bwd(i1 - KB, yy, d0, d2, d3);  // next block: rows above, not written yet
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      const double x = fma(-g1[j], x1, fma(-g2[j], x2, s0[j]));
      if (i1 - j >= 0) col[(i1 - j) * rs] = x;
      x2 = x1;
      x1 = x;
    }
  }
}

template <int KMAX, class SH>
__global__ void __launch_bounds__(kWallThreads, 2) wall_forward_kernel(const WallPlan p, int64_t L,
                                                                       const __grid_constant__ CUtensorMap tin,
                                                                       const __grid_constant__ CUtensorMap tout,
                                                                       int box_in, int box_out) {
  extern __shared__ __align__(1024) unsigned char wsm_raw[];
  const int TLs = sh_tls<SH>(p), TL = 1 << TLs;
  cd* T = reinterpret_cast<cd*>(wall_smem_base(wsm_raw));
  cd* side = T + (size_t)p.rows_smem * TL;  // [2][TL]: x0, A(0)
  uint64_t* bar = reinterpret_cast<uint64_t*>(side + 2 * TL);
  double* mf = reinterpret_cast<double*>(bar + 2);
  const int64_t l0 = (int64_t)blockIdx.x * TL;
  const int N = p.N, tid = threadIdx.x;
#ifdef SHEN_WALL_POISON
  for (int e = threadIdx.x; e < (p.rows_smem + 2) * TL; e += kWallThreads) T[e] = make_double2(__longlong_as_double(0x7ff8dead00000000LL), 0.0);
  __syncthreads();
#endif
  WALL_TS(0);
  wall_load(T, bar, &tin, N, box_in, TL, l0);
  const bool do_mass = p.mass && (p.space == 1 || p.space == 2);
  if (do_mass)
    for (int e = tid; e < 16 * (p.mmax + 1); e += kWallThreads) mf[e] = __ldg(p.mfac + e);
  if (tid < TL) side[tid] = make_double2(0.0, 0.0);
  mb_wait(bar, 0);
  __syncthreads();
  WALL_TS(1);
  const bool gauss = p.family == 0;
  fwd_dft_post<KMAX, SH>(p, T, side, tid);
  const int n = p.n_out, sp = p.space, nx = N - 1;
  __syncthreads();
  WALL_TS(2);
  // ---- Shen stencil (shen_scalar, transforms.py:89-110) and mass solve
  if (do_mass) {
    // the stencil rides the forward sweep: s_k needs w_k, w_{k+2}, w_{k+4}
    // of the same parity, all at or ahead of the sweep, so y overwrites w in
    // place.  U^T y = s then U x = y (the reference's zpbtrs, transforms.py:
    // 173) in LAPACK's row order, one thread per (line, parity, re | im) -- a chunked
    // (scan) split measured less accurate on the biharmonic mass matrix,
    // whose recurrence is only marginally stable (roots near -0.98).  The
    // host folds the stencil and the reciprocal pivots into per-row
    // coefficients ([m][8]: a0 = 1/U_ii, a2 = c2/U_ii, a4 = c4/U_ii,
    // f1 = U_{i-1,i}/U_ii, f2 = U_{i-2,i}/U_ii, g1 = U_{i,i+1}/U_ii,
    // g2 = U_{i,i+2}/U_ii): one FMA per row on the dependency chain, the
    // w window slides in registers and the next row's coefficients are
    // loaded one row ahead.
    if (tid < 4 * TL) fwd_mass_system(p, T, mf, TLs, tid);
  } else if (sp != 3) {
    // stencil alone, in place: chunks of R rows per thread walked upwards in
    // k, the 4 rows past the chunk read before anyone writes
    const int per_line = kWallThreads >> TLs;
    const int R = (n + per_line - 1) / per_line;
    const int l = tid & (TL - 1), k0 = (tid >> TLs) * R, k1 = min(n, k0 + R);
    cd ahead[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = k1 + j;
      ahead[j] = (k0 < k1 && k < N) ? T[(k << TLs) + l] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    auto wat = [&](int k) { return k < k1 ? T[(k << TLs) + l] : ahead[k - k1]; };
    for (int k = k0; k < k1; ++k) {
      const cd wk = T[(k << TLs) + l];
      cd sk;
      if (sp == 1) {
        sk = csub(wk, wat(k + 2));
      } else if (sp == 2) {
        sk = cadd(csub(wk, cscale(__ldg(p.c2 + k), wat(k + 2))), cscale(__ldg(p.c4 + k), wat(k + 4)));
      } else {
        sk = cscale(2.0 / 3.14159265358979311600, wk);  // w * (2.0 / np.pi)
        if (k == 0 || (!gauss && k == nx)) sk = cscale(0.5, sk);
      }
      T[(k << TLs) + l] = sk;
    }
  }
  WALL_TS(3);
  wall_store(T, &tout, n, box_out, TL, l0);
  WALL_TS(4);
}

// ------------------------------------------------------------------ inverse
template <int KMAX, class SH>
__global__ void __launch_bounds__(kWallThreads, 2) wall_inverse_kernel(const WallPlan p, int64_t L,
                                                                       const __grid_constant__ CUtensorMap tin,
                                                                       const __grid_constant__ CUtensorMap tout,
                                                                       int box_in, int box_out) {
  extern __shared__ __align__(1024) unsigned char wsm_raw[];
  const int TLs = sh_tls<SH>(p), TL = 1 << TLs;
  const int kind = sh_kind<SH>(p), Mv = sh_M<SH>(p);
  cd* T = reinterpret_cast<cd*>(wall_smem_base(wsm_raw));
  cd* side = T + (size_t)p.rows_smem * TL;
  uint64_t* bar = reinterpret_cast<uint64_t*>(side + 2 * TL);
  const int64_t l0 = (int64_t)blockIdx.x * TL;
  const int N = p.N, n = p.n_in, tid = threadIdx.x, nx = N - 1;
  const bool gauss = p.family == 0;
#ifdef SHEN_WALL_POISON  // debug variant: every tile row starts as NaN (reads of unwritten rows show up)
  for (int e = threadIdx.x; e < (p.rows_smem + 2) * TL; e += kWallThreads) T[e] = make_double2(__longlong_as_double(0x7ff8dead00000000LL), 0.0);
  __syncthreads();
#endif
  wall_load(T, bar, &tin, n, box_in, TL, l0);
  {  // rows the boxes do not cover, up to N: zero (the expansion reads them)
    const int covered = ((n + box_in - 1) / box_in) * box_in;
    for (int e = covered * TL + tid; e < N * TL; e += kWallThreads) T[e] = make_double2(0.0, 0.0);
  }
  mb_wait(bar, 0);
  __syncthreads();
  // ---- shen_expand -> Chebyshev coefficients c_k (k < N), reference order
  // (transforms.py:113-126), in place: chunks walked downwards in k, the 4
  // rows below the chunk read before anyone writes
  const int sp = p.space;
  if (!gauss && (sp == 1 || sp == 2)) {  // (Gauss: expanded on the fly in the FFT's gather)
    const int per_line = kWallThreads >> TLs;
    const int R = (N + per_line - 1) / per_line;
    const int l = tid & (TL - 1), k0 = (tid >> TLs) * R, k1 = min(N, k0 + R);
    cd behind[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = k0 - 4 + j;
      behind[j] = (k0 < k1 && k >= 0 && k < n) ? T[(k << TLs) + l] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    auto coef = [&](int k) {  // coefficient k < n (0 outside)
      if (k < 0 || k >= n) return make_double2(0.0, 0.0);
      return k >= k0 ? T[(k << TLs) + l] : behind[k - (k0 - 4)];
    };
    for (int k = k1 - 1; k >= k0; --k) {
      cd c = coef(k);
      if (sp == 1) {
        c = csub(c, coef(k - 2));
      } else {
        if (k >= 2 && k - 2 < n) c = csub(c, cscale(__ldg(p.c2 + k - 2), coef(k - 2)));
        if (k >= 4 && k - 4 < n) c = cadd(c, cscale(__ldg(p.c4 + k - 4), coef(k - 4)));
      }
      T[(k << TLs) + l] = c;
    }
    __syncthreads();
  }
  if (gauss) {
    // shen_expand and the DCT-III pre-twiddle are evaluated on the fly in the
    // FFT's gather from the untouched coefficient tile (below)
  } else {
    // even sequence with doubled ends: its DFT is twice the point values
    if (p.rowscale != nullptr) {  // (Chebyshev space: no expansion pass ran)
      for (int e = tid; e < N * TL; e += kWallThreads) T[e] = cscale(__ldg(p.rowscale + (e >> TLs)), T[e]);
      __syncthreads();
    }
    if (tid < TL) {
      T[tid] = cscale(2.0, T[tid]);
      T[(nx << TLs) + tid] = cscale(2.0, T[(nx << TLs) + tid]);
    }
  }
  __syncthreads();
  const double sc = p.scale;
  // Chebyshev coefficient c_k of the expansion (reference order) from the
  // coefficient tile (rows >= n are zero), and the Makhoul pre-twiddled
  // V_m = e^{i pi m / 2N} (y_m - i y_{N-m}) / 2, y_m = c_m (1 <= m < N)
  const double* rsc = p.rowscale;
  auto cheb = [&](int k, int l) -> cd {
    cd c = T[(k << TLs) + l];
    if (rsc != nullptr) c = cscale(__ldg(rsc + k), c);
    if (sp == 1 && k >= 2) c = csub(c, T[((k - 2) << TLs) + l]);
    if (sp == 2) {  // coefficient rows >= n are zero: the stencil tables (n entries) stop there
      if (k >= 2 && k - 2 < n) c = csub(c, cscale(__ldg(p.c2 + k - 2), T[((k - 2) << TLs) + l]));
      if (k >= 4 && k - 4 < n) c = cadd(c, cscale(__ldg(p.c4 + k - 4), T[((k - 4) << TLs) + l]));
    }
    return c;
  };
  auto vgauss = [&](int m, int l) -> cd {
    const cd ym = cheb(m, l), yn = cheb(N - m, l);
    return cmulc(make_double2(0.5 * (ym.x + yn.y), 0.5 * (ym.y - yn.x)), __ldg(p.mk + m));
  };
  if (kind == 0) {  // Lobatto, power of two: f_j = DFT(even extension)_j / 2
    wall_dft<SH>(p, T, TLs, nullptr, nullptr,
             [&](int i, int l) { return T[((i <= nx ? i : Mv - i) << TLs) + l]; }, [](int, int, int, auto&) {});
    const int items = N * TL;
    cd wv[KMAX];
#pragma unroll
    for (int it = 0; it < KMAX; ++it) {
      const int e = tid + it * kWallThreads;
      if (e < items) {
        const int j = e >> TLs, l = e & (TL - 1);
        wv[it] = cscale(0.5 * sc, T[(__ldg(p.pinv + j) << TLs) + l]);
      }
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < KMAX; ++it) {
      const int e = tid + it * kWallThreads;
      if (e < items) T[e] = wv[it];
    }
    __syncthreads();
  } else if (kind == 1) {  // Rader, inverse sign: X'_k = V_0 + conv; rows sigma(k)
    if (tid < TL) side[tid] = cheb(0, tid);  // V_0 = c_0 = coefficient 0
    wall_dft<SH>(p, T, TLs, p.ker_i, side + TL, [&](int i, int l) { return vgauss(__ldg(p.gin_i + i), l); },
             [&](int n1, int q, int l, auto& v) {
               constexpr int R = sizeof(v) / sizeof(cd);
               const cd v0 = side[l];
#pragma unroll
               for (int kk = 0; kk < R; ++kk) {
                 const int k = __ldg(p.gout + n1 + q * kk);
                 T[(sigma(k, N) << TLs) + l] = cscale(sc, cadd(v0, v[kk]));
               }
             });
    if (tid < TL) T[tid] = cscale(sc, cadd(side[tid], side[TL + tid]));  // row sigma(0) = 0
    __syncthreads();
  } else {  // Bluestein
    const int Ld = p.Ld;
    wall_dft<SH>(p, T, TLs, p.ker_i, nullptr,
             [&](int i, int l) {
               if (i >= Ld) return make_double2(0.0, 0.0);
               const cd v = gauss ? (i == 0 ? cheb(0, l) : vgauss(i, l)) : T[((i <= nx ? i : Ld - i) << TLs) + l];
               return cmul(v, __ldg(p.chirp_i + i));
             },
             [&](int n1, int q, int l, auto& v) {
               constexpr int R = sizeof(v) / sizeof(cd);
#pragma unroll
               for (int kk = 0; kk < R; ++kk) {
                 const int qq = n1 + q * kk;
                 if (qq >= N) continue;
                 const cd x = cmul(v[kk], __ldg(p.chirp_i + qq));
                 T[((gauss ? sigma(qq, N) : qq) << TLs) + l] = cscale(gauss ? sc : 0.5 * sc, x);
               }
             });
  }
  wall_store(T, &tout, N, box_out, TL, l0);
}

}  // namespace

size_t wall_smem_bytes(const WallPlan& p) {
  const size_t TL = (size_t)1 << p.log2_lines;
  return ((size_t)p.rows_smem + 2) * TL * sizeof(double2) + 16 + (size_t)16 * (p.mmax + 1) * sizeof(double) + 1024;
}

int wall_box_rows(int rows) {  // fewest boxes of <= 256 rows; 8-row multiples keep every box 128-B aligned
  const int nb = (rows + 255) / 256;
  return (((rows + nb - 1) / nb) + 7) & ~7;
}

template <int KMAX, class SH = WDyn>
static cudaError_t launch_wall_k(const WallPlan& p, int64_t L, const void* in, void* out, cudaStream_t st) {
  const int TL = 1 << p.log2_lines;
  const int rows_in = p.direction == 0 ? p.N : p.n_in;
  const int rows_out = p.direction == 0 ? p.n_out : p.N;
  const int bi = wall_box_rows(rows_in), bo = wall_box_rows(rows_out);
  if (((rows_in + bi - 1) / bi) * bi > p.rows_smem || ((rows_out + bo - 1) / bo) * bo > p.rows_smem)
    return cudaErrorInvalidValue;
  CUtensorMap tin, tout;
  if (!encode_tiled_2d(&tin, in, 2 * (uint64_t)L, rows_in, (uint64_t)L * sizeof(double2), 2 * TL, bi) ||
      !encode_tiled_2d(&tout, out, 2 * (uint64_t)L, rows_out, (uint64_t)L * sizeof(double2), 2 * TL, bo))
    return cudaErrorNotSupported;
  size_t smem = wall_smem_bytes(p);
#ifdef SHEN_WALL_ONE_CTA  // probe builds: one resident CTA per SM (phase times without the co-resident CTA)
  smem = smem > (size_t)120 * 1024 ? smem : (size_t)120 * 1024;
#endif
  auto kern = p.direction == 0 ? wall_forward_kernel<KMAX, SH> : wall_inverse_kernel<KMAX, SH>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  const unsigned grid = (unsigned)((L + TL - 1) / TL);
  kern<<<grid, kWallThreads, smem, st>>>(p, L, tin, tout, bi, bo);
  return cudaGetLastError();
}

cudaError_t launch_wall(const WallPlan& p, int64_t L, const void* in, void* out, cudaStream_t st) {
  if (L <= 0) return cudaSuccess;
  if ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) return cudaErrorInvalidValue;
  const int TL = 1 << p.log2_lines;
  const int items = (p.N * TL + kWallThreads - 1) / kWallThreads;  // register-staged rows per thread
  if (p.M / p.radix[0] * TL > kWallThreads) return cudaErrorInvalidValue;
  // the config-3 shapes (n_x = 256) run their compile-time instantiations
  if (p.kind == 1 && p.nstage == 2 && p.radix[0] == 16 && p.radix[1] == 16 && p.log2_lines == 4 && items <= 17)
    return launch_wall_k<17, WShape<1, 2, 16, 16, 0, 4>>(p, L, in, out, st);
  if (p.kind == 0 && p.nstage == 3 && p.radix[0] == 16 && p.radix[1] == 8 && p.radix[2] == 4 && p.log2_lines == 3 &&
      items <= 9)
    return launch_wall_k<9, WShape<0, 3, 16, 8, 4, 3>>(p, L, in, out, st);
  if (items <= 5) return launch_wall_k<5>(p, L, in, out, st);
  if (items <= 9) return launch_wall_k<9>(p, L, in, out, st);
  if (items <= 17) return launch_wall_k<17>(p, L, in, out, st);
  if (items <= 24) return launch_wall_k<24>(p, L, in, out, st);
  return cudaErrorInvalidValue;
}

}  // namespace shen

#ifdef SHEN_WALL_TIMING
extern "C" int shen_wall_ts_read(void* host, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(host, shen::g_wall_ts, bytes);
}
#endif
