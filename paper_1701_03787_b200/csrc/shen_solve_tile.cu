// Tiled chunk-parallel Helmholtz solve: the RHS is read from HBM once.
//
// The streaming solve (shen_solve_stream.cu) re-reads the RHS in its backward
// sweep because one thread per (system, parity) cannot keep y on chip; at
// config 4 that is 53.5 B of DRAM traffic per unknown against the 32 B the
// algorithm needs.  Here a persistent CTA owns a *tile* of kTileSys
// consecutive systems (all rows, both parities) in shared memory:
//
//   load   all threads copy the tile's row pieces (kTileSys x 16 B per row,
//          contiguous in the (n_modes, batch) layout) with cp.async into a
//          padded column-major tile; the next tile is in flight while this
//          one is solved (two tile buffers);
//   solve  warp = (system, parity), lanes = 32 chunks of R rows: the
//          chunk-parallel algorithm of shen_solve_chunk.cu (pass 1 from the
//          chunk checkpoint, shuffle scans of the forward / backward affine
//          maps, pass 3 back-substitution, truncated neighbour fix) reading
//          and writing the tile instead of global memory;
//   store  all threads write the solved tile back (same row pieces).
//
// DRAM traffic per unknown: 16 B in + 16 B out + the chunk checkpoints
// (3 doubles per R rows).  Padding: column entry i lives at i + i / R, so the
// 32 lanes of a warp (rows lane * R + r) hit distinct shared-memory banks.
#include <algorithm>

#include "shen_rows.cuh"
#include "shen_kernels.h"

namespace shen {
namespace {

constexpr int kTileSys = 4;                 // systems per tile: 64-B complex row pieces
constexpr int kTileWarps = 2 * kTileSys;    // warp = (system, parity)
constexpr int kTileThreads = 32 * kTileWarps;

#ifndef SHEN_FIX_STEPS
#define SHEN_FIX_STEPS 3
#endif

__device__ __forceinline__ cplx tfma(double s, cplx b, cplx a) { return {__fma_rn(s, b.re, a.re), __fma_rn(s, b.im, a.im)}; }
__device__ __forceinline__ double tfma(double s, double b, double a) { return __fma_rn(s, b, a); }
__device__ __forceinline__ cplx tmul(double s, cplx b) { return {s * b.re, s * b.im}; }
__device__ __forceinline__ double tmul(double s, double b) { return s * b; }
__device__ __forceinline__ cplx tadd(cplx a, cplx b) { return {a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ double tadd(double a, double b) { return a + b; }
__device__ __forceinline__ cplx tsub(cplx a, cplx b) { return {a.re - b.re, a.im - b.im}; }
__device__ __forceinline__ double tsub(double a, double b) { return a - b; }
template <typename V> __device__ __forceinline__ V tzero();
template <> __device__ __forceinline__ double tzero<double>() { return 0.0; }
template <> __device__ __forceinline__ cplx tzero<cplx>() { return {0.0, 0.0}; }

__device__ __forceinline__ void tcp(cplx* dst, const cplx* src, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(src), "r"(pred ? 16 : 0) : "memory");
}
__device__ __forceinline__ void tcp(double* dst, const double* src, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(src), "r"(pred ? 8 : 0) : "memory");
}
__device__ __forceinline__ void tcommit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void twait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template <int R>
__device__ __forceinline__ int col_idx(int i) { return i + i / R; }

// tile buffer layout: [kTileSys][2 parities][32 * (R + 1)] V
template <typename V, int R>
__device__ __forceinline__ void tile_load(V* buf, const V* rhs, int n_modes, int64_t B, int64_t j0, int tid) {
  constexpr int col = 32 * (R + 1);
  const int pieces = n_modes * kTileSys;
  for (int q = tid; q < pieces; q += kTileThreads) {
    const int m = q / kTileSys, s = q - m * kTileSys;
    const int p = m & 1, i = m >> 1;
    const int64_t j = j0 + s;
    const bool ok = j < B;
    tcp(buf + (s * 2 + p) * col + col_idx<R>(i), rhs + (int64_t)m * B + (ok ? j : 0), ok);
  }
}

template <typename V, int R>
__device__ __forceinline__ void tile_store(const V* buf, V* out, int n_modes, int64_t B, int64_t j0, int tid) {
  using O = VOps<V>;
  constexpr int col = 32 * (R + 1);
  const int pieces = n_modes * kTileSys;
  for (int q = tid; q < pieces; q += kTileThreads) {
    const int m = q / kTileSys, s = q - m * kTileSys;
    const int p = m & 1, i = m >> 1;
    const int64_t j = j0 + s;
    if (j < B) O::st_cs(out + (int64_t)m * B + j, buf[(s * 2 + p) * col + col_idx<R>(i)]);
  }
}

}  // namespace

// smem: two tile buffers, then the row table [2 parities][R][4][32] doubles.
template <typename V, int R>
__global__ void __launch_bounds__(kTileThreads, 1) helm_tile_kernel(HelmChunkArgs a) {
  extern __shared__ __align__(16) double smem[];
  constexpr int col = 32 * (R + 1);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int par = warp & 1, sys = warp >> 1;
  const int64_t B = a.batch;
  const int n_dir = a.n_dir;
  V* bufs = reinterpret_cast<V*>(smem);
  double* tab_all = smem + (size_t)2 * kTileSys * 2 * col * VOps<V>::ndouble;
  for (int idx = tid; idx < 2 * R * 32; idx += kTileThreads) {
    const int p = idx / (R * 32), rem = idx - p * R * 32, r = rem >> 5, c = rem & 31, i = c * R + r;
    const int np = (n_dir - p + 1) / 2;
    const int nsp = (n_dir - 2 - p + 1) / 2 > 0 ? (n_dir - 2 - p + 1) / 2 : 0;
    double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
    if (i < np) {
      const int k = p + 2 * i;
      v0 = __ldg(a.sd + k); v1 = __ldg(a.st + k); v2 = __ldg(a.md + k); v3 = i < nsp ? 1.0 : 0.0;
    }
    double* tab = tab_all + (size_t)p * R * 4 * 32;
    tab[(r * 4 + 0) * 32 + c] = v0;
    tab[(r * 4 + 1) * 32 + c] = v1;
    tab[(r * 4 + 2) * 32 + c] = v2;
    tab[(r * 4 + 3) * 32 + c] = v3;
  }
  const double* tab = tab_all + (size_t)par * R * 4 * 32;
  const int n = (n_dir - par + 1) / 2;
  const int s0 = lane * R;
  const int nr = max(0, min(R, n - s0));
  const bool use_ck = s0 > 0 && nr > 0;
  const V* rhs = static_cast<const V*>(a.rhs);
  V* out = static_cast<V*>(a.out);
  const int64_t ntiles = (B + kTileSys - 1) / kTileSys;
  int64_t t = blockIdx.x;
  if (t < ntiles) tile_load<V, R>(bufs, rhs, n_dir, B, t * kTileSys, tid);
  tcommit();
  int buf = 0;
  for (; t < ntiles; t += gridDim.x, buf ^= 1) {
    const int64_t tn = t + gridDim.x;
    if (tn < ntiles) tile_load<V, R>(bufs + (buf ^ 1) * kTileSys * 2 * col, rhs, n_dir, B, tn * kTileSys, tid);
    tcommit();
    twait<1>();
    __syncthreads();
    V* tile = bufs + buf * kTileSys * 2 * col;
    const int64_t j = t * kTileSys + sys;
    if (j < B) {
      V* Ys = tile + (sys * 2 + par) * col + lane * (R + 1);  // this lane's chunk: Ys[r]
      const double cb = __ldg(a.cb + j);
      const double sub = __dmul_rn(cb, -1.5707963267948966);
      HelmProj pj;
      if (use_ck) {
        const double* ck = a.ckpt + ((int64_t)(lane * 2 + par) * 3) * B + j;
        hp_start(pj, __ldg(ck), __ldg(ck + B), __ldg(ck + 2 * B));
      } else {
        hp_origin(pj);
      }
      // ---- pass 1
      double h_[R], rd_[R], e_[R], t_[R];
      V y = tzero<V>();
      double h = 1.0;
      double p00 = 1.0, p01 = 0.0, p10 = 0.0, p11 = 1.0;
      V t0a = tzero<V>(), t0b = tzero<V>();
      double t1a = 0.0, t1b = 0.0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const bool valid = r < nr;
        const HelmRow row = helm_row(a.ca, cb, sub, tab[(r * 4 + 0) * 32 + lane], tab[(r * 4 + 1) * 32 + lane],
                                     tab[(r * 4 + 2) * 32 + lane], tab[(r * 4 + 3) * 32 + lane] != 0.0);
        if (r > 0 && (r & 7) == 0) hp_rescale(pj);
        double d, e, tt;
        const double low = hp_step(pj, row, sub, d, e, tt);
        const V b = Ys[r];
        const V yv = tfma(-low, y, b);
        y = valid ? yv : tzero<V>();
        h = valid ? -low * h : h;
        const double rd = valid ? pj.rd : 0.0;
        e = valid ? e : 0.0;
        tt = valid ? tt : 0.0;
        Ys[r] = y;
        h_[r] = h; rd_[r] = rd; e_[r] = e; t_[r] = tt;
        const double al = -rd * e, be = -rd * tt;
        const V cy = tmul(rd, y);
        const double ch = rd * h;
        t0a = tfma(p00, cy, t0a);
        t0b = tfma(p10, cy, t0b);
        t1a = fma(p00, ch, t1a);
        t1b = fma(p10, ch, t1b);
        const double n00 = fma(p00, al, p01), n01 = fma(p00, be, p01);
        const double n10 = fma(p10, al, p11), n11 = fma(p10, be, p11);
        p00 = n00; p01 = n01; p10 = n10; p11 = n11;
      }
      // ---- scan F
      double m = h;
      V Y = y;
#pragma unroll
      for (int dd = 1; dd < 32; dd <<= 1) {
        const double mb = shfl_up_d(m, dd);
        const V Yb = shfl_up_v(Y, dd);
        const bool take = lane >= dd;
        const V Yn = tfma(m, Yb, Y);
        const double mn = m * mb;
        Y = take ? Yn : Y;
        m = take ? mn : m;
      }
      V E = shfl_up_v(Y, 1);
      if (lane == 0) E = tzero<V>();
      // ---- scan B
      V ta = tfma(t1a, E, t0a), tb = tfma(t1b, E, t0b);
      {
        double q00 = p00, q01 = p01, q10 = p10, q11 = p11;
#pragma unroll
        for (int dd = 1; dd < 32; dd <<= 1) {
          const double r00 = shfl_down_d(q00, dd), r01 = shfl_down_d(q01, dd);
          const double r10 = shfl_down_d(q10, dd), r11 = shfl_down_d(q11, dd);
          const V va = shfl_down_v(ta, dd), vb = shfl_down_v(tb, dd);
          const bool take = lane + dd < 32;
          const V tan = tfma(q00, va, tfma(q01, vb, ta));
          const V tbn = tfma(q10, va, tfma(q11, vb, tb));
          const double n00 = fma(q00, r00, q01 * r10), n01 = fma(q00, r01, q01 * r11);
          const double n10 = fma(q10, r00, q11 * r10), n11 = fma(q10, r01, q11 * r11);
          ta = take ? tan : ta;
          tb = take ? tbn : tb;
          q00 = take ? n00 : q00; q01 = take ? n01 : q01;
          q10 = take ? n10 : q10; q11 = take ? n11 : q11;
        }
      }
      V x1 = shfl_down_v(ta, 1), S = shfl_down_v(tb, 1);
      if (lane == 31) { x1 = tzero<V>(); S = tzero<V>(); }
      // ---- pass 3
#pragma unroll
      for (int r = R - 1; r >= 0; --r) {
        const V yy = tfma(h_[r], E, Ys[r]);
        const V acc = tsub(tsub(yy, tmul(e_[r], x1)), tmul(t_[r], S));
        const V x = tmul(rd_[r], acc);
        S = tadd(x1, S);
        x1 = x;
        Ys[r] = x;
      }
      // ---- fix
      const V da = tsub(x1, ta), db = tsub(S, tb);
      V wa = shfl_down_v(da, 1), wb = shfl_down_v(db, 1);
      if (lane == 31) { wa = tzero<V>(); wb = tzero<V>(); }
#pragma unroll
      for (int it = 0; it < SHEN_FIX_STEPS; ++it) {
        const V w1a = tfma(p00, wa, tfma(p01, wb, da)), w1b = tfma(p10, wa, tfma(p11, wb, db));
        wa = shfl_down_v(w1a, 1);
        wb = shfl_down_v(w1b, 1);
        if (lane == 31) { wa = tzero<V>(); wb = tzero<V>(); }
      }
      V xc1 = wa, Sc = wb;
#pragma unroll
      for (int r = R - 1; r >= 0; --r) {
        const V xc = tmul(-rd_[r], tfma(e_[r], xc1, tmul(t_[r], Sc)));
        Sc = tadd(xc1, Sc);
        xc1 = xc;
        Ys[r] = tadd(Ys[r], xc);
      }
    }
    __syncthreads();
    tile_store<V, R>(tile, out, n_dir, B, t * kTileSys, tid);
    __syncthreads();
  }
  twait<0>();
}

template <typename V, int R>
static cudaError_t helm_tile_R(const HelmChunkArgs& a, cudaStream_t st) {
  constexpr int col = 32 * (R + 1);
  const size_t smem = (size_t)2 * kTileSys * 2 * col * sizeof(V) + (size_t)2 * R * 4 * 32 * sizeof(double);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  auto kern = helm_tile_kernel<V, R>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kTileThreads, smem) != cudaSuccess || occ < 1) occ = 1;
  const int64_t ntiles = (a.batch + kTileSys - 1) / kTileSys;
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, (int64_t)sms * occ);
  kern<<<grid, kTileThreads, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_helm_tile(const HelmChunkArgs& a, bool cplx_rhs, cudaStream_t st) {
  if (a.batch <= 0) return cudaSuccess;
  switch (a.chunk_rows) {
#define SHEN_TILE_CASE(RR) \
  case RR: return cplx_rhs ? helm_tile_R<cplx, RR>(a, st) : helm_tile_R<double, RR>(a, st);
    SHEN_TILE_CASE(1) SHEN_TILE_CASE(2) SHEN_TILE_CASE(4) SHEN_TILE_CASE(8) SHEN_TILE_CASE(16)
#undef SHEN_TILE_CASE
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace shen
