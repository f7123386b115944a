// Column-resident (CR) fused factor+solve: the right-hand side is read from
// HBM once and the solution written once (32 B per complex unknown plus the
// build's chunk checkpoints), with the whole column of every system of a tile
// held in shared memory between the forward and the backward sweep.
//
// Tile = 8 consecutive systems x all rows of one parity (128-B row pieces),
// staged by 2-D TMA boxes into one of NSLOT shared-memory slots: the load of
// tile k+NSLOT-1 and the store of tile k-1 run while tile k is solved.  One
// persistent CTA per SM; even CTAs solve parity 0, odd CTAs parity 1.
//
// Inside a tile: 256 threads = 8 systems x 32 chunks of R consecutive rows
// (a quarter-warp is 8 systems of one chunk, so every shared-memory row
// access is one contiguous 128-B line: no bank conflicts).  Per thread:
//   pass 1  rows forward: factor rows recomputed from the chunk's checkpoint
//           (the build kernel's fast arithmetic, shen_rows.cuh), y with zero
//           entry and its homogeneous response h, and the chunk's backward
//           transfer map accumulated in forward order;
//   scan F  one warp per system, lanes = chunks (warp-shuffle scan of the
//           forward affine maps) -> the y entering every chunk;
//   scan B  the same for the backward maps -> the back-substitution state
//           entering every chunk;
//   pass 3  rows backward: the reference back-substitution
//           (solvers.py:118-125) writes x over y in the tile;
//   fix     the few-ulp difference between the state a chunk assumed and the
//           one its lower neighbour produced is propagated through 3
//           truncated neighbour steps and removed by a homogeneous sweep
//           (the arithmetic of the warp-per-system chunked solve).
// Replaces HelmholtzLU.solve (reference solvers.py:100-126).
#include <algorithm>
#include <cstring>

#include <cudaTypedefs.h>

#include "shen_kernels.h"
#include "shen_rows.cuh"
#include "shen_tma.cuh"

namespace shen {

static PFN_cuTensorMapEncodeTiled_v12000 cr_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool encode_tiled_2d(CUtensorMap* tm, const void* base, uint64_t dim0, uint64_t dim1, uint64_t stride1_bytes,
                     uint32_t box0, uint32_t box1) {
  auto enc = cr_encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)dim0, (cuuint64_t)dim1};
  const cuuint64_t strides[1] = {(cuuint64_t)stride1_bytes};
  const cuuint32_t box[2] = {box0, box1};
  const cuuint32_t es[2] = {1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

namespace {
constexpr int kS = 8;          // systems per tile
constexpr int kC = 32;         // chunks per (system, parity)
constexpr int kNT = kS * kC;   // threads per CTA
constexpr int kXq = 8;         // doubles exchanged per (system, chunk)
constexpr int kXs = kC + 1;    // padded chunk stride of the exchange buffer
#ifndef SHEN_CR_FIX_STEPS
#define SHEN_CR_FIX_STEPS 3
#endif

__device__ __forceinline__ cplx cfma(double s, cplx b, cplx a) { return {__fma_rn(s, b.re, a.re), __fma_rn(s, b.im, a.im)}; }
__device__ __forceinline__ cplx cmul(double s, cplx b) { return {s * b.re, s * b.im}; }
__device__ __forceinline__ cplx cadd(cplx a, cplx b) { return {a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ cplx csub(cplx a, cplx b) { return {a.re - b.re, a.im - b.im}; }
__device__ __forceinline__ cplx ld2(const cplx* p) {
  const double2 v = *reinterpret_cast<const double2*>(p);
  return {v.x, v.y};
}
__device__ __forceinline__ void st2(cplx* p, cplx v) { *reinterpret_cast<double2*>(p) = make_double2(v.re, v.im); }
}  // namespace

// smem: NSLOT x [rows_slot][8] cplx tiles | table [R][4][32] | exchange [8][8][33]
template <int R, int NSLOT>
__global__ void __launch_bounds__(kNT, 1)
    helm_cr_kernel(HelmChunkArgs a, const __grid_constant__ CUtensorMap in0, const __grid_constant__ CUtensorMap in1,
                   const __grid_constant__ CUtensorMap out0, const __grid_constant__ CUtensorMap out1, int box_rows,
                   int rows_slot) {
  // dynamic window only (no static shared memory in front of it), base
  // rounded up to 1024 B in the kernel: TMA boxes land 128-B aligned
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int s = tid & 7, c = (warp << 2) | (lane >> 3);
  const int par = (int)(blockIdx.x & 1);
  const int64_t B = a.batch;
  const int n = (a.n_dir - par + 1) / 2;
  const int nsup = max(0, (a.n_dir - 2 - par + 1) / 2);
  const size_t slot_elems = (size_t)rows_slot * kS;
  cplx* slots = reinterpret_cast<cplx*>(smem);
  double* tab = reinterpret_cast<double*>(smem + (size_t)NSLOT * slot_elems * sizeof(cplx));
  double* xch = tab + R * 4 * 32;
  uint64_t* bars = reinterpret_cast<uint64_t*>(xch + kXq * kS * kXs);
  auto X = [&](int q, int ss, int cc) -> double& { return xch[(q * kS + ss) * kXs + cc]; };
  for (int idx = tid; idx < R * 32; idx += kNT) {
    const int r = idx >> 5, cc = idx & 31, i = cc * R + r;
    double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
    if (i < n) {
      const int k = par + 2 * i;
      v0 = __ldg(a.sd + k); v1 = __ldg(a.st + k); v2 = __ldg(a.md + k); v3 = i < nsup ? 1.0 : 0.0;
    }
    tab[(r * 4 + 0) * 32 + cc] = v0;
    tab[(r * 4 + 1) * 32 + cc] = v1;
    tab[(r * 4 + 2) * 32 + cc] = v2;
    tab[(r * 4 + 3) * 32 + cc] = v3;
  }
  if (tid == 0) {
    for (int k = 0; k < NSLOT; ++k) mb_init(bars + k, 1);
    mb_fence_init();
  }
  __syncthreads();

  const int s0 = c * R;
  const int nr = max(0, min(R, n - s0));
  const bool use_ck = s0 > 0 && nr > 0;
  const int64_t jb = a.jb, je = a.je < 0 ? B : a.je;  // systems [jb, je); columns >= je are clipped by TMA
  const int64_t ntiles = (je - jb + kS - 1) / kS;
  const int64_t tfirst = blockIdx.x >> 1;
  const int64_t tstride = (gridDim.x + 1 - par) >> 1;
  if (tfirst >= ntiles) return;
  const CUtensorMap* mi = par ? &in1 : &in0;
  const CUtensorMap* mo = par ? &out1 : &out0;
  const int nbox = (n + box_rows - 1) / box_rows;
  const uint32_t tile_bytes = (uint32_t)nbox * (uint32_t)box_rows * kS * sizeof(cplx);
  auto issue_load = [&](int64_t t, int sl) {
    mb_expect(bars + sl, tile_bytes);
    for (int b = 0; b < nbox; ++b)
      tma_load_2d(slots + sl * slot_elems + (size_t)b * box_rows * kS, mi, (int)((jb + t * kS) * 2), b * box_rows,
                  bars + sl);
  };
  int64_t t_ld = tfirst;
  if (tid == 0)
    for (int k = 0; k < NSLOT - 1 && t_ld < ntiles; ++k, t_ld += tstride) issue_load(t_ld, k);

  // per-system scalars, loaded one tile ahead
  double cb_n = 1.0, ckd_n = 1.0, cke_n = 0.0, ckt_n = 0.0;
  auto load_scalars = [&](int64_t t) {
    const int64_t j = min(jb + t * kS + s, je - 1);
    cb_n = __ldg(a.cb + j);
    if (use_ck) {
      const double* ck = a.ckpt + ((int64_t)(c * 2 + par) * 3) * B + j;
      ckd_n = __ldg(ck); cke_n = __ldg(ck + B); ckt_n = __ldg(ck + 2 * B);
    }
  };
  load_scalars(tfirst);
  uint32_t phase = 0;
  int slot = 0;
  for (int64_t t = tfirst; t < ntiles; t += tstride) {
    const double cb = cb_n;
    HelmProj pj;
    if (use_ck) hp_start(pj, ckd_n, cke_n, ckt_n); else hp_origin(pj);
    if (t + tstride < ntiles) load_scalars(t + tstride);
    cplx* T = slots + slot * slot_elems + s;  // row i of this system: T[i * kS]
    mb_wait(bars + slot, (phase >> slot) & 1u);
    phase ^= 1u << slot;
    const double sub = __dmul_rn(cb, -1.5707963267948966);

    // ---- pass 1
    double h_[R], rd_[R], e_[R], t_[R];
    cplx y = {0.0, 0.0};
    double h = 1.0;
    double p00 = 1.0, p01 = 0.0, p10 = 0.0, p11 = 1.0;
    cplx t0a = {0.0, 0.0}, t0b = {0.0, 0.0};
    double t1a = 0.0, t1b = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const bool valid = r < nr;
      const HelmRow row = helm_row(a.ca, cb, sub, tab[(r * 4 + 0) * 32 + c], tab[(r * 4 + 1) * 32 + c],
                                   tab[(r * 4 + 2) * 32 + c], tab[(r * 4 + 3) * 32 + c] != 0.0);
      if (r > 0 && (r & 7) == 0) hp_rescale(pj);
      double d, e, tt;
      const double low = hp_step(pj, row, sub, d, e, tt);
      cplx* pr = T + (size_t)(s0 + r) * kS;
      const cplx b = valid ? ld2(pr) : cplx{0.0, 0.0};
      const cplx yv = cfma(-low, y, b);
      y = valid ? yv : cplx{0.0, 0.0};
      h = valid ? -low * h : h;
      const double rd = valid ? pj.rd : 0.0;
      e = valid ? e : 0.0;
      tt = valid ? tt : 0.0;
      if (valid) st2(pr, y);
      h_[r] = h; rd_[r] = rd; e_[r] = e; t_[r] = tt;
      const double al = -rd * e, be = -rd * tt;
      const cplx cy = cmul(rd, y);
      const double ch = rd * h;
      t0a = cfma(p00, cy, t0a);
      t0b = cfma(p10, cy, t0b);
      t1a = fma(p00, ch, t1a);
      t1b = fma(p10, ch, t1b);
      const double n00 = fma(p00, al, p01), n01 = fma(p00, be, p01);
      const double n10 = fma(p10, al, p11), n11 = fma(p10, be, p11);
      p00 = n00; p01 = n01; p10 = n10; p11 = n11;
    }
    X(0, s, c) = h;
    X(1, s, c) = y.re;
    X(2, s, c) = y.im;
    __syncthreads();
    // refill the slot the previous tile was stored from
    if (tid == 0 && t_ld < ntiles) {
      bulk_wait_read0();
      issue_load(t_ld, slot == 0 ? NSLOT - 1 : slot - 1);
      t_ld += tstride;
    }

    // ---- scan F (warp w = system w, lanes = chunks): exit_c = Y_c + m_c exit_{c-1}
    {
      double m = X(0, warp, lane);
      cplx Y = {X(1, warp, lane), X(2, warp, lane)};
#pragma unroll
      for (int dd = 1; dd < 32; dd <<= 1) {
        const double mb = shfl_up_d(m, dd);
        const cplx Yb = shfl_up_v(Y, dd);
        const bool take = lane >= dd;
        const cplx Yn = cfma(m, Yb, Y);
        const double mn = m * mb;
        Y = take ? Yn : Y;
        m = take ? mn : m;
      }
      cplx E = shfl_up_v(Y, 1);
      if (lane == 0) E = {0.0, 0.0};
      X(3, warp, lane) = E.re;
      X(4, warp, lane) = E.im;
    }
    __syncthreads();
    const cplx E = {X(3, s, c), X(4, s, c)};
    const cplx ta0 = cfma(t1a, E, t0a), tb0 = cfma(t1b, E, t0b);
    X(0, s, c) = p00; X(1, s, c) = p01; X(2, s, c) = p10; X(3, s, c) = p11;
    X(4, s, c) = ta0.re; X(5, s, c) = ta0.im; X(6, s, c) = tb0.re; X(7, s, c) = tb0.im;
    __syncthreads();
    // ---- scan B: sigma_c = P_c sigma_{c+1} + tau_c (suffix over chunks)
    {
      double q00 = X(0, warp, lane), q01 = X(1, warp, lane), q10 = X(2, warp, lane), q11 = X(3, warp, lane);
      cplx ta = {X(4, warp, lane), X(5, warp, lane)}, tb = {X(6, warp, lane), X(7, warp, lane)};
#pragma unroll
      for (int dd = 1; dd < 32; dd <<= 1) {
        const double r00 = shfl_down_d(q00, dd), r01 = shfl_down_d(q01, dd);
        const double r10 = shfl_down_d(q10, dd), r11 = shfl_down_d(q11, dd);
        const cplx va = shfl_down_v(ta, dd), vb = shfl_down_v(tb, dd);
        const bool take = lane + dd < 32;
        const cplx tan = cfma(q00, va, cfma(q01, vb, ta));
        const cplx tbn = cfma(q10, va, cfma(q11, vb, tb));
        const double n00 = fma(q00, r00, q01 * r10), n01 = fma(q00, r01, q01 * r11);
        const double n10 = fma(q10, r00, q11 * r10), n11 = fma(q10, r01, q11 * r11);
        ta = take ? tan : ta;
        tb = take ? tbn : tb;
        q00 = take ? n00 : q00; q01 = take ? n01 : q01;
        q10 = take ? n10 : q10; q11 = take ? n11 : q11;
      }
      cplx x1 = shfl_down_v(ta, 1), S = shfl_down_v(tb, 1);
      if (lane == 31) { x1 = {0.0, 0.0}; S = {0.0, 0.0}; }
      X(0, warp, lane) = ta.re; X(1, warp, lane) = ta.im; X(2, warp, lane) = tb.re; X(3, warp, lane) = tb.im;
      X(4, warp, lane) = x1.re; X(5, warp, lane) = x1.im; X(6, warp, lane) = S.re; X(7, warp, lane) = S.im;
    }
    __syncthreads();
    const cplx ta = {X(0, s, c), X(1, s, c)}, tb = {X(2, s, c), X(3, s, c)};
    cplx x1 = {X(4, s, c), X(5, s, c)}, S = {X(6, s, c), X(7, s, c)};

    // ---- pass 3: back-substitution over the chunk (x overwrites y in the tile)
#pragma unroll
    for (int r = R - 1; r >= 0; --r) {
      cplx* pr = T + (size_t)(s0 + r) * kS;
      const cplx yv = r < nr ? ld2(pr) : cplx{0.0, 0.0};
      const cplx yy = cfma(h_[r], E, yv);
      const cplx acc = csub(csub(yy, cmul(e_[r], x1)), cmul(t_[r], S));
      const cplx x = cmul(rd_[r], acc);
      S = cadd(x1, S);
      x1 = x;
      if (r < nr) st2(pr, x);
    }
    // ---- fix: w_c = d_{c+1} + P_{c+1} (d_{c+2} + P_{c+2} (... d_{c+1+FIX})), own (unscanned) P
    const cplx da = csub(x1, ta), db = csub(S, tb);
    X(0, s, c) = da.re; X(1, s, c) = da.im; X(2, s, c) = db.re; X(3, s, c) = db.im;
    X(4, s, c) = p00; X(5, s, c) = p01; X(6, s, c) = p10; X(7, s, c) = p11;
    __syncthreads();
    cplx wa = {0.0, 0.0}, wb = {0.0, 0.0};
#pragma unroll
    for (int k = SHEN_CR_FIX_STEPS + 1; k >= 1; --k) {
      const int cc = c + k;
      if (cc < kC) {
        const cplx ua = {X(0, s, cc), X(1, s, cc)}, ub = {X(2, s, cc), X(3, s, cc)};
        if (k == SHEN_CR_FIX_STEPS + 1) {
          wa = ua;
          wb = ub;
        } else {
          const double m00 = X(4, s, cc), m01 = X(5, s, cc), m10 = X(6, s, cc), m11 = X(7, s, cc);
          const cplx na = cfma(m00, wa, cfma(m01, wb, ua));
          const cplx nb = cfma(m10, wa, cfma(m11, wb, ub));
          wa = na;
          wb = nb;
        }
      }
    }
    cplx xc1 = wa, Sc = wb;
#pragma unroll
    for (int r = R - 1; r >= 0; --r) {
      const cplx xc = cmul(-rd_[r], cfma(e_[r], xc1, cmul(t_[r], Sc)));
      Sc = cadd(xc1, Sc);
      xc1 = xc;
      if (r < nr) {
        cplx* pr = T + (size_t)(s0 + r) * kS;
        st2(pr, cadd(ld2(pr), xc));
      }
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      const cplx* base = slots + slot * slot_elems;
      for (int b = 0; b < nbox; ++b)
        tma_store_2d(mo, (int)((jb + t * kS) * 2), b * box_rows, base + (size_t)b * box_rows * kS);
      bulk_commit();
    }
    slot = slot + 1 == NSLOT ? 0 : slot + 1;
  }
  if (tid == 0) bulk_wait0();
}

// rows of a TMA box: the fewest boxes of <= 256 rows covering n0 rows, rounded to 8
static int cr_box_rows(int n0) {
  const int nb = (n0 + 255) / 256;
  const int br = (n0 + nb - 1) / nb;
  return std::min(256, (br + 7) & ~7);
}

size_t helm_cr_smem(int n_dir, int chunk_rows, int nslot) {
  const int n0 = (n_dir + 1) / 2;
  const int br = cr_box_rows(n0);
  const int rows_slot = ((n0 + br - 1) / br) * br;
  return (size_t)nslot * rows_slot * kS * sizeof(cplx) + (size_t)chunk_rows * 4 * 32 * sizeof(double) +
         (size_t)kXq * kS * kXs * sizeof(double) + (size_t)nslot * sizeof(uint64_t) + 1024;  // + base alignment
}

template <int R, int NSLOT>
static cudaError_t helm_cr_RR(const HelmChunkArgs& a, cudaStream_t st) {
  const int n0 = (a.n_dir + 1) / 2, n1 = a.n_dir / 2;
  const int br = cr_box_rows(n0);
  const int rows_slot = ((n0 + br - 1) / br) * br;
  const size_t smem = helm_cr_smem(a.n_dir, R, NSLOT);
  CUtensorMap m[4];
  const uint64_t pitch = (uint64_t)a.batch * sizeof(cplx);
  const int64_t je = a.je < 0 ? a.batch : a.je;
  if (je <= a.jb) return cudaSuccess;
  const char* rin = static_cast<const char*>(a.rhs);
  const char* rout = static_cast<const char*>(a.out);
  // parity p: rows p, p + 2, ... -> a 2-D tensor (2 batch doubles, rows_p) with a 2-row stride
  // (the tensor ends at column je: a partial last tile is zero-filled on load and clipped on store)
  if (!encode_tiled_2d(m + 0, rin, 2 * je, n0, 2 * pitch, 2 * kS, br) ||
      (n1 > 0 && !encode_tiled_2d(m + 1, rin + pitch, 2 * je, n1, 2 * pitch, 2 * kS, br)) ||
      !encode_tiled_2d(m + 2, rout, 2 * je, n0, 2 * pitch, 2 * kS, br) ||
      (n1 > 0 && !encode_tiled_2d(m + 3, rout + pitch, 2 * je, n1, 2 * pitch, 2 * kS, br)))
    return cudaErrorNotSupported;
  if (n1 == 0) {
    m[1] = m[0];
    m[3] = m[2];
  }
  auto kern = helm_cr_kernel<R, NSLOT>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t ntiles = (je - a.jb + kS - 1) / kS;
  int64_t grid = std::min<int64_t>((int64_t)sms, 2 * ntiles);
  if (a.max_ctas > 0) grid = std::min<int64_t>(grid, a.max_ctas);
  grid = std::max<int64_t>(grid, n1 > 0 ? 2 : 1);  // parity = blockIdx.x & 1: both must exist
  if (n1 == 0) grid = 1;
  kern<<<(unsigned)grid, kNT, smem, st>>>(a, m[0], m[1], m[2], m[3], br, rows_slot);
  return cudaGetLastError();
}

template <int R>
static cudaError_t helm_cr_R(const HelmChunkArgs& a, cudaStream_t st) {
  if (helm_cr_smem(a.n_dir, R, 3) <= 227 * 1024) return helm_cr_RR<R, 3>(a, st);
  if (helm_cr_smem(a.n_dir, R, 2) <= 227 * 1024) return helm_cr_RR<R, 2>(a, st);
  return cudaErrorInvalidValue;
}

// complex RHS only; ckpt from shen_helm_factor with chunk_rows = R, 32 R >= rows of parity 0
cudaError_t launch_helm_cr(const HelmChunkArgs& a, cudaStream_t st) {
  if (a.batch <= 0) return cudaSuccess;
  if ((int64_t)a.chunk_rows * kC < (a.n_dir + 1) / 2) return cudaErrorInvalidValue;
  if ((reinterpret_cast<uintptr_t>(a.rhs) | reinterpret_cast<uintptr_t>(a.out)) & 15) return cudaErrorInvalidValue;
  switch (a.chunk_rows) {
    case 1: return helm_cr_R<1>(a, st);
    case 2: return helm_cr_R<2>(a, st);
    case 4: return helm_cr_R<4>(a, st);
    case 8: return helm_cr_R<8>(a, st);
    case 16: return helm_cr_R<16>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace shen
