// extern "C" boundary: argument validation, stream plumbing, error text.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/shen_b200.h"
#include "shen_kernels.h"
#include "shen_rows.cuh"

static_assert(SHEN_BIH_NCOL == shen::B_STRIDE, "table pitch mismatch");
static_assert(sizeof(shen_wall_plan) == sizeof(shen::WallPlan), "wall plan layout mismatch");

namespace {
thread_local std::string g_err;

int fail(int code, const char* what) {
  g_err = what;
  return code;
}
int cuda_check(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return SHEN_OK;
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return SHEN_ERR_CUDA;
}
cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

__global__ void fill_int_kernel(int* p, int n, int v) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}
}  // namespace

extern "C" {

const char* shen_version(void) { return "shen_b200 0.1 (sm_100a)"; }

const char* shen_last_error(void) { return g_err.c_str(); }

int shen_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int64_t shen_stream_scratch_bytes(int op, int n_modes, int chunk_rows, int64_t batch, int is_complex) {
  if (chunk_rows <= 0 || n_modes < 2 || batch < 0) return -1;
  return shen::stream_scratch_bytes(op, n_modes, chunk_rows, is_complex != 0);
}

int shen_memcpy2d_async(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width_bytes,
                        int64_t height, int kind, void* stream) {
  if (height == 0 || width_bytes == 0) return SHEN_OK;
  if (!dst || !src || width_bytes < 0 || height < 0 || kind < 0 || kind > 2)
    return fail(SHEN_ERR_ARG, "shen_memcpy2d_async: bad args");
  const cudaMemcpyKind k = kind == 0 ? cudaMemcpyHostToDevice : (kind == 1 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice);
  return cuda_check(cudaMemcpy2DAsync(dst, (size_t)dpitch, src, (size_t)spitch, (size_t)width_bytes, (size_t)height, k,
                                      S(stream)),
                    "shen_memcpy2d_async");
}

int shen_pivot_reset(int* pivot_dev, void* stream) {
  if (!pivot_dev) return fail(SHEN_ERR_ARG, "pivot_dev is NULL");
  fill_int_kernel<<<1, 32, 0, S(stream)>>>(pivot_dev, 2, INT_MAX);
  return cuda_check(cudaGetLastError(), "shen_pivot_reset");
}

int shen_helm_factor(int n_dir, double ca, const double* cb, int64_t batch, const double* sd, const double* st,
                     const double* md, int chunk_rows, double* ckpt, double* const* factors, int exact,
                     int* pivot_dev, void* stream) {
  if (batch == 0) return SHEN_OK;
  if (n_dir < 2 || batch < 0 || !cb || !sd || !st || !md) return fail(SHEN_ERR_ARG, "shen_helm_factor: bad args");
  if (ckpt && chunk_rows <= 0) return fail(SHEN_ERR_ARG, "shen_helm_factor: ckpt needs chunk_rows > 0");
  shen::HelmFactorArgs a{};
  a.n_dir = n_dir; a.ca = ca; a.cb = cb; a.batch = batch; a.sd = sd; a.st = st; a.md = md;
  a.chunk_rows = chunk_rows; a.ckpt = ckpt; a.pivot = pivot_dev;
  for (int p = 0; p < 2; ++p) {
    a.low[p] = factors ? factors[0 + p] : nullptr;
    a.d[p] = factors ? factors[2 + p] : nullptr;
    a.e[p] = factors ? factors[4 + p] : nullptr;
    a.t[p] = factors ? factors[6 + p] : nullptr;
    if (factors && (!a.d[p] || !a.e[p] || !a.t[p])) return fail(SHEN_ERR_ARG, "shen_helm_factor: null factor");
  }
  return cuda_check(shen::launch_helm_factor(a, exact != 0, S(stream)), "shen_helm_factor");
}

int shen_wall_transform(const shen_wall_plan* plan, int64_t L, const void* in, void* out, void* stream) {
  if (!plan) return fail(SHEN_ERR_ARG, "shen_wall_transform: plan");
  if (L == 0) return SHEN_OK;
  const shen::WallPlan& p = *reinterpret_cast<const shen::WallPlan*>(plan);
  if (L < 0 || !in || !out || in == out || p.N < 2 || p.M < 2 || (p.M & (p.M - 1)) || p.nstage < 1 || p.nstage > 4 ||
      !p.tw || p.log2_lines < 0 || p.log2_lines > 4 || p.rows_smem < p.N || p.rows_smem < p.M)
    return fail(SHEN_ERR_ARG, "shen_wall_transform: bad args");
  if ((p.kind == 1 && (!p.ker_f || !p.ker_i || !p.gin_f || !p.gin_i || !p.gout)) ||
      (p.kind == 2 && (!p.ker_f || !p.ker_i || !p.chirp_f || !p.chirp_i)) || (p.kind == 0 && !p.pinv) ||
      (p.family == 0 && !p.mk) || (p.space == 2 && (!p.c2 || !p.c4)) || (p.mass && !p.mfac))
    return fail(SHEN_ERR_ARG, "shen_wall_transform: missing table");
  return cuda_check(shen::launch_wall(p, L, in, out, S(stream)), "shen_wall_transform");
}

int64_t shen_wall_smem_bytes(const shen_wall_plan* plan) {
  if (!plan) return -1;
  return (int64_t)shen::wall_smem_bytes(*reinterpret_cast<const shen::WallPlan*>(plan));
}

int shen_helm_solve_stream(int n_dir, double ca, const double* cb, int64_t batch, const double* sd,
                           const double* st, const double* md, int chunk_rows, const double* ckpt, const void* rhs,
                           void* out, void* scratch, int is_complex, int warps_per_sm, int max_ctas,
                           int64_t j_begin, int64_t j_end, void* stream) {
  if (batch == 0) return SHEN_OK;
  if (n_dir < 2 || batch < 0 || !cb || !sd || !st || !md || !rhs || !out)
    return fail(SHEN_ERR_ARG, "shen_helm_solve_stream: bad args");
  const int rows0 = (n_dir + 1) / 2;
  if (chunk_rows != 8) return fail(SHEN_ERR_ARG, "shen_helm_solve_stream: chunk_rows (8)");
  if (rows0 > chunk_rows && !ckpt) return fail(SHEN_ERR_ARG, "shen_helm_solve_stream: ckpt required");
  if (rhs == out) return fail(SHEN_ERR_ARG, "shen_helm_solve_stream: rhs must not alias out");
  if (rows0 > chunk_rows && !scratch) return fail(SHEN_ERR_ARG, "shen_helm_solve_stream: scratch required");
  if (j_end < 0) j_end = batch;
  if (j_begin < 0 || j_begin > j_end || j_end > batch) return fail(SHEN_ERR_ARG, "shen_helm_solve_stream: range");
  if (max_ctas < 0) return fail(SHEN_ERR_ARG, "shen_helm_solve_stream: max_ctas");
  shen::HelmChunkArgs a{n_dir, ca, cb, batch, sd, st, md, chunk_rows, ckpt, rhs, out, j_begin, j_end, max_ctas};
  return cuda_check(shen::launch_helm_stream(a, scratch, is_complex != 0, warps_per_sm, S(stream)),
                    "shen_helm_solve_stream");
}

int shen_helm_solve_stored(int n_dir, int64_t batch, const double* const* factors, const void* rhs, void* out,
                           int is_complex, void* stream) {
  if (batch == 0) return SHEN_OK;
  if (n_dir < 2 || batch < 0 || !factors || !rhs || !out) return fail(SHEN_ERR_ARG, "shen_helm_solve_stored: bad args");
  shen::HelmSeqArgs a{};
  a.n_dir = n_dir; a.batch = batch; a.rhs = rhs; a.out = out;
  for (int p = 0; p < 2; ++p) {
    a.low[p] = factors[0 + p]; a.d[p] = factors[2 + p]; a.e[p] = factors[4 + p]; a.t[p] = factors[6 + p];
  }
  return cuda_check(shen::launch_helm_seq(a, is_complex != 0, S(stream)), "shen_helm_solve_stored");
}

int shen_bih_factor(int n_bih, double xi0, const double* xi1, const double* xi2, int64_t batch,
                    const double* tab, int chunk_rows, double* ckpt, double* const* factors, int exact,
                    int* pivot_dev, void* stream) {
  if (batch == 0) return SHEN_OK;
  if (n_bih < 2 || batch < 0 || !xi1 || !xi2 || !tab) return fail(SHEN_ERR_ARG, "shen_bih_factor: bad args");
  if (ckpt && chunk_rows <= 0) return fail(SHEN_ERR_ARG, "shen_bih_factor: ckpt needs chunk_rows > 0");
  shen::BihFactorArgs a{};
  a.n_bih = n_bih; a.xi0 = xi0; a.xi1 = xi1; a.xi2 = xi2; a.batch = batch; a.tab = tab;
  a.chunk_rows = chunk_rows; a.ckpt = ckpt; a.pivot = pivot_dev;
  for (int p = 0; p < 2; ++p) {
    a.low2[p] = factors ? factors[0 + p] : nullptr;
    a.low4[p] = factors ? factors[2 + p] : nullptr;
    a.d[p] = factors ? factors[4 + p] : nullptr;
    a.e[p] = factors ? factors[6 + p] : nullptr;
    a.f[p] = factors ? factors[8 + p] : nullptr;
    a.a[p] = factors ? factors[10 + p] : nullptr;
    a.b[p] = factors ? factors[12 + p] : nullptr;
  }
  return cuda_check(shen::launch_bih_factor(a, exact != 0, S(stream)), "shen_bih_factor");
}

int shen_bih_solve_stream(int n_bih, double xi0, const double* xi1, const double* xi2, int64_t batch,
                          const double* tab, int chunk_rows, const double* ckpt, const void* rhs, void* out,
                          void* scratch, int is_complex, int warps_per_sm, int max_ctas, int64_t j_begin,
                          int64_t j_end, void* stream) {
  if (batch == 0) return SHEN_OK;
  if (n_bih < 2 || batch < 0 || !xi1 || !xi2 || !tab || !rhs || !out)
    return fail(SHEN_ERR_ARG, "shen_bih_solve_stream: bad args");
  const int rows0 = (n_bih + 1) / 2;
  if (chunk_rows != 8) return fail(SHEN_ERR_ARG, "shen_bih_solve_stream: chunk_rows (8)");
  if (rows0 > chunk_rows && !ckpt) return fail(SHEN_ERR_ARG, "shen_bih_solve_stream: ckpt required");
  if (rhs == out) return fail(SHEN_ERR_ARG, "shen_bih_solve_stream: rhs must not alias out");
  if (rows0 > chunk_rows && !scratch) return fail(SHEN_ERR_ARG, "shen_bih_solve_stream: scratch required");
  if (j_end < 0) j_end = batch;
  if (j_begin < 0 || j_begin > j_end || j_end > batch) return fail(SHEN_ERR_ARG, "shen_bih_solve_stream: range");
  if (max_ctas < 0) return fail(SHEN_ERR_ARG, "shen_bih_solve_stream: max_ctas");
  shen::BihChunkArgs a{n_bih, xi0, xi1, xi2, batch, tab, chunk_rows, ckpt, rhs, out, j_begin, j_end, max_ctas};
  return cuda_check(shen::launch_bih_stream(a, scratch, is_complex != 0, warps_per_sm, S(stream)),
                    "shen_bih_solve_stream");
}

int shen_bih_solve_stream_pairs(int n_bih, double xi0, const double* xi1, const double* xi2, int64_t batch,
                                const double* tab, int chunk_rows, const double* ckpt, const void* rhs, void* out,
                                void* scratch, int is_complex, const int64_t* pairs, int64_t n_pairs, int max_ctas,
                                void* stream) {
  if (batch == 0 || n_pairs == 0) return SHEN_OK;
  if (n_bih < 2 || batch < 0 || n_pairs < 0 || n_pairs > batch || !xi1 || !xi2 || !tab || !rhs || !out || !pairs)
    return fail(SHEN_ERR_ARG, "shen_bih_solve_stream_pairs: bad args");
  const int rows0 = (n_bih + 1) / 2;
  if (chunk_rows != 8) return fail(SHEN_ERR_ARG, "shen_bih_solve_stream_pairs: chunk_rows (8)");
  if (rows0 > chunk_rows && (!ckpt || !scratch)) return fail(SHEN_ERR_ARG, "shen_bih_solve_stream_pairs: ckpt/scratch");
  if (rhs == out) return fail(SHEN_ERR_ARG, "shen_bih_solve_stream_pairs: rhs must not alias out");
  if (max_ctas < 0) return fail(SHEN_ERR_ARG, "shen_bih_solve_stream_pairs: max_ctas");
  shen::BihChunkArgs a{n_bih, xi0, xi1, xi2, batch, tab, chunk_rows, ckpt, rhs, out, 0, -1, max_ctas};
  a.pairs = pairs;
  a.n_pairs = n_pairs;
  return cuda_check(shen::launch_bih_stream(a, scratch, is_complex != 0, 8, S(stream)), "shen_bih_solve_stream_pairs");
}

int shen_bih_solve_stored(int n_bih, int64_t batch, double xi0, const double* q, const double* s,
                          const double* const* factors, const void* rhs, void* out, int is_complex,
                          void* stream) {
  if (batch == 0) return SHEN_OK;
  if (n_bih < 2 || batch < 0 || !q || !s || !factors || !rhs || !out)
    return fail(SHEN_ERR_ARG, "shen_bih_solve_stored: bad args");
  shen::BihSeqArgs a{};
  a.n_bih = n_bih; a.batch = batch; a.xi0 = xi0; a.q = q; a.s = s; a.rhs = rhs; a.out = out;
  for (int p = 0; p < 2; ++p) {
    a.low2[p] = factors[0 + p]; a.low4[p] = factors[2 + p]; a.d[p] = factors[4 + p]; a.e[p] = factors[6 + p];
    a.f[p] = factors[8 + p]; a.a[p] = factors[10 + p]; a.b[p] = factors[12 + p];
  }
  return cuda_check(shen::launch_bih_seq(a, is_complex != 0, S(stream)), "shen_bih_solve_stored");
}

int shen_xform_extend(int family, int N, int64_t L, const void* x, void* e, void* stream) {
  if (L == 0) return SHEN_OK;
  if ((family != 0 && family != 1) || N < 2 || L < 0 || !x || !e) return fail(SHEN_ERR_ARG, "shen_xform_extend: bad args");
  return cuda_check(shen::launch_xf_extend(family, N, L, x, e, S(stream)), "shen_xform_extend");
}

int shen_xform_fwd_post(int family, int space, int N, int64_t L, double scale, const void* tw, const void* Y,
                        void* out, void* stream) {
  if (L == 0) return SHEN_OK;
  if ((family != 0 && family != 1) || space < 0 || space > 3 || N < (space == 2 ? 5 : space == 1 ? 3 : 2) || L < 0 ||
      !Y || !out ||
      (family == 0 && !tw))
    return fail(SHEN_ERR_ARG, "shen_xform_fwd_post: bad args");
  return cuda_check(shen::launch_xf_fwd_post(family, space, N, L, scale, tw, Y, out, S(stream)), "shen_xform_fwd_post");
}

int shen_xform_inv_pre(int family, int space, int n, int N, int64_t L, const void* tw, const void* coef, void* Z,
                       void* cends, void* stream) {
  if (L == 0) return SHEN_OK;
  if (family < 0 || family > 2 || space < 0 || space > 2 || N < 2 || n < 1 ||
      n + (space == 2 ? 4 : space == 1 ? 2 : 0) > N || L < 0 || !coef || !Z || (family != 2 && !cends) ||
      (family == 0 && !tw))
    return fail(SHEN_ERR_ARG, "shen_xform_inv_pre: bad args");
  return cuda_check(shen::launch_xf_inv_pre(family, space, n, N, L, tw, coef, Z, cends, S(stream)), "shen_xform_inv_pre");
}

int shen_xform_inv_post(int family, int N, int64_t L, const void* F, const void* cends, void* out, void* stream) {
  if (L == 0) return SHEN_OK;
  if ((family != 0 && family != 1) || N < 2 || L < 0 || !F || !cends || !out)
    return fail(SHEN_ERR_ARG, "shen_xform_inv_post: bad args");
  return cuda_check(shen::launch_xf_inv_post(family, N, L, F, cends, out, S(stream)), "shen_xform_inv_post");
}

int shen_xform_mass_solve(int nband, int n, int mmax, int64_t L, const double* fac, const void* s, void* x,
                          void* stream) {
  if (L == 0) return SHEN_OK;
  if ((nband != 1 && nband != 2) || n < 2 || mmax < (n + 1) / 2 || L < 0 || !fac || !s || !x)
    return fail(SHEN_ERR_ARG, "shen_xform_mass_solve: bad args");
  return cuda_check(shen::launch_xf_mass(nband, n, mmax, L, fac, s, x, S(stream)), "shen_xform_mass_solve");
}

int shen_apply_banded(int nr, int nc, int64_t L, int n_off, const int* offsets, const double* diag, const void* x,
                      void* y, int is_complex, void* stream) {
  if (L == 0 || nr == 0) return SHEN_OK;
  if (nr < 0 || nc <= 0 || L < 0 || n_off < 0 || n_off > 6 || (n_off > 0 && (!offsets || !diag)) || !x || !y)
    return fail(SHEN_ERR_ARG, "shen_apply_banded: bad args");
  return cuda_check(shen::launch_apply(0, nr, nc, L, n_off, offsets, diag, nullptr, 0, nullptr, nullptr, nullptr,
                                       nullptr, nullptr, x, y, is_complex != 0, S(stream)),
                    "shen_apply_banded");
}

int shen_apply_const_tail(int nr, int nc, int64_t L, int n_off, const int* offsets, const double* diag,
                          const double* tail, int tail_start, const void* x, void* y, int is_complex, void* stream) {
  if (L == 0 || nr == 0) return SHEN_OK;
  if (nr < 0 || nc <= 0 || L < 0 || n_off < 0 || n_off > 6 || (n_off > 0 && (!offsets || !diag)) || !tail ||
      tail_start < 0 || !x || !y)
    return fail(SHEN_ERR_ARG, "shen_apply_const_tail: bad args");
  return cuda_check(shen::launch_apply(1, nr, nc, L, n_off, offsets, diag, tail, tail_start, nullptr, nullptr,
                                       nullptr, nullptr, nullptr, x, y, is_complex != 0, S(stream)),
                    "shen_apply_const_tail");
}

int shen_apply_rank2_tail(int n, int64_t L, const double* diag, const double* p, const double* q, const double* r,
                          const double* s, const void* x, void* y, int is_complex, void* stream) {
  if (L == 0 || n == 0) return SHEN_OK;
  if (n < 0 || L < 0 || !diag || !p || !q || !r || !s || !x || !y)
    return fail(SHEN_ERR_ARG, "shen_apply_rank2_tail: bad args");
  return cuda_check(shen::launch_apply(2, n, n, L, 0, nullptr, nullptr, nullptr, 0, diag, p, q, r, s, x, y,
                                       is_complex != 0, S(stream)),
                    "shen_apply_rank2_tail");
}

static bool band_ok(const shen_band& b) { return b.nr >= 0 && b.nc > 0 && b.n_off >= 0 && b.n_off <= 6 && (b.n_off == 0 || b.diag); }
static shen::RhsBand to_band(const shen_band& b) {
  shen::RhsBand o{};
  o.nr = b.nr; o.nc = b.nc; o.n_off = b.n_off; o.diag = b.diag;
  for (int i = 0; i < 6; ++i) o.off[i] = b.off[i];
  return o;
}

int shen_rhs_g(const shen_rhs_g_args* g, void* stream) {
  if (!g) return fail(SHEN_ERR_ARG, "shen_rhs_g: NULL args");
  if (g->L == 0 || g->n_dir == 0) return SHEN_OK;
  if (g->n_dir < 0 || g->L < 0 || !band_ok(g->stiff) || !band_ok(g->mass) || !g->tail || !g->cg || !g->im_m_re ||
      !g->im_m_im || !g->im_n_re || !g->im_n_im || !g->g || !g->hcy || !g->hpy || !g->hcz || !g->hpz || !g->out ||
      g->stiff.nr != g->n_dir || g->mass.nr != g->n_dir)
    return fail(SHEN_ERR_ARG, "shen_rhs_g: bad args");
  shen::RhsGArgs a{};
  a.n_dir = g->n_dir; a.L = g->L; a.stiff = to_band(g->stiff); a.mass = to_band(g->mass);
  a.tail = g->tail; a.tail_start = g->tail_start; a.c_stiff = g->c_stiff; a.dt = g->dt; a.cg = g->cg;
  a.im_m_re = g->im_m_re; a.im_m_im = g->im_m_im; a.im_n_re = g->im_n_re; a.im_n_im = g->im_n_im;
  a.g = g->g; a.hcy = g->hcy; a.hpy = g->hpy; a.hcz = g->hcz; a.hpz = g->hpz; a.out = g->out;
  return cuda_check(shen::launch_rhs_g(a, S(stream)), "shen_rhs_g");
}

int shen_rhs_u(const shen_rhs_u_args* u, void* stream) {
  if (!u) return fail(SHEN_ERR_ARG, "shen_rhs_u: NULL args");
  if (u->L == 0 || u->n_bih == 0) return SHEN_OK;
  if (u->n_bih < 0 || u->L < 0 || !u->d || !u->p || !u->q || !u->r || !u->s || !band_ok(u->stiff) ||
      !band_ok(u->mass) || !band_ok(u->mixed) || !band_ok(u->deriv) || !u->c_stiff || !u->c_mass || !u->c_mixed ||
      !u->c_dy_re || !u->c_dy_im || !u->c_dz_re || !u->c_dz_im || !u->u || !u->hcx || !u->hpx || !u->hcy ||
      !u->hpy || !u->hcz || !u->hpz || !u->out)
    return fail(SHEN_ERR_ARG, "shen_rhs_u: bad args");
  shen::RhsUArgs a{};
  a.n_bih = u->n_bih; a.L = u->L; a.d = u->d; a.p = u->p; a.q = u->q; a.r = u->r; a.s = u->s;
  a.c_fourth = u->c_fourth; a.stiff = to_band(u->stiff); a.mass = to_band(u->mass); a.mixed = to_band(u->mixed);
  a.deriv = to_band(u->deriv); a.c_stiff = u->c_stiff; a.c_mass = u->c_mass; a.c_mixed = u->c_mixed;
  a.c_dy_re = u->c_dy_re; a.c_dy_im = u->c_dy_im; a.c_dz_re = u->c_dz_re; a.c_dz_im = u->c_dz_im;
  a.u = u->u; a.hcx = u->hcx; a.hpx = u->hpx; a.hcy = u->hcy; a.hpy = u->hpy; a.hcz = u->hcz; a.hpz = u->hpz;
  a.out = u->out;
  return cuda_check(shen::launch_rhs_u(a, S(stream)), "shen_rhs_u");
}

int shen_cross(int64_t n, const double* fields, double* h, void* stream) {
  if (n == 0) return SHEN_OK;
  if (n < 0 || !fields || !h) return fail(SHEN_ERR_ARG, "shen_cross: bad args");
  return cuda_check(shen::launch_cross(n, fields, h, S(stream)), "shen_cross");
}

int shen_plane_fft_supported(int n_y, int n_z) { return shen::plane_fft_supported(n_y, n_z) ? 1 : 0; }

int shen_plane_rfft2(int64_t n_planes, int n_y, int n_z, const double* x, void* X, void* stream) {
  if (n_planes == 0) return SHEN_OK;
  if (n_planes < 0 || !x || !X || !shen::plane_fft_supported(n_y, n_z) || (reinterpret_cast<uintptr_t>(x) & 7) ||
      (reinterpret_cast<uintptr_t>(X) & 15))
    return fail(SHEN_ERR_ARG, "shen_plane_rfft2: bad args (sizes: shen_plane_fft_supported; x 8-B, X 16-B aligned)");
  return cuda_check(shen::launch_plane_rfft2(n_planes, n_y, n_z, x, X, nullptr, S(stream)), "shen_plane_rfft2");
}

int shen_plane_rfft2_fac(int64_t n_planes, int n_y, int n_z, const double* x, void* X, const double* fac,
                         void* stream) {
  if (n_planes == 0) return SHEN_OK;
  if (n_planes < 0 || !x || !X || !fac || !shen::plane_fft_supported(n_y, n_z) ||
      (reinterpret_cast<uintptr_t>(x) & 7) || (reinterpret_cast<uintptr_t>(X) & 15) ||
      (reinterpret_cast<uintptr_t>(fac) & 7))
    return fail(SHEN_ERR_ARG, "shen_plane_rfft2_fac: bad args (sizes: shen_plane_fft_supported; x, fac 8-B, X 16-B aligned)");
  return cuda_check(shen::launch_plane_rfft2(n_planes, n_y, n_z, x, X, fac, S(stream)), "shen_plane_rfft2_fac");
}

int shen_plane_irfft2(int64_t n_planes, int n_y, int n_z, const void* X, double* x, double scale, void* stream) {
  if (n_planes == 0) return SHEN_OK;
  if (n_planes < 0 || !x || !X || !shen::plane_fft_supported(n_y, n_z) || (reinterpret_cast<uintptr_t>(x) & 7) ||
      (reinterpret_cast<uintptr_t>(X) & 15))
    return fail(SHEN_ERR_ARG, "shen_plane_irfft2: bad args (sizes: shen_plane_fft_supported; x 8-B, X 16-B aligned)");
  return cuda_check(shen::launch_plane_irfft2(n_planes, n_y, n_z, X, x, scale, nullptr, nullptr, S(stream)),
                    "shen_plane_irfft2");
}

int shen_plane_irfft2_fac(int64_t n_planes, int n_y, int n_z, const void* X, double* x, double scale,
                          const double* fac_re, const double* fac_im, void* stream) {
  if (n_planes == 0) return SHEN_OK;
  if (n_planes < 0 || !x || !X || !fac_re || !fac_im || !shen::plane_fft_supported(n_y, n_z) ||
      (reinterpret_cast<uintptr_t>(x) & 7) || (reinterpret_cast<uintptr_t>(X) & 15) ||
      ((reinterpret_cast<uintptr_t>(fac_re) | reinterpret_cast<uintptr_t>(fac_im)) & 7))
    return fail(SHEN_ERR_ARG, "shen_plane_irfft2_fac: bad args (sizes: shen_plane_fft_supported; x, fac 8-B, X 16-B aligned)");
  return cuda_check(shen::launch_plane_irfft2(n_planes, n_y, n_z, X, x, scale, fac_re, fac_im, S(stream)),
                    "shen_plane_irfft2_fac");
}

// kx-row exchange descriptor from the caller's plain arrays (validated here:
// the kernels index with it unchecked)
static int make_xch(shen::PlaneXch* xc, int n_y, int world, void* const* bases, const int64_t* rows,
                    const int* owner, const int* local_row, int64_t plane0, int64_t n_planes_total,
                    int64_t n_planes) {
  if (world < 1 || world > 8 || !bases || !rows || !owner || !local_row || n_y > 256 || plane0 < 0 ||
      plane0 + n_planes > n_planes_total)
    return 0;
  for (int q = 0; q < 8; ++q) {
    xc->base[q] = q < world ? bases[q] : nullptr;
    xc->rows[q] = q < world ? rows[q] : 0;
    if (q < world && (!bases[q] || (reinterpret_cast<uintptr_t>(bases[q]) & 15) || rows[q] < 0)) return 0;
  }
  for (int y = 0; y < 256; ++y) {
    const int q = y < n_y ? owner[y] : 0, lr = y < n_y ? local_row[y] : 0;
    if (q < 0 || q >= world || lr < 0 || (y < n_y && lr >= rows[q])) return 0;
    xc->owner[y] = (unsigned char)q;
    xc->local_row[y] = (short)lr;
  }
  xc->plane0 = plane0;
  return 1;
}

int shen_plane_rfft2_scatter(int64_t n_planes, int n_y, int n_z, const double* x, int world, void* const* bases,
                             const int64_t* rows, const int* owner, const int* local_row, int64_t plane0,
                             int64_t n_planes_total, void* stream) {
  if (n_planes == 0) return SHEN_OK;
  shen::PlaneXch xc;
  if (n_planes < 0 || !x || !shen::plane_fft_supported(n_y, n_z) || (reinterpret_cast<uintptr_t>(x) & 7) ||
      !make_xch(&xc, n_y, world, bases, rows, owner, local_row, plane0, n_planes_total, n_planes))
    return fail(SHEN_ERR_ARG, "shen_plane_rfft2_scatter: bad args");
  return cuda_check(shen::launch_plane_rfft2_scatter(n_planes, n_y, n_z, x, xc, S(stream)), "shen_plane_rfft2_scatter");
}

int shen_plane_irfft2_gather(int64_t n_planes, int n_y, int n_z, int world, void* const* bases, const int64_t* rows,
                             const int* owner, const int* local_row, int64_t plane0, int64_t n_planes_total,
                             double* x, double scale, void* stream) {
  if (n_planes == 0) return SHEN_OK;
  shen::PlaneXch xc;
  if (n_planes < 0 || !x || !shen::plane_fft_supported(n_y, n_z) || (reinterpret_cast<uintptr_t>(x) & 7) ||
      !make_xch(&xc, n_y, world, bases, rows, owner, local_row, plane0, n_planes_total, n_planes))
    return fail(SHEN_ERR_ARG, "shen_plane_irfft2_gather: bad args");
  return cuda_check(shen::launch_plane_irfft2_gather(n_planes, n_y, n_z, xc, x, scale, S(stream)),
                    "shen_plane_irfft2_gather");
}

int shen_enable_peer_access(int peer_device) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(SHEN_ERR_CUDA, "shen_enable_peer_access: no device");
  if (peer_device == dev) return SHEN_OK;
  int can = 0;
  if (cudaDeviceCanAccessPeer(&can, dev, peer_device) != cudaSuccess || !can)
    return fail(SHEN_ERR_CUDA, "shen_enable_peer_access: no peer access between the devices");
  const cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return SHEN_OK;
  }
  return cuda_check(e, "shen_enable_peer_access");
}

int shen_recover_velocity(const shen_recover_args* r, void* stream) {
  if (!r) return fail(SHEN_ERR_ARG, "shen_recover_velocity: NULL args");
  if (r->L == 0 || r->n_dir == 0) return SHEN_OK;
  if (r->n_dir < 0 || r->L < 0 || !band_ok(r->deriv) || r->deriv.nr != r->n_dir || !r->fac ||
      r->mmax < (r->n_dir + 1) / 2 || !r->im_m_re || !r->im_m_im || !r->im_n_re || !r->im_n_im || !r->safe_z2 ||
      !r->u || !r->g || !r->v || !r->w)
    return fail(SHEN_ERR_ARG, "shen_recover_velocity: bad args");
  shen::RecoverArgs a{};
  a.n_dir = r->n_dir; a.L = r->L; a.d = to_band(r->deriv); a.fac = r->fac; a.mmax = r->mmax;
  a.im_m_re = r->im_m_re; a.im_m_im = r->im_m_im; a.im_n_re = r->im_n_re; a.im_n_im = r->im_n_im;
  a.safe_z2 = r->safe_z2; a.u = r->u; a.g = r->g; a.v = r->v; a.w = r->w;
  return cuda_check(shen::launch_recover(a, S(stream)), "shen_recover_velocity");
}

}  // extern "C"
