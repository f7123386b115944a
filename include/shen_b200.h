/*
 * shen_b200.h -- C ABI of the B200 (sm_100a) Shen-Galerkin wall-normal
 * solvers and transforms (the data-parallel core of arXiv 1701.03787), plus
 * the stepper-side pieces around them: structured matrix apply, fused
 * right-hand-side assembly, velocity recovery and the pointwise parts of the
 * nonlinear term.
 *
 * Plain C: device pointers, sizes and an opaque CUDA stream handle
 * (cudaStream_t passed as void*, NULL = legacy default stream).  Every call
 * is stream-ordered and asynchronous unless stated; no call allocates
 * device memory behind the caller's back.  Return value: SHEN_OK or an
 * error code; shen_last_error() gives a message (thread-local).
 *
 * Layouts follow the reference package chebchan (reference paths relative
 * to /root/reference/pkg/src/chebchan):
 *   right-hand sides / solutions: C-contiguous (n_modes, batch) arrays,
 *     complex128 (interleaved re,im) or float64, one column per
 *     wavenumber pair -- the flattened (n_modes,) + z2.shape of
 *     HelmholtzLU.solve / BiharmonicLU.solve (solvers.py:100-109,162-170);
 *   parity p rows are p, p+2, ... (the stride-2 split, solvers.py:107-108);
 *   factor arrays: per parity, (rows, batch) float64 (solvers.py:78-94,
 *     129-152).
 *
 * The reference exposes no native interface; these entry points are what
 * its Python modules bind (see INTEGRATION.md for the ctypes stub).
 */
#ifndef SHEN_B200_H
#define SHEN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum shen_status {
  SHEN_OK = 0,
  SHEN_ERR_ARG = 1,   /* invalid argument / unsupported size */
  SHEN_ERR_CUDA = 2,  /* CUDA runtime error (message via shen_last_error) */
};

/* row pitch (doubles) of the biharmonic row-constant table: 17 constants per
 * mode (see shen_rows.cuh: BihCol) + 1 pad so rows are 16-B aligned */
#define SHEN_BIH_NCOL 18

const char* shen_version(void);
const char* shen_last_error(void);
/* visible CUDA devices (0 on a machine without a GPU; never aborts) */
int shen_device_count(void);
/* scratch bytes of shen_{helm,bih}_solve_stream (op 0 = Helmholtz, 1 = biharmonic) */
int64_t shen_stream_scratch_bytes(int op, int n_modes, int chunk_rows, int64_t batch, int is_complex);
/* cudaMemcpy2DAsync (kind 0 = H2D, 1 = D2H, 2 = D2D): column slabs of
 * (n_modes, batch) arrays for pipelined host<->device solves */
int shen_memcpy2d_async(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width_bytes,
                        int64_t height, int kind, void* stream);
/* set pivot[0] = pivot[1] = INT32_MAX on the device (stream-ordered) */
int shen_pivot_reset(int* pivot_dev, void* stream);

/* ---------------------------------------------------------------------
 * Helmholtz  H = ca*K + cb*B  (Shen-Dirichlet, n_dir = n_x - 1 modes)
 * replaces build_helmholtz (solvers.py:201-241) and HelmholtzLU.solve
 * (solvers.py:100-126).
 *   cb[batch]          : 1 + nu*dt*z2/2 per system (helmholtz_coefficients,
 *                        solvers.py:67-69); ca = nu*dt/2.
 *   sd, st, md [n_dir] : stiff_dir diagonal, stiff_dir tail, mass_dir
 *                        diagonal (MatrixSet, matrices.py:264-337).
 * shen_helm_factor: sequential unpivoted elimination per (system, parity).
 *   exact != 0 -> reference evaluation order and IEEE division (bit-equal
 *   factors); exact == 0 -> reciprocal/FMA arithmetic shared with the
 *   streaming solve.  Outputs are optional (NULL to skip):
 *     factors[8] = {low_p0, low_p1, d_p0, d_p1, e_p0, e_p1, tail_p0, tail_p1}
 *                  device arrays (rows_p - 1 or rows_p, batch);
 *     ckpt       = [C][2][3][batch] factor state entering each chunk of
 *                  chunk_rows rows (C = ceil(rows_p0 / chunk_rows));
 *     pivot_dev  = int[2]; atomic-min of the first row (within parity) whose
 *                  pivot has |d| < 1e-300 (reset it first).
 * shen_helm_solve_stream: fused factor+solve from the checkpoints (ckpt made
 *   with exact == 0, chunk_rows = 8: the spacing the solve kernels are
 *   built for -- 4 doubles the checkpoint memory, 16 spills registers); one
 *   thread per (system,
 *   parity) with coalesced row access; y is
 *   checkpointed at segment ends in `scratch` (shen_stream_scratch_bytes
 *   bytes) and recomputed in the backward sweep; warps_per_sm selects the
 *   persistent CTA size (8 or 12 warps per SM; 0 = the per-operator default,
 *   12 for Helmholtz, 8 for the biharmonic); max_ctas > 0 caps the persistent
 *   grid (one CTA per SM) so that a second solve can run concurrently on the
 *   remaining SMs (0 = all SMs).  [j_begin, j_end) restricts
 *   the solve to a range of systems (j_end < 0: the whole batch) -- the row
 *   pitch stays `batch`, so host<->device copies of column slabs can be
 *   pipelined against the solve (see shen_memcpy2d_async).
 * shen_helm_solve_stored: solve with full stored factors (reference order).
 * rhs and out may alias only for the stored variant.
 * ------------------------------------------------------------------- */
int shen_helm_factor(int n_dir, double ca, const double* cb, int64_t batch, const double* sd, const double* st,
                     const double* md, int chunk_rows, double* ckpt, double* const* factors, int exact,
                     int* pivot_dev, void* stream);
int shen_helm_solve_stream(int n_dir, double ca, const double* cb, int64_t batch, const double* sd,
                           const double* st, const double* md, int chunk_rows, const double* ckpt,
                           const void* rhs, void* out, void* scratch, int is_complex, int warps_per_sm,
                           int max_ctas, int64_t j_begin, int64_t j_end, void* stream);
int shen_helm_solve_stored(int n_dir, int64_t batch, const double* const* factors, const void* rhs, void* out,
                           int is_complex, void* stream);

/* ---------------------------------------------------------------------
 * Biharmonic  H = xi0*Q + xi1*A + xi2*B  (n_bih = n_x - 3 modes)
 * replaces build_biharmonic (solvers.py:244-355) and BiharmonicLU.solve
 * (solvers.py:162-198).
 *   xi1[batch], xi2[batch] : biharmonic_coefficients (solvers.py:72-75).
 *   tab[n_bih][18]         : per-mode row constants (last column padding)
 *      {q0, -A0, B0, tail2, -A+2, B+2, tail4, B+4, -A-2(k-2), B+2(k-2),
 *       B+4(k-4), p, r, q(k+2), s(k+2), q(k+4), s(k+4)}
 *      with entries outside the band set to 0 (solvers.py:244-268).
 *   q, s [n_bih]           : tail factors (matrices.py:163-170).
 *   factors[14] = {low2_p0, low2_p1, low4_p0, low4_p1, d_p0, d_p1, e_p0,
 *                  e_p1, f_p0, f_p1, a_p0, a_p1, b_p0, b_p1}
 *   ckpt = [C][2][10][batch] (rows s-1 and s-2 of U entering each chunk).
 * ------------------------------------------------------------------- */
int shen_bih_factor(int n_bih, double xi0, const double* xi1, const double* xi2, int64_t batch,
                    const double* tab, int chunk_rows, double* ckpt, double* const* factors, int exact,
                    int* pivot_dev, void* stream);
int shen_bih_solve_stream(int n_bih, double xi0, const double* xi1, const double* xi2, int64_t batch,
                          const double* tab, int chunk_rows, const double* ckpt, const void* rhs, void* out,
                          void* scratch, int is_complex, int warps_per_sm, int max_ctas, int64_t j_begin,
                          int64_t j_end, void* stream);
/* Same solve with systems taken in mirror pairs: pairs[0..P) and
 * pairs[P..2P) are system indices with bitwise-identical z2 (for a channel
 * grid: wavenumbers (m, n) and (-m, n)); one thread runs the factor
 * recurrence once for both right-hand sides.  pairs[c] == pairs[P + c] marks
 * an unpaired system (solved once).  Every system must appear exactly once
 * over both halves; results are bit-identical to shen_bih_solve_stream. */
int shen_bih_solve_stream_pairs(int n_bih, double xi0, const double* xi1, const double* xi2, int64_t batch,
                                const double* tab, int chunk_rows, const double* ckpt, const void* rhs, void* out,
                                void* scratch, int is_complex, const int64_t* pairs, int64_t n_pairs, int max_ctas,
                                void* stream);
int shen_bih_solve_stored(int n_bih, int64_t batch, double xi0, const double* q, const double* s,
                          const double* const* factors, const void* rhs, void* out, int is_complex,
                          void* stream);

/* ---------------------------------------------------------------------
 * Wall-normal transform stages (reference transforms.py:81-205).
 * Arrays are (rows, L) complex128 with the L Fourier lines contiguous.
 * The DCT itself is an FFT of an extended sequence along the rows, done by
 * the caller's FFT library (cuFFT) between the stages below:
 *   forward  : shen_xform_extend -> FFT (forward, along rows) -> shen_xform_fwd_post
 *              -> shen_xform_mass_solve (transforms.py:178-196)
 *   inverse  : shen_xform_inv_pre -> FFT (Gauss: unnormalised inverse, GL:
 *              forward) -> shen_xform_inv_post (transforms.py:199-205)
 * family: 0 = Gauss (DCT-II/III via 2N-point FFT), 1 = Gauss-Lobatto (DCT-I
 * via 2(N-1)-point FFT); N = n_x + 1 points; space 0/1/2 = Chebyshev /
 * Dirichlet / biharmonic.
 * ------------------------------------------------------------------- */
/* x[N][L] -> e[M][L], M = 2N (Gauss, symmetric) or 2N-2 (GL, even). */
int shen_xform_extend(int family, int N, int64_t L, const void* x, void* e, void* stream);
/* Y[>=N][L] (FFT of the extension) -> out[n_modes][L]: Chebyshev scalar
 * products scaled by `scale` (pi/(2N) Gauss, pi/(2(N-1)) GL), twiddled by
 * tw[N] (exp(-i pi k / 2N), Gauss only), then the `space` stencil
 * (transforms.py:93-110); space 3 = the raw scalar products (chebyshev_scalar
 * transforms.py:81-86). */
int shen_xform_fwd_post(int family, int space, int N, int64_t L, double scale, const void* tw, const void* Y,
                        void* out, void* stream);
/* coef[n][L] of `space` -> FFT input Z[M][L] and cends[2][L] = {c_0, c_{N-1}}
 * of the Chebyshev expansion (shen_expand transforms.py:113-126).
 * family 2 writes the expanded Chebyshev coefficients Z[N][L] themselves
 * (shen_expand alone; cends may be NULL). */
int shen_xform_inv_pre(int family, int space, int n, int N, int64_t L, const void* tw, const void* coef, void* Z,
                       void* cends, void* stream);
/* F[>=N][L] -> point values out[N][L] (chebyshev_evaluate transforms.py:129-137). */
int shen_xform_inv_post(int family, int N, int64_t L, const void* F, const void* cends, void* out, void* stream);
/* Per-parity banded Cholesky solve U^T U x = s (transforms.py:163-175):
 * fac[2][nband+1][mmax] LAPACK upper band storage per parity (scipy
 * cholesky_banded), n rows, s and x may alias. */
int shen_xform_mass_solve(int nband, int n, int mmax, int64_t L, const double* fac, const void* s, void* x,
                          void* stream);

/* ---------------------------------------------------------------------
 * Fused wall-normal transform (one kernel per direction, reference
 * transforms.py:81-205): on a tile of Fourier lines held in shared memory,
 *   forward  DCT (type 2 Gauss / type 1 Gauss-Lobatto) -> Chebyshev scaling
 *            -> Shen stencil -> optional per-parity banded Cholesky mass
 *            solve (forward_transform / forward_scalar_product /
 *            shen_scalar / chebyshev_scalar);
 *   inverse  shen_expand -> Chebyshev evaluation on the points, times
 *            `scale` (inverse_transform's wall-normal stage, chebyshev_evaluate).
 * The DFT behind the DCT is a power-of-two FFT, Rader's algorithm (prime
 * length with a power-of-two predecessor: N = 257) or Bluestein's, all in
 * shared memory.  The plan (tables, all device pointers) is built by the
 * host layer (paper_1701_03787_b200/wall.py); `in` and `out` are (rows, L)
 * complex128, lines contiguous, not aliased. */
typedef struct shen_wall_plan {
  int direction, family, space, mass, N, n_out, n_in, kind, Ld, M, nstage;
  int radix[4];
  int log2_lines, rows_smem;
  double scale;
  int nband, mmax;
  const void *tw, *ker_f, *ker_i, *chirp_f, *chirp_i; /* complex128 tables */
  const int *gin_f, *gin_i, *gout, *pinv;
  const void* mk;                                     /* complex128 */
  const double *c2, *c4, *mfac;
  const double* rowscale; /* inverse, Chebyshev space: per-coefficient factor applied first, or NULL */
} shen_wall_plan;
int shen_wall_transform(const shen_wall_plan* plan, int64_t L, const void* in, void* out, void* stream);
/* shared-memory bytes per CTA of a plan (host-side plan checks) */
int64_t shen_wall_smem_bytes(const shen_wall_plan* plan);

/* ---------------------------------------------------------------------
 * Structured matrix-vector products y = M x along the rows of (rows, L)
 * arrays (reference matrices.py:62-71, 109-117, 145-152; the
 * _parity_suffix_sum of :84-90), bit-identical to the reference's.
 *   offsets[n_off] (host array), diag[n_off][nr] (device, row-indexed:
 *   entry (k, k + offsets[i]) at diag[i][k] for the offset's valid rows).
 *   constant tail: row k also gets tail[k] * sum_{j >= k + tail_start,
 *   j = k + tail_start mod 2} x[j].
 *   rank-2 tail (square n): diag[k] x[k] + p[k] sum_{j>=k+2} q[j] x[j]
 *   + r[k] sum_{j>=k+2} s[j] x[j] (same-parity j).
 * ------------------------------------------------------------------- */
int shen_apply_banded(int nr, int nc, int64_t L, int n_off, const int* offsets, const double* diag, const void* x,
                      void* y, int is_complex, void* stream);
int shen_apply_const_tail(int nr, int nc, int64_t L, int n_off, const int* offsets, const double* diag,
                          const double* tail, int tail_start, const void* x, void* y, int is_complex, void* stream);
int shen_apply_rank2_tail(int n, int64_t L, const double* diag, const double* p, const double* q, const double* r,
                          const double* s, const void* x, void* y, int is_complex, void* stream);

/* ---------------------------------------------------------------------
 * Stepper right-hand sides, fused (reference stepper.py:189-219): AB2
 * combination of the nonlinear terms and the explicit operators in one pass
 * per Fourier line, bit-identical to the reference.  Arrays are (rows, L)
 * complex128 with L = n_y (n_z/2+1) lines; per-line coefficient arrays are
 * the reference's numpy expressions evaluated on the host (see
 * paper_1701_03787_b200/rhs.py).  Matrices: row-indexed diagonal tables as
 * for shen_apply_banded (device), offsets inline.
 * ------------------------------------------------------------------- */
typedef struct shen_band {
  int nr, nc, n_off;
  int off[6];
  const double* diag; /* [n_off][nr] */
} shen_band;

typedef struct shen_rhs_g_args {
  int n_dir;
  int64_t L;
  shen_band stiff, mass; /* stiff_dir banded part, mass_dir */
  const double* tail;    /* stiff_dir tail */
  int tail_start;
  double c_stiff, dt;    /* -(nu dt/2), dt */
  const double* cg;      /* [L] 1 - nu dt z2 / 2 */
  const double *im_m_re, *im_m_im, *im_n_re, *im_n_im; /* [L] 1j m, 1j n */
  const void *g, *hcy, *hpy, *hcz, *hpz;                /* g, h_curr/h_prev y and z */
  void* out;
} shen_rhs_g_args;

typedef struct shen_rhs_u_args {
  int n_bih;
  int64_t L;
  const double *d, *p, *q, *r, *s; /* fourth_bih */
  double c_fourth;                 /* nu dt / 2 */
  shen_band stiff, mass, mixed, deriv; /* stiff_bih, mass_bih, mixed_mass, deriv_dir_to_bih */
  const double *c_stiff, *c_mass, *c_mixed;             /* [L] 1 - nu dt z2, -z2 + nu dt z2^2/2, dt z2 */
  const double *c_dy_re, *c_dy_im, *c_dz_re, *c_dz_im;  /* [L] dt 1j m, dt 1j n */
  const void *u, *hcx, *hpx, *hcy, *hpy, *hcz, *hpz;
  void* out;
} shen_rhs_u_args;

/* assemble_rhs_g (stepper.py:209-219) with _ab2 (:189-191) folded in */
int shen_rhs_g(const shen_rhs_g_args* args, void* stream);
/* assemble_rhs_u (stepper.py:193-207) with _ab2 folded in */
int shen_rhs_u(const shen_rhs_u_args* args, void* stream);

/* ---------------------------------------------------------------------
 * Velocity recovery (reference stepper.py:296-303): f = B_D^-1 (D u_new),
 * v = (1j m f + 1j n g) / z2', w = (1j n f - 1j m g) / z2' per line
 * (z2' = z2, 1 on the mean mode).  fac = per-parity LAPACK upper band
 * Cholesky factors of mass_dir, [2][2][mmax] (as for shen_xform_mass_solve).
 * ------------------------------------------------------------------- */
typedef struct shen_recover_args {
  int n_dir;
  int64_t L;
  shen_band deriv;    /* deriv_bih_to_dir (n_dir x n_bih) */
  const double* fac;
  int mmax;
  const double *im_m_re, *im_m_im, *im_n_re, *im_n_im, *safe_z2; /* [L] */
  const void *u, *g;  /* u_new (n_bih, L), g_new (n_dir, L) */
  void *v, *w;        /* (n_dir, L) outputs */
} shen_recover_args;
int shen_recover_velocity(const shen_recover_args* args, void* stream);

/* ---------------------------------------------------------------------
 * Nonlinear term H = u x omega (reference stepper.py:148-185), the pointwise
 * piece; the transforms around it are shen_wall_transform and the plane FFTs
 * below, whose _fac variants apply the per-line factors (1j m, 1j n, mask).
 * shen_cross: fields = 8 real planes-stacked arrays of n points
 *   [u, v, w, om_x, dv_dx, dw_dx, du_dy, du_dz] -> h = 3 arrays
 *   (v om_z - w om_y, w om_x - u om_z, u om_y - v om_x) with
 *   om_y = du_dz - dw_dx, om_z = dv_dx - du_dy.
 * ------------------------------------------------------------------- */
int shen_cross(int64_t n, const double* fields, double* h, void* stream);

/* ---------------------------------------------------------------------
 * Periodic (y, z) plane transforms of the 3-D transforms (reference
 * transforms.py:181-205, numpy rfft2 / irfft2 over axes (1, 2)), one
 * thread-block cluster per plane, one HBM pass each way.
 * shen_plane_rfft2:  x  (n_planes, n_y, n_z) float64 -> X (n_planes, n_y, n_z/2+1) complex128
 * shen_plane_irfft2: X -> x, times `scale` (1/(n_y n_z) = numpy's "backward"
 *   norm; 1 = "forward"); imaginary parts of the z = 0 and z = n_z/2 columns
 *   are ignored, as numpy's irfft does.
 * Sizes: shen_plane_fft_supported(n_y, n_z) (256 x 256); others -> SHEN_ERR_ARG.
 * ------------------------------------------------------------------- */
int shen_plane_fft_supported(int n_y, int n_z);
int shen_plane_rfft2(int64_t n_planes, int n_y, int n_z, const double* x, void* X, void* stream);
int shen_plane_irfft2(int64_t n_planes, int n_y, int n_z, const void* X, double* x, double scale, void* stream);
/* The same with a factor per (ky, kz) Fourier line, (n_y, n_z/2+1) float64 arrays on the device, applied to every
 * plane: shen_plane_rfft2_fac multiplies the spectrum by the real `fac` at the store (the dealiasing mask of
 * apply_mask, reference stepper.py:142-144, which commutes with the per-line wall-normal transform that follows);
 * shen_plane_irfft2_fac multiplies the spectrum by fac_re + i fac_im at the load (i m, i n: the y / z derivatives of
 * compute_nonlinear, stepper.py:171-172), so neither needs its own pass over the field. */
int shen_plane_rfft2_fac(int64_t n_planes, int n_y, int n_z, const double* x, void* X, const double* fac,
                         void* stream);
int shen_plane_irfft2_fac(int64_t n_planes, int n_y, int n_z, const void* X, double* x, double scale,
                          const double* fac_re, const double* fac_im, void* stream);

/* ---------------------------------------------------------------------
 * The same transforms with the slab decomposition's kx-row exchange fused in
 * (several GPUs of one box; the reference is single-process, so this has no
 * reference counterpart -- SURVEY.md 8(e), the paper's slab transpose).  A
 * rank holds physical x-planes [plane0, plane0 + n_planes) and the kx rows
 * {y : owner[y] == rank} of every plane.  Row y of global plane x lives in
 * rank owner[y]'s buffer bases[owner[y]], a C-contiguous complex128 array
 * (n_planes_total, rows[owner[y]], n_z/2+1), at [x][local_row[y]][:].
 * bases[q] are pointers valid on THIS device (peer memory opened by CUDA IPC
 * or the rank's own buffer); owner / local_row have n_y entries (host).
 * shen_plane_rfft2_scatter: rfft2 of the rank's planes, each spectrum row
 *   stored straight into its owner's buffer (no pack pass, no all-to-all).
 * shen_plane_irfft2_gather: irfft2 of the rank's planes, each spectrum row
 *   read from its owner's buffer.
 * Ordering is the caller's: every rank's scatter must have completed (stream
 * synchronised + a barrier across ranks) before any rank reads its buffer,
 * and a buffer must not be rewritten while a peer may still gather from it.
 * shen_enable_peer_access(d): cudaDeviceEnablePeerAccess to device d from
 *   the current one (no-op when d is the current device or already enabled).
 * ------------------------------------------------------------------- */
int shen_plane_rfft2_scatter(int64_t n_planes, int n_y, int n_z, const double* x, int world, void* const* bases,
                             const int64_t* rows, const int* owner, const int* local_row, int64_t plane0,
                             int64_t n_planes_total, void* stream);
int shen_plane_irfft2_gather(int64_t n_planes, int n_y, int n_z, int world, void* const* bases, const int64_t* rows,
                             const int* owner, const int* local_row, int64_t plane0, int64_t n_planes_total,
                             double* x, double scale, void* stream);
int shen_enable_peer_access(int peer_device);

#ifdef __cplusplus
}
#endif

#endif /* SHEN_B200_H */
