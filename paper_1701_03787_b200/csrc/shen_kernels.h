// Internal launch interface between the C-ABI layer (shen_capi.cu) and the
// kernels.  Not part of the public header (include/shen_b200.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace shen {

struct HelmFactorArgs {
  int n_dir;
  double ca;
  const double* cb;  // [batch]
  int64_t batch;
  const double* sd;  // stiff_dir diag  [n_dir]
  const double* st;  // stiff_dir tail  [n_dir]
  const double* md;  // mass_dir diag   [n_dir]
  int chunk_rows;    // R for checkpoints (0: none)
  double* ckpt;      // [C][2][3][batch] or null
  double* low[2];    // full factors per parity (null: not wanted)
  double* d[2];
  double* e[2];
  double* t[2];
  int* pivot;        // [2] min failing row per parity (INT_MAX = none), or null
};

struct BihFactorArgs {
  int n_bih;
  double xi0;
  const double* xi1;  // [batch]
  const double* xi2;  // [batch]
  int64_t batch;
  const double* tab;  // [n_bih][B_NCOL] row constants
  int chunk_rows;
  double* ckpt;       // [C][2][10][batch] or null
  double* low2[2];
  double* low4[2];
  double* d[2];
  double* e[2];
  double* f[2];
  double* a[2];
  double* b[2];
  int* pivot;
};

// Stored-factor (reference-exact) solve: one thread per (system, parity).
struct HelmSeqArgs {
  int n_dir;
  int64_t batch;
  const double* low[2];
  const double* d[2];
  const double* e[2];
  const double* t[2];
  const void* rhs;  // (n_dir, batch) complex128 or float64
  void* out;
};

struct BihSeqArgs {
  int n_bih;
  int64_t batch;
  double xi0;
  const double* q;  // [n_bih]
  const double* s;  // [n_bih]
  const double* low2[2];
  const double* low4[2];
  const double* d[2];
  const double* e[2];
  const double* f[2];
  const double* a[2];
  const double* b[2];
  const void* rhs;
  void* out;
};

// Streaming fused solve: factors recomputed from checkpoints.
struct HelmChunkArgs {
  int n_dir;
  double ca;
  const double* cb;
  int64_t batch;
  const double* sd;
  const double* st;
  const double* md;
  int chunk_rows;
  const double* ckpt;
  const void* rhs;
  void* out;
  int64_t jb = 0, je = -1;  // system range [jb, je) of the streaming solve (je < 0: whole batch)
  int max_ctas = 0;          // streaming solve: cap on persistent CTAs (0: one per SM)
};

struct BihChunkArgs {
  int n_bih;
  double xi0;
  const double* xi1;
  const double* xi2;
  int64_t batch;
  const double* tab;
  int chunk_rows;
  const double* ckpt;
  const void* rhs;
  void* out;
  int64_t jb = 0, je = -1;
  int max_ctas = 0;
  // mirror pairs (stream solve): pairs[0..P) and pairs[P..2P) are two systems
  // with bitwise-identical z2 (hence identical factors) solved by one thread;
  // equal entries mark an unpaired system.  nullptr: one system per thread.
  const int64_t* pairs = nullptr;
  int64_t n_pairs = 0;
};

cudaError_t launch_helm_factor(const HelmFactorArgs& a, bool exact, cudaStream_t st);
cudaError_t launch_bih_factor(const BihFactorArgs& a, bool exact, cudaStream_t st);
cudaError_t launch_helm_seq(const HelmSeqArgs& a, bool complex_rhs, cudaStream_t st);
cudaError_t launch_bih_seq(const BihSeqArgs& a, bool complex_rhs, cudaStream_t st);
// streaming sequential solve (lanes = systems); warps_per_sm bounds the systems in flight
cudaError_t launch_helm_stream(const HelmChunkArgs& a, void* scratch, bool complex_rhs, int warps_per_sm,
                               cudaStream_t st);
cudaError_t launch_bih_stream(const BihChunkArgs& a, void* scratch, bool complex_rhs, int warps_per_sm,
                              cudaStream_t st);
int64_t stream_scratch_bytes(int op, int n_modes, int chunk_rows, bool complex_rhs);
// structured apply along the rows (shen_apply.cu): kind 0 banded, 1 constant tail, 2 rank-2 tail
cudaError_t launch_apply(int kind, int nr, int nc, int64_t L, int n_off, const int* offs, const double* diag,
                         const double* tail, int tail_start, const double* d, const double* p, const double* q,
                         const double* r, const double* s, const void* x, void* y, bool cplx_data, cudaStream_t st);

// stepper right-hand sides (shen_rhs.cu)
struct RhsBand {  // banded matrix, row-indexed diagonals [n_off][nr] (device)
  int nr, nc, n_off;
  int off[6];
  const double* diag;
};
struct RhsGArgs {
  int n_dir;
  int64_t L;
  RhsBand stiff, mass;        // stiff_dir banded part, mass_dir
  const double* tail;         // stiff_dir tail
  int tail_start;
  double c_stiff, dt;         // -(nu dt / 2), dt
  const double* cg;           // per line: 1 - nu dt z2 / 2
  const double *im_m_re, *im_m_im, *im_n_re, *im_n_im;  // per line: 1j m, 1j n
  const void *g, *hcy, *hpy, *hcz, *hpz;
  void* out;
};
struct RhsUArgs {
  int n_bih;
  int64_t L;
  const double *d, *p, *q, *r, *s;  // fourth_bih
  double c_fourth;                  // nu dt / 2
  RhsBand stiff, mass, mixed, deriv;
  const double *c_stiff, *c_mass, *c_mixed;            // per line: 1 - nu dt z2, -z2 + nu dt z2^2 / 2, dt z2
  const double *c_dy_re, *c_dy_im, *c_dz_re, *c_dz_im;  // per line: dt 1j m, dt 1j n
  const void *u, *hcx, *hpx, *hcy, *hpy, *hcz, *hpz;
  void* out;
};
cudaError_t launch_rhs_g(const RhsGArgs& a, cudaStream_t st);
cudaError_t launch_rhs_u(const RhsUArgs& a, cudaStream_t st);

// velocity recovery (shen_recover.cu)
struct RecoverArgs {
  int n_dir;
  int64_t L;
  RhsBand d;          // deriv_bih_to_dir
  const double* fac;  // mass_dir per-parity Cholesky, [2][2][mmax] upper band storage
  int mmax;
  const double *im_m_re, *im_m_im, *im_n_re, *im_n_im, *safe_z2;  // per line
  const void *u, *g;
  void *v, *w;
};
cudaError_t launch_recover(const RecoverArgs& a, cudaStream_t st);

// nonlinear-term pointwise kernels (shen_nonlinear.cu)
cudaError_t launch_cross(int64_t n, const double* fields, double* h, cudaStream_t st);

// periodic (y, z) plane FFTs (shen_plane_fft.cu): one 8-CTA cluster per plane
// kx-row exchange fused into the plane FFTs (slab transforms over several
// GPUs): spectrum row y of global plane x lives on rank owner[y], in its
// (n_planes_total, rows[owner], n_z/2+1) complex128 buffer base[owner] at
// [x][local_row[y]][:].  Up to 8 ranks, 256 rows (the supported plane size).
struct PlaneXch {
  void* base[8];
  int64_t rows[8];
  int64_t plane0;  // global index of this launch's first plane
  unsigned char owner[256];
  short local_row[256];
};
bool plane_fft_supported(int n_y, int n_z);
cudaError_t launch_plane_rfft2_scatter(int64_t planes, int n_y, int n_z, const double* x, const PlaneXch& xc,
                                       cudaStream_t st);
cudaError_t launch_plane_irfft2_gather(int64_t planes, int n_y, int n_z, const PlaneXch& xc, double* x, double scale,
                                       cudaStream_t st);
cudaError_t launch_plane_rfft2(int64_t planes, int n_y, int n_z, const double* x, void* X, const double* fac,
                               cudaStream_t st);
cudaError_t launch_plane_irfft2(int64_t planes, int n_y, int n_z, const void* X, double* x, double scale,
                                const double* fac_re, const double* fac_im, cudaStream_t st);

// fused wall-normal transforms (shen_wall.cu); tables built on the host (wall.py)
struct WallPlan {
  int direction;   // 0 forward (points -> coefficients), 1 inverse
  int family;      // 0 Gauss, 1 Gauss-Lobatto
  int space;       // 0 Chebyshev, 1 Dirichlet, 2 biharmonic, 3 raw scalar products (forward only)
  int mass;        // forward: 1 = banded mass solve after the stencil
  int N;           // points (n_x + 1)
  int n_out;       // forward output rows
  int n_in;        // inverse input rows
  int kind;        // DFT: 0 power of two, 1 Rader, 2 Bluestein
  int Ld, M;       // DFT length, FFT size (power of two)
  int nstage;
  int radix[4];    // radix of each DIF pass, first to last (product = M)
  int log2_lines;  // lines per CTA = 1 << log2_lines
  int rows_smem;   // shared-memory rows of the tile (>= max(N, M))
  double scale;    // forward: Chebyshev scaling pi/(2N) or pi/(2 n_x); inverse: 1/(n_y n_z)
  int nband, mmax;
  const double2* tw;       // [M] exp(-2 pi i k / M)
  const double2* ker_f;    // [M] convolution kernel spectrum (digit-reversed, / M), forward DFT
  const double2* ker_i;    // [M] same for the inverse DFT
  const double2* chirp_f;  // [Ld] Bluestein chirp, forward
  const double2* chirp_i;  // [Ld] Bluestein chirp, inverse
  const int* gin_f;        // [M] Rader gather rows, forward (sigma(g^p))
  const int* gin_i;        // [M] Rader gather rows, inverse (g^p)
  const int* gout;         // [M] Rader output index g^{-q} mod N
  const int* pinv;         // [M] power of two: position of frequency k
  const double2* mk;       // [N] exp(-i pi k / 2N) (Gauss)
  const double* c2;        // [n_bih] biharmonic stencil 2(k+2)/(k+3)
  const double* c4;        // [n_bih] (k+1)/(k+3)
  const double* mfac;      // [2][mmax + 1][8] folded stencil / Cholesky coefficients per parity (wall.py)
  const double* rowscale;  // [N] inverse, Chebyshev space: coefficient k scaled first (d/dx: 1/mass_cheb), or null
};
size_t wall_smem_bytes(const WallPlan& p);
cudaError_t launch_wall(const WallPlan& p, int64_t L, const void* in, void* out, cudaStream_t st);

// transforms (shen_transform.cu)
cudaError_t launch_xf_extend(int kind, int N, int64_t L, const void* x, void* e, cudaStream_t st);
cudaError_t launch_xf_fwd_post(int gl, int space, int N, int64_t L, double scale, const void* tw, const void* Y,
                               void* out, cudaStream_t st);
cudaError_t launch_xf_inv_pre(int gl, int space, int n, int N, int64_t L, const void* tw, const void* coef, void* Z,
                              void* cends, cudaStream_t st);
cudaError_t launch_xf_inv_post(int gl, int N, int64_t L, const void* F, const void* cends, void* out, cudaStream_t st);
cudaError_t launch_xf_mass(int nband, int n, int mmax, int64_t L, const double* fac, const void* s, void* x,
                           cudaStream_t st);

}  // namespace shen
