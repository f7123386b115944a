// Row recurrences of the compressed unpivoted LU (reference solvers.py),
// written once and shared by the factor kernel and the chunked solve so the
// factors a chunk recomputes from its checkpoint are bit-identical to the
// ones the build kernel walked through.
//
// Two arithmetic modes:
//   EXACT = true : the reference's numpy evaluation order, IEEE division,
//                  no contraction  -> bit-equal to chebchan's factors.
//   EXACT = false: reciprocal-multiply and fused multiply-add (fast path).
#pragma once
#include "shen_common.cuh"

namespace shen {

// ------------------------------------------------------------ Helmholtz
// Per-system coefficients: ca (scalar), cb = 1 + nu*dt*z2/2.
// Row constants by full mode k: sd = stiff_dir diag, st = stiff_dir tail,
// md = mass_dir diag (solvers.py:209-223).
struct HelmRow {
  double diag, sup, tail;
};

__device__ __forceinline__ HelmRow helm_row(double ca, double cb, double sub, double sd, double st, double md,
                                            bool has_sup) {
  HelmRow h;
  h.diag = __dadd_rn(__dmul_rn(ca, sd), __dmul_rn(cb, md));
  h.tail = __dadd_rn(__dmul_rn(ca, st), 0.0);
  h.sup = has_sup ? __dadd_rn(h.tail, sub) : h.tail;
  return h;
}

// Factor state after row i: d, e, t.
struct HelmState {
  double d, e, t;
};

// One exact-mode elimination step (solvers.py:231-236): numpy's evaluation
// order, IEEE division, no contraction.  Returns low (0 for row 0).  The fast
// mode is the projective walk below (hp_step).
__device__ __forceinline__ double helm_step_exact(HelmState& s, const HelmRow& h, double sub, bool first) {
  if (first) {
    s.d = h.diag;
    s.e = h.sup;
    s.t = h.tail;
    return 0.0;
  }
  const double low = __ddiv_rn(sub, s.d);
  s.d = __dsub_rn(h.diag, __dmul_rn(low, s.e));
  s.e = __dsub_rn(h.sup, __dmul_rn(low, s.t));
  s.t = __dsub_rn(h.tail, __dmul_rn(low, s.t));
  return low;
}

// ---------------------------------------------------------------- fast reciprocal
// MUFU.RCP64H seed r0, then 1/x = r0 (1 + e + e^2 + ...) with e = 1 - x r0
// truncated after e^2: the seed's |e| <= 2^-19.9 leaves ~e^3 < 2^-59, i.e.
// the <= 1 ulp of two Newton steps (measured over 2^30 doubles: max 1 ulp,
// 99.97% correctly rounded, tools/rcp_check.cu) with two dependent FMAs after
// the seed instead of four.  No slow path: the
// fast-mode recurrences never see zero, inf or denormal pivots in practice;
// the exact path keeps IEEE division.
__device__ __forceinline__ double rcp_fast(double x) {
  double r0;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r0) : "d"(x));
  const double e = __fma_rn(-x, r0, 1.0);
  return __fma_rn(r0, __fma_rn(e, e, e), r0);
}

// ---------------------------------------------------------------- projective Helmholtz walk
// Fast-mode elimination with no reciprocal on the dependency chain.  With
// d_i = D_i / D_{i-1}, e_i = E_i / D_{i-1}, t_i = T_i / D_{i-1} the
// recurrence of solvers.py:231-235 becomes linear:
//     D_i = diag_i D_{i-1} - sub E_{i-1}
//     E_i = sup_i  D_{i-1} - sub T_{i-1}
//     T_i = tail_i D_{i-1} - sub T_{i-1}
// (2 dependent ops per row instead of rcp + 2).  Ratios are formed off the
// chain with one reciprocal per row.  Every chunk restarts from the rounded
// ratios (d, e, t) of its predecessor with D_{s-2} := 1, in the build kernel
// and in the solve alike, so the two see bit-identical factors.
struct HelmProj {
  double D, E, T;  // state of the last row
  double rD;       // 1 / D of the last row
  double rd;       // 1 / d of the last row
};

__device__ __forceinline__ void hp_start(HelmProj& s, double d, double e, double t) {
  s.D = d;
  s.E = e;
  s.T = t;
  s.rD = rcp_fast(d);
  s.rd = s.rD;
}

// state "before row 0": D_{-1} = 1, E = T = 0 and 1/d_{-1} := 0, so the
// generic step reproduces row 0 exactly (d_0 = diag_0, e_0 = sup_0,
// t_0 = tail_0, low_0 = 0) without a branch
__device__ __forceinline__ void hp_origin(HelmProj& s) {
  s.D = 1.0;
  s.E = 0.0;
  s.T = 0.0;
  s.rD = 1.0;
  s.rd = 0.0;
}

// generic row: returns low_i = sub / d_{i-1}; outputs ratios e_i, t_i, d_i
__device__ __forceinline__ double hp_step(HelmProj& s, const HelmRow& h, double sub, double& d, double& e,
                                          double& t) {
  const double low = __dmul_rn(sub, s.rd);
  const double se = __dmul_rn(sub, s.E), st = __dmul_rn(sub, s.T);
  const double Dn = __fma_rn(h.diag, s.D, -se);
  const double En = __fma_rn(h.sup, s.D, -st);
  const double Tn = __fma_rn(h.tail, s.D, -st);
  const double rDn = rcp_fast(Dn);
  d = __dmul_rn(Dn, s.rD);
  e = __dmul_rn(En, s.rD);
  t = __dmul_rn(Tn, s.rD);
  s.rd = __dmul_rn(s.D, rDn);
  s.D = Dn;
  s.E = En;
  s.T = Tn;
  s.rD = rDn;
  return low;
}

// exact power-of-two rescale of the projective state (overflow guard)
__device__ __forceinline__ void hp_rescale(HelmProj& s) {
  const int hi = __double2hiint(s.D);
  const int ex = (hi >> 20) & 0x7ff;
  const bool ok = ex != 0 && ex != 0x7ff;  // branch-free: zero/inf/nan left alone
  const double sc = ok ? __hiloint2double((2046 - ex) << 20, 0) : 1.0;  // 2^(1023 - ex)
  const double isc = ok ? __hiloint2double(ex << 20, 0) : 1.0;         // 2^(ex - 1023)
  s.D = __dmul_rn(s.D, sc);
  s.E = __dmul_rn(s.E, sc);
  s.T = __dmul_rn(s.T, sc);
  s.rD = __dmul_rn(s.rD, isc);
}

// ------------------------------------------------------------ biharmonic
// Row-constant table, one record per full biharmonic mode k (host built
// from MatrixSet + tail_factors, solvers.py:244-268); entries that the
// reference's band() leaves at zero are stored as 0.
enum BihCol {
  B_Q0 = 0, B_AR0, B_BB0,          // d0 band
  B_T2, B_AR2, B_BB2,              // p2 band (row k, col k+2)
  B_T4, B_BB4,                     // p4 band
  B_ARM2, B_BB2M,                  // m2 band (values at k-2)
  B_BB4M,                          // m4 band (value at k-4)
  B_P, B_R,                        // tail row factors p_k, r_k
  B_Q2, B_S2, B_Q4, B_S4,          // q, s at k+2 and k+4 (0 past the end)
  B_NCOL
};
constexpr int B_STRIDE = 18;  // table row pitch in doubles (17 used + 1 pad: 16-B aligned rows)

// the row constants of full mode k: 9 vector loads through the read-only path
__device__ __forceinline__ void load_bih_row(const double* tab, int k, double* c) {
  const double2* p = reinterpret_cast<const double2*>(tab + (int64_t)k * B_STRIDE);
#pragma unroll
  for (int q = 0; q < B_STRIDE / 2; ++q) {
    const double2 v = __ldg(p + q);
    c[2 * q] = v.x;
    if (2 * q + 1 < B_NCOL) c[2 * q + 1] = v.y;
  }
}
// same from a shared-memory copy of the table
__device__ __forceinline__ void load_bih_row_smem(const double* tab, int k, double* c) {
  const double2* p = reinterpret_cast<const double2*>(tab + (int64_t)k * B_STRIDE);
#pragma unroll
  for (int q = 0; q < B_STRIDE / 2; ++q) {
    const double2 v = p[q];
    c[2 * q] = v.x;
    if (2 * q + 1 < B_NCOL) c[2 * q + 1] = v.y;
  }
}

// Compact shared-memory row (BC_STRIDE doubles per mode, 4 virtual zero rows
// in front): the 13 per-mode values; BB2M/BB4M/Q2/S2 of mode k are the BB2 /
// BB4 / Q4 / S4 entries of modes k-2 / k-4 (virtual rows -2, -1 carry q, s of
// modes 2, 3 so that Q2/S2 of modes 0, 1 come out right).
enum BihCompactCol { BC_Q0 = 0, BC_AR0, BC_BB0, BC_T2, BC_AR2, BC_BB2, BC_T4, BC_BB4, BC_ARM2, BC_P, BC_Q4, BC_S4, BC_R,
                     BC_NCOL };
constexpr int BC_STRIDE = 14;
__host__ __device__ constexpr int bc_src(int col) {  // 18-column source of compact column `col`
  return col == BC_Q4 ? B_Q4 : col == BC_S4 ? B_S4 : col == BC_R ? B_R : col == BC_P ? B_P
       : col == BC_ARM2 ? B_ARM2 : col;  // BC_Q0..BC_BB4 coincide with B_Q0..B_BB4
}
static_assert((int)BC_BB4 == (int)B_BB4 && (int)BC_Q0 == (int)B_Q0, "compact columns 0..7 mirror the full table");

// pos = table position of the row, step = positions between rows k-2 and k
// (2 in the both-parity table, whose position is k + 4; 1 in a one-parity table)
__device__ __forceinline__ void load_bih_row_compact(const double* stab, int pos, int step, double* c) {
  const double2* r0 = reinterpret_cast<const double2*>(stab + (int64_t)pos * BC_STRIDE);
  double v[BC_STRIDE];
#pragma unroll
  for (int q = 0; q < BC_STRIDE / 2; ++q) {
    const double2 t = r0[q];
    v[2 * q] = t.x;
    v[2 * q + 1] = t.y;
  }
  c[B_Q0] = v[BC_Q0]; c[B_AR0] = v[BC_AR0]; c[B_BB0] = v[BC_BB0];
  c[B_T2] = v[BC_T2]; c[B_AR2] = v[BC_AR2]; c[B_BB2] = v[BC_BB2];
  c[B_T4] = v[BC_T4]; c[B_BB4] = v[BC_BB4]; c[B_ARM2] = v[BC_ARM2];
  c[B_P] = v[BC_P]; c[B_R] = v[BC_R]; c[B_Q4] = v[BC_Q4]; c[B_S4] = v[BC_S4];
  const double* rm2 = stab + (int64_t)(pos - step) * BC_STRIDE;
  const double2 qs = *reinterpret_cast<const double2*>(rm2 + BC_Q4);
  c[B_Q2] = qs.x;
  c[B_S2] = qs.y;
  c[B_BB2M] = rm2[BC_BB2];
  c[B_BB4M] = stab[(int64_t)(pos - 2 * step) * BC_STRIDE + BC_BB4];
}

// Sliding variant for consecutive rows k, k+2, k+4, ... of one parity: the
// row-(k-2) / row-(k-4) entries are the previous rows' own values, so they
// are carried in registers instead of re-read (7 instead of 10 shared loads
// per row).  bih_carry_init loads them for the first row of a run.
struct BihCarry {
  double q4, s4, bb2, bb4, bb4_prev;  // rows k-2 (q4, s4, bb2, bb4) and k-4 (bb4_prev)
};
__device__ __forceinline__ void bih_carry_init(const double* stab, int pos, int step, BihCarry& cr) {
  const double* rm2 = stab + (int64_t)(pos - step) * BC_STRIDE;
  const double2 qs = *reinterpret_cast<const double2*>(rm2 + BC_Q4);
  cr.q4 = qs.x;
  cr.s4 = qs.y;
  cr.bb2 = rm2[BC_BB2];
  cr.bb4 = rm2[BC_BB4];
  cr.bb4_prev = stab[(int64_t)(pos - 2 * step) * BC_STRIDE + BC_BB4];
}
__device__ __forceinline__ void load_bih_row_carry(const double* stab, int pos, double* c, BihCarry& cr) {
  const double2* r0 = reinterpret_cast<const double2*>(stab + (int64_t)pos * BC_STRIDE);
  double v[BC_STRIDE];
#pragma unroll
  for (int q = 0; q < BC_STRIDE / 2; ++q) {
    const double2 t = r0[q];
    v[2 * q] = t.x;
    v[2 * q + 1] = t.y;
  }
  c[B_Q0] = v[BC_Q0]; c[B_AR0] = v[BC_AR0]; c[B_BB0] = v[BC_BB0];
  c[B_T2] = v[BC_T2]; c[B_AR2] = v[BC_AR2]; c[B_BB2] = v[BC_BB2];
  c[B_T4] = v[BC_T4]; c[B_BB4] = v[BC_BB4]; c[B_ARM2] = v[BC_ARM2];
  c[B_P] = v[BC_P]; c[B_R] = v[BC_R]; c[B_Q4] = v[BC_Q4]; c[B_S4] = v[BC_S4];
  c[B_Q2] = cr.q4;
  c[B_S2] = cr.s4;
  c[B_BB2M] = cr.bb2;
  c[B_BB4M] = cr.bb4_prev;
  cr.bb4_prev = cr.bb4;
  cr.q4 = v[BC_Q4];
  cr.s4 = v[BC_S4];
  cr.bb2 = v[BC_BB2];
  cr.bb4 = v[BC_BB4];
}

struct BihBands {
  double hd, hp2, hp4, hm2, hm4;
};

__device__ __forceinline__ BihBands bih_bands(double xi0, double xi1, double xi2, const double* c) {
  BihBands b;
  b.hd = __dadd_rn(__dadd_rn(__dmul_rn(xi0, c[B_Q0]), __dmul_rn(xi1, c[B_AR0])), __dmul_rn(xi2, c[B_BB0]));
  b.hp2 = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(xi0, c[B_T2]), 0.0), __dmul_rn(xi1, c[B_AR2])),
                    __dmul_rn(xi2, c[B_BB2]));
  b.hp4 = __dadd_rn(__dadd_rn(__dmul_rn(xi0, c[B_T4]), 0.0), __dmul_rn(xi2, c[B_BB4]));
  b.hm2 = __dadd_rn(__dmul_rn(xi1, c[B_ARM2]), __dmul_rn(xi2, c[B_BB2M]));
  b.hm4 = __dmul_rn(xi2, c[B_BB4M]);
  return b;
}

// U-row record (d, e, f, a, b) of one eliminated row (+ 1/d in fast mode).
struct BihU {
  double d, e, f, a, b, rd;
};

// fast-mode reciprocal of a U row's pivot
__device__ __forceinline__ void bih_set_rcp(BihU& u) { u.rd = rcp_fast(u.d); }
// zero record ("row before row 0")
__device__ __forceinline__ void bih_clear_rcp(BihU& u) { u.rd = 0.0; }

// One exact-mode elimination step, rows i-1 (u1) and i-2 (u2) already
// eliminated (solvers.py:314-346), numpy's evaluation order.  i is the row
// within the parity.  Returns l2, l4.  (Fast mode: bih_step_fast below.)
__device__ __forceinline__ void bih_step_exact(BihU& u, const BihU& u1, const BihU& u2, const BihBands& h,
                                               const double* c, double xi0, int i, double& l2, double& l4) {
  if (i == 0) {
    u.d = h.hd;
    u.e = h.hp2;
    u.f = h.hp4;
    u.a = c[B_P];
    u.b = c[B_R];
    l2 = 0.0;
    l4 = 0.0;
  } else if (i == 1) {
    l4 = 0.0;
    l2 = __ddiv_rn(h.hm2, u1.d);
    const double u24 = __dmul_rn(xi0, __dadd_rn(__dmul_rn(u1.a, c[B_Q4]), __dmul_rn(u1.b, c[B_S4])));
    u.d = __dsub_rn(h.hd, __dmul_rn(l2, u1.e));
    u.e = __dsub_rn(h.hp2, __dmul_rn(l2, u1.f));
    u.f = __dsub_rn(h.hp4, __dmul_rn(l2, u24));
    u.a = __dsub_rn(c[B_P], __dmul_rn(l2, u1.a));
    u.b = __dsub_rn(c[B_R], __dmul_rn(l2, u1.b));
  } else {
    l4 = __ddiv_rn(h.hm4, u2.d);
    const double tmp = __dsub_rn(h.hm2, __dmul_rn(l4, u2.e));
    l2 = __ddiv_rn(tmp, u1.d);
    const double u42 = __dmul_rn(xi0, __dadd_rn(__dmul_rn(u2.a, c[B_Q2]), __dmul_rn(u2.b, c[B_S2])));
    const double u44 = __dmul_rn(xi0, __dadd_rn(__dmul_rn(u2.a, c[B_Q4]), __dmul_rn(u2.b, c[B_S4])));
    const double u24 = __dmul_rn(xi0, __dadd_rn(__dmul_rn(u1.a, c[B_Q4]), __dmul_rn(u1.b, c[B_S4])));
    u.d = __dsub_rn(__dsub_rn(h.hd, __dmul_rn(l4, u2.f)), __dmul_rn(l2, u1.e));
    u.e = __dsub_rn(__dsub_rn(h.hp2, __dmul_rn(l4, u42)), __dmul_rn(l2, u1.f));
    u.f = __dsub_rn(__dsub_rn(h.hp4, __dmul_rn(l4, u44)), __dmul_rn(l2, u24));
    u.a = __dsub_rn(__dsub_rn(c[B_P], __dmul_rn(l2, u1.a)), __dmul_rn(l4, u2.a));
    u.b = __dsub_rn(__dsub_rn(c[B_R], __dmul_rn(l2, u1.b)), __dmul_rn(l4, u2.b));
  }
  u.rd = 0.0;
}

// ---- fast mode (build checkpoints, chunked and streaming solves) ----------
// Own arithmetic, shared bit for bit by every fast-mode kernel: the row
// constants that multiply xi0 (Q0, T2, T4 of the bands, p_k and r_k of the
// tail) are pre-scaled by xi0 (bih_fast_prescale), and the tail factors are
// carried pre-scaled by xi0 (a~ = xi0 a, b~ = xi0 b), which removes every xi0
// product from the rows.  Checkpoints therefore hold a~, b~.
__device__ __forceinline__ void bih_fast_prescale(double* c, double xi0) {
  c[B_Q0] = __dmul_rn(xi0, c[B_Q0]);
  c[B_T2] = __dmul_rn(xi0, c[B_T2]);
  c[B_T4] = __dmul_rn(xi0, c[B_T4]);
  c[B_P] = __dmul_rn(xi0, c[B_P]);
  c[B_R] = __dmul_rn(xi0, c[B_R]);
}
// The bands keep the reference's rounding order exactly (no contraction):
// they ARE the operator's entries, and an FMA-rounded entry differs from the
// matrix the reference (and the residual check) works with by an ulp of the
// largest, mutually cancelling term -- measured: 18 of 64 config-4 systems
// above a 1e-12 residual with FMA bands against 3 for the reference.  With
// the xi0 products pre-scaled (bit-identical to computing them in place)
// this costs 14 instead of 19 fp64 ops per row.
__device__ __forceinline__ BihBands bih_bands_fast(double xi1, double xi2, const double* c) {
  BihBands b;
  b.hd = __dadd_rn(__dadd_rn(c[B_Q0], __dmul_rn(xi1, c[B_AR0])), __dmul_rn(xi2, c[B_BB0]));
  b.hp2 = __dadd_rn(__dadd_rn(c[B_T2], __dmul_rn(xi1, c[B_AR2])), __dmul_rn(xi2, c[B_BB2]));
  b.hp4 = __dadd_rn(c[B_T4], __dmul_rn(xi2, c[B_BB4]));
  b.hm2 = __dadd_rn(__dmul_rn(xi1, c[B_ARM2]), __dmul_rn(xi2, c[B_BB2M]));
  b.hm4 = __dmul_rn(xi2, c[B_BB4M]);
  return b;
}

// Branch-free fast-mode biharmonic step.  Rows "before row 0" are zero
// records with rd = 0, which makes the generic formula reproduce rows 0 and 1
// (fma(-0, 0, x) == x).
__device__ __forceinline__ void bih_step_fast(BihU& u, const BihU& u1, const BihU& u2, const BihBands& h,
                                              const double* c, double& l2, double& l4) {
  l4 = __dmul_rn(h.hm4, u2.rd);
  const double tmp = __fma_rn(-l4, u2.e, h.hm2);
  l2 = __dmul_rn(tmp, u1.rd);
  const double u42 = __fma_rn(u2.a, c[B_Q2], __dmul_rn(u2.b, c[B_S2]));
  const double u44 = __fma_rn(u2.a, c[B_Q4], __dmul_rn(u2.b, c[B_S4]));
  const double u24 = __fma_rn(u1.a, c[B_Q4], __dmul_rn(u1.b, c[B_S4]));
  u.d = __fma_rn(-l2, u1.e, __fma_rn(-l4, u2.f, h.hd));
  u.e = __fma_rn(-l2, u1.f, __fma_rn(-l4, u42, h.hp2));
  u.f = __fma_rn(-l2, u24, __fma_rn(-l4, u44, h.hp4));
  u.a = __fma_rn(-l4, u2.a, __fma_rn(-l2, u1.a, c[B_P]));
  u.b = __fma_rn(-l4, u2.b, __fma_rn(-l2, u1.b, c[B_R]));
  bih_set_rcp(u);
}

// Row step for consecutive rows of one parity with the products that repeat
// between rows carried in registers (same operations on the same operands as
// bih_bands_fast + bih_step_fast, so bit-identical results):
//   xi2 BB2(k-2) and xi2 BB4(k-4) of hm2 / hm4 are the previous rows'
//   xi2 BB2 / xi2 BB4 products of hp2 / hp4;
//   u42 of row i (a, b of row i-2 against q, s of mode k+2) is u24 of row i-1.
struct BihProd {
  double x2bb2, x2bb4, x2bb4_prev, u42;
};
__device__ __forceinline__ void bih_prod_init(double xi2, const BihCarry& cr, BihProd& pr) {
  pr.x2bb2 = __dmul_rn(xi2, cr.bb2);
  pr.x2bb4 = __dmul_rn(xi2, cr.bb4);
  pr.x2bb4_prev = __dmul_rn(xi2, cr.bb4_prev);
  pr.u42 = 0.0;
}
__device__ __forceinline__ void bih_row_fast_carried(BihU& u, const BihU& u1, const BihU& u2, const double* c,
                                                     double xi1, double xi2, BihProd& pr, bool first, double& l2,
                                                     double& l4) {
  const double x2bb2 = __dmul_rn(xi2, c[B_BB2]);
  const double x2bb4 = __dmul_rn(xi2, c[B_BB4]);
  BihBands h;
  h.hd = __dadd_rn(__dadd_rn(c[B_Q0], __dmul_rn(xi1, c[B_AR0])), __dmul_rn(xi2, c[B_BB0]));
  h.hp2 = __dadd_rn(__dadd_rn(c[B_T2], __dmul_rn(xi1, c[B_AR2])), x2bb2);
  h.hp4 = __dadd_rn(c[B_T4], x2bb4);
  h.hm2 = __dadd_rn(__dmul_rn(xi1, c[B_ARM2]), pr.x2bb2);
  h.hm4 = pr.x2bb4_prev;
  l4 = __dmul_rn(h.hm4, u2.rd);
  const double tmp = __fma_rn(-l4, u2.e, h.hm2);
  l2 = __dmul_rn(tmp, u1.rd);
  const double u42 = first ? __fma_rn(u2.a, c[B_Q2], __dmul_rn(u2.b, c[B_S2])) : pr.u42;
  const double u44 = __fma_rn(u2.a, c[B_Q4], __dmul_rn(u2.b, c[B_S4]));
  const double u24 = __fma_rn(u1.a, c[B_Q4], __dmul_rn(u1.b, c[B_S4]));
  u.d = __fma_rn(-l2, u1.e, __fma_rn(-l4, u2.f, h.hd));
  u.e = __fma_rn(-l2, u1.f, __fma_rn(-l4, u42, h.hp2));
  u.f = __fma_rn(-l2, u24, __fma_rn(-l4, u44, h.hp4));
  u.a = __fma_rn(-l4, u2.a, __fma_rn(-l2, u1.a, c[B_P]));
  u.b = __fma_rn(-l4, u2.b, __fma_rn(-l2, u1.b, c[B_R]));
  bih_set_rcp(u);
  pr.u42 = u24;
  pr.x2bb4_prev = pr.x2bb4;
  pr.x2bb4 = x2bb4;
  pr.x2bb2 = x2bb2;
}

}  // namespace shen
