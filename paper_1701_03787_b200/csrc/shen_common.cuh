// Shared device helpers for the B200 Shen solvers (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define SHEN_PIVOT_FLOOR 1e-300  // reference solvers.py:54

namespace shen {

// ---------------------------------------------------------------- values
// The right-hand side is complex128 (interleaved re/im) or float64.  Both
// map onto V below so every recurrence is written once.
struct cplx {
  double re, im;
};

__device__ __forceinline__ cplx make_v(double r, double i) { return {r, i}; }

template <typename V> struct VOps;

template <> struct VOps<double> {
  static __device__ __forceinline__ double zero() { return 0.0; }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double scale(double s, double a) { return __dmul_rn(s, a); }
  // a - s*b with the product rounded first (numpy order, no contraction)
  static __device__ __forceinline__ double sub_sc(double a, double s, double b) {
    return __dsub_rn(a, __dmul_rn(s, b));
  }
  // a + s*b fused (fast paths)
  static __device__ __forceinline__ double fma_sc(double s, double b, double a) { return __fma_rn(s, b, a); }
  static __device__ __forceinline__ double ld(const double* p) { return __ldg(p); }
  static __device__ __forceinline__ void st(double* p, double v) { *p = v; }
  static __device__ __forceinline__ double ld_cs(const double* p) { return __ldcs(p); }
  static __device__ __forceinline__ void st_cs(double* p, double v) { __stcs(p, v); }
  static constexpr int ndouble = 1;
};

template <> struct VOps<cplx> {
  static __device__ __forceinline__ cplx zero() { return {0.0, 0.0}; }
  static __device__ __forceinline__ cplx add(cplx a, cplx b) { return {__dadd_rn(a.re, b.re), __dadd_rn(a.im, b.im)}; }
  static __device__ __forceinline__ cplx sub(cplx a, cplx b) { return {__dsub_rn(a.re, b.re), __dsub_rn(a.im, b.im)}; }
  static __device__ __forceinline__ cplx scale(double s, cplx a) { return {__dmul_rn(s, a.re), __dmul_rn(s, a.im)}; }
  static __device__ __forceinline__ cplx sub_sc(cplx a, double s, cplx b) {
    return {__dsub_rn(a.re, __dmul_rn(s, b.re)), __dsub_rn(a.im, __dmul_rn(s, b.im))};
  }
  static __device__ __forceinline__ cplx fma_sc(double s, cplx b, cplx a) {
    return {__fma_rn(s, b.re, a.re), __fma_rn(s, b.im, a.im)};
  }
  static __device__ __forceinline__ cplx ld(const cplx* p) {
    double2 v = __ldg(reinterpret_cast<const double2*>(p));
    return {v.x, v.y};
  }
  static __device__ __forceinline__ void st(cplx* p, cplx v) {
    *reinterpret_cast<double2*>(p) = make_double2(v.re, v.im);
  }
  // streaming (evict-first) variants for the once-touched RHS / solution
  static __device__ __forceinline__ cplx ld_cs(const cplx* p) {
    double2 v = __ldcs(reinterpret_cast<const double2*>(p));
    return {v.x, v.y};
  }
  static __device__ __forceinline__ void st_cs(cplx* p, cplx v) {
    __stcs(reinterpret_cast<double2*>(p), make_double2(v.re, v.im));
  }
  static constexpr int ndouble = 2;
};

__device__ __forceinline__ double shfl_up_d(double v, int d) { return __shfl_up_sync(0xffffffffu, v, d); }
__device__ __forceinline__ double shfl_down_d(double v, int d) { return __shfl_down_sync(0xffffffffu, v, d); }
__device__ __forceinline__ cplx shfl_up_v(cplx v, int d) { return {shfl_up_d(v.re, d), shfl_up_d(v.im, d)}; }
__device__ __forceinline__ cplx shfl_down_v(cplx v, int d) { return {shfl_down_d(v.re, d), shfl_down_d(v.im, d)}; }
__device__ __forceinline__ double shfl_up_v(double v, int d) { return shfl_up_d(v, d); }
__device__ __forceinline__ double shfl_down_v(double v, int d) { return shfl_down_d(v, d); }

// pivot bookkeeping: the reference raises at the first row (parity 0 rows
// first, then parity 1) where any system of the batch has |d| < 1e-300.
__device__ __forceinline__ void note_pivot(int* pivot, int par, int row_in_parity, double d) {
  if (pivot != nullptr && fabs(d) < SHEN_PIVOT_FLOOR) atomicMin(pivot + par, row_in_parity);
}

}  // namespace shen
