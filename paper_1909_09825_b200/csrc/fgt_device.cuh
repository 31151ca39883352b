// Device-side building blocks of the SOE fast Gauss transform hot path.
//
// The reference evaluates, per folded SOE mode k (proj/src/transform.cpp:119-149),
//     h+_k(x_i) = sum_{y_j <= x_i} beta_j exp(-s_k (x_i - y_j))
//     h-_k(x_i) = sum_{y_j >  x_i} beta_j exp(-s_k (y_j - x_i)),   s_k = t_k/sqrt(delta)
// with two sequential merge sweeps, then u = Re sum_k mw_k (h+ + h-)
// (transform.cpp:151-196).
//
// Here the sorted targets and sources are viewed as ONE merged stream
// z_0 <= z_1 <= ... (sources before targets at equal coordinates, which is the
// reference's "y == x joins the forward pass with factor 1", transform.hpp:69-72).
// Each element i carries a gap g_i = z_i - z_{i-1} and a weight b_i (beta for a
// source, 0 for a target).  With d_i = decay(s_k, g_i):
//     forward   H_i = d_i H_{i-1} + b_i            (H at a target = h+)
//     backward  K_{i-1} = d_i (K_i + b_i)          (K at a target = h-)
// Both are first-order linear recurrences, i.e. scans under the associative
// operator (A, S) o (A', S') = (A A', A' S + S').  The stream is cut into
// tiles (one CTA) -> lane runs of R consecutive elements (one thread).
// See DESIGN.md for the full decomposition and the error analysis.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fgt_b200 {

constexpr int kMaxModes = 8;   // folded modes (reference presets use 3..7)
constexpr int kMaxDeg = 16;    // highest Taylor degree of the gap-factor fast path
constexpr double kUnderflowExponent = 745.0;  // transform.cpp:19

// Per-launch mode constants (kernel parameter, lives in the constant bank).
struct ModeParams {
  int ne;
  double s_re[kMaxModes], s_im[kMaxModes];    // s_k = t_k / sqrt(delta)
  double mw_re[kMaxModes], mw_im[kMaxModes];  // m_k * w_k
  double smax;                                // max_k |s_k|
  // rmax[D]: largest |s|*g for which the degree-D Taylor polynomial of
  // exp(-s g) has truncation error below 2^-FGT_TRUNC_BITS (relative).
  double rmax[kMaxDeg + 1];
};

struct cplx {
  double re, im;
};

__device__ __forceinline__ cplx cmul(cplx a, cplx b) {
  return {fma(a.re, b.re, -a.im * b.im), fma(a.re, b.im, a.im * b.re)};
}
// a*c + s  (complex a, c, s)
__device__ __forceinline__ cplx cmad(cplx a, cplx c, cplx s) {
  return {fma(a.re, c.re, fma(-a.im, c.im, s.re)), fma(a.re, c.im, fma(a.im, c.re, s.im))};
}

// Exact gap factor, the device restatement of decay_factor
// (transform.cpp:60-68): 1 for g == 0, exact 0 past the underflow threshold,
// otherwise exp(-a) (cos b - i sin b) with a = Re(s) g, b = Im(s) g.
__device__ __forceinline__ cplx decay_exact(double sre, double sim, double g) {
  double a = sre * g;
  if (a > kUnderflowExponent) return {0.0, 0.0};
  double e = exp(-a);
  double sn, cs;
  sincos(sim * g, &sn, &cs);
  return {e * cs, -e * sn};
}

// Warp-uniform Taylor degree for a max scaled gap r = smax * gmax;
// -1 selects the exact path.
__device__ __forceinline__ int pick_degree(const ModeParams& P, double smax, double gmax) {
  double r = smax * gmax;
  if (!(r == r)) return -1;
#pragma unroll
  for (int D = 0; D <= kMaxDeg; ++D)
    if (r <= P.rmax[D]) return D;
  return -1;
}

}  // namespace fgt_b200
