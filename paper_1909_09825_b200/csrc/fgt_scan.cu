// Merged-stream SOE scan kernels (sm_100a).  Hot path of the fast Gauss
// transform: replaces run_mode_general / run_mode_same / apply_common of the
// reference (proj/src/transform.cpp:97-149, 151-196).
//
//   K0 partition : merge-path split of the (targets, sources) stream into
//                  segments of kSeg merged elements (one warp each)
//   K1 aggregate : per segment and mode, the scan aggregate (A, F, G) from the
//                  real moments of the segment's sources (mode independent,
//                  streamed once); exact per-element fallback for wide segments
//   K2 carry scan: exclusive scan of the segment aggregates, both directions
//                  (reduce / top / down-sweep)
//   K3 main      : per warp: lane runs of kR merged elements in registers,
//                  lane aggregates from lane moments, sequential lane carries,
//                  forward/backward recurrences with the fused weighted
//                  real-part combine, staged coalesced write / scatter of u
//
// Scan operator on (A, S): (A, S) then (A', S') = (A A', A' S + S').
// Forward state at the element before a unit: Cf; after the unit it is
// A Cf + F.  Backward state at the unit's last element: Cb; before the unit
// (at the element preceding it) it is A Cb + G.
#include <cuda_runtime.h>
#include <math.h>

#include "fgt_scan.cuh"
#include "fgt_sort.cuh"

namespace fgt_b200 {

namespace {

struct LaneAgg {
  cplx A, F, G;
};

// ---------------------------------------------------------------- helpers

// Number of targets among the first `diag` merged elements.  Merged order:
// a source precedes a target unless the target is strictly smaller
// (sources before targets at equal coordinates, transform.cpp:140-143).
template <class Ptr>
__device__ __forceinline__ int64_t merge_path(Ptr x, int64_t nx, Ptr y, int64_t ny,
                                              int64_t diag) {
  int64_t lo = diag - ny > 0 ? diag - ny : 0;
  int64_t hi = diag < nx ? diag : nx;
  while (lo < hi) {
    int64_t mid = (lo + hi + 1) >> 1;
    if (x[mid - 1] < y[diag - mid])
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

// Coefficients of one mode: held in registers up to degree kRegDeg, read
// from shared memory (broadcast) above it to bound register pressure.
constexpr int kRegDeg = 8;

template <int D>
struct Coef {
  cplx c[(D >= 0 && D <= kRegDeg) ? D + 1 : 1];
  const cplx* sm;
  __device__ __forceinline__ void load(const ModeTable& mt, int k) {
    sm = mt.coef[k];
    if constexpr (D >= 0 && D <= kRegDeg) {
#pragma unroll
      for (int n = 0; n <= D; ++n) c[n] = sm[n];
    }
  }
  __device__ __forceinline__ cplx operator[](int n) const {
    if constexpr (D >= 0 && D <= kRegDeg) {
      return c[n];
    } else {
      return sm[n];
    }
  }
};

template <int D>
__device__ __forceinline__ cplx horner(const Coef<D>& c, double g) {
  cplx t = c[D];
  double pr = t.re, pi = t.im;
#pragma unroll
  for (int n = D - 1; n >= 0; --n) {
    const cplx cn = c[n];
    pr = fma(pr, g, cn.re);
    pi = fma(pi, g, cn.im);
  }
  return {pr, pi};
}

// Gap factor exp(-s g): Taylor polynomial of degree D (fast path) or exact.
template <int D>
__device__ __forceinline__ cplx gap_factor(const Coef<D>& c, cplx s, double g) {
  if constexpr (D >= 0) {
    return horner<D>(c, g);
  } else {
    return decay_exact(s.re, s.im, g);
  }
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ void load_mode_table(const ModeTable* g, ModeTable& s) {
  const double* src = reinterpret_cast<const double*>(g);
  double* dst = reinterpret_cast<double*>(&s);
  constexpr int n = sizeof(ModeTable) / sizeof(double);
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

// ---------------------------------------------------------------- geometry

struct SegGeom {
  int64_t ib, jb;  // first target / source of the segment
  int nx, ny, len;
  double zprev;  // coordinate of the merged element preceding the segment
  double zlast;  // coordinate of the segment's last merged element
};

__device__ __forceinline__ SegGeom seg_geom(const StreamArgs& a, int64_t s) {
  SegGeom g;
  const int64_t L = a.M + a.N;
  const int64_t d0 = s * kSeg;
  const int64_t d1 = (d0 + kSeg < L) ? d0 + kSeg : L;
  g.ib = a.seg_ib[s];
  const int64_t ie = a.seg_ib[s + 1];
  const double2 z = a.seg_z[s];
  g.jb = d0 - g.ib;
  const int64_t je = d1 - ie;
  g.nx = (int)(ie - g.ib);
  g.ny = (int)(je - g.jb);
  g.len = (int)(d1 - d0);
  g.zprev = s == 0 ? a.zprev0 : z.x;
  g.zlast = z.y;
  return g;
}

// ------------------------------------------------------------- lane runs

struct LaneRun {
  double g[kR];  // gap to the previous merged element
  double b[kR];  // strength if source, 0 if target / padding
  unsigned tmask;  // bit e: element e is a target
  int tfirst;      // segment-local index of the lane's first target
  double gmax;     // largest gap
  double span;     // last coordinate of the run minus the coordinate before it
};

// Lane run from the plan-time merge mask: no merge, no shared-memory
// staging; every element is an independent load.
__device__ __forceinline__ void lane_load(const StreamArgs& a, const SegGeom& g, int64_t s,
                                          int lane, LaneRun& r) {
  const uint32_t word = __ldg(a.seg_mask + s * (kSeg / 32) + (lane >> 2));
  const int d0 = lane * kR;
  const int nreal = g.len - d0 < 0 ? 0 : (g.len - d0 < kR ? g.len - d0 : kR);
  const unsigned live = nreal >= 32 ? 0xffffffffu : ((1u << nreal) - 1u);
  const unsigned byte = (word >> ((lane & 3) * 8)) & 0xffu & live;
  const int nt = __popc(byte);
  // exclusive warp prefix of the target counts
  int incl = nt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const int i0 = incl - nt;
  const int j0 = (d0 < g.len ? d0 : g.len) - i0;
  r.tfirst = i0;
  r.tmask = byte;
  double z[kR];
  double last = 0.0;
#pragma unroll
  for (int e = 0; e < kR; ++e) {
    const int t = __popc(byte & ((1u << e) - 1u));
    const int sidx = e - t;
    if (e < nreal) {
      if (byte & (1u << e)) {
        z[e] = __ldg(a.xs + g.ib + i0 + t);
        r.b[e] = 0.0;
      } else {
        z[e] = __ldg(a.ys + g.jb + j0 + sidx);
        r.b[e] = __ldg(a.bs + g.jb + j0 + sidx);
      }
      last = z[e];
    } else {
      z[e] = 0.0;
      r.b[e] = 0.0;
    }
  }
  // coordinate preceding the run: the previous lane's last element
  double prev = __shfl_up_sync(0xffffffffu, last, 1);
  if (lane == 0) prev = g.zprev;
  const double start = prev;
  r.gmax = 0.0;
#pragma unroll
  for (int e = 0; e < kR; ++e) {
    if (e < nreal) {
      r.g[e] = z[e] - prev;
      prev = z[e];
    } else {
      r.g[e] = 0.0;
    }
    r.gmax = fmax(r.gmax, r.g[e]);
  }
  r.span = nreal > 0 ? prev - start : 0.0;
}

// --------------------------------------------------------------- pass 1

// Exact per-element lane aggregates (robust path for wide runs):
//   A = prod d_i, F = forward state at the run end, G = backward state at
//   the element before the run.
template <int D>
__device__ __forceinline__ void pass1_elements(const ModeTable& mt, int ne, const LaneRun& r,
                                               LaneAgg* out) {
  for (int k = 0; k < ne; ++k) {
    Coef<D> c;
    c.load(mt, k);
    const cplx s = mt.s[k];
    cplx F = {0.0, 0.0}, P = {1.0, 0.0}, G = {0.0, 0.0};
#pragma unroll
    for (int i = 0; i < kR; ++i) {
      const cplx d = gap_factor<D>(c, s, r.g[i]);
      F = cmad(d, F, cplx{r.b[i], 0.0});
      P = cmul(P, d);
      G.re = fma(r.b[i], P.re, G.re);
      G.im = fma(r.b[i], P.im, G.im);
    }
    out[k] = LaneAgg{P, F, G};
  }
}

// Moment form of the lane aggregates: with h = span/2 and d_i the position of
// source i relative to the run's midpoint,
//   F = e^{-s h} sum_i b_i e^{+s d_i},  G = e^{-s h} sum_i b_i e^{-s d_i},
//   A = (e^{-s h})^2,
// and e^{-/+ s d} = sum_n (-/+ s)^n d^n / n! truncated at DM (|s| h <= rmax[DM]),
// so the per-source work is mode independent: M_n = sum_i b_i d_i^n.
template <int DM>
__device__ __forceinline__ void pass1_moments(const ModeTable& mt, int ne, const LaneRun& r,
                                              LaneAgg* out) {
  const double h = 0.5 * r.span;
  double M[DM + 1];
#pragma unroll
  for (int n = 0; n <= DM; ++n) M[n] = 0.0;
  double pos = 0.0;
#pragma unroll
  for (int i = 0; i < kR; ++i) {
    pos += r.g[i];
    const double d = pos - h;
    double p = r.b[i];
    M[0] += p;
#pragma unroll
    for (int n = 1; n <= DM; ++n) {
      p *= d;
      M[n] += p;
    }
  }
  for (int k = 0; k < ne; ++k) {
    Coef<DM> c;
    c.load(mt, k);
    cplx ev = {0.0, 0.0}, od = {0.0, 0.0};
#pragma unroll
    for (int n = 0; n <= DM; ++n) {
      if (n & 1) {
        od.re = fma(c[n].re, M[n], od.re);
        od.im = fma(c[n].im, M[n], od.im);
      } else {
        ev.re = fma(c[n].re, M[n], ev.re);
        ev.im = fma(c[n].im, M[n], ev.im);
      }
    }
    const cplx E = horner<DM>(c, h);
    out[k].A = cmul(E, E);
    out[k].F = cmul(E, cplx{ev.re - od.re, ev.im - od.im});
    out[k].G = cmul(E, cplx{ev.re + od.re, ev.im + od.im});
  }
}

__device__ __forceinline__ void dispatch_pass1(int D, int DM, const ModeTable& mt, int ne,
                                               const LaneRun& r, LaneAgg* out) {
  if (D >= 0 && DM >= 0) {
    switch (DM) {
#define FGT_P1M(n)                           \
  case n:                                    \
    pass1_moments<n>(mt, ne, r, out);        \
    return;
      FGT_P1M(0) FGT_P1M(1) FGT_P1M(2) FGT_P1M(3) FGT_P1M(4) FGT_P1M(5) FGT_P1M(6)
      FGT_P1M(7) FGT_P1M(8)
#undef FGT_P1M
      default:
        break;
    }
  }
  switch (D) {
#define FGT_P1E(n)                           \
  case n:                                    \
    pass1_elements<n>(mt, ne, r, out);       \
    return;
    FGT_P1E(0) FGT_P1E(1) FGT_P1E(2) FGT_P1E(3) FGT_P1E(4) FGT_P1E(5) FGT_P1E(6) FGT_P1E(7)
    FGT_P1E(8) FGT_P1E(9) FGT_P1E(10) FGT_P1E(11) FGT_P1E(12) FGT_P1E(13) FGT_P1E(14)
    FGT_P1E(15) FGT_P1E(16)
#undef FGT_P1E
    default:
      pass1_elements<-1>(mt, ne, r, out);
  }
}

// --------------------------------------------------------------- pass 2

// Mode-sums test hook (detail::mode_sums, transform.cpp:310-350): store H
// (= h+) and K (= h-) of every target per mode instead of combining.
struct ModeSumsOut {
  cplx* hp;  // [ne][M]
  cplx* hm;
  int64_t M;
  int64_t t0;  // global sorted index of this lane's first target
};

// Forward and backward recurrences seeded with the lane carries (carry[k].F
// = forward state at the element before the run, carry[k].G = backward state
// at the run's last element), accumulating Re(mw_k (H + K)) into out[] (only
// target slots are used).  Gap factors are kept in registers between the two
// sweeps.
template <int D, bool MS>
__device__ __forceinline__ void pass2(const ModeTable& mt, int ne, const LaneRun& r,
                                      const LaneAgg* carry, double (&out)[kR],
                                      const ModeSumsOut& ms) {
  for (int k = 0; k < ne; ++k) {
    Coef<D> c;
    c.load(mt, k);
    const cplx s = mt.s[k];
    const cplx mw = mt.mw[k];
    cplx d[kR];
    cplx H = carry[k].F;
    int64_t ti = ms.t0;
#pragma unroll
    for (int i = 0; i < kR; ++i) {
      d[i] = gap_factor<D>(c, s, r.g[i]);
      H = cmad(d[i], H, cplx{r.b[i], 0.0});
      if constexpr (MS) {
        if (r.tmask & (1u << i)) ms.hp[(int64_t)k * ms.M + ti++] = H;
      } else {
        out[i] = fma(mw.re, H.re, fma(-mw.im, H.im, out[i]));
      }
    }
    cplx K = carry[k].G;
#pragma unroll
    for (int i = kR - 1; i >= 0; --i) {
      if constexpr (MS) {
        if (r.tmask & (1u << i)) ms.hm[(int64_t)k * ms.M + (--ti)] = K;
      } else {
        out[i] = fma(mw.re, K.re, fma(-mw.im, K.im, out[i]));
      }
      K = cmul(d[i], cplx{K.re + r.b[i], K.im});
    }
  }
}

template <bool MS>
__device__ __forceinline__ void dispatch_pass2(int D, const ModeTable& mt, int ne,
                                               const LaneRun& r, const LaneAgg* carry,
                                               double (&out)[kR], const ModeSumsOut& ms) {
  switch (D) {
#define FGT_P2(n)                                 \
  case n:                                         \
    pass2<n, MS>(mt, ne, r, carry, out, ms);      \
    break;
    FGT_P2(0) FGT_P2(1) FGT_P2(2) FGT_P2(3) FGT_P2(4) FGT_P2(5) FGT_P2(6) FGT_P2(7)
    FGT_P2(8) FGT_P2(9) FGT_P2(10) FGT_P2(11) FGT_P2(12) FGT_P2(13) FGT_P2(14)
    FGT_P2(15) FGT_P2(16)
#undef FGT_P2
    default:
      pass2<-1, MS>(mt, ne, r, carry, out, ms);
  }
}

// ------------------------------------------------- sequential lane scans
// Lanes q < 2 ne of a warp: q < ne forward for mode q, ne <= q < 2 ne
// backward for mode q - ne.  aggs is [32 lanes][ne].

// Exclusive lane carries written in place: forward into .F, backward into .G
__device__ __forceinline__ void lanes_carry(LaneAgg* aggs, int ne, int q, cplx cin) {
  if (q < ne) {
    cplx c = cin;
    for (int l = 0; l < 32; ++l) {
      LaneAgg& x = aggs[l * ne + q];
      const cplx A = x.A, F = x.F;
      x.F = c;
      c = cmad(A, c, F);
    }
  } else {
    const int k = q - ne;
    cplx c = cin;
    for (int l = 31; l >= 0; --l) {
      LaneAgg& x = aggs[l * ne + k];
      const cplx A = x.A, G = x.G;
      x.G = c;
      c = cmad(A, c, G);
    }
  }
}

// -------------------------------------------------------- shared memory

// Per-warp region of K3: lane aggregates / carries, then the output staging.
__host__ __device__ __forceinline__ size_t warp_region_bytes(int ne) {
  return sizeof(LaneAgg) * 32 * (size_t)ne + sizeof(double) * kSeg;
}

struct SegSmemView {
  LaneAgg* aggs;
  double* su;
};

__device__ __forceinline__ SegSmemView warp_smem(unsigned char* base, int ne, int warp) {
  unsigned char* w = base + (size_t)warp * warp_region_bytes(ne);
  SegSmemView v;
  v.aggs = reinterpret_cast<LaneAgg*>(w);
  v.su = reinterpret_cast<double*>(w + sizeof(LaneAgg) * 32 * (size_t)ne);
  return v;
}

// ------------------------------------------------------------------- K1

template <int DM>
__device__ __forceinline__ void seg_moments(const StreamArgs& a, const SegGeom& g, double h,
                                            int lane, double (&M)[kMaxMom + 1]) {
#pragma unroll
  for (int n = 0; n <= DM; ++n) M[n] = 0.0;
  for (int j = lane; j < g.ny; j += 32) {
    const double y = __ldg(a.ys + g.jb + j);
    double p = __ldg(a.bs + g.jb + j);
    const double d = (y - g.zprev) - h;
    M[0] += p;
#pragma unroll
    for (int n = 1; n <= DM; ++n) {
      p *= d;
      M[n] += p;
    }
  }
#pragma unroll
  for (int n = 0; n <= DM; ++n) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M[n] += __shfl_xor_sync(0xffffffffu, M[n], o);
  }
}

template <int DM>
__device__ __forceinline__ void seg_aggregate_moments(const StreamArgs& a, const SegGeom& g,
                                                      const ModeTable& mt, int ne, int lane,
                                                      int64_t s, TileState ts) {
  const double L = g.zlast - g.zprev;
  const double h = 0.5 * L;
  double M[kMaxMom + 1];
  seg_moments<DM>(a, g, h, lane, M);
  if (lane < ne) {
    const int k = lane;
    cplx ev = {0.0, 0.0}, od = {0.0, 0.0};
#pragma unroll
    for (int n = 0; n <= DM; ++n) {
      const cplx c = mt.coef[k][n];
      if (n & 1) {
        od.re = fma(c.re, M[n], od.re);
        od.im = fma(c.im, M[n], od.im);
      } else {
        ev.re = fma(c.re, M[n], ev.re);
        ev.im = fma(c.im, M[n], ev.im);
      }
    }
    Coef<DM> c;
    c.load(mt, k);
    const cplx E = horner<DM>(c, h);
    const int64_t o = (int64_t)k * a.nseg + s;
    ts.A[o] = cmul(E, E);
    ts.F[o] = cmul(E, cplx{ev.re - od.re, ev.im - od.im});
    ts.G[o] = cmul(E, cplx{ev.re + od.re, ev.im + od.im});
  }
}

// Ordered warp reduction of lane aggregates (lane 0 ends up with the total):
// forward (A, F) left-to-right, backward G = G_left + A_left G_right.
__device__ __forceinline__ LaneAgg warp_reduce_agg(LaneAgg v) {
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    LaneAgg r;
    r.A.re = __shfl_down_sync(0xffffffffu, v.A.re, off);
    r.A.im = __shfl_down_sync(0xffffffffu, v.A.im, off);
    r.F.re = __shfl_down_sync(0xffffffffu, v.F.re, off);
    r.F.im = __shfl_down_sync(0xffffffffu, v.F.im, off);
    r.G.re = __shfl_down_sync(0xffffffffu, v.G.re, off);
    r.G.im = __shfl_down_sync(0xffffffffu, v.G.im, off);
    if (((threadIdx.x & 31) & (2 * off - 1)) == 0) {
      const cplx F = cmad(r.A, v.F, r.F);
      const cplx G = cmad(v.A, r.G, v.G);
      v.A = cmul(v.A, r.A);
      v.F = F;
      v.G = G;
    }
  }
  return v;
}

// K1: one warp per segment.  Moment path when the segment is narrow
// (|s| h <= rmax[kRegDeg]); otherwise exact per-element lane aggregates from
// the merge mask, reduced across the warp.
__global__ void __launch_bounds__(kThreads)
    seg_aggregate_kernel(StreamArgs a, ModeParams P, const ModeTable* __restrict__ mtab,
                         TileState ts) {
  __shared__ ModeTable mt;
  load_mode_table(mtab, mt);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t s = (int64_t)blockIdx.x * kSegWarps + warp;
  if (s >= a.nseg) return;
  const int ne = P.ne;
  const SegGeom g = seg_geom(a, s);
  const int DM = pick_degree(P, 0.5 * (g.zlast - g.zprev));
  switch (DM) {
#define FGT_K1(n)                                                 \
  case n:                                                         \
    seg_aggregate_moments<n>(a, g, mt, ne, lane, s, ts);          \
    return;
    FGT_K1(0) FGT_K1(1) FGT_K1(2) FGT_K1(3) FGT_K1(4) FGT_K1(5) FGT_K1(6) FGT_K1(7)
    FGT_K1(8)
#undef FGT_K1
    default:
      break;
  }
  // Wide segment: exact per-element lane aggregates, ordered warp reduction.
  LaneRun r;
  lane_load(a, g, s, lane, r);
  for (int k = 0; k < ne; ++k) {
    const cplx sk = mt.s[k];
    cplx F = {0.0, 0.0}, Pp = {1.0, 0.0}, G = {0.0, 0.0};
#pragma unroll
    for (int i = 0; i < kR; ++i) {
      const cplx d = decay_exact(sk.re, sk.im, r.g[i]);
      F = cmad(d, F, cplx{r.b[i], 0.0});
      Pp = cmul(Pp, d);
      G.re = fma(r.b[i], Pp.re, G.re);
      G.im = fma(r.b[i], Pp.im, G.im);
    }
    const LaneAgg w = warp_reduce_agg(LaneAgg{Pp, F, G});
    if (lane == 0) {
      const int64_t o = (int64_t)k * a.nseg + s;
      ts.A[o] = w.A;
      ts.F[o] = w.F;
      ts.G[o] = w.G;
    }
  }
}

// ------------------------------------------------------------------- K3

template <bool MS>
__global__ void __launch_bounds__(kThreads, 4)
    seg_main_kernel(StreamArgs a, ModeParams P, const ModeTable* __restrict__ mtab,
                    TileState ts, OutArgs o) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ModeTable& mt = *reinterpret_cast<ModeTable*>(smem_raw);
  unsigned char* wbase = smem_raw + sizeof(ModeTable);
  load_mode_table(mtab, mt);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t s = (int64_t)blockIdx.x * kSegWarps + warp;
  if (s >= a.nseg) return;
  const int ne = P.ne;
  const SegGeom g = seg_geom(a, s);
  SegSmemView v = warp_smem(wbase, ne, warp);
  LaneRun r;
  lane_load(a, g, s, lane, r);
  const int D = pick_degree(P, warp_max(r.gmax));
  const int DM = pick_degree(P, warp_max(0.5 * r.span));

  LaneAgg* mine = v.aggs + lane * ne;
  dispatch_pass1(D, DM, mt, ne, r, mine);
  __syncwarp();
  if (lane < 2 * ne) {
    const int k = lane < ne ? lane : lane - ne;
    const int64_t idx = (int64_t)k * a.nseg + s;
    lanes_carry(v.aggs, ne, lane, lane < ne ? ts.Cf[idx] : ts.Cb[idx]);
  }
  __syncwarp();

  double out[kR];
#pragma unroll
  for (int e = 0; e < kR; ++e) out[e] = 0.0;
  if constexpr (MS) {
    ModeSumsOut ms{o.hp, o.hm, a.M, o.u_offset + g.ib + r.tfirst};
    dispatch_pass2<true>(D, mt, ne, r, mine, out, ms);
    return;
  } else {
    dispatch_pass2<false>(D, mt, ne, r, mine, out, ModeSumsOut{nullptr, nullptr, 0, 0});
    int tk = r.tfirst;
#pragma unroll
    for (int e = 0; e < kR; ++e)
      if (r.tmask & (1u << e)) v.su[tk++] = out[e];
    __syncwarp();
    const int64_t base = o.u_offset + g.ib;
    if (o.tperm) {
      for (int i = lane; i < g.nx; i += 32) o.u[o.tperm[base + i]] = v.su[i];
    } else {
      for (int i = lane; i < g.nx; i += 32) o.u[base + i] = v.su[i];
    }
  }
}

// ------------------------------------------------------------------- K0

__global__ void partition_kernel(const double* __restrict__ xs, int64_t M,
                                 const double* __restrict__ ys, int64_t N, int64_t seg,
                                 int64_t nseg, int64_t* __restrict__ seg_ib) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t > nseg) return;
  int64_t diag = t * seg;
  if (diag > M + N) diag = M + N;
  seg_ib[t] = merge_path(xs, M, ys, N, diag);
}

// Plan-time segment metadata, one warp per segment: merge the segment's runs
// straight from global memory once, record (zprev, zlast) and one bit per
// merged element (1 = target) so that the apply kernels never merge.
__global__ void __launch_bounds__(128)
    seg_meta_kernel(const double* __restrict__ xs, int64_t M, const double* __restrict__ ys,
                    int64_t N, const int64_t* __restrict__ seg_ib, int64_t nseg,
                    double2* __restrict__ seg_z, uint32_t* __restrict__ seg_mask) {
  const int lane = threadIdx.x & 31;
  const int64_t s = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (s >= nseg) return;
  const int64_t L = M + N;
  const int64_t d0 = s * kSeg;
  const int64_t d1 = (d0 + kSeg < L) ? d0 + kSeg : L;
  const int64_t ib = seg_ib[s], ie = seg_ib[s + 1];
  const int64_t jb = d0 - ib, je = d1 - ie;
  const int nx = (int)(ie - ib), ny = (int)(je - jb), len = (int)(d1 - d0);
  const double* x = xs + ib;
  const double* y = ys + jb;
  const int ld = lane * kR;
  const int dd = ld < len ? ld : len;
  int i = (int)merge_path(x, (int64_t)nx, y, (int64_t)ny, (int64_t)dd);
  int j = dd - i;
  unsigned byte = 0u;
#pragma unroll
  for (int e = 0; e < kR; ++e) {
    if (ld + e < len) {
      const bool src = (j < ny) && (i >= nx || y[j] <= x[i]);
      if (src) {
        ++j;
      } else {
        byte |= 1u << e;
        ++i;
      }
    }
  }
  unsigned w = byte << ((lane & 3) * 8);
  w |= __shfl_down_sync(0xffffffffu, w, 1);
  w |= __shfl_down_sync(0xffffffffu, w, 2);
  if ((lane & 3) == 0) seg_mask[s * (kSeg / 32) + (lane >> 2)] = w;
  if (lane == 0) {
    const double px = ib > 0 ? xs[ib - 1] : -INFINITY;
    const double py = jb > 0 ? ys[jb - 1] : -INFINITY;
    const double lx = nx > 0 ? xs[ie - 1] : -INFINITY;
    const double ly = ny > 0 ? ys[je - 1] : -INFINITY;
    seg_z[s] = make_double2(fmax(px, py), fmax(lx, ly));
  }
}

// ------------------------------------------------------------------- K2
// Scan of (a, s) pairs over segments, one (mode, direction) per blockIdx.y:
// q < ne forward of mode q over F, q >= ne backward of mode q - ne over G in
// reversed segment order.  Three phases: per-block reduce, top-level scan of
// block aggregates (one CTA per q), per-block down-sweep writing carries.

constexpr int kScanThreads = 256;
constexpr int kScanItems = 4;
constexpr int kScanBlock = kScanThreads * kScanItems;

struct Pair {
  cplx a, s;
};

// earlier x then later y
__device__ __forceinline__ Pair combine(Pair x, Pair y) {
  return Pair{cmul(x.a, y.a), cmad(y.a, x.s, y.s)};
}

__device__ __forceinline__ Pair shfl_up_pair(Pair p, int off) {
  Pair r;
  r.a.re = __shfl_up_sync(0xffffffffu, p.a.re, off);
  r.a.im = __shfl_up_sync(0xffffffffu, p.a.im, off);
  r.s.re = __shfl_up_sync(0xffffffffu, p.s.re, off);
  r.s.im = __shfl_up_sync(0xffffffffu, p.s.im, off);
  return r;
}

// Block-wide exclusive scan; returns the exclusive prefix of this thread and
// the block total.
__device__ __forceinline__ Pair block_exclusive(Pair v, Pair* total) {
  __shared__ Pair wtot[kScanThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Pair incl = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const Pair p = shfl_up_pair(incl, off);
    if (lane >= off) incl = combine(p, incl);
  }
  if (lane == 31) wtot[warp] = incl;
  __syncthreads();
  Pair wpre{{1.0, 0.0}, {0.0, 0.0}};
  for (int w = 0; w < warp; ++w) wpre = combine(wpre, wtot[w]);
  Pair tot{{1.0, 0.0}, {0.0, 0.0}};
  for (int w = 0; w < kScanThreads / 32; ++w) tot = combine(tot, wtot[w]);
  *total = tot;
  Pair excl = shfl_up_pair(incl, 1);
  if (lane == 0) excl = Pair{{1.0, 0.0}, {0.0, 0.0}};
  __syncthreads();
  return combine(wpre, excl);
}

struct ScanArgs {
  const cplx* A;
  const cplx* F;
  const cplx* G;
  cplx* Cf;
  cplx* Cb;
  int64_t nseg;
  int ne;
  int64_t nblk;
  cplx* blkagg;    // [2ne][nblk] (a, s) pairs as 2 complex
  cplx* blkcarry;  // [2ne][nblk]
};

__device__ __forceinline__ Pair load_item(const ScanArgs& sa, int q, int64_t r) {
  const bool bwd = q >= sa.ne;
  const int k = bwd ? q - sa.ne : q;
  const int64_t b = bwd ? sa.nseg - 1 - r : r;
  const int64_t o = (int64_t)k * sa.nseg + b;
  return Pair{sa.A[o], bwd ? sa.G[o] : sa.F[o]};
}

__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(ScanArgs sa) {
  const int q = blockIdx.y;
  const int64_t r0 = (int64_t)blockIdx.x * kScanBlock + (int64_t)threadIdx.x * kScanItems;
  Pair acc{{1.0, 0.0}, {0.0, 0.0}};
#pragma unroll
  for (int i = 0; i < kScanItems; ++i)
    if (r0 + i < sa.nseg) acc = combine(acc, load_item(sa, q, r0 + i));
  Pair tot;
  block_exclusive(acc, &tot);
  if (threadIdx.x == 0) {
    sa.blkagg[((int64_t)q * sa.nblk + blockIdx.x) * 2 + 0] = tot.a;
    sa.blkagg[((int64_t)q * sa.nblk + blockIdx.x) * 2 + 1] = tot.s;
  }
}

__global__ void __launch_bounds__(1024)
    scan_top_kernel(ScanArgs sa, const cplx* __restrict__ carry_in, cplx* __restrict__ totals) {
  __shared__ Pair sp[1024];
  const int q = blockIdx.x;
  const int ne = sa.ne;
  const int64_t per = (sa.nblk + 1023) / 1024;
  const int64_t r0 = (int64_t)threadIdx.x * per;
  const int64_t r1 = r0 + per < sa.nblk ? r0 + per : sa.nblk;
  const cplx* ag = sa.blkagg + (int64_t)q * sa.nblk * 2;
  Pair acc{{1.0, 0.0}, {0.0, 0.0}};
  for (int64_t r = r0; r < r1; ++r) acc = combine(acc, Pair{ag[2 * r], ag[2 * r + 1]});
  // Hillis-Steele over 1024 thread aggregates (tiny)
  sp[threadIdx.x] = acc;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    Pair p{{1.0, 0.0}, {0.0, 0.0}};
    const bool has = threadIdx.x >= off;
    if (has) p = sp[threadIdx.x - off];
    __syncthreads();
    if (has) {
      acc = combine(p, acc);
      sp[threadIdx.x] = acc;
    }
    __syncthreads();
  }
  Pair ex{{1.0, 0.0}, {0.0, 0.0}};
  if (threadIdx.x > 0) ex = sp[threadIdx.x - 1];
  const cplx cin = carry_in ? carry_in[q] : cplx{0.0, 0.0};
  cplx c = cmad(ex.a, cin, ex.s);
  cplx* bc = sa.blkcarry + (int64_t)q * sa.nblk;
  for (int64_t r = r0; r < r1; ++r) {
    bc[r] = c;
    c = cmad(ag[2 * r], c, ag[2 * r + 1]);
  }
  if (totals && threadIdx.x == 1023) {
    const Pair t = sp[1023];
    if (q < ne) {
      totals[q] = t.a;       // A of the chunk
      totals[ne + q] = t.s;  // F: forward state at the chunk end
    } else {
      totals[2 * ne + (q - ne)] = t.s;  // G: backward state at the chunk's z_prev
    }
  }
}

__global__ void __launch_bounds__(kScanThreads) scan_down_kernel(ScanArgs sa) {
  const int q = blockIdx.y;
  const bool bwd = q >= sa.ne;
  const int k = bwd ? q - sa.ne : q;
  const int64_t r0 = (int64_t)blockIdx.x * kScanBlock + (int64_t)threadIdx.x * kScanItems;
  Pair items[kScanItems];
  Pair acc{{1.0, 0.0}, {0.0, 0.0}};
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    items[i] = r0 + i < sa.nseg ? load_item(sa, q, r0 + i) : Pair{{1.0, 0.0}, {0.0, 0.0}};
    acc = combine(acc, items[i]);
  }
  Pair tot;
  const Pair ex = block_exclusive(acc, &tot);
  const cplx bcin = sa.blkcarry[(int64_t)q * sa.nblk + blockIdx.x];
  cplx c = cmad(ex.a, bcin, ex.s);
  cplx* C = bwd ? sa.Cb : sa.Cf;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int64_t r = r0 + i;
    if (r < sa.nseg) {
      const int64_t b = bwd ? sa.nseg - 1 - r : r;
      C[(int64_t)k * sa.nseg + b] = c;
      c = cmad(items[i].a, c, items[i].s);
    }
  }
}

__global__ void gather_kernel(const double* __restrict__ alpha, const int32_t* __restrict__ perm,
                              int64_t n, double* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) out[i] = __ldg(alpha + perm[i]);
}

}  // namespace

// ============================================================== host side

int64_t scan_blocks(int64_t nseg) { return (nseg + kScanBlock - 1) / kScanBlock; }

size_t tile_state_elems(int64_t nseg, int ne) {
  const size_t nt = (size_t)nseg * (size_t)ne;
  return 5 * nt + (size_t)scan_blocks(nseg) * 2 * (size_t)ne * 3 + 8;
}

TileState tile_state_carve(cplx* base, int64_t nseg, int ne) {
  const size_t nt = (size_t)nseg * (size_t)ne;
  return TileState{base, base + nt, base + 2 * nt, base + 3 * nt, base + 4 * nt, base + 5 * nt};
}

size_t seg_smem_bytes(int ne) {
  return sizeof(ModeTable) + (size_t)kSegWarps * warp_region_bytes(ne);
}

cudaError_t launch_partition(const double* xs, int64_t M, const double* ys, int64_t N,
                             int64_t seg, int64_t nseg, int64_t* seg_ib, cudaStream_t st) {
  const int64_t n = nseg + 1;
  const int bs = 256;
  note_launch();
  partition_kernel<<<(unsigned)((n + bs - 1) / bs), bs, 0, st>>>(xs, M, ys, N, seg, nseg,
                                                                 seg_ib);
  return cudaGetLastError();
}

cudaError_t launch_seg_meta(const double* xs, int64_t M, const double* ys, int64_t N,
                            const int64_t* seg_ib, int64_t nseg, double2* seg_z,
                            uint32_t* seg_mask, cudaStream_t st) {
  if (nseg == 0) return cudaSuccess;
  note_launch();
  seg_meta_kernel<<<(unsigned)((nseg + 3) / 4), 128, 0, st>>>(xs, M, ys, N, seg_ib, nseg, seg_z,
                                                               seg_mask);
  return cudaGetLastError();
}

template <class K>
static cudaError_t set_smem(K kernel, bool& done) {
  if (done) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)seg_smem_bytes(kMaxModes));
  if (e == cudaSuccess) done = true;
  return e;
}

cudaError_t launch_aggregate(const StreamArgs& a, const ModeParams& P, const ModeTable* mt,
                             TileState ts, cudaStream_t st) {
  if (a.nseg == 0) return cudaSuccess;
  const unsigned grid = (unsigned)((a.nseg + kSegWarps - 1) / kSegWarps);
  note_launch();
  seg_aggregate_kernel<<<grid, kThreads, 0, st>>>(a, P, mt, ts);
  return cudaGetLastError();
}

template <bool MS>
static cudaError_t launch_seg_main(const StreamArgs& a, const ModeParams& P, const ModeTable* mt,
                                   TileState ts, OutArgs o, cudaStream_t st) {
  if (a.nseg == 0) return cudaSuccess;
  static bool done = false;
  cudaError_t e = set_smem(seg_main_kernel<MS>, done);
  if (e != cudaSuccess) return e;
  const unsigned grid = (unsigned)((a.nseg + kSegWarps - 1) / kSegWarps);
  note_launch();
  seg_main_kernel<MS><<<grid, kThreads, seg_smem_bytes(P.ne), st>>>(a, P, mt, ts, o);
  return cudaGetLastError();
}

cudaError_t launch_main(const StreamArgs& a, const ModeParams& P, const ModeTable* mt,
                        TileState ts, OutArgs o, cudaStream_t st) {
  return launch_seg_main<false>(a, P, mt, ts, o, st);
}

cudaError_t launch_mode_sums(const StreamArgs& a, const ModeParams& P, const ModeTable* mt,
                             TileState ts, OutArgs o, cudaStream_t st) {
  return launch_seg_main<true>(a, P, mt, ts, o, st);
}

cudaError_t launch_carry_scan(const TileState& ts, int64_t nseg, int ne, const cplx* carry_in,
                              cplx* totals, cudaStream_t st) {
  if (nseg == 0) return cudaSuccess;
  const int64_t nblk = scan_blocks(nseg);
  ScanArgs sa{ts.A, ts.F, ts.G, ts.Cf, ts.Cb, nseg, ne, nblk, ts.blk,
              ts.blk + (size_t)nblk * 2 * ne * 2};
  const dim3 grid((unsigned)nblk, (unsigned)(2 * ne));
  note_launch(3);
  scan_reduce_kernel<<<grid, kScanThreads, 0, st>>>(sa);
  scan_top_kernel<<<2 * ne, 1024, 0, st>>>(sa, carry_in, totals);
  scan_down_kernel<<<grid, kScanThreads, 0, st>>>(sa);
  return cudaGetLastError();
}

cudaError_t launch_gather(const double* alpha, const int32_t* perm, int64_t n, double* out,
                          cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  note_launch();
  gather_kernel<<<blocks, 256, 0, st>>>(alpha, perm, n, out);
  return cudaGetLastError();
}

}  // namespace fgt_b200
