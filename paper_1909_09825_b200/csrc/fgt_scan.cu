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
#include <stddef.h>

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

// The same split from a proportional guess (diag nx / (nx + ny): exact for
// evenly interleaved sets, within ~sqrt(diag) for random ones): gallop from
// the guess in doubling steps to bracket the answer, then bisect the bracket
// -- about 17 dependent loads instead of 27 at 2e8 elements, and at most
// kGallop + 1 more than the bisection's on any data.  The predicate is the
// bisection's, so on sorted input the result is identical.
template <class Ptr>
__device__ __forceinline__ int64_t merge_path_guess(Ptr x, int64_t nx, Ptr y, int64_t ny,
                                                    int64_t diag) {
  int64_t lo = diag - ny > 0 ? diag - ny : 0;
  int64_t hi = diag < nx ? diag : nx;
  if (lo >= hi) return lo;
  // pred(mid), lo < mid <= hi: the split is at or above mid
  auto pred = [&](int64_t mid) { return x[mid - 1] < y[diag - mid]; };
  int64_t g = (int64_t)((double)diag * ((double)nx / (double)(nx + ny)));
  g = g < lo ? lo : (g > hi ? hi : g);
  int64_t step = 1024;
  // (at most kGallop doubling steps: beyond 1024 * 2^kGallop elements from the
  // guess the remaining range is bisected as it is)
  constexpr int kGallop = 6;
  if (g > lo && pred(g)) {
    lo = g;
    for (int k = 0; k < kGallop && lo < hi; ++k) {
      const int64_t p = lo + step < hi ? lo + step : hi;
      if (pred(p)) {
        lo = p;
        step <<= 1;
      } else {
        hi = p - 1;
        break;
      }
    }
  } else {
    if (g > lo) hi = g - 1;
    for (int k = 0; k < kGallop && lo < hi; ++k) {
      const int64_t p = hi - step + 1 > lo + 1 ? hi - step + 1 : lo + 1;
      if (pred(p)) {
        lo = p;
        break;
      }
      hi = p - 1;
      step <<= 1;
    }
  }
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (pred(mid))
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

// Gap factors of a lane run, exp(-s_k g_i) for i < kR: Horner with the
// element loop inside (each coefficient read once per run, kR independent
// chains); exact for D < 0.  Same operation order as horner<D>.
template <int D>
__device__ __forceinline__ void gap_factors(const ModeTable& mt, int k, const double (&g)[kR],
                                            cplx (&d)[kR]) {
  if constexpr (D < 0) {
    const cplx s = mt.s[k];
#pragma unroll
    for (int i = 0; i < kR; ++i) d[i] = decay_exact(s.re, s.im, g[i]);
  } else {
    const cplx* cf = mt.coef[k];
    const cplx top = cf[D];
#pragma unroll
    for (int i = 0; i < kR; ++i) d[i] = top;
#pragma unroll
    for (int n = D - 1; n >= 0; --n) {
      const cplx c = cf[n];
#pragma unroll
      for (int i = 0; i < kR; ++i) {
        d[i].re = fma(d[i].re, g[i], c.re);
        d[i].im = fma(d[i].im, g[i], c.im);
      }
    }
  }
}

// Runtime-degree variant for the wide kernels (one code path for every
// degree keeps them small in the instruction cache); D < 0: exact.
__device__ __forceinline__ void gap_factors_rt(const ModeTable& mt, int k, int D,
                                               const double (&g)[kR], cplx (&d)[kR]) {
  if (D < 0) {
    const cplx s = mt.s[k];
#pragma unroll
    for (int i = 0; i < kR; ++i) d[i] = decay_exact(s.re, s.im, g[i]);
    return;
  }
  const cplx* cf = mt.coef[k];
  if (D == 0) {
#pragma unroll
    for (int i = 0; i < kR; ++i) d[i] = cf[0];
    return;
  }
  // first step folded into the initialisation (no register copies), then
  // two degrees per iteration (half the loop overhead), odd remainder last
  {
    const cplx top = cf[D], c = cf[D - 1];
#pragma unroll
    for (int i = 0; i < kR; ++i) {
      d[i].re = fma(top.re, g[i], c.re);
      d[i].im = fma(top.im, g[i], c.im);
    }
  }
  int n = D - 2;
#pragma unroll 1
  for (; n >= 1; n -= 2) {
    const cplx c1 = cf[n], c0 = cf[n - 1];
#pragma unroll
    for (int i = 0; i < kR; ++i) {
      d[i].re = fma(d[i].re, g[i], c1.re);
      d[i].im = fma(d[i].im, g[i], c1.im);
    }
#pragma unroll
    for (int i = 0; i < kR; ++i) {
      d[i].re = fma(d[i].re, g[i], c0.re);
      d[i].im = fma(d[i].im, g[i], c0.im);
    }
  }
  if (n == 0) {
    const cplx c = cf[0];
#pragma unroll
    for (int i = 0; i < kR; ++i) {
      d[i].re = fma(d[i].re, g[i], c.re);
      d[i].im = fma(d[i].im, g[i], c.im);
    }
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

// One warp copies a transform's mode table (the rows of its ne modes) into
// its shared-memory slot (batched plans).
// EXTRA: 1 also the collapsed-form rows (narrow K3), 2 the lane-collapsed
// polynomial gl, 3 both.
template <int EXTRA = 0>
__device__ __forceinline__ void warp_load_table(const ModeTable* g, ModeTable& s, int ne,
                                                int lane) {
  __syncwarp();
  const double* src = reinterpret_cast<const double*>(g);
  double* dst = reinterpret_cast<double*>(&s);
  constexpr int kHead = 4 * kMaxModes;  // s[], mw[]
  constexpr int kRow = 2 * (kMaxDeg + 1);
  const int n = kHead + kRow * ne;
  for (int i = lane; i < n; i += 32) dst[i] = __ldg(src + i);
  if (lane == 0) s.smax = __ldg(&g->smax);
  if constexpr ((EXTRA & 2) != 0) {
    constexpr int kOffL = offsetof(ModeTable, gl) / sizeof(double);
    if (lane <= kMaxDeg) dst[kOffL + lane] = __ldg(src + kOffL + lane);
  }
  if constexpr ((EXTRA & 1) != 0) {
    // collapsed-form rows and polynomial
    constexpr int kOff = offsetof(ModeTable, mwc) / sizeof(double);
    constexpr int kCRow = 2 * (kCollDeg + 1);
    const int nc = kCRow * ne;
    for (int i = lane; i < nc; i += 32) dst[kOff + i] = __ldg(src + kOff + i);
    constexpr int kOffG = offsetof(ModeTable, gpoly) / sizeof(double);
    if (lane <= kCollDeg) dst[kOffG + lane] = __ldg(src + kOffG + lane);
  }
  __syncwarp();
}
// the lane-collapsed kernel's table slots end before the collapsed-form rows
constexpr size_t kLaneTableBytes = offsetof(ModeTable, mwc);
static_assert(kLaneTableBytes % 16 == 0, "lane table slot alignment");
static_assert(offsetof(ModeTable, coef) == sizeof(double) * 4 * kMaxModes, "table layout");

// Consecutive segments a warp walks in batched plans before striding.
#ifndef FGT_BATCH_GROUP
#define FGT_BATCH_GROUP 16
#endif
constexpr int kBatchGroup = FGT_BATCH_GROUP;

// ---- TMA bulk staging on mbarriers
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// Segment walk of one warp: chunks of kWalkChunk consecutive segments dealt
// round-robin over the warps (consecutive segments keep prefetch chains and
// metadata in L1; round-robin chunks keep clustered work balanced).
#ifndef FGT_WALK_CHUNK
#define FGT_WALK_CHUNK 8
#endif
constexpr int64_t kWalkChunk = FGT_WALK_CHUNK;
static_assert((kWalkChunk & (kWalkChunk - 1)) == 0, "walk chunk: power of two");
struct WarpWalk {
  int64_t wid, nwarps, nseg;
  __device__ __forceinline__ int64_t first() const {
    const int64_t s = wid * kWalkChunk;
    return s < nseg ? s : nseg;
  }
  __device__ __forceinline__ int64_t next(int64_t s) const {
    // unsigned mask / shift (s >= 0): a signed 64-bit % or / costs more
    const uint64_t n1 = (uint64_t)s + 1;
    if ((n1 & (uint64_t)(kWalkChunk - 1)) != 0 && (int64_t)n1 < nseg) return (int64_t)n1;
    const int64_t c = (int64_t)((((uint64_t)s / (uint64_t)kWalkChunk) + (uint64_t)nwarps) *
                                (uint64_t)kWalkChunk);
    return c < nseg ? c : nseg;
  }
};

// ---------------------------------------------------------------- geometry

struct SegGeom {
  int64_t ib, jb;  // first target / source of the segment
  int nx, ny, len;
  double zprev;  // coordinate of the merged element preceding the segment
  double zlast;  // coordinate of the segment's last merged element
  int tid;       // transform of the segment (batched plans)
};

__device__ __forceinline__ SegGeom seg_geom(const StreamArgs& a, int64_t s) {
  SegGeom g;
  g.tid = 0;
  if (a.seg_info) {
    const int4 info = a.seg_info[s];
    const double2 z = a.seg_z[s];
    g.ib = a.seg_ib[s];
    g.jb = a.seg_jb[s];
    g.len = info.x;
    g.nx = info.y;
    g.ny = info.x - info.y;
    g.tid = info.z;
    g.zprev = z.x;
    g.zlast = z.y;
    return g;
  }
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
  double g[kR];    // gap to the previous merged element
  double b[kR];    // strength if source, 0 if target / padding
  unsigned tmask;  // bit e: element e is a target
  int tfirst;      // segment-local index of the lane's first target
  double gmax;     // largest gap
};

// Segment frame: centre zc and half-widths h0 = zc - zprev, h1 = zlast - zc.
struct SegFrame {
  double zc, h0, h1;
};

__device__ __forceinline__ SegFrame seg_frame(const SegGeom& g) {
  const double h = 0.5 * (g.zlast - g.zprev);
  SegFrame f;
  f.zc = g.zprev + h;
  f.h0 = f.zc - g.zprev;
  f.h1 = g.zlast - f.zc;
  return f;
}

// Lane run from the plan-time merge mask: no merge, no shared-memory
// staging; every element is an independent load.  Coordinates are left in
// r.g (converted to gaps by lane_gaps); zp = coordinate preceding the run,
// zl = coordinate of its last element.
__device__ __forceinline__ uint32_t lane_mask_word(const StreamArgs& a, int64_t s, int lane) {
  return __ldg(a.seg_mask + s * (kSeg / 32) + (lane >> 2));
}

// word: this lane's merge-mask word of segment s (prefetched by the caller)
__device__ __forceinline__ void lane_load_w(const StreamArgs& a, const SegGeom& g, uint32_t word,
                                            int lane, LaneRun& r, double& zp, double& zl);

__device__ __forceinline__ void lane_load(const StreamArgs& a, const SegGeom& g, int64_t s,
                                          int lane, LaneRun& r, double& zp, double& zl) {
  lane_load_w(a, g, lane_mask_word(a, s, lane), lane, r, zp, zl);
}

__device__ __forceinline__ void lane_load_w(const StreamArgs& a, const SegGeom& g, uint32_t word,
                                            int lane, LaneRun& r, double& zp, double& zl) {
  const int d0 = lane * kR;
  const int nreal = g.len - d0 < 0 ? 0 : (g.len - d0 < kR ? g.len - d0 : kR);
  const unsigned live = (1u << nreal) - 1u;
  const unsigned byte = (word >> ((lane & 3) * 8)) & 0xffu & live;
  const int nt = __popc(byte);
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
  // element e of the run is target number popc(byte & (2^e - 1)) or source
  // number e - that; branch-free address select, predicated loads
  const double* px = a.xs + g.ib + i0;
  const double* py = a.ys + g.jb + j0;
  const double* pb = a.bs + g.jb + j0;
  int t = 0;
#pragma unroll
  for (int e = 0; e < kR; ++e) {
    const bool tg = (byte >> e) & 1u;
    const bool real = e < nreal;
    const double* pz = tg ? px + t : py + (e - t);
    r.g[e] = real ? __ldg(pz) : 0.0;
    r.b[e] = (real && !tg) ? __ldg(pb + (e - t)) : 0.0;
    t += tg;
  }
  double last = 0.0;
#pragma unroll
  for (int e = 0; e < kR; ++e)
    if (e < nreal) last = r.g[e];
  double prev = __shfl_up_sync(0xffffffffu, last, 1);
  if (lane == 0) prev = g.zprev;
  zp = prev;
  zl = nreal > 0 ? last : prev;
  // padding elements sit on the run's last coordinate: their gaps are 0
#pragma unroll
  for (int e = 0; e < kR; ++e) r.g[e] = e < nreal ? r.g[e] : zl;
}

// ---------------------------------------------------------- segment stage
// K3 streaming: a warp's next segment (targets, sources, strengths) is
// copied into its shared-memory stage by TMA bulk copies while the current
// one is computed.  Layout: xy[kStageXY] holds x at slot ox, y at slot oy;
// b[kStageB] holds b at slot ob.  Bulk copies need 16-byte aligned source,
// destination and size: an unaligned first / last element is copied by an
// 8-byte cp.async instead (lanes 1..6).
constexpr int kStageXY = kSeg + 16;  // + alignment slots and slack for the branch-free decode
constexpr int kStageB = kSeg + 12;
// + mask words (32 B), segment carries (2 kMaxModes complex), mbarrier
constexpr size_t kStageBytes =
    sizeof(double) * (kStageXY + kStageB) + 32 + sizeof(cplx) * 2 * kMaxModes + 16;

struct StagePtrs {
  double* xy;
  double* bb;
  uint32_t* mask;  // [kSeg / 32]
  cplx* car;       // [2 kMaxModes]: forward carries of modes 0..ne-1, then backward
  uint64_t* bar;
};
__device__ __forceinline__ StagePtrs stage_ptrs(unsigned char* base) {
  StagePtrs p;
  p.xy = reinterpret_cast<double*>(base);
  p.bb = p.xy + kStageXY;
  p.mask = reinterpret_cast<uint32_t*>(p.bb + kStageB);
  p.car = reinterpret_cast<cplx*>(p.mask + kSeg / 32);
  p.bar = reinterpret_cast<uint64_t*>(p.car + 2 * kMaxModes);
  return p;
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}

struct StageSlots {
  int ox, oy, ob;
};

__device__ __forceinline__ int misaligned16(const double* p) {
  return (reinterpret_cast<uintptr_t>(p) & 15u) ? 1 : 0;
}

__device__ __forceinline__ StageSlots stage_slots(const StreamArgs& a, const SegGeom& g) {
  StageSlots o;
  const int hx = g.nx > 0 ? misaligned16(a.xs + g.ib) : 0;
  const int hy = g.ny > 0 ? misaligned16(a.ys + g.jb) : 0;
  o.ox = hx;
  o.oy = hx + g.nx;
  o.oy += (o.oy + hy) & 1;  // y's first aligned element on an even slot
  o.ob = g.ny > 0 ? misaligned16(a.bs + g.jb) : 0;
  return o;
}

__device__ __forceinline__ unsigned stage_bulk_bytes(const StageSlots& o, const SegGeom& g) {
  auto cnt = [](int h, int n) {
    if (n <= 0) return 0;
    const int c = (n - h) & ~1;
    return c > 0 ? c : 0;
  };
  return 8u * (unsigned)(cnt(o.ox & 1, g.nx) + cnt(o.oy & 1, g.ny) + cnt(o.ob & 1, g.ny));
}

// Lane-parallel issue: lanes 0..2 bulk-copy the 16-byte aligned interior of
// x / y / b (slot o + h, h = 1 when the array's first element is not
// 16-byte aligned), lane 3 the mask words, lanes 4..9 the unaligned head /
// tail elements of the three arrays by 8-byte cp.async, lanes 10.. the 2 ne
// segment carries by 16-byte cp.async.  Each lane selects its own array, so
// the warp issues one instance of each copy path.
__device__ __forceinline__ void stage_issue(const StreamArgs& a, const TileState& ts, int ne,
                                            int64_t s, const SegGeom& g, const StagePtrs& sp,
                                            int lane) {
  const StageSlots o = stage_slots(a, g);
  if (lane == 0) {
    fence_proxy_async();  // earlier generic reads of the stage before async writes
    mbar_expect(sp.bar, stage_bulk_bytes(o, g) + 32u);
  }
  __syncwarp();
  const int arr = lane < 3 ? lane : ((lane - 4) >> 1);  // 0 x, 1 y, 2 b (lanes < 10)
  const double* src = arr == 0 ? a.xs + g.ib : (arr == 1 ? a.ys + g.jb : a.bs + g.jb);
  const int n = arr == 0 ? g.nx : g.ny;
  const int so = arr == 0 ? o.ox : (arr == 1 ? o.oy : o.ob);
  double* buf = arr == 2 ? sp.bb : sp.xy;
  const int h = so & 1;
  int c = (n - h) & ~1;
  if (c < 0) c = 0;
  if (lane < 3) {
    if (n > 0 && c > 0) bulk_g2s(buf + so + h, src + h, 8u * (unsigned)c, sp.bar);
  } else if (lane == 3) {
    bulk_g2s(sp.mask, a.seg_mask + s * (kSeg / 32), 32u, sp.bar);
  } else if (lane < 10) {
    const bool tail = (lane - 4) & 1;
    const int e = tail ? n - 1 : 0;
    if (n > 0 && (tail ? h + c < n : h != 0)) cp_async8(buf + so + e, src + e);
  } else if (lane < 10 + 2 * ne) {
    const int q = lane - 10, k = q < ne ? q : q - ne;
    const int64_t idx = (int64_t)k * a.nseg + s;
    cp_async16(sp.car + q, q < ne ? ts.Cf + idx : ts.Cb + idx);
  }
  cp_async_commit();
}

// lane_load from the stage (mask word of the lane prefetched by the caller)
__device__ __forceinline__ void lane_load_stage(const StreamArgs& a, const SegGeom& g,
                                                const double* xy, const double* bb,
                                                uint32_t word, int lane, LaneRun& r, double& zp,
                                                double& zl) {
  const StageSlots so = stage_slots(a, g);
  const double* sb = bb + so.ob;
  const int d0 = lane * kR;
  const int nreal = g.len - d0 < 0 ? 0 : (g.len - d0 < kR ? g.len - d0 : kR);
  const unsigned live = (1u << nreal) - 1u;
  const unsigned byte = (word >> ((lane & 3) * 8)) & 0xffu & live;
  const int nt = __popc(byte);
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
  // branch-free: one running slot per set, the element's set picks the slot
  // (past the run, reads stay inside the stage's slack and are discarded)
  int ix = so.ox + i0, iy = so.oy + j0, ib = j0;
  double last = 0.0;
#pragma unroll
  for (int e = 0; e < kR; ++e) {
    const bool tg = (byte >> e) & 1u;
    const double v = xy[tg ? ix : iy];
    const double bv = sb[ib];
    r.g[e] = v;
    r.b[e] = (tg || e >= nreal) ? 0.0 : bv;
    if (e < nreal) last = v;
    ix += tg;
    iy += !tg;
    ib += !tg;
  }
  double prev = __shfl_up_sync(0xffffffffu, last, 1);
  if (lane == 0) prev = g.zprev;
  zp = prev;
  zl = nreal > 0 ? last : prev;
#pragma unroll
  for (int e = 0; e < kR; ++e) r.g[e] = e < nreal ? r.g[e] : zl;
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

// Lane carries of one mode: cf = forward state at the element before the
// run, cb = backward state at the run's last element.
struct Carry {
  cplx cf, cb;
};

// Forward and backward recurrences of one mode over the lane run from its
// gap factors d[], seeded with the lane carries (H = cf, K = cb),
// accumulating Re(mw_k (H + K)) into out[] (only target slots are used).
// With Kt_i = K_i + b_i the backward step is Kt_{i-1} = d_i Kt_i + b_{i-1},
// the same multiply-add as the forward step; the two chains are independent
// and interleaved for instruction-level parallelism.
template <bool MS>
__device__ __forceinline__ void chains_mode(const cplx (&d)[kR], cplx mw, const LaneRun& r,
                                            cplx H, cplx K, int k, double (&out)[kR],
                                            const ModeSumsOut& ms) {
  K.re += r.b[kR - 1];
  if constexpr (MS) {
    int64_t ti = ms.t0;
#pragma unroll
    for (int i = 0; i < kR; ++i) {
      H = cmad(d[i], H, cplx{r.b[i], 0.0});
      if (r.tmask & (1u << i)) ms.hp[(int64_t)k * ms.M + ti++] = H;
    }
#pragma unroll
    for (int i = kR - 1; i >= 0; --i) {
      if (r.tmask & (1u << i)) ms.hm[(int64_t)k * ms.M + (--ti)] = K;  // b_i = 0
      if (i > 0) K = cmad(d[i], K, cplx{r.b[i - 1], 0.0});
    }
  } else {
    (void)k;
    (void)ms;
#pragma unroll
    for (int i = 0; i < kR; ++i) {
      H = cmad(d[i], H, cplx{r.b[i], 0.0});
      out[i] = fma(mw.re, H.re, fma(-mw.im, H.im, out[i]));
      const int j = kR - 1 - i;
      out[j] = fma(mw.re, K.re, fma(-mw.im, K.im, out[j]));
      if (j > 0) K = cmad(d[j], K, cplx{r.b[j - 1], 0.0});
    }
  }
}

#ifndef FGT_CARRY_UNROLL
#define FGT_CARRY_UNROLL 1
#endif
constexpr int kCarryUnroll = FGT_CARRY_UNROLL;
#ifndef FGT_MODE_UNROLL
#define FGT_MODE_UNROLL 1
#endif
constexpr int kModeUnroll = FGT_MODE_UNROLL;

#ifndef FGT_P2_PAIRS
#define FGT_P2_PAIRS 0
#endif
// Two modes at once: four independent chains (more ILP, more registers).
template <int D>
__device__ __forceinline__ void pass2_two(const ModeTable& mt, int k, const LaneRun& r,
                                          const Carry* carry, double (&out)[kR]) {
  cplx d0[kR], d1[kR];
  gap_factors<D>(mt, k, r.g, d0);
  gap_factors<D>(mt, k + 1, r.g, d1);
  const cplx mw0 = mt.mw[k], mw1 = mt.mw[k + 1];
  cplx H0 = carry[k].cf, K0 = carry[k].cb, H1 = carry[k + 1].cf, K1 = carry[k + 1].cb;
  K0.re += r.b[kR - 1];
  K1.re += r.b[kR - 1];
#pragma unroll
  for (int i = 0; i < kR; ++i) {
    const int j = kR - 1 - i;
    H0 = cmad(d0[i], H0, cplx{r.b[i], 0.0});
    H1 = cmad(d1[i], H1, cplx{r.b[i], 0.0});
    out[i] = fma(mw0.re, H0.re, fma(-mw0.im, H0.im, out[i]));
    out[i] = fma(mw1.re, H1.re, fma(-mw1.im, H1.im, out[i]));
    out[j] = fma(mw0.re, K0.re, fma(-mw0.im, K0.im, out[j]));
    out[j] = fma(mw1.re, K1.re, fma(-mw1.im, K1.im, out[j]));
    if (j > 0) {
      K0 = cmad(d0[j], K0, cplx{r.b[j - 1], 0.0});
      K1 = cmad(d1[j], K1, cplx{r.b[j - 1], 0.0});
    }
  }
}

// Narrow segments: lane carries already in shared memory (moment form).
template <int D, bool MS>
__device__ __forceinline__ void pass2(const ModeTable& mt, int ne, const LaneRun& r,
                                      const Carry* carry, double (&out)[kR],
                                      const ModeSumsOut& ms) {
#if FGT_P2_PAIRS
  if constexpr (!MS) {
    int k = 0;
    for (; k + 1 < ne; k += 2) pass2_two<D>(mt, k, r, carry, out);
    if (k < ne) {
      cplx d[kR];
      gap_factors<D>(mt, k, r.g, d);
      chains_mode<false>(d, mt.mw[k], r, carry[k].cf, carry[k].cb, k, out, ms);
    }
    return;
  }
#endif
#pragma unroll kModeUnroll
  for (int k = 0; k < ne; ++k) {
    cplx d[kR];
    gap_factors<D>(mt, k, r.g, d);
    chains_mode<MS>(d, mt.mw[k], r, carry[k].cf, carry[k].cb, k, out, ms);
  }
}

// Degrees above MAXD are never requested by the caller; they fall through to
// the MAXD (or, for MAXD = kMaxDeg, the exact) instantiation, so the kernel
// only carries the code (and register demand) of the degrees it can see.
template <bool MS, int MAXD>
__device__ __forceinline__ void dispatch_pass2(int D, const ModeTable& mt, int ne,
                                               const LaneRun& r, const Carry* carry,
                                               double (&out)[kR], const ModeSumsOut& ms) {
  switch (D) {
#define FGT_P2(n)                                   \
  case n:                                           \
    if constexpr (n <= MAXD) {                      \
      pass2<n, MS>(mt, ne, r, carry, out, ms);      \
      return;                                       \
    }                                               \
    [[fallthrough]];
    FGT_P2(0) FGT_P2(1) FGT_P2(2) FGT_P2(3) FGT_P2(4) FGT_P2(5) FGT_P2(6) FGT_P2(7)
    FGT_P2(8) FGT_P2(9) FGT_P2(10) FGT_P2(11) FGT_P2(12) FGT_P2(13) FGT_P2(14)
    FGT_P2(15) FGT_P2(16)
#undef FGT_P2
    default:
      pass2<(MAXD < kMaxDeg ? MAXD : -1), MS>(mt, ne, r, carry, out, ms);
  }
}

// ------------------------------------------------------- lane carries

// Moment form (narrow segments, |s| max(h0, h1) <= rmax[DM]).  With
// d = z - zc and M_n = sum_{sources of the lane} b d^n (mode independent),
// P_n = exclusive prefix of M_n over lanes, S_n = suffix (lanes after):
//   cf = e^{-s u} [ sum_n s^n/n! P_n + e^{-s h0} Cf_seg ],   u = zp - zc
//   cb = e^{+s v} [ sum_n (-s)^n/n! S_n + e^{-s h1} Cb_seg ], v = zl - zc
// All exponentials have |argument| <= rmax[DM] and are Taylor polynomials.
template <int DM>
__device__ __forceinline__ void carries_moments(const ModeTable& mt, int ne, const LaneRun& r,
                                                const SegFrame& f, double zp, double zl,
                                                int lane, const cplx* terms, Carry* out) {
  double P[DM + 1], S[DM + 1];
  {
    double M[DM + 1];
#pragma unroll
    for (int n = 0; n <= DM; ++n) M[n] = 0.0;
#pragma unroll
    for (int e = 0; e < kR; ++e) {
      const double d = r.g[e] - f.zc;  // r.g holds coordinates here
      double p = r.b[e];
      M[0] += p;
#pragma unroll
      for (int n = 1; n <= DM; ++n) {
        p *= d;
        M[n] += p;
      }
    }
#pragma unroll
    for (int n = 0; n <= DM; ++n) {
      double incl = M[n];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const double tot = __shfl_sync(0xffffffffu, incl, 31);
      P[n] = incl - M[n];
      S[n] = tot - incl;
    }
  }
  const double u = zp - f.zc, v = zl - f.zc;
#pragma unroll kCarryUnroll
  for (int k = 0; k < ne; ++k) {
    Coef<DM> c;
    c.load(mt, k);
    cplx fp = {0.0, 0.0}, bs = {0.0, 0.0};
#pragma unroll
    for (int n = 0; n <= DM; ++n) {
      const cplx cn = c[n];
      const double sg = (n & 1) ? -1.0 : 1.0;  // s^n/n! = (-1)^n c_n
      fp.re = fma(sg * cn.re, P[n], fp.re);
      fp.im = fma(sg * cn.im, P[n], fp.im);
      bs.re = fma(cn.re, S[n], bs.re);
      bs.im = fma(cn.im, S[n], bs.im);
    }
    // segment carries propagated to the frame (shared memory, written by
    // lanes k and ne + k: broadcast reads)
    const cplx tf = terms[k];
    const cplx tb = terms[ne + k];
    const cplx eu = horner<DM>(c, u);
    const cplx ev = horner<DM>(c, -v);
    out[k].cf = cmul(eu, cplx{fp.re + tf.re, fp.im + tf.im});
    out[k].cb = cmul(ev, cplx{bs.re + tb.re, bs.im + tb.im});
  }
}

// Collapsed form (narrow segments, potentials only).  Every exponential of a
// narrow segment has |s t| <= rmax[DN] with DN the degree for its full width
// h0 + h1, so the modes fold into ONE real polynomial
//   G(t) = Re sum_k mw_k e^{-s_k t} = sum_{n<=DN} g_n t^n,  g_n = Re sum_k mw_k c_kn
// (c_kn = (-s_k)^n/n!, the table's Taylor coefficients).  With w = z - zc,
// v_j = z_j - zc, Pre_m / Tot_m = prefix / total over the segment's sources of
// b v^m, and the segment carries at the frame centre Tf_k = e^{-s_k h0} Cf_k,
// Tb_k = e^{-s_k h1} Cb_k, a target's potential is a degree-DN polynomial in
// its own w:
//   u = sum_q w^q [ E_q + sum_{m+q odd} 2 (-1)^m C(m+q, m) g_{m+q} Pre_m ]
//   E_q = Re sum_k mw_k c_kq (Tf_k + (-1)^q Tb_k)
//         + (-1)^q sum_m C(m+q, m) g_{m+q} Tot_m
// (forward pairs sum_n g_n (w - v)^n, backward pairs sum_n g_n (v - w)^n, and
// Suf = Tot - Pre).  Mode-independent per element: no gap factors, no chains.
// Terms: each is bounded by sum|mw| (|s| 2h)^n / n! |b|, so the rounding stays
// at eps sum|mw| sum|b| like the per-mode form.
__host__ __device__ constexpr double binom_c(int n, int m) {
  double r = 1.0;
  for (int i = 1; i <= m; ++i) r = r * (n - m + i) / i;
  return r;
}

template <int DN>
__device__ __forceinline__ void collapsed_segment(const ModeTable& mt, int ne, const LaneRun& r,
                                                  const SegFrame& f, int lane,
                                                  const cplx* terms, double* su) {
  constexpr int NM = DN + 1;
  double pre[NM], tot[NM];
  {
    double M[NM];
#pragma unroll
    for (int n = 0; n < NM; ++n) M[n] = 0.0;
#pragma unroll
    for (int e = 0; e < kR; ++e) {
      const double d = r.g[e] - f.zc;  // r.g holds coordinates here
      double p = r.b[e];
      M[0] += p;
#pragma unroll
      for (int n = 1; n < NM; ++n) {
        p *= d;
        M[n] += p;
      }
    }
#pragma unroll
    for (int n = 0; n < NM; ++n) {
      double incl = M[n];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      tot[n] = __shfl_sync(0xffffffffu, incl, 31);
      pre[n] = incl - M[n];
    }
  }
  // g_n and the carry part of E_n on lane n
  double cl = 0.0;
  if (lane < NM) {
    const double sg = (lane & 1) ? -1.0 : 1.0;
    for (int k = 0; k < ne; ++k) {
      const cplx x = mt.mwc[k][lane];
      const cplx tf = terms[k], tb = terms[ne + k];
      cl = fma(x.re, fma(sg, tb.re, tf.re), fma(-x.im, fma(sg, tb.im, tf.im), cl));
    }
  }
  double g[NM], E[NM];
#pragma unroll
  for (int n = 0; n < NM; ++n) {
    g[n] = mt.gpoly[n];
    E[n] = __shfl_sync(0xffffffffu, cl, n);
  }
#pragma unroll
  for (int q = 0; q < NM; ++q) {
    double acc = 0.0;
#pragma unroll
    for (int m = 0; m + q < NM; ++m) acc = fma(binom_c(m + q, m) * g[m + q], tot[m], acc);
    E[q] += (q & 1) ? -acc : acc;
  }
  // odd-order pair coefficients H(m, q) = 2 (-1)^m C(m+q, m) g_{m+q}
  double H[NM][NM];
#pragma unroll
  for (int q = 0; q < NM; ++q)
#pragma unroll
    for (int m = 0; m < NM; ++m)
      H[m][q] = (((m + q) & 1) && m + q < NM)
                    ? ((m & 1) ? -2.0 : 2.0) * binom_c(m + q, m) * g[(m + q) < NM ? m + q : 0]
                    : 0.0;
  int tk = r.tfirst;
#pragma unroll
  for (int e = 0; e < kR; ++e) {
    const double w = r.g[e] - f.zc;
    double p = r.b[e];  // 0 for targets: the prefix is exclusive for them
    pre[0] += p;
#pragma unroll
    for (int m = 1; m < NM; ++m) {
      p *= w;
      pre[m] += p;
    }
    double acc = 0.0;
#pragma unroll
    for (int q = DN; q >= 0; --q) {
      double c = E[q];
#pragma unroll
      for (int m = 0; m + q < NM; ++m)
        if ((m + q) & 1) c = fma(H[m][q], pre[m], c);
      acc = q == DN ? c : fma(acc, w, c);
    }
    if (r.tmask & (1u << e)) su[tk++] = acc;  // staged: coalesced stores after
  }
}

// Lane carries by shuffle (Kogge-Stone) scans of the lane aggregates (A, F,
// G) across the warp, both directions, seeded with the segment carries
// (cfs at the element before the segment, cbs at its last element).
__device__ __forceinline__ void lane_scan(cplx A, cplx F, cplx G, int lane, cplx cfs, cplx cbs,
                                          cplx& cf, cplx& cb) {
  // forward inclusive scan of (A, F) over lanes (earlier then later)
  cplx fa = A, ff = F;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    cplx pa, pf;
    pa.re = __shfl_up_sync(0xffffffffu, fa.re, o);
    pa.im = __shfl_up_sync(0xffffffffu, fa.im, o);
    pf.re = __shfl_up_sync(0xffffffffu, ff.re, o);
    pf.im = __shfl_up_sync(0xffffffffu, ff.im, o);
    if (lane >= o) {
      ff = cmad(fa, pf, ff);
      fa = cmul(pa, fa);
    }
  }
  // backward inclusive scan of (A, G) from the right
  cplx ba = A, bg = G;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    cplx pa, pg;
    pa.re = __shfl_down_sync(0xffffffffu, ba.re, o);
    pa.im = __shfl_down_sync(0xffffffffu, ba.im, o);
    pg.re = __shfl_down_sync(0xffffffffu, bg.re, o);
    pg.im = __shfl_down_sync(0xffffffffu, bg.im, o);
    if (lane + o < 32) {
      bg = cmad(ba, pg, bg);
      ba = cmul(ba, pa);
    }
  }
  // exclusive: shift by one lane and apply the segment carries
  cplx xa = {__shfl_up_sync(0xffffffffu, fa.re, 1), __shfl_up_sync(0xffffffffu, fa.im, 1)};
  cplx xf = {__shfl_up_sync(0xffffffffu, ff.re, 1), __shfl_up_sync(0xffffffffu, ff.im, 1)};
  if (lane == 0) {
    xa = {1.0, 0.0};
    xf = {0.0, 0.0};
  }
  cplx ya = {__shfl_down_sync(0xffffffffu, ba.re, 1), __shfl_down_sync(0xffffffffu, ba.im, 1)};
  cplx yg = {__shfl_down_sync(0xffffffffu, bg.re, 1), __shfl_down_sync(0xffffffffu, bg.im, 1)};
  if (lane == 31) {
    ya = {1.0, 0.0};
    yg = {0.0, 0.0};
  }
  cf = cmad(xa, cfs, xf);
  cb = cmad(ya, cbs, yg);
}

// Wide segments (no moment form): per mode, the gap factors of the lane run
// once (degree-D Taylor, exact for D < 0), the lane aggregates from them,
// the lane carries by warp scans, then both chains -- one evaluation of
// exp(-s g) per element and mode.
template <bool MS>
__device__ __forceinline__ void wide_modes(const ModeTable& mt, int ne, int D, const LaneRun& r,
                                           int lane, const cplx* terms, double (&out)[kR],
                                           const ModeSumsOut& ms) {
  for (int k = 0; k < ne; ++k) {
    cplx d[kR];
    gap_factors_rt(mt, k, D, r.g, d);
    cplx F = {0.0, 0.0}, A = {1.0, 0.0}, G = {0.0, 0.0};
#pragma unroll
    for (int i = 0; i < kR; ++i) {
      F = cmad(d[i], F, cplx{r.b[i], 0.0});
      A = cmul(A, d[i]);
      G.re = fma(r.b[i], A.re, G.re);
      G.im = fma(r.b[i], A.im, G.im);
    }
    const cplx cfs = terms[k];  // segment carries (shared memory, broadcast)
    const cplx cbs = terms[ne + k];
    cplx cf, cb;
    lane_scan(A, F, G, lane, cfs, cbs, cf, cb);
    chains_mode<MS>(d, mt.mw[k], r, cf, cb, k, out, ms);
  }
}


// ------------------------------------------ lane-collapsed wide segments
//
// Wide segments (no segment moment form) whose LANE RUNS are narrow: with W =
// zl - zp the width of a lane's run (the element before it to its last
// element) and |s| W <= rmax[DL] for every lane of the warp, every exponential
// inside a run is a degree-DL polynomial, so per run
//   * the lane aggregates follow from the run's source moments about its last
//     element, M_n = sum b v^n (v = zl - y >= 0, mode independent):
//       A = e^{-s W},  F = sum_n c_n M_n,  G = A sum_n (-1)^n c_n M_n
//     (c_n = (-s)^n / n!, the table's Taylor row): one Horner and 2 (DL + 1)
//     multiply-adds per mode instead of a gap factor per element;
//   * the lane carries come from a sequential scan of the 32 lane aggregates
//     by lanes k (forward, mode k) and ne + k (backward) through shared memory
//     (32 multiply-adds per lane) instead of 2 x 5 shuffle steps per mode;
//   * the carries' part of a target's potential is one real polynomial in its
//     own v,  sum_q v^q E_q,  E_q = Re sum_k c_kq mw_k (cb_k + (-1)^q A_k cf_k);
//   * the sources of the run itself contribute b G(|z_i - z_j|) with the
//     mode-folded polynomial G(t) = Re sum_k mw_k e^{-s_k t} = sum_n g_n t^n
//     (ModeTable::gl): symmetric, so the 28 element pairs of a run are
//     evaluated once each, branch-free.
// No per-element exponentials, no per-mode chains.  Each term is bounded by
// sum|mw| (|s| W)^n / n! |b| like the per-mode recurrences.
// Slots of one warp: A / F / G of lane l and mode k at [l * SK + k], SK odd
// (conflict-free both lane-wise and mode-wise).
__host__ __device__ __forceinline__ int lane_slot_stride(int ne) { return ne | 1; }
__host__ __device__ __forceinline__ size_t lane_slot_bytes(int ne) {
  return sizeof(cplx) * 3 * 32 * (size_t)lane_slot_stride(ne);
}

// Lanes k < ne: forward carries of mode k (exclusive, seeded with the segment
// carry) written over F; lanes ne + k: backward carries over G.
__device__ __noinline__ void lane_slot_scan(cplx* slots, int ne, int lane, cplx seed) {
  const int SK = lane_slot_stride(ne);
  const bool fwd = lane < ne;
  const int k = fwd ? lane : lane - ne;
  const cplx* sA = slots + k;
  cplx* sS = slots + (fwd ? 32 : 64) * SK + k;
  const int step = fwd ? SK : -SK;
  int at = fwd ? 0 : 31 * SK;
  cplx S = seed;
#pragma unroll 4
  for (int i = 0; i < 32; ++i) {
    const cplx a = sA[at];
    const cplx f = sS[at];
    sS[at] = S;
    S = cmad(a, S, f);
    at += step;
  }
}

// Compile-time degree DL <= kMaxDeg (lane_degree_bucket: the runtime degree
// rounded up to the next instantiated one; every loop is straight-line code).
// Offsets v_e = zl - z_e of a run's elements (r.g holds coordinates; padding
// sits on zl: v = 0, b = 0) and its source moments M_n = sum b v^n, n <= DL.
template <int DL>
__device__ __forceinline__ void lane_moments(const LaneRun& r, double zl, double (&v)[kR],
                                             double (&M)[DL + 1]) {
  double pw[kR];
  M[0] = 0.0;
#pragma unroll
  for (int e = 0; e < kR; ++e) {
    v[e] = zl - r.g[e];
    pw[e] = r.b[e];
    M[0] += pw[e];
  }
#pragma unroll
  for (int n = 1; n <= DL; ++n) {
    M[n] = 0.0;
#pragma unroll
    for (int e = 0; e < kR; ++e) {
      pw[e] *= v[e];
      M[n] += pw[e];
    }
  }
}

// One mode's lane aggregates from the moments: A = e^{-s W},
// F = sum_n c_n M_n, G = A sum_n (-1)^n c_n M_n  (cf = the mode's Taylor row).
template <int DL>
__device__ __forceinline__ void lane_mode_aggregate(const cplx* cf, const double (&M)[DL + 1],
                                                    double W, cplx& A, cplx& F, cplx& G) {
  const cplx c0 = cf[0];
  A = cf[DL];
  cplx ev = {c0.re * M[0], c0.im * M[0]}, od = {0.0, 0.0};
#pragma unroll
  for (int n = DL; n >= 1; --n) {
    const cplx cn = cf[n];
    const cplx lo = cf[n - 1];
    A.re = fma(A.re, W, lo.re);
    A.im = fma(A.im, W, lo.im);
    if (n & 1) {
      od.re = fma(cn.re, M[n], od.re);
      od.im = fma(cn.im, M[n], od.im);
    } else {
      ev.re = fma(cn.re, M[n], ev.re);
      ev.im = fma(cn.im, M[n], ev.im);
    }
  }
  F = cplx{ev.re + od.re, ev.im + od.im};
  G = cmul(A, cplx{ev.re - od.re, ev.im - od.im});
}

// The instantiated degrees: a runtime degree runs at the next one at or above
// it (a higher Taylor degree only lowers the truncation error).
#define FGT_LANE_DEGREES(X) X(4) X(6) X(8) X(10) X(12) X(14) X(16)
static_assert(kMaxDeg == 16, "lane-collapsed degree buckets");
__device__ __forceinline__ int lane_degree_bucket(int DL) { return DL <= 4 ? 4 : ((DL + 1) & ~1); }
// K1 runs only the moments / aggregates phase: multiples of 4 (fewer bodies in
// flight; measured cfg 5 K1 4.26 -> 4.08 ms, while K3 loses at these: 10.75 -> 10.91 ms)
__device__ __forceinline__ int lane_degree_bucket4(int DL) { return (DL + 3) & ~3; }

// Phase A of lane_collapsed: the run's moments and every mode's aggregates
// into the slots.
template <int DL>
__device__ __forceinline__ void lane_phase_aggregates(const ModeTable& mt, int ne,
                                                      const LaneRun& r, double zl, double W,
                                                      cplx* sA, cplx* sF, cplx* sG) {
  double v[kR], M[DL + 1];
  lane_moments<DL>(r, zl, v, M);
#pragma unroll 2
  for (int k = 0; k < ne; ++k) {
    cplx A, F, G;
    lane_mode_aggregate<DL>(mt.coef[k], M, W, A, F, G);
    sA[k] = A;
    sF[k] = F;
    sG[k] = G;
  }
}

// Phase C: the carries' polynomial sum_q v^q E_q,
// E_q = Re sum_k c_kq mw_k (cb_k + (-1)^q A_k cf_k), one Horner per element
// with E_q formed on the way down (tp / tm = mw (cb +- A cf) of every mode in
// registers; NE = the launch's mode count).  The loop over the degree is
// rolled (DL even): one body for every degree.
template <int NE>
__device__ __forceinline__ void lane_phase_carries(const ModeTable& mt, int DL,
                                                   const double (&v)[kR], const cplx* sA,
                                                   const cplx* sF, const cplx* sG,
                                                   double (&out)[kR]) {
  cplx tp[NE], tm[NE];
#pragma unroll
  for (int k = 0; k < NE; ++k) {
    const cplx mw = mt.mw[k];
    const cplx ta = cmul(mw, cmul(sA[k], sF[k]));
    const cplx tb = cmul(mw, sG[k]);
    tp[k] = cplx{tb.re + ta.re, tb.im + ta.im};
    tm[k] = cplx{tb.re - ta.re, tb.im - ta.im};
  }
  double acc[kR];
  {
    double Er = 0.0, Ei = 0.0;  // q = DL (even)
#pragma unroll
    for (int k = 0; k < NE; ++k) {
      const cplx c = mt.coef[k][DL];
      Er = fma(c.re, tp[k].re, Er);
      Ei = fma(c.im, tp[k].im, Ei);
    }
#pragma unroll
    for (int e = 0; e < kR; ++e) acc[e] = Er - Ei;
  }
#pragma unroll 1
  for (int q = DL - 1; q > 0; q -= 2) {
    double Eor = 0.0, Eoi = 0.0, Eer = 0.0, Eei = 0.0;  // q odd, q - 1 even
#pragma unroll
    for (int k = 0; k < NE; ++k) {
      const cplx co = mt.coef[k][q];
      const cplx ce = mt.coef[k][q - 1];
      Eor = fma(co.re, tm[k].re, Eor);
      Eoi = fma(co.im, tm[k].im, Eoi);
      Eer = fma(ce.re, tp[k].re, Eer);
      Eei = fma(ce.im, tp[k].im, Eei);
    }
    const double Eo = Eor - Eoi, Ee = Eer - Eei;
#pragma unroll
    for (int e = 0; e < kR; ++e) acc[e] = fma(fma(acc[e], v[e], Eo), v[e], Ee);
  }
#pragma unroll
  for (int e = 0; e < kR; ++e) out[e] += acc[e];
}
// the mode counts the carries phase is instantiated for
#define FGT_LANE_MODES(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8)
static_assert(kMaxModes == 8 && kMaxDeg % 2 == 0, "lane-collapsed form");

// DL: a degree of FGT_LANE_DEGREES (warp uniform).
__device__ __forceinline__ void lane_collapsed(const ModeTable& mt, int ne, int DL,
                                               const LaneRun& r, double zp, double zl, int lane,
                                               const cplx* terms, bool noprev, cplx* slots,
                                               double* su) {
  const int SK = lane_slot_stride(ne);
  cplx* sA = slots + lane * SK;
  cplx* sF = sA + 32 * SK;
  cplx* sG = sA + 64 * SK;
  const double W = zl - zp;
  switch (DL) {
#define FGT_LC_CASE(d)                                              \
  case d:                                                           \
    lane_phase_aggregates<d>(mt, ne, r, zl, W, sA, sF, sG);        \
    break;
    FGT_LANE_DEGREES(FGT_LC_CASE)
#undef FGT_LC_CASE
  }
  double v[kR];
#pragma unroll
  for (int e = 0; e < kR; ++e) v[e] = zl - r.g[e];
  // the run's own sources: pairs (i, j), i < j, t = z_j - z_i = v_i - v_j >= 0
  // (one loop for every degree: the polynomial's coefficients come from
  // shared memory)
  double out[kR];
#pragma unroll
  for (int e = 0; e < kR; ++e) out[e] = 0.0;
  const double gtop = mt.gl[DL];
  static_assert(kR % 4 == 0, "pair groups are evaluated two at a time");
#pragma unroll
  for (int grp = 0; grp < kR / 2; grp += 2) {
    // rows grp and kR - 1 - grp, rows grp + 1 and kR - 2 - grp: kR - 1 pairs
    // each, 2 (kR - 1) independent Horner chains per loop pass
    constexpr int NP = 2 * (kR - 1);
    double t[NP], acc[NP];
    {
      int q = 0;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int j = grp + h + 1; j < kR; ++j) t[q++] = v[grp + h] - v[j];
#pragma unroll
        for (int j = kR - grp - h; j < kR; ++j) t[q++] = v[kR - 1 - grp - h] - v[j];
      }
    }
#pragma unroll
    for (int q = 0; q < NP; ++q) acc[q] = gtop;
#pragma unroll 4
    for (int n = DL - 1; n >= 0; --n) {
      const double gn = mt.gl[n];
#pragma unroll
      for (int q = 0; q < NP; ++q) acc[q] = fma(acc[q], t[q], gn);
    }
    {
      int q = 0;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int lo = grp + h, hi = kR - 1 - grp - h;
#pragma unroll
        for (int j = lo + 1; j < kR; ++j, ++q) {
          out[lo] = fma(r.b[j], acc[q], out[lo]);
          out[j] = fma(r.b[lo], acc[q], out[j]);
        }
#pragma unroll
        for (int j = hi + 1; j < kR; ++j, ++q) {
          out[hi] = fma(r.b[j], acc[q], out[hi]);
          out[j] = fma(r.b[hi], acc[q], out[j]);
        }
      }
    }
  }
  __syncwarp();
  if (lane < 2 * ne)
    lane_slot_scan(slots, ne, lane, (noprev && lane < ne) ? cplx{0.0, 0.0} : terms[lane]);
  __syncwarp();
  switch (ne) {
#define FGT_LC_CASE(m)                                              \
  case m:                                                           \
    lane_phase_carries<m>(mt, DL, v, sA, sF, sG, out);             \
    break;
    FGT_LANE_MODES(FGT_LC_CASE)
#undef FGT_LC_CASE
  }
  __syncwarp();  // every lane has read its slots: su may alias them
  int tk = r.tfirst;
#pragma unroll
  for (int e = 0; e < kR; ++e)
    if (r.tmask & (1u << e)) su[tk++] = out[e];
}

// false: the runs are too wide for the lane-collapsed form.
#ifndef FGT_LANE_COLL
#define FGT_LANE_COLL 1
#endif
__device__ __forceinline__ bool lane_collapsed_dispatch(const ModeParams& P, const ModeTable& mt,
                                                        int ne, const LaneRun& r, double zp,
                                                        double zl, int lane, const cplx* terms,
                                                        cplx* slots, double* su) {
  // (the shuffle keeps the degree one opaque integer: the unrolled loops of
  // lane_collapsed then test it with one compare each)
  // A run without a predecessor (zp = -inf: the first segment of a batched
  // transform) starts at its own first element: nothing precedes it, so its
  // forward carry is 0 and its A / G reach no one.
  const bool noprev = __shfl_sync(0xffffffffu, zp == -INFINITY ? 1 : 0, 0) != 0;
  if (zp == -INFINITY) zp = r.g[0];
  const int DL = __shfl_sync(0xffffffffu, pick_degree(P, mt.smax, warp_max(zl - zp)), 0);
  if (DL < 0) return false;
  lane_collapsed(mt, ne, lane_degree_bucket(DL), r, zp, zl, lane, terms, noprev, slots, su);
  return true;
}

// -------------------------------------------------------- shared memory

// Per-warp region of K3: lane carries, then the output staging.
// lane_carries: false for the collapsed narrow path (potentials only),
// which keeps no per-lane carries in shared memory.
// region: 0 none (collapsed narrow path), 1 lane carries (mode sums / wide),
// 3 the lane-collapsed kernel: the lane-aggregate slots, which the output
// staging aliases, then the segment-carry terms.
__host__ __device__ __forceinline__ size_t warp_lead_bytes(int ne, int region) {
  return region == 1 ? sizeof(Carry) * 32 * (size_t)ne : 0;
}
__host__ __device__ __forceinline__ size_t lane_region_lead(int ne) {
  const size_t sl = lane_slot_bytes(ne), so = sizeof(double) * kSeg;
  return sl > so ? sl : so;
}
__host__ __device__ __forceinline__ size_t warp_region_bytes(int ne, int region) {
  if (region == 3) return lane_region_lead(ne) + sizeof(cplx) * 2 * kMaxModes;
  // lane carries, output staging, segment-carry terms
  return warp_lead_bytes(ne, region) + sizeof(double) * kSeg + sizeof(cplx) * 2 * kMaxModes;
}

// ------------------------------------------------------------------- K1

// Segment aggregates from the source moments about the segment centre.
// Moments of this lane's sources (up to kK1Per, loaded by the caller),
// warp-reduced; lanes k < ne turn them into mode k's (A, F, G).
constexpr int kK1Per = kSeg / 32;  // sources per lane (a segment has <= kSeg)

template <int DM>
__device__ __forceinline__ void seg_aggregate_from(const SegFrame& f, const ModeTable& mt, int ne,
                                                   int lane, int64_t nseg, int64_t s,
                                                   const TileState& ts,
                                                   const double (&yv)[kK1Per],
                                                   const double (&bv)[kK1Per]) {
  double M[DM + 1];
#pragma unroll
  for (int n = 0; n <= DM; ++n) M[n] = 0.0;
#pragma unroll
  for (int u = 0; u < kK1Per; ++u) {
    const double d = yv[u] - f.zc;
    double p = bv[u];
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
  if (lane < ne) {
    const int k = lane;
    Coef<DM> c;
    c.load(mt, k);
    cplx ev = {0.0, 0.0}, od = {0.0, 0.0};
#pragma unroll
    for (int n = 0; n <= DM; ++n) {
      const cplx cn = c[n];
      if (n & 1) {
        od.re = fma(cn.re, M[n], od.re);
        od.im = fma(cn.im, M[n], od.im);
      } else {
        ev.re = fma(cn.re, M[n], ev.re);
        ev.im = fma(cn.im, M[n], ev.im);
      }
    }
    const cplx E0 = horner<DM>(c, f.h0);
    const cplx E1 = horner<DM>(c, f.h1);
    const int64_t o = (int64_t)k * nseg + s;
    ts.A[o] = cmul(E0, E1);
    ts.F[o] = cmul(E1, cplx{ev.re - od.re, ev.im - od.im});
    ts.G[o] = cmul(E0, cplx{ev.re + od.re, ev.im + od.im});
  }
}

// Issue the loads of a segment's sources (lane-strided; padding = centre, 0).
__device__ __forceinline__ void k1_load(const StreamArgs& a, const SegGeom& g, double zc,
                                        int lane, double (&yv)[kK1Per], double (&bv)[kK1Per]) {
#pragma unroll
  for (int u = 0; u < kK1Per; ++u) {
    const int j = lane + u * 32;
    yv[u] = j < g.ny ? __ldg(a.ys + g.jb + j) : zc;
    bv[u] = j < g.ny ? __ldg(a.bs + g.jb + j) : 0.0;
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

// Highest segment-moment degree (narrow K1; coefficients above kRegDeg are
// read from the shared-memory table).  Segments beyond it take the wide K1.
#ifndef FGT_K1_MAXDM
#define FGT_K1_MAXDM 12
#endif
static_assert(FGT_K1_MAXDM >= kRegDeg && FGT_K1_MAXDM <= kMaxDeg, "K1 moment degree");
__device__ __forceinline__ int seg_moment_degree(const ModeParams& P, double smax,
                                                 const SegFrame& f) {
  const int DM = pick_degree(P, smax, fmax(f.h0, f.h1));
  return DM <= FGT_K1_MAXDM ? DM : -1;
}

// Highest moment degree K3 keeps in registers.  A segment narrow enough for
// it has every gap below 2 rmax[kK3Moments] < rmax[kMaxDeg], so its gap
// factors take the Taylor path.
#ifndef FGT_K3_MOMENTS
#define FGT_K3_MOMENTS 5
#endif
constexpr int kK3Moments = FGT_K3_MOMENTS;
static_assert(kK3Moments >= 0 && kK3Moments <= kRegDeg, "K3 moment degree");
// Largest gap-factor degree of a narrow segment: every gap is at most
// h0 + h1 <= 2 rmax[DM] / |s|, and 2 rmax[5] = 0.0148 < rmax[6] = 0.0197
// (rmax[D] = ((D+1)! 2^-b)^(1/(D+1)), b = FGT_TRUNC_BITS >= 48), so DM <= 5
// implies D <= 6.
#ifndef FGT_NARROW_MAXD
#define FGT_NARROW_MAXD (kK3Moments <= 5 ? 6 : kMaxDeg)
#endif
constexpr int kNarrowMaxD = FGT_NARROW_MAXD;
// Highest collapsed degree of the wide K3 (0: wide segments never collapse).
#ifndef FGT_COLL_WIDE
#define FGT_COLL_WIDE 8
#endif
constexpr int kCollWide = FGT_COLL_WIDE;
static_assert(kCollWide == 0 || (kCollWide >= 7 && kCollWide <= kCollDeg), "wide collapse");
static_assert(kNarrowMaxD >= 6 && kNarrowMaxD <= kCollDeg, "narrow degree bound");
// Highest lane-moment degree of the K1 wide path.
#ifndef FGT_LANE_MOM_MAX
#define FGT_LANE_MOM_MAX 12
#endif
constexpr int kLaneMomMax = FGT_LANE_MOM_MAX;

// Segment classes (both kernels and the plan-time count use these).
__device__ __forceinline__ bool k1_narrow(int DM) { return DM >= 0 && DM <= FGT_K1_MAXDM; }
__device__ __forceinline__ bool k3_narrow(int DM) { return DM >= 0 && DM <= kK3Moments; }

__device__ __forceinline__ int seg_deg_D(int deg) { return (deg & 0xff) - 1; }
__device__ __forceinline__ int seg_deg_DM(int deg) { return ((deg >> 8) & 0xff) - 1; }
// degree of the collapsed form (full segment width h0 + h1)
__device__ __forceinline__ int seg_deg_DN(int deg) { return ((deg >> 16) & 0xff) - 1; }

__device__ __forceinline__ double seg_smax(const StreamArgs& a, const SegGeom& g, double smax) {
  return a.mtb ? __ldg(&a.mtb[g.tid].smax) : smax;
}

// Taylor degree of a segment's gap factors from its lane runs (r.g = gaps,
// the first one from the element before the run): the largest gap of the
// segment including the one into its first element.  Warp-collective.
__device__ __forceinline__ int run_gap_degree(const ModeParams& P, double smax, const LaneRun& r) {
  double gm = r.g[0];
#pragma unroll
  for (int e = 1; e < kR; ++e) gm = fmax(gm, r.g[e]);
  return pick_degree(P, smax, warp_max(gm));
}

// Wide segments: lane aggregates from the gap factors (degree-D Taylor,
// exact for D < 0), reduced across the warp in lane order.
__device__ __forceinline__ void seg_aggregate_wide(const ModeTable& mt, int ne, int D, int lane,
                                                   const LaneRun& r, int64_t nseg, int64_t s,
                                                   TileState ts) {
  for (int k = 0; k < ne; ++k) {
    cplx d[kR];
    gap_factors_rt(mt, k, D, r.g, d);
    cplx F = {0.0, 0.0}, Pp = {1.0, 0.0}, G = {0.0, 0.0};
#pragma unroll
    for (int i = 0; i < kR; ++i) {
      F = cmad(d[i], F, cplx{r.b[i], 0.0});
      Pp = cmul(Pp, d[i]);
      G.re = fma(r.b[i], Pp.re, G.re);
      G.im = fma(r.b[i], Pp.im, G.im);
    }
    const LaneAgg w = warp_reduce_agg(LaneAgg{Pp, F, G});
    if (lane == 0) {
      const int64_t o = (int64_t)k * nseg + s;
      ts.A[o] = w.A;
      ts.F[o] = w.F;
      ts.G[o] = w.G;
    }
  }
}

// Wide segments whose lane runs are narrow: lane aggregates from the lane's
// source moments about its centre (the segment moment form of
// seg_aggregate_moments applied to one run, frame (zp, zl)), reduced across
// the warp.  r.g holds coordinates.
template <int DL>
__device__ __forceinline__ void seg_aggregate_lanes(const ModeTable& mt, int ne, int lane,
                                                    const LaneRun& r, double zp, double zl,
                                                    int64_t nseg, int64_t s, TileState ts) {
  const double h = 0.5 * (zl - zp);
  const double zc = zp + h;
  const double h0 = zc - zp, h1 = zl - zc;
  double M[DL + 1];
#pragma unroll
  for (int n = 0; n <= DL; ++n) M[n] = 0.0;
#pragma unroll
  for (int e = 0; e < kR; ++e) {
    const double d = r.g[e] - zc;
    double p = r.b[e];
    M[0] += p;
#pragma unroll
    for (int n = 1; n <= DL; ++n) {
      p *= d;
      M[n] += p;
    }
  }
  for (int k = 0; k < ne; ++k) {
    Coef<DL> c;
    c.load(mt, k);
    cplx ev = {0.0, 0.0}, od = {0.0, 0.0};
#pragma unroll
    for (int n = 0; n <= DL; ++n) {
      const cplx cn = c[n];
      if (n & 1) {
        od.re = fma(cn.re, M[n], od.re);
        od.im = fma(cn.im, M[n], od.im);
      } else {
        ev.re = fma(cn.re, M[n], ev.re);
        ev.im = fma(cn.im, M[n], ev.im);
      }
    }
    const cplx E0 = horner<DL>(c, h0);
    const cplx E1 = horner<DL>(c, h1);
    const LaneAgg w = warp_reduce_agg(LaneAgg{cmul(E0, E1), cmul(E1, cplx{ev.re - od.re, ev.im - od.im}),
                                              cmul(E0, cplx{ev.re + od.re, ev.im + od.im})});
    if (lane == 0) {
      const int64_t o = (int64_t)k * nseg + s;
      ts.A[o] = w.A;
      ts.F[o] = w.F;
      ts.G[o] = w.G;
    }
  }
}

// Wide segments whose lane runs are narrow (K1): the lane aggregates of
// lane_collapsed (one-sided moment form, degree buckets) folded across the
// warp through shared memory, kK1Pass modes at a time: 4 sub-chains of 8
// lanes per mode and direction (all 32 lanes fold), combined by shuffles --
// instead of a 5-step shuffle reduction of (A, F, G) per mode.
constexpr int kK1Pass = 4;
constexpr int kK1SlotStride = kK1Pass | 1;
constexpr size_t kK1SlotBytes = sizeof(cplx) * 3 * 32 * kK1SlotStride;
template <int DL>
__device__ __forceinline__ void seg_aggregate_slots(const ModeTable& mt, int ne, int lane,
                                                 const LaneRun& r, double zp, double zl,
                                                 bool noprev, cplx* slots, int64_t nseg, int64_t s,
                                                 TileState ts) {
  constexpr int SK = kK1SlotStride;
  cplx* sA = slots + lane * SK;
  cplx* sF = sA + 32 * SK;
  cplx* sG = sA + 64 * SK;
  const double W = zl - zp;
  double v[kR], M[DL + 1];
  lane_moments<DL>(r, zl, v, M);
  const int sub = lane >> 3, dir = (lane >> 2) & 1, kk = lane & 3;
  for (int k0 = 0; k0 < ne; k0 += kK1Pass) {
    const int np = ne - k0 < kK1Pass ? ne - k0 : kK1Pass;
    for (int q = 0; q < np; ++q) {
      cplx A, F, G;
      lane_mode_aggregate<DL>(mt.coef[k0 + q], M, W, A, F, G);
      if (noprev) {  // nothing precedes this run: its gap is infinite
        A = cplx{0.0, 0.0};
        G = cplx{0.0, 0.0};
      }
      sA[q] = A;
      sF[q] = F;
      sG[q] = G;
    }
    __syncwarp();
    // fold this thread's 8 lanes (forward: ascending, F; backward: descending, G)
    cplx Pr = {1.0, 0.0}, S = {0.0, 0.0};
    if (kk < np) {
      const cplx* pa = slots + kk;
      const cplx* px = slots + (dir ? 64 : 32) * SK + kk;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int l = 8 * sub + (dir ? 7 - i : i);
        const cplx a = pa[l * SK];
        const cplx x = px[l * SK];
        S = cmad(a, S, x);
        Pr = cmul(Pr, a);
      }
    }
    // chain the 4 sub-chains in fold order (held by sub 0 forward, sub 3 backward)
#pragma unroll
    for (int c = 1; c < 4; ++c) {
      const int src = (dir ? 3 - c : c) * 8 + (lane & 7);
      cplx Pc, Sc;
      Pc.re = __shfl_sync(0xffffffffu, Pr.re, src);
      Pc.im = __shfl_sync(0xffffffffu, Pr.im, src);
      Sc.re = __shfl_sync(0xffffffffu, S.re, src);
      Sc.im = __shfl_sync(0xffffffffu, S.im, src);
      if (sub == (dir ? 3 : 0)) {
        S = cmad(Pc, S, Sc);
        Pr = cmul(Pr, Pc);
      }
    }
    if (kk < np && sub == (dir ? 3 : 0)) {
      const int64_t o = (int64_t)(k0 + kk) * nseg + s;
      if (dir == 0) {
        ts.A[o] = Pr;
        ts.F[o] = S;
      } else {
        ts.G[o] = S;
      }
    }
    __syncwarp();
  }
}

// K1: warps loop over segments (grid-stride; groups of kBatchGroup for
// batched plans).  Two variants with their own register allocation: the
// moment path for narrow segments (WIDE = false) and per-element lane
// aggregates reduced across the warp for the others (WIDE = true); each
// skips the other's segments.
#ifndef FGT_K1_MINB
#define FGT_K1_MINB 4
#endif
template <bool WIDE>
__global__ void __launch_bounds__(kThreads, FGT_K1_MINB)
    seg_aggregate_kernel(StreamArgs a, ModeParams P, const ModeTable* __restrict__ mtab,
                         TileState ts) {
  // one mode table per warp for batched plans, one per CTA otherwise
  // (dynamic: the smaller footprint leaves more of the SM's L1 to the loads)
  extern __shared__ __align__(16) unsigned char k1_smem[];
  ModeTable* tabs = reinterpret_cast<ModeTable*>(k1_smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool batched = a.mtb != nullptr;
  if (!batched) load_mode_table(mtab, tabs[0]);
  __syncthreads();
  ModeTable& mx = batched ? tabs[warp] : tabs[0];
  int cached_tid = -1;
  const int ne = P.ne;
  // wide variant: per-warp lane-aggregate slots behind the tables
  cplx* slots = reinterpret_cast<cplx*>(k1_smem + sizeof(ModeTable) * (batched ? kSegWarps : 1) +
                                        (WIDE ? kK1SlotBytes * warp : 0));
  (void)slots;
  if constexpr (!WIDE) {
    // contiguous range per warp (metadata from L1); the next narrow
    // segment's sources are loaded into registers before this one is reduced
    const WarpWalk walk{(int64_t)blockIdx.x * kSegWarps + warp, (int64_t)gridDim.x * kSegWarps,
                        a.nseg};
    const int64_t S1 = a.nseg;
    auto next_narrow = [&](int64_t s, SegGeom& g, SegFrame& f, int& DM) -> int64_t {
      for (; s < S1; s = walk.next(s)) {
        DM = seg_deg_DM(__ldg(a.seg_deg + s));
        if (k1_narrow(DM)) {
          g = seg_geom(a, s);
          f = seg_frame(g);
          return s;
        }
      }
      return S1;
    };
    SegGeom g;
    SegFrame f;
    int DM = -1;
    double yv[kK1Per], bv[kK1Per];
    int64_t s = next_narrow(walk.first(), g, f, DM);
    if (s < S1) k1_load(a, g, f.zc, lane, yv, bv);
    while (s < S1) {
      SegGeom gn;
      SegFrame fn;
      int DMn = -1;
      double yn[kK1Per], bn[kK1Per];
      const int64_t sn = next_narrow(walk.next(s), gn, fn, DMn);
      if (sn < S1) k1_load(a, gn, fn.zc, lane, yn, bn);
      if (batched && g.tid != cached_tid) {
        warp_load_table(a.mtb + g.tid, mx, ne, lane);
        cached_tid = g.tid;
      }
      // even moment degrees only (an odd one runs at the next even one: a
      // higher degree only lowers the truncation error, and half the bodies
      // keep the kernel within the instruction cache)
      static_assert(FGT_K1_MAXDM % 2 == 0, "K1 moment degree buckets");
      switch ((DM + 1) & ~1) {
#define FGT_K1(n)                                                     \
  case n:                                                             \
    if constexpr (n <= FGT_K1_MAXDM)                                  \
      seg_aggregate_from<n>(f, mx, ne, lane, a.nseg, s, ts, yv, bv);  \
    break;
        FGT_K1(0) FGT_K1(2) FGT_K1(4) FGT_K1(6) FGT_K1(8) FGT_K1(10) FGT_K1(12) FGT_K1(14)
        FGT_K1(16)
#undef FGT_K1
        default:
          break;
      }
      s = sn;
      g = gn;
      f = fn;
      DM = DMn;
#pragma unroll
      for (int u = 0; u < kK1Per; ++u) {
        yv[u] = yn[u];
        bv[u] = bn[u];
      }
    }
    return;
  } else {
    const int64_t Gs = batched ? kBatchGroup : 1;
    for (int64_t s0 = ((int64_t)blockIdx.x * kSegWarps + warp) * Gs; s0 < a.nseg;
         s0 += (int64_t)gridDim.x * kSegWarps * Gs) {
      const int64_t s1 = s0 + Gs < a.nseg ? s0 + Gs : a.nseg;
      for (int64_t s = s0; s < s1; ++s) {
        const int deg = __ldg(a.seg_deg + s);
        if (k1_narrow(seg_deg_DM(deg))) continue;
        const SegGeom g = seg_geom(a, s);
        if (batched && g.tid != cached_tid) {
          warp_load_table(a.mtb + g.tid, mx, ne, lane);
          cached_tid = g.tid;
        }
        LaneRun r;
        double zp, zl;
        lane_load(a, g, s, lane, r, zp, zl);
#if FGT_LANE_COLL
        {
          // lane-run moment form when every run is narrow enough
          const bool noprev = zp == -INFINITY;  // first segment of a transform (lane 0)
          const double zq = noprev ? r.g[0] : zp;
          const int DLs = __shfl_sync(0xffffffffu, pick_degree(P, mx.smax, warp_max(zl - zq)), 0);
          if (DLs >= 0) {
            switch (DLs <= 4 ? 4 : lane_degree_bucket4(DLs)) {
#define FGT_LC_CASE(d)                                                                 \
  case d:                                                                              \
    seg_aggregate_slots<d>(mx, ne, lane, r, zq, zl, noprev, slots, a.nseg, s, ts);    \
    break;
              FGT_LANE_DEGREES(FGT_LC_CASE)
#undef FGT_LC_CASE
            }
            continue;
          }
        }
#endif
        // lane-run moments when the runs are narrow enough (a few degrees)
        const int DL = pick_degree(P, mx.smax, warp_max(0.5 * (zl - zp)));
        if (DL >= 0 && DL <= kLaneMomMax) {
          if (DL <= 4)
            seg_aggregate_lanes<4>(mx, ne, lane, r, zp, zl, a.nseg, s, ts);
          else if (DL <= 8)
            seg_aggregate_lanes<8>(mx, ne, lane, r, zp, zl, a.nseg, s, ts);
          else
            seg_aggregate_lanes<kLaneMomMax>(mx, ne, lane, r, zp, zl, a.nseg, s, ts);
          continue;
        }
#pragma unroll
        for (int e = kR - 1; e > 0; --e) r.g[e] -= r.g[e - 1];
        r.g[0] -= zp;
        seg_aggregate_wide(mx, ne, run_gap_degree(P, mx.smax, r), lane, r, a.nseg, s, ts);
      }
    }
  }
}

__global__ void store_table_kernel(ModeTable T, ModeTable* __restrict__ out) {
  const double* src = reinterpret_cast<const double*>(&T);
  double* dst = reinterpret_cast<double*>(out);
  for (int i = threadIdx.x; i < (int)(sizeof(ModeTable) / sizeof(double)); i += blockDim.x)
    dst[i] = src[i];
}

// Batched plans: one thread per transform writes its mode table.
__global__ void batch_modes_kernel(BatchModeBase base, const double* __restrict__ deltas, int B,
                                   ModeTable* __restrict__ out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const double isq = 1.0 / sqrt(deltas[b]);  // as build_modes (host)
  ModeTable& T = out[b];
  double smax = 0.0;
  for (int k = 0; k < kMaxModes; ++k) {
    if (k < base.ne) {
      const cplx s = {base.t[k].re * isq, base.t[k].im * isq};
      T.s[k] = s;
      T.mw[k] = base.mw[k];
      smax = fmax(smax, hypot(s.re, s.im));
      const cplx ms = {-s.re, -s.im};
      cplx c = {1.0, 0.0};
      T.coef[k][0] = c;
      T.coef[k][1] = ms;
      c = ms;
      for (int n = 2; n <= kMaxDeg; ++n) {
        c = cmul(c, ms);
        c.re /= (double)n;
        c.im /= (double)n;
        T.coef[k][n] = c;
      }
    } else {
      T.s[k] = {0.0, 0.0};
      T.mw[k] = {0.0, 0.0};
      for (int n = 0; n <= kMaxDeg; ++n) T.coef[k][n] = {0.0, 0.0};
    }
  }
  T.smax = smax;
  T.pad = 0.0;
  for (int n = 0; n <= kCollDeg; ++n) {
    double gn = 0.0;
    for (int k = 0; k < kMaxModes; ++k) {
      const cplx x = cmul(T.mw[k], T.coef[k][n]);
      T.mwc[k][n] = x;
      gn += x.re;
    }
    T.gpoly[n] = gn;
  }
  T.pad2 = 0.0;
  for (int n = 0; n <= kMaxDeg; ++n) {
    double gn = 0.0;
    for (int k = 0; k < kMaxModes; ++k) gn += cmul(T.mw[k], T.coef[k][n]).re;
    T.gl[n] = gn;
  }
  T.pad3 = 0.0;
}

// Plan-time segment classes: counts[0] = K1 wide segments, counts[1] = K3.
__global__ void classify_kernel(StreamArgs a, ModeParams P, double smax, int* __restrict__ seg_deg,
                                const int* __restrict__ skip_flags,
                                unsigned long long* __restrict__ counts) {
  // metadata of a rejected batch (non-finite / unsorted) is not valid
  if (skip_flags && (skip_flags[0] | skip_flags[1] | skip_flags[3] | skip_flags[4])) return;
  const int lane = threadIdx.x & 31;
  unsigned long long c1 = 0, c3 = 0;
  unsigned dn1 = 0;  // highest DN + 1 among this thread's K3-narrow segments
  unsigned dm1 = 0;  // highest DM + 1 among its K1-narrow segments
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t s0 = (int64_t)blockIdx.x * blockDim.x; s0 < a.nseg; s0 += stride) {
    const int64_t s = s0 + threadIdx.x;
    bool w1 = false, w3 = false;
    if (s < a.nseg) {
      SegGeom g = seg_geom(a, s);
      if (s == 0 && a.zprev0_first) {
        // a stream without a predecessor: segment 0 starts at its own first
        // element, the smaller of the first target / source
        g.zprev = fmin(a.M > 0 ? __ldg(a.xs) : INFINITY, a.N > 0 ? __ldg(a.ys) : INFINITY);
      }
      const double sm = seg_smax(a, g, smax);
      const int DM = seg_moment_degree(P, sm, seg_frame(g));
      // the gap factors' degree is chosen by the wide kernels from their own
      // lane runs (run_gap_degree)
      const int D = -1;
      const SegFrame f = seg_frame(g);
      const int DN = pick_degree(P, sm, f.h0 + f.h1);
      seg_deg[s] = (D + 1) | ((DM + 1) << 8) | ((DN + 1) << 16);
      w1 = !k1_narrow(DM);
      w3 = !k3_narrow(DM);
      if (!w3 && DN + 1 > dn1) dn1 = DN + 1;
      if (!w1 && DM + 1 > dm1) dm1 = DM + 1;
    }
    c1 += __popc(__ballot_sync(0xffffffffu, w1));
    c3 += __popc(__ballot_sync(0xffffffffu, w3));
  }
  dn1 = __reduce_max_sync(0xffffffffu, dn1);
  dm1 = __reduce_max_sync(0xffffffffu, dm1);
  if (lane == 0) {
    atomicAdd(counts, c1);
    atomicAdd(counts + 1, c3);
    if (dn1 > 0) atomicMax(counts + 2, (unsigned long long)dn1);
    if (dm1 > 0) atomicMax(counts + 3, (unsigned long long)dm1);
  }
}

// ------------------------------------------------------------------- K3

#ifndef FGT_K3_MINB
#define FGT_K3_MINB 5
#endif
// One segment of K3 once its lane runs are in registers (r.g = coordinates):
// segment carries, lane carries (moment form for narrow segments, warp scans
// for wide ones), both chains of every mode, staged write of u.
// The segment's staged potentials (su, sorted order) to global memory.
__device__ __forceinline__ void store_segment(const OutArgs& o, const SegGeom& g,
                                              const double* su, int lane) {
  __syncwarp();
  const int64_t base = o.u_offset + g.ib;
  if (o.tperm) {
    const int32_t* tp = o.tperm + base;
#pragma unroll
    for (int q = 0; q < kSeg / 32; ++q) {
      const int i = lane + 32 * q;
      if (i < g.nx) o.u[tp[i]] = su[i];
    }
  } else {
    double* up = o.u + base;
#pragma unroll
    for (int q = 0; q < kSeg / 32; ++q) {
      const int i = lane + 32 * q;
      if (i < g.nx) up[i] = su[i];
    }
  }
}

template <bool MS, bool WIDE>
__device__ __forceinline__ void seg_compute(const StreamArgs& a, const ModeParams& P,
                                            const ModeTable& mx, const OutArgs& o,
                                            const SegGeom& g, const SegFrame& f, int D, int DM,
                                            int DN, cplx seg_c, LaneRun& r, double zp, double zl,
                                            int lane, Carry* carries, double* su) {
  const int ne = P.ne;
  Carry* mine = carries + lane * ne;
  if constexpr (!WIDE && !MS) {
    (void)D;
    (void)DM;
    (void)zp;
    (void)zl;
    (void)mine;
    cplx* terms = reinterpret_cast<cplx*>(su + kSeg);  // [2 kMaxModes]
    switch (DN <= kNarrowMaxD ? DN : kNarrowMaxD) {
#define FGT_CS(n)                                                                   \
  case n:                                                                           \
    if constexpr (n <= kNarrowMaxD) {                                               \
      if (lane < 2 * ne) {                                                          \
        Coef<n> c;                                                                  \
        const int k = lane < ne ? lane : lane - ne;                                 \
        c.load(mx, k);                                                              \
        terms[lane] = cmul(horner<n>(c, lane < ne ? f.h0 : f.h1), seg_c);           \
      }                                                                             \
      __syncwarp();                                                                 \
      collapsed_segment<n>(mx, ne, r, f, lane, terms, su);                          \
      break;                                                                        \
    }                                                                               \
    [[fallthrough]];
      FGT_CS(0) FGT_CS(1) FGT_CS(2) FGT_CS(3) FGT_CS(4) FGT_CS(5) FGT_CS(6) FGT_CS(7)
      FGT_CS(8)
#undef FGT_CS
      default:
        break;
    }
  } else if constexpr (!WIDE) {
    cplx* terms = reinterpret_cast<cplx*>(su + kSeg);  // [2 kMaxModes]
    switch (DM) {
#define FGT_CM(n)                                                                   \
  case n: {                                                                         \
    if (lane < 2 * ne) {                                                            \
      Coef<n> c;                                                                    \
      const int k = lane < ne ? lane : lane - ne;                                   \
      c.load(mx, k);                                                                \
      terms[lane] = cmul(horner<n>(c, lane < ne ? f.h0 : f.h1), seg_c);             \
    }                                                                               \
    __syncwarp();                                                                   \
    carries_moments<n>(mx, ne, r, f, zp, zl, lane, terms, mine);                    \
  } break;
      FGT_CM(0) FGT_CM(1) FGT_CM(2) FGT_CM(3) FGT_CM(4) FGT_CM(5)
#if FGT_K3_MOMENTS >= 6
      FGT_CM(6)
#endif
#if FGT_K3_MOMENTS >= 7
      FGT_CM(7)
#endif
#if FGT_K3_MOMENTS >= 8
      FGT_CM(8)
#endif
#undef FGT_CM
      default:
        break;
    }
    static_assert(kK3Moments >= 5, "FGT_CM cases");
  }
  // Wide segments whose full width still allows the collapsed form at degree
  // 7..kCollWide (<= kCollDeg): mode-independent work per element instead of
  // per-mode gap factors and lane scans.
  bool coll = false;
  if constexpr (WIDE && !MS && kCollWide > 0) {
    if (DN >= 0 && DN <= kCollWide) {
      coll = true;
      cplx* terms = reinterpret_cast<cplx*>(su + kSeg);
      switch (DN < 7 ? 7 : DN) {
#define FGT_CW(n)                                                                   \
  case n:                                                                           \
    if constexpr (n <= kCollWide) {                                                 \
      if (lane < 2 * ne) {                                                          \
        Coef<n> c;                                                                  \
        const int k = lane < ne ? lane : lane - ne;                                 \
        c.load(mx, k);                                                              \
        terms[lane] = cmul(horner<n>(c, lane < ne ? f.h0 : f.h1), seg_c);           \
      }                                                                             \
      __syncwarp();                                                                 \
      collapsed_segment<n>(mx, ne, r, f, lane, terms, su);                          \
      break;                                                                        \
    }                                                                               \
    [[fallthrough]];
        FGT_CW(7) FGT_CW(8)
#undef FGT_CW
        default:
          break;
      }
    }
  }
  if constexpr (WIDE || MS) {
    if (!coll) {
#pragma unroll
    for (int e = kR - 1; e > 0; --e) r.g[e] -= r.g[e - 1];
    r.g[0] -= zp;
    D = run_gap_degree(P, mx.smax, r);
    if constexpr (!WIDE) __syncwarp();
    double out[kR];
#pragma unroll
    for (int e = 0; e < kR; ++e) out[e] = 0.0;
    const ModeSumsOut ms = MS ? ModeSumsOut{o.hp, o.hm, a.M, o.u_offset + g.ib + r.tfirst}
                              : ModeSumsOut{nullptr, nullptr, 0, 0};
    if constexpr (!WIDE) {
      dispatch_pass2<MS, kNarrowMaxD>(D, mx, ne, r, mine, out, ms);
    } else {
      cplx* terms = reinterpret_cast<cplx*>(su + kSeg);
      if (lane < 2 * ne) terms[lane] = seg_c;
      __syncwarp();
      wide_modes<MS>(mx, ne, D, r, lane, terms, out, ms);
    }
    if constexpr (!MS) {
      int tk = r.tfirst;
#pragma unroll
      for (int e = 0; e < kR; ++e)
        if (r.tmask & (1u << e)) su[tk++] = out[e];
    }
    }
  }
  if constexpr (!MS) store_segment(o, g, su, lane);
  __syncwarp();
}

__device__ __forceinline__ cplx load_seg_carry(const TileState& ts, int64_t nseg, int64_t s,
                                               int ne, int lane) {
  cplx c = {0.0, 0.0};
  if (lane < 2 * ne) {
    const int k = lane < ne ? lane : lane - ne;
    const int64_t idx = (int64_t)k * nseg + s;
    c = lane < ne ? ts.Cf[idx] : ts.Cb[idx];
  }
  return c;
}

#ifndef FGT_K3W_MINB
#define FGT_K3W_MINB 3
#endif
// Streaming (TMA-staged) segment loop per variant.  Both stream: the narrow
// kernel's collapsed form leaves it bound by its load latency, which the
// stage hides (cfg 3 K3 2.49 -> 1.52 ms on B200).
#ifndef FGT_K3_STREAM
#define FGT_K3_STREAM 1
#endif
#ifndef FGT_K3W_STREAM
#define FGT_K3W_STREAM 1
#endif
template <bool WIDE>
__host__ __device__ constexpr bool k3_stream() {
  return WIDE ? FGT_K3W_STREAM != 0 : FGT_K3_STREAM != 0;
}
// K3.  Narrow variant (WIDE = false): every warp streams a contiguous range
// of segments; the next segment's data is staged in shared memory by TMA
// bulk copies while the current one is computed.  Wide variant: grid-stride
// (groups of kBatchGroup for batched plans) with direct loads.  Each skips
// the other's segments.
// LANE (wide, potentials only): the lane-collapsed form; segments whose lane
// runs are too wide for it are flagged in seg_deg (kSegFallbackBit: a
// property of the plan's geometry, so the flag is set once and stays) and
// left to the wide kernel, launched behind it with a.fallback_only.
template <bool MS, bool WIDE, bool LANE = false>
__global__ void __launch_bounds__(kThreads, WIDE ? FGT_K3W_MINB : FGT_K3_MINB)
    seg_main_kernel(StreamArgs a, ModeParams P, const ModeTable* __restrict__ mtab,
                    TileState ts, OutArgs o) {
  static_assert(!LANE || (WIDE && !MS && k3_stream<true>()), "lane-collapsed: wide, streamed");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // mode tables (slot 0 shared by the CTA for single plans, one per warp for
  // batched plans), then the per-warp regions (+ the stage when streaming)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ne = P.ne;
  const bool batched = a.mtb != nullptr;
  constexpr bool STREAM = k3_stream<WIDE>();
  if constexpr (WIDE && !LANE) {
    // behind the lane-collapsed kernel: nothing flagged, nothing to do
    if (a.fallback_only && *seg_fallback_count(a.seg_deg, a.nseg) == 0) return;
  }
  // lead region: lane carries (mode sums of narrow segments), none otherwise
  constexpr int LC = LANE ? 3 : ((MS && !WIDE) ? 1 : 0);
  constexpr size_t kTab = LANE ? kLaneTableBytes : sizeof(ModeTable);
  const size_t wbytes = warp_region_bytes(ne, LC) + (STREAM ? kStageBytes : 0);
  unsigned char* wreg = smem_raw + kTab * (batched ? kSegWarps : 1) + (size_t)warp * wbytes;
  Carry* carries = reinterpret_cast<Carry*>(wreg);
  double* su = reinterpret_cast<double*>(wreg + warp_lead_bytes(ne, LC));
  if (!batched) {
    const double* src = reinterpret_cast<const double*>(mtab);
    double* dst = reinterpret_cast<double*>(smem_raw);
    for (int i = threadIdx.x; i < (int)(kTab / sizeof(double)); i += blockDim.x) dst[i] = src[i];
  }
  ModeTable& mx = *reinterpret_cast<ModeTable*>(smem_raw + (batched ? kTab * warp : 0));
  int cached_tid = -1;
  if constexpr (STREAM) {
    const StagePtrs sp = stage_ptrs(wreg + warp_region_bytes(ne, LC));
    if (lane == 0) mbar_init(sp.bar);
    __syncthreads();
    const WarpWalk walk{(int64_t)blockIdx.x * kSegWarps + warp, (int64_t)gridDim.x * kSegWarps,
                        a.nseg};
    const int64_t S1 = a.nseg;
    const int fb_only = a.fallback_only;
    // next segment of this variant at or after s (S1 if none); issues its staging
    auto issue_next = [&](int64_t s) -> int64_t {
      for (; s < S1; s = walk.next(s)) {
        const int deg = __ldg(a.seg_deg + s);
        bool mine = k3_narrow(seg_deg_DM(deg)) != WIDE;
        if constexpr (LANE) mine = mine && !(deg & kSegFallbackBit);
        if constexpr (WIDE && !LANE) mine = mine && (!fb_only || (deg & kSegFallbackBit));
        if (mine) {
          const SegGeom g = seg_geom(a, s);
          stage_issue(a, ts, ne, s, g, sp, lane);
          return s;
        }
      }
      return S1;
    };
    unsigned parity = 0;
    int64_t s = issue_next(walk.first());
    while (s < S1) {
      const SegGeom g = seg_geom(a, s);
      const SegFrame f = seg_frame(g);
      const int deg = __ldg(a.seg_deg + s);
      const int D = seg_deg_D(deg), DM = seg_deg_DM(deg);
      if (batched && g.tid != cached_tid) {
        warp_load_table<(LANE ? 2 : (MS ? 0 : 1))>(a.mtb + g.tid, mx, ne, lane);
        cached_tid = g.tid;
      }
      cp_async_wait_all();
      mbar_wait(sp.bar, parity);
      parity ^= 1u;
      __syncwarp();
      LaneRun r;
      double zp, zl;
      lane_load_stage(a, g, sp.xy, sp.bb, sp.mask[lane >> 2], lane, r, zp, zl);
      const cplx seg_c = lane < 2 * ne ? sp.car[lane] : cplx{0.0, 0.0};
      __syncwarp();  // stage free: the next segment's copies go in now
      const int64_t sn = issue_next(walk.next(s));
      if constexpr (LANE) {
        (void)f;
        (void)D;
        (void)DM;
        (void)carries;
        // slots (aliased by su), then the segment-carry terms
        cplx* slots = reinterpret_cast<cplx*>(wreg);
        cplx* terms = reinterpret_cast<cplx*>(wreg + lane_region_lead(ne));
        if (lane < 2 * ne) terms[lane] = seg_c;
        __syncwarp();
        if (lane_collapsed_dispatch(P, mx, ne, r, zp, zl, lane, terms, slots, su)) {
          store_segment(o, g, su, lane);
        } else if (lane == 0) {
          const_cast<int*>(a.seg_deg)[s] = deg | kSegFallbackBit;
          atomicAdd(seg_fallback_count(a.seg_deg, a.nseg), 1);
        }
        __syncwarp();
      } else {
        seg_compute<MS, WIDE>(a, P, mx, o, g, f, D, DM, seg_deg_DN(deg), seg_c, r, zp, zl, lane,
                              carries, su);
      }
      s = sn;
    }
  } else if constexpr (!WIDE) {
    // narrow, direct loads: contiguous chunks per warp (a bulk L2 prefetch
    // of the next segment measured slower: 3.60 vs 3.37 ms on cfg 3)
    __syncthreads();
    const WarpWalk walk{(int64_t)blockIdx.x * kSegWarps + warp, (int64_t)gridDim.x * kSegWarps,
                        a.nseg};
    // the next segment's mask word and carries are loaded while this one is
    // computed (its element loads then start without a dependent round trip)
    int64_t s = walk.first();
    uint32_t word = s < a.nseg ? lane_mask_word(a, s, lane) : 0u;
    cplx seg_c = s < a.nseg ? load_seg_carry(ts, a.nseg, s, ne, lane) : cplx{0.0, 0.0};
    while (s < a.nseg) {
      const int64_t sn = walk.next(s);
      const uint32_t word_n = sn < a.nseg ? lane_mask_word(a, sn, lane) : 0u;
      const cplx seg_c_n =
          sn < a.nseg ? load_seg_carry(ts, a.nseg, sn, ne, lane) : cplx{0.0, 0.0};
      const int deg = __ldg(a.seg_deg + s);
      const int D = seg_deg_D(deg), DM = seg_deg_DM(deg);
      if (k3_narrow(DM)) {
        const SegGeom g = seg_geom(a, s);
        const SegFrame f = seg_frame(g);
        if (batched && g.tid != cached_tid) {
          warp_load_table<(MS ? 0 : 1)>(a.mtb + g.tid, mx, ne, lane);
          cached_tid = g.tid;
        }
        LaneRun r;
        double zp, zl;
        lane_load_w(a, g, word, lane, r, zp, zl);
        seg_compute<MS, WIDE>(a, P, mx, o, g, f, D, DM, seg_deg_DN(deg), seg_c, r, zp, zl, lane, carries, su);
      }
      s = sn;
      word = word_n;
      seg_c = seg_c_n;
    }
  } else {
    __syncthreads();
    // batched plans walk groups of kBatchGroup consecutive segments (mostly
    // one transform: one table load per group); single plans go segment-wise
    const int64_t G = batched ? kBatchGroup : 1;
    for (int64_t s0 = ((int64_t)blockIdx.x * kSegWarps + warp) * G; s0 < a.nseg;
         s0 += (int64_t)gridDim.x * kSegWarps * G) {
      const int64_t s1 = s0 + G < a.nseg ? s0 + G : a.nseg;
      for (int64_t s = s0; s < s1; ++s) {
        const int deg = __ldg(a.seg_deg + s);
        const int D = seg_deg_D(deg), DM = seg_deg_DM(deg);
        if (k3_narrow(DM) == WIDE) continue;
        const SegGeom g = seg_geom(a, s);
        const SegFrame f = seg_frame(g);
        if (batched && g.tid != cached_tid) {
          warp_load_table<(MS ? 0 : 1)>(a.mtb + g.tid, mx, ne, lane);
          cached_tid = g.tid;
        }
        const cplx seg_c = load_seg_carry(ts, a.nseg, s, ne, lane);
        LaneRun r;
        double zp, zl;
        lane_load(a, g, s, lane, r, zp, zl);
        seg_compute<MS, WIDE>(a, P, mx, o, g, f, D, DM, seg_deg_DN(deg), seg_c, r, zp, zl, lane, carries, su);
      }
    }
  }
}

// ------------------------------------------------ collapsed-form helpers
//
// Per-warp scratch of the collapsed pass's moment scan (k3c): lane moments
// -> exclusive lane prefixes, segment totals.
struct K3nStage {
  double* su;      // unused (k3c stages its potentials per chunk)
  double* scan;    // [kCollMax + 1][32] lane moments -> exclusive lane prefixes
  double* tot;     // [kCollMax + 1 (+1)] segment totals
  double* zero;    // one 0.0 (the strength slot of every target)
};
// Exclusive warp prefix and total of NM per-lane values through shared
// memory: lane q < 4 NM takes moment q / 4 over lanes 8 (q % 4) .. + 7 (a
// sequential prefix of 8), then the 4 group sums of a moment are scanned by
// two shuffles.  ~40 warp instructions for NM = 4 against ~180 for NM
// Kogge-Stone shuffle scans of doubles.
template <int NM>
__device__ __forceinline__ void warp_moment_scan(const K3nStage& sp, int lane, const double (&M)[NM],
                                                 double (&pre)[NM], double (&tot)[NM]) {
  static_assert(NM <= 8, "moment scan width");
#pragma unroll
  for (int m = 0; m < NM; ++m) sp.scan[m * 32 + lane] = M[m];
  __syncwarp();
  constexpr unsigned kAct = NM * 4 >= 32 ? 0xffffffffu : ((1u << (NM * 4)) - 1u);
  if (lane < NM * 4) {
    const int m = lane >> 2, g = lane & 3;
    double2* row = reinterpret_cast<double2*>(sp.scan + m * 32 + g * 8);
    double v[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double2 t = row[i];
      v[2 * i] = t.x;
      v[2 * i + 1] = t.y;
    }
    double run = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const double t = v[i];
      v[i] = run;
      run += t;
    }
    double incl = run;
#pragma unroll
    for (int d = 1; d < 4; d <<= 1) {
      const double t = __shfl_up_sync(kAct, incl, d, 4);
      if (g >= d) incl += t;
    }
    const double excl = incl - run;
#pragma unroll
    for (int i = 0; i < 4; ++i) row[i] = make_double2(v[2 * i] + excl, v[2 * i + 1] + excl);
    if (g == 3) sp.tot[m] = incl;
  }
  __syncwarp();
#pragma unroll
  for (int m = 0; m < NM; ++m) {
    pre[m] = sp.scan[m * 32 + lane];
    tot[m] = sp.tot[m];
  }
}

__device__ __forceinline__ double lds_f64(unsigned addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts_f64(unsigned addr, double v) {
  asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(addr), "d"(v));
}

__device__ __forceinline__ void bulk_s2g(double* dst, const double* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

// 8-byte phase of a pointer within its 16-byte block (0 or 1)
__device__ __forceinline__ int phase8(const double* p) {
  return (int)((reinterpret_cast<uintptr_t>(p) >> 3) & 1);
}

// An opaque copy of a value: keeps a kernel-parameter constant in a register
// for the whole kernel instead of re-reading the constant bank at each use.
__device__ __forceinline__ double in_reg(double v) {
  double r;
  asm volatile("mov.b64 %0, %1;\n" : "=d"(r) : "d"(v));
  return r;
}

// ------------------------------------------- K3 narrow, CTA chunks (k3c)
//
// The collapsed narrow pass with a launch-uniform degree DN (the plan's
// highest collapsed degree over its narrow segments; a higher degree than a
// segment needs only adds terms below 2^-52).  A CTA of kCW compute warps
// takes a chunk of kCW consecutive segments (warp w: segment s0 + w); the
// chunk's targets, sources and strengths are three contiguous ranges, and so
// are its merge-mask words, collapsed carries, segment starts and frames, so
// one thread stages the whole chunk with seven bulk copies (two stages, the
// chunk after next in flight while one is computed) and writes the chunk's
// potentials back with one bulk store.  Per segment, per warp:
//   decode  : lane runs of kR merged elements from the mask and the plan's
//             per-word target prefix counts (w = z - zc, b)
//   moments : lane-run source moments, NM = DN + 1 -> exclusive lane prefix
//             Pre_m and segment totals Tot_m (transposed shared-memory scan)
//   evaluate: u(w) = sum_q w^q [E_q + sum_{m+q odd} H[m][q] Pre_m(w)],
//             E_q = E^c_q + sum_m B[q][m] Tot_m (the B terms folded into E^c
//             by K2m when FOLD)
// No per-mode work and no branches on the element loop.
constexpr int kCW = 8;
constexpr int kCThreads = 32 * kCW;
constexpr int kChunk = kCW * kSeg;
constexpr int kCStageXY = kChunk + 16;
constexpr int kCStageB = kChunk + 12;
constexpr int kCSu = kChunk + 4;
// stage header, written by the issuing thread before the copies
struct K3cHdr {
  long long ib0, jb0;  // first target / source of the chunk
  int xo, yo, bo;      // stage slots of x[ib0] (xy), y[jb0] (xy), b[jb0] (bb)
  int io;              // slot of seg_ib[s0] in the stage's seg_ib copy
  int nx;              // targets of the chunk
  int pad[3];
};
static_assert(sizeof(K3cHdr) == 48, "k3c header");
struct K3cStage {
  double* xy;        // [kCStageXY]
  double* bb;        // [kCStageB]
  double* ec;        // [kCW * kEcStride]
  double2* sz;       // [kCW] (zprev, zlast)
  long long* ib;     // [kCW + 3] seg_ib[s0 .. s1] as enclosing 16-byte blocks
  uint32_t* mask;    // [kCW * kSeg / 32]
  uint2* pre;        // [kCW] per-word target prefix counts (seg_mask_prefix)
  K3cHdr* hdr;
  uint64_t* bar;
};
constexpr size_t kCStageBytes = sizeof(double) * (kCStageXY + kCStageB + kCW * kEcStride) +
                                16 * kCW + 8 * (kCW + 4) + 4 * (kCW * kSeg / 32) + 8 * kCW +
                                sizeof(K3cHdr) + 16;
static_assert(kCStageBytes % 16 == 0, "k3c stage alignment");
__device__ __forceinline__ K3cStage k3c_stage(unsigned char* base) {
  K3cStage p;
  p.xy = reinterpret_cast<double*>(base);
  p.bb = p.xy + kCStageXY;
  p.ec = p.bb + kCStageB;
  p.sz = reinterpret_cast<double2*>(p.ec + kCW * kEcStride);
  p.ib = reinterpret_cast<long long*>(p.sz + kCW);
  p.mask = reinterpret_cast<uint32_t*>(p.ib + kCW + 4);
  p.pre = reinterpret_cast<uint2*>(p.mask + kCW * kSeg / 32);
  p.hdr = reinterpret_cast<K3cHdr*>(p.pre + kCW);
  p.bar = reinterpret_cast<uint64_t*>(p.hdr + 1);
  return p;
}
// per-warp scratch of the moment scan: [NM][32] lane values + NM totals
template <int NM>
constexpr size_t k3c_scratch_doubles() {
  return ((size_t)NM * 32 + NM + 2 + 1) & ~(size_t)1;
}
// staged potentials: two chunk buffers when two CTAs still fit an SM
template <int NM>
constexpr int k3c_nsu() {
  return 2 * (2 * kCStageBytes + 2 * sizeof(double) * kCSu +
              sizeof(double) * kCW * k3c_scratch_doubles<NM>() + 64) <= 225 * 1024
             ? 2
             : 1;
}
template <int NM>
constexpr size_t k3c_smem_bytes() {
  return 2 * kCStageBytes + sizeof(double) * kCSu * k3c_nsu<NM>() +
         sizeof(double) * kCW * k3c_scratch_doubles<NM>() + 64;
}

__device__ __forceinline__ void mbar_init_n(uint64_t* bar, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// Issue of chunk c (segments s0 .. s1) into a stage by one thread; ib0 / ib1
// = seg_ib[s0] / seg_ib[s1] (prefetched by the caller).
__device__ __forceinline__ void k3c_issue(const StreamArgs& a, const double* ec, int64_t c,
                                          int64_t ib0, int64_t ib1, const K3cStage& st) {
  auto blocks = [](const void* p, size_t nbytes, const void*& src) -> unsigned {
    const uintptr_t b0 = reinterpret_cast<uintptr_t>(p) & ~(uintptr_t)15;
    const uintptr_t b1 = (reinterpret_cast<uintptr_t>(p) + nbytes + 15) & ~(uintptr_t)15;
    src = reinterpret_cast<const void*>(b0);
    return nbytes > 0 ? (unsigned)(b1 - b0) : 0u;
  };
  const int64_t s0 = c * kCW;
  const int64_t s1 = s0 + kCW < a.nseg ? s0 + kCW : a.nseg;
  const int64_t L = a.M + a.N;
  const int64_t d0 = s0 * kSeg, d1 = s1 * kSeg < L ? s1 * kSeg : L;
  const int64_t jb0 = d0 - ib0, jb1 = d1 - ib1;
  const int nx = (int)(ib1 - ib0), ny = (int)(jb1 - jb0);
  const void *sx, *sy, *sb, *si;
  const unsigned bx = blocks(a.xs + ib0, 8u * nx, sx);
  const unsigned by = blocks(a.ys + jb0, 8u * ny, sy);
  const unsigned bb = blocks(a.bs + jb0, 8u * ny, sb);
  const unsigned bi = blocks(a.seg_ib + s0, 8u * (unsigned)(s1 - s0 + 1), si);
  const unsigned ns = (unsigned)(s1 - s0);
  K3cHdr h;
  h.ib0 = ib0;
  h.jb0 = jb0;
  h.xo = phase8(a.xs + ib0);
  const int ys = (h.xo + nx + 1) & ~1;
  h.yo = ys + phase8(a.ys + jb0);
  h.bo = phase8(a.bs + jb0);
  h.io = (int)((reinterpret_cast<uintptr_t>(a.seg_ib + s0) >> 3) & 1);
  h.nx = nx;
  *st.hdr = h;
  fence_proxy_async();  // generic accesses of the stage before the async writes
  const unsigned bp = (8u * ns + 15u) & ~15u;
  mbar_expect(st.bar, bx + by + bb + bi + bp + ns * (8u * kEcStride + 16u + 32u));
  if (bx) bulk_g2s(st.xy, sx, bx, st.bar);
  if (by) bulk_g2s(st.xy + ys, sy, by, st.bar);
  if (bb) bulk_g2s(st.bb, sb, bb, st.bar);
  bulk_g2s(st.ib, si, bi, st.bar);
  bulk_g2s(st.mask, a.seg_mask + s0 * (kSeg / 32), 32u * ns, st.bar);
  bulk_g2s(st.ec, ec + s0 * kEcStride, 8u * kEcStride * ns, st.bar);
  bulk_g2s(st.sz, a.seg_z + s0, 16u * ns, st.bar);
  bulk_g2s(st.pre, seg_mask_prefix(a.seg_mask, a.nseg) + s0, bp, st.bar);
}

// CTA layout: kCW compute warps (warp w: segment s0 + w of each chunk) and
// one producer warp whose elected lane stages the chunks and stores their
// potentials.  Hand-offs by mbarriers, no CTA-wide barrier in the loop:
//   full[k]  : chunk data landed in stage k (TMA transaction bytes)
//   empty[k] : all compute warps are done reading stage k (kCW arrivals)
//   sfull[j] : all compute warps staged their potentials in su[j]
//   sfree[j] : the bulk store of su[j] has read it (producer arrival)
// With a permutation or wide segments in the plan each warp writes its own
// targets back from a private region of su instead.
#ifndef FGT_K3C_MINB
#define FGT_K3C_MINB 2
#endif
template <int DN, bool FOLD>
__global__ void __launch_bounds__(kCThreads + 32, FGT_K3C_MINB)
    k3c_kernel(StreamArgs a, const double* __restrict__ ec, const CollConsts cc, OutArgs o) {
  constexpr int NM = DN + 1;
  constexpr int NSU = k3c_nsu<NM>();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* const su0 = reinterpret_cast<double*>(smem_raw + 2 * kCStageBytes);
  double* const scr0 = su0 + (size_t)kCSu * NSU;
  uint64_t* const bars = reinterpret_cast<uint64_t*>(scr0 + (size_t)kCW * k3c_scratch_doubles<NM>());
  uint64_t* const empty = bars;        // [2]
  uint64_t* const sfull = bars + 2;    // [NSU]
  uint64_t* const sfree = bars + 4;    // [NSU]
  double* const zero = reinterpret_cast<double*>(bars + 6);
  const int64_t nchunk = (a.nseg + kCW - 1) / kCW;
  const int64_t L = a.M + a.N;
  const bool all_narrow = a.nwide3 == 0;
  const bool bulk_out = all_narrow && !o.tperm;
  if (threadIdx.x == 0) {
    mbar_init(k3c_stage(smem_raw).bar);
    mbar_init(k3c_stage(smem_raw + kCStageBytes).bar);
    for (int i = 0; i < 2; ++i) mbar_init_n(empty + i, kCW);
    for (int j = 0; j < NSU; ++j) {
      mbar_init_n(sfull + j, kCW);
      mbar_init_n(sfree + j, 1);
    }
    zero[0] = 0.0;
  }
  __syncthreads();
  if (warp == kCW) {
    // ---------------- producer
    if (lane != 0) return;
    auto chunk_ib = [&](int64_t c, int64_t& i0, int64_t& i1) {
      const int64_t s0 = c * kCW;
      const int64_t s1 = s0 + kCW < a.nseg ? s0 + kCW : a.nseg;
      i0 = __ldg(a.seg_ib + s0);
      i1 = __ldg(a.seg_ib + s1);
    };
    // (first target, target count) of the chunk in each stage
    int64_t gib[2] = {0, 0};
    int gnx[2] = {0, 0};
    for (int i = 0; i < 2; ++i) {
      const int64_t c = blockIdx.x + (int64_t)i * gridDim.x;
      if (c < nchunk) {
        int64_t i0, i1;
        chunk_ib(c, i0, i1);
        k3c_issue(a, ec, c, i0, i1, k3c_stage(smem_raw + i * kCStageBytes));
        gib[i] = i0;
        gnx[i] = (int)(i1 - i0);
      }
    }
    int64_t nib0 = 0, nib1 = 0;
    if (blockIdx.x + 2 * (int64_t)gridDim.x < nchunk)
      chunk_ib(blockIdx.x + 2 * (int64_t)gridDim.x, nib0, nib1);
    int it = 0;
    for (int64_t c = blockIdx.x; c < nchunk; c += gridDim.x, ++it) {
      const int k = it & 1;
      const int64_t ib0 = k ? gib[1] : gib[0];
      const int nx = k ? gnx[1] : gnx[0];
      const int64_t c2 = c + 2 * (int64_t)gridDim.x;
      if (c2 < nchunk) {
        mbar_wait(empty + k, (unsigned)(it >> 1) & 1u);
        k3c_issue(a, ec, c2, nib0, nib1, k3c_stage(smem_raw + k * kCStageBytes));
        if (k) {
          gib[1] = nib0;
          gnx[1] = (int)(nib1 - nib0);
        } else {
          gib[0] = nib0;
          gnx[0] = (int)(nib1 - nib0);
        }
        if (c2 + gridDim.x < nchunk) chunk_ib(c2 + gridDim.x, nib0, nib1);
      }
      if (bulk_out) {
        const int j = NSU == 2 ? k : 0;
        double* const su = su0 + (size_t)j * kCSu;
        mbar_wait(sfull + j, (unsigned)(it / NSU) & 1u);
        double* const up = o.u + o.u_offset + ib0;
        const int uoff = (int)((reinterpret_cast<uintptr_t>(up) >> 3) & 1);
        const int cnt = (nx - uoff) & ~1;
        fence_proxy_async();  // the compute warps' stores to su before the async read
        if (cnt > 0) bulk_s2g(up + uoff, su + 2 * uoff, 8u * (unsigned)cnt);
        if (uoff && nx > 0) up[0] = su[1];
        if (uoff + cnt < nx) up[nx - 1] = su[nx - 1 + uoff];
        bulk_wait_read();
        mbar_arrive(sfree + j);
      }
    }
    bulk_wait_all();
    return;
  }
  // ---------------- compute warps
  K3nStage sp;  // the moment scan's scratch
  sp.su = nullptr;
  sp.scan = scr0 + (size_t)warp * k3c_scratch_doubles<NM>();
  sp.tot = sp.scan + NM * 32;
  sp.zero = zero;
  const unsigned az = smem_u32(zero);
  double Hr[NM][NM], Br[NM][NM];
#pragma unroll
  for (int m = 0; m < NM; ++m)
#pragma unroll
    for (int q = 0; q < NM; ++q) {
      Hr[m][q] = (m + q < NM && ((m + q) & 1)) ? in_reg(cc.H[m][q]) : 0.0;
      Br[q][m] = (!FOLD && m + q < NM) ? in_reg(cc.B[q][m]) : 0.0;
    }
  int it = 0;
  for (int64_t c = blockIdx.x; c < nchunk; c += gridDim.x, ++it) {
    const int k = it & 1;
    const K3cStage st = k3c_stage(smem_raw + k * kCStageBytes);
    mbar_wait(st.bar, (unsigned)(it >> 1) & 1u);
    const K3cHdr h = *st.hdr;
    const int64_t s = c * kCW + warp;
    // this warp's segment from the staged starts and frames
    bool live = s < a.nseg;
    int nx = 0, ny = 0, len = 0, lx = 0, ly = 0;
    double zc = 0.0;
    if (live) {
      const int64_t ib = st.ib[h.io + warp], ie = st.ib[h.io + warp + 1];
      const int64_t d0 = s * kSeg;
      len = (int)(d0 + kSeg < L ? kSeg : L - d0);
      nx = (int)(ie - ib);
      ny = len - nx;
      lx = (int)(ib - h.ib0);
      ly = (int)(d0 - ib - h.jb0);
      const double2 z = st.sz[warp];
      SegGeom g;
      g.zprev = s == 0 ? a.zprev0 : z.x;
      g.zlast = z.y;
      zc = seg_frame(g).zc;
      if (!all_narrow) live = k3_narrow(seg_deg_DM(__ldg(a.seg_deg + s)));
    }
    double w[kR], L8[kR], cq[NM];
    unsigned byte = 0;
    int i0 = 0;
    if (live) {
      const int xo = h.xo + lx, yo = h.yo + ly, bo = h.bo + ly;
      if (len < kSeg) {
        // partial (last) segment: lanes past the end decode as strength-0
        // sources at the centre (their mask bits are 0)
        for (int q = lane; q < kSeg - len + 8; q += 32) {
          st.xy[yo + ny + q] = zc;
          st.bb[bo + ny + q] = 0.0;
        }
        fence_proxy_async();  // before the stage is refilled by the async proxy
        __syncwarp();
      }
      const uint32_t word = st.mask[warp * (kSeg / 32) + (lane >> 2)];
      const unsigned sh = (lane & 3) * 8;
      byte = (word >> sh) & 0xffu;
      // targets before this lane's run: the word prefix (plan-time) + the
      // lower bytes of its own word
      const uint2 pw = st.pre[warp];
      const unsigned pq = lane & 16 ? pw.y : pw.x;
      i0 = (int)((pq >> ((lane & 12) * 2)) & 0xffu) + __popc(word & ((1u << sh) - 1u));
      const int j0 = lane * kR - i0;
      unsigned ax = smem_u32(st.xy + xo + i0);
      unsigned ay = smem_u32(st.xy + yo + j0);
      unsigned ab = smem_u32(st.bb + bo + j0);
      double lp[NM];
#pragma unroll
      for (int m = 0; m < NM; ++m) lp[m] = 0.0;
#pragma unroll
      for (int e = 0; e < kR; ++e) {
        const unsigned tg = (byte >> e) & 1u;
        const double we = lds_f64(tg ? ax : ay) - zc;
        double p = lds_f64(tg ? az : ab);
        ax += tg << 3;
        ay += (tg ^ 1u) << 3;
        ab += (tg ^ 1u) << 3;
        lp[0] += p;
#pragma unroll
        for (int m = 1; m < NM; ++m) {
          p *= we;
          lp[m] += p;
        }
        double acc = 0.0;
#pragma unroll
        for (int q = DN; q >= 0; --q) {
          double c2 = 0.0;
          bool any = false;
#pragma unroll
          for (int m = 0; m + q < NM; ++m)
            if ((m + q) & 1) {
              c2 = any ? fma(Hr[m][q], lp[m], c2) : Hr[m][q] * lp[m];
              any = true;
            }
          acc = q == DN ? c2 : fma(acc, we, c2);
        }
        w[e] = we;
        L8[e] = acc;
      }
      double ecq[NM];
#pragma unroll
      for (int q = 0; q < NM; ++q) ecq[q] = st.ec[warp * kEcStride + q];
      double pre[NM], tot[NM];
      warp_moment_scan<NM>(sp, lane, lp, pre, tot);
#pragma unroll
      for (int q = 0; q < NM; ++q) {
        double acc = ecq[q];
        if constexpr (!FOLD) {
#pragma unroll
          for (int m = 0; m + q < NM; ++m) acc = fma(Br[q][m], tot[m], acc);
        }
#pragma unroll
        for (int m = 0; m + q < NM; ++m)
          if ((m + q) & 1) acc = fma(Hr[m][q], pre[m], acc);
        cq[q] = acc;
      }
    }
    // the stage is consumed
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + k);
    const int j = NSU == 2 ? k : 0;
    double* const su = su0 + (size_t)j * kCSu;
    int base;
    if (bulk_out) {
      // chunk slots (aligned like u); wait for the store that last read su[j]
      if (it >= NSU) mbar_wait(sfree + j, (unsigned)(it / NSU - 1) & 1u);
      base = (int)((reinterpret_cast<uintptr_t>(o.u + o.u_offset + h.ib0) >> 3) & 1) + lx;
    } else {
      base = warp * kSeg;  // private region
    }
    if (live) {
      unsigned at = smem_u32(su + base + i0);
      const unsigned adis = smem_u32(su + kChunk + 2);  // discard slot of non-targets
#pragma unroll
      for (int e = 0; e < kR; ++e) {
        double acc = cq[DN];
#pragma unroll
        for (int q = DN - 1; q >= 0; --q) acc = fma(acc, w[e], cq[q]);
        const unsigned tg = (byte >> e) & 1u;
        sts_f64(tg ? at : adis, acc + L8[e]);
        at += tg << 3;
      }
    }
    __syncwarp();
    if (bulk_out) {
      if (lane == 0) mbar_arrive(sfull + j);
    } else if (live) {
      const int64_t t0 = o.u_offset + h.ib0 + lx;
      if (o.tperm) {
        const int32_t* tp = o.tperm + t0;
        for (int i = lane; i < nx; i += 32) o.u[tp[i]] = su[base + i];
      } else {
        for (int i = lane; i < nx; i += 32) o.u[t0 + i] = su[base + i];
      }
      __syncwarp();
    }
  }
}

// Collapsed carries of the narrow segments (after K2): per segment, the
// segment carries at the frame centre Tf_k = e^{-s_k h0} Cf_k, Tb_k =
// e^{-s_k h1} Cb_k folded into E^c_q = Re sum_k mw_k c_kq (Tf_k + (-1)^q Tb_k),
// q <= DN (collapsed_segment's carry part, done once per segment here
// instead of on a few lanes of every K3 warp).
__global__ void collapse_carries_kernel(StreamArgs a, const ModeTable* __restrict__ mt,
                                        int ne, TileState ts, int DN) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.nseg) return;
  if (!k3_narrow(seg_deg_DM(__ldg(a.seg_deg + s)))) return;
  const SegFrame f = seg_frame(seg_geom(a, s));
  double E[kCollMax + 1];
#pragma unroll
  for (int q = 0; q <= kCollMax; ++q) E[q] = 0.0;
  for (int k = 0; k < ne; ++k) {
    const cplx* c = mt->coef[k];
    // e^{-s h} by the degree-DN Taylor polynomial (|s h| <= rmax[DN] / 2)
    cplx e0 = c[DN], e1 = c[DN];
    for (int n = DN - 1; n >= 0; --n) {
      const cplx cn = c[n];
      e0 = {fma(e0.re, f.h0, cn.re), fma(e0.im, f.h0, cn.im)};
      e1 = {fma(e1.re, f.h1, cn.re), fma(e1.im, f.h1, cn.im)};
    }
    const int64_t idx = (int64_t)k * a.nseg + s;
    const cplx tf = cmul(e0, ts.Cf[idx]);
    const cplx tb = cmul(e1, ts.Cb[idx]);
#pragma unroll
    for (int q = 0; q <= kCollMax; ++q) {
      if (q <= DN) {
        const cplx x = mt->mwc[k][q];
        const double sg = (q & 1) ? -1.0 : 1.0;
        E[q] = fma(x.re, fma(sg, tb.re, tf.re), fma(-x.im, fma(sg, tb.im, tf.im), E[q]));
      }
    }
  }
  double* out = ts.ec + s * kEcStride;
#pragma unroll
  for (int q = 0; q <= kCollMax; ++q) out[q] = q <= DN ? E[q] : 0.0;
#pragma unroll
  for (int q = kCollMax + 1; q < kEcStride; ++q) out[q] = 0.0;
}

// ------------------------------------------------------------------- K0

__global__ void partition_kernel(const double* __restrict__ xs, int64_t M,
                                 const double* __restrict__ ys, int64_t N, int64_t seg,
                                 int64_t nseg, int64_t* __restrict__ seg_ib) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t > nseg) return;
  int64_t diag = t * seg;
  if (diag > M + N) diag = M + N;
  seg_ib[t] = merge_path_guess(xs, M, ys, N, diag);
}

// Plan-time tile pass (one CTA per tile of kPlanTile merged elements,
// speculative: run on the input as given).  Stages the tile's targets and
// sources in shared memory and, in one read of both sets:
//   - checks finiteness, sortedness (incl. the pair across the tile start)
//     and, when M == N, element-wise equality of the two vectors
//     (flags[0..4] as launch_plan_checks);
//   - splits the tile into segments by merge path in shared memory
//     (seg_ib), places every target of a segment by ranking it among the
//     segment's sources (sources at equal coordinates first) -> one bit per
//     merged element (seg_mask), and records (zprev, zlast) per segment.
// Tile context: the (transform-local) arrays a plan tile works on and where
// its segment metadata goes.
struct TileCtx {
  const double* x;  // targets of the stream the tile belongs to
  int64_t M;
  const double* y;  // sources
  int64_t N;
  int64_t ib, ie;    // local target range of the tile
  int64_t d0, d1;    // local merged range
  int64_t seg0;      // global index of the tile's first segment
  int64_t xoff, yoff;  // global offsets of the local arrays (batched plans)
  int tid;
};

#ifndef FGT_PLAN_MINB
#define FGT_PLAN_MINB 6
#endif
// Merged positions per thread: one per segment of the tile, so a tile of
// kPlanSegs segments has kSeg threads.  An odd window spreads the
// threads' merge reads over the shared-memory banks (the window starts are
// about kPlanPer / 2 doubles apart in each set; an even window of 16 put
// them 8 doubles = 64 bytes apart, i.e. on the same banks).
constexpr int kPlanPer = kPlanSegs;
constexpr int kPlanThreads = kSeg;
constexpr int kPlanWords = kPlanTile / 32;  // merge-mask words per tile
static_assert(kPlanPer < 32 && kSeg % 32 == 0, "plan tile layout");

// Staging plan of n values g[0..n) into a shared buffer: the 16-byte aligned
// interior by one bulk copy, an unaligned head / tail element by plain
// loads.  The values land at s = buf + head, s[0..n).
struct Stage {
  int head;         // 1 when g is not 16-byte aligned (g[0] loaded by a thread)
  int i0, i1;       // interior [i0, i1) (bulk)
  int tail;         // 1 when g[n-1] lies past the interior
};
__device__ __forceinline__ Stage stage_plan(const double* g, int n) {
  Stage st;
  st.head = (n > 0 && (reinterpret_cast<uintptr_t>(g) & 15u)) ? 1 : 0;
  st.i0 = st.head;
  int i1 = st.i0 + ((n - st.i0) & ~1);
  if (i1 < st.i0) i1 = st.i0;
  st.i1 = i1;
  st.tail = (n > st.i1) ? 1 : 0;
  return st;
}

// 32-bit merge path in shared memory (sources first at ties).
__device__ __forceinline__ int merge_path_smem(const double* x, int nx, const double* y, int ny,
                                               int diag) {
  int lo = diag - ny > 0 ? diag - ny : 0;
  int hi = diag < nx ? diag : nx;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (x[mid - 1] < y[diag - mid])
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

template <bool BATCH>
__device__ __forceinline__ void plan_tile_body(const TileCtx& c, int check_sorted,
                                               int64_t nseg, int64_t* __restrict__ seg_ib,
                                               int64_t* __restrict__ seg_jb,
                                               int4* __restrict__ seg_info,
                                               double2* __restrict__ seg_z,
                                               uint32_t* __restrict__ seg_mask,
                                               int* __restrict__ flags,
                                               const PlanClassify* cls = nullptr) {
  extern __shared__ __align__(16) double tsm[];
  __shared__ int sib[kPlanSegs + 1];
  __shared__ int swin[kPlanThreads];
  __shared__ uint32_t smask[kPlanWords];
  __shared__ int sflags;
  __shared__ __align__(8) uint64_t bar;
  const int64_t ib = c.ib, ie = c.ie;
  const int64_t jb = c.d0 - ib, je = c.d1 - ie;
  const int64_t nx64 = ie - ib, len64 = c.d1 - c.d0;
  if (nx64 < 0 || nx64 > len64) {
    // partition of an unsorted stream (speculative pass): the host re-checks
    // the whole input (launch_check_points) and sorts; report and bail out
    if (threadIdx.x == 0) atomicOr(flags + 3, 1);
    return;
  }
  const int nx = (int)nx64, ny = (int)(je - jb), len = (int)len64;
  const int t = threadIdx.x, lane = t & 31;
  const double* gx = c.x + ib;
  const double* gy = c.y + jb;
  const Stage stx = stage_plan(gx, nx), sty = stage_plan(gy, ny);
  // one buffer for both sets (nx + ny <= kPlanTile): x (+ sentinel) first,
  // y from the next even slot (16-byte aligned interiors)
  const int oy = (stx.head + nx + 1 + 1) & ~1;
  double* sx = tsm + stx.head;
  double* sy = tsm + oy + sty.head;
  if (t == 0) {
    sflags = 0;
    mbar_init(&bar);
  }
  for (int w = t; w < kPlanWords; w += kPlanThreads) smask[w] = 0u;
  __syncthreads();
  if (t == 0) {
    const unsigned bx = 8u * (unsigned)(stx.i1 - stx.i0), by = 8u * (unsigned)(sty.i1 - sty.i0);
    mbar_expect(&bar, bx + by);
    if (bx) bulk_g2s(sx + stx.i0, gx + stx.i0, bx, &bar);
    if (by) bulk_g2s(sy + sty.i0, gy + sty.i0, by, &bar);
  }
  if (t == 1 && stx.head) sx[0] = __ldg(gx);
  if (t == 2 && stx.tail) sx[nx - 1] = __ldg(gx + nx - 1);
  if (t == 3 && sty.head) sy[0] = __ldg(gy);
  if (t == 4 && sty.tail) sy[ny - 1] = __ldg(gy + ny - 1);
  if (t == 5) sx[nx] = INFINITY;  // merge sentinels
  if (t == 6) sy[ny] = INFINITY;
  // neighbours across the tile start (sortedness)
  const double xprev = (t == 0 && ib > 0 && nx > 0) ? __ldg(gx - 1) : -INFINITY;
  const double yprev = (t == 0 && jb > 0 && ny > 0) ? __ldg(gy - 1) : -INFINITY;
  mbar_wait(&bar, 0);
  __syncthreads();
  int f0 = 0, f1 = 0, f2 = 0, f3 = 0, f4 = 0;
  // merge-path splits in two levels: the segment starts over the whole tile,
  // then every thread's window inside its segment's split range
  const int nsegs_tile = (len + kSeg - 1) / kSeg;
  if (t < nsegs_tile) sib[t] = merge_path_smem(sx, nx, sy, ny, t * kSeg);
  if (t == 0) sib[nsegs_tile] = nx;
  __syncthreads();
  // merge: thread t owns merged positions [kPlanPer t, kPlanPer (t + 1)) and
  // sets their mask bits (1 = target).  The checks ride on the walk: every
  // consumed value is tested for finiteness and against the previous value
  // of its set, and (M == N) the stream must alternate source, equal target
  // (x == y elementwise for sorted sets, transform.cpp:214-216).  The walk
  // visits every element of the tile exactly once when the windows chain
  // (each ends where the next starts), which is checked too; a broken chain
  // reports "unsorted", and the host then re-checks the input element-wise.
  const int d0 = t * kPlanPer;
  const bool same_chk = !BATCH && c.M == c.N && *(volatile int*)(flags + 2) == 0;
  int iend = -1, istart = -1;
  if (d0 < len) {
    const int k = d0 / kSeg, D0 = k * kSeg;
    int i;
    {
      const int D1 = D0 + kSeg < len ? D0 + kSeg : len;
      const int ilo = sib[k], ihi = sib[k + 1];
      const int jhi = D1 - ihi;
      int lo = d0 - jhi > ilo ? d0 - jhi : ilo;
      int hi = ilo + (d0 - D0) < ihi ? ilo + (d0 - D0) : ihi;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (sx[mid - 1] < sy[d0 - mid])
          lo = mid;
        else
          hi = mid - 1;
      }
      i = lo;
    }
    istart = i;
    int j = d0 - i;
    // no index clamps: on sorted input the merge never reads past a set's
    // sentinel; on unsorted input (flagged, redone after the sort) it can
    // run up to kPlanPer past it, into the buffer's padding
    double cx = sx[i];
    double cy = sy[j];
    double lx = i > 0 ? sx[i - 1] : (t == 0 ? xprev : -INFINITY);
    double ly = j > 0 ? sy[j - 1] : (t == 0 ? yprev : -INFINITY);
    double zp = fmax(lx, ly);
    unsigned bits = 0u;
    const int nwin = len - d0 < kPlanPer ? len - d0 : kPlanPer;
#pragma unroll
    for (int e = 0; e < kPlanPer; ++e) {
      if (e < nwin) {
        const bool tgt = !(cy <= cx);  // sources first on ties
        const double z = tgt ? cx : cy;
        const bool fin = isfinite(z);
        if (tgt) {
          f0 |= !fin;
          f3 |= z < lx;
          lx = z;
          ++i;
          cx = sx[i];
        } else {
          f1 |= !fin;
          f4 |= z < ly;
          ly = z;
          ++j;
          cy = sy[j];
        }
        if (same_chk) f2 |= (tgt != ((e + d0) & 1)) | (tgt && z != zp);
        zp = z;
        bits |= (unsigned)tgt << e;
      }
    }
    if (!check_sorted) f3 = f4 = 0;
    iend = i;
    const int sh = d0 & 31;
    atomicOr(&smask[d0 >> 5], bits << sh);
    if (sh + kPlanPer > 32) atomicOr(&smask[(d0 >> 5) + 1], bits >> (32 - sh));
  }
  // chain check: every window starts where the previous one ended, and the
  // last one ends at the tile's end (then the walk covered every element)
  swin[t] = istart;
  __syncthreads();
  if (d0 < len) {
    const bool last = d0 + kPlanPer >= len;
    if (last ? iend != nx : iend != swin[t + 1]) f3 = 1;
  }
  __syncthreads();
  for (int w = t; w < nsegs_tile * (kSeg / 32); w += kPlanThreads)
    seg_mask[c.seg0 * (kSeg / 32) + w] = smask[w];
  if (!BATCH && t < nsegs_tile) {
    // per-word target prefix counts of the segment (byte q: targets in
    // words 0 .. q-1), read by k3c in place of a warp scan
    unsigned pre = 0, lo = 0, hi = 0;
#pragma unroll
    for (int q = 0; q < kSeg / 32; ++q) {
      if (q < 4)
        lo |= pre << (8 * q);
      else
        hi |= pre << (8 * (q - 4));
      pre += __popc(smask[t * (kSeg / 32) + q]);
    }
    seg_mask_prefix(seg_mask, nseg)[c.seg0 + t] = make_uint2(lo, hi);
  }
  bool cw1 = false, cw3 = false;
  int cdn = 0, cdm = 0;
  if (t < nsegs_tile) {
    const int k = t;
    const int i0 = sib[k], i1 = sib[k + 1];
    const int sd0 = k * kSeg;
    const int sd1 = (sd0 + kSeg < len) ? sd0 + kSeg : len;
    const int j0 = sd0 - i0, j1 = sd1 - i1;
    const int64_t sg = c.seg0 + k;
    seg_ib[sg] = c.xoff + ib + i0;
    if constexpr (BATCH) {
      seg_jb[sg] = c.yoff + jb + j0;
      seg_info[sg] = make_int4(sd1 - sd0, i1 - i0, c.tid, 0);
    }
    double px, py;
    if (k == 0) {
      // -inf at the start of a stream (a new transform never couples back)
      px = ib > 0 ? __ldg(c.x + ib - 1) : -INFINITY;
      py = jb > 0 ? __ldg(c.y + jb - 1) : -INFINITY;
    } else {
      px = i0 > 0 ? sx[i0 - 1] : -INFINITY;
      py = j0 > 0 ? sy[j0 - 1] : -INFINITY;
    }
    const double lx = i1 > i0 ? sx[i1 - 1] : -INFINITY;
    const double ly = j1 > j0 ? sy[j1 - 1] : -INFINITY;
    seg_z[sg] = make_double2(fmax(px, py), fmax(lx, ly));
    if (!BATCH && sg + 1 == nseg) seg_ib[nseg] = c.M;
    if (!BATCH && cls && cls->enabled) {
      // classify_kernel's degrees, from this segment's frame
      double zp = fmax(px, py);
      if (sg == 0)
        zp = cls->has_prev ? cls->z_prev
                           : fmin(nx > 0 ? sx[0] : INFINITY, ny > 0 ? sy[0] : INFINITY);
      SegGeom g;
      g.zprev = zp;
      g.zlast = fmax(lx, ly);
      const SegFrame f = seg_frame(g);
      const int DM = seg_moment_degree(cls->P, cls->smax, f);
      const int DN = pick_degree(cls->P, cls->smax, f.h0 + f.h1);
      cls->seg_deg[sg] = 0 | ((DM + 1) << 8) | ((DN + 1) << 16);
      cw1 = !k1_narrow(DM);
      cw3 = !k3_narrow(DM);
      cdn = !cw3 ? DN + 1 : 0;
      cdm = !cw1 ? DM + 1 : 0;
    }
  }
  if (!BATCH && cls && cls->enabled && t < 32) {
    // the tile's segments are all in warp 0: one slot update per CTA
    const unsigned n1 = __popc(__ballot_sync(0xffffffffu, cw1));
    const unsigned n3 = __popc(__ballot_sync(0xffffffffu, cw3));
    const unsigned mdn = __reduce_max_sync(0xffffffffu, (unsigned)cdn);
    const unsigned mdm = __reduce_max_sync(0xffffffffu, (unsigned)cdm);
    if (t == 0) {
      unsigned long long* slot = cls->counts + 4 * (blockIdx.x % kClassSlots);
      if (n1) atomicAdd(slot, (unsigned long long)n1);
      if (n3) atomicAdd(slot + 1, (unsigned long long)n3);
      if (mdn) atomicMax(slot + 2, (unsigned long long)mdn);
      if (mdm) atomicMax(slot + 3, (unsigned long long)mdm);
    }
  }
  int fl = (f0 ? 1 : 0) | (f1 ? 2 : 0) | (f2 ? 4 : 0) | (f3 ? 8 : 0) | (f4 ? 16 : 0);
  fl = __reduce_or_sync(0xffffffffu, fl);
  if (lane == 0 && fl) atomicOr(&sflags, fl);
  __syncthreads();
  if (t == 0 && sflags) {
    for (int q = 0; q < 5; ++q)
      if (sflags & (1 << q)) atomicOr(flags + q, 1);
  }
}

__global__ void __launch_bounds__(kPlanThreads, FGT_PLAN_MINB)
    plan_tile_kernel(const double* __restrict__ xs, int64_t M, const double* __restrict__ ys,
                     int64_t N, const int64_t* __restrict__ tile_ib, int64_t nseg,
                     int check_sorted, int64_t* __restrict__ seg_ib, double2* __restrict__ seg_z,
                     uint32_t* __restrict__ seg_mask, int* __restrict__ flags,
                     const __grid_constant__ PlanClassify cls) {
  const int64_t t = blockIdx.x;
  const int64_t L = M + N;
  TileCtx c;
  c.x = xs;
  c.M = M;
  c.y = ys;
  c.N = N;
  c.ib = tile_ib[t];
  c.ie = tile_ib[t + 1];
  c.d0 = t * kPlanTile;
  c.d1 = (c.d0 + kPlanTile < L) ? c.d0 + kPlanTile : L;
  c.seg0 = t * kPlanSegs;
  c.xoff = c.yoff = 0;
  c.tid = 0;
  plan_tile_body<false>(c, check_sorted, nseg, seg_ib, nullptr, nullptr, seg_z, seg_mask, flags,
                        &cls);
}

struct BatchArgs {
  const double* xs;
  const double* ys;
  const int64_t* t_off;
  const int64_t* s_off;
  const int64_t* seg_base;
  const int64_t* tile_base;
  const int32_t* tile_tid;
};

__device__ __forceinline__ TileCtx batch_ctx(const BatchArgs& b, int64_t gt, const int64_t* tile_ib) {
  TileCtx c;
  const int tid = b.tile_tid[gt];
  const int64_t lt = gt - b.tile_base[tid];
  c.tid = tid;
  c.xoff = b.t_off[tid];
  c.yoff = b.s_off[tid];
  c.x = b.xs + c.xoff;
  c.M = b.t_off[tid + 1] - c.xoff;
  c.y = b.ys + c.yoff;
  c.N = b.s_off[tid + 1] - c.yoff;
  const int64_t L = c.M + c.N;
  c.d0 = lt * kPlanTile;
  c.d1 = (c.d0 + kPlanTile < L) ? c.d0 + kPlanTile : L;
  c.seg0 = b.seg_base[tid] + lt * kPlanSegs;
  if (tile_ib) {
    c.ib = tile_ib[gt];
    c.ie = gt + 1 < b.tile_base[tid + 1] ? tile_ib[gt + 1] : c.M;
  }
  return c;
}

__global__ void batch_partition_kernel(BatchArgs b, int64_t ntiles, int64_t* __restrict__ tile_ib) {
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gt >= ntiles) return;
  const TileCtx c = batch_ctx(b, gt, nullptr);
  tile_ib[gt] = merge_path(c.x, c.M, c.y, c.N, c.d0);
}

__global__ void __launch_bounds__(kPlanThreads, FGT_PLAN_MINB)
    batch_plan_tile_kernel(BatchArgs b, const int64_t* __restrict__ tile_ib,
                           int64_t* __restrict__ seg_ib, int64_t* __restrict__ seg_jb,
                           int4* __restrict__ seg_info, double2* __restrict__ seg_z,
                           uint32_t* __restrict__ seg_mask, int* __restrict__ flags) {
  const TileCtx c = batch_ctx(b, blockIdx.x, tile_ib);
  plan_tile_body<true>(c, 1, 0, seg_ib, seg_jb, seg_info, seg_z, seg_mask, flags);
}

// Element-wise checks of the input as given (no partition involved):
// flags[0] / [1] a non-finite target / source, [2] x[i] != y[i] somewhere
// (M == N only), [3] / [4] targets / sources out of order.  The plan's tile
// pass checks a sorted input in the same read as its metadata; on input it
// finds unsorted (whose merge-path tiles need not cover every element) the
// host runs this pass over the original arrays (check_points, transform.cpp:
// 21-25; same_points, :214-216).
__global__ void check_points_kernel(const double* __restrict__ x, int64_t M,
                                    const double* __restrict__ y, int64_t N,
                                    int* __restrict__ flags) {
  const int64_t L = M > N ? M : N;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int f = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < L; i += stride) {
    double xv = 0.0, yv = 0.0;
    if (i < M) {
      xv = __ldg(x + i);
      f |= !isfinite(xv) ? 1 : 0;
      if (i > 0 && __ldg(x + i - 1) > xv) f |= 8;
    }
    if (i < N) {
      yv = __ldg(y + i);
      f |= !isfinite(yv) ? 2 : 0;
      if (i > 0 && __ldg(y + i - 1) > yv) f |= 16;
    }
    if (M == N && !(xv == yv)) f |= 4;
  }
  f = __reduce_or_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0 && f) {
    for (int q = 0; q < 5; ++q)
      if (f & (1 << q)) atomicOr(flags + q, 1);
  }
}

// ------------------------------------------------------------------- K2
// Scan of (a, s) pairs over segments, one (mode, direction) per blockIdx.y:
// q < ne forward of mode q over F, q >= ne backward of mode q - ne over G in
// reversed segment order.  Three phases: per-block reduce, top-level scan of
// block aggregates (one CTA per q), per-block down-sweep writing carries.

#ifndef FGT_SCAN_THREADS
#define FGT_SCAN_THREADS 128
#endif
constexpr int kScanThreads = FGT_SCAN_THREADS;
// Grid caps (CTAs per SM) of K1 and of the K3 non-streaming variants; waves
// of resident CTAs for the streaming (wide) K3.
#ifndef FGT_K3N_WAVES
#define FGT_K3N_WAVES 32
#endif
#ifndef FGT_K3W_WAVES
#define FGT_K3W_WAVES 32
#endif
// (batched plans: segment costs differ by the lane-run degree, 4 .. 16, so
// smaller ranges per CTA balance better: cfg 5 K3 10.75 ms at 32 waves, 10.41
// at 128, 10.43 at 256, 10.62 at 512, 11.2 at 8)
#ifndef FGT_K3W_WAVES_BATCH
#define FGT_K3W_WAVES_BATCH 128
#endif
#ifndef FGT_K1_GRID
#define FGT_K1_GRID 64
#endif
// batched plans: segment costs vary from transform to transform (their own
// delta), so the grids are finer (cfg 5 K1: 4.09 ms at 64, 4.00 at 256)
#ifndef FGT_K1_GRID_BATCH
#define FGT_K1_GRID_BATCH 256
#endif
#ifndef FGT_K3_GRID
#define FGT_K3_GRID 64
#endif
#ifndef FGT_SCAN_ITEMS
#define FGT_SCAN_ITEMS 2
#endif
constexpr int kScanItems = FGT_SCAN_ITEMS;
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
  cplx* blka = nullptr;  // [2ne][nblk] exclusive products of the block A's (moment path)
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
  // thread aggregates of contiguous runs, then an inclusive scan over the
  // 1024 threads: warp shuffles, the 32 warp totals by warp 0 (two barriers
  // instead of a 10-step Hillis-Steele over shared memory)
  __shared__ Pair sp[1024];
  __shared__ Pair wsp[32];
  const int q = blockIdx.x;
  const int ne = sa.ne;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t per = (sa.nblk + 1023) / 1024;
  const int64_t r0 = (int64_t)threadIdx.x * per;
  const int64_t r1 = r0 + per < sa.nblk ? r0 + per : sa.nblk;
  const cplx* ag = sa.blkagg + (int64_t)q * sa.nblk * 2;
  Pair acc{{1.0, 0.0}, {0.0, 0.0}};
  for (int64_t r = r0; r < r1; ++r) acc = combine(acc, Pair{ag[2 * r], ag[2 * r + 1]});
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const Pair p = shfl_up_pair(acc, off);
    if (lane >= off) acc = combine(p, acc);
  }
  if (lane == 31) wsp[warp] = acc;
  __syncthreads();
  if (warp == 0) {
    Pair w = wsp[lane];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const Pair p = shfl_up_pair(w, off);
      if (lane >= off) w = combine(p, w);
    }
    wsp[lane] = w;
  }
  __syncthreads();
  if (warp > 0) acc = combine(wsp[warp - 1], acc);
  sp[threadIdx.x] = acc;
  __syncthreads();
  Pair ex{{1.0, 0.0}, {0.0, 0.0}};
  if (threadIdx.x > 0) ex = sp[threadIdx.x - 1];
  const cplx cin = carry_in ? carry_in[q] : cplx{0.0, 0.0};
  cplx c = cmad(ex.a, cin, ex.s);
  cplx* bc = sa.blkcarry + (int64_t)q * sa.nblk;
  if (sa.blka) {
    // also the exclusive A products, so that a later carry-in applies
    // without another top-level pass (chunk phase 2: c = A cin + carry)
    cplx* ba = sa.blka + (int64_t)q * sa.nblk;
    cplx ar = ex.a;
    for (int64_t r = r0; r < r1; ++r) {
      bc[r] = c;
      ba[r] = ar;
      c = cmad(ag[2 * r], c, ag[2 * r + 1]);
      ar = cmul(ag[2 * r], ar);
    }
  } else {
    for (int64_t r = r0; r < r1; ++r) {
      bc[r] = c;
      c = cmad(ag[2 * r], c, ag[2 * r + 1]);
    }
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

// ------------------------------------------- moment path: K1m and K2m
//
// Single plans carry the narrow segments' aggregates as their source
// moments about the segment centre, Mom_n = sum b (y - zc)^n, n < NMk (the
// plan's highest K1 moment degree + 1): 8 NMk bytes per segment instead of
// 48 ne (A, F, G per mode).  The per-mode pairs are formed from them inside
// the carry scan (K2m), whose down-sweep also folds every K3-narrow
// segment's carries into its collapsed carries E^c (the collapse kernel's
// job) so the per-mode carries of those segments never reach memory.

constexpr int kMomMax = FGT_K1_MAXDM + 1;
// Scan blocks of the moment path: kMomBlock consecutive segments per warp.
constexpr int kMomBlock = 64;
constexpr int kMomPerLane = kMomBlock / 32;
static_assert(kMomPerLane == 2, "moment-path scan block layout");

struct MomScanArgs {
  StreamArgs a;
  int ne;
  double* mom;  // [nseg][nm]
  int nm;       // K1 moments per segment (launch-uniform)
  int dn;       // collapsed degree of the narrow K3 (E^c rows)
  TileState ts;
  int64_t nblk;
  cplx* blkagg;    // [2ne][nblk] pairs (backward blocks stored right to left)
  cplx* blkcarry;  // [2ne][nblk]
  cplx* blka;      // [2ne][nblk] exclusive block A products (top level)
  // chunk phase 2: carries = blka * carry_in + blkcarry (no second top pass)
  const cplx* carry_in = nullptr;
  // K2m also folds the segment-total terms sum_m B[q][m] Tot_m of the
  // collapsed form into E^c (k3_folds: the moments reach degree dn)
  int fold = 0;
  CollConsts cc;
};

__device__ __forceinline__ bool mom_n1(const StreamArgs& a, int DM) {
  return a.nwide1 == 0 || k1_narrow(DM);
}
__device__ __forceinline__ bool mom_n3(const StreamArgs& a, int DM) {
  return a.nwide3 == 0 || k3_narrow(DM);
}

// Mode k of a segment from its moments about its centre (seg_aggregate_from's
// algebra): A = e^{-s (h0 + h1)}, F = forward state after the segment, G =
// backward state before it; E0 / E1 = e^{-s h0} / e^{-s h1} (degree NM-1
// Taylor polynomials, |s h| <= rmax[DM]).
template <int NM>
__device__ __forceinline__ void mom_pairs(const ModeTable& mt, int k, const double (&M)[NM],
                                          double h0, double h1, cplx& A, cplx& F, cplx& G,
                                          cplx& E0, cplx& E1) {
  const cplx* c = mt.coef[k];
  cplx e0 = c[NM - 1], e1 = c[NM - 1];
  cplx ev = {0.0, 0.0}, od = {0.0, 0.0};
#pragma unroll
  for (int n = NM - 1; n >= 0; --n) {
    const cplx cn = c[n];
    if (n < NM - 1) {
      e0 = {fma(e0.re, h0, cn.re), fma(e0.im, h0, cn.im)};
      e1 = {fma(e1.re, h1, cn.re), fma(e1.im, h1, cn.im)};
    }
    if (n & 1) {
      od.re = fma(cn.re, M[n], od.re);
      od.im = fma(cn.im, M[n], od.im);
    } else {
      ev.re = fma(cn.re, M[n], ev.re);
      ev.im = fma(cn.im, M[n], ev.im);
    }
  }
  E0 = e0;
  E1 = e1;
  A = cmul(e0, e1);
  F = cmul(e1, cplx{ev.re - od.re, ev.im - od.im});
  G = cmul(e0, cplx{ev.re + od.re, ev.im + od.im});
}

// Scan blocks of the moment path: kMomCta consecutive segments (K1agg's block
// aggregates, K2's top level, K2m's down-sweep CTAs).
constexpr int kMomCta = kSegWarps * kMomBlock;

// K1c: the segment source moments with CTA-level staging (k3c's scheme).
// Each CTA takes an equal contiguous range of chunks of kCW consecutive
// segments (compute warp w: segment s0 + w), whose sources and strengths are
// one contiguous range each: a producer warp stages a chunk (y, beta, segment
// starts and frames: four bulk copies) into one of two stages while the
// compute warps reduce the previous one to segment moments.  A warp's element
// loop runs only over its segment's sources (warp-uniform trip count), not
// over all kSeg merged slots.  The scan blocks' aggregates follow in K1agg.
constexpr int kK1cStageD = kChunk + 8;  // doubles per set and stage
struct K1cHdr {
  long long jb0;
  int yo, bo, io;
  int pad[3];
};
struct K1cStage {
  double* y;
  double* b;
  double2* sz;
  long long* ib;
  K1cHdr* hdr;
  uint64_t* bar;
};
constexpr size_t kK1cStageBytes =
    sizeof(double) * 2 * kK1cStageD + 16 * kCW + 8 * (kCW + 4) + sizeof(K1cHdr) + 16;
static_assert(kK1cStageBytes % 16 == 0, "k1c stage alignment");
static_assert(kMomCta % kCW == 0, "k1c: scan blocks are whole chunks");
__device__ __forceinline__ K1cStage k1c_stage(unsigned char* base) {
  K1cStage p;
  p.y = reinterpret_cast<double*>(base);
  p.b = p.y + kK1cStageD;
  p.sz = reinterpret_cast<double2*>(p.b + kK1cStageD);
  p.ib = reinterpret_cast<long long*>(p.sz + kCW);
  p.hdr = reinterpret_cast<K1cHdr*>(p.ib + kCW + 4);
  p.bar = reinterpret_cast<uint64_t*>(p.hdr + 1);
  return p;
}
template <int NM>
constexpr size_t k1c_smem_bytes() {
  return 2 * kK1cStageBytes + 64;
}

__device__ __forceinline__ void k1c_issue(const StreamArgs& a, int64_t c, int64_t ib0, int64_t ib1,
                                          const K1cStage& st) {
  auto blocks = [](const void* p, size_t nbytes, const void*& src) -> unsigned {
    const uintptr_t b0 = reinterpret_cast<uintptr_t>(p) & ~(uintptr_t)15;
    const uintptr_t b1 = (reinterpret_cast<uintptr_t>(p) + nbytes + 15) & ~(uintptr_t)15;
    src = reinterpret_cast<const void*>(b0);
    return nbytes > 0 ? (unsigned)(b1 - b0) : 0u;
  };
  const int64_t s0 = c * kCW;
  const int64_t s1 = s0 + kCW < a.nseg ? s0 + kCW : a.nseg;
  const int64_t L = a.M + a.N;
  const int64_t d0 = s0 * kSeg, d1 = s1 * kSeg < L ? s1 * kSeg : L;
  const int64_t jb0 = d0 - ib0, jb1 = d1 - ib1;
  const int ny = (int)(jb1 - jb0);
  const void *sy, *sb, *si;
  const unsigned by = blocks(a.ys + jb0, 8u * ny, sy);
  const unsigned bb = blocks(a.bs + jb0, 8u * ny, sb);
  const unsigned bi = blocks(a.seg_ib + s0, 8u * (unsigned)(s1 - s0 + 1), si);
  const unsigned ns = (unsigned)(s1 - s0);
  K1cHdr h;
  h.jb0 = jb0;
  h.yo = phase8(a.ys + jb0);
  h.bo = phase8(a.bs + jb0);
  h.io = (int)((reinterpret_cast<uintptr_t>(a.seg_ib + s0) >> 3) & 1);
  *st.hdr = h;
  fence_proxy_async();
  mbar_expect(st.bar, by + bb + bi + 16u * ns);
  if (by) bulk_g2s(st.y, sy, by, st.bar);
  if (bb) bulk_g2s(st.b, sb, bb, st.bar);
  bulk_g2s(st.ib, si, bi, st.bar);
  bulk_g2s(st.sz, a.seg_z + s0, 16u * ns, st.bar);
}


#ifndef FGT_K1C_MINB
#define FGT_K1C_MINB 3
#endif
template <int NM>
__global__ void __launch_bounds__(kCThreads + 32, FGT_K1C_MINB) k1c_kernel(MomScanArgs q,
                                                          const ModeTable* __restrict__ mtab) {
  (void)mtab;
  extern __shared__ __align__(16) unsigned char k1c_smem[];
  __shared__ __align__(16) double kred[kCW][32 * 4];
  const StreamArgs& a = q.a;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* const empty = reinterpret_cast<uint64_t*>(k1c_smem + 2 * kK1cStageBytes);
  if (threadIdx.x == 0) {
    mbar_init(k1c_stage(k1c_smem).bar);
    mbar_init(k1c_stage(k1c_smem + kK1cStageBytes).bar);
    mbar_init_n(empty, kCW);
    mbar_init_n(empty + 1, kCW);
  }
  __syncthreads();
  const int64_t nchunk = (a.nseg + kCW - 1) / kCW;
  // the CTA's chunks: an equal contiguous range (balanced to one chunk; the
  // block aggregates are formed afterwards by k1agg_kernel)
  const int64_t cbeg = nchunk * blockIdx.x / gridDim.x;
  const int64_t cend = nchunk * (blockIdx.x + 1) / gridDim.x;
  if (warp == kCW) {
    if (lane != 0) return;
    auto chunk_ib = [&](int64_t c, int64_t& i0, int64_t& i1) {
      const int64_t s0 = c * kCW;
      const int64_t s1 = s0 + kCW < a.nseg ? s0 + kCW : a.nseg;
      i0 = __ldg(a.seg_ib + s0);
      i1 = __ldg(a.seg_ib + s1);
    };
    for (int i = 0; i < 2; ++i) {
      const int64_t c = cbeg + i;
      if (c < cend) {
        int64_t i0, i1;
        chunk_ib(c, i0, i1);
        k1c_issue(a, c, i0, i1, k1c_stage(k1c_smem + i * kK1cStageBytes));
      }
    }
    int64_t nib0 = 0, nib1 = 0;
    if (cbeg + 2 < cend) chunk_ib(cbeg + 2, nib0, nib1);
    for (int64_t it = 0;; ++it) {
      const int64_t c2 = cbeg + it + 2;
      if (c2 >= cend) break;
      const int k = (int)(it & 1);
      mbar_wait(empty + k, (unsigned)(it >> 1) & 1u);
      k1c_issue(a, c2, nib0, nib1, k1c_stage(k1c_smem + k * kK1cStageBytes));
      if (c2 + 1 < cend) chunk_ib(c2 + 1, nib0, nib1);
    }
    return;
  }
  const int64_t L = a.M + a.N;
  int64_t it = 0;
  for (int64_t c = cbeg; c < cend; ++c, ++it) {
      const int k = (int)(it & 1);
      const K1cStage st = k1c_stage(k1c_smem + k * kK1cStageBytes);
      mbar_wait(st.bar, (unsigned)(it >> 1) & 1u);
      const int64_t s = c * kCW + warp;
      double M[NM];
#pragma unroll
      for (int n = 0; n < NM; ++n) M[n] = 0.0;
      const bool live = s < a.nseg;
      if (live) {
        const K1cHdr h = *st.hdr;
        const int64_t ib = st.ib[h.io + warp], ie = st.ib[h.io + warp + 1];
        const int64_t d0 = s * kSeg;
        const int len = (int)(d0 + kSeg < L ? kSeg : L - d0);
        const int ny = len - (int)(ie - ib);
        const int ly = (int)(d0 - ib - h.jb0);
        const double2 z = st.sz[warp];
        SegGeom g;
        g.zprev = s == 0 ? a.zprev0 : z.x;
        g.zlast = z.y;
        const SegFrame f = seg_frame(g);
        const double zc = f.zc;
        const double* yy = st.y + h.yo + ly;
        const double* bb = st.b + h.bo + ly;
        // two warp-uniform halves of kSeg / 64 source slots per lane (a
        // segment holds about kSeg / 2 sources); no branch inside a half
        auto half = [&](int u0) {
          double d[kSeg / 64], p[kSeg / 64];
#pragma unroll
          for (int u = 0; u < kSeg / 64; ++u) {
            const int j = lane + 32 * (u0 + u);
            const bool in = j < ny;
            d[u] = in ? yy[j] - zc : 0.0;
            p[u] = in ? bb[j] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < kSeg / 64; ++u) {
            double q = p[u];
            M[0] += q;
#pragma unroll
            for (int n = 1; n < NM; ++n) {
              q *= d[u];
              M[n] += q;
            }
          }
        };
        half(0);
        if (ny > kSeg / 2) half(kSeg / 64);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + k);  // stage consumed
      if constexpr (NM <= 4) {
        double* red = kred[warp];
#pragma unroll
        for (int n = 0; n < NM; ++n) red[n * 32 + lane] = M[n];
        __syncwarp();
        const int n = lane >> 3, g = lane & 7;
        double v = 0.0;
        if (n < NM) {
          const double2 a0 = *reinterpret_cast<const double2*>(red + n * 32 + 4 * g);
          const double2 a1 = *reinterpret_cast<const double2*>(red + n * 32 + 4 * g + 2);
          v = (a0.x + a0.y) + (a1.x + a1.y);
        }
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (live && n < NM && g == 0) {
          q.mom[s * NM + n] = v;
        }
        __syncwarp();
      } else {
#pragma unroll
        for (int n = 0; n < NM; ++n) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) M[n] += __shfl_xor_sync(0xffffffffu, M[n], o);
        }
        if (live && lane < NM) {
          double v = M[0];
#pragma unroll
          for (int n = 1; n < NM; ++n)
            if (lane == n) v = M[n];
          q.mom[s * NM + lane] = v;
        }
      }
  }
}

// Block aggregates of the moment path (K1c's second half): two warps per
// scan block of kMomCta segments, lane l of a warp holding kAggPer
// consecutive segments (their moments and frames loaded once, before the
// mode loop).  Per mode: each segment's (A, F) / (A, G) pairs from its
// moments, combined in order in registers (forward: earlier first;
// backward: later first), one ordered warp reduction, the two warps'
// results combined in order -- under half the FP64 work of a warp reduction
// over single segments.
constexpr int kAggPer = 4;                       // segments per lane
constexpr int kAggWarps = kMomCta / (32 * kAggPer);  // warps per scan block
static_assert(kAggWarps == 2 && kCW % kAggWarps == 0, "k1agg layout");
template <int NM>
__global__ void __launch_bounds__(kCThreads) k1agg_kernel(MomScanArgs q,
                                                         const ModeTable* __restrict__ mtab) {
  __shared__ ModeTable mt;
  __shared__ Pair wagg[kCW][2 * kMaxModes];
  load_mode_table(mtab, mt);
  const StreamArgs& a = q.a;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ne = q.ne;
  const bool all1 = a.nwide1 == 0;
  const int64_t b = (int64_t)blockIdx.x * (kCW / kAggWarps) + warp / kAggWarps;
  const int64_t s0 = b * kMomCta + (int64_t)(warp % kAggWarps) * 32 * kAggPer +
                     (int64_t)lane * kAggPer;
  double Mm[kAggPer][NM];
  double h0[kAggPer], h1[kAggPer];
  bool lv[kAggPer], n1[kAggPer];
#pragma unroll
  for (int i = 0; i < kAggPer; ++i) {
    const int64_t sg = s0 + i;
    lv[i] = b < q.nblk && sg < a.nseg;
    n1[i] = false;
    h0[i] = h1[i] = 0.0;
#pragma unroll
    for (int n = 0; n < NM; ++n) Mm[i][n] = 0.0;
    if (lv[i]) {
      n1[i] = all1 || k1_narrow(seg_deg_DM(__ldg(a.seg_deg + sg)));
      const double2 z = __ldg(a.seg_z + sg);
      SegGeom g;
      g.zprev = sg == 0 ? a.zprev0 : z.x;
      g.zlast = z.y;
      const SegFrame f = seg_frame(g);
      h0[i] = f.h0;
      h1[i] = f.h1;
      if (n1[i]) {
#pragma unroll
        for (int n = 0; n < NM; ++n) Mm[i][n] = __ldg(q.mom + sg * NM + n);
      }
    }
  }
  __syncthreads();  // the mode table
  for (int k = 0; k < ne; ++k) {
    Pair fw{{1.0, 0.0}, {0.0, 0.0}}, bw{{1.0, 0.0}, {0.0, 0.0}};
#pragma unroll
    for (int i = 0; i < kAggPer; ++i) {
      if (!lv[i]) continue;
      cplx A, F, G;
      if (n1[i]) {
        cplx E0, E1;
        mom_pairs<NM>(mt, k, Mm[i], h0[i], h1[i], A, F, G, E0, E1);
      } else {
        const int64_t o = (int64_t)k * a.nseg + s0 + i;
        A = q.ts.A[o];
        F = q.ts.F[o];
        G = q.ts.G[o];
      }
      fw = combine(fw, Pair{A, F});
      bw = combine(Pair{A, G}, bw);
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      Pair of, ob;
      of.a.re = __shfl_xor_sync(0xffffffffu, fw.a.re, off);
      of.a.im = __shfl_xor_sync(0xffffffffu, fw.a.im, off);
      of.s.re = __shfl_xor_sync(0xffffffffu, fw.s.re, off);
      of.s.im = __shfl_xor_sync(0xffffffffu, fw.s.im, off);
      ob.a.re = __shfl_xor_sync(0xffffffffu, bw.a.re, off);
      ob.a.im = __shfl_xor_sync(0xffffffffu, bw.a.im, off);
      ob.s.re = __shfl_xor_sync(0xffffffffu, bw.s.re, off);
      ob.s.im = __shfl_xor_sync(0xffffffffu, bw.s.im, off);
      const bool lower = (lane & off) == 0;
      fw = lower ? combine(fw, of) : combine(of, fw);
      bw = lower ? combine(ob, bw) : combine(bw, ob);
    }
    if (lane == 0) {
      wagg[warp][k] = fw;
      wagg[warp][ne + k] = bw;
    }
  }
  __syncthreads();
  // the scan blocks of this CTA: thread t < (kCW / kAggWarps) 2 ne
  const int per = 2 * ne;
  if ((int)threadIdx.x < (kCW / kAggWarps) * per) {
    const int bl = threadIdx.x / per, q2 = threadIdx.x % per;
    const int64_t bb = (int64_t)blockIdx.x * (kCW / kAggWarps) + bl;
    if (bb < q.nblk) {
      const bool bwd = q2 >= ne;
      const Pair p0 = wagg[bl * kAggWarps][q2], p1 = wagg[bl * kAggWarps + 1][q2];
      const Pair acc = bwd ? combine(p1, p0) : combine(p0, p1);
      cplx* out = q.blkagg + ((int64_t)q2 * q.nblk + (bwd ? q.nblk - 1 - bb : bb)) * 2;
      out[0] = acc.a;
      out[1] = acc.s;
    }
  }
}

// K2m down-sweep, one CTA per scan block (kMomBlock segments per warp, two
// per lane: s0 + 2l, s0 + 2l + 1).  Per mode: exclusive warp scans of the
// lane pairs (forward by shfl_up, backward by shfl_down), the warps' totals
// combined through shared memory into each warp's carry-in, seeded with the
// block carries of the top level.  K3-narrow segments fold their carries
// into the collapsed carries E^c, K3-wide ones store them.
template <int NM>
__global__ void __launch_bounds__(kThreads) k2m_down_kernel(MomScanArgs q,
                                                            const ModeTable* __restrict__ mtab) {
  __shared__ ModeTable mt;
  __shared__ Pair wtot[kMaxModes][2][kSegWarps];
  load_mode_table(mtab, mt);
  __syncthreads();
  const StreamArgs& a = q.a;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t b = blockIdx.x;
  const int ne = q.ne;
  bool live[2], n1[2], n3[2];
  double h0[2], h1[2];
  double M[2][NM];
  int64_t sg[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    sg[i] = b * kMomCta + (int64_t)warp * kMomBlock + 2 * lane + i;
    live[i] = sg[i] < a.nseg;
    n1[i] = n3[i] = false;
    h0[i] = h1[i] = 0.0;
#pragma unroll
    for (int n = 0; n < NM; ++n) M[i][n] = 0.0;
    if (live[i]) {
      const int DM = a.nwide1 == 0 && a.nwide3 == 0 ? 0 : seg_deg_DM(__ldg(a.seg_deg + sg[i]));
      n1[i] = mom_n1(a, DM);
      n3[i] = mom_n3(a, DM);
      const double2 z = __ldg(a.seg_z + sg[i]);
      SegGeom g;
      g.zprev = sg[i] == 0 ? a.zprev0 : z.x;
      g.zlast = z.y;
      const SegFrame f = seg_frame(g);
      h0[i] = f.h0;
      h1[i] = f.h1;
      if (n1[i]) {
        const double* m = q.mom + sg[i] * NM;
#pragma unroll
        for (int n = 0; n < NM; ++n) M[i][n] = __ldg(m + n);
      }
    }
  }
  double E[2][kCollMax + 1];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int n = 0; n <= kCollMax; ++n) E[i][n] = 0.0;
  const Pair id{{1.0, 0.0}, {0.0, 0.0}};
  for (int k = 0; k < ne; ++k) {
    cplx A[2], F[2], G[2], E0[2], E1[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      if (!live[i]) {
        A[i] = {1.0, 0.0};
        F[i] = G[i] = E0[i] = E1[i] = {0.0, 0.0};
      } else if (n1[i]) {
        mom_pairs<NM>(mt, k, M[i], h0[i], h1[i], A[i], F[i], G[i], E0[i], E1[i]);
      } else {
        const int64_t o = (int64_t)k * a.nseg + sg[i];
        A[i] = q.ts.A[o];
        F[i] = q.ts.F[o];
        G[i] = q.ts.G[o];
        E0[i] = E1[i] = {0.0, 0.0};
      }
    }
    // forward: lane aggregate (item 0 then 1), inclusive scan over lanes
    Pair fincl = combine(Pair{A[0], F[0]}, Pair{A[1], F[1]});
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const Pair p = shfl_up_pair(fincl, off);
      if (lane >= off) fincl = combine(p, fincl);
    }
    Pair fex = shfl_up_pair(fincl, 1);
    if (lane == 0) fex = id;
    // backward: lane aggregate in reverse order (item 1 then 0), inclusive
    // scan from the right
    Pair bincl = combine(Pair{A[1], G[1]}, Pair{A[0], G[0]});
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      Pair p;
      p.a.re = __shfl_down_sync(0xffffffffu, bincl.a.re, off);
      p.a.im = __shfl_down_sync(0xffffffffu, bincl.a.im, off);
      p.s.re = __shfl_down_sync(0xffffffffu, bincl.s.re, off);
      p.s.im = __shfl_down_sync(0xffffffffu, bincl.s.im, off);
      if (lane + off < 32) bincl = combine(p, bincl);
    }
    Pair bex;
    bex.a.re = __shfl_down_sync(0xffffffffu, bincl.a.re, 1);
    bex.a.im = __shfl_down_sync(0xffffffffu, bincl.a.im, 1);
    bex.s.re = __shfl_down_sync(0xffffffffu, bincl.s.re, 1);
    bex.s.im = __shfl_down_sync(0xffffffffu, bincl.s.im, 1);
    if (lane == 31) bex = id;
    if (lane == 31) wtot[k][0][warp] = fincl;
    if (lane == 0) wtot[k][1][warp] = bincl;
    __syncthreads();
    // this warp's carries in: the block's carry through the earlier warps
    // (forward) / the later warps (backward)
    const int64_t of = (int64_t)k * q.nblk + b, ob = (int64_t)(ne + k) * q.nblk + (q.nblk - 1 - b);
    cplx cinf = q.blkcarry[of];
    cplx cinb = q.blkcarry[ob];
    if (q.carry_in) {
      cinf = cmad(q.blka[of], q.carry_in[k], cinf);
      cinb = cmad(q.blka[ob], q.carry_in[ne + k], cinb);
    }
    for (int w = 0; w < warp; ++w) {
      const Pair t = wtot[k][0][w];
      cinf = cmad(t.a, cinf, t.s);
    }
    for (int w = kSegWarps - 1; w > warp; --w) {
      const Pair t = wtot[k][1][w];
      cinb = cmad(t.a, cinb, t.s);
    }
    cplx cf[2], cb[2];
    cf[0] = cmad(fex.a, cinf, fex.s);  // forward state before item 0
    cf[1] = cmad(A[0], cf[0], F[0]);   // ... before item 1
    cb[1] = cmad(bex.a, cinb, bex.s);  // backward state at item 1's last element
    cb[0] = cmad(A[1], cb[1], G[1]);   // ... at item 0's last element
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      if (!live[i]) continue;
      if (n3[i]) {
        // collapsed carries: Re sum_k mw_k c_kq (e^{-s h0} Cf + (-1)^q e^{-s h1} Cb)
        const cplx tf = cmul(E0[i], cf[i]), tb = cmul(E1[i], cb[i]);
#pragma unroll
        for (int n = 0; n <= kCollMax; ++n) {
          if (n <= q.dn) {
            const cplx x = mt.mwc[k][n];
            const double sgn = (n & 1) ? -1.0 : 1.0;
            E[i][n] = fma(x.re, fma(sgn, tb.re, tf.re), fma(-x.im, fma(sgn, tb.im, tf.im), E[i][n]));
          }
        }
      } else {
        const int64_t o = (int64_t)k * a.nseg + sg[i];
        q.ts.Cf[o] = cf[i];
        q.ts.Cb[o] = cb[i];
      }
    }
  }
  if (q.fold) {
    // E_q += sum_m B[q][m] Tot_m (Tot = the segment's source moments)
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int n = 0; n <= kCollMax; ++n)
#pragma unroll
        for (int m = 0; m < NM; ++m)
          if (n + m <= kCollMax && n + m <= q.dn) E[i][n] = fma(q.cc.B[n][m], M[i][m], E[i][n]);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    if (live[i] && n3[i]) {
      double* out = q.ts.ec + sg[i] * kEcStride;
#pragma unroll
      for (int n = 0; n <= kCollMax; ++n) out[n] = n <= q.dn ? E[i][n] : 0.0;
#pragma unroll
      for (int n = kCollMax + 1; n < kEcStride; ++n) out[n] = 0.0;
    }
  }
}

// out[i] = alpha[perm[i]]: random reads; kGatherILP independent gathers per
// thread in flight (coalesced index loads first, then the data loads).
constexpr int kGatherILP = 8;
__global__ void gather_kernel(const double* __restrict__ alpha, const int32_t* __restrict__ perm,
                              int64_t n, double* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n;
       i0 += stride * kGatherILP) {
    int32_t p[kGatherILP];
#pragma unroll
    for (int u = 0; u < kGatherILP; ++u) {
      const int64_t i = i0 + u * stride;
      p[u] = i < n ? __ldg(perm + i) : 0;
    }
    double v[kGatherILP];
#pragma unroll
    for (int u = 0; u < kGatherILP; ++u) v[u] = __ldg(alpha + p[u]);
#pragma unroll
    for (int u = 0; u < kGatherILP; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < n) out[i] = v[u];
    }
  }
}

}  // namespace

// ============================================================== host side

static int num_sms() {
  static int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
      return v;
    cudaGetLastError();
    return 148;
  }();
  return n;
}

int64_t scan_blocks(int64_t nseg) { return (nseg + kScanBlock - 1) / kScanBlock; }

// the moment path's smaller scan blocks set the workspace size
static int64_t ws_blocks(int64_t nseg) { return (nseg + 255) / 256; }
size_t tile_state_elems(int64_t nseg, int ne) {
  const size_t nt = (size_t)nseg * (size_t)ne;
  const size_t blk = (size_t)ws_blocks(nseg) * 2 * (size_t)ne * 4 + 8;
  return 5 * nt + blk + (size_t)nseg * (kEcStride / 2) + 4;
}

TileState tile_state_carve(cplx* base, int64_t nseg, int ne) {
  const size_t nt = (size_t)nseg * (size_t)ne;
  const size_t blk = (size_t)ws_blocks(nseg) * 2 * (size_t)ne * 4 + 8;
  // collapsed carries: 64-byte aligned rows (one bulk copy per segment)
  uintptr_t ecp = reinterpret_cast<uintptr_t>(base + 5 * nt + blk);
  ecp = (ecp + 63) & ~(uintptr_t)63;
  return TileState{base,           base + nt,      base + 2 * nt,
                   base + 3 * nt,  base + 4 * nt,  base + 5 * nt,
                   reinterpret_cast<double*>(ecp)};
}

CollConsts coll_consts(const double* g) {
  CollConsts c{};
  auto binom = [](int n, int m) {
    double r = 1.0;
    for (int i = 1; i <= m; ++i) r = r * (n - m + i) / i;
    return r;
  };
  for (int m = 0; m <= kCollMax; ++m)
    for (int q = 0; q <= kCollMax; ++q) {
      const int n = m + q;
      if (n > kCollMax) continue;
      if (n & 1) c.H[m][q] = ((m & 1) ? -2.0 : 2.0) * binom(n, m) * g[n];
      c.B[q][m] = ((q & 1) ? -1.0 : 1.0) * binom(n, m) * g[n];
    }
  return c;
}

size_t seg_smem_bytes(int ne, bool batched, bool stream, int region) {
  return (region == 3 ? kLaneTableBytes : sizeof(ModeTable)) * (batched ? kSegWarps : 1) +
         (size_t)kSegWarps * (warp_region_bytes(ne, region) + (stream ? kStageBytes : 0));
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

cudaError_t launch_plan_tiles(const double* xs, int64_t M, const double* ys, int64_t N,
                              const int64_t* tile_ib, int64_t ntiles, int64_t nseg,
                              int check_sorted, int64_t* seg_ib, double2* seg_z,
                              uint32_t* seg_mask, int* flags, cudaStream_t st,
                              const PlanClassify* cls) {
  if (ntiles == 0) return cudaSuccess;
  PlanClassify cl;
  if (cls && cls->enabled) {
    cl = *cls;
    cudaError_t e0 = cudaMemsetAsync(cl.counts, 0, sizeof(unsigned long long) * 4 * kClassSlots, st);
    if (e0 != cudaSuccess) return e0;
  }
  // both sets, heads, sentinels + padding for merge overruns on unsorted input
  const size_t smem = sizeof(double) * (kPlanTile + 8 + 2 * kPlanPer);
  static std::atomic<unsigned long long> done{0};
  cudaError_t e = ensure_dynamic_smem(plan_tile_kernel, (int)smem, done);
  if (e != cudaSuccess) return e;
  note_launch();
  plan_tile_kernel<<<(unsigned)ntiles, kPlanThreads, smem, st>>>(xs, M, ys, N, tile_ib, nseg, check_sorted,
                                                         seg_ib, seg_z, seg_mask, flags, cl);
  return cudaGetLastError();
}

cudaError_t launch_check_points(const double* xs, int64_t M, const double* ys, int64_t N,
                                int* flags, cudaStream_t st) {
  const int64_t L = M > N ? M : N;
  if (L == 0) return cudaSuccess;
  int64_t blocks = (L + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  note_launch();
  check_points_kernel<<<(unsigned)blocks, 256, 0, st>>>(xs, M, ys, N, flags);
  return cudaGetLastError();
}

cudaError_t launch_batch_plan(const double* xs, const double* ys, const int64_t* t_off,
                              const int64_t* s_off, const int64_t* seg_base,
                              const int64_t* tile_base, const int32_t* tile_tid, int B,
                              int64_t ntiles, int64_t* tile_ib, int64_t* seg_ib, int64_t* seg_jb,
                              int4* seg_info, double2* seg_z, uint32_t* seg_mask,
                              int* flags, cudaStream_t st) {
  (void)B;
  if (ntiles == 0) return cudaSuccess;
  const BatchArgs b{xs, ys, t_off, s_off, seg_base, tile_base, tile_tid};
  note_launch(2);
  batch_partition_kernel<<<(unsigned)((ntiles + 255) / 256), 256, 0, st>>>(b, ntiles, tile_ib);
  // both sets, heads, sentinels + padding for merge overruns on unsorted input
  const size_t smem = sizeof(double) * (kPlanTile + 8 + 2 * kPlanPer);
  static std::atomic<unsigned long long> done{0};
  cudaError_t e = ensure_dynamic_smem(batch_plan_tile_kernel, (int)smem, done);
  if (e != cudaSuccess) return e;
  batch_plan_tile_kernel<<<(unsigned)ntiles, kPlanThreads, smem, st>>>(b, tile_ib, seg_ib, seg_jb, seg_info,
                                                              seg_z, seg_mask, flags);
  return cudaGetLastError();
}

template <class K>
static cudaError_t set_smem(K kernel, std::atomic<unsigned long long>& done, int region) {
  return ensure_dynamic_smem(kernel, (int)seg_smem_bytes(kMaxModes, true, true, region), done);
}

cudaError_t launch_aggregate(const StreamArgs& a, const ModeParams& P, const ModeTable* mt,
                             TileState ts, cudaStream_t st) {
  if (a.nseg == 0) return cudaSuccess;
  const int64_t per_cta = (int64_t)kSegWarps * (a.mtb ? kBatchGroup : 1);
  int64_t want = (a.nseg + per_cta - 1) / per_cta;
  const int64_t cap = (int64_t)num_sms() * (a.mtb ? FGT_K1_GRID_BATCH : FGT_K1_GRID);
  const unsigned grid = (unsigned)(want < cap ? want : cap);
  const size_t smem = sizeof(ModeTable) * (a.mtb ? kSegWarps : 1);
  if (a.nwide1 != 0) {
    note_launch();
    seg_aggregate_kernel<true><<<grid, kThreads, smem + kK1SlotBytes * kSegWarps, st>>>(a, P, mt,
                                                                                        ts);
  }
  if (a.nwide1 != a.nseg) {
    note_launch();
    seg_aggregate_kernel<false><<<grid, kThreads, smem, st>>>(a, P, mt, ts);
  }
  return cudaGetLastError();
}

cudaError_t launch_store_table(const ModeTable& T, ModeTable* out, cudaStream_t st) {
  note_launch();
  store_table_kernel<<<1, 128, 0, st>>>(T, out);
  return cudaGetLastError();
}

cudaError_t launch_batch_modes(const BatchModeBase& base, const double* deltas, int B,
                               ModeTable* out, cudaStream_t st) {
  if (B <= 0) return cudaSuccess;
  note_launch();
  batch_modes_kernel<<<(B + 127) / 128, 128, 0, st>>>(base, deltas, B, out);
  return cudaGetLastError();
}

cudaError_t launch_classify(const StreamArgs& a, const ModeParams& P, double smax,
                            int* seg_deg, const int* skip_flags,
                            unsigned long long* counts, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(counts, 0, 4 * sizeof(unsigned long long), st);
  if (e != cudaSuccess || a.nseg == 0) return e;
  const int64_t want = (a.nseg + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 8;
  note_launch();
  classify_kernel<<<(unsigned)(want < cap ? want : cap), 256, 0, st>>>(a, P, smax, seg_deg,
                                                                       skip_flags, counts);
  return cudaGetLastError();
}

template <bool MS, bool WIDE, bool LANE = false>
static cudaError_t launch_seg_main_variant(const StreamArgs& a, const ModeParams& P,
                                           const ModeTable* mt, TileState ts, OutArgs o,
                                           cudaStream_t st) {
  if constexpr (WIDE && !MS && !LANE && FGT_LANE_COLL && k3_stream<true>()) {
    // lane-collapsed kernel first; what it flags goes to the per-mode kernel
    if (!a.fallback_only) {
      cudaError_t e = launch_seg_main_variant<MS, WIDE, true>(a, P, mt, ts, o, st);
      if (e != cudaSuccess) return e;
      StreamArgs fb = a;
      fb.fallback_only = 1;
      return launch_seg_main_variant<MS, WIDE, false>(fb, P, mt, ts, o, st);
    }
  }
  constexpr int region = LANE ? 3 : ((MS && !WIDE) ? 1 : 0);
  static std::atomic<unsigned long long> done{0};
  cudaError_t e = set_smem(seg_main_kernel<MS, WIDE, LANE>, done, region);
  if (e != cudaSuccess) return e;
  const size_t smem = seg_smem_bytes(P.ne, a.mtb != nullptr, k3_stream<WIDE>(), region);
  int64_t want, cap;
  if constexpr (!k3_stream<WIDE>()) {
    const int64_t per_cta = (int64_t)kSegWarps * (a.mtb ? kBatchGroup : 1);
    want = (a.nseg + per_cta - 1) / per_cta;
    cap = (int64_t)num_sms() * FGT_K3_GRID;
  } else {
    // streaming: one resident wave, contiguous segment ranges per warp
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, seg_main_kernel<MS, WIDE, LANE>,
                                                      kThreads, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    want = (a.nseg + kSegWarps - 1) / kSegWarps;
    cap = (int64_t)num_sms() * per_sm *
          (WIDE ? (a.mtb ? FGT_K3W_WAVES_BATCH : FGT_K3W_WAVES) : FGT_K3N_WAVES);
  }
  const unsigned grid = (unsigned)(want < cap ? want : cap);
  note_launch();
  seg_main_kernel<MS, WIDE, LANE><<<grid, kThreads, smem, st>>>(a, P, mt, ts, o);
  return cudaGetLastError();
}

template <bool MS>
static cudaError_t launch_seg_main(const StreamArgs& a, const ModeParams& P, const ModeTable* mt,
                                   TileState ts, OutArgs o, cudaStream_t st) {
  if (a.nseg == 0) return cudaSuccess;
  if (a.nwide3 != 0) {
    cudaError_t e = launch_seg_main_variant<MS, true>(a, P, mt, ts, o, st);
    if (e != cudaSuccess) return e;
  }
  if (a.nwide3 != a.nseg) return launch_seg_main_variant<MS, false>(a, P, mt, ts, o, st);
  return cudaSuccess;
}

// Chunk g's forward carry is the forward state at its z_prev from all chunks
// to its left, C+_g = A_{g-1} C+_{g-1} + F_{g-1}; the backward carry is the
// mirror image, C-_g = A_{g+1} C-_{g+1} + G_{g+1} (fgt_chunk_carries).
__global__ void chunk_carries_kernel(const cplx* __restrict__ a, int G, int ne, int rank,
                                     cplx* __restrict__ out) {
  const int k = threadIdx.x;
  if (k >= ne) return;
  cplx f = {0.0, 0.0};
  for (int g = 0; g < rank; ++g) {
    const cplx A = a[g * 3 * ne + k], F = a[g * 3 * ne + ne + k];
    f = cplx{A.re * f.re - A.im * f.im + F.re, A.re * f.im + A.im * f.re + F.im};
  }
  cplx b = {0.0, 0.0};
  for (int g = G - 1; g > rank; --g) {
    const cplx A = a[g * 3 * ne + k], Gg = a[g * 3 * ne + 2 * ne + k];
    b = cplx{A.re * b.re - A.im * b.im + Gg.re, A.re * b.im + A.im * b.re + Gg.im};
  }
  out[k] = f;
  out[ne + k] = b;
}

cudaError_t launch_chunk_carries(const cplx* aggs, int n_chunks, int ne, int rank, cplx* out,
                                 cudaStream_t st) {
  note_launch();
  chunk_carries_kernel<<<1, 32, 0, st>>>(aggs, n_chunks, ne, rank, out);
  return cudaGetLastError();
}

template <int DN, bool FOLD>
static cudaError_t launch_k3c_dnf(const StreamArgs& a, const TileState& ts, const CollConsts& cc,
                                  OutArgs o, cudaStream_t st) {
  static std::atomic<unsigned long long> done{0};
  const size_t smem = k3c_smem_bytes<DN + 1>();
  cudaError_t e = ensure_dynamic_smem(k3c_kernel<DN, FOLD>, (int)smem, done);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k3c_kernel<DN, FOLD>, kCThreads + 32,
                                                    smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t want = (a.nseg + kCW - 1) / kCW;
  const int64_t cap = (int64_t)num_sms() * per_sm;
  note_launch();
  k3c_kernel<DN, FOLD><<<(unsigned)(want < cap ? want : cap), kCThreads + 32, smem, st>>>(a, ts.ec,
                                                                                         cc, o);
  return cudaGetLastError();
}
template <int DN>
static cudaError_t launch_k3c_dn(const StreamArgs& a, const TileState& ts, const CollConsts& cc,
                                 OutArgs o, cudaStream_t st, bool folded) {
  return folded ? launch_k3c_dnf<DN, true>(a, ts, cc, o, st)
                : launch_k3c_dnf<DN, false>(a, ts, cc, o, st);
}

template <int DN>
static cudaError_t launch_k3n_dn(const StreamArgs& a, const TileState& ts, const CollConsts& cc,
                                 OutArgs o, cudaStream_t st, bool folded) {
  return launch_k3c_dn<DN>(a, ts, cc, o, st, folded);
}

int k3n_degree(const StreamArgs& a) {
  return a.dn_narrow >= 0 ? (a.dn_narrow < kCollMax ? a.dn_narrow : kCollMax) : kCollMax;
}

bool k3_folds(const StreamArgs& a) { return k3n_degree(a) + 1 <= k1m_moments(a); }

cudaError_t launch_main(const StreamArgs& a, const ModeParams& P, const ModeTable* mt,
                        TileState ts, OutArgs o, cudaStream_t st, const CollConsts* cc,
                        bool ec_ready, bool folded) {
  if (!cc || a.mtb || a.nseg == 0) return launch_seg_main<false>(a, P, mt, ts, o, st);
  // single plan: wide segments on the per-segment kernel, narrow ones on the
  // collapsed kernel at the plan's highest narrow degree
  if (a.nwide3 != 0) {
    cudaError_t e = launch_seg_main_variant<false, true>(a, P, mt, ts, o, st);
    if (e != cudaSuccess) return e;
  }
  if (a.nwide3 == a.nseg) return cudaSuccess;
  const int DN = k3n_degree(a);
  if (!ec_ready) {
    note_launch();
    collapse_carries_kernel<<<(unsigned)((a.nseg + 255) / 256), 256, 0, st>>>(a, mt, P.ne, ts, DN);
  }
  switch (DN) {
    case 0: return launch_k3n_dn<0>(a, ts, *cc, o, st, folded);
    case 1: return launch_k3n_dn<1>(a, ts, *cc, o, st, folded);
    case 2: return launch_k3n_dn<2>(a, ts, *cc, o, st, folded);
    case 3: return launch_k3n_dn<3>(a, ts, *cc, o, st, folded);
    case 4: return launch_k3n_dn<4>(a, ts, *cc, o, st, folded);
    case 5: return launch_k3n_dn<5>(a, ts, *cc, o, st, folded);
    default: return launch_k3n_dn<6>(a, ts, *cc, o, st, folded);
  }
}

cudaError_t launch_mode_sums(const StreamArgs& a, const ModeParams& P, const ModeTable* mt,
                             TileState ts, OutArgs o, cudaStream_t st) {
  return launch_seg_main<true>(a, P, mt, ts, o, st);
}

cudaError_t launch_carry_scan(const TileState& ts, int64_t nseg, int ne, const cplx* carry_in,
                              cplx* totals, cudaStream_t st, bool reduce, bool down) {
  if (nseg == 0) return cudaSuccess;
  const int64_t nblk = scan_blocks(nseg);
  ScanArgs sa{ts.A, ts.F, ts.G, ts.Cf, ts.Cb, nseg, ne, nblk, ts.blk,
              ts.blk + (size_t)nblk * 2 * ne * 2};
  const dim3 grid((unsigned)nblk, (unsigned)(2 * ne));
  note_launch(1 + (reduce ? 1 : 0) + (down ? 1 : 0));
  if (reduce) scan_reduce_kernel<<<grid, kScanThreads, 0, st>>>(sa);
  scan_top_kernel<<<2 * ne, 1024, 0, st>>>(sa, carry_in, totals);
  if (down) scan_down_kernel<<<grid, kScanThreads, 0, st>>>(sa);
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

// ---- moment path launchers

int k1m_moments(const StreamArgs& a) {
  return a.dm_narrow >= 0 ? a.dm_narrow + 1 : kMomMax;
}

int64_t mom_scan_blocks(int64_t nseg) { return (nseg + kMomCta - 1) / kMomCta; }

cudaError_t launch_moments(const StreamArgs& a, const ModeParams& P, const ModeTable* mt,
                           TileState ts, double* mom, cudaStream_t st) {
  (void)mom;
  if (a.nseg == 0 || a.nwide1 == 0) return cudaSuccess;
  // K1-wide segments keep their per-mode (A, F, G) (wide K1); the narrow
  // ones' moments are formed by K1c inside launch_mom_scan
  const int64_t want = (a.nseg + kSegWarps - 1) / kSegWarps;
  const int64_t cap = (int64_t)num_sms() * FGT_K1_GRID;
  note_launch();
  seg_aggregate_kernel<true><<<(unsigned)(want < cap ? want : cap), kThreads,
                               sizeof(ModeTable) + kK1SlotBytes * kSegWarps, st>>>(a, P, mt, ts);
  return cudaGetLastError();
}

template <int NM>
static cudaError_t launch_mom_nm(const MomScanArgs& q, const ModeTable* mt, bool reduce, bool down,
                                 const ScanArgs& sa, const cplx* carry_in, cplx* totals,
                                 cudaStream_t st) {
  const unsigned grid = (unsigned)q.nblk;
  const bool top = reduce || !down || !carry_in;
  note_launch((top ? 1 : 0) + (reduce ? 2 : 0) + (down ? 1 : 0));
  if (reduce) {
    const size_t smem = k1c_smem_bytes<NM>();
    static std::atomic<unsigned long long> done{0};
    cudaError_t e = ensure_dynamic_smem(k1c_kernel<NM>, (int)smem, done);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k1c_kernel<NM>, kCThreads + 32, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    const int64_t nchunk = (q.a.nseg + kCW - 1) / kCW;
    const int64_t cap = (int64_t)num_sms() * per_sm;
    k1c_kernel<NM><<<(unsigned)(nchunk < cap ? nchunk : cap), kCThreads + 32, smem, st>>>(q, mt);
    k1agg_kernel<NM><<<(unsigned)((q.nblk + kCW / kAggWarps - 1) / (kCW / kAggWarps)), kCThreads, 0,
                       st>>>(q, mt);
  }
  if (top) scan_top_kernel<<<2 * q.ne, 1024, 0, st>>>(sa, carry_in, totals);
  if (down) k2m_down_kernel<NM><<<grid, kThreads, 0, st>>>(q, mt);
  return cudaGetLastError();
}

cudaError_t launch_mom_scan(const StreamArgs& a, int ne, const ModeTable* mt, const TileState& ts,
                            double* mom, const cplx* carry_in, cplx* totals, cudaStream_t st,
                            bool reduce, bool down, const CollConsts* cc) {
  if (a.nseg == 0) return cudaSuccess;
  const int64_t nblk = mom_scan_blocks(a.nseg);
  MomScanArgs q;
  q.a = a;
  q.ne = ne;
  q.mom = mom;
  q.nm = k1m_moments(a);
  q.dn = k3n_degree(a);
  q.ts = ts;
  q.nblk = nblk;
  q.blkagg = ts.blk;
  q.blkcarry = ts.blk + (size_t)nblk * 2 * ne * 2;
  q.blka = ts.blk + (size_t)nblk * 2 * ne * 3;
  if (cc && k3_folds(a)) {
    q.fold = 1;
    q.cc = *cc;
  }
  ScanArgs sa{ts.A, ts.F, ts.G, ts.Cf, ts.Cb, a.nseg, ne, nblk, q.blkagg, q.blkcarry};
  sa.blka = q.blka;
  if (!reduce && down) {
    // chunk phase 2: phase 1's top level left the block carries without a
    // carry-in and the exclusive A products; K2m applies carry_in itself
    q.carry_in = carry_in;
  }
  switch (q.nm) {
#define FGT_MNM(n)                                                 \
  case n:                                                          \
    return launch_mom_nm<n>(q, mt, reduce, down, sa, carry_in, totals, st);
    FGT_MNM(1) FGT_MNM(2) FGT_MNM(3) FGT_MNM(4) FGT_MNM(5) FGT_MNM(6) FGT_MNM(7) FGT_MNM(8)
    FGT_MNM(9) FGT_MNM(10) FGT_MNM(11) FGT_MNM(12) FGT_MNM(13)
#undef FGT_MNM
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace fgt_b200
