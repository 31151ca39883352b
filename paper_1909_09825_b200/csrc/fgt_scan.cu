// Merged-stream SOE scan kernels (sm_100a).  Hot path of the fast Gauss
// transform: replaces run_mode_general / apply_common of the reference
// (proj/src/transform.cpp:119-149, 151-196).
//
//   K0 partition : merge-path split of the (targets, sources) stream into tiles
//   K1 aggregate : per tile, per mode, the scan aggregate (A, F, G)
//   K2 carry scan: exclusive scan of tile aggregates in both directions
//   K3 main      : per tile, lane carries -> forward/backward recurrences ->
//                  fused weighted real-part combine and scatter of u
//
// Within a tile (CTA, kTile merged elements) each lane owns a run of kR
// consecutive merged elements held in registers as (gap, weight) pairs.
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

template <int D>
__device__ __forceinline__ cplx horner(const cplx (&c)[kMaxDeg + 1], double g) {
  double pr = c[D].re, pi = c[D].im;
#pragma unroll
  for (int n = D - 1; n >= 0; --n) {
    pr = fma(pr, g, c[n].re);
    pi = fma(pi, g, c[n].im);
  }
  return {pr, pi};
}

// Gap factor for mode coefficients c (fast path, degree D) or exact (D < 0).
template <int D>
__device__ __forceinline__ cplx gap_factor(const cplx (&c)[kMaxDeg + 1], cplx s, double g) {
  if constexpr (D >= 0) {
    return horner<D>(c, g);
  } else {
    return decay_exact(s.re, s.im, g);
  }
}

template <int D>
__device__ __forceinline__ void load_coef(const ModeTable& mt, int k, cplx (&c)[kMaxDeg + 1]) {
  if constexpr (D >= 0) {
#pragma unroll
    for (int n = 0; n <= D; ++n) c[n] = mt.coef[k][n];
  }
}

// Pass 1: lane-run aggregates for every mode, carries in = 0.
//   A = prod d_i, F = forward state at the run end, G = backward state at the
//   element before the run.
template <int D>
__device__ __forceinline__ void pass1(const ModeTable& mt, int ne, const double (&g)[kR],
                                   const double (&b)[kR], LaneAgg* out) {
  for (int k = 0; k < ne; ++k) {
    cplx c[kMaxDeg + 1];
    load_coef<D>(mt, k, c);
    const cplx s = mt.s[k];
    cplx F = {0.0, 0.0}, P = {1.0, 0.0}, G = {0.0, 0.0};
#pragma unroll
    for (int i = 0; i < kR; ++i) {
      cplx d = gap_factor<D>(c, s, g[i]);
      F = cmad(d, F, cplx{b[i], 0.0});
      P = cmul(P, d);
      G.re = fma(b[i], P.re, G.re);
      G.im = fma(b[i], P.im, G.im);
    }
    out[k] = LaneAgg{P, F, G};
  }
}

// Pass 2: forward and backward recurrences seeded with the lane carries,
// accumulating Re(mw_k (H + K)) into out[] (only target slots are used).
// MS (mode-sums test hook, detail::mode_sums transform.cpp:310-350): instead
// store H (= h+) and K (= h-) of every target, per mode, to ms.
struct ModeSumsOut {
  cplx* hp;  // [ne][M]
  cplx* hm;
  int64_t M;
  int64_t t0;  // global sorted index of this lane's first target
};

template <int D, bool MS>
__device__ __forceinline__ void pass2(const ModeTable& mt, int ne, const double (&g)[kR],
                                      const double (&b)[kR], unsigned tmask, const LaneAgg* carry,
                                      double (&out)[kR], const ModeSumsOut& ms) {
  for (int k = 0; k < ne; ++k) {
    cplx c[kMaxDeg + 1];
    load_coef<D>(mt, k, c);
    const cplx s = mt.s[k];
    const cplx mw = mt.mw[k];
    cplx d[kR];
    cplx H = carry[k].F;  // forward state at the element before the run
    int64_t ti = ms.t0;
#pragma unroll
    for (int i = 0; i < kR; ++i) {
      d[i] = gap_factor<D>(c, s, g[i]);
      H = cmad(d[i], H, cplx{b[i], 0.0});
      if constexpr (MS) {
        if (tmask & (1u << i)) ms.hp[(int64_t)k * ms.M + ti++] = H;
      } else {
        out[i] = fma(mw.re, H.re, fma(-mw.im, H.im, out[i]));
      }
    }
    cplx K = carry[k].G;  // backward state at the run's last element
#pragma unroll
    for (int i = kR - 1; i >= 0; --i) {
      if constexpr (MS) {
        if (tmask & (1u << i)) ms.hm[(int64_t)k * ms.M + (--ti)] = K;
      } else {
        out[i] = fma(mw.re, K.re, fma(-mw.im, K.im, out[i]));
      }
      K = cmul(d[i], cplx{K.re + b[i], K.im});
    }
  }
}

// ------------------------------------------------------------ tile body

struct TileGeom {
  int64_t ib, jb;  // first target / source of the tile
  int nx, ny, len;
  double zprev;
};

__device__ __forceinline__ TileGeom tile_geom(const StreamArgs& a, int64_t t) {
  TileGeom tg;
  const int64_t L = a.M + a.N;
  const int64_t d0 = t * kTile;
  const int64_t d1 = (d0 + kTile < L) ? d0 + kTile : L;
  tg.ib = a.tile_ib[t];
  const int64_t ie = a.tile_ib[t + 1];
  tg.jb = d0 - tg.ib;
  tg.nx = (int)(ie - tg.ib);
  tg.ny = (int)((d1 - ie) - tg.jb);
  tg.len = (int)(d1 - d0);
  if (t == 0) {
    tg.zprev = a.zprev0;
  } else {
    double px = tg.ib > 0 ? a.xs[tg.ib - 1] : -INFINITY;
    double py = tg.jb > 0 ? a.ys[tg.jb - 1] : -INFINITY;
    tg.zprev = fmax(px, py);
  }
  return tg;
}

struct LaneRun {
  double g[kR];
  double b[kR];
  unsigned tmask;
  int tfirst;
  double gmax;
};

// Loads the tile into shared memory and merges this lane's run into registers.
__device__ __forceinline__ void load_and_merge(const StreamArgs& a, const TileGeom& tg,
                                               double* sx, double* sy, double* sb, LaneRun& r) {
  for (int i = threadIdx.x; i < tg.nx; i += kThreads) sx[i] = __ldg(a.xs + tg.ib + i);
  for (int j = threadIdx.x; j < tg.ny; j += kThreads) {
    sy[j] = __ldg(a.ys + tg.jb + j);
    sb[j] = __ldg(a.bs + tg.jb + j);
  }
  __syncthreads();
  const int d0 = threadIdx.x * kR;
  const int dd = d0 < tg.len ? d0 : tg.len;
  int i = (int)merge_path(sx, tg.nx, sy, tg.ny, dd);
  int j = dd - i;
  double prev;
  if (d0 == 0) {
    prev = tg.zprev;
  } else {
    double px = i > 0 ? sx[i - 1] : -INFINITY;
    double py = j > 0 ? sy[j - 1] : -INFINITY;
    prev = fmax(px, py);
  }
  r.tfirst = i;
  r.tmask = 0u;
  r.gmax = 0.0;
#pragma unroll
  for (int e = 0; e < kR; ++e) {
    if (d0 + e < tg.len) {
      const bool src = (j < tg.ny) && (i >= tg.nx || sy[j] <= sx[i]);
      double z;
      if (src) {
        z = sy[j];
        r.b[e] = sb[j];
        ++j;
      } else {
        z = sx[i];
        r.b[e] = 0.0;
        r.tmask |= 1u << e;
        ++i;
      }
      r.g[e] = z - prev;
      prev = z;
    } else {
      r.g[e] = 0.0;
      r.b[e] = 0.0;
    }
    r.gmax = fmax(r.gmax, r.g[e]);
  }
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Dispatch on the warp-uniform Taylor degree.
__device__ __forceinline__ void dispatch_pass1(int D, const ModeTable& mt, int ne,
                                               const LaneRun& r, LaneAgg* out) {
  switch (D) {
#define FGT_P1(n) \
  case n:         \
    pass1<n>(mt, ne, r.g, r.b, out); \
    break;
    FGT_P1(0) FGT_P1(1) FGT_P1(2) FGT_P1(3) FGT_P1(4) FGT_P1(5) FGT_P1(6) FGT_P1(7)
    FGT_P1(8) FGT_P1(9) FGT_P1(10) FGT_P1(11) FGT_P1(12) FGT_P1(13) FGT_P1(14)
    FGT_P1(15) FGT_P1(16)
#undef FGT_P1
    default:
      pass1<-1>(mt, ne, r.g, r.b, out);
  }
}

template <bool MS>
__device__ __forceinline__ void dispatch_pass2(int D, const ModeTable& mt, int ne,
                                               const LaneRun& r, const LaneAgg* carry,
                                               double (&out)[kR], const ModeSumsOut& ms) {
  switch (D) {
#define FGT_P2(n) \
  case n:         \
    pass2<n, MS>(mt, ne, r.g, r.b, r.tmask, carry, out, ms); \
    break;
    FGT_P2(0) FGT_P2(1) FGT_P2(2) FGT_P2(3) FGT_P2(4) FGT_P2(5) FGT_P2(6) FGT_P2(7)
    FGT_P2(8) FGT_P2(9) FGT_P2(10) FGT_P2(11) FGT_P2(12) FGT_P2(13) FGT_P2(14)
    FGT_P2(15) FGT_P2(16)
#undef FGT_P2
    default:
      pass2<-1, MS>(mt, ne, r.g, r.b, r.tmask, carry, out, ms);
  }
}

// Bytes of the aliased region: tile data (x, y, beta) during the merge, lane
// aggregates / carries afterwards.
__host__ __device__ __forceinline__ size_t tile_dyn_bytes(int ne) {
  size_t data = sizeof(double) * 3 * kTile;
  size_t aggs = sizeof(LaneAgg) * kThreads * (size_t)ne;
  return data > aggs ? data : aggs;
}

// Shared-memory layout of one tile CTA.
struct TileSmem {
  ModeTable mt;
  LaneAgg wagg[kWarps][kMaxModes];  // warp aggregates, then warp carries
  // followed by the dynamic region: max(3*kTile doubles, kThreads*ne LaneAgg)
};

__device__ __forceinline__ void load_mode_table(const ModeTable* g, ModeTable& s) {
  const double* src = reinterpret_cast<const double*>(g);
  double* dst = reinterpret_cast<double*>(&s);
  constexpr int n = sizeof(ModeTable) / sizeof(double);
  for (int i = threadIdx.x; i < n; i += kThreads) dst[i] = src[i];
}

// Sequential scans by lanes q < 2*ne of a warp: q < ne forward of mode q,
// ne <= q < 2ne backward of mode q-ne.  `aggs` is [lanes][ne] LaneAgg.
// reduce: combine lanes [l0, l0+n) into (A, F) / G.
__device__ __forceinline__ LaneAgg seq_reduce(const LaneAgg* aggs, int ne, int l0, int n, int q) {
  LaneAgg res{{1.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
  if (q < ne) {
    const int k = q;
    cplx A = {1.0, 0.0}, F = {0.0, 0.0};
    for (int l = l0; l < l0 + n; ++l) {
      const LaneAgg& x = aggs[l * ne + k];
      F = cmad(x.A, F, x.F);
      A = cmul(A, x.A);
    }
    res.A = A;
    res.F = F;
  } else {
    const int k = q - ne;
    cplx G = {0.0, 0.0};
    for (int l = l0 + n - 1; l >= l0; --l) {
      const LaneAgg& x = aggs[l * ne + k];
      G = cmad(x.A, G, x.G);
    }
    res.G = G;
  }
  return res;
}

// Exclusive carries, written in place: forward carry into .F, backward into .G
__device__ __forceinline__ void seq_carry(LaneAgg* aggs, int ne, int l0, int n, int q, cplx cin) {
  if (q < ne) {
    const int k = q;
    cplx c = cin;
    for (int l = l0; l < l0 + n; ++l) {
      LaneAgg& x = aggs[l * ne + k];
      const cplx A = x.A, F = x.F;
      x.F = c;
      c = cmad(A, c, F);
    }
  } else {
    const int k = q - ne;
    cplx c = cin;
    for (int l = l0 + n - 1; l >= l0; --l) {
      LaneAgg& x = aggs[l * ne + k];
      const cplx A = x.A, G = x.G;
      x.G = c;
      c = cmad(A, c, G);
    }
  }
}

// KIND: 0 = tile aggregates (K1), 1 = main pass (K3), 2 = mode sums (test hook)
template <int KIND>
__global__ void __launch_bounds__(kThreads, 4)
    tile_kernel(StreamArgs a, ModeParams P, const ModeTable* __restrict__ mtab, TileState ts,
                OutArgs o) {
  constexpr bool MAIN = KIND != 0;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TileSmem& S = *reinterpret_cast<TileSmem*>(smem_raw);
  unsigned char* dyn = smem_raw + sizeof(TileSmem);
  double* sx = reinterpret_cast<double*>(dyn);
  double* sy = sx + kTile;
  double* sb = sy + kTile;
  LaneAgg* aggs = reinterpret_cast<LaneAgg*>(dyn);  // aliases sx/sy/sb after merge
  double* su = reinterpret_cast<double*>(dyn + tile_dyn_bytes(P.ne));  // output staging

  const int64_t t = blockIdx.x;
  const int ne = P.ne;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  load_mode_table(mtab, S.mt);
  const TileGeom tg = tile_geom(a, t);
  LaneRun r;
  load_and_merge(a, tg, sx, sy, sb, r);
  const int D = pick_degree(P, warp_max(r.gmax));
  __syncthreads();  // tile data dead from here on; aggs alias it

  LaneAgg* mine = aggs + threadIdx.x * ne;
  dispatch_pass1(D, S.mt, ne, r, mine);
  __syncwarp();

  // Level A: warp aggregates.
  if (lane < 2 * ne) {
    LaneAgg w = seq_reduce(aggs, ne, warp * 32, 32, lane);
    const int k = lane < ne ? lane : lane - ne;
    if (lane < ne) {
      S.wagg[warp][k].A = w.A;
      S.wagg[warp][k].F = w.F;
    } else {
      S.wagg[warp][k].G = w.G;
    }
  }
  __syncthreads();

  if constexpr (!MAIN) {
    // Tile aggregate -> global.
    if (warp == 0 && lane < 2 * ne) {
      const int k = lane < ne ? lane : lane - ne;
      if (lane < ne) {
        cplx A = {1.0, 0.0}, F = {0.0, 0.0};
        for (int w = 0; w < kWarps; ++w) {
          F = cmad(S.wagg[w][k].A, F, S.wagg[w][k].F);
          A = cmul(A, S.wagg[w][k].A);
        }
        ts.A[(int64_t)k * a.ntiles + t] = A;
        ts.F[(int64_t)k * a.ntiles + t] = F;
      } else {
        cplx G = {0.0, 0.0};
        for (int w = kWarps - 1; w >= 0; --w) G = cmad(S.wagg[w][k].A, G, S.wagg[w][k].G);
        ts.G[(int64_t)k * a.ntiles + t] = G;
      }
    }
    return;
  } else {
    // Level B: warp carries from the tile carries.
    if (warp == 0 && lane < 2 * ne) {
      const int k = lane < ne ? lane : lane - ne;
      if (lane < ne) {
        cplx c = ts.Cf[(int64_t)k * a.ntiles + t];
        for (int w = 0; w < kWarps; ++w) {
          const cplx A = S.wagg[w][k].A, F = S.wagg[w][k].F;
          S.wagg[w][k].F = c;
          c = cmad(A, c, F);
        }
      } else {
        cplx c = ts.Cb[(int64_t)k * a.ntiles + t];
        for (int w = kWarps - 1; w >= 0; --w) {
          const cplx A = S.wagg[w][k].A, G = S.wagg[w][k].G;
          S.wagg[w][k].G = c;
          c = cmad(A, c, G);
        }
      }
    }
    __syncthreads();
    // Level C: lane carries inside each warp.
    if (lane < 2 * ne) {
      const int k = lane < ne ? lane : lane - ne;
      const cplx cin = lane < ne ? S.wagg[warp][k].F : S.wagg[warp][k].G;
      seq_carry(aggs, ne, warp * 32, 32, lane, cin);
    }
    __syncwarp();

    double out[kR];
#pragma unroll
    for (int e = 0; e < kR; ++e) out[e] = 0.0;
    if constexpr (KIND == 2) {
      ModeSumsOut ms{o.hp, o.hm, a.M, o.u_offset + tg.ib + r.tfirst};
      dispatch_pass2<true>(D, S.mt, ne, r, mine, out, ms);
      return;
    } else {
      dispatch_pass2<false>(D, S.mt, ne, r, mine, out, ModeSumsOut{nullptr, nullptr, 0, 0});
    }

    int tk = r.tfirst;
#pragma unroll
    for (int e = 0; e < kR; ++e)
      if (r.tmask & (1u << e)) su[tk++] = out[e];
    __syncthreads();
    const int64_t base = o.u_offset + tg.ib;
    if (o.tperm) {
      for (int i = threadIdx.x; i < tg.nx; i += kThreads) o.u[o.tperm[base + i]] = su[i];
    } else {
      for (int i = threadIdx.x; i < tg.nx; i += kThreads) o.u[base + i] = su[i];
    }
  }
}

// ------------------------------------------------------------ K0 / K2

__global__ void partition_kernel(const double* __restrict__ xs, int64_t M,
                                 const double* __restrict__ ys, int64_t N, int64_t tile,
                                 int64_t ntiles, int64_t* __restrict__ tile_ib) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t > ntiles) return;
  int64_t diag = t * tile;
  if (diag > M + N) diag = M + N;
  tile_ib[t] = merge_path(xs, M, ys, N, diag);
}

constexpr int kScanThreads = 1024;

// One CTA per (mode, direction).  Thread-serial segments + a block scan of
// the segment aggregates under (a, s) o (a', s') = (a a', a' s + s').
__global__ void __launch_bounds__(kScanThreads)
    carry_scan_kernel(TileState ts, int64_t ntiles, int ne, const cplx* __restrict__ carry_in,
                      cplx* __restrict__ totals) {
  __shared__ cplx sa[kScanThreads];
  __shared__ cplx ss[kScanThreads];
  const int k = blockIdx.x % ne;
  const bool bwd = blockIdx.x >= ne;
  const cplx* A = ts.A + (int64_t)k * ntiles;
  const cplx* Sv = (bwd ? ts.G : ts.F) + (int64_t)k * ntiles;
  cplx* C = (bwd ? ts.Cb : ts.Cf) + (int64_t)k * ntiles;
  const int64_t per = (ntiles + kScanThreads - 1) / kScanThreads;
  const int64_t r0 = (int64_t)threadIdx.x * per;
  const int64_t r1 = (r0 + per < ntiles) ? r0 + per : ntiles;
  cplx a = {1.0, 0.0}, s = {0.0, 0.0};
  for (int64_t r = r0; r < r1; ++r) {
    const int64_t b = bwd ? ntiles - 1 - r : r;
    const cplx Ab = A[b];
    s = cmad(Ab, s, Sv[b]);
    a = cmul(a, Ab);
  }
  // inclusive Hillis-Steele scan over threads
  sa[threadIdx.x] = a;
  ss[threadIdx.x] = s;
  __syncthreads();
  for (int off = 1; off < kScanThreads; off <<= 1) {
    cplx pa = {1.0, 0.0}, ps = {0.0, 0.0};
    const bool has = threadIdx.x >= off;
    if (has) {
      pa = sa[threadIdx.x - off];
      ps = ss[threadIdx.x - off];
    }
    __syncthreads();
    if (has) {
      // earlier (pa, ps) then later (a, s)
      s = cmad(a, ps, s);
      a = cmul(pa, a);
      sa[threadIdx.x] = a;
      ss[threadIdx.x] = s;
    }
    __syncthreads();
  }
  // exclusive prefix for this thread
  cplx ea = {1.0, 0.0}, es = {0.0, 0.0};
  if (threadIdx.x > 0) {
    ea = sa[threadIdx.x - 1];
    es = ss[threadIdx.x - 1];
  }
  const cplx cin = carry_in ? carry_in[(bwd ? ne : 0) + k] : cplx{0.0, 0.0};
  cplx c = cmad(ea, cin, es);
  for (int64_t r = r0; r < r1; ++r) {
    const int64_t b = bwd ? ntiles - 1 - r : r;
    C[b] = c;
    c = cmad(A[b], c, Sv[b]);
  }
  if (totals && threadIdx.x == kScanThreads - 1) {
    // totals layout: [ne] A, [ne] F-total, [ne] G-total
    if (!bwd) {
      totals[k] = a;
      totals[ne + k] = s;
    } else {
      totals[2 * ne + k] = s;
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

size_t tile_smem_bytes(int ne) {
  return sizeof(TileSmem) + tile_dyn_bytes(ne) + sizeof(double) * kTile;
}

cudaError_t launch_partition(const double* xs, int64_t M, const double* ys, int64_t N,
                             int64_t tile, int64_t ntiles, int64_t* tile_ib, cudaStream_t st) {
  const int64_t n = ntiles + 1;
  const int bs = 256;
  note_launch();
  partition_kernel<<<(unsigned)((n + bs - 1) / bs), bs, 0, st>>>(xs, M, ys, N, tile, ntiles,
                                                                 tile_ib);
  return cudaGetLastError();
}

template <int KIND>
static cudaError_t launch_tile(const StreamArgs& a, const ModeParams& P, const ModeTable* mt,
                               TileState ts, OutArgs o, cudaStream_t st) {
  if (a.ntiles == 0) return cudaSuccess;
  const size_t smem = tile_smem_bytes(P.ne);
  static bool configured[3] = {false, false, false};
  if (!configured[KIND]) {
    cudaError_t e = cudaFuncSetAttribute(tile_kernel<KIND>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)tile_smem_bytes(kMaxModes));
    if (e != cudaSuccess) return e;
    configured[KIND] = true;
  }
  note_launch();
  tile_kernel<KIND><<<(unsigned)a.ntiles, kThreads, smem, st>>>(a, P, mt, ts, o);
  return cudaGetLastError();
}

cudaError_t launch_aggregate(const StreamArgs& a, const ModeParams& P, const ModeTable* mt,
                             TileState ts, cudaStream_t st) {
  return launch_tile<0>(a, P, mt, ts, OutArgs{}, st);
}

cudaError_t launch_main(const StreamArgs& a, const ModeParams& P, const ModeTable* mt,
                        TileState ts, OutArgs o, cudaStream_t st) {
  return launch_tile<1>(a, P, mt, ts, o, st);
}

cudaError_t launch_mode_sums(const StreamArgs& a, const ModeParams& P, const ModeTable* mt,
                             TileState ts, OutArgs o, cudaStream_t st) {
  return launch_tile<2>(a, P, mt, ts, o, st);
}

cudaError_t launch_carry_scan(const TileState& ts, int64_t ntiles, int ne, const cplx* carry_in,
                              cplx* totals, cudaStream_t st) {
  if (ntiles == 0) return cudaSuccess;
  note_launch();
  carry_scan_kernel<<<2 * ne, kScanThreads, 0, st>>>(ts, ntiles, ne, carry_in, totals);
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
