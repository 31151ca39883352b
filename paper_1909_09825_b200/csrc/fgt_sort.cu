// Sort / permutation plumbing of plan(): the device replacement of
// sort_with_perm (proj/src/transform.cpp:27-39, std::sort of (value, index)
// pairs => ascending, ties in original order).  The structural checks
// (finite, sorted, same points) run in the plan tile pass (fgt_scan.cu).
//
//   radix sort      : stable LSD, 8-bit digits over order-preserving u64 keys
//                     with a u32 index payload; passes whose digit is constant
//                     across all keys are skipped (one global histogram pass);
//                     the first pass forms the keys from the values, the last
//                     writes the sorted values and the permutation
#include <cuda_runtime.h>
#include <stdint.h>

#include "fgt_sort.cuh"

namespace fgt_b200 {

namespace {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
#ifndef FGT_SORT_ITEMS
#define FGT_SORT_ITEMS 12
#endif
constexpr int kItems = FGT_SORT_ITEMS;                      // keys per lane per tile
constexpr int kSortTile = kSortThreads * kItems;            // 2048 keys per CTA
constexpr int kRadix = 256;

// -0.0 and +0.0 compare equal in the reference's std::sort; canonicalise so
// that both map to the same key (the stable index order then decides).
__device__ __forceinline__ uint64_t key_of(double x) {
  uint64_t k = (uint64_t)__double_as_longlong(x + 0.0);
  return (k >> 63) ? ~k : (k | 0x8000000000000000ull);
}
__device__ __forceinline__ double value_of(uint64_t k) {
  k = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)k);
}

// Every digit constant: all keys equal, the stable order is the input order.
__global__ void identity_sort_kernel(const double* __restrict__ x, int64_t n,
                                     double* __restrict__ sorted, int32_t* __restrict__ perm) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    sorted[i] = value_of(key_of(x[i]));
    perm[i] = (int32_t)i;
  }
}

// All 8 digit histograms in one read: hist8[pass][digit].
__global__ void global_hist_kernel(const double* __restrict__ x, int64_t n,
                                   unsigned long long* __restrict__ hist8) {
  __shared__ unsigned int h[8][kRadix];
  for (int i = threadIdx.x; i < 8 * kRadix; i += blockDim.x) (&h[0][0])[i] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = key_of(__ldg(x + i));
#pragma unroll
    for (int p = 0; p < 8; ++p) atomicAdd(&h[p][(k >> (8 * p)) & 0xff], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 8 * kRadix; i += blockDim.x) {
    unsigned int v = (&h[0][0])[i];
    if (v) atomicAdd(hist8 + i, (unsigned long long)v);
  }
}

// Per-tile digit counts, digit-major: cnt[digit * ntiles + tile].  FIRST:
// the keys are formed from the input values on the fly (no key array yet).
template <bool FIRST>
__global__ void __launch_bounds__(kSortThreads)
    tile_hist_kernel(const uint64_t* __restrict__ keys, const double* __restrict__ x, int64_t n,
                     int shift, uint32_t* __restrict__ cnt, int64_t ntiles) {
  __shared__ unsigned int h[kRadix];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kSortTile;
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    int64_t i = base + it * kSortThreads + threadIdx.x;
    if (i < n) {
      const uint64_t k = FIRST ? key_of(__ldg(x + i)) : keys[i];
      atomicAdd(&h[(k >> shift) & 0xff], 1u);
    }
  }
  __syncthreads();
  cnt[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

constexpr size_t kScatterSmem = (sizeof(uint64_t) + sizeof(uint32_t)) * kSortTile;

// Stable scatter.  Warp w owns tile keys [w*256, (w+1)*256) and ranks them in
// order with __match_any_sync; warp counters are scanned digit-wise across
// warps, keys are staged digit-sorted in shared memory and written out in
// contiguous per-digit runs.
// FIRST: keys from the input values and the identity payload; LAST: the
// sorted values and the permutation written instead of keys / payload.
template <bool FIRST, bool LAST>
__global__ void __launch_bounds__(kSortThreads)
    scatter_kernel(const uint64_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                   const double* __restrict__ x, int64_t n, int shift,
                   const uint32_t* __restrict__ offs, int64_t ntiles, uint64_t* __restrict__ kout,
                   uint32_t* __restrict__ vout, double* __restrict__ sorted,
                   int32_t* __restrict__ perm) {
  __shared__ unsigned int wc[kSortWarps][kRadix];
  __shared__ unsigned int loff[kRadix];
  __shared__ unsigned int goff[kRadix];
  extern __shared__ __align__(16) unsigned char sort_dyn[];  // staging (kScatterSmem)
  uint64_t* sk = reinterpret_cast<uint64_t*>(sort_dyn);
  uint32_t* sv = reinterpret_cast<uint32_t*>(sk + kSortTile);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < kSortWarps * kRadix; i += kSortThreads) (&wc[0][0])[i] = 0;
  goff[threadIdx.x] = offs[(int64_t)threadIdx.x * ntiles + blockIdx.x];
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kSortTile;
  const int64_t tn64 = n - base < kSortTile ? n - base : kSortTile;
  const int tn = (int)tn64;
  const unsigned lt = (1u << lane) - 1u;
  uint64_t key[kItems];
  uint32_t val[kItems];
  int dig[kItems];
  unsigned rank[kItems];
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    const int li = warp * 32 * kItems + it * 32 + lane;  // tile-local index, in order
    const bool ok = li < tn;
    if constexpr (FIRST) {
      key[it] = ok ? key_of(__ldg(x + base + li)) : 0ull;
      val[it] = (uint32_t)(base + li);
    } else {
      key[it] = ok ? kin[base + li] : 0ull;
      val[it] = ok ? vin[base + li] : 0u;
    }
    const int d = ok ? (int)((key[it] >> shift) & 0xff) : -1;
    dig[it] = d;
    const unsigned active = __ballot_sync(0xffffffffu, ok);
    unsigned peers = __match_any_sync(0xffffffffu, d);
    if (ok) {
      peers &= active;
      rank[it] = wc[warp][d] + __popc(peers & lt);
    }
    __syncwarp();
    if (ok && (lane == __ffs(peers) - 1)) wc[warp][d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  {
    const int d = threadIdx.x;
    unsigned run = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
      unsigned c = wc[w][d];
      wc[w][d] = run;
      run += c;
    }
    loff[d] = run;  // tile total for digit d (scanned below)
  }
  __syncthreads();
  // exclusive scan of loff over digits (256 entries, one per thread)
  {
    unsigned v = loff[threadIdx.x];
    unsigned incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    __shared__ unsigned int wsum[kSortWarps];
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    unsigned wpre = 0;
    for (int w = 0; w < warp; ++w) wpre += wsum[w];
    __syncthreads();
    loff[threadIdx.x] = wpre + incl - v;
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    if (dig[it] >= 0) {
      const int d = dig[it];
      const unsigned p = loff[d] + wc[warp][d] + rank[it];
      sk[p] = key[it];
      sv[p] = val[it];
    }
  }
  __syncthreads();
  for (int p = threadIdx.x; p < tn; p += kSortThreads) {
    const uint64_t k = sk[p];
    const int d = (int)((k >> shift) & 0xff);
    const int64_t o = (int64_t)goff[d] + (p - (int)loff[d]);
    if constexpr (LAST) {
      sorted[o] = value_of(k);
      perm[o] = (int32_t)sv[p];
    } else {
      kout[o] = k;
      vout[o] = sv[p];
    }
  }
}

// ---- block-wide exclusive scan of uint32 (values fit: counts <= 2^32) -----
constexpr int kScanBlock = 1024;
constexpr int kScanItems = 8;
constexpr int kScanChunk = kScanBlock * kScanItems;

__device__ __forceinline__ unsigned block_excl_scan(unsigned v, unsigned* total) {
  __shared__ unsigned ws[kScanBlock / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) ws[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    unsigned w = lane < kScanBlock / 32 ? ws[lane] : 0u;
    unsigned wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < kScanBlock / 32) ws[lane] = wi - w;
    if (lane == kScanBlock / 32 - 1) ws[kScanBlock / 32 - 1] = wi - w, *total = wi;
  }
  __syncthreads();
  unsigned r = ws[warp] + incl - v;
  __syncthreads();
  return r;
}

// The scatter offsets of one pass in one launch: CTA d scans the tile counts
// of digit d (cnt is digit-major) on top of the digit's base, the number of
// keys with a smaller digit (from the global histogram of the pass).
__global__ void __launch_bounds__(kScanBlock)
    digit_scan_kernel(const uint32_t* __restrict__ cnt, int64_t ntiles,
                      const unsigned long long* __restrict__ hist, uint32_t* __restrict__ offs) {
  __shared__ unsigned tot;
  const int d = blockIdx.x;
  const unsigned hb = (int)threadIdx.x < d ? (unsigned)hist[threadIdx.x] : 0u;
  block_excl_scan(hb, &tot);
  unsigned run = tot;
  const uint32_t* in = cnt + (int64_t)d * ntiles;
  uint32_t* out = offs + (int64_t)d * ntiles;
  for (int64_t c0 = 0; c0 < ntiles; c0 += kScanChunk) {
    const int64_t base = c0 + (int64_t)threadIdx.x * kScanItems;
    unsigned v[kScanItems];
    unsigned s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      v[i] = base + i < ntiles ? in[base + i] : 0u;
      s += v[i];
    }
    unsigned r = run + block_excl_scan(s, &tot);
    run += tot;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      if (base + i < ntiles) out[base + i] = r;
      r += v[i];
    }
  }
}
static_assert(kScanBlock >= kRadix, "digit_scan_kernel: one thread per smaller digit");

inline unsigned grid_for(int64_t n, int bs) {
  int64_t g = (n + bs - 1) / bs;
  if (g > 148 * 32) g = 148 * 32;
  if (g < 1) g = 1;
  return (unsigned)g;
}

}  // namespace

size_t radix_sort_workspace_bytes(int64_t n) {
  const int64_t ntiles = (n + kSortTile - 1) / kSortTile;
  size_t b = 0;
  b += 2 * sizeof(uint64_t) * (size_t)n;                 // keys x2
  b += 2 * sizeof(uint32_t) * (size_t)n;                 // vals x2
  b += 2 * sizeof(uint32_t) * (size_t)(ntiles * kRadix); // cnt + offs
  b += sizeof(unsigned long long) * 8 * kRadix;
  return b + 16 * 256;  // 8 regions, each re-aligned to 256 B
}

static inline char* align_up(char* p) {
  return (char*)(((uintptr_t)p + 255) & ~(uintptr_t)255);
}

// Workspace layout of one sort.
struct SortWs {
  uint64_t *k0, *k1;
  uint32_t *v0, *v1, *cnt, *offs;
  unsigned long long* hist8;
};
static SortWs sort_ws(void* workspace, int64_t n) {
  const int64_t ntiles = (n + kSortTile - 1) / kSortTile;
  SortWs w;
  char* p = align_up((char*)workspace);
  w.k0 = (uint64_t*)p; p = align_up(p + sizeof(uint64_t) * n);
  w.k1 = (uint64_t*)p; p = align_up(p + sizeof(uint64_t) * n);
  w.v0 = (uint32_t*)p; p = align_up(p + sizeof(uint32_t) * n);
  w.v1 = (uint32_t*)p; p = align_up(p + sizeof(uint32_t) * n);
  w.cnt = (uint32_t*)p; p = align_up(p + sizeof(uint32_t) * ntiles * kRadix);
  w.offs = (uint32_t*)p; p = align_up(p + sizeof(uint32_t) * ntiles * kRadix);
  w.hist8 = (unsigned long long*)p;
  return w;
}

cudaError_t radix_sort_begin(const double* x, int64_t n, void* workspace,
                             unsigned long long* hist_host, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const SortWs w = sort_ws(workspace, n);
  note_launch(1);
  cudaError_t e = cudaMemsetAsync(w.hist8, 0, sizeof(unsigned long long) * 8 * kRadix, st);
  if (e != cudaSuccess) return e;
  global_hist_kernel<<<grid_for(n, 256) < 1184 ? grid_for(n, 256) : 1184, 256, 0, st>>>(x, n,
                                                                                       w.hist8);
  return cudaMemcpyAsync(hist_host, w.hist8, sizeof(unsigned long long) * 8 * kRadix,
                         cudaMemcpyDeviceToHost, st);
}

template <bool F, bool L>
static cudaError_t scatter_pass(const uint64_t* kin, const uint32_t* vin, const double* x,
                                int64_t n, int shift, const uint32_t* offs, int64_t ntiles,
                                uint64_t* kout, uint32_t* vout, double* sorted, int32_t* perm,
                                cudaStream_t st) {
  static std::atomic<unsigned long long> smem_set{0};
  cudaError_t e = ensure_dynamic_smem(scatter_kernel<F, L>, (int)kScatterSmem, smem_set);
  if (e != cudaSuccess) return e;
  scatter_kernel<F, L><<<(unsigned)ntiles, kSortThreads, kScatterSmem, st>>>(
      kin, vin, x, n, shift, offs, ntiles, kout, vout, sorted, perm);
  return cudaGetLastError();
}

// The first pass reads the values (keys formed on the fly), the last one
// writes the sorted values and the permutation: no separate key / unkey pass.
cudaError_t radix_sort_end(const double* x, int64_t n, double* sorted, int32_t* perm,
                           void* workspace, const unsigned long long* h8, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int64_t ntiles = (n + kSortTile - 1) / kSortTile;
  const SortWs w = sort_ws(workspace, n);
  int passes[8], np = 0;
  for (int p = 0; p < 8; ++p) {
    bool trivial = false;
    for (int d = 0; d < kRadix; ++d)
      if (h8[p * kRadix + d] == (unsigned long long)n) trivial = true;
    if (!trivial) passes[np++] = p;  // a constant digit's pass is the identity
  }
  if (np == 0) {
    note_launch();
    identity_sort_kernel<<<grid_for(n, 256), 256, 0, st>>>(x, n, sorted, perm);
    return cudaGetLastError();
  }
  uint64_t* kin = w.k0;
  uint64_t* kout = w.k1;
  uint32_t* vin = w.v0;
  uint32_t* vout = w.v1;
  cudaError_t e = cudaSuccess;
  for (int q = 0; q < np; ++q) {
    const int shift = 8 * passes[q];
    const bool first = q == 0, last = q + 1 == np;
    note_launch(2);
    if (first)
      tile_hist_kernel<true><<<(unsigned)ntiles, kSortThreads, 0, st>>>(nullptr, x, n, shift, w.cnt,
                                                                        ntiles);
    else
      tile_hist_kernel<false><<<(unsigned)ntiles, kSortThreads, 0, st>>>(kin, nullptr, n, shift,
                                                                         w.cnt, ntiles);
    note_launch();
    digit_scan_kernel<<<kRadix, kScanBlock, 0, st>>>(w.cnt, ntiles, w.hist8 + passes[q] * kRadix,
                                                     w.offs);
    if (first && last)
      e = scatter_pass<true, true>(nullptr, nullptr, x, n, shift, w.offs, ntiles, nullptr, nullptr,
                                   sorted, perm, st);
    else if (first)
      e = scatter_pass<true, false>(nullptr, nullptr, x, n, shift, w.offs, ntiles, kout, vout,
                                    nullptr, nullptr, st);
    else if (last)
      e = scatter_pass<false, true>(kin, vin, nullptr, n, shift, w.offs, ntiles, nullptr, nullptr,
                                    sorted, perm, st);
    else
      e = scatter_pass<false, false>(kin, vin, nullptr, n, shift, w.offs, ntiles, kout, vout,
                                     nullptr, nullptr, st);
    if (e != cudaSuccess) return e;
    uint64_t* tk = kin; kin = kout; kout = tk;
    uint32_t* tv = vin; vin = vout; vout = tv;
  }
  return cudaSuccess;
}

cudaError_t radix_sort_with_perm(const double* x, int64_t n, double* sorted, int32_t* perm,
                                 void* workspace, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  unsigned long long h8[8 * kRadix];
  cudaError_t e = radix_sort_begin(x, n, workspace, h8, st);
  if (e != cudaSuccess) return e;
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return e;
  return radix_sort_end(x, n, sorted, perm, workspace, h8, st);
}

}  // namespace fgt_b200
