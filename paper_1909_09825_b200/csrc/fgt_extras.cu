// Device kernels around the hot path:
//   fgt_direct            <- fgt::direct (proj/src/transform.cpp:255-288): O(|S| N)
//                            sum; long double in the reference, double-double here
//   fgt_plan_gap_table    <- precompute_gap_table (transform.cpp:221-237)
//   fgt_uniform_points_device <- rng::uniform_points (proj/src/rng.cpp:7-29)
//   fgt_sort_device       <- sort_with_perm (transform.cpp:27-39)
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "../../include/fgt1d_b200.h"
#include "fgt_device.cuh"
#include "fgt_scan.cuh"
#include "fgt_sort.cuh"

using namespace fgt_b200;

namespace fgt_b200 {
void set_last_error(const std::string& m);  // fgt_capi.cu
}

namespace {

struct ErrSink {
  ErrSink& operator=(const std::string& m) {
    set_last_error(m);
    return *this;
  }
};
ErrSink g_err;

int cuda_fail(cudaError_t e, const char* what) {
  cudaGetLastError();
  g_err = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? FGT_ERR_NOMEM : FGT_ERR_CUDA;
}

#define CKR(expr, what)                          \
  do {                                           \
    cudaError_t e_ = (expr);                     \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

struct dd {
  double hi, lo;
};

__device__ __forceinline__ dd two_sum(double a, double b) {
  double s = a + b;
  double bb = s - a;
  double e = (a - (s - bb)) + (b - bb);
  return {s, e};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  double lo = s.lo + a.lo + b.lo;
  double hi = s.hi + lo;
  return {hi, lo - (hi - s.hi)};
}

constexpr int kDirThreads = 256;
constexpr int kDirPerThread = 32;
constexpr int64_t kDirChunk = (int64_t)kDirThreads * kDirPerThread;

// One block per (target, source chunk); deterministic in-order reduction.
__global__ void __launch_bounds__(kDirThreads)
    direct_partial_kernel(const double* __restrict__ x, const int64_t* __restrict__ subset,
                          int64_t ntarg, const double* __restrict__ y,
                          const double* __restrict__ a, int64_t N, double q_hi, double q_lo,
                          int64_t nchunks, dd* __restrict__ partial) {
  const int64_t t = blockIdx.x / nchunks;
  const int64_t ch = blockIdx.x % nchunks;
  const double xv = x[subset ? subset[t] : t];
  dd acc = {0.0, 0.0};
  const int64_t j0 = ch * kDirChunk;
  for (int r = 0; r < kDirPerThread; ++r) {
    const int64_t j = j0 + (int64_t)r * kDirThreads + threadIdx.x;
    if (j >= N) break;
    const double yv = y[j];
    // d = x - y exactly (two-diff)
    dd d = two_sum(xv, -yv);
    // d^2 (double-double)
    double p = d.hi * d.hi;
    double pe = fma(d.hi, d.hi, -p) + 2.0 * d.hi * d.lo;
    // arg = d^2 / (4 delta)
    double ah = p * q_hi;
    double al = fma(p, q_hi, -ah) + (pe * q_hi + p * q_lo);
    dd arg = two_sum(ah, al);
    if (arg.hi > 745.5) continue;
    double eh = exp(-arg.hi);
    double el = -eh * arg.lo;  // exp(-hi - lo) ~ eh (1 - lo)
    const double av = a[j];
    double th = eh * av;
    double tl = fma(eh, av, -th) + el * av;
    acc = dd_add(acc, dd{th, tl});
  }
  // block reduction (fixed order)
  __shared__ dd sh[kDirThreads];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kDirThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = dd_add(sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

__global__ void direct_final_kernel(const dd* __restrict__ partial, int64_t ntarg,
                                    int64_t nchunks, double* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntarg) return;
  dd acc = {0.0, 0.0};
  for (int64_t c = 0; c < nchunks; ++c) acc = dd_add(acc, partial[t * nchunks + c]);
  out[t] = acc.hi + acc.lo;
}

__global__ void gap_table_kernel(const double* __restrict__ xs, int64_t M, int ne,
                                 const double* __restrict__ sre, const double* __restrict__ sim,
                                 double2* __restrict__ out) {
  const int64_t n = (M - 1) * ne;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(idx / (M - 1));
    const int64_t i = idx % (M - 1);
    const double d = xs[i + 1] - xs[i];
    double2 r;
    if (d == 0.0) {
      r = make_double2(1.0, 0.0);
    } else {
      cplx e = decay_exact(sre[k], sim[k], d);
      const double n2 = e.re * e.re + e.im * e.im;
      if (n2 > 1.0) {
        const double s = sqrt(n2);
        e.re /= s;
        e.im /= s;
      }
      r = make_double2(e.re, e.im);
    }
    out[idx] = r;
  }
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void uniform_kernel(double* __restrict__ out, int64_t n, uint64_t seed, uint64_t stream,
                               uint64_t offset) {
  const uint64_t base = mix64(seed ^ stream * 0xA24BAED4963EE407ull);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t r = mix64(base + ((uint64_t)i + offset) * 0x9E3779B97F4A7C15ull);
    out[i] = (double)(r >> 11) * 0x1.0p-53;
  }
}

// out[perm[i]] = src[i] (the inverse of launch_gather's out[i] = src[perm[i]]).
__global__ void scatter_kernel(const double* __restrict__ src, const int32_t* __restrict__ perm,
                               int64_t n, double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[__ldg(perm + i)] = __ldg(src + i);
}

// Stable merge of two sorted runs A (na) and B (nb) with int32 payloads:
// out[d] for d in [0, na + nb); A's element precedes B's at equal values
// (A is the earlier run).  Thread t writes kMergePer consecutive outputs
// from its merge-path split.
constexpr int kMergePer = 16;
__global__ void merge2_kernel(const double* __restrict__ av, const int32_t* __restrict__ ai,
                              int64_t na, const double* __restrict__ bv,
                              const int32_t* __restrict__ bi, int64_t nb,
                              double* __restrict__ ov, int32_t* __restrict__ oi) {
  const int64_t n = na + nb;
  const int64_t d0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * kMergePer;
  if (d0 >= n) return;
  int64_t lo = d0 - nb > 0 ? d0 - nb : 0, hi = d0 < na ? d0 : na;
  while (lo < hi) {  // i = number of A elements among the first d0 outputs
    const int64_t mid = (lo + hi + 1) >> 1;
    if (av[mid - 1] <= bv[d0 - mid])
      lo = mid;
    else
      hi = mid - 1;
  }
  int64_t i = lo, j = d0 - lo;
  const int64_t d1 = d0 + kMergePer < n ? d0 + kMergePer : n;
  for (int64_t d = d0; d < d1; ++d) {
    const bool takea = j >= nb || (i < na && av[i] <= bv[j]);
    if (takea) {
      ov[d] = av[i];
      oi[d] = ai[i];
      ++i;
    } else {
      ov[d] = bv[j];
      oi[d] = bi[j];
      ++j;
    }
  }
}

__global__ void iota_kernel(int32_t* __restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)i;
}

// FP64 pipe probe: 8 independent DFMA chains per thread, fully unrolled.
__global__ void __launch_bounds__(256) fp64_probe_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1e-9, x2 = x0 + 2e-9, x3 = x0 + 3e-9;
  double x4 = x0 + 4e-9, x5 = x0 + 5e-9, x6 = x0 + 6e-9, x7 = x0 + 7e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  const double r = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (r == 1.2345) out[0] = r;  // keep the chains alive
}

}  // namespace

extern "C" {

// Measured FP64 FMA throughput (TFLOP/s, FMA = 2 flops) of the current device
// at its current clocks; used by bench.py as the fp64 roofline denominator.
int fgt_fp64_peak(double* tflops, double* ms_out) {
  int dev = 0, sms = 0;
  CKR(cudaGetDevice(&dev), "device");
  CKR(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "attr");
  double* d = nullptr;
  CKR(cudaMalloc(&d, 8), "malloc");
  const int blocks = sms * 8, threads = 256, iters = 2048;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  fp64_probe_kernel<<<blocks, threads>>>(d, 64, 0.999999, 1e-7);  // warm-up
  cudaEventRecord(e0);
  fp64_probe_kernel<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
  cudaEventRecord(e1);
  CKR(cudaEventSynchronize(e1), "probe");
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  const double fmas = (double)blocks * threads * iters * 16.0 * 8.0;
  if (tflops) *tflops = 2.0 * fmas / (ms * 1e-3) / 1e12;
  if (ms_out) *ms_out = ms;
  return FGT_OK;
}


int fgt_direct(const double* targets, int64_t M, const double* sources, int64_t N,
               const double* strengths, double delta, const int64_t* subset, int64_t nsub,
               double* out) {
  if (!std::isfinite(delta) || !(delta > 0.0)) {
    g_err = "delta must be positive and finite";
    return FGT_ERR_DOMAIN;
  }
  for (int64_t i = 0; i < M; ++i)
    if (!std::isfinite(targets[i])) {
      g_err = "target coordinates must be finite";
      return FGT_ERR_DOMAIN;
    }
  for (int64_t j = 0; j < N; ++j)
    if (!std::isfinite(sources[j])) {
      g_err = "source coordinates must be finite";
      return FGT_ERR_DOMAIN;
    }
  const int64_t ntarg = (subset && nsub > 0) ? nsub : M;
  if (subset && nsub > 0)
    for (int64_t i = 0; i < nsub; ++i)
      if (subset[i] < 0 || subset[i] >= M) {
        g_err = "target subset index out of range";
        return FGT_ERR_INVALID;
      }
  if (ntarg == 0) return FGT_OK;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    g_err = "no CUDA device available: the B200 transform has no CPU fallback";
    return FGT_ERR_CUDA;
  }
  if (N == 0) {
    for (int64_t i = 0; i < ntarg; ++i) out[i] = 0.0;
    return FGT_OK;
  }
  // 0.25 / delta in double-double (reference: 0.25L / (long double)delta)
  const long double q = 0.25L / (long double)delta;
  const double q_hi = (double)q;
  const double q_lo = (double)(q - (long double)q_hi);
  const int64_t nchunks = (N + kDirChunk - 1) / kDirChunk;
  double *dx = nullptr, *dy = nullptr, *da = nullptr, *dout = nullptr;
  int64_t* ds = nullptr;
  dd* dpart = nullptr;
  int rc = FGT_OK;
  cudaError_t e;
#define CK2(expr, what)                 \
  if ((e = (expr)) != cudaSuccess) {    \
    rc = cuda_fail(e, what);            \
    goto done;                          \
  }
  CK2(cudaMalloc(&dx, 8 * (M > 0 ? M : 1)), "malloc");
  CK2(cudaMalloc(&dy, 8 * N), "malloc");
  CK2(cudaMalloc(&da, 8 * N), "malloc");
  CK2(cudaMalloc(&dout, 8 * ntarg), "malloc");
  CK2(cudaMalloc(&dpart, sizeof(dd) * ntarg * nchunks), "malloc");
  CK2(cudaMemcpy(dx, targets, 8 * M, cudaMemcpyHostToDevice), "copy");
  CK2(cudaMemcpy(dy, sources, 8 * N, cudaMemcpyHostToDevice), "copy");
  CK2(cudaMemcpy(da, strengths, 8 * N, cudaMemcpyHostToDevice), "copy");
  if (subset && nsub > 0) {
    CK2(cudaMalloc(&ds, 8 * nsub), "malloc");
    CK2(cudaMemcpy(ds, subset, 8 * nsub, cudaMemcpyHostToDevice), "copy");
  }
  {
    // grid.x limit is 2^31-1: process targets in batches
    const int64_t max_blocks = (int64_t)1 << 30;
    const int64_t tb = max_blocks / nchunks > 0 ? max_blocks / nchunks : 1;
    for (int64_t t0 = 0; t0 < ntarg; t0 += tb) {
      const int64_t nt = ntarg - t0 < tb ? ntarg - t0 : tb;
      direct_partial_kernel<<<(unsigned)(nt * nchunks), kDirThreads>>>(
          ds ? dx : dx + t0, ds ? ds + t0 : nullptr, nt, dy, da, N, q_hi, q_lo, nchunks,
          dpart + t0 * nchunks);
      CK2(cudaGetLastError(), "direct kernel");
    }
    direct_final_kernel<<<(unsigned)((ntarg + 255) / 256), 256>>>(dpart, ntarg, nchunks, dout);
    CK2(cudaGetLastError(), "direct final");
    CK2(cudaMemcpy(out, dout, 8 * ntarg, cudaMemcpyDeviceToHost), "copy out");
  }
done:
  cudaFree(dx);
  cudaFree(dy);
  cudaFree(da);
  cudaFree(dout);
  cudaFree(ds);
  cudaFree(dpart);
#undef CK2
  return rc;
}

int fgt_uniform_points_device(double* out_device, int64_t count, uint64_t seed, uint64_t stream,
                              uint64_t offset, void* cuda_stream) {
  if (count <= 0) return FGT_OK;
  int64_t blocks = (count + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  uniform_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)cuda_stream>>>(out_device, count, seed,
                                                                         stream, offset);
  CKR(cudaGetLastError(), "uniform kernel");
  return FGT_OK;
}

int fgt_gather_device(const double* src, const int32_t* perm, int64_t n, double* out,
                      void* stream) {
  if (n <= 0) return FGT_OK;
  CKR(launch_gather(src, perm, n, out, (cudaStream_t)stream), "gather");
  return FGT_OK;
}

int fgt_scatter_device(const double* src, const int32_t* perm, int64_t n, double* out,
                       void* stream) {
  if (n <= 0) return FGT_OK;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  note_launch();
  scatter_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(src, perm, n, out);
  CKR(cudaGetLastError(), "scatter");
  return FGT_OK;
}

// Stable merge of G sorted runs v[off[r] .. off[r+1]) (host offsets) by a
// tree of pairwise merge-path merges: merged values and the permutation
// (merged[i] == v[perm[i]]), ties in run order -- the order a stable sort of
// the concatenation gives.
int fgt_merge_runs_device(const double* v, const int64_t* off, int G, double* merged,
                          int32_t* perm, void* stream) {
  if (G < 1) {
    g_err = std::string("merge needs at least one run");
    return FGT_ERR_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = off[G];
  if (n <= 0) return FGT_OK;
  std::vector<int64_t> o(off, off + G + 1);
  double* bufv[2] = {nullptr, nullptr};
  int32_t* bufi[2] = {nullptr, nullptr};
  for (int b = 0; b < 2; ++b) {
    CKR(cudaMallocAsync(reinterpret_cast<void**>(&bufv[b]), sizeof(double) * n, st), "merge ws");
    CKR(cudaMallocAsync(reinterpret_cast<void**>(&bufi[b]), sizeof(int32_t) * n, st), "merge ws");
  }
  CKR(cudaMemcpyAsync(bufv[0], v, sizeof(double) * n, cudaMemcpyDeviceToDevice, st), "copy");
  note_launch();
  iota_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(bufi[0], n);
  int cur = 0;
  while (o.size() > 2) {
    std::vector<int64_t> no{0};
    for (size_t r = 0; r + 1 < o.size(); r += 2) {
      const int64_t a0 = o[r], a1 = o[r + 1];
      const int64_t b1 = r + 2 < o.size() ? o[r + 2] : a1;
      const int64_t tot = b1 - a0;
      if (tot > 0) {
        const int64_t threads = (tot + kMergePer - 1) / kMergePer;
        note_launch();
        merge2_kernel<<<(unsigned)((threads + 127) / 128), 128, 0, st>>>(
            bufv[cur] + a0, bufi[cur] + a0, a1 - a0, bufv[cur] + a1, bufi[cur] + a1, b1 - a1,
            bufv[cur ^ 1] + a0, bufi[cur ^ 1] + a0);
      }
      no.push_back(b1);
    }
    o.swap(no);
    cur ^= 1;
  }
  CKR(cudaMemcpyAsync(merged, bufv[cur], sizeof(double) * n, cudaMemcpyDeviceToDevice, st), "copy");
  CKR(cudaMemcpyAsync(perm, bufi[cur], sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st), "copy");
  for (int b = 0; b < 2; ++b) {
    cudaFreeAsync(bufv[b], st);
    cudaFreeAsync(bufi[b], st);
  }
  CKR(cudaGetLastError(), "merge");
  return FGT_OK;
}

int fgt_sort_device(const double* x, int64_t n, double* sorted, int32_t* perm, void* stream) {
  if (n <= 0) return FGT_OK;
  cudaStream_t st = (cudaStream_t)stream;
  void* ws = nullptr;
  CKR(cudaMallocAsync(&ws, radix_sort_workspace_bytes(n), st), "sort workspace");
  cudaError_t e = radix_sort_with_perm(x, n, sorted, perm, ws, st);
  cudaFreeAsync(ws, st);
  CKR(e, "radix sort");
  return FGT_OK;
}

// Gap table of sorted targets, interleaved complex, mode-major:
// out[(k*(M-1) + i)*2 + {0,1}].
int fgt_gap_table_device(const double* d_sorted_targets, int64_t M, int ne, const double* s_re,
                         const double* s_im, double* out_host) {
  if (M < 2 || ne <= 0) return FGT_OK;
  double *dsr = nullptr, *dsi = nullptr;
  double2* dout = nullptr;
  const int64_t n = (M - 1) * ne;
  CKR(cudaMalloc(&dsr, 8 * ne), "malloc");
  CKR(cudaMalloc(&dsi, 8 * ne), "malloc");
  CKR(cudaMalloc(&dout, sizeof(double2) * n), "malloc");
  CKR(cudaMemcpy(dsr, s_re, 8 * ne, cudaMemcpyHostToDevice), "copy");
  CKR(cudaMemcpy(dsi, s_im, 8 * ne, cudaMemcpyHostToDevice), "copy");
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  gap_table_kernel<<<(unsigned)blocks, 256>>>(d_sorted_targets, M, ne, dsr, dsi, dout);
  CKR(cudaGetLastError(), "gap table");
  CKR(cudaMemcpy(out_host, dout, sizeof(double2) * n, cudaMemcpyDeviceToHost), "copy");
  cudaFree(dsr);
  cudaFree(dsi);
  cudaFree(dout);
  return FGT_OK;
}

}  // extern "C"
