// C ABI of the B200 SOE fast Gauss transform (include/fgt1d_b200.h).
//
// Plan / apply orchestration on the device.  Maps to the reference:
//   fgt_plan_create    <- fgt::plan              proj/src/transform.cpp:200-219
//   fgt_plan_gap_table <- precompute_gap_table   proj/src/transform.cpp:221-237
//   fgt_apply_general  <- apply_general          proj/src/transform.cpp:249-253
//   fgt_apply_same     <- apply_same             proj/src/transform.cpp:239-247
//   fgt_direct         <- direct                 proj/src/transform.cpp:255-288
//   fgt_mode_sums      <- detail::mode_sums      proj/src/transform.cpp:310-350
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <cmath>
#include <complex>
#include <memory>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/fgt1d_b200.h"
#include "fgt_scan.cuh"
#include "fgt_soe.hpp"
#include "fgt_sort.cuh"

using namespace fgt_b200;

namespace {
thread_local std::string g_last_error;
}

namespace fgt_b200 {
void set_last_error(const std::string& m) { g_last_error = m; }
}  // namespace fgt_b200

namespace {
std::atomic<long long> g_launch_count{0};
}
namespace fgt_b200 {
void note_launch(int n) { g_launch_count.fetch_add(n); }
}  // namespace fgt_b200

extern "C" int fgt_gap_table_device(const double* d_sorted_targets, int64_t M, int ne,
                                    const double* s_re, const double* s_im, double* out_host);

namespace {

struct ApiError {
  int code;
  std::string msg;
};

[[noreturn]] void raise(int code, const std::string& m) { throw ApiError{code, m}; }

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();  // clear sticky-free errors
    raise(e == cudaErrorMemoryAllocation ? FGT_ERR_NOMEM : FGT_ERR_CUDA,
          std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
  }
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return FGT_OK;
  } catch (const ApiError& e) {
    g_last_error = e.msg;
    return e.code;
  } catch (const SoeError& e) {
    g_last_error = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return FGT_ERR_NOMEM;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return FGT_ERR_CUDA;
  }
}

// Device context guard: a usable device is mandatory (no CPU fallback).
void require_device(int device) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    raise(FGT_ERR_CUDA, "no CUDA device available: the B200 transform has no CPU fallback");
  }
  if (device >= 0) ck(cudaSetDevice(device), "cudaSetDevice");
  // Keep stream-ordered allocations cached across plans/applies instead of
  // returning them to the driver at every synchronization.
  int dev = 0;
  ck(cudaGetDevice(&dev), "cudaGetDevice");
  static std::once_flag once[64];
  if (dev < 64)
    std::call_once(once[dev], [dev] {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
      cudaGetLastError();
    });
}

template <class T>
T* dmalloc(size_t n, cudaStream_t st) {
  if (n == 0) n = 1;
  void* p = nullptr;
  ck(cudaMallocAsync(&p, n * sizeof(T), st), "cudaMallocAsync");
  return static_cast<T*>(p);
}
void dfree(void* p, cudaStream_t st) {
  if (p) cudaFreeAsync(p, st);
}

Soe soe_from_arrays(const double* t_re, const double* t_im, const double* w_re, const double* w_im,
                    const uint8_t* sc, int n, int form) {
  if (n < 0) raise(FGT_ERR_INVALID, "negative SOE size");
  if (n > 0 && (!t_re || !t_im || !w_re || !w_im))
    raise(FGT_ERR_INVALID, "SOE arrays must not be NULL");
  Soe s;
  s.folded = form == FGT_SOE_FOLDED;
  for (int k = 0; k < n; ++k) {
    s.nodes.emplace_back(t_re[k], t_im[k]);
    s.weights.emplace_back(w_re[k], w_im[k]);
    if (s.folded) s.self_conj.push_back(sc ? sc[k] : (t_im[k] == 0.0 ? 1 : 0));
  }
  return s;
}

// Taylor degree thresholds: largest r with r^(D+1)/(D+1)! <= 2^-FGT_TRUNC_BITS.
// A truncated term is then below 2^-FGT_TRUNC_BITS of the exponential it
// replaces; summed over sources and weighted modes the transform error stays
// below 2^-FGT_TRUNC_BITS * sum|m w| * sum|alpha| (sum|m w| = 131 at
// n_e = 6): 2^-52 keeps it 1/35 of the 1e-12 * sum|alpha| parity bar.
#ifndef FGT_TRUNC_BITS
#define FGT_TRUNC_BITS 52
#endif
void fill_rmax(ModeParams& P) {
  long double fact = 1.0L;
  for (int D = 0; D <= kMaxDeg; ++D) {
    fact *= (long double)(D + 1);
    P.rmax[D] =
        (double)powl(fact * ldexpl(1.0L, -FGT_TRUNC_BITS), 1.0L / (long double)(D + 1));
  }
}

// mode_coefs (transform.cpp:47-56): s_k = t_k * (1/sqrt(delta)) exactly as the
// reference forms it, mw_k = m_k w_k; plus the Taylor coefficients of
// exp(-s g) computed in extended precision.
void build_modes(const Soe& folded, double delta, ModeParams& P, ModeTable& T) {
  std::memset(&P, 0, sizeof(P));
  std::memset(&T, 0, sizeof(T));
  const int ne = (int)folded.nodes.size();
  if (ne > kMaxModes)
    raise(FGT_ERR_INVALID, "at most " + std::to_string(kMaxModes) + " folded SOE modes supported");
  P.ne = ne;
  const double isq = 1.0 / std::sqrt(delta);
  double smax = 0.0;
  long double gpoly[kCollDeg + 1] = {};
  long double gl[kMaxDeg + 1] = {};
  for (int k = 0; k < ne; ++k) {
    const double sre = folded.nodes[k].real() * isq;
    const double sim = folded.nodes[k].imag() * isq;
    const std::complex<double> mw = folded.multiplier(k) * folded.weights[k];
    P.s_re[k] = sre;
    P.s_im[k] = sim;
    P.mw_re[k] = mw.real();
    P.mw_im[k] = mw.imag();
    T.s[k] = {sre, sim};
    T.mw[k] = {mw.real(), mw.imag()};
    smax = std::fmax(smax, std::hypot(sre, sim));
    std::complex<long double> c(1.0L, 0.0L);
    const std::complex<long double> ms(-(long double)sre, -(long double)sim);
    const std::complex<long double> lmw((long double)mw.real(), (long double)mw.imag());
    for (int n = 0; n <= kMaxDeg; ++n) {
      T.coef[k][n] = {(double)c.real(), (double)c.imag()};
      gl[n] += (lmw * c).real();
      if (n <= kCollDeg) {
        const std::complex<long double> x = lmw * c;
        T.mwc[k][n] = {(double)x.real(), (double)x.imag()};
        gpoly[n] += x.real();
      }
      c = c * ms / (long double)(n + 1);
    }
  }
  for (int n = 0; n <= kCollDeg; ++n) T.gpoly[n] = (double)gpoly[n];
  for (int n = 0; n <= kMaxDeg; ++n) T.gl[n] = (double)gl[n];
  P.smax = smax;
  T.smax = smax;
  fill_rmax(P);
}

}  // namespace

// Per-chunk persistent state for the two-phase (multi-GPU) apply.
struct ChunkState {
  double* mom = nullptr;           // segment moments between the phases (moment path)
  double* bs = nullptr;            // strengths, sorted-source order (owned copy)
  const double* bs_dev = nullptr;  // or the caller's device strengths (already sorted order)
  cplx* tile = nullptr;            // 5 * ne * ntiles
};

struct fgt_plan_s {
  int device = 0;
  int64_t M = 0, N = 0;
  double delta = 1.0;
  Soe soe;  // folded
  ModeParams P{};
  ModeTable* d_mt = nullptr;
  double* d_xs = nullptr;  // sorted targets
  double* d_ys = nullptr;  // sorted sources
  bool own_xs = true, own_ys = true;
  int32_t* d_tperm = nullptr;  // nullptr: identity
  int32_t* d_sperm = nullptr;
  bool t_sorted = true, s_sorted = true;
  bool same_points = false;
  int64_t ntiles = 0;  // segments of kSeg merged elements
  int64_t* d_tile_ib = nullptr;
  double2* d_seg_z = nullptr;
  int* d_seg_deg = nullptr;      // per segment: packed degrees (classify_kernel)
  uint32_t* d_seg_mask = nullptr;
  unsigned long long* d_cls = nullptr;  // slotted class counts of the fused classification
  // batched plans (fgt_batch_create)
  bool batch = false;
  int nbatch = 0;
  int64_t* d_seg_jb = nullptr;
  int4* d_seg_info = nullptr;
  ModeTable* d_mtb = nullptr;
  // segment classes (launch_classify): K1 / K3 wide-path segment counts
  int64_t nwide1 = -1, nwide3 = -1;
  int dn_narrow = -1;  // highest collapsed degree of the K3-narrow segments
  int dm_narrow = -1;  // highest moment degree of the K1-narrow segments
  CollConsts cc{};     // collapsed-form constants of the plan (single plans)
  double zprev0 = 0.0;
  int* d_flag = nullptr;
  ChunkState cs;
  cudaStream_t stream = nullptr;  // stream the plan was built on (teardown)
  // Applies may run on other streams than the plan's: each such stream's
  // last use is an event the teardown waits on before the memory is reused.
  std::mutex use_mu;
  std::vector<std::pair<cudaStream_t, cudaEvent_t>> uses;
};

namespace {

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- kernel-time profiling hook (bench.py roofline) -------------------------
std::atomic<bool> g_profile{false};
std::mutex g_prof_mu;
struct ProfEv {
  int kind;
  cudaEvent_t a, b;
};
std::vector<ProfEv> g_prof_pending;
double g_prof_ms[8] = {0};
long long g_prof_cnt[8] = {0};

struct ProfScope {
  int kind;
  cudaStream_t st;
  cudaEvent_t a = nullptr, b = nullptr;
  ProfScope(int k, cudaStream_t s) : kind(k), st(s) {
    if (g_profile.load()) {
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, st);
    }
  }
  ~ProfScope() {
    if (a) {
      cudaEventRecord(b, st);
      std::lock_guard<std::mutex> lk(g_prof_mu);
      g_prof_pending.push_back({kind, a, b});
    }
  }
};

// Plan construction: device-resident originals -> all checks in one round
// trip -> borrow / adopt / sort each set.
struct SetSrc {
  const double* dptr = nullptr;  // device copy of the input as given
  bool tmp = false;              // dptr is a temporary we own
};

SetSrc stage_set(const double* src, int64_t n, uint32_t flags, cudaStream_t st) {
  SetSrc r;
  if (n == 0) return r;
  if (flags & FGT_DEVICE_PTRS) {
    r.dptr = src;
    return r;
  }
  double* d = dmalloc<double>(n, st);
  ck(cudaMemcpyAsync(d, src, sizeof(double) * n, cudaMemcpyHostToDevice, st), "upload points");
  r.dptr = d;
  r.tmp = true;
  return r;
}

void adopt_set(const SetSrc& in, int64_t n, bool is_sorted, uint32_t flags, cudaStream_t st,
               double** d_sorted, bool* own, int32_t** d_perm) {
  *d_sorted = nullptr;
  *d_perm = nullptr;
  *own = true;
  if (n == 0) return;
  if (is_sorted) {
    if (in.tmp) {
      *d_sorted = const_cast<double*>(in.dptr);
    } else if (flags & FGT_BORROW) {
      *d_sorted = const_cast<double*>(in.dptr);
      *own = false;
    } else {
      double* d = dmalloc<double>(n, st);
      ck(cudaMemcpyAsync(d, in.dptr, sizeof(double) * n, cudaMemcpyDeviceToDevice, st), "copy");
      *d_sorted = d;
    }
    return;
  }
  double* d_out = dmalloc<double>(n, st);
  int32_t* d_p = dmalloc<int32_t>(n, st);
  void* ws = dmalloc<char>(radix_sort_workspace_bytes(n), st);
  ck(radix_sort_with_perm(in.dptr, n, d_out, d_p, ws, st), "radix sort");
  dfree(ws, st);
  if (in.tmp) dfree(const_cast<double*>(in.dptr), st);
  *d_sorted = d_out;
  *d_perm = d_p;
}

struct PinnedBuf {
  void* p = nullptr;
  explicit PinnedBuf(size_t n) { ck(cudaMallocHost(&p, n), "pinned buffer"); }
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
};

// Both sets unsorted: the two radix sorts run concurrently, the second on a
// side stream, and share one host read of their digit histograms (small
// sorts are launch / latency bound: overlapping them hides most of it).
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  ~SideStream() {
    if (fork) cudaEventDestroy(fork);
    if (join) cudaEventDestroy(join);
    if (s) cudaStreamDestroy(s);
  }
};
SideStream& side_stream() {
  thread_local SideStream ss;
  int dev = 0;
  cudaGetDevice(&dev);
  thread_local int ss_dev = -1;
  if (ss.s && ss_dev != dev) {  // a stream belongs to one device
    cudaEventDestroy(ss.fork);
    cudaEventDestroy(ss.join);
    cudaStreamDestroy(ss.s);
    ss.s = nullptr;
  }
  if (!ss.s) {
    ck(cudaStreamCreateWithFlags(&ss.s, cudaStreamNonBlocking), "side stream");
    ck(cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming), "event");
    ss_dev = dev;
  }
  return ss;
}

void sort_both_sets(const SetSrc& xs, int64_t M, const SetSrc& ys, int64_t N, cudaStream_t st,
                    double** d_xs, int32_t** d_tperm, double** d_ys, int32_t** d_sperm) {
  SideStream& ss = side_stream();
  double* xo = dmalloc<double>(M, st);
  int32_t* xp = dmalloc<int32_t>(M, st);
  void* xw = dmalloc<char>(radix_sort_workspace_bytes(M), st);
  double* yo = dmalloc<double>(N, st);
  int32_t* yp = dmalloc<int32_t>(N, st);
  void* yw = dmalloc<char>(radix_sort_workspace_bytes(N), st);
  ck(cudaEventRecord(ss.fork, st), "fork");
  ck(cudaStreamWaitEvent(ss.s, ss.fork, 0), "fork");
  thread_local std::unique_ptr<PinnedBuf> pin;  // two histograms, pinned (async copies)
  if (!pin) pin.reset(new PinnedBuf(2 * sizeof(unsigned long long) * kSortHistWords));
  unsigned long long* h = static_cast<unsigned long long*>(pin->p);
  ck(radix_sort_begin(xs.dptr, M, xw, h, st), "radix sort");
  ck(radix_sort_begin(ys.dptr, N, yw, h + kSortHistWords, ss.s), "radix sort");
  ck(cudaStreamSynchronize(st), "sort sync");
  ck(cudaStreamSynchronize(ss.s), "sort sync");
  ck(radix_sort_end(xs.dptr, M, xo, xp, xw, h, st), "radix sort");
  ck(radix_sort_end(ys.dptr, N, yo, yp, yw, h + kSortHistWords, ss.s), "radix sort");
  ck(cudaEventRecord(ss.join, ss.s), "join");
  ck(cudaStreamWaitEvent(st, ss.join, 0), "join");
  dfree(xw, st);
  dfree(yw, st);
  if (xs.tmp) dfree(const_cast<double*>(xs.dptr), st);
  if (ys.tmp) dfree(const_cast<double*>(ys.dptr), st);
  *d_xs = xo;
  *d_tperm = xp;
  *d_ys = yo;
  *d_sperm = yp;
}

// Small per-thread pinned buffer for the plan's device -> host reads (flags,
// first coordinates, class counts): async copies into pageable memory would
// synchronise the stream each.  Falls back to nullptr (pageable) if pinned
// allocation fails.
struct PinnedScratch {
  unsigned char* p = nullptr;
  ~PinnedScratch() {
    if (p) cudaFreeHost(p);
  }
};
unsigned char* pinned_scratch() {
  thread_local PinnedScratch s;
  if (!s.p) {
    void* q = nullptr;
    if (cudaMallocHost(&q, 2048) == cudaSuccess) {
      s.p = static_cast<unsigned char*>(q);
    } else {
      cudaGetLastError();
    }
  }
  return s.p;
}

// d_flag: tile-pass check flags 0..4, three 64-bit segment-class counters at
// ints 8..13 (launch_classify), element-wise check flags
// (launch_check_points) at 16..20.
constexpr int kFlagInts = 24;
constexpr int kFullCheck = 16;
unsigned long long* class_counts(fgt_plan_s* p) {
  return reinterpret_cast<unsigned long long*>(p->d_flag + 8);
}

// Packed segment degrees plus, behind them, the plan's count of segments the
// lane-collapsed K3 flagged for the per-mode kernel (seg_fallback_count).
int* alloc_seg_deg(int64_t nseg, cudaStream_t st) {
  int* d = dmalloc<int>(nseg + 2, st);
  ck(cudaMemsetAsync(d + nseg, 0, 2 * sizeof(int), st), "seg_deg tail");
  return d;
}

StreamArgs stream_args(const fgt_plan_s* p, const double* bs) {
  StreamArgs sa{p->d_xs, p->M, p->d_ys, p->N, bs, p->d_tile_ib, p->ntiles, p->zprev0,
                p->d_seg_z, p->d_seg_mask, p->d_seg_info, p->d_seg_jb, p->d_mtb};
  sa.nwide1 = p->nwide1;
  sa.nwide3 = p->nwide3;
  sa.dn_narrow = p->dn_narrow;
  sa.dm_narrow = p->dm_narrow;
  sa.seg_deg = p->d_seg_deg;
  return sa;
}

// Queue the segment classification; the counts land in h[0..1] once the
// stream is synchronized (see take_classes).
// xd / yd: the arrays the segments were cut from (the plan's own sorted
// arrays when null).
void queue_classify(fgt_plan_s* p, unsigned long long* h, cudaStream_t st,
                    bool check_flags = false, bool zprev0_first = false,
                    const double* xd = nullptr, const double* yd = nullptr) {
  StreamArgs sa = stream_args(p, nullptr);
  if (xd) sa.xs = xd;
  if (yd) sa.ys = yd;
  sa.zprev0_first = zprev0_first;
  ck(launch_classify(sa, p->P, p->P.smax, p->d_seg_deg,
                     check_flags ? p->d_flag : nullptr, class_counts(p), st),
     "classify");
  ck(cudaMemcpyAsync(h, class_counts(p), 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                     st),
     "class counts");
}
void take_classes(fgt_plan_s* p, const unsigned long long* h) {
  p->nwide1 = (int64_t)h[0];
  p->nwide3 = (int64_t)h[1];
  p->dn_narrow = (int)h[2] - 1;
  p->dm_narrow = (int)h[3] - 1;
}

// Partition + speculative tile pass (checks and segment metadata) on the
// arrays as given; valid metadata whenever they turn out to be sorted.
// classify: also write the segment degrees and the slotted class counts
// (p->d_cls; p->P must be set), read back by read_classes.
void plan_tiles(fgt_plan_s* p, const double* xd, const double* yd, bool check_sorted,
                cudaStream_t st, bool classify = false, bool has_prev = false,
                double z_prev = 0.0) {
  const int64_t L = p->M + p->N;
  const int64_t ntl = (L + kPlanTile - 1) / kPlanTile;
  if (ntl == 0) return;
  int64_t* tib = dmalloc<int64_t>(ntl + 1, st);
  ck(launch_partition(xd, p->M, yd, p->N, kPlanTile, ntl, tib, st), "partition");
  PlanClassify cls;
  if (classify) {
    if (!p->d_cls) p->d_cls = dmalloc<unsigned long long>(4 * kClassSlots, st);
    cls.enabled = 1;
    cls.P = p->P;
    cls.smax = p->P.smax;
    cls.seg_deg = p->d_seg_deg;
    cls.counts = p->d_cls;
    cls.has_prev = has_prev ? 1 : 0;
    cls.z_prev = z_prev;
  }
  ck(launch_plan_tiles(xd, p->M, yd, p->N, tib, ntl, p->ntiles, check_sorted ? 1 : 0,
                       p->d_tile_ib, p->d_seg_z, p->d_seg_mask, p->d_flag, st, &cls),
     "plan tiles");
  dfree(tib, st);
}

// The fused classification's slotted counts -> host (h: 4 kClassSlots u64,
// pinned), reduced by take_slotted_classes once the stream is synchronized.
void queue_slotted_classes(fgt_plan_s* p, unsigned long long* h, cudaStream_t st) {
  if (!p->d_cls) {  // no tiles (empty sets)
    for (int q = 0; q < 4 * kClassSlots; ++q) h[q] = 0;
    return;
  }
  ck(cudaMemcpyAsync(h, p->d_cls, sizeof(unsigned long long) * 4 * kClassSlots,
                     cudaMemcpyDeviceToHost, st),
     "class counts");
}
void take_slotted_classes(fgt_plan_s* p, const unsigned long long* h) {
  unsigned long long r[4] = {0, 0, 0, 0};
  for (int q = 0; q < kClassSlots; ++q) {
    r[0] += h[4 * q];
    r[1] += h[4 * q + 1];
    r[2] = h[4 * q + 2] > r[2] ? h[4 * q + 2] : r[2];
    r[3] = h[4 * q + 3] > r[3] ? h[4 * q + 3] : r[3];
  }
  take_classes(p, r);
}

// Mode table of a single plan: built on the host, stored by a kernel
// parameter (stream-ordered, no synchronisation).
void upload_modes(fgt_plan_s* p, cudaStream_t st) {
  ModeTable T;
  build_modes(p->soe, p->delta, p->P, T);
  p->cc = coll_consts(T.gpoly);
  p->d_mt = dmalloc<ModeTable>(1, st);
  ck(launch_store_table(T, p->d_mt, st), "store mode table");
}


// Record that work using plan p was queued on stream st (st != the plan's
// stream): destroy_plan orders its frees after it.
void note_use(fgt_plan_s* p, cudaStream_t st) {
  if (st == p->stream) return;
  std::lock_guard<std::mutex> lk(p->use_mu);
  for (auto& u : p->uses)
    if (u.first == st) {
      ck(cudaEventRecord(u.second, st), "record plan use");
      return;
    }
  cudaEvent_t ev = nullptr;
  ck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "plan use event");
  p->uses.emplace_back(st, ev);
  ck(cudaEventRecord(ev, st), "record plan use");
}

// Stream-ordered teardown on the plan's stream: work already queued on it
// that uses the plan, and the last use on every other stream an apply ran
// on, completes before the memory is reused.
void destroy_plan(fgt_plan_s* p) {
  if (!p) return;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(p->device);
  cudaStream_t st = p->stream;
  for (auto& u : p->uses) {
    cudaStreamWaitEvent(st, u.second, 0);
    cudaEventDestroy(u.second);  // released once it has completed
  }
  if (p->own_xs) dfree(p->d_xs, st);
  if (p->own_ys) dfree(p->d_ys, st);
  dfree(p->d_tperm, st);
  dfree(p->d_sperm, st);
  dfree(p->d_tile_ib, st);
  dfree(p->d_seg_z, st);
  dfree(p->d_seg_deg, st);
  dfree(p->d_seg_mask, st);
  dfree(p->d_cls, st);
  dfree(p->d_seg_jb, st);
  dfree(p->d_seg_info, st);
  dfree(p->d_mtb, st);
  dfree(p->d_mt, st);
  dfree(p->d_flag, st);
  dfree(p->cs.bs, st);
  dfree(p->cs.mom, st);
  dfree(p->cs.tile, st);
  cudaGetLastError();
  cudaSetDevice(cur);
  delete p;
}

Soe resolve_soe(const double* t_re, const double* t_im, const double* w_re, const double* w_im,
                const uint8_t* sc, int n_modes, int form) {
  Soe s = soe_from_arrays(t_re, t_im, w_re, w_im, sc, n_modes, form);
  soe_validate(s);
  return soe_fold(s);
}

void check_delta(double delta) {
  if (!std::isfinite(delta) || !(delta > 0.0))
    raise(FGT_ERR_DOMAIN, "delta must be positive and finite");
}

// Per-apply device workspace, stream ordered.
struct Work {
  cudaStream_t st;
  std::vector<void*> ptrs;
  template <class T>
  T* get(size_t n) {
    T* p = dmalloc<T>(n, st);
    ptrs.push_back(p);
    return p;
  }
  ~Work() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
};

// Strengths in sorted-source order (upload + gather as needed).
const double* sorted_strengths(fgt_plan_s* p, const double* strengths, uint32_t flags, Work& w,
                               double* into) {
  const bool dev = flags & FGT_DEVICE_PTRS;
  const double* alpha = strengths;
  if (p->N == 0) return alpha;
  if (!dev) {
    double* d = (p->d_sperm || !into) ? w.get<double>(p->N) : into;
    ck(cudaMemcpyAsync(d, strengths, sizeof(double) * p->N, cudaMemcpyHostToDevice, w.st),
       "upload strengths");
    alpha = d;
  }
  if (p->d_sperm) {
    double* g = into ? into : w.get<double>(p->N);
    ck(launch_gather(alpha, p->d_sperm, p->N, g, w.st), "gather strengths");
    return g;
  }
  if (into && alpha != into)
    ck(cudaMemcpyAsync(into, alpha, sizeof(double) * p->N, cudaMemcpyDeviceToDevice, w.st), "copy");
  return into ? into : alpha;
}


// apply_general / apply_same: K1 aggregates -> K2 carries -> K3 main.
void run_apply(fgt_plan_s* p, const double* strengths, double* potentials, uint32_t flags,
               cudaStream_t st) {
  ck(cudaSetDevice(p->device), "cudaSetDevice");
  const bool dev = flags & FGT_DEVICE_PTRS;
  if (p->M == 0) return;
  Work w{st, {}};
  double* u = dev ? potentials : w.get<double>(p->M);
  if (p->N == 0) {
    ck(cudaMemsetAsync(u, 0, sizeof(double) * p->M, st), "zero potentials");
  } else {
    const double* bs = sorted_strengths(p, strengths, flags, w, nullptr);
    const StreamArgs sa = stream_args(p, bs);
    const TileState ts = tile_state_carve(w.get<cplx>(tile_state_elems(p->ntiles, p->P.ne)),
                                          p->ntiles, p->P.ne);
    OutArgs o;
    o.u = u;
    o.tperm = p->d_tperm;
    if (!p->batch) {
      // moment path: K1m -> K2m (collapsed carries) -> K3
      double* mom = w.get<double>((size_t)p->ntiles * k1m_moments(sa));
      {
        ProfScope ps(0, st);
        ck(launch_moments(sa, p->P, p->d_mt, ts, mom, st), "segment moments");
      }
      {
        ProfScope ps(1, st);
        ck(launch_mom_scan(sa, p->P.ne, p->d_mt, ts, mom, nullptr, nullptr, st, true, true, &p->cc),
           "carry scan");
      }
      {
        ProfScope ps(2, st);
        ck(launch_main(sa, p->P, p->d_mt, ts, o, st, &p->cc, true, k3_folds(sa)), "main pass");
      }
    } else {
      {
        ProfScope ps(0, st);
        ck(launch_aggregate(sa, p->P, p->d_mt, ts, st), "tile aggregates");
      }
      {
        ProfScope ps(1, st);
        ck(launch_carry_scan(ts, p->ntiles, p->P.ne, nullptr, nullptr, st), "carry scan");
      }
      {
        ProfScope ps(2, st);
        ck(launch_main(sa, p->P, p->d_mt, ts, o, st), "main pass");
      }
    }
  }
  note_use(p, st);
  if (!dev) {
    ck(cudaMemcpyAsync(potentials, u, sizeof(double) * p->M, cudaMemcpyDeviceToHost, st),
       "download potentials");
    ck(cudaStreamSynchronize(st), "apply sync");
  }
}

// Two-phase chunk apply.  Phase 1 keeps the sorted strengths and the tile
// aggregates in the plan so phase 2 only runs the carry scan and K3.
void run_chunk_aggregate(fgt_plan_s* p, const double* strengths, cplx* totals_out,
                         uint32_t flags, cudaStream_t st) {
  const bool dev_aggs = flags & FGT_DEVICE_AGGS;
  ck(cudaSetDevice(p->device), "cudaSetDevice");
  const int ne = p->P.ne;
  Work w{st, {}};
  if (!p->cs.tile) p->cs.tile = dmalloc<cplx>(tile_state_elems(p->ntiles, ne), p->stream);
  // device strengths of presorted sources are used in place (the caller
  // passes them again to phase 2); otherwise the plan keeps a sorted copy
  const bool borrow = (flags & FGT_DEVICE_PTRS) && !p->d_sperm;
  if (!borrow && !p->cs.bs && p->N) p->cs.bs = dmalloc<double>(p->N, p->stream);
  if (st != p->stream) ck(cudaStreamSynchronize(p->stream), "sync");
  if (borrow)
    p->cs.bs_dev = strengths;
  else
    sorted_strengths(p, strengths, flags, w, p->cs.bs);
  const double* bs = borrow ? strengths : p->cs.bs;
  if (p->ntiles == 0) {
    std::vector<cplx> id(3 * ne, cplx{0.0, 0.0});
    for (int k = 0; k < ne; ++k) id[k] = {1.0, 0.0};
    if (dev_aggs) {
      ck(cudaMemcpyAsync(totals_out, id.data(), sizeof(cplx) * 3 * ne, cudaMemcpyHostToDevice, st),
         "identity aggregates");
    } else {
      std::memcpy(totals_out, id.data(), sizeof(cplx) * 3 * ne);
    }
    ck(cudaStreamSynchronize(st), "sync");
    return;
  }
  const StreamArgs sa = stream_args(p, bs);
  const TileState ts = tile_state_carve(p->cs.tile, p->ntiles, ne);
  if (!p->cs.mom) p->cs.mom = dmalloc<double>((size_t)p->ntiles * k1m_moments(sa), st);
  {
    ProfScope ps(0, st);
    ck(launch_moments(sa, p->P, p->d_mt, ts, p->cs.mom, st), "segment moments");
  }
  cplx* d_tot = dev_aggs ? totals_out : w.get<cplx>(3 * ne);
  {
    // block reduce + top level only: phase 2's down-sweep writes the carries
    ProfScope ps(1, st);
    ck(launch_mom_scan(sa, ne, p->d_mt, ts, p->cs.mom, nullptr, d_tot, st, true, false),
       "chunk totals");
  }
  note_use(p, st);
  if (dev_aggs) return;  // stream-ordered: the caller gathers the device totals
  ck(cudaMemcpyAsync(totals_out, d_tot, sizeof(cplx) * 3 * ne, cudaMemcpyDeviceToHost, st),
     "totals");
  ck(cudaStreamSynchronize(st), "sync");
}

void run_chunk_finish(fgt_plan_s* p, const double* strengths, const cplx* carry_in,
                      double* potentials, uint32_t flags, cudaStream_t st) {
  const bool dev_aggs = flags & FGT_DEVICE_AGGS;
  ck(cudaSetDevice(p->device), "cudaSetDevice");
  if (p->M == 0) return;
  const bool dev = flags & FGT_DEVICE_PTRS;
  const int ne = p->P.ne;
  Work w{st, {}};
  double* u = dev ? potentials : w.get<double>(p->M);
  if (p->N == 0 && p->ntiles > 0 && !p->cs.tile)
    raise(FGT_ERR_INVALID, "fgt_apply_chunk_finish before fgt_apply_chunk_aggregate");
  if (!p->cs.tile) raise(FGT_ERR_INVALID, "fgt_apply_chunk_finish before fgt_apply_chunk_aggregate");
  if (p->cs.bs_dev && p->cs.bs_dev != strengths)
    raise(FGT_ERR_INVALID, "fgt_apply_chunk_finish: pass the strengths given to phase 1");
  const StreamArgs sa = stream_args(p, p->cs.bs_dev ? p->cs.bs_dev : p->cs.bs);
  const TileState ts = tile_state_carve(p->cs.tile, p->ntiles, ne);
  const cplx* d_cin = carry_in;
  if (!dev_aggs) {
    cplx* d = w.get<cplx>(2 * ne);
    ck(cudaMemcpyAsync(d, carry_in, sizeof(cplx) * 2 * ne, cudaMemcpyHostToDevice, st),
       "carry in");
    d_cin = d;
  }
  {
    ProfScope ps(1, st);
    // phase 1's block aggregates are still in the tile state: top + down only
    ck(launch_mom_scan(sa, ne, p->d_mt, ts, p->cs.mom, d_cin, nullptr, st, false, true, &p->cc),
       "carry scan");
  }
  OutArgs o;
  o.u = u;
  o.tperm = p->d_tperm;
  {
    ProfScope ps(2, st);
    ck(launch_main(sa, p->P, p->d_mt, ts, o, st, &p->cc, true, k3_folds(sa)), "main pass");
  }
  note_use(p, st);
  if (!dev) {
    ck(cudaMemcpyAsync(potentials, u, sizeof(double) * p->M, cudaMemcpyDeviceToHost, st),
       "download potentials");
  }
  // a host carry_in was staged through pageable memory: complete before return
  if (!dev_aggs || !dev) ck(cudaStreamSynchronize(st), "sync");
}

// ------------------------------------------------ pipelined host transform
//
// One-shot transform from host buffers with the PCIe copies overlapped.  A
// plan-then-apply call must upload x, y, alpha and download u back to back
// (57 ms of link time at N = M = 1e8); here the sources go first, the
// targets follow in G chunks, and each chunk's potentials download while
// the next chunk's targets upload (the link is full duplex), so the
// download hides behind the target upload.  This works because a chunk's
// aggregates (A, F, G of the merged-stream chunk) depend on its
// sources and its two boundary coordinates only: they are computed from
// source-only chunk plans while the targets are still in flight, the
// carries follow with the multi-GPU chunk algebra (fgt_chunk_carries), and
// every target chunk is planned and finished as soon as it lands.  Chunk
// boundaries are merge-path splits of the host arrays.
//
// The device work is queued without host round trips (a small device ->
// host copy on the compute stream would queue behind the multi-megabyte
// potential downloads on the copy engine): the chunk plans' checks land in
// one flag array read once per phase, and the kernel variants of both
// segment classes run (each skips the other's segments).  Sortedness and
// finiteness are checked on the device (chunk tile passes) and at the chunk
// boundaries on the host; any violation drops to the full plan / apply path
// on the already uploaded arrays, which sorts, reports errors and returns
// the reference's results and exceptions.

int64_t merge_split_host(const double* x, int64_t M, const double* y, int64_t N, int64_t d) {
  // targets among the first d merged elements (sources first on ties)
  int64_t lo = d - N > 0 ? d - N : 0, hi = d < M ? d : M;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) / 2;
    if (x[mid - 1] < y[d - mid])
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

// decay_factor (transform.cpp:60-68) on the host: 1 at d = 0, exactly 0 past
// the underflow exponent.
std::complex<double> host_decay(double sre, double sim, double d) {
  if (d == 0.0) return {1.0, 0.0};
  if (sre * d > 745.0) return {0.0, 0.0};
  return std::exp(std::complex<double>(-sre * d, -sim * d));
}

// Pipeline sizes: merged points below which one plan / apply is used, and
// merged points per chunk.  The environment variables FGT_PIPE_MIN /
// FGT_PIPE_CHUNK override them (test hook: many small chunks).
int64_t pipe_knob(const char* name, int64_t dflt) {
  const char* v = std::getenv(name);
  if (!v || !*v) return dflt;
  const long long n = std::atoll(v);
  return n > 0 ? (int64_t)n : dflt;
}

// Chunk plan over device slices, queued on st with no host round trip: the
// checks (sortedness of each slice included) land in flag[0..7], segment
// classes stay unknown.  The caller owns flag.
fgt_plan_s* pipe_chunk_plan(const double* dx, int64_t M, const double* dy, int64_t N,
                            const Soe& soe, double delta, const ModeTable& T, const ModeParams& P,
                            double zprev, int* flag, cudaStream_t st) {
  fgt_plan_s* p = new fgt_plan_s();
  try {
    ck(cudaGetDevice(&p->device), "cudaGetDevice");
    p->M = M;
    p->N = N;
    p->soe = soe;
    p->P = P;
    p->delta = delta;
    p->stream = st;
    p->ntiles = (M + N + kSeg - 1) / kSeg;
    p->d_tile_ib = dmalloc<int64_t>(p->ntiles + 1, st);
    p->d_seg_z = dmalloc<double2>(p->ntiles, st);
    p->d_seg_deg = alloc_seg_deg(p->ntiles, st);
    p->d_seg_mask = dmalloc<uint32_t>(seg_mask_words(p->ntiles), st);
    p->d_xs = const_cast<double*>(dx);
    p->d_ys = const_cast<double*>(dy);
    p->own_xs = p->own_ys = false;
    p->d_flag = flag;
    plan_tiles(p, dx, dy, true, st);
    p->d_mt = dmalloc<ModeTable>(1, st);
    ck(launch_store_table(T, p->d_mt, st), "store mode table");
    p->cc = coll_consts(T.gpoly);
    p->zprev0 = zprev;
    const StreamArgs sa = stream_args(p, nullptr);
    ck(launch_classify(sa, p->P, p->P.smax, p->d_seg_deg, nullptr,
                       class_counts(p), st),
       "classify");
    p->nwide1 = p->nwide3 = -1;
  } catch (...) {
    p->d_flag = nullptr;
    destroy_plan(p);
    throw;
  }
  return p;
}
void pipe_chunk_destroy(fgt_plan_s* p) {
  p->d_flag = nullptr;  // owned by the pipeline
  destroy_plan(p);
}

struct PipeChunk {
  int64_t i0, i1, j0, j1;
  double zprev, zlast;
};

struct PipeStreams {
  cudaStream_t in = nullptr, out = nullptr;
  std::vector<cudaEvent_t> ev;
  cudaEvent_t event() {
    cudaEvent_t e;
    ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    ev.push_back(e);
    return e;
  }
  ~PipeStreams() {
    if (in) cudaStreamSynchronize(in);
    if (out) cudaStreamSynchronize(out);
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    if (in) cudaStreamDestroy(in);
    if (out) cudaStreamDestroy(out);
  }
};


// Plan / apply (host or device pointers per flags) for the small and the
// fallback cases.
void plan_apply(const double* x, int64_t M, const double* y, int64_t N, const double* a,
                double* u, double delta, const Soe& soe, uint32_t flags, cudaStream_t st) {
  std::vector<double> tr, ti, wr, wi;
  std::vector<uint8_t> sc;
  for (size_t k = 0; k < soe.nodes.size(); ++k) {
    tr.push_back(soe.nodes[k].real());
    ti.push_back(soe.nodes[k].imag());
    wr.push_back(soe.weights[k].real());
    wi.push_back(soe.weights[k].imag());
    sc.push_back(soe.self_conj[k]);
  }
  fgt_plan_t p = nullptr;
  int rc = fgt_plan_create(x, M, y, N, delta, tr.data(), ti.data(), wr.data(), wi.data(),
                           sc.data(), (int)tr.size(), FGT_SOE_FOLDED, flags, -1, st, &p);
  if (rc != FGT_OK) raise(rc, g_last_error);
  rc = fgt_apply_general(p, a, N, u, 1, flags, st);
  fgt_plan_destroy(p);
  if (rc != FGT_OK) raise(rc, g_last_error);
}

void transform_host(const double* x, int64_t M, const double* y, int64_t N, const double* alpha,
                    double* u, double delta, const Soe& soe, cudaStream_t st) {
  if (M == 0) return;
  const int64_t L = M + N;
  if (N == 0 || L < pipe_knob("FGT_PIPE_MIN", (int64_t)1 << 22)) {
    plan_apply(x, M, y, N, alpha, u, delta, soe, 0, st);
    return;
  }
  // chunks of the merged stream (merge path on the host arrays; validated below)
  // chunk: about L / 4 merged points, within [2.5M, 12.5M] (measured: fewer,
  // larger chunks leave a long last-chunk tail; smaller ones cost per-chunk
  // plan overhead)
  int64_t dflt = L / 4;
  dflt = dflt < 2500000 ? 2500000 : (dflt > 12500000 ? 12500000 : dflt);
  int64_t G = L / pipe_knob("FGT_PIPE_CHUNK", dflt);
  G = G < 2 ? 2 : (G > 64 ? 64 : G);
  std::vector<PipeChunk> ch(G);
  bool ok = true;
  int64_t ip = 0;
  for (int64_t g = 0; g < G; ++g) {
    const int64_t d0 = L * g / G, d1 = L * (g + 1) / G;
    const int64_t i1 = g + 1 == G ? M : merge_split_host(x, M, y, N, d1);
    PipeChunk& c = ch[g];
    c.i0 = ip;
    c.i1 = i1;
    c.j0 = d0 - ip;
    c.j1 = d1 - i1;
    ok = ok && c.i1 >= c.i0 && c.j1 >= c.j0;
    ip = i1;
  }
  if (ok) {
    // merged element before the chunk / the chunk's last one: the larger of
    // the last target and the last source so far (sorted prefixes)
    auto last = [&](int64_t i, int64_t j) {
      const double a = i > 0 ? x[i - 1] : -INFINITY, b = j > 0 ? y[j - 1] : -INFINITY;
      return a > b ? a : b;
    };
    for (int64_t g = 0; g < G; ++g) {
      PipeChunk& c = ch[g];
      // boundary order between chunks (each chunk's inside is checked on the device)
      if (c.i0 > 0 && c.i0 < M) ok = ok && x[c.i0 - 1] <= x[c.i0];
      if (c.j0 > 0 && c.j0 < N) ok = ok && y[c.j0 - 1] <= y[c.j0];
      c.zprev = g == 0 ? std::fmin(x[0], y[0]) : last(c.i0, c.j0);
      c.zlast = last(c.i1, c.j1);
    }
  }
  const int ne = (int)soe.nodes.size();
  ModeParams P;
  ModeTable T;
  build_modes(soe, delta, P, T);
  // FGT_PIPE_TRACE=1: host timestamps of the phases and device arrival
  // times of the target chunks on stderr
  const bool trace = pipe_knob("FGT_PIPE_TRACE", 0) != 0;
  const auto t0 = std::chrono::steady_clock::now();
  auto stamp = [&](const char* what) {
    if (trace)
      std::fprintf(stderr, "pipe %-24s %8.3f ms\n", what,
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                       .count());
  };

  double* dx = dmalloc<double>(M, st);
  double* dy = dmalloc<double>(N, st);
  double* da = dmalloc<double>(N, st);
  double* du = dmalloc<double>(M, st);
  int* dflag = dmalloc<int>((size_t)2 * G * kFlagInts, st);
  cplx* d_agg = dmalloc<cplx>((size_t)G * 3 * ne, st);
  cplx* d_car = dmalloc<cplx>((size_t)G * 2 * ne, st);
  struct Free {
    cudaStream_t st;
    std::vector<void*> p;
    ~Free() {
      for (void* q : p) cudaFreeAsync(q, st);
      cudaStreamSynchronize(st);
    }
  } fr{st, {dx, dy, da, du, dflag, d_agg, d_car}};
  ck(cudaMemsetAsync(dflag, 0, sizeof(int) * 2 * G * kFlagInts, st), "flags");
  PipeStreams ps;
  ck(cudaStreamCreateWithFlags(&ps.in, cudaStreamNonBlocking), "stream");
  ck(cudaStreamCreateWithFlags(&ps.out, cudaStreamNonBlocking), "stream");
  // the buffers were allocated on st: the copy streams start after that
  cudaEvent_t ready = ps.event();
  ck(cudaEventRecord(ready, st), "event");
  ck(cudaStreamWaitEvent(ps.in, ready, 0), "wait");
  auto h2d = [&](double* d, const double* h, int64_t n) {
    if (n > 0)
      ck(cudaMemcpyAsync(d, h, sizeof(double) * n, cudaMemcpyHostToDevice, ps.in), "upload");
  };
  // the full path on the uploaded arrays: sorts, checks, reference errors
  auto fallback = [&]() {
    ck(cudaStreamSynchronize(ps.in), "upload sync");
    ck(cudaStreamSynchronize(ps.out), "download sync");
    ck(cudaStreamSynchronize(st), "sync");
    plan_apply(dx, M, dy, N, da, du, delta, soe, FGT_DEVICE_PTRS, st);
    ck(cudaMemcpyAsync(u, du, sizeof(double) * M, cudaMemcpyDeviceToHost, st), "download");
    ck(cudaStreamSynchronize(st), "download sync");
  };
  if (!ok) {  // not sorted (or NaN at a split)
    h2d(dx, x, M);
    h2d(dy, y, N);
    h2d(da, alpha, N);
    return fallback();
  }
  // every upload is queued up front: sources by chunk, then targets by chunk
  std::vector<cudaEvent_t> ev_src(G), ev_tgt(G);
  for (int64_t g = 0; g < G; ++g) {
    h2d(dy + ch[g].j0, y + ch[g].j0, ch[g].j1 - ch[g].j0);
    h2d(da + ch[g].j0, alpha + ch[g].j0, ch[g].j1 - ch[g].j0);
    ev_src[g] = ps.event();
    ck(cudaEventRecord(ev_src[g], ps.in), "event");
  }
  std::vector<cudaEvent_t> tev;  // trace: timing events on the copy streams
  auto tmark = [&](cudaStream_t s) {
    if (!trace) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    tev.push_back(e);
  };
  tmark(ps.in);
  for (int64_t g = 0; g < G; ++g) {
    h2d(dx + ch[g].i0, x + ch[g].i0, ch[g].i1 - ch[g].i0);
    ev_tgt[g] = ps.event();
    ck(cudaEventRecord(ev_tgt[g], ps.in), "event");
  }
  tmark(ps.in);
  stamp("uploads queued");
  PinnedBuf pin(sizeof(cplx) * (size_t)G * 5 * ne + sizeof(int) * 2 * G * kFlagInts);
  cplx* h_agg = static_cast<cplx*>(pin.p);   // [G][3 ne]: A', F', G' (source span)
  cplx* h_car = h_agg + (size_t)G * 3 * ne;  // [G][2 ne]: carries
  int* h_flag = reinterpret_cast<int*>(h_car + (size_t)G * 2 * ne);
  auto flags_bad = [&](int64_t g0, int64_t g1) {
    for (int64_t g = g0; g < g1; ++g) {
      const int* f = h_flag + g * kFlagInts;
      if (f[0] || f[1] || f[3] || f[4]) return true;
    }
    return false;
  };
  // phase 1: aggregates of every chunk from its sources alone
  for (int64_t g = 0; g < G; ++g) {
    const PipeChunk& c = ch[g];
    const int64_t Ng = c.j1 - c.j0;
    if (!Ng) continue;
    ck(cudaStreamWaitEvent(st, ev_src[g], 0), "wait");
    fgt_plan_s* p = pipe_chunk_plan(dx, 0, dy + c.j0, Ng, soe, delta, T, P, c.zprev,
                                    dflag + g * kFlagInts, st);
    {
      Work w{st, {}};
      const StreamArgs sa = stream_args(p, da + c.j0);
      const TileState ts =
          tile_state_carve(w.get<cplx>(tile_state_elems(p->ntiles, ne)), p->ntiles, ne);
      ck(launch_aggregate(sa, P, p->d_mt, ts, st), "chunk aggregates");
      ck(launch_carry_scan(ts, p->ntiles, ne, nullptr, d_agg + g * 3 * ne, st), "chunk totals");
    }
    pipe_chunk_destroy(p);
  }
  ck(cudaMemcpyAsync(h_agg, d_agg, sizeof(cplx) * G * 3 * ne, cudaMemcpyDeviceToHost, st),
     "aggregates");
  ck(cudaMemcpyAsync(h_flag, dflag, sizeof(int) * G * kFlagInts, cudaMemcpyDeviceToHost, st),
     "flags");
  ck(cudaStreamSynchronize(st), "aggregates sync");
  stamp("sources + aggregates");
  if (flags_bad(0, G)) return fallback();
  // extend each source span to the chunk's last merged element, then the
  // carry algebra of the multi-GPU path
  std::vector<double> aggs((size_t)G * 6 * ne);
  using C = std::complex<double>;
  C* A = reinterpret_cast<C*>(aggs.data());
  for (int64_t g = 0; g < G; ++g) {
    const PipeChunk& c = ch[g];
    const bool src = c.j1 > c.j0;
    const double ylast = src ? y[c.j1 - 1] : c.zprev;
    for (int k = 0; k < ne; ++k) {
      const C e = host_decay(P.s_re[k], P.s_im[k], c.zlast - ylast);
      C a1(1.0, 0.0), f1(0.0, 0.0), g1(0.0, 0.0);
      if (src) {
        const cplx* h = h_agg + g * 3 * ne;
        a1 = C(h[k].re, h[k].im);
        f1 = C(h[ne + k].re, h[ne + k].im);
        g1 = C(h[2 * ne + k].re, h[2 * ne + k].im);
      }
      A[g * 3 * ne + k] = a1 * e;
      A[g * 3 * ne + ne + k] = f1 * e;
      A[g * 3 * ne + 2 * ne + k] = g1;
    }
  }
  {
    const int rc = fgt_chunk_carries(aggs.data(), (int)G, ne, reinterpret_cast<double*>(h_car));
    if (rc != FGT_OK) raise(rc, g_last_error);
  }
  ck(cudaMemcpyAsync(d_car, h_car, sizeof(cplx) * G * 2 * ne, cudaMemcpyHostToDevice, st), "carries");
  // phase 2: every target chunk is planned and finished as it lands; its
  // potentials download on the out stream while the next chunk uploads
  int* dflag2 = dflag + G * kFlagInts;
  for (int64_t g = 0; g < G; ++g) {
    const PipeChunk& c = ch[g];
    const int64_t Mg = c.i1 - c.i0, Ng = c.j1 - c.j0;
    if (!Mg) continue;
    ck(cudaStreamWaitEvent(st, ev_tgt[g], 0), "wait");
    fgt_plan_s* p = pipe_chunk_plan(dx + c.i0, Mg, dy + c.j0, Ng, soe, delta, T, P, c.zprev,
                                    dflag2 + g * kFlagInts, st);
    {
      Work w{st, {}};
      const StreamArgs sa = stream_args(p, Ng ? da + c.j0 : da);
      const TileState ts =
          tile_state_carve(w.get<cplx>(tile_state_elems(p->ntiles, ne)), p->ntiles, ne);
      ck(launch_aggregate(sa, P, p->d_mt, ts, st), "tile aggregates");
      ck(launch_carry_scan(ts, p->ntiles, ne, d_car + g * 2 * ne, nullptr, st), "carry scan");
      OutArgs o;
      o.u = du + c.i0;
      ck(launch_main(sa, P, p->d_mt, ts, o, st, &p->cc), "main pass");
    }
    pipe_chunk_destroy(p);
    cudaEvent_t done = ps.event();
    ck(cudaEventRecord(done, st), "event");
    ck(cudaStreamWaitEvent(ps.out, done, 0), "wait");
    if (g == 0) tmark(ps.out);
    ck(cudaMemcpyAsync(u + c.i0, du + c.i0, sizeof(double) * Mg, cudaMemcpyDeviceToHost, ps.out),
       "download");
  }
  tmark(ps.out);
  stamp("phase 2 queued");
  ck(cudaMemcpyAsync(h_flag + G * kFlagInts, dflag2, sizeof(int) * G * kFlagInts,
                     cudaMemcpyDeviceToHost, st),
     "flags");
  ck(cudaStreamSynchronize(st), "sync");
  if (flags_bad(G, 2 * G)) return fallback();
  ck(cudaStreamSynchronize(ps.out), "download sync");
  stamp("downloads done");
  if (trace && tev.size() == 4) {
    float a = 0.f, b = 0.f, c = 0.f;
    cudaEventElapsedTime(&a, tev[0], tev[1]);
    cudaEventElapsedTime(&b, tev[0], tev[2]);
    cudaEventElapsedTime(&c, tev[0], tev[3]);
    std::fprintf(stderr, "pipe device: targets uploaded %.3f, first download start %.3f, "
                 "downloads done %.3f ms after the sources\n", a, b, c);
  }
  for (cudaEvent_t e : tev) cudaEventDestroy(e);
}

}  // namespace

// ======================================================================= C

extern "C" {

const char* fgt_last_error(void) { return g_last_error.c_str(); }

int fgt_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int fgt_cf_soe(int n, int folded, double* t_re, double* t_im, double* w_re, double* w_im,
               uint8_t* self_conj) {
  int count = 0;
  int rc = guarded([&] {
    Soe s = soe_cf(n);
    if (folded) s = soe_fold(s);
    count = (int)s.nodes.size();
    for (int k = 0; k < count; ++k) {
      if (t_re) t_re[k] = s.nodes[k].real();
      if (t_im) t_im[k] = s.nodes[k].imag();
      if (w_re) w_re[k] = s.weights[k].real();
      if (w_im) w_im[k] = s.weights[k].imag();
      if (self_conj) self_conj[k] = s.folded ? s.self_conj[k] : 0;
    }
  });
  return rc == FGT_OK ? count : -rc;
}

int fgt_preset_mode_count(int p) {
  switch (p) {  // transform.cpp:290-302
    case 0: return 3;
    case 1: return 4;
    case 2: return 5;
    case 3: return 6;
    default:
      g_last_error = "unknown precision preset";
      return -FGT_ERR_DOMAIN;
  }
}

int fgt_mode_count_for_tolerance(double tol) {
  // proj/README.md:184-189 documented transform errors per preset
  if (!(tol > 0.0) || !std::isfinite(tol)) {
    g_last_error = "tolerance must be positive and finite";
    return -FGT_ERR_DOMAIN;
  }
  if (tol >= 1e-3) return 3;
  if (tol >= 1e-6) return 4;
  if (tol >= 1e-8) return 5;
  if (tol >= 1e-10) return 6;
  if (tol >= 1e-11) return 7;
  g_last_error = "tolerance below the reach of the double-precision CF tables";
  return -FGT_ERR_DOMAIN;
}

}  // extern "C"

namespace {
// fgt_plan_create; has_prev: a chunk plan whose stream continues after z_prev
// (segment 0 is framed from z_prev, classified in the same round trip)
int plan_create_impl(const double* targets, int64_t M, const double* sources, int64_t N,
                     double delta, const double* t_re, const double* t_im, const double* w_re,
                     const double* w_im, const uint8_t* self_conj, int n_modes, int form,
                     uint32_t flags, int device, void* stream, fgt_plan_t* out, bool has_prev,
                     double z_prev) {
  return guarded([&] {
    if (!out) raise(FGT_ERR_INVALID, "out must not be NULL");
    *out = nullptr;
    if (M < 0 || N < 0) raise(FGT_ERR_INVALID, "negative point count");
    check_delta(delta);
    Soe soe = resolve_soe(t_re, t_im, w_re, w_im, self_conj, n_modes, form);
    require_device(device);
    cudaStream_t st = as_stream(stream);
    fgt_plan_s* p = new fgt_plan_s();
    std::vector<void*> temps;
    try {
      ck(cudaGetDevice(&p->device), "cudaGetDevice");
      p->M = M;
      p->N = N;
      p->delta = delta;
      p->soe = soe;
      if (M >= ((int64_t)1 << 31) || N >= ((int64_t)1 << 31))
        raise(FGT_ERR_INVALID, "at most 2^31-1 points per set");
      p->stream = st;
      p->d_flag = dmalloc<int>(kFlagInts, st);
      ck(cudaMemsetAsync(p->d_flag, 0, sizeof(int) * kFlagInts, st), "flag");
      SetSrc xs = stage_set(targets, M, flags, st);
      if (xs.tmp) temps.push_back((void*)xs.dptr);
      SetSrc ys = stage_set(sources, N, flags, st);
      if (ys.tmp) temps.push_back((void*)ys.dptr);
      const int64_t L = M + N;
      p->ntiles = (L + kSeg - 1) / kSeg;
      p->d_tile_ib = dmalloc<int64_t>(p->ntiles + 1, st);
      p->d_seg_z = dmalloc<double2>(p->ntiles, st);
        p->d_seg_deg = alloc_seg_deg(p->ntiles, st);
      p->d_seg_mask = dmalloc<uint32_t>(seg_mask_words(p->ntiles), st);
      upload_modes(p, st);
      // one read of both sets: checks + (speculative) segment metadata and
      // classification (valid when both sets are sorted: segment 0 starts at
      // its own first element, or after z_prev); flags, first coordinates
      // and class counts in one round trip (pinned scratch)
      plan_tiles(p, xs.dptr, ys.dptr, !(flags & FGT_ASSUME_SORTED), st, true, has_prev, z_prev);
      unsigned char* pin = pinned_scratch();
      int hfl[8] = {0};
      double xyl[2] = {0.0, 0.0};
      std::vector<unsigned long long> hcl(4 * kClassSlots, 0);
      int* hf = pin ? reinterpret_cast<int*>(pin) : hfl;
      double* xy0 = pin ? reinterpret_cast<double*>(pin + 32) : xyl;
      unsigned long long* hc = pin ? reinterpret_cast<unsigned long long*>(pin + 128) : hcl.data();
      xy0[0] = xy0[1] = 0.0;
      if (has_prev) p->zprev0 = z_prev;
      queue_slotted_classes(p, hc, st);
      ck(cudaMemcpyAsync(hf, p->d_flag, sizeof(int) * 8, cudaMemcpyDeviceToHost, st), "flags");
      if (M > 0) ck(cudaMemcpyAsync(xy0, xs.dptr, 8, cudaMemcpyDeviceToHost, st), "x0");
      if (N > 0) ck(cudaMemcpyAsync(xy0 + 1, ys.dptr, 8, cudaMemcpyDeviceToHost, st), "y0");
      ck(cudaStreamSynchronize(st), "flags sync");
      const bool tile_flagged = hf[3] || hf[4];
      if (tile_flagged && !(flags & FGT_ASSUME_SORTED)) {
        // unsorted input: the merge-path tiles of the speculative pass need
        // not cover every element, so every check is redone element-wise on
        // the arrays as given
        int* fc = p->d_flag + kFullCheck;
        ck(cudaMemsetAsync(fc, 0, sizeof(int) * 5, st), "flag");
        ck(launch_check_points(xs.dptr, M, ys.dptr, N, fc, st), "check points");
        ck(cudaMemcpyAsync(hf, fc, sizeof(int) * 5, cudaMemcpyDeviceToHost, st), "flags");
        ck(cudaStreamSynchronize(st), "flags sync");
      }
      // the reference checks targets, then sources (transform.cpp:202-204)
      if (hf[0]) raise(FGT_ERR_DOMAIN, "target coordinates must be finite");
      if (hf[1]) raise(FGT_ERR_DOMAIN, "source coordinates must be finite");
      p->same_points = (M == N) && !hf[2];  // transform.cpp:214-216
      p->t_sorted = !hf[3];
      p->s_sorted = !hf[4];
      temps.clear();  // ownership moves into adopt_set / sort_both_sets
      if (!p->t_sorted && !p->s_sorted && M > 0 && N > 0) {
        sort_both_sets(xs, M, ys, N, st, &p->d_xs, &p->d_tperm, &p->d_ys, &p->d_sperm);
        p->own_xs = p->own_ys = true;
      } else {
        adopt_set(xs, M, p->t_sorted, flags, st, &p->d_xs, &p->own_xs, &p->d_tperm);
        adopt_set(ys, N, p->s_sorted, flags, st, &p->d_ys, &p->own_ys, &p->d_sperm);
      }
      if (!p->t_sorted || !p->s_sorted || tile_flagged) {
        // metadata and classes of the sorted stream; first coordinates after
        // sorting
        plan_tiles(p, p->d_xs, p->d_ys, false, st, true, has_prev, z_prev);
        queue_slotted_classes(p, hc, st);
        if (M > 0) ck(cudaMemcpyAsync(xy0, p->d_xs, 8, cudaMemcpyDeviceToHost, st), "x0");
        if (N > 0) ck(cudaMemcpyAsync(xy0 + 1, p->d_ys, 8, cudaMemcpyDeviceToHost, st), "y0");
        ck(cudaStreamSynchronize(st), "sorted sync");
      }
      // coordinate before the first merged element: the element itself
      const double x0 = xy0[0], y0 = xy0[1];
      p->zprev0 = has_prev ? z_prev : (M > 0 && N > 0) ? std::fmin(x0, y0) : (M > 0 ? x0 : y0);
      take_slotted_classes(p, hc);
    } catch (...) {
      for (void* t : temps) cudaFreeAsync(t, st);
      destroy_plan(p);
      throw;
    }
    *out = p;
  });
}

}  // namespace

extern "C" {

int fgt_plan_create(const double* targets, int64_t M, const double* sources, int64_t N,
                    double delta, const double* t_re, const double* t_im, const double* w_re,
                    const double* w_im, const uint8_t* self_conj, int n_modes, int form,
                    uint32_t flags, int device, void* stream, fgt_plan_t* out) {
  return plan_create_impl(targets, M, sources, N, delta, t_re, t_im, w_re, w_im, self_conj,
                          n_modes, form, flags, device, stream, out, false, 0.0);
}

int fgt_plan_create_chunk(const double* sorted_targets, int64_t M, const double* sorted_sources,
                          int64_t N, double z_prev, int has_prev, double delta,
                          const double* t_re, const double* t_im, const double* w_re,
                          const double* w_im, const uint8_t* self_conj, int n_modes, int form,
                          uint32_t flags, int device, void* stream, fgt_plan_t* out) {
  int rc = plan_create_impl(sorted_targets, M, sorted_sources, N, delta, t_re, t_im, w_re, w_im,
                            self_conj, n_modes, form, flags | FGT_ASSUME_SORTED, device, stream,
                            out, has_prev != 0, z_prev);
  if (rc != FGT_OK) return rc;
  (*out)->same_points = false;
  return FGT_OK;
}

void fgt_plan_destroy(fgt_plan_t plan) { destroy_plan(plan); }

int fgt_plan_info(fgt_plan_t p, int64_t* M, int64_t* N, int* n_modes, int* same_points,
                  int* tsorted, int* ssorted, int64_t* ntiles) {
  return guarded([&] {
    if (!p) raise(FGT_ERR_INVALID, "NULL plan");
    if (M) *M = p->M;
    if (N) *N = p->N;
    if (n_modes) *n_modes = p->P.ne;
    if (same_points) *same_points = p->same_points;
    if (tsorted) *tsorted = p->t_sorted;
    if (ssorted) *ssorted = p->s_sorted;
    if (ntiles) *ntiles = p->ntiles;
  });
}

int fgt_plan_copy_sorted(fgt_plan_t p, double* sx, int64_t* tperm, double* sy, int64_t* sperm) {
  return guarded([&] {
    if (!p) raise(FGT_ERR_INVALID, "NULL plan");
    ck(cudaSetDevice(p->device), "cudaSetDevice");
    if (sx && p->M) ck(cudaMemcpy(sx, p->d_xs, 8 * p->M, cudaMemcpyDeviceToHost), "copy x");
    if (sy && p->N) ck(cudaMemcpy(sy, p->d_ys, 8 * p->N, cudaMemcpyDeviceToHost), "copy y");
    auto perm = [&](int32_t* d, int64_t n, int64_t* out) {
      if (!out || n == 0) return;
      if (!d) {
        for (int64_t i = 0; i < n; ++i) out[i] = i;
        return;
      }
      std::vector<int32_t> h(n);
      ck(cudaMemcpy(h.data(), d, 4 * n, cudaMemcpyDeviceToHost), "copy perm");
      for (int64_t i = 0; i < n; ++i) out[i] = h[i];
    };
    perm(p->d_tperm, p->M, tperm);
    perm(p->d_sperm, p->N, sperm);
  });
}

int fgt_plan_copy_soe(fgt_plan_t p, double* t_re, double* t_im, double* w_re, double* w_im,
                      uint8_t* sc) {
  return guarded([&] {
    if (!p) raise(FGT_ERR_INVALID, "NULL plan");
    for (size_t k = 0; k < p->soe.nodes.size(); ++k) {
      if (t_re) t_re[k] = p->soe.nodes[k].real();
      if (t_im) t_im[k] = p->soe.nodes[k].imag();
      if (w_re) w_re[k] = p->soe.weights[k].real();
      if (w_im) w_im[k] = p->soe.weights[k].imag();
      if (sc) sc[k] = p->soe.self_conj[k];
    }
  });
}

int fgt_apply_general(fgt_plan_t p, const double* strengths, int64_t n_strengths,
                      double* potentials, int num_threads, uint32_t flags, void* stream) {
  (void)num_threads;  // results never depend on it (transform.hpp:60-64)
  return guarded([&] {
    if (!p) raise(FGT_ERR_INVALID, "NULL plan");
    if (n_strengths != p->N)
      raise(FGT_ERR_INVALID, "strengths length must match the planned source count");
    run_apply(p, strengths, potentials, flags, as_stream(stream));
  });
}

int fgt_apply_same(fgt_plan_t p, const double* strengths, int64_t n_strengths,
                   double* potentials, int num_threads, uint32_t flags, void* stream) {
  return guarded([&] {
    if (!p) raise(FGT_ERR_INVALID, "NULL plan");
    if (!p->same_points)
      raise(FGT_ERR_INVALID,
            "apply_same requires a plan built from identical target and source sets");
    if (n_strengths != p->N)
      raise(FGT_ERR_INVALID, "strengths length must match the planned source count");
    // Same points: the merged stream puts every source before its equal
    // target, so forward includes self and backward excludes it, exactly the
    // run_mode_same split (transform.cpp:97-113).
    (void)num_threads;
    run_apply(p, strengths, potentials, flags, as_stream(stream));
  });
}

int fgt_apply_chunk_aggregate(fgt_plan_t p, const double* strengths, double* agg_out,
                              uint32_t flags, void* stream) {
  return guarded([&] {
    if (!p) raise(FGT_ERR_INVALID, "NULL plan");
    if (!agg_out) raise(FGT_ERR_INVALID, "agg_out must not be NULL");
    run_chunk_aggregate(p, strengths, reinterpret_cast<cplx*>(agg_out), flags, as_stream(stream));
  });
}

int fgt_apply_chunk_finish(fgt_plan_t p, const double* strengths, const double* carry_in,
                           double* potentials, uint32_t flags, void* stream) {
  return guarded([&] {
    if (!p) raise(FGT_ERR_INVALID, "NULL plan");
    if (!carry_in) raise(FGT_ERR_INVALID, "carry_in must not be NULL");
    run_chunk_finish(p, strengths, reinterpret_cast<const cplx*>(carry_in), potentials, flags,
                     as_stream(stream));
  });
}

// Chunk g's forward carry is the forward state at its z_prev from all chunks
// to its left: C+_g = A_{g-1} C+_{g-1} + F_{g-1}; the backward carry is the
// backward state at its last element from all chunks to its right:
// C-_g = A_{g+1} C-_{g+1} + G_{g+1}.  Each chunk's A already includes the gap
// from the previous chunk's last element.
int fgt_chunk_carries(const double* aggs, int n_chunks, int ne, double* carries_out) {
  return guarded([&] {
    if (n_chunks < 0 || ne < 0 || ne > kMaxModes) raise(FGT_ERR_INVALID, "bad sizes");
    using C = std::complex<double>;
    const C* a = reinterpret_cast<const C*>(aggs);
    C* c = reinterpret_cast<C*>(carries_out);
    for (int k = 0; k < ne; ++k) {
      C f(0.0, 0.0);
      for (int g = 0; g < n_chunks; ++g) {
        c[g * 2 * ne + k] = f;
        const C A = a[g * 3 * ne + k], F = a[g * 3 * ne + ne + k];
        f = C(A.real() * f.real() - A.imag() * f.imag() + F.real(),
              A.real() * f.imag() + A.imag() * f.real() + F.imag());
      }
      C b(0.0, 0.0);
      for (int g = n_chunks - 1; g >= 0; --g) {
        c[g * 2 * ne + ne + k] = b;
        const C A = a[g * 3 * ne + k], G = a[g * 3 * ne + 2 * ne + k];
        b = C(A.real() * b.real() - A.imag() * b.imag() + G.real(),
              A.real() * b.imag() + A.imag() * b.real() + G.imag());
      }
    }
  });
}

int fgt_chunk_carries_device(const double* aggs, int n_chunks, int ne, int rank,
                             double* carry_out, void* stream) {
  return guarded([&] {
    if (n_chunks < 1 || ne < 0 || ne > kMaxModes || rank < 0 || rank >= n_chunks)
      raise(FGT_ERR_INVALID, "bad sizes");
    if (!aggs || !carry_out) raise(FGT_ERR_INVALID, "NULL buffer");
    ck(launch_chunk_carries(reinterpret_cast<const cplx*>(aggs), n_chunks, ne, rank,
                            reinterpret_cast<cplx*>(carry_out), as_stream(stream)),
       "chunk carries");
  });
}

int fgt_gauss_transform(const double* targets, int64_t M, const double* sources, int64_t N,
                        const double* strengths, double delta, const double* t_re,
                        const double* t_im, const double* w_re, const double* w_im,
                        const uint8_t* self_conj, int n_modes, int form, int ne, int threads,
                        double* potentials) {
  // pymodule.cpp:37-60: custom SOE (folded if full) or fold(cf_soe(2*ne)).
  std::vector<double> tr, ti, wr, wi;
  std::vector<uint8_t> sc;
  if (n_modes <= 0) {
    int cnt = fgt_cf_soe(2 * ne, 1, nullptr, nullptr, nullptr, nullptr, nullptr);
    if (cnt < 0) return -cnt;
    tr.resize(cnt), ti.resize(cnt), wr.resize(cnt), wi.resize(cnt), sc.resize(cnt);
    fgt_cf_soe(2 * ne, 1, tr.data(), ti.data(), wr.data(), wi.data(), sc.data());
    t_re = tr.data(), t_im = ti.data(), w_re = wr.data(), w_im = wi.data();
    self_conj = sc.data();
    n_modes = cnt;
    form = FGT_SOE_FOLDED;
  }
  // same_points: apply_same and apply_general agree on the merged stream
  // (every source precedes its equal target), so one path serves both
  (void)threads;
  return fgt_transform_host(targets, M, sources, N, strengths, delta, t_re, t_im, w_re, w_im,
                            self_conj, n_modes, form, potentials, -1, nullptr);
}

int fgt_transform_host(const double* targets, int64_t M, const double* sources, int64_t N,
                       const double* strengths, double delta, const double* t_re,
                       const double* t_im, const double* w_re, const double* w_im,
                       const uint8_t* self_conj, int n_modes, int form, double* potentials,
                       int device, void* stream) {
  return guarded([&] {
    if (M < 0 || N < 0) raise(FGT_ERR_INVALID, "negative point count");
    if ((M > 0 && (!targets || !potentials)) || (N > 0 && (!sources || !strengths)))
      raise(FGT_ERR_INVALID, "NULL buffer");
    if (M >= ((int64_t)1 << 31) || N >= ((int64_t)1 << 31))
      raise(FGT_ERR_INVALID, "at most 2^31-1 points per set");
    check_delta(delta);
    Soe soe = resolve_soe(t_re, t_im, w_re, w_im, self_conj, n_modes, form);
    require_device(device);
    transform_host(targets, M, sources, N, strengths, potentials, delta, soe, as_stream(stream));
  });
}

}  // extern "C"

// ---------------------------------------------------------------- extras

extern "C" int fgt_plan_gap_table(fgt_plan_t p, double* out) {
  return guarded([&] {
    if (!p) raise(FGT_ERR_INVALID, "NULL plan");
    ck(cudaSetDevice(p->device), "cudaSetDevice");
    int rc = fgt_gap_table_device(p->d_xs, p->M, p->P.ne, p->P.s_re, p->P.s_im, out);
    if (rc != FGT_OK) throw ApiError{rc, g_last_error};
  });
}

extern "C" int fgt_mode_sums(fgt_plan_t p, const double* strengths, double* hp, double* hm) {
  return guarded([&] {
    if (!p) raise(FGT_ERR_INVALID, "NULL plan");
    ck(cudaSetDevice(p->device), "cudaSetDevice");
    cudaStream_t st = nullptr;
    Work w{st, {}};
    const int ne = p->P.ne;
    const size_t cnt = (size_t)ne * (size_t)p->M;
    cplx* d_hp = w.get<cplx>(cnt);
    cplx* d_hm = w.get<cplx>(cnt);
    if (p->N == 0 || p->M == 0) {
      ck(cudaMemsetAsync(d_hp, 0, sizeof(cplx) * cnt, st), "zero");
      ck(cudaMemsetAsync(d_hm, 0, sizeof(cplx) * cnt, st), "zero");
    } else {
      const double* bs = sorted_strengths(p, strengths, 0, w, nullptr);
      const StreamArgs sa = stream_args(p, bs);
      const TileState ts = tile_state_carve(w.get<cplx>(tile_state_elems(p->ntiles, ne)),
                                            p->ntiles, ne);
      ck(launch_aggregate(sa, p->P, p->d_mt, ts, st), "aggregates");
      ck(launch_carry_scan(ts, p->ntiles, ne, nullptr, nullptr, st), "carry scan");
      OutArgs o;
      o.hp = d_hp;
      o.hm = d_hm;
      ck(launch_mode_sums(sa, p->P, p->d_mt, ts, o, st), "mode sums");
    }
    if (cnt) {
      ck(cudaMemcpyAsync(hp, d_hp, sizeof(cplx) * cnt, cudaMemcpyDeviceToHost, st), "hp");
      ck(cudaMemcpyAsync(hm, d_hm, sizeof(cplx) * cnt, cudaMemcpyDeviceToHost, st), "hm");
    }
    ck(cudaStreamSynchronize(st), "sync");
  });
}

// ---- instrumentation used by bench.py ------------------------------------

extern "C" long long fgt_launch_counter(void) { return g_launch_count.load(); }

extern "C" void fgt_profile_enable(int on) { g_profile.store(on != 0); }

// ms[kind], counts[kind] for kind 0 = tile aggregates (K1), 1 = carry scan
// (K2), 2 = main pass (K3); accumulated since the last read.  Synchronizes
// on the recorded events.
extern "C" int fgt_profile_read(double* ms, long long* counts, int nkinds) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto& e : g_prof_pending) {
    float t = 0.f;
    cudaEventSynchronize(e.b);
    cudaEventElapsedTime(&t, e.a, e.b);
    g_prof_ms[e.kind] += t;
    g_prof_cnt[e.kind] += 1;
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  g_prof_pending.clear();
  for (int k = 0; k < nkinds && k < 8; ++k) {
    if (ms) ms[k] = g_prof_ms[k];
    if (counts) counts[k] = g_prof_cnt[k];
    g_prof_ms[k] = 0.0;
    g_prof_cnt[k] = 0;
  }
  return FGT_OK;
}

// ---- batched transforms (BASELINE cfg 5) ---------------------------------
// B independent presorted transforms in one plan: targets / sources are the
// concatenation of the transforms' sets (host offsets t_off / s_off, B+1
// entries), one delta per transform, one SOE for all.  Every transform's
// stream starts at a segment boundary with zprev = -inf, so transforms never
// couple; each segment reads its transform's mode table.  Apply with
// fgt_apply_general (strengths / potentials concatenated the same way).
extern "C" int fgt_batch_create(int B, const double* targets, const int64_t* t_off,
                                const double* sources, const int64_t* s_off,
                                const double* deltas, const double* t_re, const double* t_im,
                                const double* w_re, const double* w_im, const uint8_t* self_conj,
                                int n_modes, int form, uint32_t flags, int device, void* stream,
                                fgt_plan_t* out) {
  return guarded([&] {
    if (!out) raise(FGT_ERR_INVALID, "out must not be NULL");
    *out = nullptr;
    if (B < 1) raise(FGT_ERR_INVALID, "batch needs at least one transform");
    if (!t_off || !s_off || !deltas) raise(FGT_ERR_INVALID, "offsets / deltas must not be NULL");
    if (t_off[0] != 0 || s_off[0] != 0) raise(FGT_ERR_INVALID, "offsets must start at 0");
    for (int b = 0; b < B; ++b) {
      if (t_off[b + 1] < t_off[b] || s_off[b + 1] < s_off[b])
        raise(FGT_ERR_INVALID, "offsets must be non-decreasing");
      check_delta(deltas[b]);
    }
    const int64_t M = t_off[B], N = s_off[B];
    if (M >= ((int64_t)1 << 31) || N >= ((int64_t)1 << 31))
      raise(FGT_ERR_INVALID, "at most 2^31-1 points per set");
    Soe soe = resolve_soe(t_re, t_im, w_re, w_im, self_conj, n_modes, form);
    require_device(device);
    cudaStream_t st = as_stream(stream);
    fgt_plan_s* p = new fgt_plan_s();
    std::vector<void*> temps;
    try {
      ck(cudaGetDevice(&p->device), "cudaGetDevice");
      p->M = M;
      p->N = N;
      p->delta = deltas[0];
      p->soe = soe;
      p->batch = true;
      p->nbatch = B;
      p->stream = st;
      p->d_flag = dmalloc<int>(kFlagInts, st);
      ck(cudaMemsetAsync(p->d_flag, 0, sizeof(int) * kFlagInts, st), "flag");
      SetSrc xs = stage_set(targets, M, flags, st);
      SetSrc ys = stage_set(sources, N, flags, st);
      if (xs.tmp) temps.push_back((void*)xs.dptr);
      if (ys.tmp) temps.push_back((void*)ys.dptr);
      // segment / tile layout per transform
      std::vector<int64_t> seg_base(B + 1, 0), tile_base(B + 1, 0);
      for (int b = 0; b < B; ++b) {
        const int64_t L = (t_off[b + 1] - t_off[b]) + (s_off[b + 1] - s_off[b]);
        seg_base[b + 1] = seg_base[b] + (L + kSeg - 1) / kSeg;
        tile_base[b + 1] = tile_base[b] + (L + kPlanTile - 1) / kPlanTile;
      }
      const int64_t nseg = seg_base[B], ntl = tile_base[B];
      std::vector<int32_t> tile_tid(ntl);
      for (int b = 0; b < B; ++b)
        for (int64_t t = tile_base[b]; t < tile_base[b + 1]; ++t) tile_tid[t] = b;
      p->ntiles = nseg;
      p->d_tile_ib = dmalloc<int64_t>(nseg + 1, st);
      p->d_seg_jb = dmalloc<int64_t>(nseg + 1, st);
      p->d_seg_info = dmalloc<int4>(nseg + 1, st);
      p->d_seg_z = dmalloc<double2>(nseg + 1, st);
      p->d_seg_deg = alloc_seg_deg(nseg, st);
      p->d_seg_mask = dmalloc<uint32_t>((size_t)(nseg + 1) * (kSeg / 32), st);
      Work w{st, {}};
      int64_t* d_toff = w.get<int64_t>(B + 1);
      int64_t* d_soff = w.get<int64_t>(B + 1);
      int64_t* d_sbase = w.get<int64_t>(B + 1);
      int64_t* d_tbase = w.get<int64_t>(B + 1);
      int32_t* d_ttid = w.get<int32_t>(ntl + 1);
      int64_t* d_tib = w.get<int64_t>(ntl + 1);
      ck(cudaMemcpyAsync(d_toff, t_off, 8 * (B + 1), cudaMemcpyHostToDevice, st), "offsets");
      ck(cudaMemcpyAsync(d_soff, s_off, 8 * (B + 1), cudaMemcpyHostToDevice, st), "offsets");
      ck(cudaMemcpyAsync(d_sbase, seg_base.data(), 8 * (B + 1), cudaMemcpyHostToDevice, st), "bases");
      ck(cudaMemcpyAsync(d_tbase, tile_base.data(), 8 * (B + 1), cudaMemcpyHostToDevice, st), "bases");
      if (ntl)
        ck(cudaMemcpyAsync(d_ttid, tile_tid.data(), 4 * ntl, cudaMemcpyHostToDevice, st), "tile map");
      ck(launch_batch_plan(xs.dptr, ys.dptr, d_toff, d_soff, d_sbase, d_tbase, d_ttid, B, ntl,
                           d_tib, p->d_tile_ib, p->d_seg_jb, p->d_seg_info, p->d_seg_z,
                           p->d_seg_mask, p->d_flag, st),
         "batch plan");
      unsigned char* pin = pinned_scratch();
      int hfl[8] = {0};
      int* hf = pin ? reinterpret_cast<int*>(pin) : hfl;
      ck(cudaMemcpyAsync(hf, p->d_flag, sizeof(int) * 8, cudaMemcpyDeviceToHost, st), "flags");
      // per-transform mode tables (device-built), the shared one of transform 0
      ModeTable T0;
      build_modes(p->soe, deltas[0], p->P, T0);
      BatchModeBase base{};
      base.ne = p->P.ne;
      for (int k = 0; k < base.ne; ++k) {
        base.t[k] = {p->soe.nodes[k].real(), p->soe.nodes[k].imag()};
        base.mw[k] = {p->P.mw_re[k], p->P.mw_im[k]};
      }
      double* d_deltas = w.get<double>(B);
      ck(cudaMemcpyAsync(d_deltas, deltas, sizeof(double) * B, cudaMemcpyHostToDevice, st),
         "deltas");
      p->d_mtb = dmalloc<ModeTable>(B, st);
      ck(launch_batch_modes(base, d_deltas, B, p->d_mtb, st), "mode tables");
      p->d_mt = dmalloc<ModeTable>(1, st);
      ck(launch_store_table(T0, p->d_mt, st), "mode table");
      unsigned long long hcl[4] = {0, 0, 0, 0};
      unsigned long long* hc = pin ? reinterpret_cast<unsigned long long*>(pin + 64) : hcl;
      queue_classify(p, hc, st, true);
      ck(cudaStreamSynchronize(st), "batch plan sync");
      take_classes(p, hc);
      if (hf[0]) raise(FGT_ERR_DOMAIN, "target coordinates must be finite");
      if (hf[1]) raise(FGT_ERR_DOMAIN, "source coordinates must be finite");
      if (hf[3] || hf[4])
        raise(FGT_ERR_INVALID, "batched transforms require each transform's points sorted");
      temps.clear();
      adopt_set(xs, M, true, flags, st, &p->d_xs, &p->own_xs, &p->d_tperm);
      adopt_set(ys, N, true, flags, st, &p->d_ys, &p->own_ys, &p->d_sperm);
      p->same_points = false;
    } catch (...) {
      for (void* t : temps) cudaFreeAsync(t, st);
      destroy_plan(p);
      throw;
    }
    *out = p;
  });
}
