// Segment kernels of the merged-stream SOE scan: K0 partition, K1 segment
// aggregates, K2 carry scan over segments, K3 main pass (see fgt_device.cuh
// and DESIGN.md §3).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "fgt_device.cuh"

namespace fgt_b200 {

#ifndef FGT_KR
#define FGT_KR 8
#endif
constexpr int kR = FGT_KR;              // merged elements per lane run
constexpr int kSeg = 32 * kR;           // merged elements per segment (one warp)
#ifndef FGT_SEG_WARPS
#define FGT_SEG_WARPS 4
#endif
constexpr int kSegWarps = FGT_SEG_WARPS;  // segments (warps) per CTA in K1 / K3
constexpr int kThreads = 32 * kSegWarps;
constexpr int kMaxMom = kMaxDeg;        // highest moment order of the expansions
// (21: the largest odd tile that keeps 5 CTAs per SM in the tile pass; cfg 3
// plan + other 0.563 ms at 15, 0.545 at 19, 0.52-0.53 at 21, 0.556 at 23, 0.537 at 25)
#ifndef FGT_PLAN_SEGS
#define FGT_PLAN_SEGS 21
#endif
constexpr int kPlanSegs = FGT_PLAN_SEGS;  // segments per plan tile
constexpr int kPlanTile = kPlanSegs * kSeg;  // merged elements per plan tile

// Per-mode constants laid out in device memory (plan-owned): s_k, mw_k and the
// Taylor coefficients c_{k,n} = (-s_k)^n / n! of exp(-s_k g).
// Highest degree of the collapsed (mode-folded) polynomial of narrow segments.
constexpr int kCollDeg = 8;

struct ModeTable {
  cplx s[kMaxModes];
  cplx mw[kMaxModes];
  cplx coef[kMaxModes][kMaxDeg + 1];
  double smax;  // max_k |s_k| (degree selection)
  double pad;
  // lane-collapsed wide segments (fgt_scan.cu lane_collapsed): the mode-folded
  // polynomial up to the highest Taylor degree, gl[n] = Re sum_k mw_k coef[k][n]
  double gl[kMaxDeg + 1];
  double pad3;
  // collapsed form of narrow segments (fgt_scan.cu collapsed_segment):
  // mwc[k][n] = mw_k coef[k][n], gpoly[n] = Re sum_k mwc[k][n]
  // (the lane-collapsed kernel stages only the fields before mwc)
  cplx mwc[kMaxModes][kCollDeg + 1];
  double gpoly[kCollDeg + 1];
  double pad2;
};
static_assert(sizeof(ModeTable) <= 4096, "ModeTable is passed as a kernel parameter");
// tables are staged ahead of 16-byte aligned stages in shared memory
static_assert(sizeof(ModeTable) % 16 == 0, "ModeTable size must be a multiple of 16 bytes");

// Constants of the collapsed narrow K3 (k3n), derived from the collapsed
// polynomial G(t) = sum_n g_n t^n of a plan (ModeTable::gpoly):
//   H[m][q] = 2 (-1)^m C(m+q, m) g_{m+q}   (m + q odd)  prefix-moment terms
//   B[q][m] = (-1)^q C(m+q, m) g_{m+q}                  total-moment terms
// (fgt_scan.cu, collapsed form).  Passed as a kernel parameter: the FMAs read
// them from the constant bank.
constexpr int kSegFallbackBit = 1 << 30;  // seg_deg: not lane-collapsible (set by K3)
// seg_deg is allocated with two trailing ints; the second counts the flagged
// segments of the plan (the per-mode kernel behind the lane-collapsed one
// leaves at once while it is 0).
__host__ __device__ inline int* seg_fallback_count(const int* seg_deg, int64_t nseg) {
  return const_cast<int*>(seg_deg) + nseg + 1;
}
constexpr int kCollMax = 6;   // highest collapsed degree of the narrow K3
constexpr int kEcStride = 8;  // doubles per segment of the collapsed carries
struct CollConsts {
  double H[kCollMax + 1][kCollMax + 1];
  double B[kCollMax + 1][kCollMax + 1];
};
CollConsts coll_consts(const double* gpoly);

struct StreamArgs {
  const double* xs;  // sorted targets (this chunk)
  int64_t M;
  const double* ys;  // sorted sources (this chunk)
  int64_t N;
  const double* bs;  // strengths in sorted-source order
  const int64_t* seg_ib;  // [nseg+1] targets preceding each segment
  int64_t nseg;
  double zprev0;  // coordinate of the element before this chunk (or its first)
  // plan-time segment metadata (seg_meta): (zprev, zlast) per segment and
  // the merged order as one bit per element (1 = target), 8 words/segment;
  // single plans append per-segment word prefix counts (seg_mask_prefix)
  const double2* seg_z;
  const uint32_t* seg_mask;
  // batched transforms (nullptr for a single stream): per segment
  // (len, nx, transform, 0) with seg_ib = global first target and
  // seg_jb = global first source; per-transform mode tables
  const int4* seg_info = nullptr;
  const int64_t* seg_jb = nullptr;
  const ModeTable* mtb = nullptr;
  // plan-time segment classes (classify_segments): segments too wide for the
  // moment form of K1 / K3; -1 = unknown (both kernel variants run)
  int64_t nwide1 = -1, nwide3 = -1;
  // plan-time degrees per segment: (D + 1) | (DM + 1) << 8 with D the Taylor
  // degree of its gap factors and DM its moment degree (-1 = none)
  const int* seg_deg = nullptr;
  // wide K3 after the lane-collapsed kernel: only the segments that kernel
  // flagged (kSegFallbackBit of seg_deg: lane runs too wide for it)
  int fallback_only = 0;
  // classify_kernel only: segment 0's zprev is its own first element (a
  // plan without a predecessor, classified before zprev0 is known on the host)
  bool zprev0_first = false;
  // plan-time highest collapsed degree DN over the narrow segments (-1:
  // unknown -> the narrow K3 runs at kCollMax)
  int dn_narrow = -1;
  // plan-time highest moment degree DM over the K1-narrow segments (-1:
  // unknown -> kMomMax moments)
  int dm_narrow = -1;
};

// Single plans: seg_mask holds kSeg / 32 words per segment followed by one
// uint2 per segment whose byte q counts the targets in words 0 .. q-1 (plan
// tile pass); seg_mask_words sizes that allocation (+ one padding entry).
constexpr int kSegMaskWords = kSeg / 32;
__host__ __device__ inline size_t seg_mask_words(int64_t nseg) {
  return (size_t)nseg * kSegMaskWords + 2 * (size_t)nseg + 4;
}
__host__ __device__ inline uint2* seg_mask_prefix(uint32_t* seg_mask, int64_t nseg) {
  return reinterpret_cast<uint2*>(seg_mask + (size_t)nseg * kSegMaskWords);
}
__host__ __device__ inline const uint2* seg_mask_prefix(const uint32_t* seg_mask, int64_t nseg) {
  return reinterpret_cast<const uint2*>(seg_mask + (size_t)nseg * kSegMaskWords);
}

struct OutArgs {
  double* u = nullptr;             // potentials (original target order if tperm)
  const int32_t* tperm = nullptr;  // sorted -> original target index, or nullptr (identity)
  int64_t u_offset = 0;            // global sorted index of this chunk's first target
  cplx* hp = nullptr;              // mode sums (test hook): [ne][M] h+ and h-
  cplx* hm = nullptr;
};

// Segment aggregates / carries, [ne][nseg] each, plus the K2 workspace.
struct TileState {
  cplx* A;
  cplx* F;
  cplx* G;
  cplx* Cf;
  cplx* Cb;
  cplx* blk;  // scan workspace: scan_blocks(nseg) * 2 * ne * 3 complex
  double* ec;  // collapsed carries of the narrow segments, [nseg][kEcStride]
};

int64_t scan_blocks(int64_t nseg);
// complex values needed for a TileState of nseg segments and ne modes
size_t tile_state_elems(int64_t nseg, int ne);
TileState tile_state_carve(cplx* base, int64_t nseg, int ne);

size_t seg_smem_bytes(int ne, bool batched, bool stream, int region = 1);

cudaError_t launch_partition(const double* xs, int64_t M, const double* ys, int64_t N,
                             int64_t seg, int64_t nseg, int64_t* seg_ib, cudaStream_t st);
// Plan-time tile pass (speculative on unsorted input): checks (flags[0..4] =
// x non-finite, y non-finite, x != y when M == N, x unsorted, y unsorted;
// zeroed by the caller) and segment metadata seg_ib / seg_z / seg_mask.
// tile_ib: launch_partition output at kPlanTile granularity.
// Segment classification folded into the tile pass (single plans): the
// degrees classify_kernel would write (seg_deg) and the class counts, summed
// per CTA into kClassSlots slots of 4 u64 each (wide-K1 count, wide-K3 count,
// max DN + 1, max DM + 1), which the host reduces.  z_prev: the coordinate
// before segment 0 when has_prev (chunk plans), else its own first element.
constexpr int kClassSlots = 32;
struct PlanClassify {
  int enabled = 0;
  ModeParams P;
  double smax = 0.0;
  int* seg_deg = nullptr;
  unsigned long long* counts = nullptr;  // [kClassSlots][4]
  int has_prev = 0;
  double z_prev = 0.0;
};
cudaError_t launch_plan_tiles(const double* xs, int64_t M, const double* ys, int64_t N,
                              const int64_t* tile_ib, int64_t ntiles, int64_t nseg,
                              int check_sorted, int64_t* seg_ib, double2* seg_z,
                              uint32_t* seg_mask, int* flags, cudaStream_t st,
                              const PlanClassify* cls = nullptr);
// Element-wise checks of unsorted input (flags[0..4] as launch_plan_tiles,
// zeroed by the caller) over the arrays as given.
cudaError_t launch_check_points(const double* xs, int64_t M, const double* ys, int64_t N,
                                int* flags, cudaStream_t st);
// Batched plans: per-transform offsets (B+1 each, concatenated arrays) and
// the first global segment of each transform (B+1).  Partition at
// kPlanTile granularity inside each transform, then the tile pass writes the
// per-segment metadata (seg_ib, seg_jb, seg_info, seg_z, seg_mask; zprev of
// each transform's first segment = -inf, so transforms never couple) and the
// flags (0/1: non-finite, 3/4: a transform's targets / sources unsorted).
cudaError_t launch_batch_plan(const double* xs, const double* ys, const int64_t* t_off,
                              const int64_t* s_off, const int64_t* seg_base,
                              const int64_t* tile_base, const int32_t* tile_tid, int B,
                              int64_t ntiles, int64_t* tile_ib, int64_t* seg_ib, int64_t* seg_jb,
                              int4* seg_info, double2* seg_z, uint32_t* seg_mask,
                              int* flags, cudaStream_t st);
// Per-transform mode tables of a batched plan, built on the device:
// s_k = t_k / sqrt(delta_b), mw_k, Taylor coefficients of exp(-s g)
// (c_0 = 1 and c_1 = -s exact), smax.  deltas: device array of B.
struct BatchModeBase {
  int ne;
  cplx t[kMaxModes];   // folded SOE nodes
  cplx mw[kMaxModes];  // multiplier * weight
};
// Store a mode table built on the host through a kernel parameter (no
// pageable copy, no implicit stream synchronisation).
cudaError_t launch_store_table(const ModeTable& T, ModeTable* out, cudaStream_t st);
cudaError_t launch_batch_modes(const BatchModeBase& base, const double* deltas, int B,
                               ModeTable* out, cudaStream_t st);
// Plan-time classification: counts[0] / counts[1] = segments that K1 / K3
// process on their wide (per-element) path, counts[2] = the highest
// collapsed degree DN among the K3-narrow segments.  smax: the single plan's
// max |s_k| (batched plans read their tables).
// Also writes seg_deg (see StreamArgs) from seg_gap and the segment frames.
cudaError_t launch_classify(const StreamArgs& a, const ModeParams& P, double smax,
                            int* seg_deg, const int* skip_flags,
                            unsigned long long* counts, cudaStream_t st);
cudaError_t launch_aggregate(const StreamArgs& a, const ModeParams& P, const ModeTable* mt,
                             TileState ts, cudaStream_t st);
// K2: exclusive carries per segment.  carry_in: 2*ne complex (forward carry at
// the chunk's z_prev, backward carry at the chunk end) or nullptr; totals:
// 3*ne complex (A, F, G of the whole chunk) or nullptr.  reduce = false
// reuses the block aggregates of an earlier scan of the same TileState (a
// chunk's phase 2: only the carry-in changed); down = false stops after the
// top level (a chunk's phase 1: only the totals are needed).
cudaError_t launch_carry_scan(const TileState& ts, int64_t nseg, int ne, const cplx* carry_in,
                              cplx* totals, cudaStream_t st, bool reduce = true,
                              bool down = true);
// Chunk carries of one chunk from the gathered chunk aggregates (the
// algebra of fgt_chunk_carries, one thread per mode).
cudaError_t launch_chunk_carries(const cplx* aggs, int n_chunks, int ne, int rank, cplx* out,
                                 cudaStream_t st);
// K3.  cc: the plan's collapsed-form constants (single plans); nullptr runs
// the per-segment-degree narrow kernel (batched plans, per-transform tables).
// folded: ts.ec already holds the segment-total terms (launch_mom_scan with
// cc and k3_folds(a)).
cudaError_t launch_main(const StreamArgs& a, const ModeParams& P, const ModeTable* mt,
                        TileState ts, OutArgs o, cudaStream_t st, const CollConsts* cc = nullptr,
                        bool ec_ready = false, bool folded = false);
// Moment path (single plans): K1m writes the narrow segments' source
// moments (k1m_moments(a) per segment, mom[nseg][..]) and the wide K1 the
// others' (A, F, G); K2m scans them per mode and direction and writes the
// K3-narrow segments' collapsed carries (ts.ec, launch_main(..., ec_ready))
// and the K3-wide segments' carries (ts.Cf / Cb).  carry_in / totals /
// reduce / down as launch_carry_scan.
int k1m_moments(const StreamArgs& a);
int k3n_degree(const StreamArgs& a);
cudaError_t launch_moments(const StreamArgs& a, const ModeParams& P, const ModeTable* mt,
                           TileState ts, double* mom, cudaStream_t st);
// cc: fold the collapsed form's segment-total terms into E^c when
// k3_folds(a) (the K1 moments reach the collapsed degree).
bool k3_folds(const StreamArgs& a);
cudaError_t launch_mom_scan(const StreamArgs& a, int ne, const ModeTable* mt, const TileState& ts,
                            double* mom, const cplx* carry_in, cplx* totals,
                            cudaStream_t st, bool reduce = true, bool down = true,
                            const CollConsts* cc = nullptr);
cudaError_t launch_mode_sums(const StreamArgs& a, const ModeParams& P, const ModeTable* mt,
                             TileState ts, OutArgs o, cudaStream_t st);
cudaError_t launch_gather(const double* alpha, const int32_t* perm, int64_t n, double* out,
                          cudaStream_t st);

}  // namespace fgt_b200
