// Tile kernels of the merged-stream SOE scan: K0 partition, K1 tile
// aggregates, K2 carry scan over tiles, K3 main pass (see fgt_device.cuh and
// DESIGN.md §3).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "fgt_device.cuh"

namespace fgt_b200 {

constexpr int kWarps = 4;               // warps per CTA (one tile per CTA)
constexpr int kR = 8;                   // merged elements per lane run
constexpr int kThreads = kWarps * 32;   // 128
constexpr int kTile = kThreads * kR;    // 1024 merged elements per tile

// Per-mode constants laid out in device memory (plan-owned), copied into
// shared memory by every CTA: s_k, mw_k and the Taylor coefficients
// c_{k,n} = (-s_k)^n / n! of the gap factor exp(-s_k g).
struct ModeTable {
  cplx s[kMaxModes];
  cplx mw[kMaxModes];
  cplx coef[kMaxModes][kMaxDeg + 1];
};

struct StreamArgs {
  const double* xs;  // sorted targets (this chunk)
  int64_t M;
  const double* ys;  // sorted sources (this chunk)
  int64_t N;
  const double* bs;  // strengths in sorted-source order
  const int64_t* tile_ib;  // [ntiles+1] targets preceding each tile
  int64_t ntiles;
  double zprev0;  // coordinate of the element before this chunk (or its first)
};

struct OutArgs {
  double* u = nullptr;             // potentials (original target order if tperm)
  const int32_t* tperm = nullptr;  // sorted -> original target index, or nullptr (identity)
  int64_t u_offset = 0;            // global sorted index of this chunk's first target
  cplx* hp = nullptr;              // mode sums (test hook): [ne][M] h+ and h-
  cplx* hm = nullptr;
};

// Aggregates / carries, [ne][ntiles] each.
struct TileState {
  cplx* A;
  cplx* F;
  cplx* G;
  cplx* Cf;
  cplx* Cb;
};

size_t tile_smem_bytes(int ne);

cudaError_t launch_partition(const double* xs, int64_t M, const double* ys, int64_t N,
                             int64_t tile, int64_t ntiles, int64_t* tile_ib,
                             cudaStream_t st);
cudaError_t launch_aggregate(const StreamArgs& a, const ModeParams& P, const ModeTable* mt,
                             TileState ts, cudaStream_t st);
cudaError_t launch_mode_sums(const StreamArgs& a, const ModeParams& P, const ModeTable* mt,
                             TileState ts, OutArgs o, cudaStream_t st);
cudaError_t launch_carry_scan(const TileState& ts, int64_t ntiles, int ne, const cplx* carry_in,
                              cplx* totals, cudaStream_t st);
cudaError_t launch_main(const StreamArgs& a, const ModeParams& P, const ModeTable* mt,
                        TileState ts, OutArgs o, cudaStream_t st);
cudaError_t launch_gather(const double* alpha, const int32_t* perm, int64_t n, double* out,
                          cudaStream_t st);

}  // namespace fgt_b200
