#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <atomic>

namespace fgt_b200 {

// Launch accounting for bench.py's gpu_launches (fgt_capi.cu).
void note_launch(int n = 1);

size_t radix_sort_workspace_bytes(int64_t n);
// Stable ascending sort of x (n < 2^31) -> sorted values and the permutation
// (sorted[i] == x[perm[i]]; ties keep original order, like the reference).
cudaError_t radix_sort_with_perm(const double* x, int64_t n, double* sorted, int32_t* perm,
                                 void* workspace, cudaStream_t st);
cudaError_t check_sorted(const double* x, int64_t n, int* d_flag, int* is_sorted,
                         cudaStream_t st);
cudaError_t check_equal(const double* x, const double* y, int64_t n, int* d_flag, int* equal,
                        cudaStream_t st);
cudaError_t check_finite(const double* x, int64_t n, int* d_flag, int* finite, cudaStream_t st);
// Flag kernels (no sync): set *flag = 1 if the condition is found.
cudaError_t launch_flag_unsorted(const double* x, int64_t n, int* flag, cudaStream_t st);
cudaError_t launch_flag_unequal(const double* x, const double* y, int64_t n, int* flag,
                                cudaStream_t st);
cudaError_t launch_flag_nonfinite(const double* x, int64_t n, int* flag, cudaStream_t st);
// Fused plan checks (flags[0..4]: x non-finite, y non-finite, x != y when
// M == N, x unsorted, y unsorted); flags must be zeroed by the caller.
cudaError_t launch_plan_checks(const double* x, int64_t M, const double* y, int64_t N,
                               int check_sorted, int* flags, cudaStream_t st);
cudaError_t launch_iota(int32_t* p, int64_t n, cudaStream_t st);


// Raise a kernel's dynamic shared-memory limit once per device (the
// attribute is per device; mask: one bit per device ordinal < 64).
template <class K>
inline cudaError_t ensure_dynamic_smem(K kernel, int bytes, std::atomic<unsigned long long>& mask) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = 1ull << (dev & 63);
  if (mask.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) mask.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

}  // namespace fgt_b200
