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
// The same in two halves around one host read, so that several sorts can
// share it: begin queues the keys and the digit histograms and copies the
// histograms (8 * 256 u64) to hist_host; once they have landed (the caller
// synchronizes st), end queues the passes that are not the identity.
constexpr int kSortHistWords = 8 * 256;
cudaError_t radix_sort_begin(const double* x, int64_t n, void* workspace,
                             unsigned long long* hist_host, cudaStream_t st);
cudaError_t radix_sort_end(const double* x, int64_t n, double* sorted, int32_t* perm,
                           void* workspace, const unsigned long long* hist_host, cudaStream_t st);
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
