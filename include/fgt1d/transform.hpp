#pragma once
// Discrete Gauss transform u_i = sum_j exp(-(x_i - y_j)^2 / (4 delta)) alpha_j
// -- drop-in for the reference's proj/include/fgt1d/transform.hpp:17-106.
// Same types, names, argument meaning and exception behaviour; the work runs
// on the GPU through the C ABI (include/fgt1d_b200.h).
#include <complex>
#include <cstdint>
#include <memory>
#include <vector>

#include "fgt1d/soe.hpp"

namespace fgt {

struct TransformRequest {
  std::vector<double> targets;    // x_i
  std::vector<double> sources;    // y_j
  std::vector<double> strengths;  // alpha_j, one per source
  double delta = 1.0;             // > 0
};

struct TransformResult {
  std::vector<double> potentials;  // u_i, one per target, original order
};

// Reusable plan (transform.hpp:28-47).  The public fields are populated as in
// the reference; `device` owns the GPU-resident plan the applies run on.
struct TransformPlan {
  std::vector<double> sorted_targets;
  std::vector<double> sorted_sources;
  std::vector<std::int64_t> target_perm;
  std::vector<std::int64_t> source_perm;
  SoeApprox soe;  // folded form
  double delta = 1.0;
  bool same_points = false;
  bool precomputed = false;
  std::vector<std::complex<double>> gap_exponentials;
  std::shared_ptr<void> device;  // fgt_plan_t
};

TransformPlan plan(const TransformRequest& request, const SoeApprox& soe, bool precompute);
void precompute_gap_table(TransformPlan& plan);
TransformResult apply_same(const TransformPlan& plan, const std::vector<double>& strengths,
                           int num_threads = 1);
TransformResult apply_general(const TransformPlan& plan, const std::vector<double>& strengths,
                              int num_threads = 1);
TransformResult direct(const TransformRequest& request,
                       const std::vector<std::int64_t>& target_subset = {});

enum class Precision { Digits4, Digits7, Digits9, Digits11 };
int preset_mode_count(Precision p);  // 3, 4, 5, 6
SoeApprox preset_soe(Precision p);   // folded

namespace detail {
struct ModeSums {
  std::vector<std::vector<std::complex<double>>> hp;
  std::vector<std::vector<std::complex<double>>> hm;
};
ModeSums mode_sums(const TransformPlan& plan, const std::vector<double>& strengths);
}  // namespace detail

}  // namespace fgt
