#pragma once
// Discrete Gauss transform u_i = sum_j exp(-(x_i - y_j)^2 / (4 delta)) alpha_j
// -- drop-in for the reference's proj/include/fgt1d/transform.hpp:17-106.
// Same types, names, argument meaning and exception behaviour; the work runs
// on the GPU through the C ABI (include/fgt1d_b200.h).
#include <complex>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <memory>
#include <mutex>
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

// Read-only host view of a plan array that lives on the GPU.  It reads like
// the reference's std::vector field (size, [], iteration, data, comparison,
// conversion to const std::vector&); the size is known at plan time and the
// contents are copied from the device on first access (once, thread-safe),
// so a plan that is only applied never moves its sorted arrays or
// permutations back to the host.
template <class T>
class HostMirror {
 public:
  HostMirror() : st_(std::make_shared<State>()) { st_->ready = true; }
  HostMirror(std::size_t n, std::function<void(T*)> load) : st_(std::make_shared<State>()) {
    st_->n = n;
    st_->load = std::move(load);
  }
  std::size_t size() const { return st_->n; }
  bool empty() const { return st_->n == 0; }
  const std::vector<T>& get() const {
    std::call_once(st_->once, [s = st_.get()] {
      if (s->ready) return;
      s->v.resize(s->n);
      if (s->n && s->load) s->load(s->v.data());
      s->ready = true;
    });
    return st_->v;
  }
  operator const std::vector<T>&() const { return get(); }
  const T& operator[](std::size_t i) const { return get()[i]; }
  const T* data() const { return get().data(); }
  typename std::vector<T>::const_iterator begin() const { return get().begin(); }
  typename std::vector<T>::const_iterator end() const { return get().end(); }
  friend bool operator==(const HostMirror& a, const std::vector<T>& b) { return a.get() == b; }
  friend bool operator==(const std::vector<T>& b, const HostMirror& a) { return a.get() == b; }
  friend bool operator!=(const HostMirror& a, const std::vector<T>& b) { return !(a == b); }

 private:
  struct State {
    std::size_t n = 0;
    std::function<void(T*)> load;
    std::once_flag once;
    std::vector<T> v;
    bool ready = false;
  };
  std::shared_ptr<State> st_;
};

// Reusable plan (transform.hpp:28-47).  The public fields read as in the
// reference (sorted copies, stable permutations sorted[i] = orig[perm[i]]);
// their contents are fetched from the GPU plan on first access.  `device`
// owns the GPU-resident plan the applies run on.
struct TransformPlan {
  HostMirror<double> sorted_targets;
  HostMirror<double> sorted_sources;
  HostMirror<std::int64_t> target_perm;
  HostMirror<std::int64_t> source_perm;
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
