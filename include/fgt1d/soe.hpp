#pragma once
// Sum-of-exponentials approximation of the Gaussian kernel -- the API of the
// reference's proj/include/fgt1d/soe.hpp:24-108 (SoeApprox, validate,
// evaluate, fold / unfold, max_error, coefficient-table I/O).
#include <complex>
#include <cstddef>
#include <cstdint>
#include <iosfwd>
#include <string>
#include <vector>

namespace fgt {

enum class SoeForm { Full, Folded };

struct SoeApprox {
  std::vector<std::complex<double>> nodes;    // t_k, Re(t_k) > 0
  std::vector<std::complex<double>> weights;  // w_k
  SoeForm form = SoeForm::Full;
  std::vector<std::uint8_t> self_conjugate;   // folded only

  std::size_t size() const { return nodes.size(); }
  double multiplier(std::size_t k) const {
    if (form == SoeForm::Full) return 1.0;
    return self_conjugate[k] ? 1.0 : 2.0;
  }
};

void validate(const SoeApprox& soe);
double evaluate(const SoeApprox& soe, double x, double delta);
SoeApprox fold(const SoeApprox& soe);
SoeApprox unfold(const SoeApprox& soe);

struct ErrorReport {
  int n = 0;
  double max_abs_error = 0.0;
  double argmax_x = 0.0;
};

inline constexpr int kErrorGridLogPoints = 100000;
double error_grid_point(int i);
ErrorReport max_error(const SoeApprox& soe);
ErrorReport max_error_extended(const SoeApprox& soe);

void write_coefficient_table(std::ostream& os, const SoeApprox& soe,
                             const std::string& source_tag);
SoeApprox read_coefficient_table(std::istream& is);
void save_coefficient_table(const std::string& path, const SoeApprox& soe,
                            const std::string& source_tag);
SoeApprox load_coefficient_table(const std::string& path);

}  // namespace fgt
