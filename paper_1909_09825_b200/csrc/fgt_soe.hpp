// Host-side SOE representation used behind the C ABI.
// Semantics follow the reference SoeApprox (proj/include/fgt1d/soe.hpp:24-39),
// validate (proj/src/soe.cpp:107-132) and fold (proj/src/soe.cpp:143-215).
#pragma once

#include <complex>
#include <cstdint>
#include <string>
#include <vector>

namespace fgt_b200 {

struct Soe {
  std::vector<std::complex<double>> nodes;
  std::vector<std::complex<double>> weights;
  bool folded = false;
  std::vector<uint8_t> self_conj;  // folded only
  double multiplier(size_t k) const { return !folded ? 1.0 : (self_conj[k] ? 1.0 : 2.0); }
};

struct SoeError {
  int code;  // FGT_ERR_*
  std::string msg;
};

// Throw SoeError on violation.
void soe_validate(const Soe& s);
Soe soe_fold(const Soe& s);
Soe soe_unfold(const Soe& s);
Soe soe_cf(int n);  // compiled-in table, full form

}  // namespace fgt_b200
