// Host SOE utilities behind the C ABI: table lookup, validation, folding.
#include "fgt_soe.hpp"

#include <algorithm>
#include <cmath>
#include <sstream>

#include "../../include/fgt1d_b200.h"

namespace fgt_b200 {

namespace {
#include "soe_tables.inc"

[[noreturn]] void fail(int code, const std::string& m) { throw SoeError{code, m}; }

bool finite_c(std::complex<double> z) { return std::isfinite(z.real()) && std::isfinite(z.imag()); }

bool node_less(const std::pair<std::complex<double>, std::complex<double>>& a,
               const std::pair<std::complex<double>, std::complex<double>>& b) {
  if (a.first.real() != b.first.real()) return a.first.real() < b.first.real();
  return a.first.imag() < b.first.imag();
}
}  // namespace

// soe.cpp:107-132 -- same checks, same error class (invalid_argument).
void soe_validate(const Soe& s) {
  if (s.nodes.size() != s.weights.size()) fail(FGT_ERR_INVALID, "SOE node/weight count mismatch");
  if (s.folded) {
    if (s.self_conj.size() != s.nodes.size())
      fail(FGT_ERR_INVALID, "folded SOE requires one self-conjugate flag per node");
  } else if (!s.self_conj.empty()) {
    fail(FGT_ERR_INVALID, "full-form SOE must not carry fold flags");
  }
  for (size_t k = 0; k < s.nodes.size(); ++k) {
    if (!finite_c(s.nodes[k]) || !finite_c(s.weights[k]))
      fail(FGT_ERR_INVALID, "SOE coefficients must be finite");
    if (!(s.nodes[k].real() > 0.0))
      fail(FGT_ERR_INVALID, "SOE nodes must lie in the open right half-plane");
    if (s.folded) {
      if (s.nodes[k].imag() < 0.0)
        fail(FGT_ERR_INVALID, "folded SOE stores the Im(t) >= 0 representative of each pair");
      if (s.self_conj[k] && s.nodes[k].imag() != 0.0)
        fail(FGT_ERR_INVALID, "self-conjugate folded node must have a real t");
    }
  }
}

// soe.cpp:143-215: canonicalise near-real nodes (|Im t| <= 1e-12 |t|), pair
// each upper node with its unused conjugate (tolerance 1e-12 |t|), average the
// pair, order by (Re t, Im t).
Soe soe_fold(const Soe& s) {
  soe_validate(s);
  if (s.folded) return s;
  const size_t n = s.nodes.size();
  std::vector<int> kind(n, 0);
  for (size_t k = 0; k < n; ++k) {
    const double mag = std::abs(s.nodes[k]);
    if (std::fabs(s.nodes[k].imag()) <= 1e-12 * mag) {
      if (std::fabs(s.weights[k].imag()) > 1e-9 * (1.0 + std::abs(s.weights[k])))
        fail(FGT_ERR_INVALID, "fold: real node " + std::to_string(k) +
                                  " carries a non-real weight; the sum cannot be real-valued");
      kind[k] = 0;
    } else {
      kind[k] = s.nodes[k].imag() > 0.0 ? 1 : -1;
    }
  }
  std::vector<char> used(n, 0);
  std::vector<std::pair<std::complex<double>, std::complex<double>>> ent;
  std::vector<uint8_t> flags;
  for (size_t k = 0; k < n; ++k) {
    if (used[k]) continue;
    if (kind[k] == 0) {
      used[k] = 1;
      ent.push_back({{s.nodes[k].real(), 0.0}, {s.weights[k].real(), 0.0}});
      flags.push_back(1);
      continue;
    }
    const std::complex<double> want = std::conj(s.nodes[k]);
    const double tol = 1e-12 * std::abs(s.nodes[k]);
    size_t match = n;
    for (size_t j = 0; j < n; ++j) {
      if (j == k || used[j] || kind[j] == 0 || kind[j] == kind[k]) continue;
      if (std::abs(s.nodes[j] - want) <= tol) {
        match = j;
        break;
      }
    }
    if (match == n) {
      std::ostringstream m;
      m << "fold: node " << k << " (t = " << s.nodes[k].real() << " + " << s.nodes[k].imag()
        << "i) has no conjugate partner";
      fail(FGT_ERR_INVALID, m.str());
    }
    used[k] = used[match] = 1;
    const size_t up = kind[k] > 0 ? k : match;
    const size_t dn = kind[k] > 0 ? match : k;
    ent.push_back({0.5 * (s.nodes[up] + std::conj(s.nodes[dn])),
                   0.5 * (s.weights[up] + std::conj(s.weights[dn]))});
    flags.push_back(0);
  }
  std::vector<size_t> idx(ent.size());
  for (size_t i = 0; i < idx.size(); ++i) idx[i] = i;
  std::sort(idx.begin(), idx.end(), [&](size_t a, size_t b) { return node_less(ent[a], ent[b]); });
  Soe out;
  out.folded = true;
  for (size_t i : idx) {
    out.nodes.push_back(ent[i].first);
    out.weights.push_back(ent[i].second);
    out.self_conj.push_back(flags[i]);
  }
  return out;
}

// soe.cpp:217-235
Soe soe_unfold(const Soe& s) {
  soe_validate(s);
  if (!s.folded) return s;
  std::vector<std::pair<std::complex<double>, std::complex<double>>> ent;
  for (size_t k = 0; k < s.nodes.size(); ++k) {
    ent.push_back({s.nodes[k], s.weights[k]});
    if (!s.self_conj[k]) ent.push_back({std::conj(s.nodes[k]), std::conj(s.weights[k])});
  }
  std::sort(ent.begin(), ent.end(), node_less);
  Soe out;
  for (auto& e : ent) {
    out.nodes.push_back(e.first);
    out.weights.push_back(e.second);
  }
  return out;
}

Soe soe_cf(int n) {
  if (n < 2 || n > 14)
    fail(FGT_ERR_DOMAIN,
         "rational construction supports orders 2..14 (beyond that the double-precision "
         "Hankel SVD cannot resolve the coefficients)");
  Soe s;
  const double* r = kCfTable + kCfOffset[n];
  for (int k = 0; k < n; ++k) {
    s.nodes.emplace_back(r[4 * k + 0], r[4 * k + 1]);
    s.weights.emplace_back(r[4 * k + 2], r[4 * k + 3]);
  }
  return s;
}

}  // namespace fgt_b200
