// C++ host API (include/fgt1d/*.hpp, namespace fgt) over the C ABI of the
// B200 transform (include/fgt1d_b200.h).  Mirrors the reference library's
// public surface for the transform path: same types, names, argument
// meaning and exception classes (proj/include/fgt1d/{transform,soe,cf,rng,
// errors}.hpp); every transform runs on the GPU.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iomanip>
#include <map>
#include <istream>
#include <limits>
#include <ostream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>

#include "../../include/fgt1d/cf.hpp"
#include "../../include/fgt1d/errors.hpp"
#include "../../include/fgt1d/rng.hpp"
#include "../../include/fgt1d/soe.hpp"
#include "../../include/fgt1d/transform.hpp"
#include "../../include/fgt1d_b200.h"
#include "../csrc/fgt_soe.hpp"

namespace fgt {

namespace {

[[noreturn]] void throw_status(int rc) {
  const std::string msg = fgt_last_error();
  switch (rc) {
    case FGT_ERR_DOMAIN:
      throw std::domain_error(msg);
    case FGT_ERR_INVALID:
      throw std::invalid_argument(msg);
    case FGT_ERR_NUMERICAL:
      throw numerical_error(msg);
    case FGT_ERR_NOMEM:
      throw std::bad_alloc();
    default:
      throw device_error(msg);
  }
}

void check(int rc) {
  if (rc != FGT_OK) throw_status(rc);
}

fgt_b200::Soe to_internal(const SoeApprox& s) {
  fgt_b200::Soe o;
  o.nodes = s.nodes;
  o.weights = s.weights;
  o.folded = s.form == SoeForm::Folded;
  o.self_conj = s.self_conjugate;
  return o;
}

SoeApprox from_internal(const fgt_b200::Soe& s) {
  SoeApprox o;
  o.nodes = s.nodes;
  o.weights = s.weights;
  o.form = s.folded ? SoeForm::Folded : SoeForm::Full;
  if (s.folded) o.self_conjugate = s.self_conj;
  return o;
}

template <class F>
auto soe_call(F&& f) -> decltype(f()) {
  try {
    return f();
  } catch (const fgt_b200::SoeError& e) {
    if (e.code == FGT_ERR_DOMAIN) throw std::domain_error(e.msg);
    throw std::invalid_argument(e.msg);
  }
}

constexpr double kUnderflowExponent = 745.0;  // transform.cpp:19

// Mode-by-mode evaluation of the folded / full SOE sum over a whole vector of
// scaled arguments s (sum_k m_k w_k exp(-t_k s), terms past the underflow
// exponent dropped), accumulated in Real.  One pass per mode keeps the
// per-mode constants in registers; the accumulation order over k is the
// mode order, as in the reference's scalar sum (soe.cpp:22-35).
template <class Real>
void soe_sum_into(const SoeApprox& soe, const std::vector<Real>& s, std::vector<Real>& out) {
  std::vector<std::complex<Real>> acc(s.size());
  for (std::size_t k = 0; k < soe.size(); ++k) {
    const std::complex<Real> t(soe.nodes[k].real(), soe.nodes[k].imag());
    const std::complex<Real> mw =
        Real(soe.multiplier(k)) *
        std::complex<Real>(soe.weights[k].real(), soe.weights[k].imag());
    for (std::size_t i = 0; i < s.size(); ++i)
      if (!(t.real() * s[i] > Real(kUnderflowExponent))) acc[i] += mw * std::exp(-t * s[i]);
  }
  out.resize(s.size());
  for (std::size_t i = 0; i < s.size(); ++i) out[i] = acc[i].real();
}

// max |exp(-x^2/4) - SOE(x)| over the standard log grid (soe.hpp:70-81).
// The grid is cut into one contiguous slice per hardware thread; each slice
// is evaluated vectorised (soe_sum_into) and reduced to its first maximum,
// then the slices are combined in grid order (first maximum overall).
template <class Real>
ErrorReport max_error_impl(const SoeApprox& soe) {
  validate(soe);
  const int total = kErrorGridLogPoints + 1;
  const unsigned hw = std::thread::hardware_concurrency();
  const int nslice = std::max(1, std::min(hw ? (int)hw : 1, 64));
  struct Best {
    double err = -1.0, x = 0.0;
  };
  std::vector<Best> best(nslice);
  auto slice = [&](int q) {
    const int i0 = (int)((int64_t)total * q / nslice), i1 = (int)((int64_t)total * (q + 1) / nslice);
    std::vector<Real> s(i1 - i0), g;
    for (int i = i0; i < i1; ++i) s[i - i0] = Real(error_grid_point(i));
    soe_sum_into<Real>(soe, s, g);
    for (int i = i0; i < i1; ++i) {
      const Real v = s[i - i0];
      const double e = (double)std::fabs(std::exp(-v * v / Real(4)) - g[i - i0]);
      if (e > best[q].err) best[q] = Best{e, (double)v};
    }
  };
  std::vector<std::thread> pool;
  for (int q = 1; q < nslice; ++q) pool.emplace_back(slice, q);
  slice(0);
  for (auto& th : pool) th.join();
  ErrorReport rep;
  for (std::size_t k = 0; k < soe.size(); ++k) rep.n += (int)soe.multiplier(k);
  Best b;
  for (const Best& q : best)
    if (q.err > b.err) b = q;
  rep.max_abs_error = b.err;
  rep.argmax_x = b.x;
  return rep;
}

struct PlanDeleter {
  void operator()(void* p) const { fgt_plan_destroy(static_cast<fgt_plan_t>(p)); }
};

fgt_plan_t handle(const TransformPlan& p) {
  if (!p.device) throw std::invalid_argument("plan has no device state");
  return static_cast<fgt_plan_t>(p.device.get());
}

TransformResult apply_impl(const TransformPlan& p, const std::vector<double>& strengths,
                           int threads, bool same) {
  if (strengths.size() != p.sorted_sources.size())
    throw std::invalid_argument("strengths length must match the planned source count");
  TransformResult res;
  res.potentials.assign(p.sorted_targets.size(), 0.0);
  const auto fn = same ? fgt_apply_same : fgt_apply_general;
  check(fn(handle(p), strengths.data(), (int64_t)strengths.size(), res.potentials.data(), threads,
           0, nullptr));
  return res;
}

}  // namespace

// ------------------------------------------------------------------ SOE

void validate(const SoeApprox& soe) {
  soe_call([&] {
    fgt_b200::soe_validate(to_internal(soe));
    return 0;
  });
}

double evaluate(const SoeApprox& soe, double x, double delta) {
  validate(soe);
  if (!std::isfinite(x)) throw std::domain_error("evaluate: x must be finite");
  if (!std::isfinite(delta) || !(delta > 0.0))
    throw std::domain_error("evaluate: delta must be positive and finite");
  std::vector<double> v{std::fabs(x) / std::sqrt(delta)}, g;
  soe_sum_into<double>(soe, v, g);
  return g[0];
}

SoeApprox fold(const SoeApprox& soe) {
  return soe_call([&] { return from_internal(fgt_b200::soe_fold(to_internal(soe))); });
}

SoeApprox unfold(const SoeApprox& soe) {
  return soe_call([&] { return from_internal(fgt_b200::soe_unfold(to_internal(soe))); });
}

double error_grid_point(int i) {
  if (i <= 0) return 0.0;
  const double frac = static_cast<double>(i - 1) / (kErrorGridLogPoints - 1);
  return std::pow(10.0, -5.0 + 7.0 * frac);
}

ErrorReport max_error(const SoeApprox& soe) { return max_error_impl<double>(soe); }
ErrorReport max_error_extended(const SoeApprox& soe) { return max_error_impl<long double>(soe); }

// Coefficient-table text format (soe.hpp:90-100): a header line
// "soe n=<count> form=<full|folded>[ source=<tag>]" and one row per node,
// "Re t  Im t  Re w  Im w" with 17 significant digits (exact round trip).
void write_coefficient_table(std::ostream& os, const SoeApprox& soe, const std::string& tag) {
  validate(soe);
  std::ostringstream out;
  out << "soe n=" << soe.size() << " form=" << (soe.form == SoeForm::Folded ? "folded" : "full")
      << (tag.empty() ? "" : " source=") << tag << '\n';
  out << std::scientific << std::setprecision(16);
  for (std::size_t k = 0; k < soe.size(); ++k)
    out << soe.nodes[k].real() << ' ' << soe.nodes[k].imag() << ' ' << soe.weights[k].real()
        << ' ' << soe.weights[k].imag() << '\n';
  os << out.str();
}

namespace {

// "key=value" fields of the header after the leading "soe" token.
std::map<std::string, std::string> table_header_fields(const std::string& line) {
  std::istringstream hs(line);
  std::string word;
  if (!(hs >> word) || word != "soe")
    throw std::invalid_argument("coefficient table: first line is not an 'soe' header");
  std::map<std::string, std::string> kv;
  while (hs >> word) {
    const std::size_t at = word.find('=');
    if (at == std::string::npos || at == 0)
      throw std::invalid_argument("coefficient table: header field without '=': " + word);
    kv[word.substr(0, at)] = word.substr(at + 1);
  }
  return kv;
}

// Four doubles of one row; false when the line holds anything else.
bool parse_row(const std::string& line, double (&v)[4]) {
  const char* p = line.c_str();
  for (double& d : v) {
    char* end = nullptr;
    d = std::strtod(p, &end);
    if (end == p) return false;
    p = end;
  }
  while (*p == ' ' || *p == '\t' || *p == '\r') ++p;
  return *p == '\0';
}

}  // namespace

SoeApprox read_coefficient_table(std::istream& is) {
  std::string line;
  if (!std::getline(is, line)) throw std::invalid_argument("coefficient table: no header line");
  const auto kv = table_header_fields(line);
  const auto fn = kv.find("n"), ff = kv.find("form");
  long n = -1;
  if (fn != kv.end()) {
    char* end = nullptr;
    n = std::strtol(fn->second.c_str(), &end, 10);
    if (fn->second.empty() || *end != '\0' || n < 0)
      throw std::invalid_argument("coefficient table: n is not a count: " + fn->second);
  }
  if (n < 0) throw std::invalid_argument("coefficient table: header has no n");
  if (ff == kv.end() || (ff->second != "full" && ff->second != "folded"))
    throw std::invalid_argument("coefficient table: form must be full or folded");
  SoeApprox out;
  out.form = ff->second == "folded" ? SoeForm::Folded : SoeForm::Full;
  while (std::getline(is, line)) {
    if (line.find_first_not_of(" \t\r") == std::string::npos) continue;  // blank
    double v[4];
    if (!parse_row(line, v))
      throw std::invalid_argument("coefficient table: row is not four numbers: " + line);
    if (out.form == SoeForm::Folded && v[1] < 0.0)
      throw std::invalid_argument("coefficient table: a folded node needs Im(t) >= 0");
    out.nodes.emplace_back(v[0], v[1]);
    out.weights.emplace_back(v[2], v[3]);
    if (out.form == SoeForm::Folded) out.self_conjugate.push_back(v[1] == 0.0 ? 1 : 0);
  }
  if ((long)out.size() != n)
    throw std::invalid_argument("coefficient table: " + std::to_string(out.size()) +
                                " rows, header says " + std::to_string(n));
  validate(out);
  return out;
}

void save_coefficient_table(const std::string& path, const SoeApprox& soe,
                            const std::string& tag) {
  std::ofstream f(path);
  if (!f) throw std::invalid_argument("cannot open for writing: " + path);
  write_coefficient_table(f, soe, tag);
}

SoeApprox load_coefficient_table(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw std::invalid_argument("cannot open for reading: " + path);
  return read_coefficient_table(f);
}

SoeApprox cf_soe(int n) {
  return soe_call([&] { return from_internal(fgt_b200::soe_cf(n)); });
}

SoeApprox soe_for_tolerance(double tol) {
  const int ne = fgt_mode_count_for_tolerance(tol);
  if (ne < 0) throw_status(-ne);
  return fold(cf_soe(2 * ne));
}

// ------------------------------------------------------------ transform

namespace {

fgt_plan_t device_plan(const TransformRequest& req, const SoeApprox& folded) {
  const std::size_t ne = folded.size();
  std::vector<double> tr(ne), ti(ne), wr(ne), wi(ne);
  std::vector<std::uint8_t> sc(ne, 0);
  for (std::size_t k = 0; k < ne; ++k) {
    tr[k] = folded.nodes[k].real();
    ti[k] = folded.nodes[k].imag();
    wr[k] = folded.weights[k].real();
    wi[k] = folded.weights[k].imag();
    sc[k] = folded.self_conjugate[k];
  }
  fgt_plan_t h = nullptr;
  check(fgt_plan_create(req.targets.data(), (int64_t)req.targets.size(), req.sources.data(),
                        (int64_t)req.sources.size(), req.delta, tr.data(), ti.data(), wr.data(),
                        wi.data(), sc.data(), (int)ne, FGT_SOE_FOLDED, 0, -1, nullptr, &h));
  return h;
}

}  // namespace

TransformPlan plan(const TransformRequest& req, const SoeApprox& soe, bool precompute) {
  // Validation order of transform.cpp:200-211: delta, target / source
  // coordinates (checked on the device by the plan's check pass), strength
  // count, SOE.
  if (!std::isfinite(req.delta) || !(req.delta > 0.0))
    throw std::domain_error("delta must be positive and finite");
  const bool count_ok = req.strengths.size() == req.sources.size();
  bool soe_ok = true;
  try {
    validate(soe);
  } catch (const std::invalid_argument&) {
    soe_ok = false;
  }
  if (!count_ok || !soe_ok) {
    // the coordinates are still checked first (a stand-in SOE for the check)
    fgt_plan_destroy(device_plan(req, fold(cf_soe(2))));
    if (!count_ok) throw std::invalid_argument("one strength per source required");
    validate(soe);  // throws
  }
  TransformPlan p;
  p.soe = soe.form == SoeForm::Folded ? soe : fold(soe);
  p.delta = req.delta;
  fgt_plan_t h = device_plan(req, p.soe);
  std::shared_ptr<void> dev(h, PlanDeleter{});
  p.device = dev;
  int same = 0;
  check(fgt_plan_info(h, nullptr, nullptr, nullptr, &same, nullptr, nullptr, nullptr));
  p.same_points = same != 0;
  // host fields on first access (lazily populated)
  p.sorted_targets = HostMirror<double>(req.targets.size(), [dev](double* o) {
    check(fgt_plan_copy_sorted(static_cast<fgt_plan_t>(dev.get()), o, nullptr, nullptr, nullptr));
  });
  p.sorted_sources = HostMirror<double>(req.sources.size(), [dev](double* o) {
    check(fgt_plan_copy_sorted(static_cast<fgt_plan_t>(dev.get()), nullptr, nullptr, o, nullptr));
  });
  p.target_perm = HostMirror<std::int64_t>(req.targets.size(), [dev](std::int64_t* o) {
    check(fgt_plan_copy_sorted(static_cast<fgt_plan_t>(dev.get()), nullptr, o, nullptr, nullptr));
  });
  p.source_perm = HostMirror<std::int64_t>(req.sources.size(), [dev](std::int64_t* o) {
    check(fgt_plan_copy_sorted(static_cast<fgt_plan_t>(dev.get()), nullptr, nullptr, nullptr, o));
  });
  if (precompute) precompute_gap_table(p);
  return p;
}

void precompute_gap_table(TransformPlan& p) {
  if (p.precomputed) return;
  const std::size_t M = p.sorted_targets.size(), ne = p.soe.size();
  p.gap_exponentials.clear();
  if (M >= 2 && ne > 0) {
    p.gap_exponentials.resize(ne * (M - 1));
    check(fgt_plan_gap_table(handle(p), reinterpret_cast<double*>(p.gap_exponentials.data())));
  }
  p.precomputed = true;
}

TransformResult apply_same(const TransformPlan& p, const std::vector<double>& strengths,
                           int num_threads) {
  if (!p.same_points)
    throw std::invalid_argument(
        "apply_same requires a plan built from identical target and source sets");
  return apply_impl(p, strengths, num_threads, true);
}

TransformResult apply_general(const TransformPlan& p, const std::vector<double>& strengths,
                              int num_threads) {
  return apply_impl(p, strengths, num_threads, false);
}

TransformResult direct(const TransformRequest& req, const std::vector<std::int64_t>& subset) {
  if (req.strengths.size() != req.sources.size())
    throw std::invalid_argument("one strength per source required");
  TransformResult res;
  res.potentials.resize(subset.empty() ? req.targets.size() : subset.size());
  check(fgt_direct(req.targets.data(), (int64_t)req.targets.size(), req.sources.data(),
                   (int64_t)req.sources.size(), req.strengths.data(), req.delta,
                   subset.empty() ? nullptr : subset.data(), (int64_t)subset.size(),
                   res.potentials.data()));
  return res;
}

int preset_mode_count(Precision p) {
  const int r = fgt_preset_mode_count(static_cast<int>(p));
  if (r < 0) throw std::domain_error("unknown precision preset");
  return r;
}

SoeApprox preset_soe(Precision p) { return fold(cf_soe(2 * preset_mode_count(p))); }

namespace detail {

ModeSums mode_sums(const TransformPlan& p, const std::vector<double>& strengths) {
  if (strengths.size() != p.sorted_sources.size())
    throw std::invalid_argument("strengths length must match the planned source count");
  const std::size_t ne = p.soe.size(), M = p.sorted_targets.size();
  std::vector<std::complex<double>> hp(ne * M), hm(ne * M);
  check(fgt_mode_sums(handle(p), strengths.data(), reinterpret_cast<double*>(hp.data()),
                      reinterpret_cast<double*>(hm.data())));
  ModeSums out;
  out.hp.assign(ne, {});
  out.hm.assign(ne, {});
  for (std::size_t k = 0; k < ne; ++k) {
    out.hp[k].assign(hp.begin() + k * M, hp.begin() + (k + 1) * M);
    out.hm[k].assign(hm.begin() + k * M, hm.begin() + (k + 1) * M);
  }
  return out;
}

}  // namespace detail

// ------------------------------------------------------------------ rng

namespace rng {

std::uint64_t mix64(std::uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

std::uint64_t counter_rand(std::uint64_t seed, std::uint64_t stream, std::uint64_t i) {
  return mix64(mix64(seed ^ stream * 0xA24BAED4963EE407ull) + i * 0x9E3779B97F4A7C15ull);
}

double uniform01(std::uint64_t seed, std::uint64_t stream, std::uint64_t i) {
  return static_cast<double>(counter_rand(seed, stream, i) >> 11) * 0x1.0p-53;
}

std::vector<double> uniform_points(std::size_t count, std::uint64_t seed, std::uint64_t stream) {
  std::vector<double> out(count);
  for (std::size_t i = 0; i < count; ++i) out[i] = uniform01(seed, stream, i);
  return out;
}

std::vector<double> chebyshev_points(std::size_t count) {
  const double pi = 3.14159265358979323846;
  std::vector<double> out(count);
  for (std::size_t i = 1; i <= count; ++i)
    out[i - 1] = (1.0 + std::cos(pi * (2.0 * (double)i - 1.0) / (2.0 * (double)count))) / 2.0;
  return out;
}

}  // namespace rng

}  // namespace fgt
