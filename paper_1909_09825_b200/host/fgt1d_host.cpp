// C++ host API (include/fgt1d/*.hpp, namespace fgt) over the C ABI of the
// B200 transform (include/fgt1d_b200.h).  Mirrors the reference library's
// public surface for the transform path: same types, names, argument
// meaning and exception classes (proj/include/fgt1d/{transform,soe,cf,rng,
// errors}.hpp); every transform runs on the GPU.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <fstream>
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

constexpr double kUnderflowExponent = 745.0;

template <class Real>
Real eval_sum(const SoeApprox& soe, Real s) {
  std::complex<Real> acc{};
  for (std::size_t k = 0; k < soe.size(); ++k) {
    std::complex<Real> t(soe.nodes[k].real(), soe.nodes[k].imag());
    if (t.real() * s > Real(kUnderflowExponent)) continue;
    std::complex<Real> w(soe.weights[k].real(), soe.weights[k].imag());
    acc += Real(soe.multiplier(k)) * w * std::exp(-t * s);
  }
  return acc.real();
}

template <class Real>
ErrorReport max_error_impl(const SoeApprox& soe) {
  validate(soe);
  constexpr int kChunk = 4096;
  const int total = kErrorGridLogPoints + 1;
  const int nchunks = (total + kChunk - 1) / kChunk;
  std::vector<double> err(nchunks, 0.0), arg(nchunks, 0.0);
  auto run = [&](int c) {
    double best = -1.0, bx = 0.0;
    for (int i = c * kChunk; i < std::min(total, (c + 1) * kChunk); ++i) {
      const double x = error_grid_point(i);
      const Real s = Real(x);
      const double e =
          static_cast<double>(std::fabs(std::exp(-s * s / Real(4)) - eval_sum<Real>(soe, s)));
      if (e > best) {
        best = e;
        bx = x;
      }
    }
    err[c] = best;
    arg[c] = bx;
  };
  unsigned hw = std::thread::hardware_concurrency();
  int nt = std::max(1, std::min<int>(hw ? (int)hw : 1, nchunks));
  std::vector<std::thread> pool;
  for (int t = 0; t < nt; ++t)
    pool.emplace_back([&, t] {
      for (int c = t; c < nchunks; c += nt) run(c);
    });
  for (auto& th : pool) th.join();
  ErrorReport rep;
  for (std::size_t k = 0; k < soe.size(); ++k) rep.n += (int)soe.multiplier(k);
  double best = -1.0;
  for (int c = 0; c < nchunks; ++c)
    if (err[c] > best) {
      best = err[c];
      rep.argmax_x = arg[c];
    }
  rep.max_abs_error = best;
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
  return eval_sum<double>(soe, std::fabs(x) / std::sqrt(delta));
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

void write_coefficient_table(std::ostream& os, const SoeApprox& soe, const std::string& tag) {
  validate(soe);
  os << "soe n=" << soe.size() << " form=" << (soe.form == SoeForm::Folded ? "folded" : "full");
  if (!tag.empty()) os << " source=" << tag;
  os << "\n";
  char buf[160];
  for (std::size_t k = 0; k < soe.size(); ++k) {
    std::snprintf(buf, sizeof buf, "%.16e %.16e %.16e %.16e\n", soe.nodes[k].real(),
                  soe.nodes[k].imag(), soe.weights[k].real(), soe.weights[k].imag());
    os << buf;
  }
}

SoeApprox read_coefficient_table(std::istream& is) {
  std::string header;
  if (!std::getline(is, header)) throw std::invalid_argument("coefficient table: empty input");
  std::istringstream hs(header);
  std::string tag;
  hs >> tag;
  if (tag != "soe") throw std::invalid_argument("coefficient table: header must start with 'soe'");
  long n = -1;
  std::string form, kv;
  while (hs >> kv) {
    const auto eq = kv.find('=');
    if (eq == std::string::npos)
      throw std::invalid_argument("coefficient table: malformed header field '" + kv + "'");
    const std::string key = kv.substr(0, eq), val = kv.substr(eq + 1);
    if (key == "n") {
      try {
        n = std::stol(val);
      } catch (const std::exception&) {
        throw std::invalid_argument("coefficient table: bad n value");
      }
    } else if (key == "form") {
      form = val;
    }
  }
  if (n < 0) throw std::invalid_argument("coefficient table: missing n");
  if (form != "full" && form != "folded")
    throw std::invalid_argument("coefficient table: missing or bad form");
  SoeApprox out;
  out.form = form == "folded" ? SoeForm::Folded : SoeForm::Full;
  std::string line;
  while (std::getline(is, line)) {
    if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
    std::istringstream ls(line);
    double tr, ti, wr, wi;
    if (!(ls >> tr >> ti >> wr >> wi))
      throw std::invalid_argument("coefficient table: malformed row '" + line + "'");
    out.nodes.emplace_back(tr, ti);
    out.weights.emplace_back(wr, wi);
    if (out.form == SoeForm::Folded) {
      if (ti < 0.0) throw std::invalid_argument("coefficient table: folded rows must have Im(t) >= 0");
      out.self_conjugate.push_back(ti == 0.0 ? 1 : 0);
    }
  }
  if (static_cast<long>(out.size()) != n)
    throw std::invalid_argument("coefficient table: row count does not match header n");
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

TransformPlan plan(const TransformRequest& req, const SoeApprox& soe, bool precompute) {
  // validation order of transform.cpp:200-211
  if (!std::isfinite(req.delta) || !(req.delta > 0.0))
    throw std::domain_error("delta must be positive and finite");
  for (double x : req.targets)
    if (!std::isfinite(x)) throw std::domain_error("target coordinates must be finite");
  for (double y : req.sources)
    if (!std::isfinite(y)) throw std::domain_error("source coordinates must be finite");
  if (req.strengths.size() != req.sources.size())
    throw std::invalid_argument("one strength per source required");
  validate(soe);
  TransformPlan p;
  p.soe = soe.form == SoeForm::Folded ? soe : fold(soe);
  p.delta = req.delta;
  const std::size_t ne = p.soe.size();
  std::vector<double> tr(ne), ti(ne), wr(ne), wi(ne);
  for (std::size_t k = 0; k < ne; ++k) {
    tr[k] = p.soe.nodes[k].real();
    ti[k] = p.soe.nodes[k].imag();
    wr[k] = p.soe.weights[k].real();
    wi[k] = p.soe.weights[k].imag();
  }
  fgt_plan_t h = nullptr;
  check(fgt_plan_create(req.targets.data(), (int64_t)req.targets.size(), req.sources.data(),
                        (int64_t)req.sources.size(), req.delta, tr.data(), ti.data(), wr.data(),
                        wi.data(), p.soe.self_conjugate.data(), (int)ne, FGT_SOE_FOLDED, 0, -1,
                        nullptr, &h));
  p.device = std::shared_ptr<void>(h, PlanDeleter{});
  int same = 0;
  check(fgt_plan_info(h, nullptr, nullptr, nullptr, &same, nullptr, nullptr, nullptr));
  p.same_points = same != 0;
  p.sorted_targets.resize(req.targets.size());
  p.sorted_sources.resize(req.sources.size());
  p.target_perm.resize(req.targets.size());
  p.source_perm.resize(req.sources.size());
  check(fgt_plan_copy_sorted(h, p.sorted_targets.data(), p.target_perm.data(),
                             p.sorted_sources.data(), p.source_perm.data()));
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
