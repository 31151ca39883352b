// C++ API tests of the drop-in host library (include/fgt1d/*.hpp).
// The cases follow the reference's own unit tests for the transform path
// (proj/tests/test_transform.cpp, test_rng.cpp, test_soe.cpp) through the
// same public interface.  Usage: test_fgt1d_api cpu|gpu  (exit code = #fails)
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <functional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "fgt1d/cf.hpp"
#include "fgt1d/errors.hpp"
#include "fgt1d/rng.hpp"
#include "fgt1d/soe.hpp"
#include "fgt1d/transform.hpp"

namespace {

int g_fail = 0, g_checks = 0;
std::string g_case;

#define CHECK(cond)                                                          \
  do {                                                                       \
    ++g_checks;                                                              \
    if (!(cond)) {                                                           \
      ++g_fail;                                                              \
      std::printf("FAIL [%s] %s:%d: %s\n", g_case.c_str(), __FILE__, __LINE__, #cond); \
    }                                                                        \
  } while (0)

template <class E, class F>
bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

using fgt::TransformRequest;

const std::vector<double> kYs = {0.0, 0.1, 0.35, 0.5, 0.75, 1.0};
const std::vector<double> kAs = {0.5, -0.25, 1.0, 0.8, -0.6, 0.9};
const std::vector<double> kXs = {0.0, 0.5, 1.0};
const std::vector<double> kGold = {0.53026354628615822, 1.3078174711896560, 0.66552744606900788};

TransformRequest golden() { return TransformRequest{kXs, kYs, kAs, 0.02}; }

TransformRequest random_request(std::uint64_t seed, std::size_t n, std::size_t m, double delta) {
  TransformRequest r;
  r.targets = fgt::rng::uniform_points(n, seed, fgt::rng::kStreamTargets);
  r.sources = fgt::rng::uniform_points(m, seed, fgt::rng::kStreamSources);
  r.strengths.resize(m);
  for (std::size_t j = 0; j < m; ++j)
    r.strengths[j] = 2.0 * fgt::rng::uniform01(seed, fgt::rng::kStreamStrengths, j) - 1.0;
  r.delta = delta;
  return r;
}

double max_abs_diff(const std::vector<double>& a, const std::vector<double>& b) {
  if (a.size() != b.size()) return INFINITY;
  double w = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) w = std::max(w, std::fabs(a[i] - b[i]));
  return w;
}

void run(const char* name, const std::function<void()>& f) {
  g_case = name;
  try {
    f();
  } catch (const std::exception& e) {
    ++g_fail;
    std::printf("FAIL [%s] unexpected exception: %s\n", name, e.what());
  }
}

// ----------------------------------------------------------------- CPU

void cpu_tests() {
  run("rng pins", [] {
    CHECK(fgt::rng::counter_rand(0, 0, 0) == 0xa706dd2f4d197e6full);
    CHECK(fgt::rng::counter_rand(42, 1, 7) == 0x8d3b7fd7abb430aeull);
    CHECK(fgt::rng::counter_rand(123456789, 3, 1000000) == 0x2ca992c901c93cedull);
    CHECK(fgt::rng::uniform01(0, 0, 0) == 0.65244848637403219);
    auto ch = fgt::rng::chebyshev_points(5);
    CHECK(ch.size() == 5 && std::fabs(ch[0] - (1 + std::cos(M_PI / 10)) / 2) < 1e-15);
  });
  run("cf tables and presets", [] {
    CHECK(fgt::cf_soe(12).size() == 12);
    CHECK(fgt::cf_soe(12).form == fgt::SoeForm::Full);
    CHECK(throws<std::domain_error>([] { fgt::cf_soe(1); }));
    CHECK(throws<std::domain_error>([] { fgt::cf_soe(15); }));
    using fgt::Precision;
    CHECK(fgt::preset_mode_count(Precision::Digits4) == 3);
    CHECK(fgt::preset_mode_count(Precision::Digits11) == 6);
    auto s = fgt::preset_soe(Precision::Digits9);
    CHECK(s.form == fgt::SoeForm::Folded && s.size() == 5);
    CHECK(fgt::soe_for_tolerance(1e-10).size() == 6);
    CHECK(fgt::soe_for_tolerance(1e-6).size() == 4);
  });
  run("max_error pins (test_cf.cpp:20-23)", [] {
    const struct {
      int n;
      double e;
    } pins[] = {{6, 7.2279e-5}, {8, 1.2570e-6}, {12, 3.0208e-10}};
    for (auto p : pins) {
      auto rep = fgt::max_error(fgt::cf_soe(p.n));
      CHECK(rep.n == p.n);
      CHECK(std::fabs(rep.max_abs_error - p.e) <= 0.05 * p.e);
      CHECK(rep.argmax_x == 0.0);
    }
    // folding changes the sum only at roundoff
    auto f = fgt::fold(fgt::cf_soe(12));
    CHECK(std::fabs(fgt::max_error(f).max_abs_error - 3.0208e-10) <= 0.05 * 3.0208e-10);
  });
  run("fold / unfold / evaluate", [] {
    auto full = fgt::cf_soe(7);
    auto fo = fgt::fold(full);
    CHECK(fo.size() == 4);
    int selfc = 0;
    for (auto b : fo.self_conjugate) selfc += b;
    CHECK(selfc == 1);
    CHECK(fgt::unfold(fo).size() == 7);
    for (double x : {0.0, 0.3, 1.7})
      CHECK(std::fabs(fgt::evaluate(full, x, 1.0) - fgt::evaluate(fo, x, 1.0)) < 1e-13);
    fgt::SoeApprox bad;
    bad.nodes = {{1.0, 1.0}};
    bad.weights = {{1.0, 0.0}};
    CHECK(throws<std::invalid_argument>([&] { fgt::fold(bad); }));
    CHECK(throws<std::domain_error>([&] { fgt::evaluate(full, NAN, 1.0); }));
  });
  run("coefficient table round trip", [] {
    auto s = fgt::fold(fgt::cf_soe(9));
    std::stringstream ss;
    fgt::write_coefficient_table(ss, s, "test");
    auto back = fgt::read_coefficient_table(ss);
    CHECK(back.form == s.form && back.nodes == s.nodes && back.weights == s.weights &&
          back.self_conjugate == s.self_conjugate);
    std::stringstream bad("soe n=2 form=full\n1 0 1 0\n");
    CHECK(throws<std::invalid_argument>([&] { fgt::read_coefficient_table(bad); }));
  });
  run("plan validation (test_transform.cpp:260-280)", [] {
    auto soe = fgt::fold(fgt::cf_soe(8));
    auto r = golden();
    r.delta = 0.0;
    CHECK(throws<std::domain_error>([&] { fgt::plan(r, soe, false); }));
    r = golden();
    r.delta = -2.0;
    CHECK(throws<std::domain_error>([&] { fgt::plan(r, soe, false); }));
    // coordinates and the strength count are checked after the device's
    // coordinate pass (gpu_tests: "plan validation on the device")
  });
}

// ----------------------------------------------------------------- GPU

void gpu_tests() {
  run("plan validation on the device (test_transform.cpp:260-280)", [] {
    auto soe = fgt::fold(fgt::cf_soe(8));
    auto r = golden();
    r.targets[1] = NAN;
    CHECK(throws<std::domain_error>([&] { fgt::plan(r, soe, false); }));
    r = golden();
    r.sources[4] = INFINITY;
    CHECK(throws<std::domain_error>([&] { fgt::plan(r, soe, false); }));
    r = golden();
    r.strengths.pop_back();
    CHECK(throws<std::invalid_argument>([&] { fgt::plan(r, soe, false); }));
    // coordinates first: a NaN and a short strength vector -> domain_error
    r.targets[0] = NAN;
    CHECK(throws<std::domain_error>([&] { fgt::plan(r, soe, false); }));
    // strength count before the SOE (transform.cpp:205-208)
    auto bad = soe;
    bad.nodes[0] = {-1.0, 0.0};
    r = golden();
    r.strengths.pop_back();
    bool msg_ok = false;
    try {
      fgt::plan(r, bad, false);
    } catch (const std::invalid_argument& e) {
      msg_ok = std::string(e.what()).find("strength") != std::string::npos;
    }
    CHECK(msg_ok);
    // lazily populated host fields: sizes known, contents on first access
    r = golden();
    std::swap(r.targets[0], r.targets[2]);
    auto p = fgt::plan(r, soe, false);
    CHECK(p.sorted_targets.size() == 3 && p.target_perm.size() == 3);
    CHECK(p.target_perm == (std::vector<std::int64_t>{2, 1, 0}));
    CHECK(p.sorted_targets[0] == 0.0 && p.sorted_targets[2] == 1.0);
    const std::vector<double>& sv = p.sorted_sources;
    CHECK(sv == kYs);
  });
  run("direct matches the 50-digit reference", [] {
    auto res = fgt::direct(golden());
    for (int i = 0; i < 3; ++i) CHECK(std::fabs(res.potentials[i] - kGold[i]) <= 1e-15 * kGold[i]);
  });
  run("fast transform within SOE accuracy", [] {
    auto p = fgt::plan(golden(), fgt::fold(fgt::cf_soe(12)), true);
    CHECK(!p.same_points);
    auto r = fgt::apply_general(p, kAs);
    for (int i = 0; i < 3; ++i) CHECK(std::fabs(r.potentials[i] - kGold[i]) < 5e-9);
  });
  run("direct subset", [] {
    auto all = fgt::direct(golden());
    auto sub = fgt::direct(golden(), {2, 0});
    CHECK(sub.potentials.size() == 2 && sub.potentials[0] == all.potentials[2] &&
          sub.potentials[1] == all.potentials[0]);
    CHECK(throws<std::invalid_argument>([] { fgt::direct(golden(), {3}); }));
    CHECK(throws<std::invalid_argument>([] { fgt::direct(golden(), {-1}); }));
  });
  run("same-point and general scans agree", [] {
    auto r = random_request(11, 500, 500, 0.37);
    r.targets = r.sources;
    auto soe = fgt::fold(fgt::cf_soe(10));
    auto p = fgt::plan(r, soe, false);
    CHECK(p.same_points);
    auto a = fgt::apply_same(p, r.strengths);
    auto b = fgt::apply_general(p, r.strengths);
    CHECK(max_abs_diff(a.potentials, b.potentials) < 1e-13);
    auto o = fgt::direct(r);
    double mass = 0;
    for (double v : r.strengths) mass += std::fabs(v);
    CHECK(max_abs_diff(a.potentials, o.potentials) < fgt::max_error(soe).max_abs_error * mass);
  });
  run("ties", [] {
    TransformRequest r{{0.3, 0.5, 0.7, 0.9, 0.3}, {0.3, 0.3, 0.7, 0.7, 0.7},
                       {1.0, -2.0, 0.5, 0.5, 0.25}, 0.05};
    auto p = fgt::plan(r, fgt::fold(fgt::cf_soe(12)), false);
    CHECK(max_abs_diff(fgt::apply_general(p, r.strengths).potentials, fgt::direct(r).potentials) <
          1e-8);
  });
  run("empty inputs", [] {
    auto soe = fgt::fold(fgt::cf_soe(8));
    TransformRequest a{{0.1, 0.9}, {}, {}, 1.0};
    auto r1 = fgt::apply_general(fgt::plan(a, soe, false), {});
    CHECK(r1.potentials.size() == 2 && r1.potentials[0] == 0.0 && r1.potentials[1] == 0.0);
    CHECK(fgt::direct(a).potentials[0] == 0.0);
    TransformRequest b{{}, {0.5}, {2.0}, 1.0};
    CHECK(fgt::apply_general(fgt::plan(b, soe, false), {2.0}).potentials.empty());
  });
  run("plan reuse across strength vectors", [] {
    auto r = random_request(3, 200, 300, 2.0);
    auto p = fgt::plan(r, fgt::fold(fgt::cf_soe(12)), true);
    auto r1 = fgt::apply_general(p, r.strengths);
    std::vector<double> b2(300);
    for (int j = 0; j < 300; ++j) b2[j] = std::sin(0.1 * (j + 1));
    auto r2 = fgt::apply_general(p, b2);
    auto r2req = r;
    r2req.strengths = b2;
    double scale = 0;
    for (double v : b2) scale += std::fabs(v);
    CHECK(max_abs_diff(r2.potentials, fgt::direct(r2req).potentials) < 1e-9 * scale);
    CHECK(max_abs_diff(r1.potentials, fgt::apply_general(p, r.strengths).potentials) == 0.0);
  });
  run("gap table", [] {
    auto r = random_request(5, 400, 400, 0.8);
    r.targets = r.sources;
    auto soe = fgt::fold(fgt::cf_soe(10));
    auto lazy = fgt::plan(r, soe, false);
    auto eager = fgt::plan(r, soe, true);
    CHECK(!lazy.precomputed && eager.precomputed);
    CHECK(eager.gap_exponentials.size() == soe.size() * 399);
    bool bounded = true;
    for (auto g : eager.gap_exponentials) bounded = bounded && std::abs(g) <= 1.0;
    CHECK(bounded);
    CHECK(max_abs_diff(fgt::apply_same(lazy, r.strengths).potentials,
                       fgt::apply_same(eager, r.strengths).potentials) == 0.0);
  });
  run("thread count invariance", [] {
    auto r = random_request(8, 700, 900, 0.25);
    auto p = fgt::plan(r, fgt::fold(fgt::cf_soe(12)), false);
    CHECK(max_abs_diff(fgt::apply_general(p, r.strengths, 1).potentials,
                       fgt::apply_general(p, r.strengths, 4).potentials) == 0.0);
  });
  run("widely separated clusters", [] {
    TransformRequest r{{5e-4, 100.0005}, {0.0, 1e-3, 100.0, 100.001}, {1.0, 2.0, -3.0, 4.0}, 1e-8};
    auto p = fgt::plan(r, fgt::fold(fgt::cf_soe(12)), true);
    auto u = fgt::apply_general(p, r.strengths);
    for (double v : u.potentials) CHECK(std::isfinite(v));
    CHECK(max_abs_diff(u.potentials, fgt::direct(r).potentials) < 1e-8);
  });
  run("mode sums vs quadratic definition", [] {
    auto r = random_request(21, 120, 120, 0.6);
    r.targets = r.sources;
    auto soe = fgt::fold(fgt::cf_soe(8));
    auto p = fgt::plan(r, soe, false);
    auto sums = fgt::detail::mode_sums(p, r.strengths);
    CHECK(sums.hp.size() == soe.size() && sums.hm.size() == soe.size());
    const double rs = 1.0 / std::sqrt(r.delta);
    double bscale = 0;
    for (double b : r.strengths) bscale += std::fabs(b);
    double worst = 0;
    for (std::size_t k = 0; k < soe.size(); ++k)
      for (std::size_t i = 0; i < p.sorted_targets.size(); ++i) {
        std::complex<double> hp{}, hm{};
        for (std::size_t j = 0; j < p.sorted_sources.size(); ++j) {
          const double beta = r.strengths[p.source_perm[j]];
          const double gap = p.sorted_targets[i] - p.sorted_sources[j];
          if (p.sorted_sources[j] <= p.sorted_targets[i])
            hp += beta * std::exp(-p.soe.nodes[k] * gap * rs);
          else
            hm += beta * std::exp(p.soe.nodes[k] * gap * rs);
        }
        worst = std::max(worst, std::abs(sums.hp[k][i] - hp) / bscale);
        worst = std::max(worst, std::abs(sums.hm[k][i] - hm) / bscale);
      }
    CHECK(worst <= 1e-12);
  });
  run("apply-time validation", [] {
    auto p = fgt::plan(golden(), fgt::fold(fgt::cf_soe(8)), false);
    CHECK(throws<std::invalid_argument>([&] { fgt::apply_general(p, {1.0}); }));
    CHECK(throws<std::invalid_argument>([&] { fgt::apply_same(p, kAs); }));
  });
  run("same-point detection needs identical vectors", [] {
    TransformRequest r{{0.1, 0.5, 0.9}, {0.9, 0.1, 0.5}, {1.0, 1.0, 1.0}, 1.0};
    auto soe = fgt::fold(fgt::cf_soe(8));
    auto p = fgt::plan(r, soe, false);
    CHECK(!p.same_points);
    CHECK(max_abs_diff(fgt::apply_general(p, r.strengths).potentials, fgt::direct(r).potentials) <
          fgt::max_error(soe).max_abs_error * 3.0);
  });
  run("stable sort permutation", [] {
    TransformRequest r{{0.5, 0.2, 0.5, 0.2}, {0.4}, {1.0}, 1.0};
    auto p = fgt::plan(r, fgt::fold(fgt::cf_soe(8)), false);
    CHECK(p.target_perm == (std::vector<std::int64_t>{1, 3, 0, 2}));
  });
}

}  // namespace

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
  if (gpu)
    gpu_tests();
  else
    cpu_tests();
  std::printf("%s: %d checks, %d failures\n", gpu ? "gpu" : "cpu", g_checks, g_fail);
  return g_fail;
}
