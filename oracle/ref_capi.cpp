// TEST INFRASTRUCTURE ONLY (oracle).  Never linked into the product.
//
// A thin extern "C" shim over the UNMODIFIED reference fgt1d library
// (/root/reference/proj/src/{transform,soe,rng}.cpp, compiled in place by
// oracle/build_ref.sh into oracle/_ref/libfgt1d_ref.so).  It lets the Python
// tests and bench.py's reference arm call the reference's own public API:
//
//   plan()              proj/src/transform.cpp:200-219 (here :306-325 numbering of the file)
//   precompute_gap_table proj/src/transform.cpp:221-237
//   apply_same/general  proj/src/transform.cpp:239-253
//   direct              proj/src/transform.cpp:255-288
//   detail::mode_sums   proj/src/transform.cpp:310-350
//
// The reference's cf_soe() (proj/src/cf.cpp:194) needs Eigen, which this
// image lacks; it is supplied here by loading the regenerated table
// cf_n<n>.soe (tools/gen_soe_tables.py) through the reference's own
// load_coefficient_table (proj/src/soe.cpp:333-337).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "fgt1d/cf.hpp"
#include "fgt1d/errors.hpp"
#include "fgt1d/soe.hpp"
#include "fgt1d/rng.hpp"
#include "fgt1d/transform.hpp"

namespace {
std::string g_table_dir = ".";
thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

#define FGT_REF_TRY(body)                                   \
  try {                                                     \
    body;                                                   \
    return 0;                                               \
  } catch (const fgt::numerical_error& e) {                 \
    return fail(e, 3);                                      \
  } catch (const std::domain_error& e) {                    \
    return fail(e, 1);                                      \
  } catch (const std::invalid_argument& e) {                \
    return fail(e, 2);                                      \
  } catch (const std::exception& e) {                       \
    return fail(e, 4);                                      \
  }

fgt::SoeApprox make_soe(int ne, const double* t_re, const double* t_im,
                        const double* w_re, const double* w_im, int nsoe,
                        int folded) {
  if (nsoe <= 0) return fgt::fold(fgt::cf_soe(2 * ne));
  fgt::SoeApprox s;
  s.form = folded ? fgt::SoeForm::Folded : fgt::SoeForm::Full;
  for (int k = 0; k < nsoe; ++k) {
    s.nodes.emplace_back(t_re[k], t_im[k]);
    s.weights.emplace_back(w_re[k], w_im[k]);
    if (folded) s.self_conjugate.push_back(t_im[k] == 0.0 ? 1 : 0);
  }
  return s;
}

fgt::TransformRequest make_req(const double* x, int64_t M, const double* y,
                               int64_t N, const double* a, double delta) {
  fgt::TransformRequest req;
  req.targets.assign(x, x + M);
  req.sources.assign(y, y + N);
  req.strengths.assign(a, a + N);
  req.delta = delta;
  return req;
}
}  // namespace

namespace fgt {
SoeApprox cf_soe(int n) {
  if (n < 2 || n > 14)
    throw std::domain_error("rational construction supports orders 2..14");
  return load_coefficient_table(g_table_dir + "/cf_n" + std::to_string(n) +
                                ".soe");
}
}  // namespace fgt

extern "C" {

const char* fgt_ref_last_error(void) { return g_err.c_str(); }

void fgt_ref_set_table_dir(const char* dir) { g_table_dir = dir; }

// One reference transform, timed per phase exactly like run_bench_once
// (proj/tools/fgt1d_cli.cpp:240-251).  mode: 0 general, 1 same, 2 auto
// (same if plan.same_points, like pymodule.cpp:56-58).  precompute != 0
// runs precompute_gap_table between plan and apply.
int fgt_ref_transform(const double* x, int64_t M, const double* y, int64_t N,
                      const double* a, double delta, int ne,
                      const double* t_re, const double* t_im,
                      const double* w_re, const double* w_im, int nsoe,
                      int folded, int mode, int threads, int precompute,
                      double* u_out, double* times3) {
  FGT_REF_TRY({
    auto req = make_req(x, M, y, N, a, delta);
    auto soe = make_soe(ne, t_re, t_im, w_re, w_im, nsoe, folded);
    using Clock = std::chrono::steady_clock;
    auto t0 = Clock::now();
    fgt::TransformPlan plan = fgt::plan(req, soe, false);
    auto t1 = Clock::now();
    if (precompute) fgt::precompute_gap_table(plan);
    auto t2 = Clock::now();
    bool same = mode == 1 || (mode == 2 && plan.same_points);
    fgt::TransformResult res =
        same ? fgt::apply_same(plan, req.strengths, threads)
             : fgt::apply_general(plan, req.strengths, threads);
    auto t3 = Clock::now();
    std::memcpy(u_out, res.potentials.data(), sizeof(double) * res.potentials.size());
    if (times3) {
      times3[0] = std::chrono::duration<double>(t1 - t0).count();
      times3[1] = std::chrono::duration<double>(t2 - t1).count();
      times3[2] = std::chrono::duration<double>(t3 - t2).count();
    }
  })
}

// plan() only: sorted copies, permutations and same_points flag.
int fgt_ref_plan(const double* x, int64_t M, const double* y, int64_t N,
                 const double* a, double delta, int ne, double* sorted_x,
                 int64_t* tperm, double* sorted_y, int64_t* sperm,
                 int* same_points) {
  FGT_REF_TRY({
    auto req = make_req(x, M, y, N, a, delta);
    auto plan = fgt::plan(req, fgt::fold(fgt::cf_soe(2 * ne)), false);
    std::memcpy(sorted_x, plan.sorted_targets.data(), sizeof(double) * M);
    std::memcpy(sorted_y, plan.sorted_sources.data(), sizeof(double) * N);
    std::memcpy(tperm, plan.target_perm.data(), sizeof(int64_t) * M);
    std::memcpy(sperm, plan.source_perm.data(), sizeof(int64_t) * N);
    *same_points = plan.same_points ? 1 : 0;
  })
}

int fgt_ref_direct(const double* x, int64_t M, const double* y, int64_t N,
                   const double* a, double delta, const int64_t* subset,
                   int64_t nsub, double* out) {
  FGT_REF_TRY({
    auto req = make_req(x, M, y, N, a, delta);
    std::vector<int64_t> idx;
    if (nsub > 0) idx.assign(subset, subset + nsub);
    auto res = fgt::direct(req, idx);
    std::memcpy(out, res.potentials.data(), sizeof(double) * res.potentials.size());
  })
}

// Per-mode h+ / h- (sorted-target order), interleaved re/im:
// hp[(k*M + i)*2 + {0,1}].
int fgt_ref_mode_sums(const double* x, int64_t M, const double* y, int64_t N,
                      const double* a, double delta, int ne, double* hp,
                      double* hm) {
  FGT_REF_TRY({
    auto req = make_req(x, M, y, N, a, delta);
    auto plan = fgt::plan(req, fgt::fold(fgt::cf_soe(2 * ne)), false);
    auto ms = fgt::detail::mode_sums(plan, req.strengths);
    for (std::size_t k = 0; k < ms.hp.size(); ++k)
      for (int64_t i = 0; i < M; ++i) {
        hp[(k * M + i) * 2 + 0] = ms.hp[k][i].real();
        hp[(k * M + i) * 2 + 1] = ms.hp[k][i].imag();
        hm[(k * M + i) * 2 + 0] = ms.hm[k][i].real();
        hm[(k * M + i) * 2 + 1] = ms.hm[k][i].imag();
      }
  })
}

// Grid error of a full or folded SOE (proj/src/soe.cpp:242-248).
int fgt_ref_max_error(int n, int fold_it, double* err, double* argmax) {
  FGT_REF_TRY({
    auto s = fgt::cf_soe(n);
    if (fold_it) s = fgt::fold(s);
    auto rep = fgt::max_error(s);
    *err = rep.max_abs_error;
    *argmax = rep.argmax_x;
  })
}

// precompute_gap_table (transform.cpp:221-237) of the plan of sorted or
// unsorted targets x (sources = x): mode-major, interleaved re/im,
// out[(k*(M-1) + i)*2 + {0,1}].
int fgt_ref_gap_table(const double* x, int64_t M, double delta, int ne, double* out) {
  FGT_REF_TRY({
    std::vector<double> a(M, 1.0);
    auto req = make_req(x, M, x, M, a.data(), delta);
    auto plan = fgt::plan(req, fgt::fold(fgt::cf_soe(2 * ne)), true);
    for (std::size_t i = 0; i < plan.gap_exponentials.size(); ++i) {
      out[2 * i] = plan.gap_exponentials[i].real();
      out[2 * i + 1] = plan.gap_exponentials[i].imag();
    }
  })
}

// rng::uniform_points (rng.cpp:24-29) and rng::counter_rand (rng.cpp:7-17).
int fgt_ref_uniform_points(int64_t count, uint64_t seed, uint64_t stream, double* out) {
  FGT_REF_TRY({
    auto v = fgt::rng::uniform_points((std::size_t)count, seed, stream);
    std::memcpy(out, v.data(), sizeof(double) * v.size());
  })
}

uint64_t fgt_ref_counter_rand(uint64_t seed, uint64_t stream, uint64_t i) {
  return fgt::rng::counter_rand(seed, stream, i);
}

}  // extern "C"
