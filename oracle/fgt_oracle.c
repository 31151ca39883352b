/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle for the SOE fast Gauss transform
 * hot path.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load this library, and only as the checker.  The product path
 * (paper_1909_09825_b200/csrc, libfgt1d_b200.so) never calls it.
 *
 * A plain-C restatement of the reference algorithm, operation for operation,
 * so that (with gcc -O2, no FMA contraction, glibc cexp) it reproduces the
 * reference bit for bit.  Pinned by tests/test_oracle.py against
 *   - the reference's golden potentials (proj/tests/test_transform.cpp:19-26),
 *   - the reference library itself compiled in place (oracle/_ref, bit-exact
 *     comparison on seeded inputs).
 *
 * Reference map (paths under /root/reference/proj):
 *   sort_with_perm        src/transform.cpp:27-39   -> oracle_sort_with_perm
 *   mode_coefs            src/transform.cpp:47-56   -> (done by the caller: s_re, s_im, mw)
 *   decay_factor          src/transform.cpp:60-68   -> decay_factor
 *   permuted_strengths    src/transform.cpp:88-93   -> inside oracle_apply
 *   run_mode_same         src/transform.cpp:97-113  -> run_mode_same
 *   run_mode_general      src/transform.cpp:119-149 -> run_mode_general
 *   apply_common          src/transform.cpp:151-196 -> oracle_apply
 *   direct                src/transform.cpp:255-288 -> oracle_direct
 *   detail::mode_sums     src/transform.cpp:310-350 -> oracle_mode_sums
 *   rng counter_rand      src/rng.cpp:7-22          -> oracle_counter_rand
 */
#include <complex.h>
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cplx;

/* transform.cpp:19 */
#define K_UNDERFLOW_EXPONENT 745.0

/* ---------------------------------------------------------------- rng -- */
/* rng.cpp:7-22 */
static uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
uint64_t oracle_counter_rand(uint64_t seed, uint64_t stream, uint64_t i) {
  return mix64(mix64(seed ^ stream * 0xA24BAED4963EE407ull) + i * 0x9E3779B97F4A7C15ull);
}
double oracle_uniform01(uint64_t seed, uint64_t stream, uint64_t i) {
  return (double)(oracle_counter_rand(seed, stream, i) >> 11) * 0x1.0p-53;
}
void oracle_uniform_points(int64_t n, uint64_t seed, uint64_t stream, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = oracle_uniform01(seed, stream, (uint64_t)i);
}

/* --------------------------------------------------------------- sort -- */
typedef struct {
  double v;
  int64_t i;
} pair_t;

static int pair_less(const void* a, const void* b) {
  const pair_t* p = (const pair_t*)a;
  const pair_t* q = (const pair_t*)b;
  if (p->v < q->v) return -1;
  if (q->v < p->v) return 1;
  return (p->i > q->i) - (p->i < q->i);
}

/* transform.cpp:27-39: std::sort of (value, index) pairs -> ties keep
 * original order; -0.0 and +0.0 compare equal. */
void oracle_sort_with_perm(const double* v, int64_t n, double* sorted, int64_t* perm) {
  pair_t* tmp = (pair_t*)malloc(sizeof(pair_t) * (size_t)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) {
    tmp[i].v = v[i];
    tmp[i].i = i;
  }
  qsort(tmp, (size_t)n, sizeof(pair_t), pair_less);
  for (int64_t i = 0; i < n; ++i) {
    sorted[i] = tmp[i].v;
    perm[i] = tmp[i].i;
  }
  free(tmp);
}

/* ------------------------------------------------------------ kernels -- */
typedef struct {
  double tre, tim;
  cplx mw;
} mode_coef_t;

/* transform.cpp:60-68 */
static inline cplx decay_factor(const mode_coef_t* m, double d) {
  if (d == 0.0) return CMPLX(1.0, 0.0);
  double a = m->tre * d;
  if (a > K_UNDERFLOW_EXPONENT) return CMPLX(0.0, 0.0);
  cplx e = cexp(CMPLX(-a, -m->tim * d));
  double re = creal(e), im = cimag(e);
  double n2 = re * re + im * im; /* std::norm (libstdc++ _Norm_helper) */
  if (n2 > 1.0) {
    double s = sqrt(n2);
    e = CMPLX(re / s, im / s);
  }
  return e;
}

/* Multiplication exactly as std::complex<double> operator* (GCC lowers both
 * to the same __muldc3 semantics; finite operands give (ac-bd, ad+bc)). */
static inline cplx cmul(cplx a, cplx b) { return a * b; }

typedef struct {
  const double* xs; /* sorted targets (M) */
  const double* ys; /* sorted sources (N) */
  const double* bs; /* permuted strengths (N) */
  int64_t M, N;
  const mode_coef_t* mc;
  const cplx* gaps; /* optional precomputed gap table (ne * (M-1)) or NULL */
} problem_t;

static inline cplx gap(const problem_t* p, int k, int64_t i) {
  if (p->gaps) return p->gaps[(int64_t)k * (p->M - 1) + i];
  return decay_factor(&p->mc[k], p->xs[i + 1] - p->xs[i]);
}

/* transform.cpp:97-113 */
static void run_mode_same(const problem_t* p, int k, cplx* buf) {
  const int64_t N = p->N;
  const mode_coef_t* m = &p->mc[k];
  cplx run = 0;
  buf[N - 1] = 0;
  for (int64_t i = N - 1; i >= 1; --i) {
    run = cmul(gap(p, k, i - 1), run + p->bs[i]);
    buf[i - 1] = run;
  }
  run = 0;
  for (int64_t i = 0; i < N; ++i) {
    run = i == 0 ? CMPLX(p->bs[0], 0.0) : p->bs[i] + cmul(gap(p, k, i - 1), run);
    buf[i] = cmul(m->mw, run + buf[i]);
  }
}

/* transform.cpp:119-149 (reference names: N = #targets, M = #sources) */
static void run_mode_general(const problem_t* p, int k, cplx* buf) {
  const double* xs = p->xs;
  const double* ys = p->ys;
  const int64_t NT = p->M, NS = p->N;
  const mode_coef_t* m = &p->mc[k];
  cplx run = 0;
  int64_t j = NS;
  for (int64_t ii = NT; ii-- > 0;) {
    if (ii + 1 < NT) run = cmul(run, gap(p, k, ii));
    while (j > 0 && ys[j - 1] > xs[ii]) {
      run += p->bs[j - 1] * decay_factor(m, ys[j - 1] - xs[ii]);
      --j;
    }
    buf[ii] = run;
  }
  run = 0;
  j = 0;
  for (int64_t i = 0; i < NT; ++i) {
    if (i > 0) run = cmul(run, gap(p, k, i - 1));
    while (j < NS && ys[j] <= xs[i]) {
      if (ys[j] == xs[i])
        run += p->bs[j];
      else
        run += p->bs[j] * decay_factor(m, xs[i] - ys[j]);
      ++j;
    }
    buf[i] = cmul(m->mw, run + buf[i]);
  }
}

typedef struct {
  const problem_t* p;
  int same, k0, stride, ne;
  cplx** bufs;
} worker_t;

static void* worker(void* arg) {
  worker_t* w = (worker_t*)arg;
  for (int k = w->k0; k < w->ne; k += w->stride) {
    if (w->same)
      run_mode_same(w->p, k, w->bufs[k]);
    else
      run_mode_general(w->p, k, w->bufs[k]);
  }
  return NULL;
}

static void fill_modes(mode_coef_t* mc, int ne, double delta, const double* t_re,
                       const double* t_im, const double* mw_re, const double* mw_im) {
  const double isq = 1.0 / sqrt(delta); /* transform.cpp:49 */
  for (int k = 0; k < ne; ++k) {
    mc[k].tre = t_re[k] * isq;
    mc[k].tim = t_im[k] * isq;
    mc[k].mw = CMPLX(mw_re[k], mw_im[k]);
  }
}

/*
 * apply_common (transform.cpp:151-196) on an already-sorted problem.
 *   xs, ys: sorted targets / sources; tperm, sperm: the plan permutations
 *   alpha: strengths in ORIGINAL source order; mw = multiplier * weight.
 *   gaps: NULL (lazy) or the precomputed table from oracle_gap_table.
 *   u_out: potentials in ORIGINAL target order (M entries).
 */
int oracle_apply(const double* xs, const int64_t* tperm, int64_t M, const double* ys,
                 const int64_t* sperm, int64_t N, const double* alpha, double delta,
                 const double* t_re, const double* t_im, const double* mw_re,
                 const double* mw_im, int ne, int same, int num_threads,
                 const double* gaps_interleaved, double* u_out) {
  for (int64_t i = 0; i < M; ++i) u_out[i] = 0.0;
  if (M == 0) return 0;
  mode_coef_t* mc = (mode_coef_t*)malloc(sizeof(mode_coef_t) * (size_t)(ne > 0 ? ne : 1));
  fill_modes(mc, ne, delta, t_re, t_im, mw_re, mw_im);
  double* bs = (double*)malloc(sizeof(double) * (size_t)(N > 0 ? N : 1));
  for (int64_t j = 0; j < N; ++j) bs[j] = alpha[sperm[j]];
  problem_t p = {xs, ys, bs, M, N, mc, (const cplx*)gaps_interleaved};
  cplx* acc = (cplx*)calloc((size_t)M, sizeof(cplx));
  cplx** bufs = (cplx**)malloc(sizeof(cplx*) * (size_t)(ne > 0 ? ne : 1));
  int threads = num_threads < 1 ? 1 : num_threads;
  if (threads > ne) threads = ne > 0 ? ne : 1;
  for (int k = 0; k < ne; ++k) bufs[k] = (cplx*)calloc((size_t)M, sizeof(cplx));
  if (threads <= 1) {
    worker_t w = {&p, same, 0, 1, ne, bufs};
    worker(&w);
  } else {
    pthread_t th[64];
    worker_t ws[64];
    if (threads > 64) threads = 64;
    for (int t = 0; t < threads; ++t) {
      ws[t] = (worker_t){&p, same, t, threads, ne, bufs};
      pthread_create(&th[t], NULL, worker, &ws[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  }
  /* fixed mode order combine (transform.cpp:190-191) */
  for (int k = 0; k < ne; ++k)
    for (int64_t i = 0; i < M; ++i) acc[i] += bufs[k][i];
  /* scatter of the real part (transform.cpp:193-194) */
  for (int64_t i = 0; i < M; ++i) u_out[tperm[i]] = creal(acc[i]);
  for (int k = 0; k < ne; ++k) free(bufs[k]);
  free(bufs);
  free(acc);
  free(bs);
  free(mc);
  return 0;
}

/* precompute_gap_table (transform.cpp:221-237); out: ne*(M-1) complex,
 * interleaved re/im. */
void oracle_gap_table(const double* xs, int64_t M, double delta, const double* t_re,
                      const double* t_im, int ne, double* out) {
  if (M < 2) return;
  mode_coef_t mc[64];
  double z[64] = {0};
  fill_modes(mc, ne, delta, t_re, t_im, z, z);
  cplx* o = (cplx*)out;
  for (int k = 0; k < ne; ++k)
    for (int64_t i = 0; i + 1 < M; ++i)
      o[(int64_t)k * (M - 1) + i] = decay_factor(&mc[k], xs[i + 1] - xs[i]);
}

/* Whole pipeline: plan (sort) + apply, original order in and out. */
int oracle_transform(const double* x, int64_t M, const double* y, int64_t N,
                     const double* alpha, double delta, const double* t_re,
                     const double* t_im, const double* mw_re, const double* mw_im,
                     int ne, int mode, int num_threads, double* u_out) {
  if (!(delta > 0.0) || !isfinite(delta)) return 1;
  for (int64_t i = 0; i < M; ++i)
    if (!isfinite(x[i])) return 1;
  for (int64_t j = 0; j < N; ++j)
    if (!isfinite(y[j])) return 1;
  double* xs = (double*)malloc(sizeof(double) * (size_t)(M > 0 ? M : 1));
  double* ys = (double*)malloc(sizeof(double) * (size_t)(N > 0 ? N : 1));
  int64_t* tp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(M > 0 ? M : 1));
  int64_t* sp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(N > 0 ? N : 1));
  oracle_sort_with_perm(x, M, xs, tp);
  oracle_sort_with_perm(y, N, ys, sp);
  /* transform.cpp:214-216: std::equal on the vectors as given */
  int same_points = (M == N);
  if (same_points)
    for (int64_t i = 0; i < M; ++i)
      if (!(x[i] == y[i])) {
        same_points = 0;
        break;
      }
  int same = mode == 1 || (mode == 2 && same_points);
  int rc = oracle_apply(xs, tp, M, ys, sp, N, alpha, delta, t_re, t_im, mw_re, mw_im,
                        ne, same, num_threads, NULL, u_out);
  free(xs);
  free(ys);
  free(tp);
  free(sp);
  return rc;
}

/* direct (transform.cpp:255-288): long double accumulation. */
int oracle_direct(const double* x, int64_t M, const double* y, int64_t N,
                  const double* alpha, double delta, const int64_t* subset, int64_t nsub,
                  double* out) {
  const long double inv4d = 0.25L / (long double)delta;
  int64_t cnt = nsub > 0 ? nsub : M;
  for (int64_t m = 0; m < cnt; ++m) {
    int64_t idx = nsub > 0 ? subset[m] : m;
    if (idx < 0 || idx >= M) return 2;
    const long double xv = x[idx];
    long double acc = 0.0L;
    for (int64_t j = 0; j < N; ++j) {
      long double d = xv - (long double)y[j];
      long double e = -d * d * inv4d;
      if (e < -11350.0L) continue;
      acc += expl(e) * (long double)alpha[j];
    }
    out[m] = (double)acc;
  }
  return 0;
}

/* detail::mode_sums (transform.cpp:310-350) on sorted inputs; hp/hm are
 * ne*M complex (interleaved), mode-major, sorted-target order. */
int oracle_mode_sums(const double* xs, int64_t M, const double* ys, const int64_t* sperm,
                     int64_t N, const double* alpha, double delta, const double* t_re,
                     const double* t_im, int ne, double* hp_out, double* hm_out) {
  mode_coef_t mc[64];
  double z[64] = {0};
  fill_modes(mc, ne, delta, t_re, t_im, z, z);
  double* bs = (double*)malloc(sizeof(double) * (size_t)(N > 0 ? N : 1));
  for (int64_t j = 0; j < N; ++j) bs[j] = alpha[sperm[j]];
  problem_t p = {xs, ys, bs, M, N, mc, NULL};
  cplx* hp = (cplx*)hp_out;
  cplx* hm = (cplx*)hm_out;
  for (int k = 0; k < ne; ++k) {
    cplx run = 0;
    int64_t j = N;
    for (int64_t ii = M; ii-- > 0;) {
      if (ii + 1 < M) run = cmul(run, gap(&p, k, ii));
      while (j > 0 && ys[j - 1] > xs[ii]) {
        run += bs[j - 1] * decay_factor(&mc[k], ys[j - 1] - xs[ii]);
        --j;
      }
      hm[(int64_t)k * M + ii] = run;
    }
    run = 0;
    j = 0;
    for (int64_t i = 0; i < M; ++i) {
      if (i > 0) run = cmul(run, gap(&p, k, i - 1));
      while (j < N && ys[j] <= xs[i]) {
        run += ys[j] == xs[i] ? CMPLX(bs[j], 0.0) : bs[j] * decay_factor(&mc[k], xs[i] - ys[j]);
        ++j;
      }
      hp[(int64_t)k * M + i] = run;
    }
  }
  free(bs);
  return 0;
}
