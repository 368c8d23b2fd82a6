// TEST INFRASTRUCTURE ONLY — extern "C" shim over the REAL reference.
//
// Compiled by oracle/Makefile directly against the read-only reference
// headers (-I /root/reference/proj/include); output goes to oracle/_ref/
// (git-ignored).  No reference source is copied into this repo.  Used to
// (a) pin the C restatement (oracle/oracle_impl.h) and (b) time the
// reference CPU path (bench.py --impl reference / cpu_baseline).
//
// Each ref_<op>_<s> mirrors oracle/oracle_impl.h's o_<op>_<s> signature and
// maps the reference's exceptions onto dla_status codes.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "dlinalg/adjoints.hpp"
#include "dlinalg/blas.hpp"
#include "dlinalg/cholesky.hpp"
#include "dlinalg/eigen_sym.hpp"
#include "dlinalg/lq.hpp"
#include "dlinalg/matrix.hpp"
#include "dlinalg/models.hpp"
#include "dlinalg/svd.hpp"
#include "dlinalg/tape.hpp"
#include "dlinalg/transforms.hpp"

#include "../include/dla.h"
#include "kalman_oracle.hpp"  // the reference's own dense joint-Gaussian oracle (proj/tests)

using dla::ConstMatrixView;
using dla::index_t;
using dla::MatrixView;

namespace {

template <typename T>
MatrixView<T> mv(T* p, int64_t r, int64_t c) { return MatrixView<T>{p, r, c}; }
template <typename T>
ConstMatrixView<T> cv(const T* p, int64_t r, int64_t c) { return ConstMatrixView<T>(p, r, c); }

template <typename F>
int guarded(F&& f, int64_t* idx) {
  try {
    f();
    return DLA_OK;
  } catch (const dla::NotPositiveDefiniteError& e) {
    if (idx) *idx = e.step;
    return DLA_ERR_NOT_SPD;
  } catch (const dla::SingularError& e) {
    if (idx) *idx = e.index;
    return DLA_ERR_SINGULAR;
  } catch (const dla::ConvergenceError& e) {
    if (idx) *idx = e.iterations;
    return DLA_ERR_CONVERGENCE;
  } catch (const dla::ShapeError& e) {
    const std::string w = e.what();
    return w.find("not symmetric") != std::string::npos ? DLA_ERR_ASYMMETRIC : DLA_ERR_SHAPE;
  } catch (const dla::Error& e) {
    const std::string w = e.what();
    return w.find("alias") != std::string::npos ? DLA_ERR_ALIAS : DLA_ERR_INVALID;
  }
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

#define REF_OPS(T, S)                                                                           \
  int ref_gemm_##S(int64_t m, int64_t n, int64_t k, T* c, const T* a, const T* b, int ta,       \
                   int tb, T alpha, int acc) {                                                  \
    return guarded([&] {                                                                        \
      dla::detail::gemm_accum<T>(mv(c, m, n), cv(a, ta ? k : m, ta ? m : k),                    \
                                 cv(b, tb ? n : k, tb ? k : n), ta, tb, alpha, acc);            \
    }, nullptr);                                                                                \
  }                                                                                             \
  int ref_syrk_##S(int64_t n, int64_t k, T* b, const T* a, int ta, T alpha) {                   \
    return guarded([&] {                                                                        \
      dla::syrk_into<T>(mv(b, n, n), cv(a, ta ? k : n, ta ? n : k), ta, alpha);                 \
    }, nullptr);                                                                                \
  }                                                                                             \
  int ref_trmm_##S(int64_t m, int64_t n, const T* t, T* x, int r, int tr, int lo, T alpha) {    \
    const int64_t mt = r ? n : m;                                                               \
    return guarded([&] { dla::trmm_inplace<T>(cv(t, mt, mt), mv(x, m, n), r, tr, lo, alpha); }, \
                   nullptr);                                                                    \
  }                                                                                             \
  int ref_trsm_##S(int64_t m, int64_t n, const T* t, T* x, int r, int tr, int lo, T alpha,      \
                   int64_t* idx) {                                                              \
    const int64_t mt = r ? n : m;                                                               \
    return guarded([&] { dla::trsm_inplace<T>(cv(t, mt, mt), mv(x, m, n), r, tr, lo, alpha); }, \
                   idx);                                                                        \
  }                                                                                             \
  int ref_potrf_##S(int64_t n, T* a, int lower, int64_t* idx) {                                 \
    return guarded([&] { dla::potrf_inplace<T>(mv(a, n, n), lower); }, idx);                    \
  }                                                                                             \
  int ref_potri_##S(int64_t n, T* a, int lower, int64_t* idx) {                                 \
    return guarded([&] { dla::potri_inplace<T>(mv(a, n, n), lower); }, idx);                    \
  }                                                                                             \
  int ref_gelqf_##S(int64_t m, int64_t n, T* q, T* l, int64_t* idx) {                           \
    return guarded([&] { dla::gelqf_inplace<T>(mv(q, m, n), mv(l, m, m)); }, idx);              \
  }                                                                                             \
  int ref_syevd_##S(int64_t n, T* u, T* lambda, int64_t* idx) {                                 \
    return guarded([&] { dla::syevd_inplace<T>(mv(u, n, n), lambda); }, idx);                   \
  }                                                                                             \
  int ref_gemm2_bwd_##S(int64_t m, int64_t n, int64_t k, T* abar, T* bbar, const T* cbar,       \
                        const T* a, const T* b, int ta, int tb, T alpha) {                      \
    return guarded([&] {                                                                        \
      dla::gemm2_backward_into<T>(mv(abar, ta ? k : m, ta ? m : k),                             \
                                  mv(bbar, tb ? n : k, tb ? k : n), cv(cbar, m, n),             \
                                  cv(a, ta ? k : m, ta ? m : k), cv(b, tb ? n : k, tb ? k : n), \
                                  ta, tb, alpha);                                               \
    }, nullptr);                                                                                \
  }                                                                                             \
  int ref_syrk_bwd_##S(int64_t n, int64_t k, T* abar, const T* bbar, const T* a, int ta,        \
                       T alpha) {                                                               \
    return guarded([&] {                                                                        \
      dla::syrk_backward_into<T>(mv(abar, ta ? k : n, ta ? n : k), cv(bbar, n, n),              \
                                 cv(a, ta ? k : n, ta ? n : k), ta, alpha);                     \
    }, nullptr);                                                                                \
  }                                                                                             \
  int ref_trmm_bwd_##S(int64_t m, int64_t n, T* abar, T* tbar, const T* bbar, const T* t,       \
                       const T* a, int r, int tr, int lo, T alpha) {                            \
    const int64_t mt = r ? n : m;                                                               \
    return guarded([&] {                                                                        \
      dla::trmm_backward_into<T>(mv(abar, m, n), mv(tbar, mt, mt), cv(bbar, m, n),              \
                                 cv(t, mt, mt), cv(a, m, n), r, tr, lo, alpha);                 \
    }, nullptr);                                                                                \
  }                                                                                             \
  int ref_trsm_bwd_##S(int64_t m, int64_t n, T* abar, T* tbar, const T* bbar, const T* t,       \
                       const T* b, int r, int tr, int lo, T alpha, int64_t* idx) {              \
    const int64_t mt = r ? n : m;                                                               \
    return guarded([&] {                                                                        \
      dla::trsm_backward_into<T>(mv(abar, m, n), mv(tbar, mt, mt), cv(bbar, m, n),              \
                                 cv(t, mt, mt), cv(b, m, n), r, tr, lo, alpha);                 \
    }, idx);                                                                                    \
  }                                                                                             \
  int ref_potrf_bwd_##S(int64_t n, T* abar, const T* lbar, const T* l, int lower) {             \
    return guarded([&] {                                                                        \
      dla::potrf_backward_into<T>(mv(abar, n, n), cv(lbar, n, n), cv(l, n, n), lower);          \
    }, nullptr);                                                                                \
  }                                                                                             \
  int ref_potri_bwd_##S(int64_t n, T* lbar, const T* bbar, const T* l, const T* b, int lower) { \
    return guarded([&] {                                                                        \
      dla::potri_backward_into<T>(mv(lbar, n, n), cv(bbar, n, n), cv(l, n, n), cv(b, n, n),     \
                                  lower);                                                       \
    }, nullptr);                                                                                \
  }                                                                                             \
  int ref_gelqf_bwd_##S(int64_t m, int64_t n, T* abar, const T* qbar, const T* lbar,            \
                        const T* q, const T* l) {                                               \
    return guarded([&] {                                                                        \
      dla::gelqf_backward_into<T>(mv(abar, m, n), cv(qbar, m, n), cv(lbar, m, m), cv(q, m, n),  \
                                  cv(l, m, m));                                                 \
    }, nullptr);                                                                                \
  }                                                                                             \
  int ref_gesvd_##S(int64_t m, int64_t n, T* v, T* u, T* lambda, int64_t* idx) {               \
    return guarded([&] { dla::gesvd_inplace<T>(mv(v, m, n), mv(u, m, m), lambda); }, idx);      \
  }                                                                                             \
  int ref_gesvd_bwd_##S(int64_t m, int64_t n, T* abar, const T* ubar, const T* lambdabar,       \
                        const T* vbar, const T* u, const T* lambda, const T* v, T eps_gap,      \
                        int64_t* idx) {                                                         \
    auto cfg = dla::ToleranceConfig<T>::defaults();                                             \
    cfg.eps_gap = eps_gap;                                                                      \
    return guarded([&] {                                                                        \
      dla::gesvd_backward_into<T>(mv(abar, m, n), cv(ubar, m, m), lambdabar, cv(vbar, m, n),    \
                                  cv(u, m, m), lambda, cv(v, m, n), cfg);                       \
    }, idx);                                                                                    \
  }                                                                                             \
  int ref_syevd_bwd_##S(int64_t n, T* abar, const T* ubar, const T* lambdabar, const T* u,      \
                        const T* lambda, T eps_gap) {                                           \
    auto cfg = dla::ToleranceConfig<T>::defaults();                                             \
    cfg.eps_gap = eps_gap;                                                                      \
    return guarded([&] {                                                                        \
      dla::syevd_backward_into<T>(mv(abar, n, n), cv(ubar, n, n), lambdabar, cv(u, n, n),       \
                                  lambda, cfg);                                                 \
    }, nullptr);                                                                                \
  }

extern "C" {

REF_OPS(double, f64)
REF_OPS(float, f32)

// sumlogdiag through the reference tape chain ExtractDiag -> Log -> Sum
// (dl/tape.hpp:389-393, :342, :371) and its pullback via Graph::backward.
int ref_sumlogdiag_f64(int64_t n, const double* a, double* out, double* abar) {
  return guarded([&] {
    dla::Graph<double> g;
    dla::Matrix<double> m(n, n);
    std::memcpy(m.data(), a, sizeof(double) * n * n);
    dla::NodeId x = g.leaf(m, "a");
    dla::NodeId s = g.sum(g.log(g.extract_diag(x)));
    *out = g.value(s)(0, 0);
    if (abar) {
      auto gs = g.backward(s);
      std::memcpy(abar, gs.at(x).data(), sizeof(double) * n * n);
    }
  }, nullptr);
}

// GP NLL + gradient w.r.t. (log sigma2, log ell2, log lam) through the
// reference's make_gp + Graph::backward (dl/models.hpp:115-135,
// dl/tape.hpp:461-484).  out = {nll, d/dlog_sigma2, d/dlog_ell2, d/dlog_lam}.
// Single-threaded by construction (the tape never fans out).
int ref_gp_nll_grad_f64(int64_t n, int64_t d, const double* x, const double* y, double sigma2,
                        double ell2, double lam, double* out, double* xbar, double* ybar) {
  return guarded([&] {
    dla::Matrix<double> xm(n, d), ym(n, 1);
    std::memcpy(xm.data(), x, sizeof(double) * n * d);
    std::memcpy(ym.data(), y, sizeof(double) * n);
    dla::Graph<double> g;
    auto m = dla::make_gp(g, xm, ym, sigma2, ell2, lam);
    out[0] = g.value(m.loss)(0, 0);
    auto gs = g.backward(m.loss);
    out[1] = gs.at(m.log_sigma2)(0, 0);
    out[2] = gs.at(m.log_ell2)(0, 0);
    out[3] = gs.at(m.log_lam)(0, 0);
    if (xbar) std::memcpy(xbar, gs.at(m.x).data(), sizeof(double) * n * d);
    if (ybar) std::memcpy(ybar, gs.at(m.y).data(), sizeof(double) * n);
  }, nullptr);
}

// C1 chain over a batch with the reference's own batch loop (for_each_slice,
// dl/matrix.hpp:217-240): L = potrf(A); z = trsm(L, y); phi = 1/2|z|^2 +
// sumlogdiag(L); backward with phibar = 1: zbar = z; (ybar, Lbar) =
// trsm_backward; Lbar(i,i) += 1/L(i,i); Abar = potrf_backward(Lbar).
// a: [batch,n,n] (overwritten by L), y: [batch,n] (overwritten by ybar),
// abar: [batch,n,n], phi: [batch].  Returns seconds of wall time.
double ref_c1_chain_f64(int64_t batch, int64_t n, double* a, double* y, double* abar,
                        double* phi, int threads) {
  const double t0 = now_s();
  dla::for_each_slice(batch, threads, [&](index_t b) {
    double* ab = a + b * n * n;
    double* yb = y + b * n;
    double* gb = abar + b * n * n;
    dla::potrf_inplace<double>(mv(ab, n, n), true);
    std::vector<double> z(yb, yb + n), zbar(n), ybar(n);
    dla::trsm_inplace<double>(cv<double>(ab, n, n), mv(z.data(), n, 1), false, false, true, 1.0);
    double quad = 0.0, logdet = 0.0;
    for (int64_t i = 0; i < n; ++i) quad += z[i] * z[i];
    for (int64_t i = 0; i < n; ++i) logdet += std::log(ab[i * n + i]);
    phi[b] = 0.5 * quad + logdet;
    for (int64_t i = 0; i < n; ++i) zbar[i] = z[i];
    dla::trsm_backward_into<double>(mv(ybar.data(), n, 1), mv(gb, n, n),
                                    cv<double>(zbar.data(), n, 1), cv<double>(ab, n, n),
                                    cv<double>(z.data(), n, 1), false, false, true, 1.0);
    for (int64_t i = 0; i < n; ++i) gb[i * n + i] += 1.0 / ab[i * n + i];
    dla::potrf_backward_into<double>(mv(gb, n, n), cv<double>(gb, n, n), cv<double>(ab, n, n),
                                     true);
    std::memcpy(yb, ybar.data(), sizeof(double) * n);
  });
  return now_s() - t0;
}

// potrf fwd+bwd over a batch (north-star / C5-shaped op timing):
// a -> L in place; abar <- potrf_backward(lbar, L) (lbar may alias abar).
double ref_potrf_fwdbwd_batch_f64(int64_t batch, int64_t n, double* a, double* abar,
                                  const double* lbar, int threads) {
  const double t0 = now_s();
  dla::for_each_slice(batch, threads, [&](index_t b) {
    double* ab = a + b * n * n;
    dla::potrf_inplace<double>(mv(ab, n, n), true);
    dla::potrf_backward_into<double>(mv(abar + b * n * n, n, n),
                                     cv<double>(lbar + b * n * n, n, n), cv<double>(ab, n, n),
                                     true);
  });
  return now_s() - t0;
}

#define REF_BATCH_LQ_EIG(T, S)                                                                  \
  double ref_gelqf_fwdbwd_batch_##S(int64_t batch, int64_t m, int64_t n, T* q, T* l, T* abar,   \
                                    const T* qbar, const T* lbar, int threads) {                \
    const double t0 = now_s();                                                                  \
    dla::for_each_slice(batch, threads, [&](index_t b) {                                        \
      dla::gelqf_inplace<T>(mv(q + b * m * n, m, n), mv(l + b * m * m, m, m));                  \
      dla::gelqf_backward_into<T>(mv(abar + b * m * n, m, n), cv(qbar + b * m * n, m, n),       \
                                  cv(lbar + b * m * m, m, m), cv<T>(q + b * m * n, m, n),       \
                                  cv<T>(l + b * m * m, m, m));                                  \
    });                                                                                         \
    return now_s() - t0;                                                                        \
  }                                                                                             \
  double ref_syevd_fwdbwd_batch_##S(int64_t batch, int64_t n, T* u, T* lambda, T* abar,         \
                                    const T* ubar, const T* lambdabar, int threads) {           \
    const double t0 = now_s();                                                                  \
    auto cfg = dla::ToleranceConfig<T>::defaults();                                             \
    dla::for_each_slice(batch, threads, [&](index_t b) {                                        \
      dla::syevd_inplace<T>(mv(u + b * n * n, n, n), lambda + b * n);                           \
      dla::syevd_backward_into<T>(mv(abar + b * n * n, n, n), cv(ubar + b * n * n, n, n),       \
                                  lambdabar + b * n, cv<T>(u + b * n * n, n, n),                \
                                  lambda + b * n, cfg);                                         \
    });                                                                                         \
    return now_s() - t0;                                                                        \
  }

REF_BATCH_LQ_EIG(double, f64)
REF_BATCH_LQ_EIG(float, f32)


// Kalman filter NLL + gradient of every leaf through the reference's
// make_kalman + Graph::backward (dl/models.hpp:285-369, dl/tape.hpp).
// obs: T x d (row t = observation t); gradients in the input shapes; the
// observation gradients land in obsbar.  joint (nullable): the reference
// test oracle's dense joint-Gaussian NLL (proj/tests/kalman_oracle.hpp:16-79).
int ref_kalman_f64(int64_t h, int64_t d, int64_t T, const double* a, const double* b, const double* sh,
                   const double* sv, const double* mu0, const double* s0, const double* obs, double* nll,
                   double* abar, double* bbar, double* shbar, double* svbar, double* mu0bar, double* s0bar,
                   double* obsbar, double* joint) {
  return guarded([&] {
    auto mat = [](const double* p, int64_t r, int64_t c) {
      dla::Matrix<double> m(r, c);
      std::memcpy(m.data(), p, sizeof(double) * r * c);
      return m;
    };
    dla::Matrix<double> am = mat(a, h, h), bm = mat(b, d, h), shm = mat(sh, h, h), svm = mat(sv, d, d),
                        m0 = mat(mu0, h, 1), s0m = mat(s0, h, h);
    std::vector<dla::Matrix<double>> ob;
    for (int64_t t = 0; t < T; ++t) ob.push_back(mat(obs + t * d, d, 1));
    dla::Graph<double> g;
    auto m = dla::make_kalman(g, am, bm, shm, svm, m0, s0m, ob);
    *nll = g.value(m.loss)(0, 0);
    auto gs = g.backward(m.loss);
    std::memcpy(abar, gs.at(m.a).data(), sizeof(double) * h * h);
    std::memcpy(bbar, gs.at(m.b).data(), sizeof(double) * d * h);
    std::memcpy(shbar, gs.at(m.sh).data(), sizeof(double) * h * h);
    std::memcpy(svbar, gs.at(m.sv).data(), sizeof(double) * d * d);
    std::memcpy(mu0bar, gs.at(m.mu0).data(), sizeof(double) * h);
    std::memcpy(s0bar, gs.at(m.s0).data(), sizeof(double) * h * h);
    for (int64_t t = 0; t < T; ++t) std::memcpy(obsbar + t * d, gs.at(m.obs[t]).data(), sizeof(double) * d);
    if (joint) *joint = oracle::lgssm_joint_nll(am, bm, shm, svm, m0, s0m, ob);
  }, nullptr);
}

// Batched Kalman NLL + gradients with the reference's own batch loop
// (timing leg of bench.py): sequence s uses parameters + s * (its size).
double ref_kalman_batch_f64(int64_t batch, int64_t h, int64_t d, int64_t T, const double* a, const double* b,
                            const double* sh, const double* sv, const double* mu0, const double* s0,
                            const double* obs, double* nll, int threads) {
  const double t0 = now_s();
  dla::for_each_slice(batch, threads, [&](index_t s) {
    std::vector<double> ga(h * h), gb(d * h), gsh(h * h), gsv(d * d), gm(h), gs0(h * h), go(T * d);
    ref_kalman_f64(h, d, T, a + s * h * h, b + s * d * h, sh + s * h * h, sv + s * d * d, mu0 + s * h,
                   s0 + s * h * h, obs + s * T * d, nll + s, ga.data(), gb.data(), gsh.data(), gsv.data(),
                   gm.data(), gs0.data(), go.data(), nullptr);
  });
  return now_s() - t0;
}


// Memory-plan hand-off counts of the reference tape (Graph::planned_reuse_count,
// dl/tape.hpp:486-491) for make_gp and make_kalman graphs: the device tape's
// restated build_plan must make the same hand-offs.
int64_t ref_gp_plan_count(int64_t n, int64_t d, const double* x, const double* y) {
  int64_t c = -1;
  guarded([&] {
    dla::Matrix<double> xm(n, d), ym(n, 1);
    std::memcpy(xm.data(), x, sizeof(double) * n * d);
    std::memcpy(ym.data(), y, sizeof(double) * n);
    dla::Graph<double> g;
    dla::make_gp(g, xm, ym, 1.0, 1.0, 0.1);
    c = g.planned_reuse_count();
  }, nullptr);
  return c;
}
int64_t ref_kalman_plan_count(int64_t h, int64_t d, int64_t T, const double* a, const double* b, const double* sh,
                              const double* sv, const double* mu0, const double* s0, const double* obs) {
  int64_t c = -1;
  guarded([&] {
    auto mat = [](const double* p, int64_t r, int64_t cc) {
      dla::Matrix<double> m(r, cc);
      std::memcpy(m.data(), p, sizeof(double) * r * cc);
      return m;
    };
    std::vector<dla::Matrix<double>> ob;
    for (int64_t t = 0; t < T; ++t) ob.push_back(mat(obs + t * d, d, 1));
    dla::Graph<double> g;
    dla::make_kalman(g, mat(a, h, h), mat(b, d, h), mat(sh, h, h), mat(sv, d, d), mat(mu0, h, 1), mat(s0, h, h), ob);
    c = g.planned_reuse_count();
  }, nullptr);
  return c;
}

}  // extern "C"
