// C++ host caller of libdla_b200's C-ABI, from the REFERENCE's side of the
// boundary.  Compiled by __graft_entry__.build() (where
// /root/reference exists) against the reference's own headers
// (-I /root/reference/proj/include) into tests/cpp/_bin/backend_hook, which
// travels to the GPU box; tests/test_gpu_cpp_backend.py runs it there.
//
//  1. replays the reference's hook test (proj/tests/test_blas_kernels.cpp:
//     98-129): a declining hook falls through to the reference loops
//     bit-for-bit, a claiming hook's sentinel shows up, clearing restores;
//  2. installs the B200 backend -- kernel_backend<T>().gemm over
//     dla_gemm_fwd_{f32,f64} (dl/blas.hpp:17-29, consulted by gemm_accum
//     :61-63) -- and runs the reference's own gemm2 and pullbacks
//     (gemm2/potri/gelqf/syevd backward: their products go to the device)
//     against the same calls with the hook cleared;
//  3. calls the operator entry points directly from C++ (potrf, potrf
//     pullback, trsm, syevd) on device buffers and checks them against the
//     reference's potrf_inplace / potrf_backward_into / trsm_inplace /
//     syevd_inplace on the same inputs.
// Prints one line per check and "ALL OK" at the end; exit code 0 = pass.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "dla.h"
#include "dlinalg/adjoints.hpp"
#include "dlinalg/blas.hpp"
#include "dlinalg/cholesky.hpp"
#include "dlinalg/eigen_sym.hpp"
#include "dlinalg/lq.hpp"
#include "dlinalg/matrix.hpp"

using namespace dla;

static int g_fail = 0;

static void check(bool ok, const char* what, double v = 0.0) {
  std::printf("%-60s %s (%.3g)\n", what, ok ? "ok" : "FAIL", v);
  if (!ok) ++g_fail;
}

template <typename T>
static Matrix<T> rnd(index_t r, index_t c, std::mt19937_64& g) {
  std::normal_distribution<double> nd(0.0, 1.0);  // inputs only; both sides see the same values
  Matrix<T> m(r, c);
  for (index_t i = 0; i < r * c; ++i) m.data()[i] = T(nd(g));
  return m;
}

template <typename T>
static Matrix<T> spd(index_t n, std::mt19937_64& g) {
  Matrix<T> x = rnd<T>(n, n, g), a(n, n);
  for (index_t i = 0; i < n; ++i)
    for (index_t j = 0; j < n; ++j) {
      double s = 0;
      for (index_t k = 0; k < n; ++k) s += double(x(i, k)) * double(x(j, k));
      a(i, j) = T(s + (i == j ? n : 0));
    }
  return a;
}

template <typename T>
static double rel(ConstMatrixView<T> a, ConstMatrixView<T> b) {
  double d = 0, m = 1e-300;
  for (index_t i = 0; i < a.size(); ++i) {
    d = std::fmax(d, std::fabs(double(a.data[i]) - double(b.data[i])));
    m = std::fmax(m, std::fabs(double(b.data[i])));
  }
  return d / m;
}

// ---------------------------------------------------------------- device
struct Dev {
  void* p = nullptr;
  explicit Dev(size_t bytes) {
    if (bytes && cudaMalloc(&p, bytes) != cudaSuccess) {
      std::fprintf(stderr, "cudaMalloc failed\n");
      std::exit(2);
    }
  }
  ~Dev() {
    if (p) cudaFree(p);
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

template <typename T>
dla_status gemm_fwd(int64_t m, int64_t n, int64_t k, T* c, const T* a, const T* b, int ta, int tb, T alpha,
                    T beta, void* ws, size_t wsb);
template <>
dla_status gemm_fwd<double>(int64_t m, int64_t n, int64_t k, double* c, const double* a, const double* b, int ta,
                            int tb, double alpha, double beta, void* ws, size_t wsb) {
  return dla_gemm_fwd_f64(1, m, n, k, c, a, b, ta, tb, alpha, beta, ws, wsb, nullptr);
}
template <>
dla_status gemm_fwd<float>(int64_t m, int64_t n, int64_t k, float* c, const float* a, const float* b, int ta, int tb,
                           float alpha, float beta, void* ws, size_t wsb) {
  return dla_gemm_fwd_f32(1, m, n, k, c, a, b, ta, tb, alpha, beta, ws, wsb, nullptr);
}

static long g_device_gemms = 0;

// The backend a maintainer installs: gemm_accum's product on the B200
// (host views in, host view out; accumulate = beta 1).
template <typename T>
static void install_device_backend() {
  kernel_backend<T>().gemm = [](MatrixView<T> c, ConstMatrixView<T> a, ConstMatrixView<T> b, bool ta, bool tb,
                                T alpha, bool accumulate) -> bool {
    const int64_t m = c.rows, n = c.cols, k = ta ? a.rows : a.cols;
    if (m == 0 || n == 0) return false;
    const size_t sa = sizeof(T) * a.size(), sb = sizeof(T) * b.size(), sc = sizeof(T) * c.size();
    Dev da(sa), db(sb), dc(sc);
    const size_t wsb =
        dla_workspace_bytes(DLA_OP_GEMM, sizeof(T) == 8 ? DLA_F64 : DLA_F32, 1, m, n, k, 0);
    Dev ws(wsb);
    cudaMemcpy(da.p, a.data, sa, cudaMemcpyHostToDevice);
    cudaMemcpy(db.p, b.data, sb, cudaMemcpyHostToDevice);
    if (accumulate) cudaMemcpy(dc.p, c.data, sc, cudaMemcpyHostToDevice);
    const dla_status st = gemm_fwd<T>(m, n, k, dc.as<T>(), da.as<T>(), db.as<T>(), ta, tb, alpha,
                                      accumulate ? T(1) : T(0), ws.p, wsb);
    if (st != DLA_OK) return false;  // decline: the reference loops take over
    cudaMemcpy(c.data, dc.p, sc, cudaMemcpyDeviceToHost);
    ++g_device_gemms;
    return true;
  };
}

// ------------------------------------------------------------------ tests
static void replay_reference_hook_test() {
  // proj/tests/test_blas_kernels.cpp:98-129
  std::mt19937_64 rng(19);
  Matrix<double> a = rnd<double>(3, 3, rng), b = rnd<double>(3, 3, rng);
  Matrix<double> base = gemm2(a, b);
  int calls = 0;
  kernel_backend<double>().gemm = [&](MatrixView<double>, ConstMatrixView<double>, ConstMatrixView<double>, bool,
                                      bool, double, bool) {
    ++calls;
    return false;
  };
  Matrix<double> declined = gemm2(a, b);
  check(calls > 0 && rel<double>(declined.view(), base.view()) == 0, "hook: decline falls through bitwise");
  kernel_backend<double>().gemm = [&](MatrixView<double> c, ConstMatrixView<double>, ConstMatrixView<double>, bool,
                                      bool, double, bool accumulate) {
    if (!accumulate)
      for (index_t i = 0; i < c.rows; ++i)
        for (index_t j = 0; j < c.cols; ++j) c(i, j) = 42.0;
    return true;
  };
  Matrix<double> hijacked = gemm2(a, b);
  check(hijacked(0, 0) == 42.0, "hook: claiming backend's sentinel shows up");
  kernel_backend<double>().gemm = nullptr;
  Matrix<double> restored = gemm2(a, b);
  check(rel<double>(restored.view(), base.view()) == 0, "hook: cleared hook restores the reference");
}

template <typename T>
static void device_backend_runs_reference_ops(double tol) {
  const char* tn = sizeof(T) == 8 ? "f64" : "f32";
  char buf[128];
  std::mt19937_64 rng(20260816);
  // gemm2, all flag cases, a size that takes the tiled DMMA / tcgen05 routes
  for (int ta = 0; ta < 2; ++ta)
    for (int tb = 0; tb < 2; ++tb) {
      const index_t m = 300, n = 260, k = 270;
      Matrix<T> a = ta ? rnd<T>(k, m, rng) : rnd<T>(m, k, rng);
      Matrix<T> b = tb ? rnd<T>(n, k, rng) : rnd<T>(k, n, rng);
      kernel_backend<T>().gemm = nullptr;
      Matrix<T> want = gemm2(a, b, ta, tb, T(0.75));
      install_device_backend<T>();
      const long before = g_device_gemms;
      Matrix<T> got = gemm2(a, b, ta, tb, T(0.75));
      std::snprintf(buf, sizeof buf, "backend %s: gemm2 ta=%d tb=%d on device", tn, ta, tb);
      check(g_device_gemms > before && rel<T>(got.view(), want.view()) < tol, buf, rel<T>(got.view(), want.view()));
    }
  // the reference's own pullbacks route their products through the hook
  {
    const index_t n = 96;
    Matrix<T> a = spd<T>(n, rng);
    Matrix<T> l = potrf(a);
    Matrix<T> bi = potri(l);
    Matrix<T> bbar = rnd<T>(n, n, rng);
    kernel_backend<T>().gemm = nullptr;
    Matrix<T> want = potri_backward(bbar, l, bi);
    install_device_backend<T>();
    const long before = g_device_gemms;
    Matrix<T> got = potri_backward(bbar, l, bi);
    std::snprintf(buf, sizeof buf, "backend %s: reference potri_backward, products on device", tn);
    check(g_device_gemms > before && rel<T>(got.view(), want.view()) < tol * 10, buf, rel<T>(got.view(), want.view()));
  }
  {
    const index_t m = 24, n = 80;
    Matrix<T> a = rnd<T>(m, n, rng);
    Matrix<T> q(a), l(m, m);
    gelqf_inplace<T>(q.view(), l.view());
    Matrix<T> qbar = rnd<T>(m, n, rng), lbar = rnd<T>(m, m, rng);
    kernel_backend<T>().gemm = nullptr;
    Matrix<T> want(m, n), got(m, n);
    gelqf_backward_into<T>(want.view(), qbar.view(), lbar.view(), q.view(), l.view());
    install_device_backend<T>();
    const long before = g_device_gemms;
    gelqf_backward_into<T>(got.view(), qbar.view(), lbar.view(), q.view(), l.view());
    std::snprintf(buf, sizeof buf, "backend %s: reference gelqf_backward, products on device", tn);
    check(g_device_gemms > before && rel<T>(got.view(), want.view()) < tol * 10, buf, rel<T>(got.view(), want.view()));
  }
  kernel_backend<T>().gemm = nullptr;
}

// Direct C-ABI calls from C++ vs the reference on the same inputs.
static void direct_operator_calls() {
  std::mt19937_64 rng(7);
  const index_t n = 256, batch = 2;
  std::vector<Matrix<double>> as, lbars;
  for (index_t b = 0; b < batch; ++b) {
    as.push_back(spd<double>(n, rng));
    Matrix<double> lb = rnd<double>(n, n, rng);
    for (index_t i = 0; i < n; ++i)
      for (index_t j = i + 1; j < n; ++j) lb(i, j) = 0;
    lbars.push_back(lb);
  }
  const size_t mat = sizeof(double) * n * n;
  Dev da(mat * batch), dlb(mat * batch), dab(mat * batch), dinfo(sizeof(int32_t) * batch);
  for (index_t b = 0; b < batch; ++b) {
    cudaMemcpy(da.as<double>() + b * n * n, as[b].data(), mat, cudaMemcpyHostToDevice);
    cudaMemcpy(dlb.as<double>() + b * n * n, lbars[b].data(), mat, cudaMemcpyHostToDevice);
  }
  cudaStream_t s;
  cudaStreamCreate(&s);
  size_t wsf = dla_workspace_bytes(DLA_OP_POTRF, DLA_F64, batch, n, n, 0, 0);
  size_t wsbk = dla_workspace_bytes(DLA_OP_POTRF, DLA_F64, batch, n, n, 0, DLA_WS_BACKWARD);
  Dev w1(wsf), w2(wsbk);
  dla_status st = dla_potrf_fwd_f64(batch, n, da.as<double>(), 1, dinfo.as<int32_t>(), w1.p, wsf, s);
  int64_t bad = -1, idx = -1;
  if (st == DLA_OK) st = dla_info_check(dinfo.as<int32_t>(), batch, s, &bad, &idx);
  check(st == DLA_OK, "C-ABI: dla_potrf_fwd_f64 status");
  st = dla_potrf_bwd_f64(batch, n, dab.as<double>(), dlb.as<double>(), da.as<double>(), 1, w2.p, wsbk, s);
  cudaStreamSynchronize(s);
  check(st == DLA_OK, "C-ABI: dla_potrf_bwd_f64 status");
  double el = 0, eb = 0;
  for (index_t b = 0; b < batch; ++b) {
    Matrix<double> l(n, n), ab(n, n);
    cudaMemcpy(l.data(), da.as<double>() + b * n * n, mat, cudaMemcpyDeviceToHost);
    cudaMemcpy(ab.data(), dab.as<double>() + b * n * n, mat, cudaMemcpyDeviceToHost);
    Matrix<double> lr(as[b]);
    potrf_inplace<double>(lr.view(), true);
    Matrix<double> abr(n, n);
    potrf_backward_into<double>(abr.view(), lbars[b].view(), lr.view(), true);
    el = std::fmax(el, rel<double>(l.view(), lr.view()));
    eb = std::fmax(eb, rel<double>(ab.view(), abr.view()));
  }
  check(el < 1e-12, "C-ABI: potrf (batch 2 x 256^2) vs reference potrf_inplace", el);
  check(eb < 1e-10, "C-ABI: potrf pullback vs reference potrf_backward_into", eb);
  // singular trsm: the reference's SingularError index through info
  {
    Matrix<double> t = Matrix<double>::from_rows({{1, 0}, {5, 0}});
    Matrix<double> x = Matrix<double>::from_rows({{2}, {3}});
    Dev dt(sizeof(double) * 4), dx(sizeof(double) * 2), di(sizeof(int32_t));
    cudaMemcpy(dt.p, t.data(), sizeof(double) * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dx.p, x.data(), sizeof(double) * 2, cudaMemcpyHostToDevice);
    st = dla_trsm_fwd_f64(1, 2, 1, dt.as<double>(), dx.as<double>(), 0, 0, 1, 1.0, di.as<int32_t>(), nullptr, 0, s);
    dla_status code = st == DLA_OK ? dla_info_check(di.as<int32_t>(), 1, s, &bad, &idx) : st;
    check(code == DLA_ERR_SINGULAR && idx == 1, "C-ABI: singular trsm -> SINGULAR(1) (test_blas_kernels.cpp:94)");
  }
  // syevd KAT (proj/tests/test_eigen.cpp:14-26)
  {
    Matrix<double> a = Matrix<double>::from_rows({{0, 1}, {1, 0}});
    Dev du(sizeof(double) * 4), dl(sizeof(double) * 2), di(sizeof(int32_t));
    cudaMemcpy(du.p, a.data(), sizeof(double) * 4, cudaMemcpyHostToDevice);
    size_t wse = dla_workspace_bytes(DLA_OP_SYEVD, DLA_F64, 1, 2, 2, 0, 0);
    Dev we(wse);
    st = dla_syevd_fwd_f64(1, 2, du.as<double>(), dl.as<double>(), di.as<int32_t>(), we.p, wse, s);
    double u[4], lam[2];
    cudaMemcpy(u, du.p, sizeof u, cudaMemcpyDeviceToHost);
    cudaMemcpy(lam, dl.p, sizeof lam, cudaMemcpyDeviceToHost);
    const double h = std::sqrt(0.5);
    const bool ok = st == DLA_OK && std::fabs(lam[0] + 1) < 1e-14 && std::fabs(lam[1] - 1) < 1e-14 &&
                    std::fabs(u[0] - h) < 1e-14 && std::fabs(u[1] + h) < 1e-14 && std::fabs(u[2] - h) < 1e-14 &&
                    std::fabs(u[3] - h) < 1e-14;
    check(ok, "C-ABI: syevd [[0,1],[1,0]] KAT (test_eigen.cpp:14-26)");
  }
  cudaStreamDestroy(s);
}

int main() {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    std::printf("no CUDA device\n");
    return 3;
  }
  replay_reference_hook_test();
  device_backend_runs_reference_ops<double>(1e-13);
  device_backend_runs_reference_ops<float>(2e-5);
  direct_operator_calls();
  std::printf("device gemms through the hook: %ld\n", g_device_gemms);
  std::printf(g_fail ? "FAILED %d\n" : "ALL OK\n", g_fail);
  return g_fail ? 1 : 0;
}
