// Internal declarations of the fused / special-purpose operator kernels.
#pragma once

#include "common.cuh"

namespace dlab {

// small.cu — one CTA per matrix, whole matrix in shared memory (n <= 64).
template <typename T>
bool potrf_small_eligible(int64_t n);
template <typename T>
bool potrf_fwd_small_eligible(int64_t n);
template <typename T>
// check_sym: the public op's symmetry precheck (dl/cholesky.hpp:19-25); internal
// callers that factor a lower triangle (strict upper unspecified) pass false
// (honoured by the 64 < n <= 128 kernel; the smaller ones are public-op only).
dla_status potrf_small(const Ctx& c, int64_t batch, int64_t n, MatB<T> a, bool lower, bool check_sym = true);
template <typename T>
dla_status potrf_bwd_small(const Ctx& c, int64_t batch, int64_t n, MatB<T> abar, MatB<const T> lbar,
                           MatB<const T> l, bool lower);

// Fused C1 chain (n <= 32, warp per matrix): phi = 1/2 |L^-1 y|^2 + sumlogdiag(L),
// L = potrf(A), with ybar and Abar at phibar = 1.
template <typename T>
dla_status chol_chain_small(const Ctx& c, int64_t batch, int64_t n, MatB<const T> a, const T* y, T* phi, MatB<T> abar,
                            T* ybar);

// inv.cu — inverse-based large-n paths (n = 64 * 2^k, n >= 256)
template <typename T>
bool inv_eligible(int64_t n);
template <typename T>
int64_t inv_pad(int64_t n);
template <typename T>
dla_status trsm_inv_from(const Ctx& c, int64_t batch, int64_t m, int64_t n, MatB<const T> t, MatB<const T> src,
                         MatB<T> x, bool right, bool trans, bool lower, T alpha);
template <typename T>
size_t ws_trsm_inv_from(int64_t batch, int64_t m, int64_t n, bool right);
template <typename T>
bool potri_fused_eligible(int64_t n);
dla_status potri128_into(const Ctx& c, int64_t batch, int64_t n, MatB<const double> l, bool from_upper,
                         MatB<double> b);
template <typename T>
dla_status trsm_inv(const Ctx& c, int64_t batch, int64_t m, int64_t n, MatB<const T> t, MatB<T> x, bool right,
                    bool trans, bool lower, T alpha);
template <typename T>
dla_status potrf_bwd_inv(const Ctx& c, int64_t batch, int64_t n, MatB<T> abar, MatB<const T> lbar, MatB<const T> l,
                         bool lower);
template <typename T>
size_t trtri_levels_tmp(int64_t n);
template <typename T>
dla_status trtri_levels(const Ctx& c, int64_t batch, int64_t n, MatB<T> w, T* tmp,
                        const MatB<const T>* src = nullptr, bool from_upper = false);
template <typename T>
dla_status potrf_inv_prepare(const Ctx& c, int64_t batch, int64_t n, MatB<const T> l, bool lower, MatB<T> wi, T* tmp);
template <typename T>
dla_status potrf_bwd_from_inv(const Ctx& c, int64_t batch, int64_t n, MatB<T> abar, MatB<const T> lbar, MatB<const T> l,
                              bool lower, MatB<const T> wi, MatB<T> tt);
template <typename T>
dla_status potrf_bwd_phi(const Ctx& c, int64_t batch, int64_t n, MatB<const T> lbar, MatB<const T> l, bool lower,
                         MatB<T> tt);
template <typename T>
dla_status potrf_bwd_finish(const Ctx& c, int64_t batch, int64_t n, MatB<T> abar, MatB<const T> wi, MatB<T> tt);
template <typename T>
dla_status potrf_bwd_finish_z(const Ctx& c, int64_t batch, int64_t n, MatB<T> abar, MatB<const T> wi, MatB<T> tt);

// gp.cu: the symmetric RBF pullback straight from potrf_bwd's Z (fused GP tail)
bool gp_rbf_sym_ok(int64_t d);
dla_status gp_rbf_bwd_sym(int64_t batch, int64_t n, int64_t d, const double* x, double sigma2, double ell2, double lam,
                          const double* z, double* xbar, double* grads, void* ws, size_t ws_bytes, cudaStream_t s);
template <typename T>
dla_status trmm_gemm(const Ctx& c, int64_t batch, int64_t m, int64_t n, MatB<const T> t, MatB<T> x, bool right,
                     bool trans, bool lower, T alpha);
template <typename T>
dla_status potri_inv(const Ctx& c, int64_t batch, int64_t n, MatB<T> a);
template <typename T>
size_t ws_trtri_levels(int64_t batch, int64_t n);
template <typename T>
size_t ws_trsm_inv(int64_t batch, int64_t m, int64_t n, bool right);
template <typename T>
size_t ws_potrf_inv_prepare(int64_t batch, int64_t n);
template <typename T>
size_t ws_potrf_bwd_tail(int64_t batch, int64_t n);
template <typename T>
size_t ws_potrf_bwd_inv(int64_t batch, int64_t n);
template <typename T>
size_t ws_trmm_gemm(int64_t batch, int64_t m, int64_t n, bool right);
template <typename T>
size_t ws_potri_inv(int64_t batch, int64_t n);

// trsv.cu — one-launch solve for <= 8 right-hand sides (flag-synchronised)
template <typename T>
bool trsv_eligible(int64_t nt, int64_t nvec);
template <typename T>
size_t ws_trsv(int64_t batch, int64_t m, int64_t n, bool right);
template <typename T>
dla_status trsv(const Ctx& c, int64_t batch, int64_t m, int64_t n, MatB<const T> t, MatB<T> x, bool right, bool trans,
                bool lower, T alpha);

// gelqf_blk.cu: blocked (compact WY) LQ, m >= 64
template <typename T>
bool gelqf_blocked_eligible(int64_t m, int64_t n);
template <typename T>
size_t gelqf_blocked_ws_bytes(int64_t batch, int64_t m, int64_t n);
template <typename T>
dla_status gelqf_blocked(const Ctx& c, int64_t batch, int64_t m, int64_t n, T* q, T* l, void* ws,
                         bool rank_check = true);

// gelqf_cqr.cu: CholeskyQR2 LQ (f64) with a per-slice Householder fallback
bool gelqf_cqr_eligible(int64_t m, int64_t n);
size_t ws_gelqf_cqr(int64_t batch, int64_t m, int64_t n);
dla_status gelqf_cqr(const Ctx& c, int64_t batch, int64_t m, int64_t n, double* q, double* l);

// gelqf.cu
template <typename T>
size_t gelqf_ws_bytes(int64_t batch, int64_t m, int64_t n, bool backward);
template <typename T>
dla_status gelqf_fwd(const Ctx& c, int64_t batch, int64_t m, int64_t n, T* q, T* l, void* ws,
                     bool rank_check = true);

// potrf_tiles.cu: persistent tile-dataflow Cholesky (f64, lower, in place;
// strict upper untouched)
bool potrf_tiles_eligible(int64_t batch, int64_t n, const MatB<double>& a);
dla_status potrf_tiles(const Ctx& c, int64_t batch, int64_t n, MatB<double> a, int64_t kbase);
size_t ws_potrf_tiles(int64_t batch, int64_t n);

// gemm_tma.cu: TMA-fed persistent fp64 GEMM for large products (false = not taken)
bool gemm_tma(const Ctx& c, int64_t batch, int64_t m, int64_t n, int64_t k, double alpha, MatB<const double> a,
              bool ta, MatB<const double> b, bool tb, double beta, MatB<double> cm, int mask, const int32_t* skip,
              int tri_a, int tri_b, int64_t inner, dla_status* st);
// syrk_tma.cu: TMA-fed persistent trailing update C[lower] = alpha P P^T + beta C (f64)
bool syrk_tma_eligible(int64_t m, int64_t k, const MatB<const double>& p, const MatB<double>& c, int64_t batch);
dla_status syrk_tma(const Ctx& c, int64_t batch, int64_t m, int64_t k, double alpha, MatB<const double> p, double beta,
                    MatB<double> cm, int max_ctas);

// gesvd.cu: LQ-preconditioned one-sided Jacobi SVD (m <= n) and its pullback
template <typename T>
size_t ws_gesvd_fwd(int64_t batch, int64_t m, int64_t n);
template <typename T>
size_t ws_gesvd_bwd(int64_t batch, int64_t m, int64_t n);
template <typename T>
dla_status gesvd_fwd(const Ctx& c, int64_t batch, int64_t m, int64_t n, T* v, T* u, T* lambda);
template <typename T>
dla_status gesvd_bwd(const Ctx& c, int64_t batch, int64_t m, int64_t n, T* abar, const T* ubar, const T* lambdabar,
                     const T* vbar, const T* u, const T* lambda, const T* v, T eps_gap);

// syevd.cu
template <typename T>
size_t syevd_ws_bytes(int64_t batch, int64_t n, bool backward);
template <typename T>
dla_status syevd_fwd(const Ctx& c, int64_t batch, int64_t n, T* u, T* lambda, void* ws);
template <typename T>
dla_status syevd_gap_kernel(const Ctx& c, int64_t batch, int64_t n, MatB<T> w, const T* lambdabar, const T* lambda,
                            T eps_gap);
template <typename T>
dla_status ew_sym_into(const Ctx& c, int64_t batch, int64_t n, MatB<const T> w, MatB<T> out);

}  // namespace dlab
