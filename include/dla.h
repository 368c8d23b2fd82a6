/*
 * dla.h — C-ABI of the B200-native batched differentiable linear-algebra
 * operator set (libdla_b200.so).
 *
 * This is the drop-in boundary for the reference's operator layer
 * (/root/reference/proj/include/dlinalg; "dl/" below).  Every entry point is
 * a batched, stream-ordered replacement of one reference `*_inplace` /
 * `*_into` / `*_backward_into` function, with the same argument meaning,
 * flags, aliasing rules and error taxonomy:
 *
 *   layout     packed row-major, batch-major: matrix b of an r x c operand
 *              starts at ptr + b*r*c (dl/matrix.hpp:181-213, BatchTensor).
 *   pointers   all matrix/vector pointers are DEVICE pointers.
 *   flags      int 0/1, exactly the reference's bool flags.
 *   info       optional (nullable) device int32[batch].  0 = slice OK, else
 *              DLA_INFO(code, index): code is a dla_status, index the
 *              reference exception's payload (pivot step, zero-diagonal
 *              index, rank row, QL iteration count).  The first failing
 *              slice's info is what the reference would have thrown
 *              (dl/matrix.hpp:232-239); use dla_info_check() to read it.
 *   workspace  every operator takes (ws, ws_bytes): caller-owned device
 *              scratch of at least dla_workspace_bytes() bytes (any
 *              alignment; NULL/0 when the query returns 0).  ALL internal
 *              scratch is carved from it -- no entry point allocates device
 *              memory -- and a too-small workspace returns DLA_ERR_WORKSPACE
 *              before any launch that would need it.  The workspace must stay
 *              untouched until the op's work on `stream` has completed
 *              (stream order: the next call on the same stream may reuse it).
 *   stream     cudaStream_t passed as void*; 0 = legacy default stream.
 *   threading  no process-global mutable state on the compute path: device
 *              properties and kernel attributes are per device (the current
 *              device at the call), fork/join side streams and events are
 *              per (device, caller stream) and locked for the enqueue, so
 *              calls from different host threads on different streams or
 *              devices are independent.  Calls on ONE stream from several
 *              threads are serialised by the caller (stream order).
 *
 * Host-side validation (shape, aliasing) runs before any launch and
 * returns a status synchronously; numerical failures are per-slice and
 * land in info[].  The reference throws for aliasing that it forbids
 * (dl/blas.hpp:33-38, :58-59, :146, :197): these return DLA_ERR_ALIAS.
 *
 * Precision: the f64 path computes in IEEE binary64 end to end (FP64 DMMA
 * tensor cores for the blocked contractions).  The f32 path computes in
 * binary32: FFMA for small products, and for large products (m, n >= 256,
 * k >= 128) 3xTF32 on the tcgen05 tensor cores -- each operand split once
 * into TF32 hi + lo, C += hi*hi + hi*lo + lo*hi with fp32 accumulation,
 * i.e. binary32-level accuracy (DLA_SGEMM_TC=0
 * keeps every f32 product on FFMA).
 */
#ifndef DLA_B200_H_
#define DLA_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error taxonomy: dl/common.hpp:20-57. */
typedef enum dla_status {
  DLA_OK = 0,
  DLA_ERR_SHAPE = 1,        /* ShapeError: dims / non-square / m > n       */
  DLA_ERR_NOT_SPD = 2,      /* NotPositiveDefiniteError{step}              */
  DLA_ERR_SINGULAR = 3,     /* SingularError{index}                        */
  DLA_ERR_CONVERGENCE = 4,  /* ConvergenceError{iterations}                */
  DLA_ERR_ALIAS = 5,        /* Error: output must not alias this input     */
  DLA_ERR_ASYMMETRIC = 6,   /* ShapeError: input is not symmetric          */
  DLA_ERR_CUDA = 7,         /* launch / runtime failure                    */
  DLA_ERR_WORKSPACE = 8,    /* workspace missing or too small              */
  DLA_ERR_INVALID = 9       /* bad argument (negative batch, null pointer) */
} dla_status;

#define DLA_INFO(code, index) (((int32_t)(code) << 24) | ((int32_t)(index) & 0xFFFFFF))
#define DLA_INFO_CODE(v) ((int32_t)(v) >> 24)
#define DLA_INFO_INDEX(v) ((int32_t)(v) & 0xFFFFFF)

typedef enum dla_op {
  DLA_OP_GEMM = 0, DLA_OP_GEMM2 = 1, DLA_OP_SYRK = 2, DLA_OP_TRMM = 3,
  DLA_OP_TRSM = 4, DLA_OP_POTRF = 5, DLA_OP_POTRI = 6, DLA_OP_SUMLOGDIAG = 7,
  DLA_OP_GELQF = 8, DLA_OP_SYEVD = 9, DLA_OP_CHOL_CHAIN = 10, DLA_OP_GESVD = 11
} dla_op;

typedef enum dla_dtype { DLA_F32 = 0, DLA_F64 = 1 } dla_dtype;

/* dla_workspace_bytes phase flags */
#define DLA_WS_BACKWARD 1  /* the op's pullback (else its forward)          */
#define DLA_WS_RIGHTSIDE 2 /* trmm / trsm with rightside = 1                */

const char* dla_status_string(dla_status s);
const char* dla_version(void);

/* Device workspace (bytes) one call of the op needs; 0 = none.  Host-only
 * (no device access), deterministic in its arguments.  Dimensions as the op
 * takes them: gemm/gemm2 (m, n, k); syrk (n, k); trmm/trsm (m, n) of X plus
 * DLA_WS_RIGHTSIDE; potrf/potri/sumlogdiag/syevd/chol_chain n; gelqf/gesvd
 * (m, n).  `phase`: DLA_WS_BACKWARD for the pullback.  The reference's own
 * budgets (dl/adjoints.hpp:1-9: gelqf tau m, gelqf bwd m*m, syevd n*n + 9n,
 * syevd bwd n*n; zero for gemm2/syrk/trmm/trsm/potrf/potri pullbacks) are
 * what the CPU needs; the device schedules here add their own scratch (the
 * inverse-based pullbacks' n*n factor inverse, the narrow solve's publish
 * buffer, packed tcgen05 operands for large f32 products) and the query
 * returns that sum. */
size_t dla_workspace_bytes(dla_op op, dla_dtype dtype, int64_t batch, int64_t m,
                           int64_t n, int64_t k, int phase);

/* Reads info[0..batch) (synchronises `stream`).  Returns DLA_OK when every
 * slice is clean, else the first failing slice's code, with *first_bad /
 * *index set (each nullable). */
dla_status dla_info_check(const int32_t* info, int64_t batch, void* stream,
                          int64_t* first_bad, int64_t* index);

/* ---------------------------------------------------------------- macros */
/* Each operator is declared for f32 and f64 through one prototype list.   */

#define DLA_DECLARE_OPS(T, S)                                                       \
  /* gemm2: C = alpha op(A) op(B); dl/blas.hpp:119-122 (gemm_accum :43-110).      \
     A is (ta ? k x m : m x k), B is (tb ? n x k : k x n), C is m x n.           \
     C must not alias A or B. */                                                    \
  dla_status dla_gemm2_fwd_##S(int64_t batch, int64_t m, int64_t n, int64_t k,      \
                               T* c, const T* a, const T* b, int ta, int tb,        \
                               T alpha, void* ws, size_t ws_bytes, void* stream);                              \
  /* gemm: C = alpha op(A) op(B) + beta C.  beta = 0 / 1 are the reference's        \
     gemm_accum(accumulate = false / true) (dl/blas.hpp:43-110); other beta         \
     scale C first. */                                                              \
  dla_status dla_gemm_fwd_##S(int64_t batch, int64_t m, int64_t n, int64_t k,       \
                              T* c, const T* a, const T* b, int ta, int tb,         \
                              T alpha, T beta, void* ws, size_t ws_bytes, void* stream);                       \
  /* gemm2 / gemm pullback: dl/adjoints.hpp:36-49 (Abar written before Bbar). */    \
  dla_status dla_gemm2_bwd_##S(int64_t batch, int64_t m, int64_t n, int64_t k,      \
                               T* abar, T* bbar, const T* cbar, const T* a,         \
                               const T* b, int ta, int tb, T alpha, void* ws, size_t ws_bytes, void* stream);  \
  /* gemm pullback: abar/bbar as gemm2; cbar_io <- beta * cbar_io (the C-input     \
     cotangent), after abar/bbar are formed. */                                     \
  dla_status dla_gemm_bwd_##S(int64_t batch, int64_t m, int64_t n, int64_t k,       \
                              T* abar, T* bbar, T* cbar_io, const T* a,             \
                              const T* b, int ta, int tb, T alpha, T beta,          \
                              void* ws, size_t ws_bytes, void* stream);                                        \
  /* syrk: B = alpha A A^T (ta=0, A n x k) / alpha A^T A (ta=1, A k x n),           \
     bit-exactly symmetric; dl/blas.hpp:138-169. */                                 \
  dla_status dla_syrk_fwd_##S(int64_t batch, int64_t n, int64_t k, T* b,            \
                              const T* a, int ta, T alpha, void* ws, size_t ws_bytes, void* stream);           \
  /* syrk pullback: dl/adjoints.hpp:69-78. */                                       \
  dla_status dla_syrk_bwd_##S(int64_t batch, int64_t n, int64_t k, T* abar,         \
                              const T* bbar, const T* a, int ta, T alpha,           \
                              void* ws, size_t ws_bytes, void* stream);                                        \
  /* trmm: X <- alpha op(T) X (right=0) / alpha X op(T) (right=1); X m x n,         \
     T m x m (left) or n x n (right); dl/blas.hpp:202-291. */                       \
  dla_status dla_trmm_fwd_##S(int64_t batch, int64_t m, int64_t n, const T* t,      \
                              T* x, int rightside, int transpose, int lower,        \
                              T alpha, void* ws, size_t ws_bytes, void* stream);                               \
  /* trmm out of place: y = alpha op(T) x / alpha x op(T); x, t unchanged, y may  \
     alias neither; same workspace as dla_trmm_fwd. */                              \
  dla_status dla_trmm_into_##S(int64_t batch, int64_t m, int64_t n, const T* t,     \
                               const T* x, T* y, int rightside, int transpose,      \
                               int lower, T alpha, void* ws, size_t ws_bytes, void* stream);                   \
  /* trmm pullback (reads the forward INPUT a); abar may alias bbar;                \
     dl/adjoints.hpp:94-110. */                                                     \
  dla_status dla_trmm_bwd_##S(int64_t batch, int64_t m, int64_t n, T* abar,         \
                              T* tbar, const T* bbar, const T* t, const T* a,       \
                              int rightside, int transpose, int lower, T alpha,     \
                              void* ws, size_t ws_bytes, void* stream);                                        \
  /* trsm: X <- alpha op(T)^-1 X / alpha X op(T)^-1; exact zero diagonal =>         \
     SINGULAR(k) in info and the slice is left untouched; dl/blas.hpp:307-395. */   \
  dla_status dla_trsm_fwd_##S(int64_t batch, int64_t m, int64_t n, const T* t,      \
                              T* x, int rightside, int transpose, int lower,        \
                              T alpha, int32_t* info, void* ws, size_t ws_bytes, void* stream);                \
  /* trsm pullback (reads the forward OUTPUT b); abar may alias bbar;               \
     dl/adjoints.hpp:131-153. */                                                    \
  dla_status dla_trsm_bwd_##S(int64_t batch, int64_t m, int64_t n, T* abar,         \
                              T* tbar, const T* bbar, const T* t, const T* b,       \
                              int rightside, int transpose, int lower, T alpha,     \
                              void* ws, size_t ws_bytes, void* stream);                                        \
  /* potrf: A = L L^T (lower=1, strict upper zeroed) / A = R^T R (lower=0), in      \
     place.  Asymmetric input => ASYMMETRIC (slice untouched); failed pivot =>      \
     NOT_SPD(step); dl/cholesky.hpp:79-88. */                                       \
  dla_status dla_potrf_fwd_##S(int64_t batch, int64_t n, T* a, int lower,           \
                               int32_t* info, void* ws, size_t ws_bytes, void* stream);                        \
  /* potrf pullback: Abar = 1/2 L^-T copyltu(L^T Lbar) L^-1, exactly symmetric;     \
     abar may alias lbar; dl/adjoints.hpp:175-191. */                               \
  dla_status dla_potrf_bwd_##S(int64_t batch, int64_t n, T* abar, const T* lbar,    \
                               const T* l, int lower, void* ws, size_t ws_bytes, void* stream);                \
  /* potri: B = A^-1 from the Cholesky factor, in place, exactly symmetric;         \
     zero diagonal => SINGULAR(j); dl/cholesky.hpp:141-147. */                      \
  dla_status dla_potri_fwd_##S(int64_t batch, int64_t n, T* a, int lower,           \
                               int32_t* info, void* ws, size_t ws_bytes, void* stream);                        \
  /* potri out of place: b = inv(L L^T) from the factor l (unchanged); same info  \
     and workspace as the in-place potri; fp64 64 < n <= 128: one fused launch */ \
  dla_status dla_potri_into_##S(int64_t batch, int64_t n, const T* l, T* b,         \
                                int lower, int32_t* info, void* ws, size_t ws_bytes, void* stream);            \
  /* potri pullback: Lbar = -tril((B Bbar + B Bbar^T) L^-T); dl/adjoints.hpp:207. */\
  dla_status dla_potri_bwd_##S(int64_t batch, int64_t n, T* lbar, const T* bbar,    \
                               const T* l, const T* b, int lower, void* ws, size_t ws_bytes, void* stream);    \
  /* sumlogdiag: out[b] = sum_i log A_b(i,i) (tape chain ExtractDiag->Log->Sum,   \
     dl/tape.hpp:789-795, :714, :747-755), summed as per-thread strided partials    \
     reduced by a fixed-order tree: deterministic, NOT the reference's sequential  \
     i order (agrees to ~n u). */                                                   \
  dla_status dla_sumlogdiag_fwd_##S(int64_t batch, int64_t n, T* out, const T* a,   \
                                    void* ws, size_t ws_bytes, void* stream);                                  \
  /* sumlogdiag pullback: abar(i,i) = gbar[b] / A(i,i), off-diagonal exactly 0      \
     (accumulate=0) or untouched (accumulate=1: added onto the diagonal). */        \
  dla_status dla_sumlogdiag_bwd_##S(int64_t batch, int64_t n, T* abar,              \
                                    const T* gbar, const T* a, int accumulate,      \
                                    void* ws, size_t ws_bytes, void* stream);                                  \
  /* gelqf: A (m x n, m <= n) = L Q; q: in A, out Q; l: out L (m x m, positive      \
     diagonal); rank deficiency => SINGULAR(row); dl/lq.hpp:24-106.                 \
     workspace: dla_workspace_bytes(DLA_OP_GELQF, ..., 0) (m reals per slice;       \
     m >= 64 runs the blocked compact-WY path: 2mn + 64m + m + 1 reals). */         \
  dla_status dla_gelqf_fwd_##S(int64_t batch, int64_t m, int64_t n, T* q, T* l,     \
                               int32_t* info, void* ws, size_t ws_bytes,            \
                               void* stream);                                       \
  /* gelqf pullback: Abar = L^-T (Qbar + copyltu(L^T Lbar - Qbar Q^T) Q);           \
     one m x m workspace per slice; dl/adjoints.hpp:239-252. */                     \
  dla_status dla_gelqf_bwd_##S(int64_t batch, int64_t m, int64_t n, T* abar,        \
                               const T* qbar, const T* lbar, const T* q,            \
                               const T* l, void* ws, size_t ws_bytes,               \
                               void* stream);                                       \
  /* syevd: A = U^T diag(lambda) U, ROWS of U are eigenvectors, lambda              \
     ascending, sign rule of dl/eigen_sym.hpp:316-333; u: in A, out U;              \
     dl/eigen_sym.hpp:339-367. */                                                   \
  dla_status dla_syevd_fwd_##S(int64_t batch, int64_t n, T* u, T* lambda,           \
                               int32_t* info, void* ws, size_t ws_bytes,            \
                               void* stream);                                       \
  /* syevd pullback with the eps_gap guard; one n x n workspace per slice;          \
     dl/adjoints.hpp:272-295. */                                                    \
  dla_status dla_syevd_bwd_##S(int64_t batch, int64_t n, T* abar, const T* ubar,    \
                               const T* lambdabar, const T* u, const T* lambda,     \
                               T eps_gap, void* ws, size_t ws_bytes, void* stream);

/* gesvd: thin SVD of a wide A (m x n, m <= n), A = U^T diag(lambda) V; ROWS of U
 * (m x m) / V (m x n) are the singular vectors, lambda ascending >= 0, the sign
 * rule of dl/eigen_sym.hpp:316-333 on U's rows with V's rows flipped in
 * lockstep; v: in A, out V (dl/svd.hpp:229-284).  info: CONVERGENCE(sweeps).
 * Pullback (dl/adjoints.hpp:315-382): abar may alias vbar; every lambda_i must
 * exceed eps_gap, else SINGULAR(i) in info and the slice is left untouched. */
#define DLA_DECLARE_GESVD(T, S)                                                                   \
  dla_status dla_gesvd_fwd_##S(int64_t batch, int64_t m, int64_t n, T* v, T* u, T* lambda,      \
                               int32_t* info, void* ws, size_t ws_bytes, void* stream);         \
  dla_status dla_gesvd_bwd_##S(int64_t batch, int64_t m, int64_t n, T* abar, const T* ubar,     \
                               const T* lambdabar, const T* vbar, const T* u, const T* lambda,  \
                               const T* v, T eps_gap, int32_t* info, void* ws, size_t ws_bytes, \
                               void* stream);

DLA_DECLARE_GESVD(float, f32)
DLA_DECLARE_GESVD(double, f64)

DLA_DECLARE_OPS(float, f32)
DLA_DECLARE_OPS(double, f64)

/* --------------------------------------------------------- instrumentation */
/* Kernels launched by this library so far (host-side counter). */
long long dla_launch_count(void);
/* GEMM launch timing with CUDA events on the launching stream (off by
 * default; enabling clears previous records). */
void dla_prof_enable(int on);
long long dla_prof_read(double* ms, double* flops);
/* The recorded GEMM launch(es) with the largest flop count: average event
 * time (ms) and that flop count; returns how many launches tied. */
long long dla_prof_read_max(double* ms, double* flops);

/* --------------------------------------------- split potrf pullback (driver) */
/* dla_potrf_bwd_f64 in two stream-ordered halves so a driver can overlap the
 * factor's inverse with work that only reads L (the GP driver's solves):
 * _begin forks L^-1 onto an internal side stream; _end joins and produces
 * Abar bitwise identical to dla_potrf_bwd_f64 (dl/adjoints.hpp:175-191).  L
 * must not change in between; one begin/end pair in flight per (device,
 * stream).  Sizes where the inverse path does not apply (n != 64 * 2^k) make
 * _begin a no-op and _end the plain pullback.  Workspace: one buffer of
 * dla_potrf_bwd_ws_bytes_f64 bytes, the SAME buffer for every call of a
 * pair (its head holds L^-1 between the calls). */
size_t dla_potrf_bwd_ws_bytes_f64(int64_t batch, int64_t n);
/* dla_potrf_fwd_f64 (lower) fused with _begin for a driver that needs the
 * pullback next: the blocked factorization signals once block columns
 * [0, n/2) are final, and L11^-1 and L21 L11^-1 (half of the inverse's
 * flops) form on the side stream during its chain-bound second half; the
 * rest follows the factorization.  Finish with dla_potrf_bwd_end_f64; L's
 * strict upper triangle is zeroed on the side stream and is complete (stream-
 * ordered) once _end -- or, for a caller that does not need the pullback,
 * dla_potrf_inv_join_f64 -- has been enqueued on `stream`. */
dla_status dla_gp_potrf_inv_f64(int64_t batch, int64_t n, double* a, int32_t* info, void* ws,
                                size_t ws_bytes, void* stream);
dla_status dla_potrf_bwd_begin_f64(int64_t batch, int64_t n, const double* l, int lower, void* ws,
                                   size_t ws_bytes, void* stream);
dla_status dla_potrf_bwd_end_f64(int64_t batch, int64_t n, double* abar, const double* lbar,
                                 const double* l, int lower, void* ws, size_t ws_bytes, void* stream);
/* Makes `stream` wait for the side-stream work of the last _begin /
 * dla_gp_potrf_inv_f64 on it (the join _end performs), without the pullback. */
dla_status dla_potrf_inv_join_f64(void* stream);

/* ----------------------------------------------- fused C1 likelihood chain */
/* Gaussian log-likelihood chain over a batch of small SPD matrices
 * (BASELINE config C1; the make_gp graph dl/models.hpp:99-103 given A):
 *   L = potrf(A);  z = L^-1 y;  phi[b] = 1/2 z^T z + sum_i log L_ii
 * and its pullback at phibar = 1: ybar = L^-T z and Abar = dphi/dA (trsm,
 * sumlogdiag and potrf backward: dl/adjoints.hpp:131-153, 175-191,
 * dl/tape.hpp:1038-1045).  a, abar: [batch, n, n]; y, ybar: [batch, n, 1];
 * phi: [batch].  n <= 32 runs as ONE launch (one warp per matrix); larger n
 * composes the operators.  Failures as potrf (info: ASYMMETRIC, NOT_SPD(step));
 * outputs of a failed slice are untouched.  No output may overlap an input. */
dla_status dla_chol_chain_fwdbwd_f64(int64_t batch, int64_t n, const double* a, const double* y,
                                     double* phi, double* abar, double* ybar, int32_t* info,
                                     void* ws, size_t ws_bytes, void* stream);
dla_status dla_chol_chain_fwdbwd_f32(int64_t batch, int64_t n, const float* a, const float* y,
                                     float* phi, float* abar, float* ybar, int32_t* info,
                                     void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------ GP driver */
/* Fused RBF-kernel build and pullback for the Gaussian-process NLL driver
 * (dl/models.hpp:50-65 rbf_kernel + :95-98 K + lam I; pullbacks of the tape
 * chain dl/tape.hpp:930-1036).  x: [batch, n, d] (d <= 32), a/abar:
 * [batch, n, n].  grads: [batch, 3] = d phi / d(log sigma2, log ell2,
 * log lam) given abar = d phi / dA; xbar (nullable): [batch, n, d].
 * workspace: dla_gp_rbf_ws_bytes(batch, n, d). */
size_t dla_gp_rbf_ws_bytes(int64_t batch, int64_t n, int64_t d);
dla_status dla_gp_rbf_fwd_f64(int64_t batch, int64_t n, int64_t d, const double* x, double sigma2,
                              double ell2, double lam, double* a, void* ws, size_t ws_bytes,
                              void* stream);
dla_status dla_gp_rbf_bwd_f64(int64_t batch, int64_t n, int64_t d, const double* x, double sigma2,
                              double ell2, double lam, const double* abar, double* xbar,
                              double* grads, void* ws, size_t ws_bytes, void* stream);
/* Device tape node kernels: the reference tape's
 * elementwise / structural nodes and their pullbacks (dl/tape.hpp
 * compute_node :615-790, pull_node :930-1120, acc :920-929) for the device
 * Graph (paper_1710_08717_b200/tape.py).  One matrix (no batch), row-major.
 *   out = f(x[, y][, s[0]][, c])      accumulate != 0:  out += f(...)
 * x is rows x cols unless stated.  out may alias x (in-place nodes of the
 * memory plan) for the map ops (COPY .. ABS_BWD).  SUM / DOT / DOT_NEG_DIV
 * need dla_tape_ew_ws_bytes() of workspace (fixed-order reduction). */
typedef enum {
  DLA_EW_COPY = 0, DLA_EW_ADD = 1, DLA_EW_SUB = 2, DLA_EW_MUL = 3,
  DLA_EW_SQUARE = 4, DLA_EW_SQRT = 5, DLA_EW_LOG = 6, DLA_EW_EXP = 7,
  DLA_EW_ABS = 8, DLA_EW_NEG = 9,
  DLA_EW_SCALE = 10,      /* x * c                                         */
  DLA_EW_ADDC = 11,       /* x + c                                         */
  DLA_EW_MULS = 12,       /* x * s[0]  (MulScalar)                         */
  DLA_EW_DIVS = 13,       /* x / s[0]  (DivScalar)                         */
  DLA_EW_FILL = 14,       /* s[0] everywhere (Sum pullback)                */
  DLA_EW_SQUARE_BWD = 15, /* x * (2 y)       x = gbar, y = input           */
  DLA_EW_SQRT_BWD = 16,   /* x / (2 y)       y = output                    */
  DLA_EW_LOG_BWD = 17,    /* x / y           y = input                     */
  DLA_EW_ABS_BWD = 18,    /* x * sign(y)     y = input                     */
  DLA_EW_TRIL = 19, DLA_EW_TRIU = 20,  /* square x                         */
  DLA_EW_TILECOLS = 21,   /* x rows x 1 -> rows x aux                      */
  DLA_EW_TILEROWS = 22,   /* x rows x 1 -> aux x rows                      */
  DLA_EW_EXTRACTDIAG = 23,/* x n x n -> n x 1                              */
  DLA_EW_MAKEDIAG = 24,   /* x n x 1 -> n x n                              */
  DLA_EW_CONCATCOLS = 25, /* [x | y], y rows x aux                         */
  DLA_EW_SLICECOLS = 26,  /* x rows x aux -> columns [c, c + cols)         */
  DLA_EW_SUMROWS = 27,    /* -> rows x 1                                   */
  DLA_EW_SUMCOLS = 28,    /* -> cols x 1                                   */
  DLA_EW_SUM = 29,        /* -> 1 x 1                                      */
  DLA_EW_DOT = 30,        /* sum(x * y) -> 1 x 1                           */
  DLA_EW_DOT_NEG_DIV = 31 /* -sum(x * y) / s[0] -> 1 x 1                   */
} dla_ew_op;
size_t dla_tape_ew_ws_bytes(void);
dla_status dla_tape_ew_f64(int op, int64_t rows, int64_t cols, int64_t aux, const double* x,
                           const double* y, const double* s, double c, double* out, int accumulate,
                           void* ws, size_t ws_bytes, void* stream);
dla_status dla_tape_ew_f32(int op, int64_t rows, int64_t cols, int64_t aux, const float* x,
                           const float* y, const float* s, float c, float* out, int accumulate,
                           void* ws, size_t ws_bytes, void* stream);

/* Batched Kalman filter NLL + gradient of every leaf:
 * the reference's build_kalman_nll graph (dl/models.hpp:285-337, Joseph-form
 * covariance update, first observation scored against the prior) and
 * Graph::backward over it, one launch for `batch` sequences.
 *   a [h,h] transition, b [d,h] emission, sh [h,h] / sv [d,d] process /
 *   observation noise, mu0 [h,1] / s0 [h,h] prior, obs [batch][T][d]
 *   (row t = observation t of that sequence).  param_stride 1: every
 *   parameter carries a leading [batch] dimension; 0: one model shared by
 *   all sequences.
 *   nll [batch]; abar bbar shbar svbar mu0bar s0bar: [batch] x the parameter
 *   shapes (per-sequence gradients; a shared model sums them); obsbar
 *   (nullable) [batch][T][d].  h, d <= 32 (SHAPE otherwise; T >= 1).
 *   info[b]: NOT_SPD with index t*d + pivot when step t's innovation
 *   covariance is not positive definite (that sequence's outputs untouched).
 *   workspace: dla_kalman_ws_bytes_{f32,f64} (the device tape of the
 *   intermediates of every step). */
size_t dla_kalman_ws_bytes_f64(int64_t batch, int64_t h, int64_t d, int64_t T);
size_t dla_kalman_ws_bytes_f32(int64_t batch, int64_t h, int64_t d, int64_t T);
dla_status dla_kalman_nll_fwdbwd_f64(int64_t batch, int64_t h, int64_t d, int64_t T, const double* a,
                                     const double* b, const double* sh, const double* sv,
                                     const double* mu0, const double* s0, const double* obs,
                                     int64_t param_stride, double* nll, double* abar, double* bbar,
                                     double* shbar, double* svbar, double* mu0bar, double* s0bar,
                                     double* obsbar, int32_t* info, void* ws, size_t ws_bytes,
                                     void* stream);
dla_status dla_kalman_nll_fwdbwd_f32(int64_t batch, int64_t h, int64_t d, int64_t T, const float* a,
                                     const float* b, const float* sh, const float* sv,
                                     const float* mu0, const float* s0, const float* obs,
                                     int64_t param_stride, float* nll, float* abar, float* bbar,
                                     float* shbar, float* svbar, float* mu0bar, float* s0bar,
                                     float* obsbar, int32_t* info, void* ws, size_t ws_bytes,
                                     void* stream);
/* The GP step's pullback tail fused (dl/models.hpp:115-135 backward from
 * Lbar): potrf_backward_into (dl/adjoints.hpp:175-191) up to
 * Z = L^-T P' L^-1 with L^-1 from dla_gp_potrf_inv_f64 / _begin (iws, the
 * same workspace), then the RBF pullback reading Abar = 1/2 (Z + Z^T) tile
 * pair by tile pair (Abar is never materialized; lbar is clobbered).  grads
 * and xbar as dla_gp_rbf_bwd_f64.  rws: dla_gp_pullback_ws_bytes. */
size_t dla_gp_rbf_bwd_sym_ws_bytes(int64_t batch, int64_t n, int64_t d);
size_t dla_gp_pullback_ws_bytes(int64_t batch, int64_t n, int64_t d);
dla_status dla_gp_pullback_f64(int64_t batch, int64_t n, int64_t d, const double* x, double sigma2,
                               double ell2, double lam, double* lbar, const double* l, double* xbar,
                               double* grads, void* iws, size_t iws_bytes, void* rws, size_t rws_bytes,
                               void* stream);
/* nll[b] = quad[b] + logdet[b] + n/2 log(2 pi)  (dl/models.hpp:100-103). */
dla_status dla_gp_nll_assemble_f64(int64_t batch, int64_t n, const double* quad,
                                   const double* logdet, double* nll, void* stream);

/* ------------------------------------- batched marginal-likelihood driver */
/* Helpers of the C5 driver (batched GP marginal likelihoods; the graph is
 * SURVEY §8d's, built from reference ops): a = s + lam I (batch of n x n);
 * y += alpha x (count elements); out[0] = sum_b (quad_b + logdet_b) +
 * batch n/2 log 2 pi and out[1] = lam sum_b tr(abar_b), summed in a fixed
 * order (deterministic). */
dla_status dla_ml_shift_copy_f64(int64_t batch, int64_t n, const double* s, double* a, double lam,
                                 void* stream);
dla_status dla_axpy_f64(int64_t count, double alpha, const double* x, double* y, void* stream);
size_t dla_ml_reduce_ws_bytes(int64_t batch);
dla_status dla_ml_reduce_f64(int64_t batch, int64_t n, const double* quad, const double* logdet,
                             const double* abar, double lam, double* out, void* ws, size_t ws_bytes,
                             void* stream);

#ifdef __cplusplus
}
#endif

#endif /* DLA_B200_H_ */
