/* CPU oracle — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's dense kernels and closed-form
 * pullbacks (dlinalg, /root/reference/proj/include/dlinalg).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this code, and only as the checker.  The product path
 * (paper_1710_08717_b200, libdla_b200.so) never links or calls it.
 *
 * Parity pinning: every function here is checked against (1) the reference's
 * own known-answer tests (tests/golden/kat.json, restated from
 * proj/tests/test_*.cpp) and (2) the real reference compiled from its headers
 * into oracle/_ref/libdla_ref.so (tests/test_oracle_vs_ref.py).
 *
 * This header is instantiated twice by dla_oracle.c: R = double / suffix _f64,
 * R = float / suffix _f32.  Matrices are packed row-major, element (i, j) of an
 * r x c matrix at p[i*c + j] — the reference MatrixView layout
 * (dl/matrix.hpp:64-89).  Return value: a dla status code (include/dla.h);
 * *idx receives the failing index where the reference exception carries one.
 */

#define AT(p, ld, i, j) ((p)[(size_t)(i) * (size_t)(ld) + (size_t)(j)])

/* ----------------------------------------------------------------- helpers */

static R FN(absr)(R v) { return v < (R)0 ? -v : v; }

static R FN(max_abs)(const R* a, int64_t count) {
  R m = (R)0;
  for (int64_t i = 0; i < count; ++i) {
    R v = FN(absr)(a[i]);
    if (v > m) m = v;
  }
  return m;
}

/* dl/transforms.hpp:133-141 + dl/cholesky.hpp:19-25 */
static int FN(symmetric_ok)(int64_t n, const R* a, R rtol) {
  R asym = (R)0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i + 1; j < n; ++j) {
      R d = FN(absr)(AT(a, n, i, j) - AT(a, n, j, i));
      if (d > asym) asym = d;
    }
  R scale = FN(max_abs)(a, n * n);
  return !(asym > rtol * (scale > (R)0 ? scale : (R)1));
}

static void FN(transpose_sq)(int64_t n, R* a) {
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i + 1; j < n; ++j) {
      R t = AT(a, n, i, j);
      AT(a, n, i, j) = AT(a, n, j, i);
      AT(a, n, j, i) = t;
    }
}

/* dl/transforms.hpp:18-32, 49-61, 78-87 */
void FN(o_copyltu)(int64_t n, R* a) {
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i + 1; j < n; ++j) AT(a, n, i, j) = AT(a, n, j, i);
}
void FN(o_copyutl)(int64_t n, R* a) {
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i + 1; j < n; ++j) AT(a, n, j, i) = AT(a, n, i, j);
}
void FN(o_tril)(int64_t n, R* a) {
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i + 1; j < n; ++j) AT(a, n, i, j) = (R)0;
}
void FN(o_triu)(int64_t n, R* a) {
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < i; ++j) AT(a, n, i, j) = (R)0;
}
void FN(o_sym)(int64_t n, R* a) {
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i + 1; j < n; ++j) {
      R v = (AT(a, n, i, j) + AT(a, n, j, i)) / (R)2;
      AT(a, n, i, j) = v;
      AT(a, n, j, i) = v;
    }
}
static void FN(scale)(R* a, int64_t count, R s) {
  for (int64_t i = 0; i < count; ++i) a[i] *= s;
}

/* ------------------------------------------------------------------- gemm */

/* C (+)= alpha op(A) op(B); dl/blas.hpp:43-110.  A is (ta ? k x m : m x k),
 * B is (tb ? n x k : k x n), C is m x n.  Same four loop orders as the
 * reference so rounding matches. */
int FN(o_gemm)(int64_t m, int64_t n, int64_t k, R* c, const R* a, const R* b,
               int ta, int tb, R alpha, int accumulate) {
  if (m < 0 || n < 0 || k < 0) return DLA_ERR_SHAPE;
  if (c == a || c == b) return DLA_ERR_ALIAS;
  const int64_t lda = ta ? m : k, ldb = tb ? k : n;
  if (!accumulate)
    for (int64_t i = 0; i < m * n; ++i) c[i] = (R)0;
  if (!ta && !tb) {
    for (int64_t i = 0; i < m; ++i)
      for (int64_t p = 0; p < k; ++p) {
        const R av = alpha * AT(a, lda, i, p);
        for (int64_t j = 0; j < n; ++j) AT(c, n, i, j) += av * AT(b, ldb, p, j);
      }
  } else if (ta && !tb) {
    for (int64_t p = 0; p < k; ++p)
      for (int64_t i = 0; i < m; ++i) {
        const R av = alpha * AT(a, lda, p, i);
        for (int64_t j = 0; j < n; ++j) AT(c, n, i, j) += av * AT(b, ldb, p, j);
      }
  } else if (!ta && tb) {
    for (int64_t i = 0; i < m; ++i)
      for (int64_t j = 0; j < n; ++j) {
        R acc = (R)0;
        for (int64_t p = 0; p < k; ++p) acc += AT(a, lda, i, p) * AT(b, ldb, j, p);
        AT(c, n, i, j) += alpha * acc;
      }
  } else {
    for (int64_t i = 0; i < m; ++i)
      for (int64_t j = 0; j < n; ++j) {
        R acc = (R)0;
        for (int64_t p = 0; p < k; ++p) acc += AT(a, lda, p, i) * AT(b, ldb, j, p);
        AT(c, n, i, j) += alpha * acc;
      }
  }
  return DLA_OK;
}

/* dl/blas.hpp:119-122 */
int FN(o_gemm2)(int64_t m, int64_t n, int64_t k, R* c, const R* a, const R* b,
                int ta, int tb, R alpha) {
  return FN(o_gemm)(m, n, k, c, a, b, ta, tb, alpha, 0);
}

/* syrk: B = alpha A A^T (ta=0, A n x k) or alpha A^T A (ta=1, A k x n);
 * lower triangle computed, then mirrored (bit-exact symmetry);
 * dl/blas.hpp:138-169. */
int FN(o_syrk)(int64_t n, int64_t k, R* bo, const R* a, int ta, R alpha) {
  if (bo == a) return DLA_ERR_ALIAS;
  for (int64_t i = 0; i < n * n; ++i) bo[i] = (R)0;
  if (!ta) {
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j <= i; ++j) {
        R acc = (R)0;
        for (int64_t p = 0; p < k; ++p) acc += AT(a, k, i, p) * AT(a, k, j, p);
        AT(bo, n, i, j) = alpha * acc;
      }
  } else {
    for (int64_t p = 0; p < k; ++p)
      for (int64_t i = 0; i < n; ++i) {
        const R av = alpha * AT(a, n, p, i);
        for (int64_t j = 0; j <= i; ++j) AT(bo, n, i, j) += av * AT(a, n, p, j);
      }
  }
  FN(o_copyltu)(n, bo);
  return DLA_OK;
}

/* ------------------------------------------------------------- trmm / trsm */

/* Effective element of op(T) restricted to the `lower`-selected triangle. */
static R FN(tri_at)(const R* t, int64_t ld, int64_t i, int64_t j, int transpose, int lower) {
  int64_t r = transpose ? j : i, c = transpose ? i : j;
  if (lower ? (c > r) : (c < r)) return (R)0;
  return AT(t, ld, r, c);
}

/* X <- alpha op(T) X (left) or alpha X op(T) (right); dl/blas.hpp:202-291.
 * X is m x n; T is m x m (left) or n x n (right). */
int FN(o_trmm)(int64_t m, int64_t n, const R* t, R* x, int rightside, int transpose,
               int lower, R alpha) {
  if (x == t) return DLA_ERR_ALIAS;
  if (!rightside) {
    /* effective lower => rows bottom-up keep the untouched rows above intact */
    const int eff_lower = (lower != transpose);
    for (int64_t s = 0; s < m; ++s) {
      const int64_t i = eff_lower ? m - 1 - s : s;
      const R dii = AT(t, m, i, i);
      for (int64_t j = 0; j < n; ++j) AT(x, n, i, j) *= dii;
      const int64_t p0 = eff_lower ? 0 : i + 1, p1 = eff_lower ? i : m;
      for (int64_t p = p0; p < p1; ++p) {
        const R tv = FN(tri_at)(t, m, i, p, transpose, lower);
        if (tv == (R)0) continue;
        for (int64_t j = 0; j < n; ++j) AT(x, n, i, j) += tv * AT(x, n, p, j);
      }
      if (alpha != (R)1)
        for (int64_t j = 0; j < n; ++j) AT(x, n, i, j) *= alpha;
    }
    return DLA_OK;
  }
  for (int64_t r = 0; r < m; ++r) {
    R* xr = x + r * n;
    if (lower && !transpose) {
      for (int64_t k = 0; k < n; ++k) {
        const R v = xr[k];
        for (int64_t j = 0; j < k; ++j) xr[j] += v * AT(t, n, k, j);
        xr[k] = v * AT(t, n, k, k);
      }
    } else if (lower && transpose) {
      for (int64_t j = n - 1; j >= 0; --j) {
        R acc = (R)0;
        for (int64_t k = 0; k <= j; ++k) acc += xr[k] * AT(t, n, j, k);
        xr[j] = acc;
      }
    } else if (!lower && !transpose) {
      for (int64_t k = n - 1; k >= 0; --k) {
        const R v = xr[k];
        for (int64_t j = k + 1; j < n; ++j) xr[j] += v * AT(t, n, k, j);
        xr[k] = v * AT(t, n, k, k);
      }
    } else {
      for (int64_t j = 0; j < n; ++j) {
        R acc = (R)0;
        for (int64_t k = j; k < n; ++k) acc += xr[k] * AT(t, n, j, k);
        xr[j] = acc;
      }
    }
    if (alpha != (R)1)
      for (int64_t j = 0; j < n; ++j) xr[j] *= alpha;
  }
  return DLA_OK;
}

/* Solve op(T) Y = alpha X (left) or Y op(T) = alpha X (right), Y over X;
 * dl/blas.hpp:307-395.  Exact zero diagonal => SINGULAR(k), checked over the
 * whole diagonal before any write. */
int FN(o_trsm)(int64_t m, int64_t n, const R* t, R* x, int rightside, int transpose,
               int lower, R alpha, int64_t* idx) {
  if (x == t) return DLA_ERR_ALIAS;
  const int64_t nt = rightside ? n : m;
  for (int64_t k = 0; k < nt; ++k)
    if (AT(t, nt, k, k) == (R)0) {
      if (idx) *idx = k;
      return DLA_ERR_SINGULAR;
    }
  if (alpha != (R)1) FN(scale)(x, m * n, alpha);
  if (!rightside) {
    const int forward = (lower != transpose);
    for (int64_t s = 0; s < m; ++s) {
      const int64_t i = forward ? s : m - 1 - s;
      const int64_t p0 = forward ? 0 : i + 1, p1 = forward ? i : m;
      for (int64_t p = p0; p < p1; ++p) {
        const R tv = FN(tri_at)(t, m, i, p, transpose, lower);
        if (tv == (R)0) continue;
        for (int64_t j = 0; j < n; ++j) AT(x, n, i, j) -= tv * AT(x, n, p, j);
      }
      const R inv = (R)1 / AT(t, m, i, i);
      for (int64_t j = 0; j < n; ++j) AT(x, n, i, j) *= inv;
    }
    return DLA_OK;
  }
  for (int64_t r = 0; r < m; ++r) {
    R* xr = x + r * n;
    if (lower && !transpose) {
      for (int64_t k = n - 1; k >= 0; --k) {
        const R yk = xr[k] / AT(t, n, k, k);
        xr[k] = yk;
        for (int64_t j = 0; j < k; ++j) xr[j] -= yk * AT(t, n, k, j);
      }
    } else if (lower && transpose) {
      for (int64_t j = 0; j < n; ++j) {
        R acc = xr[j];
        for (int64_t k = 0; k < j; ++k) acc -= xr[k] * AT(t, n, j, k);
        xr[j] = acc / AT(t, n, j, j);
      }
    } else if (!lower && !transpose) {
      for (int64_t k = 0; k < n; ++k) {
        const R yk = xr[k] / AT(t, n, k, k);
        xr[k] = yk;
        for (int64_t j = k + 1; j < n; ++j) xr[j] -= yk * AT(t, n, k, j);
      }
    } else {
      for (int64_t j = n - 1; j >= 0; --j) {
        R acc = xr[j];
        for (int64_t k = j + 1; k < n; ++k) acc -= xr[k] * AT(t, n, j, k);
        xr[j] = acc / AT(t, n, j, j);
      }
    }
  }
  return DLA_OK;
}

/* --------------------------------------------------------- potrf / potri */

static R FN(sym_rtol)(void) { return sizeof(R) == 8 ? (R)1e-10 : (R)1e-4; }

/* dl/cholesky.hpp:35-72: nb = 64 panels, left-looking inside the panel,
 * right-looking lower trailing update; strict upper zeroed at the end. */
static int FN(potrf_lower)(int64_t n, R* a, int64_t* idx) {
  const int64_t nb = 64;
  for (int64_t k0 = 0; k0 < n; k0 += nb) {
    const int64_t k1 = k0 + nb < n ? k0 + nb : n;
    for (int64_t j = k0; j < k1; ++j) {
      for (int64_t i = j; i < n; ++i) {
        R acc = AT(a, n, i, j);
        for (int64_t p = k0; p < j; ++p) acc -= AT(a, n, i, p) * AT(a, n, j, p);
        AT(a, n, i, j) = acc;
      }
      const R d = AT(a, n, j, j);
      if (!(d > (R)0)) {
        if (idx) *idx = j;
        return DLA_ERR_NOT_SPD;
      }
      const R r = (R)SQRT(d);
      AT(a, n, j, j) = r;
      const R inv = (R)1 / r;
      for (int64_t i = j + 1; i < n; ++i) AT(a, n, i, j) *= inv;
    }
    for (int64_t i = k1; i < n; ++i)
      for (int64_t j = k1; j <= i; ++j) {
        R acc = (R)0;
        for (int64_t p = k0; p < k1; ++p) acc += AT(a, n, i, p) * AT(a, n, j, p);
        AT(a, n, i, j) -= acc;
      }
  }
  FN(o_tril)(n, a);
  return DLA_OK;
}

/* dl/cholesky.hpp:79-88 */
int FN(o_potrf)(int64_t n, R* a, int lower, int64_t* idx) {
  if (!FN(symmetric_ok)(n, a, FN(sym_rtol)())) return DLA_ERR_ASYMMETRIC;
  int st = FN(potrf_lower)(n, a, idx);
  if (st != DLA_OK) return st;
  if (!lower) FN(transpose_sq)(n, a);
  return DLA_OK;
}

/* dl/cholesky.hpp:105-147: trtri (column by column) + lauum + copyltu. */
int FN(o_potri)(int64_t n, R* a, int lower, int64_t* idx) {
  if (!lower) FN(transpose_sq)(n, a);
  for (int64_t j = 0; j < n; ++j) {
    if (AT(a, n, j, j) == (R)0) {
      if (idx) *idx = j;
      return DLA_ERR_SINGULAR;
    }
    AT(a, n, j, j) = (R)1 / AT(a, n, j, j);
    for (int64_t i = j + 1; i < n; ++i) {
      R acc = (R)0;
      for (int64_t k = j; k < i; ++k) acc += AT(a, n, i, k) * AT(a, n, k, j);
      AT(a, n, i, j) = -acc / AT(a, n, i, i);
    }
  }
  for (int64_t i = 0; i < n; ++i) {
    const R wii = AT(a, n, i, i);
    for (int64_t j = 0; j <= i; ++j) {
      R acc = wii * AT(a, n, i, j);
      for (int64_t k = i + 1; k < n; ++k) acc += AT(a, n, k, i) * AT(a, n, k, j);
      AT(a, n, i, j) = acc;
    }
  }
  FN(o_copyltu)(n, a);
  return DLA_OK;
}

/* ------------------------------------------------------------- sumlogdiag */

/* Tape chain ExtractDiag -> Log -> Sum (dl/tape.hpp:789-795, :714, :747-755):
 * sequential sum over i = 0..n-1. */
R FN(o_sumlogdiag)(int64_t n, const R* a) {
  R acc = (R)0;
  for (int64_t i = 0; i < n; ++i) acc += (R)LOG(AT(a, n, i, i));
  return acc;
}

/* Pullback (dl/tape.hpp:1038-1045, :969-975, :1080-1086): abar zero except
 * abar_ii = g / a_ii.  accumulate=1 adds onto the diagonal only. */
void FN(o_sumlogdiag_bwd)(int64_t n, R* abar, R g, const R* a, int accumulate) {
  if (!accumulate)
    for (int64_t i = 0; i < n * n; ++i) abar[i] = (R)0;
  for (int64_t i = 0; i < n; ++i) AT(abar, n, i, i) += g / AT(a, n, i, i);
}

/* ------------------------------------------------------------------ gelqf */

/* A (m x n, m <= n) = L Q; q: in A, out Q; l: out L (m x m).
 * dl/lq.hpp:24-106. */
int FN(o_gelqf)(int64_t m, int64_t n, R* q, R* l, R* tau, int64_t* idx) {
  if (m > n) return DLA_ERR_SHAPE;
  const R norm_a = FN(max_abs)(q, m * n);
  if (norm_a == (R)0) {
    if (idx) *idx = 0;
    return DLA_ERR_SINGULAR;
  }
  for (int64_t k = 0; k < m; ++k) {
    R* xk = q + k * n;
    R sigma = (R)0;
    for (int64_t j = k + 1; j < n; ++j) sigma += xk[j] * xk[j];
    const R alpha = xk[k];
    if (sigma == (R)0) {
      tau[k] = (R)0;
      continue;
    }
    const R nrm = (R)SQRT(alpha * alpha + sigma);
    const R beta = alpha >= (R)0 ? -nrm : nrm;
    tau[k] = (beta - alpha) / beta;
    const R sc = (R)1 / (alpha - beta);
    for (int64_t j = k + 1; j < n; ++j) xk[j] *= sc;
    xk[k] = beta;
    for (int64_t i = k + 1; i < m; ++i) {
      R* xi = q + i * n;
      R w = xi[k];
      for (int64_t j = k + 1; j < n; ++j) w += xi[j] * xk[j];
      w *= tau[k];
      xi[k] -= w;
      for (int64_t j = k + 1; j < n; ++j) xi[j] -= w * xk[j];
    }
  }
  const R rank_tol = (sizeof(R) == 8 ? (R)1e-12 : (R)1e-5) * norm_a;
  for (int64_t i = 0; i < m; ++i) {
    for (int64_t j = 0; j < m; ++j) AT(l, m, i, j) = j <= i ? AT(q, n, i, j) : (R)0;
    if (FN(absr)(AT(l, m, i, i)) < rank_tol) {
      if (idx) *idx = i;
      return DLA_ERR_SINGULAR;
    }
  }
  for (int64_t k = m - 1; k >= 0; --k) {
    const R* vk = q + k * n;
    const R tk = tau[k];
    for (int64_t i = k + 1; i < m; ++i) {
      R* xi = q + i * n;
      R w = xi[k];
      for (int64_t j = k + 1; j < n; ++j) w += xi[j] * vk[j];
      w *= tk;
      xi[k] -= w;
      for (int64_t j = k + 1; j < n; ++j) xi[j] -= w * vk[j];
    }
    R* xk = q + k * n;
    for (int64_t j = 0; j < k; ++j) xk[j] = (R)0;
    for (int64_t j = k + 1; j < n; ++j) xk[j] = -tk * xk[j];
    xk[k] = (R)1 - tk;
  }
  for (int64_t k = 0; k < m; ++k)
    if (AT(l, m, k, k) < (R)0) {
      for (int64_t i = k; i < m; ++i) AT(l, m, i, k) = -AT(l, m, i, k);
      for (int64_t j = 0; j < n; ++j) AT(q, n, k, j) = -AT(q, n, k, j);
    }
  return DLA_OK;
}

/* ------------------------------------------------------------------ syevd */

static R FN(pythag)(R a, R b) {  /* dl/common.hpp:109-119 */
  const R aa = FN(absr)(a), ab = FN(absr)(b);
  if (aa > ab) {
    const R r = ab / aa;
    return aa * (R)SQRT((R)1 + r * r);
  }
  if (ab == (R)0) return (R)0;
  const R r = aa / ab;
  return ab * (R)SQRT((R)1 + r * r);
}

static R FN(sign_like)(R a, R b) { return b >= (R)0 ? FN(absr)(a) : -FN(absr)(a); }

/* Householder tridiagonalization, reflectors kept (dl/eigen_sym.hpp:34-97). */
static void FN(tred1)(int64_t n, R* u, R* d, R* e, R* hout, R* v, R* y) {
  for (int64_t i = n - 1; i >= 1; --i) {
    const int64_t l = i - 1;
    R h = (R)0, scale = (R)0;
    if (l > 0) {
      for (int64_t k = 0; k <= l; ++k) scale += FN(absr)(AT(u, n, k, i));
      if (scale == (R)0) {
        e[i] = AT(u, n, l, i);
      } else {
        for (int64_t k = 0; k <= l; ++k) {
          AT(u, n, k, i) /= scale;
          v[k] = AT(u, n, k, i);
          h += v[k] * v[k];
        }
        R f = v[l];
        const R g = f >= (R)0 ? -(R)SQRT(h) : (R)SQRT(h);
        e[i] = scale * g;
        h -= f * g;
        AT(u, n, l, i) = f - g;
        v[l] = f - g;
        for (int64_t k = 0; k <= l; ++k) y[k] = (R)0;
        for (int64_t r = 0; r <= l; ++r) {
          const R vr = v[r];
          R acc = AT(u, n, r, r) * vr;
          for (int64_t c = r + 1; c <= l; ++c) {
            acc += AT(u, n, r, c) * v[c];
            y[c] += AT(u, n, r, c) * vr;
          }
          y[r] += acc;
        }
        f = (R)0;
        for (int64_t j = 0; j <= l; ++j) {
          AT(u, n, i, j) = v[j] / h;
          e[j] = y[j] / h;
          f += e[j] * v[j];
        }
        const R hh = f / (h + h);
        for (int64_t j = 0; j <= l; ++j) e[j] -= hh * v[j];
        for (int64_t r = 0; r <= l; ++r) {
          const R fr = v[r], gr = e[r];
          for (int64_t c = r; c <= l; ++c) AT(u, n, r, c) -= fr * e[c] + gr * v[c];
        }
      }
    } else {
      e[i] = AT(u, n, l, i);
    }
    hout[i] = h;
  }
  hout[0] = (R)0;
  e[0] = (R)0;
  for (int64_t i = 0; i < n; ++i) d[i] = AT(u, n, i, i);
  for (int64_t i = 0; i + 1 < n; ++i) e[i] = e[i + 1];
  e[n - 1] = (R)0;
}

static int FN(cmp)(const void* pa, const void* pb) {
  const R a = *(const R*)pa, b = *(const R*)pb;
  return a < b ? -1 : (a > b ? 1 : 0);
}

/* Implicit-shift QL, eigenvalues only, ascending (dl/eigen_sym.hpp:102-150). */
static int FN(tql1)(int64_t n, R* d, R* e, int64_t cap, int64_t* iters) {
  const R eps = EPS;
  int64_t total = 0;
  for (int64_t l = 0; l < n; ++l) {
    int64_t m;
    do {
      for (m = l; m < n - 1; ++m) {
        const R dd = FN(absr)(d[m]) + FN(absr)(d[m + 1]);
        if (FN(absr)(e[m]) <= eps * dd) break;
      }
      if (m != l) {
        if (++total > cap) {
          if (iters) *iters = total;
          return DLA_ERR_CONVERGENCE;
        }
        R g = (d[l + 1] - d[l]) / ((R)2 * e[l]);
        R r = FN(pythag)(g, (R)1);
        g = d[m] - d[l] + e[l] / (g + FN(sign_like)(r, g));
        R s = (R)1, c = (R)1, p = (R)0;
        int64_t i;
        for (i = m - 1; i >= l; --i) {
          R f = s * e[i];
          const R b = c * e[i];
          r = FN(pythag)(f, g);
          e[i + 1] = r;
          if (r == (R)0) {
            d[i + 1] -= p;
            e[m] = (R)0;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + (R)2 * c * b;
          p = s * r;
          d[i + 1] = g + p;
          g = c * r - b;
        }
        if (r == (R)0 && i >= l) continue;
        d[l] -= p;
        e[l] = g;
        e[m] = (R)0;
      }
    } while (m != l);
  }
  qsort(d, (size_t)n, sizeof(R), FN(cmp));
  return DLA_OK;
}

/* Deterministic start vector (dl/eigen_sym.hpp:155-162). */
static R FN(invit_seed)(int64_t salt, int64_t k) {
  uint64_t x = ((uint64_t)salt + 1) * 0x9E3779B97F4A7C15ull;
  x ^= ((uint64_t)k + 1) * 0xBF58476D1CE4E5B9ull;
  x ^= x >> 31;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 29;
  return (R)1 + (R)0.5 * (R)((double)(x >> 11) * 0x1.0p-53);
}

/* Inverse iteration on the tridiagonal (dl/eigen_sym.hpp:170-275). */
static void FN(tinvit)(int64_t n, const R* d, const R* e, const R* w, R* z, R* alp,
                       R* bet, R* gam, R* mul, R* swp) {
  R norm = FN(absr)(d[0]) + FN(absr)(e[0]);
  for (int64_t i = 1; i < n; ++i) {
    R t = FN(absr)(e[i - 1]) + FN(absr)(d[i]) + FN(absr)(e[i]);
    if (t > norm) norm = t;
  }
  if (norm == (R)0) {
    for (int64_t i = 0; i < n; ++i)
      for (int64_t k = 0; k < n; ++k) AT(z, n, i, k) = k == i ? (R)1 : (R)0;
    return;
  }
  const R eps = EPS;
  const R eps3 = eps * norm;
  const R gtol = (R)100 * (R)SQRT(eps) * norm;
  const R piv_min = RMIN / eps;
  int64_t gs = 0;
  R lam_used = (R)0;
  for (int64_t idx = 0; idx < n; ++idx) {
    if (idx > 0 && w[idx] - w[idx - 1] > gtol) gs = idx;
    R lam = w[idx];
    if (idx > gs && lam < lam_used + eps3) lam = lam_used + eps3;
    lam_used = lam;
    R* x = z + idx * n;
    for (int attempt = 0; attempt < 3; ++attempt) {
      R a = d[0] - lam;
      R b = n > 1 ? e[0] : (R)0;
      for (int64_t i = 0; i + 1 < n; ++i) {
        const R sub = e[i], dia = d[i + 1] - lam;
        const R sup = i + 2 < n ? e[i + 1] : (R)0;
        if (FN(absr)(sub) > FN(absr)(a)) {
          swp[i] = (R)1;
          bet[i] = dia;
          gam[i] = sup;
          const R mm = a / sub;
          mul[i] = mm;
          alp[i] = (R)1 / sub;
          a = b - mm * dia;
          b = -mm * sup;
        } else {
          swp[i] = (R)0;
          R piv = a;
          if (FN(absr)(piv) < piv_min) piv = eps3;
          bet[i] = b;
          gam[i] = (R)0;
          const R mm = sub / piv;
          mul[i] = mm;
          alp[i] = (R)1 / piv;
          a = dia - mm * b;
          b = sup;
        }
      }
      if (FN(absr)(a) < piv_min) a = eps3;
      alp[n - 1] = (R)1 / a;
      for (int64_t k = 0; k < n; ++k) x[k] = FN(invit_seed)(idx + 131 * attempt, k);
      for (int it = 0; it < 2; ++it) {
        if (it > 0)
          for (int64_t i = 0; i + 1 < n; ++i) {
            if (swp[i] != (R)0) {
              R t = x[i];
              x[i] = x[i + 1];
              x[i + 1] = t;
            }
            x[i + 1] -= mul[i] * x[i];
          }
        x[n - 1] *= alp[n - 1];
        if (n >= 2) x[n - 2] = (x[n - 2] - bet[n - 2] * x[n - 1]) * alp[n - 2];
        for (int64_t i = n - 3; i >= 0; --i)
          x[i] = (x[i] - bet[i] * x[i + 1] - gam[i] * x[i + 2]) * alp[i];
        R amax = (R)0;
        for (int64_t k = 0; k < n; ++k)
          if (FN(absr)(x[k]) > amax) amax = FN(absr)(x[k]);
        const R inv = (R)1 / amax;
        for (int64_t k = 0; k < n; ++k) x[k] *= inv;
      }
      R nrm = (R)0;
      for (int64_t k = 0; k < n; ++k) nrm += x[k] * x[k];
      nrm = (R)SQRT(nrm);
      for (int64_t k = 0; k < n; ++k) x[k] /= nrm;
      R drop = (R)1;
      for (int pass = 0; pass < 2 && idx > gs; ++pass) {
        for (int64_t j = gs; j < idx; ++j) {
          const R* zj = z + j * n;
          R dot = (R)0;
          for (int64_t k = 0; k < n; ++k) dot += x[k] * zj[k];
          for (int64_t k = 0; k < n; ++k) x[k] -= dot * zj[k];
        }
        R s = (R)0;
        for (int64_t k = 0; k < n; ++k) s += x[k] * x[k];
        s = (R)SQRT(s);
        if (pass == 0) drop = s;
        if (s > (R)0)
          for (int64_t k = 0; k < n; ++k) x[k] /= s;
      }
      if (drop >= (R)0.01) break;
    }
  }
}

/* Reflector back-transform onto the rows of z (dl/eigen_sym.hpp:282-310). */
static void FN(trbak)(int64_t n, const R* refl, const R* h, R* z, R* v) {
  for (int64_t i = 1; i < n; ++i) {
    if (h[i] == (R)0) continue;
    for (int64_t k = 0; k < i; ++k) v[k] = AT(refl, n, k, i);
    const R* vh = refl + i * n;
    for (int64_t j = 0; j < n; ++j) {
      R* zj = z + j * n;
      R g = (R)0;
      for (int64_t k = 0; k < i; ++k) g += v[k] * zj[k];
      for (int64_t k = 0; k < i; ++k) zj[k] -= g * vh[k];
    }
  }
}

/* Sign rule (dl/eigen_sym.hpp:316-333): flip row i when its largest-|.| entry
 * (first index on ties, strict >) is negative. */
void FN(o_fix_row_signs)(int64_t rows, int64_t cols, R* u) {
  for (int64_t i = 0; i < rows; ++i) {
    R* row = u + i * cols;
    int64_t kmax = 0;
    R best = FN(absr)(row[0]);
    for (int64_t k = 1; k < cols; ++k)
      if (FN(absr)(row[k]) > best) {
        best = FN(absr)(row[k]);
        kmax = k;
      }
    if (row[kmax] < (R)0)
      for (int64_t k = 0; k < cols; ++k) row[k] = -row[k];
  }
}

/* A = U^T diag(lambda) U, rows of U eigenvectors, lambda ascending.
 * dl/eigen_sym.hpp:339-367.  ws: n*n + 9n reals. */
int FN(o_syevd)(int64_t n, R* u, R* lambda, R* ws, int64_t* idx) {
  if (!FN(symmetric_ok)(n, u, FN(sym_rtol)())) return DLA_ERR_ASYMMETRIC;
  if (n == 1) {
    lambda[0] = u[0];
    u[0] = (R)1;
    return DLA_OK;
  }
  if (n == 0) return DLA_OK;
  R* refl = ws;
  R* d = refl + n * n;
  R* e = d + n;
  R* h = e + n;
  R* v = h + n;
  R* y = v + n;
  R* alp = y + n;
  R* bet = alp + n;
  R* gam = bet + n;
  R* mul = gam + n;
  FN(tred1)(n, u, d, e, h, v, y);
  memcpy(refl, u, sizeof(R) * (size_t)(n * n));
  memcpy(lambda, d, sizeof(R) * (size_t)n);
  memcpy(v, e, sizeof(R) * (size_t)n);
  int st = FN(tql1)(n, lambda, v, 30 * n, idx);
  if (st != DLA_OK) return st;
  FN(tinvit)(n, d, e, lambda, u, alp, bet, gam, mul, y);
  FN(trbak)(n, refl, h, u, v);
  FN(o_fix_row_signs)(n, n, u);
  return DLA_OK;
}

/* --------------------------------------------------------------- backward */

/* dl/adjoints.hpp:36-49 */
int FN(o_gemm2_bwd)(int64_t m, int64_t n, int64_t k, R* abar, R* bbar, const R* cbar,
                    const R* a, const R* b, int ta, int tb, R alpha) {
  /* A is (ta ? k x m : m x k), B is (tb ? n x k : k x n), C m x n */
  int st;
  if (!ta) st = FN(o_gemm)(m, k, n, abar, cbar, b, 0, !tb, alpha, 0);
  else st = FN(o_gemm)(k, m, n, abar, b, cbar, tb, 1, alpha, 0);
  if (st) return st;
  if (!tb) st = FN(o_gemm)(k, n, m, bbar, a, cbar, !ta, 0, alpha, 0);
  else st = FN(o_gemm)(n, k, m, bbar, cbar, a, 1, ta, alpha, 0);
  return st;
}

/* dl/adjoints.hpp:69-78 */
int FN(o_syrk_bwd)(int64_t n, int64_t k, R* abar, const R* bbar, const R* a, int ta, R alpha) {
  if (!ta) {  /* A n x k: abar = alpha (Bbar + Bbar^T) A */
    FN(o_gemm)(n, k, n, abar, bbar, a, 0, 0, alpha, 0);
    FN(o_gemm)(n, k, n, abar, bbar, a, 1, 0, alpha, 1);
  } else {    /* A k x n: abar = alpha A (Bbar + Bbar^T) */
    FN(o_gemm)(k, n, n, abar, a, bbar, 0, 0, alpha, 0);
    FN(o_gemm)(k, n, n, abar, a, bbar, 0, 1, alpha, 1);
  }
  return DLA_OK;
}

static void FN(mask)(int64_t n, R* x, int lower) {
  if (lower) FN(o_tril)(n, x);
  else FN(o_triu)(n, x);
}

/* dl/adjoints.hpp:94-110.  X/A/Bbar are m x n; T is mt x mt. */
int FN(o_trmm_bwd)(int64_t m, int64_t n, R* abar, R* tbar, const R* bbar, const R* t,
                   const R* a, int rightside, int transpose, int lower, R alpha) {
  const int64_t mt = rightside ? n : m;
  if (!rightside && !transpose) FN(o_gemm)(m, m, n, tbar, bbar, a, 0, 1, alpha, 0);
  else if (!rightside && transpose) FN(o_gemm)(m, m, n, tbar, a, bbar, 0, 1, alpha, 0);
  else if (rightside && !transpose) FN(o_gemm)(n, n, m, tbar, a, bbar, 1, 0, alpha, 0);
  else FN(o_gemm)(n, n, m, tbar, bbar, a, 1, 0, alpha, 0);
  FN(mask)(mt, tbar, lower);
  if (abar != bbar) memcpy(abar, bbar, sizeof(R) * (size_t)(m * n));
  return FN(o_trmm)(m, n, t, abar, rightside, !transpose, lower, alpha);
}

/* dl/adjoints.hpp:131-153.  b is the forward OUTPUT. */
int FN(o_trsm_bwd)(int64_t m, int64_t n, R* abar, R* tbar, const R* bbar, const R* t,
                   const R* b, int rightside, int transpose, int lower, R alpha,
                   int64_t* idx) {
  const int64_t mt = rightside ? n : m;
  if (abar != bbar) memcpy(abar, bbar, sizeof(R) * (size_t)(m * n));
  int st = FN(o_trsm)(m, n, t, abar, rightside, !transpose, lower, (R)1, idx);
  if (st) return st;
  if (!rightside) {
    if (!transpose) FN(o_gemm)(m, m, n, tbar, abar, b, 0, 1, (R)-1, 0);
    else FN(o_gemm)(m, m, n, tbar, b, abar, 0, 1, (R)-1, 0);
  } else {
    if (!transpose) FN(o_gemm)(n, n, m, tbar, b, abar, 1, 0, (R)-1, 0);
    else FN(o_gemm)(n, n, m, tbar, abar, b, 1, 0, (R)-1, 0);
  }
  FN(mask)(mt, tbar, lower);
  if (alpha != (R)1) FN(scale)(abar, m * n, alpha);
  return DLA_OK;
}

/* dl/adjoints.hpp:175-191; abar may alias lbar. */
int FN(o_potrf_bwd)(int64_t n, R* abar, const R* lbar, const R* l, int lower) {
  if (abar != lbar) memcpy(abar, lbar, sizeof(R) * (size_t)(n * n));
  if (lower) {
    FN(o_trmm)(n, n, l, abar, 0, 1, 1, (R)1);
    FN(o_copyltu)(n, abar);
    FN(o_trsm)(n, n, l, abar, 0, 1, 1, (R)1, NULL);
    FN(o_trsm)(n, n, l, abar, 1, 0, 1, (R)1, NULL);
  } else {
    FN(o_trmm)(n, n, l, abar, 1, 1, 0, (R)1);
    FN(o_copyutl)(n, abar);
    FN(o_trsm)(n, n, l, abar, 0, 0, 0, (R)1, NULL);
    FN(o_trsm)(n, n, l, abar, 1, 1, 0, (R)1, NULL);
  }
  FN(scale)(abar, n * n, (R)0.5);
  FN(o_sym)(n, abar);
  return DLA_OK;
}

/* dl/adjoints.hpp:207-223 */
int FN(o_potri_bwd)(int64_t n, R* lbar, const R* bbar, const R* l, const R* b, int lower) {
  if (lower) {
    FN(o_gemm)(n, n, n, lbar, b, bbar, 0, 0, (R)1, 0);
    FN(o_gemm)(n, n, n, lbar, b, bbar, 0, 1, (R)1, 1);
    FN(o_trsm)(n, n, l, lbar, 1, 1, 1, (R)1, NULL);
    FN(scale)(lbar, n * n, (R)-1);
    FN(o_tril)(n, lbar);
  } else {
    FN(o_gemm)(n, n, n, lbar, bbar, b, 0, 0, (R)1, 0);
    FN(o_gemm)(n, n, n, lbar, bbar, b, 1, 0, (R)1, 1);
    FN(o_trsm)(n, n, l, lbar, 0, 1, 0, (R)1, NULL);
    FN(scale)(lbar, n * n, (R)-1);
    FN(o_triu)(n, lbar);
  }
  return DLA_OK;
}

/* dl/adjoints.hpp:239-252; work: m*m reals. */
int FN(o_gelqf_bwd)(int64_t m, int64_t n, R* abar, const R* qbar, const R* lbar,
                    const R* q, const R* l, R* work) {
  memcpy(work, lbar, sizeof(R) * (size_t)(m * m));
  FN(o_trmm)(m, m, l, work, 0, 1, 1, (R)1);
  FN(o_gemm)(m, m, n, work, qbar, q, 0, 1, (R)-1, 1);
  FN(o_copyltu)(m, work);
  if (abar != qbar) memcpy(abar, qbar, sizeof(R) * (size_t)(m * n));
  FN(o_gemm)(m, n, m, abar, work, q, 0, 0, (R)1, 1);
  return FN(o_trsm)(m, n, l, abar, 0, 1, 1, (R)1, NULL);
}

/* dl/adjoints.hpp:272-295; work: n*n reals. */
int FN(o_syevd_bwd)(int64_t n, R* abar, const R* ubar, const R* lambdabar, const R* u,
                    const R* lambda, R eps_gap, R* work) {
  FN(o_gemm)(n, n, n, work, ubar, u, 0, 1, (R)1, 0);
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t j = 0; j < i; ++j) {
      R gap = lambda[i] - lambda[j];
      if (gap < eps_gap) gap = eps_gap;
      const R yv = (AT(work, n, i, j) - AT(work, n, j, i)) / ((R)2 * gap);
      AT(work, n, i, j) = yv;
      AT(work, n, j, i) = yv;
    }
    AT(work, n, i, i) = lambdabar[i];
  }
  FN(o_gemm)(n, n, n, abar, u, work, 1, 0, (R)1, 0);
  FN(o_gemm)(n, n, n, work, abar, u, 0, 0, (R)1, 0);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j <= i; ++j) {
      const R yv = (AT(work, n, i, j) + AT(work, n, j, i)) / (R)2;
      AT(abar, n, i, j) = yv;
      AT(abar, n, j, i) = yv;
    }
  return DLA_OK;
}

/* ------------------------------------------------------------------ gesvd */

/* Golub-Kahan-Reinsch on a (rows M >= cols N), dl/svd.hpp:26-223: a becomes
 * the economy left factor, w the singular values, v (N x N) the right factor.
 * rv1: N reals.  Returns DLA_ERR_CONVERGENCE (*idx = total iterations) after
 * 30 sweeps on one singular value. */
static int FN(svd_gkr)(int64_t m, int64_t n, R* a, R* w, R* v, R* rv1, int64_t* idx) {
  const R eps = (R)EPS;
  R g = 0, scale = 0, anorm = 0, s, f, h, c, x, y, z;
  int64_t l = 0, nm = 0;
#define A_(i, j) AT(a, n, i, j)
#define V_(i, j) AT(v, n, i, j)
  for (int64_t i = 0; i < n; ++i) {
    l = i + 1;
    rv1[i] = scale * g;
    g = scale = 0;
    if (i < m) {
      for (int64_t k = i; k < m; ++k) scale += FN(absr)(A_(k, i));
      if (scale != (R)0) {
        s = 0;
        for (int64_t k = i; k < m; ++k) {
          A_(k, i) /= scale;
          s += A_(k, i) * A_(k, i);
        }
        f = A_(i, i);
        g = -FN(sign_like)((R)SQRT(s), f);
        h = f * g - s;
        A_(i, i) = f - g;
        for (int64_t j = l; j < n; ++j) {
          s = 0;
          for (int64_t k = i; k < m; ++k) s += A_(k, i) * A_(k, j);
          f = s / h;
          for (int64_t k = i; k < m; ++k) A_(k, j) += f * A_(k, i);
        }
        for (int64_t k = i; k < m; ++k) A_(k, i) *= scale;
      }
    }
    w[i] = scale * g;
    g = scale = 0;
    if (i < m && i != n - 1) {
      for (int64_t k = l; k < n; ++k) scale += FN(absr)(A_(i, k));
      if (scale != (R)0) {
        s = 0;
        for (int64_t k = l; k < n; ++k) {
          A_(i, k) /= scale;
          s += A_(i, k) * A_(i, k);
        }
        f = A_(i, l);
        g = -FN(sign_like)((R)SQRT(s), f);
        h = f * g - s;
        A_(i, l) = f - g;
        for (int64_t k = l; k < n; ++k) rv1[k] = A_(i, k) / h;
        for (int64_t j = l; j < m; ++j) {
          s = 0;
          for (int64_t k = l; k < n; ++k) s += A_(j, k) * A_(i, k);
          for (int64_t k = l; k < n; ++k) A_(j, k) += s * rv1[k];
        }
        for (int64_t k = l; k < n; ++k) A_(i, k) *= scale;
      }
    }
    {
      const R t = FN(absr)(w[i]) + FN(absr)(rv1[i]);
      if (t > anorm) anorm = t;
    }
  }
  for (int64_t i = n - 1; i >= 0; --i) {
    if (i < n - 1) {
      if (g != (R)0) {
        for (int64_t j = l; j < n; ++j) V_(j, i) = (A_(i, j) / A_(i, l)) / g;
        for (int64_t j = l; j < n; ++j) {
          s = 0;
          for (int64_t k = l; k < n; ++k) s += A_(i, k) * V_(k, j);
          for (int64_t k = l; k < n; ++k) V_(k, j) += s * V_(k, i);
        }
      }
      for (int64_t j = l; j < n; ++j) V_(i, j) = V_(j, i) = 0;
    }
    V_(i, i) = 1;
    g = rv1[i];
    l = i;
  }
  for (int64_t i = (m < n ? m : n) - 1; i >= 0; --i) {
    l = i + 1;
    g = w[i];
    for (int64_t j = l; j < n; ++j) A_(i, j) = 0;
    if (g != (R)0) {
      g = (R)1 / g;
      for (int64_t j = l; j < n; ++j) {
        s = 0;
        for (int64_t k = l; k < m; ++k) s += A_(k, i) * A_(k, j);
        f = (s / A_(i, i)) * g;
        for (int64_t k = i; k < m; ++k) A_(k, j) += f * A_(k, i);
      }
      for (int64_t j = i; j < m; ++j) A_(j, i) *= g;
    } else {
      for (int64_t j = i; j < m; ++j) A_(j, i) = 0;
    }
    A_(i, i) += (R)1;
  }
  int64_t total_iter = 0;
  for (int64_t k = n - 1; k >= 0; --k) {
    for (int64_t its = 1;; ++its) {
      int flag = 1;
      for (l = k; l >= 0; --l) {
        nm = l - 1;
        if (FN(absr)(rv1[l]) <= eps * anorm) {
          flag = 0;
          break;
        }
        if (FN(absr)(w[nm]) <= eps * anorm) break;
      }
      if (flag) {
        c = 0;
        s = 1;
        for (int64_t i = l; i <= k; ++i) {
          f = s * rv1[i];
          rv1[i] = c * rv1[i];
          if (FN(absr)(f) <= eps * anorm) break;
          g = w[i];
          h = FN(pythag)(f, g);
          w[i] = h;
          h = (R)1 / h;
          c = g * h;
          s = -f * h;
          for (int64_t j = 0; j < m; ++j) {
            y = A_(j, nm);
            z = A_(j, i);
            A_(j, nm) = y * c + z * s;
            A_(j, i) = z * c - y * s;
          }
        }
      }
      z = w[k];
      if (l == k) {
        if (z < (R)0) {
          w[k] = -z;
          for (int64_t j = 0; j < n; ++j) V_(j, k) = -V_(j, k);
        }
        break;
      }
      if (its == 30) {
        if (idx) *idx = total_iter;
        return DLA_ERR_CONVERGENCE;
      }
      ++total_iter;
      x = w[l];
      nm = k - 1;
      y = w[nm];
      g = rv1[nm];
      h = rv1[k];
      f = ((y - z) * (y + z) + (g - h) * (g + h)) / ((R)2 * h * y);
      g = FN(pythag)(f, (R)1);
      f = ((x - z) * (x + z) + h * ((y / (f + FN(sign_like)(g, f))) - h)) / x;
      c = s = 1;
      for (int64_t j = l; j <= nm; ++j) {
        const int64_t i = j + 1;
        g = rv1[i];
        y = w[i];
        h = s * g;
        g = c * g;
        z = FN(pythag)(f, h);
        rv1[j] = z;
        c = f / z;
        s = h / z;
        f = x * c + g * s;
        g = g * c - x * s;
        h = y * s;
        y *= c;
        for (int64_t jj = 0; jj < n; ++jj) {
          x = V_(jj, j);
          z = V_(jj, i);
          V_(jj, j) = x * c + z * s;
          V_(jj, i) = z * c - x * s;
        }
        z = FN(pythag)(f, h);
        w[j] = z;
        if (z != (R)0) {
          z = (R)1 / z;
          c = f * z;
          s = h * z;
        }
        f = c * g + s * y;
        x = c * y - s * g;
        for (int64_t jj = 0; jj < m; ++jj) {
          y = A_(jj, j);
          z = A_(jj, i);
          A_(jj, j) = y * c + z * s;
          A_(jj, i) = z * c - y * s;
        }
      }
      rv1[l] = 0;
      rv1[k] = f;
      w[k] = x;
    }
  }
#undef A_
#undef V_
  return DLA_OK;
}

/* v: in A (m x n, m <= n), out V; u: out U (m x m); lambda ascending (stable
 * sort), sign rule on U's rows mirrored onto V (dl/svd.hpp:229-284).
 * ws: n*m + m*m + m*m + m*n + 2m reals. */
int FN(o_gesvd)(int64_t m, int64_t n, R* v, R* u, R* lambda, R* ws, int64_t* idx) {
  if (m > n) return DLA_ERR_SHAPE;
  if (m == 0) return DLA_OK;
  R* wt = ws;             /* n x m */
  R* vs = wt + n * m;     /* m x m */
  R* ut = vs + m * m;     /* m x m */
  R* vt = ut + m * m;     /* m x n */
  R* rv1 = vt + m * n;    /* m */
  R* lt = rv1 + m;        /* m */
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) AT(wt, m, j, i) = AT(v, n, i, j);
  int st = FN(svd_gkr)(n, m, wt, lambda, vs, rv1, idx);
  if (st != DLA_OK) return st;
  for (int64_t i = 0; i < m; ++i)
    for (int64_t k = 0; k < m; ++k) AT(u, m, i, k) = AT(vs, m, k, i);
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) AT(v, n, i, j) = AT(wt, m, j, i);
  /* stable ascending sort: insertion sort of the permutation (ties keep order) */
  int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)m);
  for (int64_t i = 0; i < m; ++i) perm[i] = i;
  for (int64_t i = 1; i < m; ++i) {
    const int64_t p = perm[i];
    int64_t j = i - 1;
    while (j >= 0 && lambda[p] < lambda[perm[j]]) {
      perm[j + 1] = perm[j];
      --j;
    }
    perm[j + 1] = p;
  }
  for (int64_t i = 0; i < m; ++i) {
    const int64_t sidx = perm[i];
    lt[i] = lambda[sidx];
    memcpy(ut + i * m, u + sidx * m, sizeof(R) * (size_t)m);
    memcpy(vt + i * n, v + sidx * n, sizeof(R) * (size_t)n);
  }
  free(perm);
  memcpy(lambda, lt, sizeof(R) * (size_t)m);
  memcpy(u, ut, sizeof(R) * (size_t)(m * m));
  memcpy(v, vt, sizeof(R) * (size_t)(m * n));
  /* sign rule on U, V's row flipped in lockstep */
  for (int64_t i = 0; i < m; ++i) {
    R* row = u + i * m;
    int64_t kmax = 0;
    R best = FN(absr)(row[0]);
    for (int64_t k = 1; k < m; ++k)
      if (FN(absr)(row[k]) > best) {
        best = FN(absr)(row[k]);
        kmax = k;
      }
    if (row[kmax] < (R)0) {
      for (int64_t k = 0; k < m; ++k) row[k] = -row[k];
      for (int64_t j = 0; j < n; ++j) AT(v, n, i, j) = -AT(v, n, i, j);
    }
  }
  return DLA_OK;
}

/* dl/adjoints.hpp:315-382; work: m*m + m + m*n reals.  SINGULAR(i) when a
 * singular value is not above eps_gap. */
int FN(o_gesvd_bwd)(int64_t m, int64_t n, R* abar, const R* ubar, const R* lambdabar, const R* vbar,
                    const R* u, const R* lambda, const R* v, R eps_gap, R* work, int64_t* idx) {
  for (int64_t i = 0; i < m; ++i)
    if (!(lambda[i] > eps_gap)) {
      if (idx) *idx = i;
      return DLA_ERR_SINGULAR;
    }
  R* w = work;
  R* dvec = w + m * m;
  R* tmp = dvec + m;
  for (int64_t i = 0; i < m; ++i) {
    const R inv = (R)1 / lambda[i];
    for (int64_t j = 0; j < n; ++j) AT(abar, n, i, j) = inv * AT(vbar, n, i, j);
  }
  FN(o_gemm)(m, m, n, w, abar, v, 0, 1, (R)1, 0);
  for (int64_t i = 0; i < m; ++i) dvec[i] = AT(w, m, i, i);
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < m; ++j) AT(w, m, i, j) *= lambda[j];
  FN(o_gemm)(m, m, m, w, ubar, u, 0, 1, (R)1, 1);
  for (int64_t i = 0; i < m; ++i) {
    for (int64_t j = 0; j < i; ++j) {
      R hd = lambda[i] - lambda[j], hs = lambda[i] + lambda[j];
      if (hd < eps_gap) hd = eps_gap;
      if (hs < eps_gap) hs = eps_gap;
      const R yv = (AT(w, m, i, j) - AT(w, m, j, i)) / (hd * hs);
      AT(w, m, i, j) = yv * lambda[j];
      AT(w, m, j, i) = yv * lambda[i];
    }
    AT(w, m, i, i) = lambdabar[i] - dvec[i];
  }
  FN(o_gemm)(m, n, m, abar, w, v, 0, 0, (R)1, 1);
  memcpy(tmp, abar, sizeof(R) * (size_t)(m * n));
  FN(o_gemm)(m, n, m, abar, u, tmp, 1, 0, (R)1, 0);
  return DLA_OK;
}


/* ------------------------------------------------------------------------
 * Batched Kalman filter NLL: the reference's
 * build_kalman_nll graph (dl/models.hpp:285-337, Joseph-form covariance
 * update) evaluated forward, and its reverse-mode gradient w.r.t. every leaf
 * (A, B, S_h, S_v, mu0, S0, the observations) written out op by op — the
 * pullbacks the tape applies (dl/tape.hpp:841-917: gemm2, potrf, trsm; the
 * elementwise add / sub / square / log / sum chain, :930-1086).
 *
 * Per step t (mu, S = predicted state; v = obs[t]):
 *   M1 = B S;  Svv = M1 B^T + Sv;  L = chol(Svv);  e = v - B mu;  z = L^-1 e
 *   phi_t = 1/2 z^T z + sum log L_ii + d/2 log 2 pi
 *   X = S B^T;  Y = X L^-T;  K = Y L^-1;  mu_f = mu + K e;  I_KB = I - K B
 *   P1 = I_KB S;  S_f = P1 I_KB^T + (K Sv) K^T
 *   (t < T-1)  mu' = A mu_f;  S' = (A S_f) A^T + Sh
 * nll = sum_t phi_t.  Layout: a h x h, b d x h, sh h x h, sv d x d, mu0 h,
 * s0 h x h, obs T x d (row t = observation t); gradients in the same shapes.
 * The tape (intermediates of every step) is malloc'ed here. */
int FN(o_kalman)(int64_t h, int64_t d, int64_t T, const R* a, const R* b, const R* sh, const R* sv,
                 const R* mu0, const R* s0, const R* obs, R* nll, R* abar, R* bbar, R* shbar, R* svbar,
                 R* mu0bar, R* s0bar, R* obsbar, int64_t* idx) {
  if (h < 1 || d < 1 || T < 1) return DLA_ERR_SHAPE;
  const int64_t hh = h * h, hd = h * d, dd = d * d;
  /* tape per step: S mu M1 L e z X Y K IKB P1 Q1 Sf muf */
  const int64_t step = hh + h + hd + dd + d + d + hd + hd + hd + hh + hh + hd + hh + h;
  R* tape = (R*)calloc((size_t)(step * T), sizeof(R));
  R* w = (R*)calloc((size_t)(16 * (hh + hd + dd + h + d) + 64), sizeof(R));
  if (!tape || !w) {
    free(tape);
    free(w);
    return DLA_ERR_INVALID;
  }
#define TP(t, off) (tape + (t) * step + (off))
  const int64_t oS = 0, oMu = oS + hh, oM1 = oMu + h, oL = oM1 + hd, oE = oL + dd, oZ = oE + d, oX = oZ + d,
                oY = oX + hd, oK = oY + hd, oI = oK + hd, oP1 = oI + hh, oQ1 = oP1 + hh, oSf = oQ1 + hd,
                oMuf = oSf + hh;
  R* t1 = w;            /* h x h scratch */
  R* t2 = t1 + hh;      /* h x h */
  R* t3 = t2 + hh;      /* h x h */
  R* vd = t3 + hh;      /* d x d */
  R* vhd = vd + dd;     /* h x d */
  R* vhd2 = vhd + hd;   /* h x d */
  R* vh = vhd2 + hd;    /* h */
  R* vdv = vh + h;      /* d */
  R* sbar = vdv + d;    /* h x h: adjoint of S_pred (running) */
  R* mubar = sbar + hh; /* h */
  R* sbn = mubar + h;   /* h x h: adjoint of the next S_pred */
  R* mbn = sbn + hh;    /* h */
  R* lbar = mbn + h;    /* d x d */
  R* kbar = lbar + dd;  /* h x d */
  R* ybar = kbar + hd;  /* h x d */
  R* ebar = ybar + hd;  /* d */
  R* ibar = ebar + d;   /* h x h */
  R* p1bar = ibar + hh; /* h x h */
  R* m1bar = p1bar + hh; /* d x h */
  int st = DLA_OK;
  const R log2pi = (R)1.8378770664093454835606594728112353L;
  R total = (R)0;
  memcpy(TP(0, oS), s0, sizeof(R) * (size_t)hh);
  memcpy(TP(0, oMu), mu0, sizeof(R) * (size_t)h);
  for (int64_t t = 0; t < T && st == DLA_OK; ++t) {
    R *S = TP(t, oS), *mu = TP(t, oMu), *M1 = TP(t, oM1), *L = TP(t, oL), *e = TP(t, oE), *z = TP(t, oZ);
    R *X = TP(t, oX), *Y = TP(t, oY), *K = TP(t, oK), *I = TP(t, oI), *P1 = TP(t, oP1), *Q1 = TP(t, oQ1);
    R *Sf = TP(t, oSf), *muf = TP(t, oMuf);
    FN(o_gemm)(d, h, h, M1, b, S, 0, 0, (R)1, 0);
    FN(o_gemm)(d, d, h, L, M1, b, 0, 1, (R)1, 0);
    for (int64_t q = 0; q < dd; ++q) L[q] += sv[q];
    if (!FN(symmetric_ok)(d, L, FN(sym_rtol)())) {
      st = DLA_ERR_ASYMMETRIC;
      break;
    }
    st = FN(potrf_lower)(d, L, idx);
    if (st) break;
    FN(o_tril)(d, L);
    FN(o_gemm)(d, 1, h, vdv, b, mu, 0, 0, (R)1, 0);
    for (int64_t i = 0; i < d; ++i) e[i] = obs[t * d + i] - vdv[i];
    memcpy(z, e, sizeof(R) * (size_t)d);
    FN(o_trsm)(d, 1, L, z, 0, 0, 1, (R)1, NULL);
    R quad = (R)0, ld = (R)0;
    for (int64_t i = 0; i < d; ++i) quad += z[i] * z[i];
    for (int64_t i = 0; i < d; ++i) ld += LOG(AT(L, d, i, i));
    const R term = ((R)0.5 * quad + ld) + (R)0.5 * (R)d * log2pi;
    total = t == 0 ? term : total + term;
    FN(o_gemm)(h, d, h, X, S, b, 0, 1, (R)1, 0);
    memcpy(Y, X, sizeof(R) * (size_t)hd);
    FN(o_trsm)(h, d, L, Y, 1, 1, 1, (R)1, NULL);
    memcpy(K, Y, sizeof(R) * (size_t)hd);
    FN(o_trsm)(h, d, L, K, 1, 0, 1, (R)1, NULL);
    FN(o_gemm)(h, 1, d, vh, K, e, 0, 0, (R)1, 0);
    for (int64_t i = 0; i < h; ++i) muf[i] = mu[i] + vh[i];
    FN(o_gemm)(h, h, d, t1, K, b, 0, 0, (R)1, 0);
    for (int64_t i = 0; i < h; ++i)
      for (int64_t j = 0; j < h; ++j) AT(I, h, i, j) = (i == j ? (R)1 : (R)0) - AT(t1, h, i, j);
    FN(o_gemm)(h, h, h, P1, I, S, 0, 0, (R)1, 0);
    FN(o_gemm)(h, h, h, t2, P1, I, 0, 1, (R)1, 0);
    FN(o_gemm)(h, d, d, Q1, K, sv, 0, 0, (R)1, 0);
    FN(o_gemm)(h, h, d, t3, Q1, K, 0, 1, (R)1, 0);
    for (int64_t q = 0; q < hh; ++q) Sf[q] = t2[q] + t3[q];
    if (t + 1 < T) {
      FN(o_gemm)(h, 1, h, TP(t + 1, oMu), a, muf, 0, 0, (R)1, 0);
      FN(o_gemm)(h, h, h, t1, a, Sf, 0, 0, (R)1, 0);
      FN(o_gemm)(h, h, h, TP(t + 1, oS), t1, a, 0, 1, (R)1, 0);
      for (int64_t q = 0; q < hh; ++q) TP(t + 1, oS)[q] += sh[q];
    }
  }
  if (st == DLA_OK) {
    *nll = total;
    memset(abar, 0, sizeof(R) * (size_t)hh);
    memset(bbar, 0, sizeof(R) * (size_t)hd);
    memset(shbar, 0, sizeof(R) * (size_t)hh);
    memset(svbar, 0, sizeof(R) * (size_t)dd);
    memset(sbn, 0, sizeof(R) * (size_t)hh);
    memset(mbn, 0, sizeof(R) * (size_t)h);
    for (int64_t t = T - 1; t >= 0; --t) {
      R *S = TP(t, oS), *mu = TP(t, oMu), *M1 = TP(t, oM1), *L = TP(t, oL), *e = TP(t, oE), *z = TP(t, oZ);
      R *Y = TP(t, oY), *K = TP(t, oK), *I = TP(t, oI), *P1 = TP(t, oP1), *Q1 = TP(t, oQ1);
      R *Sf = TP(t, oSf), *muf = TP(t, oMuf);
      R* sfbar = t1; /* h x h */
      R* mufbar = vh;
      if (t + 1 < T) { /* S' = (A Sf) A^T + Sh, mu' = A muf */
        for (int64_t q = 0; q < hh; ++q) shbar[q] += sbn[q];
        FN(o_gemm)(h, h, h, t2, a, Sf, 0, 0, (R)1, 0);       /* R1 = A Sf */
        FN(o_gemm)(h, h, h, abar, sbn, t2, 1, 0, (R)1, 1);   /* Abar += S'bar^T R1 */
        FN(o_gemm)(h, h, h, t3, sbn, a, 0, 0, (R)1, 0);      /* R1bar = S'bar A */
        FN(o_gemm)(h, h, h, abar, t3, Sf, 0, 1, (R)1, 1);    /* Abar += R1bar Sf^T */
        FN(o_gemm)(h, h, h, sfbar, a, t3, 1, 0, (R)1, 0);    /* Sfbar = A^T R1bar */
        FN(o_gemm)(h, h, 1, abar, mbn, muf, 0, 1, (R)1, 1);  /* Abar += mu'bar muf^T */
        FN(o_gemm)(h, 1, h, mufbar, a, mbn, 1, 0, (R)1, 0);  /* mufbar = A^T mu'bar */
      } else {
        memset(sfbar, 0, sizeof(R) * (size_t)hh);
        memset(mufbar, 0, sizeof(R) * (size_t)h);
      }
      /* Q2 = Q1 K^T, Q1 = K Sv */
      FN(o_gemm)(h, d, h, vhd, sfbar, K, 0, 0, (R)1, 0);     /* Q1bar = Sfbar K */
      FN(o_gemm)(h, d, h, kbar, sfbar, Q1, 1, 0, (R)1, 0);   /* Kbar = Sfbar^T Q1 */
      FN(o_gemm)(h, d, d, kbar, vhd, sv, 0, 1, (R)1, 1);     /* Kbar += Q1bar Sv^T */
      FN(o_gemm)(d, d, h, svbar, K, vhd, 1, 0, (R)1, 1);     /* Svbar += K^T Q1bar */
      /* P2 = P1 I^T, P1 = I S */
      FN(o_gemm)(h, h, h, p1bar, sfbar, I, 0, 0, (R)1, 0);   /* P1bar = Sfbar I */
      FN(o_gemm)(h, h, h, ibar, sfbar, P1, 1, 0, (R)1, 0);   /* Ibar = Sfbar^T P1 */
      FN(o_gemm)(h, h, h, ibar, p1bar, S, 0, 1, (R)1, 1);    /* Ibar += P1bar S^T */
      FN(o_gemm)(h, h, h, sbar, I, p1bar, 1, 0, (R)1, 0);    /* Sbar = I^T P1bar */
      /* I = Id - K B */
      FN(o_gemm)(h, d, h, kbar, ibar, b, 0, 1, (R)-1, 1);    /* Kbar -= Ibar B^T */
      FN(o_gemm)(d, h, h, bbar, K, ibar, 1, 0, (R)-1, 1);    /* Bbar -= K^T Ibar */
      /* muf = mu + K e */
      memcpy(mubar, mufbar, sizeof(R) * (size_t)h);
      FN(o_gemm)(h, d, 1, kbar, mufbar, e, 0, 1, (R)1, 1);   /* Kbar += mufbar e^T */
      FN(o_gemm)(d, 1, h, ebar, K, mufbar, 1, 0, (R)1, 0);   /* ebar = K^T mufbar */
      /* K = Y L^-1, Y = X L^-T: trsm pullbacks (dl/adjoints.hpp:131-153) */
      FN(o_trsm_bwd)(h, d, ybar, lbar, kbar, L, K, 1, 0, 1, (R)1, NULL);
      FN(o_trsm_bwd)(h, d, vhd2, vd, ybar, L, Y, 1, 1, 1, (R)1, NULL);  /* vhd2 = Xbar */
      for (int64_t q = 0; q < dd; ++q) lbar[q] += vd[q];
      /* X = S B^T */
      FN(o_gemm)(h, h, d, sbar, vhd2, b, 0, 0, (R)1, 1);     /* Sbar += Xbar B */
      FN(o_gemm)(d, h, h, bbar, vhd2, S, 1, 0, (R)1, 1);     /* Bbar += Xbar^T S */
      /* phi_t: zbar = z, Lbar_ii += 1 / L_ii; z = L^-1 e */
      FN(o_trsm_bwd)(d, 1, vdv, vd, z, L, z, 0, 0, 1, (R)1, NULL);
      for (int64_t q = 0; q < dd; ++q) lbar[q] += vd[q];
      for (int64_t i = 0; i < d; ++i) AT(lbar, d, i, i) += (R)1 / AT(L, d, i, i);
      for (int64_t i = 0; i < d; ++i) ebar[i] += vdv[i];
      /* e = v - B mu */
      for (int64_t i = 0; i < d; ++i) obsbar[t * d + i] = ebar[i];
      FN(o_gemm)(d, h, 1, bbar, ebar, mu, 0, 1, (R)-1, 1);   /* Bbar -= ebar mu^T */
      FN(o_gemm)(h, 1, d, mubar, b, ebar, 1, 0, (R)-1, 1);   /* mubar -= B^T ebar */
      /* L = chol(Svv); Svv = M1 B^T + Sv; M1 = B S */
      FN(o_potrf_bwd)(d, vd, lbar, L, 1);
      for (int64_t q = 0; q < dd; ++q) svbar[q] += vd[q];
      FN(o_gemm)(d, h, d, m1bar, vd, b, 0, 0, (R)1, 0);      /* M1bar = Svvbar B */
      FN(o_gemm)(d, h, d, bbar, vd, M1, 1, 0, (R)1, 1);      /* Bbar += Svvbar^T M1 */
      FN(o_gemm)(d, h, h, bbar, m1bar, S, 0, 1, (R)1, 1);    /* Bbar += M1bar S^T */
      FN(o_gemm)(h, h, d, sbar, b, m1bar, 1, 0, (R)1, 1);    /* Sbar += B^T M1bar */
      memcpy(sbn, sbar, sizeof(R) * (size_t)hh);
      memcpy(mbn, mubar, sizeof(R) * (size_t)h);
    }
    memcpy(s0bar, sbn, sizeof(R) * (size_t)hh);
    memcpy(mu0bar, mbn, sizeof(R) * (size_t)h);
  }
#undef TP
  free(tape);
  free(w);
  return st;
}

#undef AT
