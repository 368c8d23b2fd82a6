// Batched LQ (f64) by CholeskyQR2 on DMMA, with a per-slice Householder
// fallback — the gelqf forward for the BLR shapes (BASELINE C3: 128 x 512).
//
// The reference's LQ (dl/lq.hpp:24-106, sign-normalized so diag(L) > 0) is
// unique for a full-rank A, so any stable factorization returns the same
// (Q, L) to rounding.  The blocked Householder path (gelqf_blk.cu) spends its
// time in 32-reflector panel chains (one CTA per slice, ~350 us per panel at
// 256 x 128 x 512, 0 % tensor pipe).  CholeskyQR2 is all batched DMMA work:
//
//   G1 = A A^T,  R1 = chol(G1),  Q1 = R1^-1 A        (pass 1)
//   G2 = Q1 Q1^T, R2 = chol(G2), Q  = R2^-1 Q1       (pass 2: restores
//                                                     orthogonality to O(eps))
//   L  = R2 R1  (lower x lower; positive diagonal, = the reference's sign rule)
//
// It is accurate while kappa(A)^2 eps << 1.  A slice falls back to the
// Householder path when (a) either Cholesky breaks down, (b) the pass-1
// diagonal spread max R1_ii / min R1_ii (a lower bound on kappa(A)) exceeds
// 1e5, or (c) the reference's rank test |L_ii| < 1e-12 max|A| fires (so the
// SingularError index comes from the reference's own algorithm).  The
// fallback runs on a copy of A for the flagged slices only (the other slices
// are masked through the skip array every kernel honours), so a batch with
// no flagged slice pays only early-exit launches.
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "ops.cuh"

namespace dlab {
namespace {

constexpr double KAPPA_MAX = 1e5;

inline MatB<double> pk(double* p, int64_t r, int64_t c) { return MatB<double>{p, c, r * c}; }
inline MatB<const double> C_(MatB<double> m) { return MatB<const double>{m.p, m.ld, m.bs, m.bsi}; }

// per slice: fb[b] = 1 when the CholeskyQR2 result must be replaced; the
// Householder pass's skip mask hinfo[b] = 0 (run) / 1 (skip)
__global__ void __launch_bounds__(256) k_cqr_flags(int64_t batch, int64_t m, int64_t n, const double* a,
                                                   const double* r1, const double* l, const int32_t* cinfo,
                                                   int32_t* fb, int32_t* hinfo) {
  __shared__ double red[3][8];
  const int64_t b = blockIdx.x;
  const double* ab = a + b * m * n;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  double mx = 0.0, dmin = INFINITY, dmax = 0.0, lmin = INFINITY;
  for (int64_t e = t; e < m * n; e += 256) mx = fmax(mx, fabs(ab[e]));
  for (int64_t i = t; i < m; i += 256) {
    const double d = fabs(r1[b * m * m + i * m + i]);
    dmin = fmin(dmin, d);
    dmax = fmax(dmax, d);
    lmin = fmin(lmin, fabs(l[b * m * m + i * m + i]));
  }
  for (int o = 16; o; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    dmin = fmin(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
    lmin = fmin(lmin, __shfl_xor_sync(0xffffffffu, lmin, o));
  }
  __shared__ double red2[8];
  if (lane == 0) {
    red[0][w] = mx;
    red[1][w] = dmax;
    red[2][w] = dmin;
    red2[w] = lmin;
  }
  __syncthreads();
  if (t == 0) {
    double amax = 0.0, dx = 0.0, dn = INFINITY, ln = INFINITY;
    for (int k = 0; k < 8; ++k) {
      amax = fmax(amax, red[0][k]);
      dx = fmax(dx, red[1][k]);
      dn = fmin(dn, red[2][k]);
      ln = fmin(ln, red2[k]);
    }
    // NaN-safe: a breakdown anywhere leaves a NaN / non-positive pivot
    const bool bad = cinfo[b] != 0 || !(ln >= Num<double>::rank_rtol * amax) || !(dx <= KAPPA_MAX * dn);
    fb[b] = bad ? 1 : 0;
    hinfo[b] = bad ? 0 : 1;
  }
}

// q[b] <- a[b] for the flagged slices (the Householder fallback's input)
__global__ void k_cqr_restore(int64_t batch, int64_t count, const double* a, double* q, const int32_t* fb) {
  for (int64_t b = blockIdx.y; b < batch; b += gridDim.y) {
    if (!fb[b]) continue;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x)
      q[b * count + e] = a[b * count + e];
  }
}

// the fallback's per-slice status (a rank failure) becomes the call's info
__global__ void k_cqr_merge(int64_t batch, const int32_t* fb, const int32_t* hinfo, int32_t* info) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < batch; b += (int64_t)gridDim.x * blockDim.x)
    if (fb[b] && hinfo[b] != 0 && info) info[b] = hinfo[b];
}

}  // namespace

bool gelqf_cqr_eligible(int64_t m, int64_t n) {
  static const bool on = [] {
    const char* e = getenv("DLA_GELQF_CQR");  // tuning switch: 0 keeps the blocked Householder path
    return e ? atoi(e) != 0 : true;
  }();
  return on && m >= 64 && m <= 512 && n >= m;
}

size_t ws_gelqf_cqr(int64_t batch, int64_t m, int64_t n) {
  const size_t mm = sizeof(double) * (size_t)(batch * m * m);
  // the call's arena is carved monotonically: every carve of the call tree adds up
  return carve_bound(sizeof(double) * (size_t)(batch * m * n)) + 2 * carve_bound(mm) +
         3 * carve_bound(sizeof(int32_t) * (size_t)batch) +
         2 * (ws_gemm<double>(batch, m, m, n) + ws_potrf_lower<double>(batch, m) + ws_trsm<double>(batch, m, n, false)) +
         ws_gemm<double>(batch, m, m, m) + carve_bound(gelqf_ws_bytes<double>(batch, m, n, false));
}

dla_status gelqf_cqr(const Ctx& c, int64_t batch, int64_t m, int64_t n, double* q, double* l) {
  DLAB_SCRATCH(sa, c, sizeof(double) * (size_t)(batch * m * n));  // A, kept for the fallback
  DLAB_SCRATCH(sg, c, sizeof(double) * (size_t)(batch * m * m));  // G1 -> R1
  DLAB_SCRATCH(sh, c, sizeof(double) * (size_t)(batch * m * m));  // G2 -> R2
  DLAB_SCRATCH(sfb, c, sizeof(int32_t) * (size_t)batch);
  DLAB_SCRATCH(shi, c, sizeof(int32_t) * (size_t)batch);
  DLAB_SCRATCH(sci, c, sizeof(int32_t) * (size_t)batch);  // the Cholesky breakdowns of both passes
  int32_t* fb = sfb.as<int32_t>();
  int32_t* hinfo = shi.as<int32_t>();
  int32_t* cinfo = sci.as<int32_t>();
  if (cudaMemsetAsync(cinfo, 0, sizeof(int32_t) * (size_t)batch, c.stream) != cudaSuccess) return DLA_ERR_CUDA;
  MatB<double> qa = pk(q, m, n), r1 = pk(sg.as<double>(), m, m), r2 = pk(sh.as<double>(), m, m);
  DLAB_TRY(ew_copy<double>(c, batch, m, n, C_(qa), pk(sa.as<double>(), m, n)));
  Ctx cc = c;
  cc.info = cinfo;  // breakdowns flag the slice, the call's info is left to the fallback
  for (int pass = 0; pass < 2; ++pass) {
    MatB<double> r = pass == 0 ? r1 : r2;
    // G = Q Q^T (lower), R = chol(G), Q <- R^-1 Q
    DLAB_TRY(gemm<double>(cc, batch, m, m, n, 1.0, C_(qa), false, C_(qa), true, 0.0, r, MASK_LOWER, nullptr));
    DLAB_TRY(potrf_lower<double>(cc, batch, m, r, /*zero_upper*/ true));
    DLAB_TRY(trsm<double>(cc, batch, m, n, C_(r), qa, false, false, true, 1.0, false));
  }
  // L = R2 R1 (lower x lower: the full-output product is lower, zeros above)
  DLAB_TRY(gemm<double>(cc, batch, m, m, m, 1.0, C_(r2), false, C_(r1), false, 0.0, pk(l, m, m), MASK_FULL, nullptr,
                        TRI_LOWER, TRI_LOWER));
  k_cqr_flags<<<(unsigned)batch, 256, 0, c.stream>>>(batch, m, n, sa.as<double>(), r1.p, l, cinfo, fb, hinfo);
  DLAB_LAUNCH_CHECK();
  // Householder fallback on the flagged slices (masked by hinfo)
  {
    const int64_t count = m * n;
    const unsigned gx = blocks_for(count, 256, 64), gy = (unsigned)std::min<int64_t>(batch, 65535);
    k_cqr_restore<<<dim3(gx, gy), 256, 0, c.stream>>>(batch, count, sa.as<double>(), q, fb);
    DLAB_LAUNCH_CHECK();
  }
  DLAB_SCRATCH(hws, c, gelqf_ws_bytes<double>(batch, m, n, false));
  Ctx hc = c;
  hc.info = hinfo;
  DLAB_TRY(gelqf_fwd<double>(hc, batch, m, n, q, l, hws.p, true));
  k_cqr_merge<<<blocks_for(batch, 256), 256, 0, c.stream>>>(batch, fb, hinfo, c.info);
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}

}  // namespace dlab
