// Batched Kalman filter NLL + gradient of every leaf.
//
// The reference builds the filter as a tape of tiny nodes, T steps of
// gemm2 / potrf / trsm on h x h and d x d blocks (dl/models.hpp:285-337), and
// differentiates it with Graph::backward; its test oracle is the dense
// joint Gaussian (proj/tests/kalman_oracle.hpp:16-79).  Here one CTA runs a
// whole sequence: the forward recursion with every step's intermediates
// written to a device tape (caller workspace), then the reverse sweep that
// applies the same pullbacks the tape would (gemm2, trsm, potrf:
// dl/adjoints.hpp:36-49, :131-153, :175-191; the elementwise add / sub /
// square / log / sum chain) — step for step the math of
// oracle/oracle_impl.h o_kalman (pinned to the reference, ≤ 3e-15).
// All blocks of a step live in shared memory; a batch of independent
// sequences (or one model over many sequences, param_stride = 0) fills the
// GPU with CTAs, so the per-step barrier chain is hidden by occupancy
// (the launch-bound "small-n" regime of the north star).
//
// Per step t (mu, S predicted; v = obs[t]):
//   M1 = B S;  Svv = M1 B^T + Sv;  L = chol(Svv);  e = v - B mu;  z = L^-1 e
//   phi_t = 1/2 z^T z + sum log L_ii + d/2 log 2 pi
//   X = S B^T;  Y = X L^-T;  K = Y L^-1;  mu_f = mu + K e;  I_KB = I - K B
//   P1 = I_KB S;  S_f = P1 I_KB^T + (K Sv) K^T
//   (t < T-1)  mu' = A mu_f;  S' = (A S_f) A^T + Sh
#include "common.cuh"

namespace dlab {
namespace {

constexpr int KT = 128;    // max threads per sequence (the launch uses kalman_threads())
constexpr int KMAX = 32;   // h, d <= 32
constexpr int KMSLOTS = 22, KVSLOTS = 9;  // shared-memory matrix / vector slots

struct KDims {
  int h, d, T;
  int64_t hh, hd, dd, step;  // tape floats per step
  // tape offsets within a step
  int64_t oS, oMu, oM1, oL, oE, oZ, oY, oK, oI, oP1, oQ1, oSf, oMuf;
};

inline KDims kdims(int64_t h, int64_t d, int64_t T) {
  KDims k;
  k.h = (int)h;
  k.d = (int)d;
  k.T = (int)T;
  k.hh = h * h;
  k.hd = h * d;
  k.dd = d * d;
  int64_t o = 0;
  k.oS = o; o += k.hh;
  k.oMu = o; o += h;
  k.oM1 = o; o += k.hd;
  k.oL = o; o += k.dd;
  k.oE = o; o += d;
  k.oZ = o; o += d;
  k.oY = o; o += k.hd;
  k.oK = o; o += k.hd;
  k.oI = o; o += k.hh;
  k.oP1 = o; o += k.hh;
  k.oQ1 = o; o += k.hd;
  k.oSf = o; o += k.hh;
  k.oMuf = o; o += h;
  k.step = (o + 1) & ~int64_t(1);  // 16-byte aligned steps
  return k;
}

// C (m x n) = alpha op(A) op(B) (+ C if acc); A: ta ? k x m : m x k;
// B: tb ? n x k : k x n; sequential k (no barrier inside).
// NT: threads per sequence (compile time); with the block sizes compile-time
// constants too (the specialised kernels) every loop below unrolls into
// straight-line FMAs on constant shared-memory offsets.
template <int NT, typename T>
__device__ __forceinline__ void mm(T* C, const T* A, const T* B, int m, int n, int k, bool ta, bool tb, T alpha,
                                   bool acc) {
#pragma unroll
  for (int idx = threadIdx.x; idx < m * n; idx += NT) {
    const int i = idx / n, j = idx - i * n;
    T s = T(0);
#pragma unroll
    for (int p = 0; p < k; ++p) {
      const T av = ta ? A[p * m + i] : A[i * k + p];
      const T bv = tb ? B[j * k + p] : B[p * n + j];
      s += av * bv;
    }
    C[idx] = acc ? C[idx] + alpha * s : alpha * s;
  }
}

template <int NT, typename T>
__device__ __forceinline__ void cpy(T* dst, const T* src, int n) {
#pragma unroll
  for (int i = threadIdx.x; i < n; i += NT) dst[i] = src[i];
}

// Cholesky of the d x d block S (lower, in place, strict upper zeroed) by
// warp 0: right-looking, lane = row.  Returns the failing step or -1
// (uniform after the caller's barrier through *fail).
template <typename T>
__device__ __forceinline__ void chol_warp(T* S, int d, int* fail) {
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  for (int j = 0; j < d; ++j) {
    const T piv = S[j * d + j];
    if (!(piv > T(0))) {
      if (lane == 0) *fail = j;
      return;
    }
    const T r = Num<T>::sqrt_(piv);
    __syncwarp();
    if (lane == j) S[j * d + j] = r;
    if (lane > j && lane < d) S[lane * d + j] /= r;
    __syncwarp();
    if (lane > j && lane < d) {
      const T lij = S[lane * d + j];
      for (int k = j + 1; k <= lane; ++k) S[lane * d + k] -= lij * S[k * d + j];
    }
    __syncwarp();
  }
  if (lane < d)
    for (int k = lane + 1; k < d; ++k) S[lane * d + k] = T(0);
}

// Row-wise triangular solves with L (d x d lower), one thread per row of the
// (rows x d) operand X, in place:
//   mode 0: x <- x L^-T  (L x'^T = x^T: forward substitution)
//   mode 1: x <- x L^-1  (L^T x'^T = x^T: back substitution)
// `extra` (optional): one more row vector solved the same way, by the lane
// after the last row (in the same instruction stream as the rows).
template <int NT, typename T>
__device__ __forceinline__ void rows_solve(T* X, int rows, const T* L, int d, int mode, T* extra = nullptr) {
  const int nr = extra ? rows + 1 : rows;
#pragma unroll
  for (int i = threadIdx.x; i < nr; i += NT) {
    T* x = i < rows ? X + i * d : extra;
    if (mode == 0) {
      for (int j = 0; j < d; ++j) {
        T s = x[j];
        for (int k = 0; k < j; ++k) s -= L[j * d + k] * x[k];
        x[j] = s / L[j * d + j];
      }
    } else {
      for (int j = d - 1; j >= 0; --j) {
        T s = x[j];
        for (int k = j + 1; k < d; ++k) s -= L[k * d + j] * x[k];
        x[j] = s / L[j * d + j];
      }
    }
  }
}

template <typename T>
struct KArgs {
  KDims k;
  int64_t batch, pstride;  // pstride: 1 = per-sequence parameters, 0 = shared
  const T *a, *b, *sh, *sv, *mu0, *s0, *obs;
  T *nll, *abar, *bbar, *shbar, *svbar, *mu0bar, *s0bar, *obsbar;
  T* tape;
  int32_t* info;
};

// NT threads per sequence: 128 (8 CTAs/SM by registers), 64 (16) or 32 (32):
// the per-step chain is latency-bound on 8 x 8 blocks, so smaller CTAs keep
// more sequences in flight per SM.
// H, D > 0: the state / observation sizes as compile-time constants (the
// common small models; same operation order as the runtime-size kernel, so
// the results are bitwise identical); 0 = read from the arguments.
template <typename T, int NT, int H = 0, int D = 0>
__global__ void __launch_bounds__(NT, (NT == 128 ? 8 : NT == 64 ? 16 : 32)) k_kalman(KArgs<T> g) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  const KDims& K = g.k;
  const int h = H > 0 ? H : K.h, d = D > 0 ? D : K.d, nT = K.T;
  const int hh = h * h, hd = h * d, dd = d * d;
  const int64_t seq = blockIdx.x;
  if (slice_failed(g.info, seq)) return;
  __shared__ int fail;
  if (threadIdx.x == 0) fail = -1;
  // parameters
  const int64_t ps = g.pstride;
  T* A = sm;
  T* B = A + hh;
  T* Sh = B + hd;
  T* Sv = Sh + hh;
  T* W = Sv + dd;  // work slots of KMAX^2 / general sizes below
  cpy<NT>(A, g.a + ps * seq * hh, hh);
  cpy<NT>(B, g.b + ps * seq * hd, hd);
  cpy<NT>(Sh, g.sh + ps * seq * hh, hh);
  cpy<NT>(Sv, g.sv + ps * seq * dd, dd);
  const int64_t mx = h > d ? h : d;
  const int64_t slot = (mx * mx + 1) & ~int64_t(1), vslot = (mx + 1) & ~int64_t(1);
  auto S_ = [&](int i) { return W + i * slot; };                                  // matrix slots
  auto V_ = [&](int i) { return W + KMSLOTS * slot + i * vslot; };                 // vector slots
  T* tape = g.tape + seq * nT * K.step;
  const T* obs = g.obs + seq * (int64_t)nT * d;
  const T log2pi = T(1.8378770664093454835606594728112353L);
  // ------------------------------------------------------------ forward
  {
    T* S = tape + K.oS;  // step 0's predicted state comes from the prior
    cpy<NT>(S, g.s0 + ps * seq * hh, hh);
    cpy<NT>(tape + K.oMu, g.mu0 + ps * seq * h, h);
  }
  T total = T(0);
  __syncthreads();
  for (int t = 0; t < nT; ++t) {
    T* tp = tape + t * K.step;
    T *S = S_(0), *M1 = S_(1), *L = S_(2), *Y = S_(3), *Kg = S_(4), *I = S_(5), *P1 = S_(6), *Q1 = S_(7);
    T *Sf = S_(8), *t1 = S_(9), *t2 = S_(10);
    T *mu = V_(0), *e = V_(1), *z = V_(2), *muf = V_(3), *lg = V_(4);  // (V_(4): the backward's mbn)
    cpy<NT>(S, tp + K.oS, hh);
    cpy<NT>(mu, tp + K.oMu, h);
    __syncthreads();
    mm<NT>(M1, B, S, d, h, h, false, false, T(1), false);        // M1 = B S
    mm<NT>(Y, S, B, h, d, h, false, true, T(1), false);          // X = S B^T (into Y)
    mm<NT>(e, B, mu, d, 1, h, false, false, T(-1), false);       // e = -B mu
    __syncthreads();
    mm<NT>(L, M1, B, d, d, h, false, true, T(1), false);         // Svv = M1 B^T
    for (int i = threadIdx.x; i < d; i += NT) e[i] += obs[t * d + i];
    __syncthreads();
    for (int i = threadIdx.x; i < dd; i += NT) L[i] += Sv[i];
    __syncthreads();
    chol_warp(L, d, &fail);
    __syncthreads();
    if (fail >= 0) {
      if (threadIdx.x == 0) record_failure(g.info, seq, DLA_ERR_NOT_SPD, (int64_t)t * d + fail);
      return;
    }
    for (int i = threadIdx.x; i < d; i += NT) {
      z[i] = e[i];
      lg[i] = Num<T>::log_(L[i * d + i]);  // the d logs in parallel; summed in order below
    }
    __syncthreads();
    rows_solve<NT>(Y, h, L, d, 0, z);                             // Y = X L^-T;  z = L^-1 e (one more row)
    __syncthreads();
    if (threadIdx.x == 0) {  // phi_t (sequential sums as the tape's Sum)
      T quad = T(0), ld = T(0);
      for (int i = 0; i < d; ++i) quad += z[i] * z[i];
      for (int i = 0; i < d; ++i) ld += lg[i];
      const T term = (T(0.5) * quad + ld) + T(0.5) * T(d) * log2pi;
      total = t == 0 ? term : total + term;
    }
    cpy<NT>(Kg, Y, hd);
    __syncthreads();
    rows_solve<NT>(Kg, h, L, d, 1);                               // K = Y L^-1
    __syncthreads();
    mm<NT>(muf, Kg, e, h, 1, d, false, false, T(1), false);      // K e
    mm<NT>(I, Kg, B, h, h, d, false, false, T(-1), false);       // -K B
    mm<NT>(Q1, Kg, Sv, h, d, d, false, false, T(1), false);      // Q1 = K Sv
    __syncthreads();
    for (int i = threadIdx.x; i < h; i += NT) muf[i] += mu[i];
    for (int i = threadIdx.x; i < h; i += NT) I[i * h + i] += T(1);
    __syncthreads();
    mm<NT>(P1, I, S, h, h, h, false, false, T(1), false);        // P1 = I_KB S
    mm<NT>(t1, Q1, Kg, h, h, d, false, true, T(1), false);       // Q2 = Q1 K^T
    __syncthreads();
    mm<NT>(Sf, P1, I, h, h, h, false, true, T(1), false);        // P2 = P1 I_KB^T
    __syncthreads();
    for (int i = threadIdx.x; i < hh; i += NT) Sf[i] += t1[i];
    __syncthreads();
    // tape of this step
    cpy<NT>(tp + K.oM1, M1, hd);
    cpy<NT>(tp + K.oL, L, dd);
    cpy<NT>(tp + K.oE, e, d);
    cpy<NT>(tp + K.oZ, z, d);
    cpy<NT>(tp + K.oY, Y, hd);
    cpy<NT>(tp + K.oK, Kg, hd);
    cpy<NT>(tp + K.oI, I, hh);
    cpy<NT>(tp + K.oP1, P1, hh);
    cpy<NT>(tp + K.oQ1, Q1, hd);
    cpy<NT>(tp + K.oSf, Sf, hh);
    cpy<NT>(tp + K.oMuf, muf, h);
    if (t + 1 < nT) {
      T* tn = tp + K.step;
      mm<NT>(tn + K.oMu, A, muf, h, 1, h, false, false, T(1), false);  // mu' = A mu_f
      mm<NT>(t2, A, Sf, h, h, h, false, false, T(1), false);           // A S_f
      __syncthreads();
      mm<NT>(tn + K.oS, t2, A, h, h, h, false, true, T(1), false);     // (A S_f) A^T
      __syncthreads();
      for (int i = threadIdx.x; i < hh; i += NT) tn[K.oS + i] += Sh[i];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) g.nll[seq] = total;
  // ------------------------------------------------------------ backward
  T* gA = g.abar + seq * hh;
  T* gB = g.bbar + seq * hd;
  T* gSh = g.shbar + seq * hh;
  T* gSv = g.svbar + seq * dd;
  T *aA = S_(11), *aB = S_(12), *aSh = S_(13), *aSv = S_(14), *sbn = S_(15), *mbn = V_(4);
  for (int i = threadIdx.x; i < hh; i += NT) aA[i] = aSh[i] = sbn[i] = T(0);
  for (int i = threadIdx.x; i < hd; i += NT) aB[i] = T(0);
  for (int i = threadIdx.x; i < dd; i += NT) aSv[i] = T(0);
  for (int i = threadIdx.x; i < h; i += NT) mbn[i] = T(0);
  __syncthreads();
  for (int t = nT - 1; t >= 0; --t) {
    const T* tp = tape + t * K.step;
    T *S = S_(0), *M1 = S_(1), *L = S_(2), *Y = S_(3), *Kg = S_(4), *I = S_(5), *P1 = S_(6), *Q1 = S_(7);
    T *Sf = S_(8), *t1 = S_(9), *t2 = S_(10);
    T *mu = V_(0), *e = V_(1), *z = V_(2), *muf = V_(3);
    // S_f bar, Q1bar, P1bar and Ibar are dead once Kbar / Sbar have absorbed
    // them: M1bar, Xbar, Ybar and Lbar reuse their slots
    T *sfb = S_(16), *q1b = S_(17), *kb = S_(18), *p1b = S_(19), *ib = S_(20), *sb = S_(21);
    T *yb = p1b, *xb = q1b, *lb = ib, *m1b = sfb;
    T *mufb = V_(5), *mub = V_(6), *eb = V_(7), *sv_ = V_(8);
    cpy<NT>(S, tp + K.oS, hh);
    cpy<NT>(mu, tp + K.oMu, h);
    cpy<NT>(M1, tp + K.oM1, hd);
    cpy<NT>(L, tp + K.oL, dd);
    cpy<NT>(e, tp + K.oE, d);
    cpy<NT>(z, tp + K.oZ, d);
    cpy<NT>(Y, tp + K.oY, hd);
    cpy<NT>(Kg, tp + K.oK, hd);
    cpy<NT>(I, tp + K.oI, hh);
    cpy<NT>(P1, tp + K.oP1, hh);
    cpy<NT>(Q1, tp + K.oQ1, hd);
    cpy<NT>(Sf, tp + K.oSf, hh);
    cpy<NT>(muf, tp + K.oMuf, h);
    __syncthreads();
    if (t + 1 < nT) {  // S' = (A S_f) A^T + Sh,  mu' = A mu_f
      for (int i = threadIdx.x; i < hh; i += NT) aSh[i] += sbn[i];
      mm<NT>(t1, A, Sf, h, h, h, false, false, T(1), false);     // R1 = A S_f
      mm<NT>(t2, sbn, A, h, h, h, false, false, T(1), false);    // R1bar = S'bar A
      mm<NT>(mufb, A, mbn, h, 1, h, true, false, T(1), false);   // mu_f bar = A^T mu'bar
      __syncthreads();
      mm<NT>(aA, sbn, t1, h, h, h, true, false, T(1), true);     // Abar += S'bar^T R1
      mm<NT>(sfb, A, t2, h, h, h, true, false, T(1), false);     // S_f bar = A^T R1bar
      __syncthreads();
      mm<NT>(aA, t2, Sf, h, h, h, false, true, T(1), true);      // Abar += R1bar S_f^T
      __syncthreads();
      mm<NT>(aA, mbn, muf, h, h, 1, false, true, T(1), true);    // Abar += mu'bar mu_f^T
    } else {
      for (int i = threadIdx.x; i < hh; i += NT) sfb[i] = T(0);
      for (int i = threadIdx.x; i < h; i += NT) mufb[i] = T(0);
    }
    __syncthreads();
    // S_f = P1 I^T + (K Sv) K^T
    mm<NT>(q1b, sfb, Kg, h, d, h, false, false, T(1), false);   // Q1bar = S_f bar K
    mm<NT>(kb, sfb, Q1, h, d, h, true, false, T(1), false);     // Kbar = S_f bar^T Q1
    mm<NT>(p1b, sfb, I, h, h, h, false, false, T(1), false);    // P1bar = S_f bar I
    mm<NT>(ib, sfb, P1, h, h, h, true, false, T(1), false);     // Ibar = S_f bar^T P1
    __syncthreads();
    mm<NT>(kb, q1b, Sv, h, d, d, false, true, T(1), true);      // Kbar += Q1bar Sv^T
    mm<NT>(aSv, Kg, q1b, d, d, h, true, false, T(1), true);     // Svbar += K^T Q1bar
    mm<NT>(ib, p1b, S, h, h, h, false, true, T(1), true);       // Ibar += P1bar S^T
    mm<NT>(sb, I, p1b, h, h, h, true, false, T(1), false);      // Sbar = I^T P1bar
    __syncthreads();
    // I = Id - K B;  mu_f = mu + K e
    mm<NT>(kb, ib, B, h, d, h, false, true, T(-1), true);       // Kbar -= Ibar B^T
    mm<NT>(aB, Kg, ib, d, h, h, true, false, T(-1), true);      // Bbar -= K^T Ibar
    cpy<NT>(mub, mufb, h);
    mm<NT>(eb, Kg, mufb, d, 1, h, true, false, T(1), false);    // ebar = K^T mu_f bar
    __syncthreads();
    mm<NT>(kb, mufb, e, h, d, 1, false, true, T(1), true);      // Kbar += mu_f bar e^T
    __syncthreads();
    // K = Y L^-1: Ybar = Kbar L^-T, Lbar = -tril(K^T Ybar)
    cpy<NT>(yb, kb, hd);
    __syncthreads();
    rows_solve<NT>(yb, h, L, d, 0);
    __syncthreads();
    mm<NT>(lb, Kg, yb, d, d, h, true, false, T(-1), false);
    // Y = X L^-T: Xbar = Ybar L^-1, Lbar += -tril(Xbar^T Y)
    cpy<NT>(xb, yb, hd);
    cpy<NT>(sv_, z, d);
    __syncthreads();
    // phi_t: zbar = z;  z = L^-1 e:  s = L^-T zbar (one more row of the solve)
    rows_solve<NT>(xb, h, L, d, 1, sv_);
    __syncthreads();
    mm<NT>(lb, xb, Y, d, d, h, true, false, T(-1), true);
    // X = S B^T
    mm<NT>(sb, xb, B, h, h, d, false, false, T(1), true);       // Sbar += Xbar B
    mm<NT>(aB, xb, S, d, h, h, true, false, T(1), true);        // Bbar += Xbar^T S
    __syncthreads();
    // ebar += s;  Lbar += -tril(s z^T);  Lbar_ii += 1 / L_ii
    for (int i = threadIdx.x; i < d; i += NT) eb[i] += sv_[i];
    __syncthreads();
    for (int idx = threadIdx.x; idx < dd; idx += NT) {
      const int i = idx / d, j = idx - i * d;
      if (j <= i) {
        T v = lb[idx] - sv_[i] * z[j];
        if (i == j) v += T(1) / L[i * d + i];
        lb[idx] = v;
      } else {
        lb[idx] = T(0);  // only tril(Lbar) enters the potrf pullback
      }
    }
    // e = v - B mu
    if (g.obsbar)
      for (int i = threadIdx.x; i < d; i += NT) g.obsbar[(seq * nT + t) * (int64_t)d + i] = eb[i];
    __syncthreads();
    mm<NT>(aB, eb, mu, d, h, 1, false, true, T(-1), true);      // Bbar -= ebar mu^T
    mm<NT>(mub, B, eb, h, 1, d, true, false, T(-1), true);      // mubar -= B^T ebar
    // L = chol(Svv):  Svvbar = 1/2 sym(L^-T copyltu(L^T Lbar) L^-1)  (dl/adjoints.hpp:175-191)
    mm<NT>(t1, L, lb, d, d, d, true, false, T(1), false);       // L^T Lbar
    __syncthreads();
    for (int idx = threadIdx.x; idx < dd; idx += NT) {  // copyltu
      const int i = idx / d, j = idx - i * d;
      t2[idx] = j > i ? t1[j * d + i] : t1[idx];
    }
    __syncthreads();
    for (int j = threadIdx.x; j < d; j += NT) {  // column j: t2(:, j) <- L^-T t2(:, j)
      for (int r = d - 1; r >= 0; --r) {
        T acc = t2[r * d + j];
        for (int k = r + 1; k < d; ++k) acc -= L[k * d + r] * t2[k * d + j];
        t2[r * d + j] = acc / L[r * d + r];
      }
    }
    __syncthreads();
    rows_solve<NT>(t2, d, L, d, 1);                             // (.) L^-1
    __syncthreads();
    for (int idx = threadIdx.x; idx < dd; idx += NT) {  // 1/2, then exact symmetrization
      const int i = idx / d, j = idx - i * d;
      t1[idx] = (T(0.5) * t2[idx] + T(0.5) * t2[j * d + i]) / T(2);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < dd; i += NT) aSv[i] += t1[i];
    mm<NT>(m1b, t1, B, d, h, d, false, false, T(1), false);     // M1bar = Svvbar B
    mm<NT>(aB, t1, M1, d, h, d, true, false, T(1), true);       // Bbar += Svvbar^T M1
    __syncthreads();
    mm<NT>(aB, m1b, S, d, h, h, false, true, T(1), true);       // Bbar += M1bar S^T
    mm<NT>(sb, B, m1b, h, h, d, true, false, T(1), true);       // Sbar += B^T M1bar
    __syncthreads();
    cpy<NT>(sbn, sb, hh);
    cpy<NT>(mbn, mub, h);
    __syncthreads();
  }
  cpy<NT>(gA, aA, hh);
  cpy<NT>(gB, aB, hd);
  cpy<NT>(gSh, aSh, hh);
  cpy<NT>(gSv, aSv, dd);
  cpy<NT>(g.s0bar + seq * hh, sbn, hh);
  cpy<NT>(g.mu0bar + seq * h, mbn, h);
}

template <typename T>
size_t kalman_smem(int64_t h, int64_t d) {
  const int64_t m = h > d ? h : d;
  const int64_t slot = (m * m + 1) & ~int64_t(1), vslot = (m + 1) & ~int64_t(1);
  return sizeof(T) * (size_t)(2 * h * h + h * d + d * d + KMSLOTS * slot + KVSLOTS * vslot + 2);
}

}  // namespace

template <typename T>
size_t kalman_ws_bytes(int64_t batch, int64_t h, int64_t d, int64_t T_) {
  if (batch <= 0 || h <= 0 || d <= 0 || T_ <= 0) return 0;
  return sizeof(T) * (size_t)batch * (size_t)T_ * (size_t)kdims(h, d, T_).step;
}

template <typename T>
dla_status kalman_fwdbwd(const Ctx& c, int64_t batch, int64_t h, int64_t d, int64_t T_, const T* a, const T* b,
                         const T* sh, const T* sv, const T* mu0, const T* s0, const T* obs, int64_t pstride, T* nll,
                         T* abar, T* bbar, T* shbar, T* svbar, T* mu0bar, T* s0bar, T* obsbar, T* tape) {
  KArgs<T> g;
  g.k = kdims(h, d, T_);
  g.batch = batch;
  g.pstride = pstride;
  g.a = a;
  g.b = b;
  g.sh = sh;
  g.sv = sv;
  g.mu0 = mu0;
  g.s0 = s0;
  g.obs = obs;
  g.nll = nll;
  g.abar = abar;
  g.bbar = bbar;
  g.shbar = shbar;
  g.svbar = svbar;
  g.mu0bar = mu0bar;
  g.s0bar = s0bar;
  g.obsbar = obsbar;
  g.tape = tape;
  g.info = c.info;
  const size_t sm = kalman_smem<T>(h, d);
  static const int nt = [] {
    // tuning switch: 32 / 64 / 128 threads per sequence (measured at 4096 x (8, 8, 128):
    // 196k / 181k / 146k sequences/s -- one warp per sequence keeps 32 in flight per SM)
    const char* e = getenv("DLA_KALMAN_THREADS");
    const int v = e ? atoi(e) : 32;
    return v == 64 || v == 128 ? v : 32;
  }();
  auto go = [&](auto kern, int threads) {
    ensure_smem_attr(kern, sm);
    kern<<<(unsigned)batch, threads, sm, c.stream>>>(g);
  };
  static const bool spec = [] {
    const char* e = getenv("DLA_KALMAN_SPECIALISE");  // tuning switch: 0 = runtime-size kernel only
    return e ? atoi(e) != 0 : true;
  }();
  if (nt == 32 && spec && h == 8 && d == 8) go(k_kalman<T, 32, 8, 8>, 32);
  else if (nt == 32 && spec && h == 4 && d == 4) go(k_kalman<T, 32, 4, 4>, 32);
  else if (nt == 32 && spec && h == 8 && d == 4) go(k_kalman<T, 32, 8, 4>, 32);
  else if (nt == 32) go(k_kalman<T, 32>, 32);
  else if (nt == 128) go(k_kalman<T, 128>, 128);
  else go(k_kalman<T, 64>, 64);
  DLAB_LAUNCH_CHECK();
  note_launch(1);
  return DLA_OK;
}

bool kalman_dims_ok(int64_t h, int64_t d) { return h >= 1 && d >= 1 && h <= KMAX && d <= KMAX; }

template <typename T>
dla_status kalman_entry(int64_t batch, int64_t h, int64_t d, int64_t T_, const T* a, const T* b, const T* sh,
                        const T* sv, const T* mu0, const T* s0, const T* obs, int64_t pstride, T* nll, T* abar,
                        T* bbar, T* shbar, T* svbar, T* mu0bar, T* s0bar, T* obsbar, int32_t* info, void* ws,
                        size_t ws_bytes, void* stream) {
  // build_kalman_nll's checks (dl/models.hpp:288-302): no observations or
  // inconsistent shapes are ShapeErrors; blocks above 32 are outside this
  // kernel's shared-memory design (reported as SHAPE as well)
  if (batch < 0 || T_ < 1 || !kalman_dims_ok(h, d)) return DLA_ERR_SHAPE;
  if (pstride != 0 && pstride != 1) return DLA_ERR_INVALID;
  if (batch == 0) return DLA_OK;
  if (!a || !b || !sh || !sv || !mu0 || !s0 || !obs || !nll || !abar || !bbar || !shbar || !svbar || !mu0bar ||
      !s0bar)
    return DLA_ERR_INVALID;
  if (!ws || ws_bytes < kalman_ws_bytes<T>(batch, h, d, T_)) return DLA_ERR_WORKSPACE;
  Ctx c = make_ctx(stream, info);
  if (info && cudaMemsetAsync(info, 0, sizeof(int32_t) * (size_t)batch, c.stream) != cudaSuccess)
    return DLA_ERR_CUDA;
  return kalman_fwdbwd<T>(c, batch, h, d, T_, a, b, sh, sv, mu0, s0, obs, pstride, nll, abar, bbar, shbar, svbar,
                          mu0bar, s0bar, obsbar, static_cast<T*>(ws));
}

#define INST(T)                                                                                                  \
  template size_t kalman_ws_bytes<T>(int64_t, int64_t, int64_t, int64_t);                                       \
  template dla_status kalman_fwdbwd<T>(const Ctx&, int64_t, int64_t, int64_t, int64_t, const T*, const T*,       \
                                       const T*, const T*, const T*, const T*, const T*, int64_t, T*, T*, T*, T*, \
                                       T*, T*, T*, T*, T*);
INST(double)
INST(float)

}  // namespace dlab

using namespace dlab;

extern "C" {

size_t dla_kalman_ws_bytes_f64(int64_t batch, int64_t h, int64_t d, int64_t T) {
  return kalman_ws_bytes<double>(batch, h, d, T);
}
size_t dla_kalman_ws_bytes_f32(int64_t batch, int64_t h, int64_t d, int64_t T) {
  return kalman_ws_bytes<float>(batch, h, d, T);
}

#define DLA_KALMAN(Tp, S)                                                                                          \
  dla_status dla_kalman_nll_fwdbwd_##S(int64_t batch, int64_t h, int64_t d, int64_t T, const Tp* a, const Tp* b,   \
                                       const Tp* sh, const Tp* sv, const Tp* mu0, const Tp* s0, const Tp* obs,     \
                                       int64_t param_stride, Tp* nll, Tp* abar, Tp* bbar, Tp* shbar, Tp* svbar,    \
                                       Tp* mu0bar, Tp* s0bar, Tp* obsbar, int32_t* info, void* ws,                \
                                       size_t ws_bytes, void* stream) {                                           \
    return kalman_entry<Tp>(batch, h, d, T, a, b, sh, sv, mu0, s0, obs, param_stride, nll, abar, bbar, shbar,     \
                            svbar, mu0bar, s0bar, obsbar, info, ws, ws_bytes, stream);                            \
  }
DLA_KALMAN(double, f64)
DLA_KALMAN(float, f32)
#undef DLA_KALMAN

}  // extern "C"
