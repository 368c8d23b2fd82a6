// Batched symmetric eigensolver: A = U^T diag(lambda) U with the ROWS of U as
// eigenvectors, lambda ascending and the reference's deterministic sign rule
// (dl/eigen_sym.hpp:316-333: flip row i when its largest-|.| entry, first
// index on ties, is negative).  Symmetry precheck as potrf
// (dl/eigen_sym.hpp:340, dl/cholesky.hpp:19-25); n = 1 special case (:342-346).
//
// Algorithm (B200-first, not the reference's EISPACK tred1/tql1/tinvit
// pipeline, which is a chain of scalar recurrences): two-sided cyclic Jacobi
// with the round-robin parallel ordering.  Each round applies n/2 disjoint
// rotations to whole rows, then whole columns, then the eigenvector
// accumulator — every thread of the CTA busy, A and V resident in shared
// memory for n <= 64 (one CTA per matrix), in the caller's workspace
// otherwise.  The input is pre-scaled by an exact power of two so the
// convergence test is scale invariant (tests/test_eigen.cpp:127-135).
// Sweeps are capped (ConvergenceError as dl/eigen_sym.hpp:113-118).
//
// Also here: the syevd-backward gap kernel (dl/adjoints.hpp:278-286) and the
// symmetrizing copy (:289-294).
#include "common.cuh"
#include "ops.cuh"

namespace dlab {
namespace {

constexpr int EN = 64;        // shared-memory path limit
constexpr int ET = 256;       // threads per CTA
constexpr int MAX_SWEEPS = 40;

template <typename T>
struct Eps;
template <>
struct Eps<double> {
  static constexpr double v = 2.220446049250313e-16;
};
template <>
struct Eps<float> {
  static constexpr float v = 1.1920929e-07f;
};

template <typename T>
__device__ T bmax(T v, T* red) {
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  T r = red[0];
  for (int k = 1; k < ET / 32; ++k) r = fmax(r, red[k]);
  return r;
}

// Round-robin pairing (circle method) over N = even players; round r, pair k.
__device__ __forceinline__ void rr_pair(int N, int r, int k, int& p, int& q) {
  const int M = N - 1;
  if (k == 0) {
    p = M;
    q = r % M;
  } else {
    p = (r + k) % M;
    q = (r - k + M) % M;
  }
  if (p > q) {
    int t = p;
    p = q;
    q = t;
  }
}

// A (lda = ld) and V in shared or global memory; n real size, N = padded even.
template <typename T>
__device__ void jacobi(int n, T* A, T* V, int ld, T* cs, int* pq, T* red, int* sweeps_out) {
  const int N = n + (n & 1);
  const int half = N / 2;
  for (int e = threadIdx.x; e < n * n; e += ET) V[(e / n) * ld + e % n] = (e / n == e % n) ? T(1) : T(0);
  __syncthreads();
  int sweep = 0;
  for (; sweep < MAX_SWEEPS; ++sweep) {
    // convergence: max off-diagonal vs max diagonal (matrix pre-scaled to O(1))
    T off = T(0), dia = T(0);
    for (int e = threadIdx.x; e < n * n; e += ET) {
      const int i = e / n, j = e % n;
      const T v = fabs(A[i * ld + j]);
      if (i != j) off = fmax(off, v);
      else dia = fmax(dia, v);
    }
    off = bmax(off, red);
    dia = bmax(dia, red);
    if (off <= Eps<T>::v * dia) break;
    if (off == T(0)) break;
    for (int r = 0; r < N - 1; ++r) {
      // rotation parameters for each pair (Rutishauser)
      for (int k = threadIdx.x; k < half; k += ET) {
        int p, q;
        rr_pair(N, r, k, p, q);
        T c = T(1), s = T(0);
        if (q < n) {
          const T apq = A[p * ld + q];
          if (apq != T(0)) {
            const T theta = (A[q * ld + q] - A[p * ld + p]) / (T(2) * apq);
            T t;
            if (fabs(theta) > (sizeof(T) == 8 ? T(1e150) : T(1e15))) t = T(0.5) / theta;
            else t = (theta >= T(0) ? T(1) : T(-1)) / (fabs(theta) + sqrt(theta * theta + T(1)));
            c = T(1) / sqrt(t * t + T(1));
            s = t * c;
          }
        }
        cs[2 * k] = c;
        cs[2 * k + 1] = s;
        pq[2 * k] = p;
        pq[2 * k + 1] = q;
      }
      __syncthreads();
      // rows: A <- J^T A
      for (int e = threadIdx.x; e < half * n; e += ET) {
        const int k = e / n, j = e % n;
        const int p = pq[2 * k], q = pq[2 * k + 1];
        if (q >= n) continue;
        const T c = cs[2 * k], s = cs[2 * k + 1];
        if (s == T(0)) continue;
        const T ap = A[p * ld + j], aq = A[q * ld + j];
        A[p * ld + j] = c * ap - s * aq;
        A[q * ld + j] = s * ap + c * aq;
      }
      __syncthreads();
      // columns: A <- A J ; V <- V J
      for (int e = threadIdx.x; e < half * n; e += ET) {
        const int k = e / n, i = e % n;
        const int p = pq[2 * k], q = pq[2 * k + 1];
        if (q >= n) continue;
        const T c = cs[2 * k], s = cs[2 * k + 1];
        if (s == T(0)) continue;
        const T ap = A[i * ld + p], aq = A[i * ld + q];
        A[i * ld + p] = c * ap - s * aq;
        A[i * ld + q] = s * ap + c * aq;
        const T vp = V[i * ld + p], vq = V[i * ld + q];
        V[i * ld + p] = c * vp - s * vq;
        V[i * ld + q] = s * vp + c * vq;
      }
      __syncthreads();
      // the annihilated pairs are exactly zero
      for (int k = threadIdx.x; k < half; k += ET) {
        const int p = pq[2 * k], q = pq[2 * k + 1];
        if (q < n && cs[2 * k + 1] != T(0)) {
          A[p * ld + q] = T(0);
          A[q * ld + p] = T(0);
        }
      }
      __syncthreads();
    }
  }
  *sweeps_out = sweep;
}

template <typename T>
__global__ void __launch_bounds__(ET) k_syevd(int n, T* uall, T* lamall, T* wsall, int32_t* info, bool in_smem) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ T red[ET / 32];
  __shared__ int order[EN];
  const int64_t b = blockIdx.x;
  T* u = uall + b * (int64_t)n * n;
  T* lam = lamall + b * (int64_t)n;
  T *A, *V;
  int ld;
  const int npairs = (n + 1) / 2;
  T* cs = reinterpret_cast<T*>(smem_raw) + (in_smem ? 2 * EN * (EN + 1) : 0);
  int* pq = reinterpret_cast<int*>(cs + 2 * npairs);
  if (in_smem) {
    A = reinterpret_cast<T*>(smem_raw);
    V = A + EN * (EN + 1);
    ld = EN + 1;
  } else {
    A = wsall + b * (int64_t)2 * n * n;
    V = A + (int64_t)n * n;
    ld = n;
  }
  for (int e = threadIdx.x; e < n * n; e += ET) A[(e / n) * ld + e % n] = u[e];
  __syncthreads();
  // symmetry precheck
  T mabs = T(0), masym = T(0);
  for (int e = threadIdx.x; e < n * n; e += ET) {
    const int i = e / n, j = e % n;
    const T v = A[i * ld + j];
    if (fabs(v) > mabs) mabs = fabs(v);
    if (j > i) masym = fmax(masym, fabs(v - A[j * ld + i]));
  }
  mabs = bmax(mabs, red);
  masym = bmax(masym, red);
  if (masym > Num<T>::sym_rtol * (mabs > T(0) ? mabs : T(1))) {
    if (threadIdx.x == 0) record_failure(info, b, DLA_ERR_ASYMMETRIC, 0);
    return;
  }
  if (n == 1) {
    if (threadIdx.x == 0) {
      lam[0] = u[0];
      u[0] = T(1);
    }
    return;
  }
  // exact power-of-two pre-scaling; symmetrize from the lower triangle
  int ex = 0;
  if (mabs > T(0)) frexp(mabs, &ex);
  for (int e = threadIdx.x; e < n * n; e += ET) {
    const int i = e / n, j = e % n;
    if (j <= i) {
      const T v = ldexp(A[i * ld + j], -ex);
      A[i * ld + j] = v;
      A[j * ld + i] = v;
    }
  }
  __syncthreads();
  int sweeps = 0;
  jacobi<T>(n, A, V, ld, cs, pq, red, &sweeps);
  if (sweeps >= MAX_SWEEPS) {
    if (threadIdx.x == 0) record_failure(info, b, DLA_ERR_CONVERGENCE, sweeps);
    return;
  }
  // ascending order of the diagonal (stable: ties keep index order)
  if (n <= EN) {
    for (int i = threadIdx.x; i < n; i += ET) {
      const T di = A[i * ld + i];
      int rank = 0;
      for (int j = 0; j < n; ++j) {
        const T dj = A[j * ld + j];
        rank += (dj < di) || (dj == di && j < i);
      }
      order[rank] = i;
    }
    __syncthreads();
  }
  // U row r = eigenvector order[r] (column of V), sign rule, lambda
  for (int r = threadIdx.x >> 5; r < n; r += ET / 32) {
    const int lane = threadIdx.x & 31;
    int col;
    if (n <= EN) {
      col = order[r];
    } else {  // rank selection without the shared order table
      col = -1;
      for (int i = 0; i < n && col < 0; ++i) {
        const T di = A[i * ld + i];
        int rank = 0;
        for (int j = 0; j < n; ++j) {
          const T dj = A[j * ld + j];
          rank += (dj < di) || (dj == di && j < i);
        }
        if (rank == r) col = i;
      }
    }
    // largest |entry|, first index on ties
    T best = T(-1);
    int kbest = 0;
    for (int k = lane; k < n; k += 32) {
      const T v = fabs(V[k * ld + col]);
      if (v > best) {
        best = v;
        kbest = k;
      }
    }
    for (int o = 16; o; o >>= 1) {
      const T ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int ok = __shfl_xor_sync(0xffffffffu, kbest, o);
      if (ob > best || (ob == best && ok < kbest)) {
        best = ob;
        kbest = ok;
      }
    }
    const T sgn = V[kbest * ld + col] < T(0) ? T(-1) : T(1);
    for (int k = lane; k < n; k += 32) u[(int64_t)r * n + k] = sgn * V[k * ld + col];
    if (lane == 0) lam[r] = ldexp(A[col * ld + col], ex);
  }
}


// ---------------------------------------------------- n <= 64: one pass/round
// The same cyclic Jacobi (round-robin ordering, Rutishauser rotations), with
// each round applied as ONE pass over 2 x 2 blocks: rows {p_a, q_a} x columns
// {p_b, q_b} of A become J_a^T A_blk J_b, so a thread owns every element it
// reads and writes (no row pass / column pass / zeroing pass, 2 barriers per
// round instead of 4).  Only blocks a <= b are computed and mirrored, so A
// stays exactly symmetric.  The eigenvector accumulator is kept transposed
// (Vt = V^T, rotated by rows), which makes the output rows contiguous.
constexpr int SP = 32;                 // max pairs
constexpr int NUB = SP * (SP + 1) / 2;  // upper 2x2 blocks
static_assert(ET == 8 * SP, "Vt pass: 8 threads per pair");

struct BlkTab {  // (a, b), a <= b, packed a << 8 | b
  unsigned short v[NUB];
  constexpr BlkTab() : v() {
    int e = 0;
    for (int a = 0; a < SP; ++a)
      for (int b = a; b < SP; ++b) v[e++] = (unsigned short)(a << 8 | b);
  }
};
__device__ const BlkTab kBlkTab = BlkTab();

// Packed upper triangle of the symmetric A: (i, j), i <= j, at i (129 - i) / 2 + j - i
// (row i starts after rows 0 .. i-1 of lengths 64, 63, ...): 2080 doubles.
// With the transposed eigenvector accumulator (64 x 65) the CTA needs 50 KB,
// so four matrices share an SM (full storage: three).
constexpr int PK = EN * (EN + 1) / 2;
__device__ __forceinline__ int pidx(int i, int j) {
  const int lo = i < j ? i : j, hi = i < j ? j : i;
  return (lo * (2 * EN + 1 - lo)) / 2 + hi - lo;
}

template <typename T>
__global__ void __launch_bounds__(ET, 4) k_syevd_small(int n, T* uall, T* lamall, int32_t* info) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* A = reinterpret_cast<T*>(smem_raw);  // packed upper triangle, PK
  T* Vt = A + PK + (PK & 1);              // EN x (EN+1)
  __shared__ T red[ET / 32];
  __shared__ T cs[2 * SP];
  __shared__ int pq[2 * SP];
  __shared__ unsigned short blk[NUB];
  __shared__ int order[EN];
  constexpr int ld = EN + 1;
  const int64_t b = blockIdx.x;
  T* u = uall + b * (int64_t)n * n;
  T* lam = lamall + b * (int64_t)n;
  const int tid = threadIdx.x;
  const int N = n + (n & 1), half = N / 2;
  for (int e = tid; e < NUB; e += ET) blk[e] = kBlkTab.v[e];
  // symmetry precheck straight from global memory (both triangles)
  T mabs = T(0), masym = T(0);
  for (int e = tid; e < n * n; e += ET) {
    const int i = e / n, j = e % n;
    const T v = u[e];
    if (fabs(v) > mabs) mabs = fabs(v);
    if (j > i) masym = fmax(masym, fabs(v - u[j * n + i]));
  }
  mabs = bmax(mabs, red);
  masym = bmax(masym, red);
  if (masym > Num<T>::sym_rtol * (mabs > T(0) ? mabs : T(1))) {
    if (tid == 0) record_failure(info, b, DLA_ERR_ASYMMETRIC, 0);
    return;
  }
  if (n == 1) {
    if (tid == 0) {
      lam[0] = u[0];
      u[0] = T(1);
    }
    return;
  }
  int ex = 0;
  if (mabs > T(0)) frexp(mabs, &ex);
  // exact power-of-two pre-scaling; the symmetric matrix from the lower triangle
  for (int e = tid; e < PK; e += ET) A[e] = T(0);
  for (int e = tid; e < EN * EN; e += ET) {
    const int i = e / EN, j = e % EN;
    Vt[i * ld + j] = (i == j) ? T(1) : T(0);
  }
  __syncthreads();
  for (int e = tid; e < n * n; e += ET) {
    const int i = e / n, j = e % n;
    if (j <= i) A[pidx(j, i)] = ldexp(u[e], -ex);
  }
  __syncthreads();
  int sweep = 0;
  for (; sweep < MAX_SWEEPS; ++sweep) {
    T off = T(0), dia = T(0);
    for (int e = tid; e < PK; e += ET) {
      // row i of the packed triangle: e in [i (129 - i) / 2, ...)
      int i = (int)((2 * EN + 1 - sqrtf((float)((2 * EN + 1) * (2 * EN + 1) - 8 * e))) * 0.5f);
      while (i > 0 && (i * (2 * EN + 1 - i)) / 2 > e) --i;
      while ((i + 1) * (2 * EN + 1 - (i + 1)) / 2 <= e) ++i;
      const int j = i + e - (i * (2 * EN + 1 - i)) / 2;
      if (i >= n || j >= n) continue;
      const T v = fabs(A[e]);
      if (i != j) off = fmax(off, v);
      else dia = fmax(dia, v);
    }
    off = bmax(off, red);
    dia = bmax(dia, red);
    if (off <= Eps<T>::v * dia || off == T(0)) break;
    for (int r = 0; r < N - 1; ++r) {
      if (tid < half) {
        int p, q;
        rr_pair(N, r, tid, p, q);
        T c = T(1), sn = T(0);
        if (q < n) {
          const T apq = A[pidx(p, q)];
          if (apq != T(0)) {
            // the rotation on the round's serial chain with MUFU-seeded
            // reciprocal / reciprocal-sqrt (two Newton steps each, ~1 ulp)
            // instead of IEEE divide / sqrt sequences
            const T theta = (A[pidx(q, q)] - A[pidx(p, p)]) * Num<T>::rcp_(T(2) * apq);
            T t;
            if (fabs(theta) > (sizeof(T) == 8 ? T(1e150) : T(1e15))) {
              t = T(0.5) * Num<T>::rcp_(theta);
            } else {
              const T r2 = theta * theta + T(1);
              t = (theta >= T(0) ? T(1) : T(-1)) * Num<T>::rcp_(fabs(theta) + r2 * Num<T>::rsqrt_(r2));
            }
            c = Num<T>::rsqrt_(t * t + T(1));
            sn = t * c;
          }
        }
        cs[2 * tid] = c;
        cs[2 * tid + 1] = sn;
        pq[2 * tid] = p;
        pq[2 * tid + 1] = q;
      }
      __syncthreads();
      // A <- J^T A J on the 2x2 blocks {p_a, q_a} x {p_b, q_b}, a <= b (each
      // packed element is owned by exactly one block)
      for (int e = tid; e < NUB; e += ET) {
        const int ba = blk[e] >> 8, bb = blk[e] & 255;
        if (bb >= half) continue;
        const int pa = pq[2 * ba], qa = pq[2 * ba + 1], pb = pq[2 * bb], qb = pq[2 * bb + 1];
        const T ca = cs[2 * ba], sa = cs[2 * ba + 1], cb = cs[2 * bb], sb = cs[2 * bb + 1];
        if (ba == bb) {
          if (sa == T(0)) continue;
          const int ipp = pidx(pa, pa), ipq = pidx(pa, qa), iqq = pidx(qa, qa);
          const T x = A[ipp], y = A[ipq], w = A[iqq];
          const T x1 = ca * x - sa * y, y1 = ca * y - sa * w;
          const T z1 = sa * x + ca * y, w1 = sa * y + ca * w;
          A[ipp] = ca * x1 - sa * y1;
          A[iqq] = sa * z1 + ca * w1;
          A[ipq] = T(0);  // the annihilated pair is exactly zero
          continue;
        }
        if (sa == T(0) && sb == T(0)) continue;
        const int i0 = pidx(pa, pb), i1 = pidx(pa, qb), i2 = pidx(qa, pb), i3 = pidx(qa, qb);
        const T x = A[i0], y = A[i1], z = A[i2], w = A[i3];
        const T x1 = ca * x - sa * z, y1 = ca * y - sa * w;
        const T z1 = sa * x + ca * z, w1 = sa * y + ca * w;
        A[i0] = cb * x1 - sb * y1;
        A[i1] = sb * x1 + cb * y1;
        A[i2] = cb * z1 - sb * w1;
        A[i3] = sb * z1 + cb * w1;
      }
      // Vt <- J^T Vt (rows p, q of Vt = columns of V): a warp per row pair,
      // lanes along contiguous columns (2 wavefronts per access whatever p,
      // q are; the previous 4-pairs-per-warp split collided across rows)
      {
        const int wp = tid >> 5, lane = tid & 31;
        for (int k = wp; k < half; k += ET / 32) {
          const T sn = cs[2 * k + 1];
          if (sn == T(0)) continue;
          const T c = cs[2 * k];
          T* vp = Vt + pq[2 * k] * ld;
          T* vq = Vt + pq[2 * k + 1] * ld;
#pragma unroll
          for (int v = 0; v < EN / 32; ++v) {
            const int i = lane + 32 * v;
            const T a0 = vp[i], a1 = vq[i];
            vp[i] = c * a0 - sn * a1;
            vq[i] = sn * a0 + c * a1;
          }
        }
      }
      __syncthreads();
    }
  }
  if (sweep >= MAX_SWEEPS) {
    if (tid == 0) record_failure(info, b, DLA_ERR_CONVERGENCE, sweep);
    return;
  }
  for (int i = tid; i < n; i += ET) {
    const T di = A[pidx(i, i)];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const T dj = A[pidx(j, j)];
      rank += (dj < di) || (dj == di && j < i);
    }
    order[rank] = i;
  }
  __syncthreads();
  for (int r = tid >> 5; r < n; r += ET / 32) {
    const int lane = tid & 31;
    const int col = order[r];
    const T* vr = Vt + col * ld;
    T best = T(-1);
    int kbest = 0;
    for (int k = lane; k < n; k += 32) {
      const T v = fabs(vr[k]);
      if (v > best) {
        best = v;
        kbest = k;
      }
    }
    for (int o = 16; o; o >>= 1) {
      const T ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int ok = __shfl_xor_sync(0xffffffffu, kbest, o);
      if (ob > best || (ob == best && ok < kbest)) {
        best = ob;
        kbest = ok;
      }
    }
    const T sgn = vr[kbest] < T(0) ? T(-1) : T(1);
    for (int k = lane; k < n; k += 32) u[(int64_t)r * n + k] = sgn * vr[k];
    if (lane == 0) lam[r] = ldexp(A[pidx(col, col)], ex);
  }
}

template <typename T>
__global__ void k_gap(int64_t batch, int64_t n, MatB<T> w, const T* lambdabar, const T* lambda, T eps_gap) {
  const int64_t total = batch * n * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t / (n * n), r = t % (n * n), i = r / n, j = r % n;
    if (j > i) continue;
    T* wij = w.at(b, i, j);
    if (i == j) {
      *wij = lambdabar[b * n + i];
      continue;
    }
    T* wji = w.at(b, j, i);
    const T gap = fmax(lambda[b * n + i] - lambda[b * n + j], eps_gap);
    const T y = (*wij - *wji) / (T(2) * gap);
    *wij = y;
    *wji = y;
  }
}

template <typename T>
__global__ void k_sym_into(int64_t batch, int64_t n, MatB<const T> w, MatB<T> out) {
  const int64_t total = batch * n * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t / (n * n), r = t % (n * n), i = r / n, j = r % n;
    const int64_t hi = i > j ? i : j, lo = i > j ? j : i;
    *out.at(b, i, j) = (*w.at(b, hi, lo) + *w.at(b, lo, hi)) / T(2);
  }
}

}  // namespace

template <typename T>
size_t syevd_ws_bytes(int64_t batch, int64_t n, bool backward) {
  if (backward) return sizeof(T) * (size_t)(batch * n * n);
  return n <= EN ? 0 : sizeof(T) * (size_t)(batch * 2 * n * n);
}

template <typename T>
dla_status syevd_fwd(const Ctx& c, int64_t batch, int64_t n, T* u, T* lambda, void* ws) {
  const bool sm = n <= EN;
  if (sm) {
    const size_t smem = sizeof(T) * (PK + (PK & 1) + EN * (EN + 1));
    ensure_smem_attr(k_syevd_small<T>, smem);
    k_syevd_small<T><<<(unsigned)batch, ET, smem, c.stream>>>((int)n, u, lambda, c.info);
    DLAB_LAUNCH_CHECK();
    return DLA_OK;
  }
  if (!ws) return DLA_ERR_WORKSPACE;
  const int64_t npairs = (n + 1) / 2;
  const size_t smem = (sm ? sizeof(T) * 2 * EN * (EN + 1) : 0) + npairs * 2 * (sizeof(T) + sizeof(int));
  if (smem > 200 * 1024) return DLA_ERR_SHAPE;  // n > ~8000: out of the supported range
  ensure_smem_attr(k_syevd<T>, smem);
  k_syevd<T><<<(unsigned)batch, ET, smem, c.stream>>>((int)n, u, lambda, static_cast<T*>(ws), c.info, sm);
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}

template <typename T>
dla_status syevd_gap_kernel(const Ctx& c, int64_t batch, int64_t n, MatB<T> w, const T* lambdabar, const T* lambda,
                            T eps_gap) {
  k_gap<T><<<blocks_for(batch * n * n, 256), 256, 0, c.stream>>>(batch, n, w, lambdabar, lambda, eps_gap);
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}

template <typename T>
dla_status ew_sym_into(const Ctx& c, int64_t batch, int64_t n, MatB<const T> w, MatB<T> out) {
  k_sym_into<T><<<blocks_for(batch * n * n, 256), 256, 0, c.stream>>>(batch, n, w, out);
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}

#define INST(T)                                                                                        \
  template size_t syevd_ws_bytes<T>(int64_t, int64_t, bool);                                           \
  template dla_status syevd_fwd<T>(const Ctx&, int64_t, int64_t, T*, T*, void*);                       \
  template dla_status syevd_gap_kernel<T>(const Ctx&, int64_t, int64_t, MatB<T>, const T*, const T*, T); \
  template dla_status ew_sym_into<T>(const Ctx&, int64_t, int64_t, MatB<const T>, MatB<T>);
INST(double)
INST(float)

}  // namespace dlab
