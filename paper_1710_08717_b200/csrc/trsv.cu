// Narrow triangular solve: op(T)^{-1} applied to <= 8 vectors (the GP
// driver's L z = y and L^T s = zbar, dl/models.hpp:99 and its trsm pullback,
// dl/adjoints.hpp:136-137).  A recursive solve would be 2 n/64 dependent
// launches of almost no work each; here ONE launch covers the whole solve:
// CTA i owns block row i (64 rows), streams the blocks S(i, j), j < i, of the
// triangle as soon as block j is published (per-block ready flags in global
// memory, release/acquire via __threadfence), then solves its diagonal block
// with a warp per vector.  The triangle is read once (n^2/2 elements), in
// parallel across all CTAs: HBM-bound instead of launch-bound.
//
// Semantics are trsm_inplace's (dl/blas.hpp:307-395): S is op(T) (left) or
// op(T)^T (right, vectors are rows of X); an upper S is handled by reversing
// the row order so the kernel always runs a forward substitution.
#include "chol64.cuh"
#include "common.cuh"
#include "ops.cuh"

namespace dlab {
namespace {

constexpr int BR = 64;   // rows per block
constexpr int NR = 8;    // max vectors
constexpr int TT = 256;  // threads per CTA
constexpr int SLD = BR + 1;

struct TrsvGeo {
  int64_t nt, nblk, nvec;
  bool right, s_tt, slower;
};

// physical index of logical row r (forward-substitution order)
__device__ __forceinline__ int64_t phys(const TrsvGeo& g, int64_t r) { return g.slower ? r : g.nt - 1 - r; }

template <typename T>
__device__ __forceinline__ T s_at(const TrsvGeo& g, MatB<const T> t, int64_t b, int64_t r, int64_t c) {
  const int64_t pr = phys(g, r), pc = phys(g, c);
  return g.s_tt ? *t.at(b, pc, pr) : *t.at(b, pr, pc);
}

template <typename T>
__device__ __forceinline__ T* x_at(const TrsvGeo& g, MatB<T> x, int64_t b, int64_t r, int v) {
  return g.right ? x.at(b, v, phys(g, r)) : x.at(b, phys(g, r), v);
}

template <typename T>
__global__ void __launch_bounds__(TT) k_trsv(TrsvGeo g, MatB<const T> t, MatB<T> x, T alpha, int* flags,
                                             const int32_t* skip) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* SP = reinterpret_cast<T*>(smem_raw);  // diagonal block, then partial sums P[4][NR][BR]
  T* Xi = SP + BR * SLD;                   // inverse of the diagonal block, vector-major: Xi[v*SLD + r] = Sinv(r, v)
  T* rd = Xi + BR * SLD;
  T(*Y)[BR] = reinterpret_cast<T(*)[BR]>(rd + BR);  // [NR][BR]
  T* S = SP;
  const int64_t b = blockIdx.x / g.nblk, i = blockIdx.x % g.nblk;
  if (slice_failed(skip, b)) return;
  const int tid = threadIdx.x;
  const int64_t r0 = i * BR;
  const int rows = (int)min((int64_t)BR, g.nt - r0);
  const int nv = (int)g.nvec;
  // Off the critical path (before waiting on any earlier block): invert the
  // diagonal block, so the dependent step is a 64 x 64 matrix-vector product
  // instead of a 64-step substitution.
  for (int e = tid; e < BR * BR; e += TT) {
    const int rr = e / BR, c = e % BR;
    S[rr * SLD + c] = (rr < rows && c <= rr) ? s_at(g, t, b, r0 + rr, r0 + c) : (rr == c ? T(1) : T(0));
    Xi[rr * SLD + c] = (rr == c) ? T(1) : T(0);
  }
  __syncthreads();
  if (tid < BR) rd[tid] = T(1) / S[tid * SLD + tid];
  __syncthreads();
  blocked_fwd_subst<T>(S, Xi, rd, BR, BR);
  // (row, 16-column chunk) per thread; lanes walk contiguous memory of T
  const int r = g.s_tt ? tid % BR : tid / 4, cq = g.s_tt ? tid / BR : tid % 4;
  T part[NR];
#pragma unroll
  for (int v = 0; v < NR; ++v) part[v] = T(0);
  // off-diagonal blocks j < i, in publication order
  for (int64_t j = 0; j < i; ++j) {
    // the triangle's block (i, j) does not depend on block j's result:
    // fetch it before waiting for the flag
    T s[16];
#pragma unroll
    for (int cc = 0; cc < 16; ++cc) s[cc] = (r < rows) ? s_at(g, t, b, r0 + r, j * BR + cq * 16 + cc) : T(0);
    if (tid == 0) {
      volatile int* f = flags + b * g.nblk + j;
      while (*f == 0) __nanosleep(32);
      __threadfence();
    }
    __syncthreads();
    for (int e = tid; e < nv * BR; e += TT) {
      const int v = e / BR, c = e % BR;
      Y[v][c] = __ldcg(x_at(g, x, b, j * BR + c, v));  // L2: written by another CTA
    }
    __syncthreads();
#pragma unroll
    for (int cc = 0; cc < 16; ++cc) {
      const int c = cq * 16 + cc;
#pragma unroll
      for (int v = 0; v < NR; ++v)
        if (v < nv) part[v] += s[cc] * Y[v][c];
    }
  }
  // right-hand side: alpha x_i minus the four column-chunk partial sums
#pragma unroll
  for (int v = 0; v < NR; ++v) SP[(cq * NR + v) * BR + r] = part[v];
  __syncthreads();
  for (int e = tid; e < NR * BR; e += TT) {
    const int v = e / BR, rr = e % BR;
    T acc = T(0);
    if (v < nv && rr < rows)
      acc = alpha * *x_at(g, x, b, r0 + rr, v) - (SP[(0 * NR + v) * BR + rr] + SP[(1 * NR + v) * BR + rr] +
                                                   SP[(2 * NR + v) * BR + rr] + SP[(3 * NR + v) * BR + rr]);
    Y[v][rr] = acc;
  }
  __syncthreads();
  // y_i = S_ii^{-1} rhs: thread (row, vector) dots the lower row of S^{-1}
  for (int e = tid; e < nv * BR; e += TT) {
    const int v = e / BR, rr = e % BR;
    if (rr >= rows) continue;
    T acc = T(0);
    for (int c = 0; c <= rr; ++c) acc += Xi[c * SLD + rr] * Y[v][c];
    *x_at(g, x, b, r0 + rr, v) = acc;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) atomicExch(flags + b * g.nblk + i, 1);
}

}  // namespace

template <typename T>
bool trsv_eligible(int64_t nt, int64_t nvec) {
  return nt > 64 && nvec >= 1 && nvec <= NR;
}

template <typename T>
dla_status trsv(const Ctx& c, int64_t batch, int64_t m, int64_t n, MatB<const T> t, MatB<T> x, bool right, bool trans,
                bool lower, T alpha) {
  const bool op_lower = (lower != trans);
  TrsvGeo g;
  g.nt = right ? n : m;
  g.nvec = right ? m : n;
  g.nblk = (g.nt + BR - 1) / BR;
  g.right = right;
  g.s_tt = right ? !trans : trans;
  g.slower = right ? !op_lower : op_lower;
  Scratch flags(sizeof(int) * (size_t)(batch * g.nblk), c.stream);
  if (!flags.p) return DLA_ERR_CUDA;
  if (cudaMemsetAsync(flags.p, 0, sizeof(int) * batch * g.nblk, c.stream) != cudaSuccess) return DLA_ERR_CUDA;
  const size_t sm = sizeof(T) * (2 * BR * SLD + BR + NR * BR);
  static bool once = false;
  if (!once) {
    cudaFuncSetAttribute(k_trsv<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    once = true;
  }
  k_trsv<T><<<(unsigned)(batch * g.nblk), TT, sm, c.stream>>>(g, t, x, alpha, flags.as<int>(), c.info);
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}

template bool trsv_eligible<double>(int64_t, int64_t);
template bool trsv_eligible<float>(int64_t, int64_t);
template dla_status trsv<double>(const Ctx&, int64_t, int64_t, int64_t, MatB<const double>, MatB<double>, bool, bool,
                                 bool, double);
template dla_status trsv<float>(const Ctx&, int64_t, int64_t, int64_t, MatB<const float>, MatB<float>, bool, bool,
                                bool, float);

}  // namespace dlab
