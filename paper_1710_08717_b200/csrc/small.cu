// Fused small-matrix kernels (n <= 64): one CTA per matrix, the whole
// operator chain in shared memory, one HBM read of each input and one write
// of each output.  This is the batched small-n regime of the north star
// (C1: batch 64 x 32^2; any batch x n <= 64).
//
//   potrf fwd : symmetry precheck (dl/cholesky.hpp:19-25) + Cholesky
//               (dl/cholesky.hpp:35-72) + tril / transpose (:71, :85-86).
//   potrf bwd : Abar = 1/2 sym(L^-T copyltu(L^T Lbar) L^-1)
//               (dl/adjoints.hpp:175-191), upper variant by transposition.
#include "chol64.cuh"
#include "common.cuh"
#include "ops.cuh"

namespace dlab {
namespace {

constexpr int SN = 64;
constexpr int SLD = SN + 1;

template <typename T>
__device__ T block_max(T v, T* red) {
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  T r = red[0];
  for (int k = 1; k < (int)(blockDim.x >> 5); ++k) r = fmax(r, red[k]);
  return r;
}

template <typename T>
__global__ void __launch_bounds__(256) k_potrf_small(int n, MatB<T> a, bool lower, int32_t* info) {
  __shared__ T S[SN * SLD];
  __shared__ T red[8];
  __shared__ int flag;
  static_assert(SLD == CH_LD, "shared layout");
  const int64_t b = blockIdx.x;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) S[(e / n) * SLD + e % n] = *a.at(b, e / n, e % n);
  __syncthreads();
  // symmetry precheck: max|a_ij - a_ji| <= rtol * max|a|  (NaN ignored as in max_abs)
  T mabs = T(0), masym = T(0);
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e % n;
    const T v = S[i * SLD + j];
    if (fabs(v) > mabs) mabs = fabs(v);
    if (j > i) {
      const T d = fabs(v - S[j * SLD + i]);
      if (d > masym) masym = d;
    }
  }
  mabs = block_max(mabs, red);
  masym = block_max(masym, red);
  if (masym > Num<T>::sym_rtol * (mabs > T(0) ? mabs : T(1))) {
    if (threadIdx.x == 0) record_failure(info, b, DLA_ERR_ASYMMETRIC, 0);
    return;
  }
  const int failed = chol_smem64<T>(S, n, &flag);
  if (failed >= 0) {
    if (threadIdx.x == 0) record_failure(info, b, DLA_ERR_NOT_SPD, failed);
    return;
  }
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e % n;
    T v;
    if (lower) v = j <= i ? S[i * SLD + j] : T(0);
    else v = i <= j ? S[j * SLD + i] : T(0);
    *a.at(b, i, j) = v;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_potrf_bwd_small(int n, MatB<T> abar, MatB<const T> lbar, MatB<const T> l,
                                                         bool lower) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* L = reinterpret_cast<T*>(smem_raw);
  T* G = L + SN * SLD;  // Lbar (lower view)
  T* W = G + SN * SLD;
  const int64_t b = blockIdx.x;
  // Upper variant: L = R^T, Lbar = Rbar^T (dl/adjoints.hpp:183-188 is the
  // transpose of the lower composition).
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e % n;
    T lv = lower ? *l.at(b, i, j) : *l.at(b, j, i);
    T gv = lower ? *lbar.at(b, i, j) : *lbar.at(b, j, i);
    L[i * SLD + j] = j <= i ? lv : T(0);
    G[i * SLD + j] = gv;
  }
  __syncthreads();
  // Phi = copyltu(L^T Lbar): Phi_ij (i >= j) = sum_{k >= i} L_ki Lbar_kj
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e % n;
    if (j > i) continue;
    T acc = T(0);
    for (int k = i; k < n; ++k) acc += L[k * SLD + i] * G[k * SLD + j];
    W[i * SLD + j] = acc;
    W[j * SLD + i] = acc;
  }
  __syncthreads();
  // X = L^{-T} Phi: back substitution per column
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    for (int i = n - 1; i >= 0; --i) {
      T acc = W[i * SLD + j];
      for (int k = i + 1; k < n; ++k) acc -= L[k * SLD + i] * W[k * SLD + j];
      W[i * SLD + j] = acc / L[i * SLD + i];
    }
  }
  __syncthreads();
  // Y = X L^{-1}: per row, y_k = (x_k - sum_{j>k} y_j L_jk) / L_kk, k descending
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    T* wr = W + r * SLD;
    for (int k = n - 1; k >= 0; --k) {
      T acc = wr[k];
      for (int j = k + 1; j < n; ++j) acc -= wr[j] * L[j * SLD + k];
      wr[k] = acc / L[k * SLD + k];
    }
  }
  __syncthreads();
  // Abar = sym(Y / 2), exactly symmetric
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e % n;
    const T hi = W[i * SLD + j] * T(0.5), hj = W[j * SLD + i] * T(0.5);
    *abar.at(b, i, j) = (i == j) ? hi : (hi + hj) / T(2);
  }
}

}  // namespace

template <typename T>
bool potrf_small_eligible(int64_t n) {
  return n >= 1 && n <= SN;
}

template <typename T>
dla_status potrf_small(const Ctx& c, int64_t batch, int64_t n, MatB<T> a, bool lower) {
  k_potrf_small<T><<<(unsigned)batch, 256, 0, c.stream>>>((int)n, a, lower, c.info);
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}

template <typename T>
dla_status potrf_bwd_small(const Ctx& c, int64_t batch, int64_t n, MatB<T> abar, MatB<const T> lbar,
                           MatB<const T> l, bool lower) {
  const size_t sm = sizeof(T) * 3 * SN * SLD;
  static bool once = false;
  if (!once) {
    cudaFuncSetAttribute(k_potrf_bwd_small<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    once = true;
  }
  k_potrf_bwd_small<T><<<(unsigned)batch, 256, sm, c.stream>>>((int)n, abar, lbar, l, lower);
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}

#define INST(T)                                                                                     \
  template bool potrf_small_eligible<T>(int64_t);                                                   \
  template dla_status potrf_small<T>(const Ctx&, int64_t, int64_t, MatB<T>, bool);                  \
  template dla_status potrf_bwd_small<T>(const Ctx&, int64_t, int64_t, MatB<T>, MatB<const T>, MatB<const T>, bool);
INST(double)
INST(float)

}  // namespace dlab
