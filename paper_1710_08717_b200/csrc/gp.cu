// Gaussian-process driver kernels either side of the Cholesky path (SURVEY
// §8f row 1): the RBF kernel build and its pullback, fused into one HBM pass
// each instead of the reference tape's ~15 elementwise n x n nodes.
//
// Forward  (dl/models.hpp:50-65, :95-98):
//   dist_ij = (s_i + s_j) - 2 G_ij,   s = sum_rows(x∘x),  G = syrk(x)
//   A_ij    = sigma2 * exp(-(dist_ij / (2 ell2))) + lam * I_ij
// Backward (tape pullbacks dl/tape.hpp:930-1036 composed by hand), given
// Abar = dphi/dA (symmetric):
//   dsigma2 = sum Abar∘E,   dlam = tr(Abar),
//   d(2 ell2) = sum Nbar∘D / (2 ell2),  Nbar = Abar sigma2 E,  D = dist/(2 ell2)
//   xbar_i  = 4 sum_j W_ij (x_i - x_j),  W = -Nbar / (2 ell2)   (syrk + square
//             + tile pullbacks with W symmetric)
//   returned as gradients w.r.t. the log-parameters (dl/models.hpp:126-131).
// Reductions are two-level with fixed order (no atomics): run-to-run
// deterministic.
#include "common.cuh"

namespace dlab {
namespace {

constexpr int RT = 256;
constexpr int MAXD = 32;

// s_i = sum_f x_if^2 (sequential f, like SumRows)
__global__ void k_rowsq(int64_t batch, int64_t n, int64_t d, const double* x, double* s) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < batch * n; t += (int64_t)gridDim.x * blockDim.x) {
    const double* xi = x + t * d;
    double acc = 0.0;
    for (int64_t f = 0; f < d; ++f) acc += xi[f] * xi[f];
    s[t] = acc;
  }
}

__device__ __forceinline__ double gram(const double* xa, const double* xb, int64_t d) {
  double acc = 0.0;
  for (int64_t f = 0; f < d; ++f) acc += xa[f] * xb[f];
  return acc;
}

// One CTA per (slice, row i); threads sweep j.  Writes full rows (coalesced).
__global__ void __launch_bounds__(RT) k_rbf_fwd(int64_t n, int64_t d, const double* x, const double* s, double sigma2,
                                                double two_ell2, double lam, double* a) {
  __shared__ double xi_s[MAXD];
  const int64_t row = blockIdx.x;  // b * n + i
  const int64_t b = row / n, i = row % n;
  const double* xb = x + b * n * d;
  if (threadIdx.x < d) xi_s[threadIdx.x] = xb[i * d + threadIdx.x];
  __syncthreads();
  const double si = s[b * n + i];
  double* arow = a + b * n * n + i * n;
  for (int64_t j = threadIdx.x; j < n; j += RT) {
    // G_ij from the (max, min) pair: syrk fills the lower triangle and mirrors
    const double g = gram(xi_s, xb + j * d, d);
    const double dist = (si + s[b * n + j]) - 2.0 * g;
    double v = sigma2 * exp(-(dist / two_ell2));
    if (j == i) v += lam;
    arow[j] = v;
  }
}

// Per (slice, row-block) partial sums + xbar rows.
__global__ void __launch_bounds__(RT) k_rbf_bwd(int64_t n, int64_t d, const double* x, const double* s, double sigma2,
                                                double two_ell2, const double* abar, double* xbar, double* part) {
  __shared__ double xi_s[MAXD];
  __shared__ double red[3][RT / 32];
  __shared__ double xred[RT / 32][MAXD];
  const int64_t row = blockIdx.x;
  const int64_t b = row / n, i = row % n;
  const double* xb = x + b * n * d;
  if (threadIdx.x < d) xi_s[threadIdx.x] = xb[i * d + threadIdx.x];
  __syncthreads();
  const double si = s[b * n + i];
  const double* ar = abar + b * n * n + i * n;
  double ps = 0.0, pl = 0.0, pe = 0.0;
  double xacc[MAXD];
  for (int f = 0; f < d; ++f) xacc[f] = 0.0;
  for (int64_t j = threadIdx.x; j < n; j += RT) {
    const double* xj = xb + j * d;
    const double g = gram(xi_s, xj, d);
    const double dist = (si + s[b * n + j]) - 2.0 * g;
    const double D = dist / two_ell2;
    const double E = exp(-D);
    const double kb = ar[j];
    ps += kb * E;                   // sigma2-bar
    const double nb = kb * sigma2 * E;
    pe += nb * D;                   // (2 ell2)-bar * (2 ell2)
    if (j == i) pl += kb;           // lam-bar (trace)
    if (xbar) {
      const double w = -nb / two_ell2;  // dist-bar
      for (int f = 0; f < d; ++f) xacc[f] += w * (xi_s[f] - xj[f]);
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int o = 16; o; o >>= 1) {
    ps += __shfl_xor_sync(0xffffffffu, ps, o);
    pl += __shfl_xor_sync(0xffffffffu, pl, o);
    pe += __shfl_xor_sync(0xffffffffu, pe, o);
  }
  if (lane == 0) {
    red[0][warp] = ps;
    red[1][warp] = pl;
    red[2][warp] = pe;
  }
  if (xbar) {
    for (int f = 0; f < d; ++f) {
      double v = xacc[f];
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) xred[warp][f] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double acc = 0.0;
    for (int w = 0; w < RT / 32; ++w) acc += red[threadIdx.x][w];
    part[row * 3 + threadIdx.x] = acc;
  }
  if (xbar && threadIdx.x < d) {
    double acc = 0.0;
    for (int w = 0; w < RT / 32; ++w) acc += xred[w][threadIdx.x];
    xbar[(b * n + i) * d + threadIdx.x] = 4.0 * acc;
  }
}

// Tiled variants for a compile-time feature count D (the C2 workload has
// d = 8): a CTA owns 16 rows; warp w handles rows w and w + 8, its lanes
// stride the columns, so every A / Abar access of a warp is one contiguous
// 256-byte row segment; x_j tiles are staged in shared memory once per CTA.
constexpr int TRW = 16;   // rows per CTA
constexpr int TCJ = 128;  // columns per staged tile
constexpr int TCS = 512;  // columns per CTA (grid = rows/16 x n/512: enough CTAs to fill 148 SMs at n = 4096)

__host__ __device__ inline int64_t rbf_splits(int64_t n) { return (n + TCS - 1) / TCS; }

template <int D, bool FWD>
__global__ void __launch_bounds__(256) k_rbf_tiled(int64_t n, const double* x, const double* s, double sigma2,
                                                   double two_ell2, double lam, double* a, const double* abar,
                                                   double* xpart, double* part) {
  __shared__ double xs[TCJ][D + 1];  // odd row stride: lane-strided reads are conflict-free
  __shared__ double ss[TCJ];
  const int64_t rb = (n + TRW - 1) / TRW, splits = rbf_splits(n);
  const int64_t sp = blockIdx.x % splits, blk = blockIdx.x / splits;
  const int64_t b = blk / rb, i0 = (blk % rb) * TRW;
  const int64_t jbeg = sp * TCS, jend = min(n, jbeg + TCS);
  const double inv2l = 1.0 / two_ell2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* xb = x + b * n * D;
  const double* sb = s + b * n;
  int64_t ii[2] = {i0 + warp, i0 + warp + 8};
  double xi[2][D], si[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const bool ok = ii[q] < n;
#pragma unroll
    for (int f = 0; f < D; ++f) xi[q][f] = ok ? xb[ii[q] * D + f] : 0.0;
    si[q] = ok ? sb[ii[q]] : 0.0;
  }
  double ps[2] = {0, 0}, pl[2] = {0, 0}, pe[2] = {0, 0}, xacc[2][D];
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int f = 0; f < D; ++f) xacc[q][f] = 0.0;
  for (int64_t j0 = jbeg; j0 < jend; j0 += TCJ) {
    __syncthreads();
    for (int e = threadIdx.x; e < TCJ * D; e += 256) {
      const int64_t j = j0 + e / D;
      xs[e / D][e % D] = j < jend ? xb[j * D + e % D] : 0.0;
    }
    for (int e = threadIdx.x; e < TCJ; e += 256) ss[e] = (j0 + e < jend) ? sb[j0 + e] : 0.0;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < TCJ / 32; ++k) {
      const int jj = lane + 32 * k;
      const int64_t j = j0 + jj;
      if (j >= jend) continue;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int64_t i = ii[q];
        if (i >= n) continue;
        double g = 0.0;
#pragma unroll
        for (int f = 0; f < D; ++f) g += xi[q][f] * xs[jj][f];
        const double dist = (si[q] + ss[jj]) - 2.0 * g;
        const double Dv = dist * inv2l;
        const double E = exp(-Dv);
        double* ap = a + (b * n + i) * n + j;
        if constexpr (FWD) {
          double v = sigma2 * E;
          if (j == i) v += lam;
          *ap = v;
        } else {
          const double kb = abar[(b * n + i) * n + j];
          ps[q] += kb * E;
          const double nb = kb * sigma2 * E;
          pe[q] += nb * Dv;
          if (j == i) pl[q] += kb;
          if (xpart) {
            const double w = -nb * inv2l;
#pragma unroll
            for (int f = 0; f < D; ++f) xacc[q][f] += w * (xi[q][f] - xs[jj][f]);
          }
        }
      }
    }
  }
  if constexpr (!FWD) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      double v0 = ps[q], v1 = pl[q], v2 = pe[q];
      for (int o = 16; o; o >>= 1) {
        v0 += __shfl_xor_sync(0xffffffffu, v0, o);
        v1 += __shfl_xor_sync(0xffffffffu, v1, o);
        v2 += __shfl_xor_sync(0xffffffffu, v2, o);
      }
      double xv[D];
#pragma unroll
      for (int f = 0; f < D; ++f) {
        double t = xacc[q][f];
        for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        xv[f] = t;
      }
      const int64_t i = ii[q];
      if (lane == 0 && i < n) {  // per-(row, column split) partials, reduced in a fixed order later
        double* pp = part + ((b * n + i) * splits + sp) * 3;
        pp[0] = v0;
        pp[1] = v1;
        pp[2] = v2;
        if (xpart)
#pragma unroll
          for (int f = 0; f < D; ++f) xpart[((b * n + i) * splits + sp) * D + f] = xv[f];
      }
    }
  }
}

template <bool FWD>
bool launch_tiled(int64_t d, int64_t batch, int64_t n, const double* x, const double* s, double sigma2,
                  double two_ell2, double lam, double* a, const double* abar, double* xbar, double* part,
                  cudaStream_t st) {
  const unsigned grid = (unsigned)(batch * ((n + TRW - 1) / TRW) * rbf_splits(n));
#define DLAB_RBF_CASE(DD)                                                                                  \
  case DD:                                                                                                 \
    k_rbf_tiled<DD, FWD><<<grid, 256, 0, st>>>(n, x, s, sigma2, two_ell2, lam, a, abar, xbar, part);      \
    return true;
  switch (d) {
    DLAB_RBF_CASE(1)
    DLAB_RBF_CASE(2)
    DLAB_RBF_CASE(3)
    DLAB_RBF_CASE(4)
    DLAB_RBF_CASE(8)
    DLAB_RBF_CASE(16)
    default:
      return false;
  }
#undef DLAB_RBF_CASE
}

// xbar rows from the per-split partials (fixed split order).
__global__ void k_rbf_xbar(int64_t rows, int64_t splits, int d, const double* xpart, double* xbar) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows * d; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / d, f = t % d;
    double acc = 0.0;
    for (int64_t sp = 0; sp < splits; ++sp) acc += xpart[(r * splits + sp) * d + f];
    xbar[t] = 4.0 * acc;
  }
}

// Fixed-order finalization per slice: grads w.r.t. (log sigma2, log ell2, log lam).
constexpr int FT = 1024;  // one CTA per slice: wide, so the partial sweep is not a serial chain
__global__ void k_rbf_finalize(int64_t batch, int64_t n, int64_t splits, const double* part, double sigma2,
                               double ell2, double lam, double two_ell2, double* grads) {
  const int64_t b = blockIdx.x;
  __shared__ double red[3][FT];
  double a0 = 0, a1 = 0, a2 = 0;
#pragma unroll 4
  for (int64_t i = threadIdx.x; i < n; i += FT)
    for (int64_t sp = 0; sp < splits; ++sp) {
      const double* pp = part + ((b * n + i) * splits + sp) * 3;
      a0 += pp[0];
      a1 += pp[1];
      a2 += pp[2];
    }
  red[0][threadIdx.x] = a0;
  red[1][threadIdx.x] = a1;
  red[2][threadIdx.x] = a2;
  __syncthreads();
  for (int st = FT / 2; st; st >>= 1) {
    if (threadIdx.x < st)
      for (int k = 0; k < 3; ++k) red[k][threadIdx.x] += red[k][threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double sbar = red[0][0], lbar = red[1][0];
    const double two_ell2_bar = red[2][0] / two_ell2;  // -sum(Dbar∘D)/(2 ell2), Dbar = -Nbar
    const double ell2_bar = 2.0 * two_ell2_bar;
    grads[b * 3 + 0] = sbar * sigma2;
    grads[b * 3 + 1] = ell2_bar * ell2;
    grads[b * 3 + 2] = lbar * lam;
  }
}

// ---- symmetric pullback straight from Z (the GP step's fused tail) ----
// potrf_backward's last two products leave Z = L^-T P' L^-1 and the operator
// would materialize Abar = 1/2 (Z + Z^T) (one more 3 n^2 HBM pass) before the
// RBF pullback reads Abar back.  Here one CTA takes a 64 x 64 tile PAIR
// (I, J), I >= J, of the symmetric problem: it reads Z(I,J) and Z(J,I),
// forms Abar_ij = 0.5 (Z_ij + Z_ji) exactly as that add-transpose pass does
// (same bits), evaluates the RBF entry ONCE for (i,j) and (j,i) (they are the
// same bits: the distance formula commutes), and contributes the pullback of
// both: scalar sums twice, xbar rows of I (sum over j) and of J (sum over i).
// Half the exp work of the row-wise kernel, no Abar pass.  Per-(row, tile)
// xbar partials and per-pair scalar partials are reduced in a fixed order
// afterwards: deterministic.
constexpr int SBT = 64;  // tile
constexpr size_t SYM_SMEM = sizeof(double) * SBT * (SBT + 1);
template <int D>
__global__ void __launch_bounds__(256) k_rbf_bwd_sym(int64_t n, int64_t tiles, int64_t npairs, const double* x,
                                                    const double* s, double sigma2, double two_ell2,
                                                    const double* z, double* xpart, double* part) {
  extern __shared__ double sym_smem[];
  double(*zr)[SBT + 1] = reinterpret_cast<double(*)[SBT + 1]>(sym_smem);  // Z(I,J) -> Abar(I,J) -> W(I,J)
  __shared__ double xI[SBT][D + 1], xJ[SBT][D + 1];
  __shared__ double sI[SBT], sJ[SBT];
  __shared__ double red[3][8];
  const int64_t b = blockIdx.x / npairs, pr = blockIdx.x % npairs;
  int64_t I = (int64_t)((sqrt(8.0 * (double)pr + 1.0) - 1.0) * 0.5);
  while (I * (I + 1) / 2 > pr) --I;
  while ((I + 1) * (I + 2) / 2 <= pr) ++I;
  const int64_t J = pr - I * (I + 1) / 2;
  const bool diag = I == J;
  const int64_t i0 = I * SBT, j0 = J * SBT;
  const double* xb = x + b * n * D;
  const double* sb = s + b * n;
  const double* zb = z + b * n * n;
  const int t = threadIdx.x;
  for (int e = t; e < SBT * D; e += 256) {
    const int r = e / D, f = e % D;
    xI[r][f] = i0 + r < n ? xb[(i0 + r) * D + f] : 0.0;
    xJ[r][f] = j0 + r < n ? xb[(j0 + r) * D + f] : 0.0;
  }
  if (t < SBT) {
    sI[t] = i0 + t < n ? sb[i0 + t] : 0.0;
    sJ[t] = j0 + t < n ? sb[j0 + t] : 0.0;
  }
  for (int e = t; e < SBT * SBT; e += 256) {
    const int r = e >> 6, c = e & 63;
    zr[r][c] = (i0 + r < n && j0 + c < n) ? zb[(i0 + r) * n + j0 + c] : 0.0;
  }
  __syncthreads();
  // Abar_ij = 0.5 (Z_ij + Z_ji) (k_add_transpose's bits): Z(J,I) read by
  // coalesced rows and folded in transposed; every element has one owner
  for (int e = t; e < SBT * SBT; e += 256) {
    const int r = e >> 6, c = e & 63;  // Z(J,I)[r][c] = Z_{i0+c, j0+r}^T partner of (c, r)
    const double zji = (j0 + r < n && i0 + c < n) ? zb[(j0 + r) * n + i0 + c] : 0.0;
    zr[c][r] = 0.5 * (zr[c][r] + zji);
  }
  __syncthreads();
  const double inv2l = 1.0 / two_ell2;
  double ps = 0.0, pe = 0.0, pl = 0.0;
  const int jl = t & 63;
  for (int rr = 0; rr < 16; ++rr) {
    const int il = (t >> 6) + 4 * rr;
    const int64_t gi = i0 + il, gj = j0 + jl;
    double w = 0.0;
    if (gi < n && gj < n) {
      double g = 0.0;
#pragma unroll
      for (int f = 0; f < D; ++f) g += xI[il][f] * xJ[jl][f];
      const double dist = (sI[il] + sJ[jl]) - 2.0 * g;
      const double Dv = dist * inv2l;
      const double E = exp(-Dv);
      const double kb = zr[il][jl];  // Abar_ij
      ps += kb * E;
      const double nb = kb * sigma2 * E;
      pe += nb * Dv;
      if (gi == gj) pl += kb;
      w = -nb * inv2l;
    }
    zr[il][jl] = w;  // owned by this thread
  }
  // scalar partials: the off-diagonal pair stands for (i,j) and (j,i)
  const double mult = diag ? 1.0 : 2.0;
  ps *= mult;
  pe *= mult;
  const int warp = t >> 5, lane = t & 31;
  for (int o = 16; o; o >>= 1) {
    ps += __shfl_xor_sync(0xffffffffu, ps, o);
    pe += __shfl_xor_sync(0xffffffffu, pe, o);
    pl += __shfl_xor_sync(0xffffffffu, pl, o);
  }
  if (lane == 0) {
    red[0][warp] = ps;
    red[1][warp] = pl;
    red[2][warp] = pe;
  }
  __syncthreads();
  if (t < 3) {
    double a = 0.0;
    for (int w8 = 0; w8 < 8; ++w8) a += red[t][w8];
    part[(b * npairs + pr) * 3 + t] = a;
  }
  // xbar partials: row side (I rows, sum over j) and, off the diagonal, the
  // column side (J rows, sum over i): x_r sum w - sum w x_other, split over
  // two threads per line (halves of the tile) and combined by one shuffle
  const int side = t >> 7, line = (t >> 1) & 63, half = t & 1;
  if (side == 1 && diag) return;  // (warp-uniform: warps 4..7)
  double sw = 0.0, acc[D];
#pragma unroll
  for (int f = 0; f < D; ++f) acc[f] = 0.0;
  for (int k = half * 32; k < half * 32 + 32; ++k) {
    const double w = side == 0 ? zr[line][k] : zr[k][line];
    sw += w;
#pragma unroll
    for (int f = 0; f < D; ++f) acc[f] += w * (side == 0 ? xJ[k][f] : xI[k][f]);
  }
  sw += __shfl_xor_sync(0xffffffffu, sw, 1);
#pragma unroll
  for (int f = 0; f < D; ++f) acc[f] += __shfl_xor_sync(0xffffffffu, acc[f], 1);
  const int64_t row = (side == 0 ? i0 : j0) + line;
  const int64_t other = side == 0 ? J : I;
  if (half == 0 && row < n) {
    double* xp = xpart + ((b * n + row) * tiles + other) * D;
#pragma unroll
    for (int f = 0; f < D; ++f) xp[f] = (side == 0 ? xI[line][f] : xJ[line][f]) * sw - acc[f];
  }
}

// fixed-order finalization of the tile-pair partials
__global__ void k_rbf_sym_xbar(int64_t rows, int64_t tiles, int d, const double* xpart, double* xbar) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows * d; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / d, f = t % d;
    double acc = 0.0;
    for (int64_t q = 0; q < tiles; ++q) acc += xpart[(r * tiles + q) * d + f];
    xbar[t] = 4.0 * acc;
  }
}

__global__ void k_nll(int64_t batch, int64_t n, const double* quad, const double* logdet, double* nll) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b < batch) nll[b] = (quad[b] + logdet[b]) + 0.5 * (double)n * 1.8378770664093454835606594728112353;
}


// ---- batched marginal-likelihood driver helpers (BASELINE config C5) ----
// dst = src + lam I over a batch of n x n matrices (copy with diagonal shift)
__global__ void k_shift_copy(int64_t total, int64_t n, const double* src, double* dst, double lam) {
  const int64_t nn = n * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t % nn;
    const double v = src[t];
    dst[t] = (r / n == r % n) ? v + lam : v;
  }
}

__global__ void k_axpy(int64_t count, double alpha, const double* x, double* y) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x)
    y[t] += alpha * x[t];
}

// out[0] = sum_b (quad_b + logdet_b) + batch n/2 log 2 pi, out[1] = lam sum_b tr(abar_b).
// Two fixed-order passes (deterministic; no atomics):
// k_ml_partial — one warp per slice computes the slice's (phi_b, tr_b), CTAs
// reduce 64 consecutive slices each into part[]; k_ml_final — one CTA sums
// the parts in order.
constexpr int MLT = 1024;
constexpr int MLS = 64;  // slices per partial CTA (2 per warp)
__global__ void __launch_bounds__(MLT) k_ml_partial(int64_t batch, int64_t n, const double* quad,
                                                     const double* logdet, const double* abar, double* part) {
  __shared__ double s0[MLS], s1[MLS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int q = warp; q < MLS; q += MLT / 32) {
    const int64_t b = blockIdx.x * (int64_t)MLS + q;
    double tr = 0.0;
    if (b < batch) {
      const double* ab = abar + b * n * n;
      for (int64_t i = lane; i < n; i += 32) tr += ab[i * (n + 1)];
    }
    for (int o = 16; o; o >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, o);
    if (lane == 0) {
      s0[q] = b < batch ? quad[b] + logdet[b] : 0.0;
      s1[q] = tr;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, g = 0.0;
    for (int q = 0; q < MLS; ++q) {
      a += s0[q];
      g += s1[q];
    }
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = g;
  }
}

__global__ void __launch_bounds__(MLT) k_ml_final(int64_t nparts, int64_t batch, int64_t n, const double* part,
                                                   double lam, double* out) {
  __shared__ double r0[MLT], r1[MLT];
  double a = 0.0, g = 0.0;
  for (int64_t p = threadIdx.x; p < nparts; p += MLT) {
    a += part[2 * p];
    g += part[2 * p + 1];
  }
  r0[threadIdx.x] = a;
  r1[threadIdx.x] = g;
  __syncthreads();
  for (int st = MLT / 2; st; st >>= 1) {
    if (threadIdx.x < st) {
      r0[threadIdx.x] += r0[threadIdx.x + st];
      r1[threadIdx.x] += r1[threadIdx.x + st];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = r0[0] + (double)batch * 0.5 * (double)n * 1.8378770664093454835606594728112353;
    out[1] = lam * r1[0];
  }
}

}  // namespace

// Symmetric RBF pullback from Z (the fused GP tail): workspace = row norms +
// per-(row, tile) xbar partials + per-pair scalar partials.
extern "C" size_t dla_gp_rbf_bwd_sym_ws_bytes(int64_t batch, int64_t n, int64_t d) {
  const int64_t tiles = (n + SBT - 1) / SBT, npairs = tiles * (tiles + 1) / 2;
  return sizeof(double) * (size_t)(batch * n + batch * n * tiles * d + batch * npairs * 3);
}

dla_status gp_rbf_bwd_sym(int64_t batch, int64_t n, int64_t d, const double* x, double sigma2, double ell2, double lam,
                          const double* z, double* xbar, double* grads, void* ws, size_t ws_bytes, cudaStream_t s) {
  const int64_t tiles = (n + SBT - 1) / SBT, npairs = tiles * (tiles + 1) / 2;
  if (!ws || ws_bytes < dla_gp_rbf_bwd_sym_ws_bytes(batch, n, d)) return DLA_ERR_WORKSPACE;
  double* sq = static_cast<double*>(ws);
  double* xpart = sq + batch * n;
  double* part = xpart + batch * n * tiles * d;
  k_rowsq<<<blocks_for(batch * n, 256), 256, 0, s>>>(batch, n, d, x, sq);
  const unsigned grid = (unsigned)(batch * npairs);
  switch (d) {
#define DLAB_SYM_CASE(DD)                                                                                  \
  case DD:                                                                                                 \
    ensure_smem_attr(k_rbf_bwd_sym<DD>, SYM_SMEM);                                                        \
    k_rbf_bwd_sym<DD><<<grid, 256, SYM_SMEM, s>>>(n, tiles, npairs, x, sq, sigma2, ell2 * 2.0, z, xpart, part); \
    break;
    DLAB_SYM_CASE(1)
    DLAB_SYM_CASE(2)
    DLAB_SYM_CASE(3)
    DLAB_SYM_CASE(4)
    DLAB_SYM_CASE(8)
    DLAB_SYM_CASE(16)
#undef DLAB_SYM_CASE
    default:
      return DLA_ERR_SHAPE;
  }
  k_rbf_finalize<<<(unsigned)batch, FT, 0, s>>>(batch, npairs, 1, part, sigma2, ell2, lam, ell2 * 2.0, grads);
  if (xbar) k_rbf_sym_xbar<<<blocks_for(batch * n * d, 256), 256, 0, s>>>(batch * n, tiles, (int)d, xpart, xbar);
  note_launch(xbar ? 3 : 2);
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}
bool gp_rbf_sym_ok(int64_t d) { return d == 1 || d == 2 || d == 3 || d == 4 || d == 8 || d == 16; }
}  // namespace dlab

using namespace dlab;

extern "C" {

size_t dla_gp_rbf_ws_bytes(int64_t batch, int64_t n, int64_t d) {
  // row norms + per-(row, column split) partials of (s, l, e) and xbar
  return sizeof(double) * (size_t)(batch * n + batch * n * rbf_splits(n) * (3 + d));
}

dla_status dla_gp_rbf_fwd_f64(int64_t batch, int64_t n, int64_t d, const double* x, double sigma2, double ell2,
                              double lam, double* a, void* ws, size_t ws_bytes, void* stream) {
  if (batch < 0 || n < 0 || d < 0 || d > MAXD) return DLA_ERR_SHAPE;
  if (batch * n == 0) return DLA_OK;
  if (!ws || ws_bytes < dla_gp_rbf_ws_bytes(batch, n, d)) return DLA_ERR_WORKSPACE;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  double* sq = static_cast<double*>(ws);
  k_rowsq<<<blocks_for(batch * n, 256), 256, 0, s>>>(batch, n, d, x, sq);
  if (!launch_tiled<true>(d, batch, n, x, sq, sigma2, ell2 * 2.0, lam, a, nullptr, nullptr, nullptr, s))
    k_rbf_fwd<<<(unsigned)(batch * n), RT, 0, s>>>(n, d, x, sq, sigma2, ell2 * 2.0, lam, a);
  note_launch(1);  // + 1 in DLAB_LAUNCH_CHECK
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}

dla_status dla_gp_rbf_bwd_f64(int64_t batch, int64_t n, int64_t d, const double* x, double sigma2, double ell2,
                              double lam, const double* abar, double* xbar, double* grads, void* ws,
                              size_t ws_bytes, void* stream) {
  if (batch < 0 || n < 0 || d < 0 || d > MAXD) return DLA_ERR_SHAPE;
  if (batch * n == 0) return DLA_OK;
  if (!ws || ws_bytes < dla_gp_rbf_ws_bytes(batch, n, d)) return DLA_ERR_WORKSPACE;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  double* sq = static_cast<double*>(ws);
  double* part = sq + batch * n;
  const int64_t splits = rbf_splits(n);
  double* xpart = part + batch * n * splits * 3;
  k_rowsq<<<blocks_for(batch * n, 256), 256, 0, s>>>(batch, n, d, x, sq);
  int launches = 2;  // + 1 in DLAB_LAUNCH_CHECK
  if (launch_tiled<false>(d, batch, n, x, sq, sigma2, ell2 * 2.0, lam, nullptr, abar, xbar ? xpart : nullptr, part,
                          s)) {
    k_rbf_finalize<<<(unsigned)batch, FT, 0, s>>>(batch, n, splits, part, sigma2, ell2, lam, ell2 * 2.0, grads);
    if (xbar) {
      k_rbf_xbar<<<blocks_for(batch * n * d, 256), 256, 0, s>>>(batch * n, splits, (int)d, xpart, xbar);
      ++launches;
    }
  } else {  // generic d: one CTA per row, partials already per row
    k_rbf_bwd<<<(unsigned)(batch * n), RT, 0, s>>>(n, d, x, sq, sigma2, ell2 * 2.0, abar, xbar, part);
    k_rbf_finalize<<<(unsigned)batch, FT, 0, s>>>(batch, n, 1, part, sigma2, ell2, lam, ell2 * 2.0, grads);
  }
  note_launch(launches);
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}

dla_status dla_gp_nll_assemble_f64(int64_t batch, int64_t n, const double* quad, const double* logdet, double* nll,
                                   void* stream) {
  if (batch <= 0) return DLA_OK;
  k_nll<<<blocks_for(batch, 128), 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(batch, n, quad, logdet, nll);
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}

dla_status dla_ml_shift_copy_f64(int64_t batch, int64_t n, const double* s, double* a, double lam, void* stream) {
  if (batch < 0 || n < 0) return DLA_ERR_SHAPE;
  if (batch * n == 0) return DLA_OK;
  const int64_t total = batch * n * n;
  k_shift_copy<<<blocks_for(total, 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(total, n, s, a, lam);
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}

dla_status dla_axpy_f64(int64_t count, double alpha, const double* x, double* y, void* stream) {
  if (count < 0) return DLA_ERR_SHAPE;
  if (count == 0) return DLA_OK;
  k_axpy<<<blocks_for(count, 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(count, alpha, x, y);
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}

size_t dla_ml_reduce_ws_bytes(int64_t batch) {
  const int64_t nparts = batch > 0 ? (batch + MLS - 1) / MLS : 0;
  return sizeof(double) * (size_t)(2 * (nparts > 0 ? nparts : 1));
}

dla_status dla_ml_reduce_f64(int64_t batch, int64_t n, const double* quad, const double* logdet, const double* abar,
                             double lam, double* out, void* ws, size_t ws_bytes, void* stream) {
  if (batch < 0 || n < 0) return DLA_ERR_SHAPE;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t nparts = batch > 0 ? (batch + MLS - 1) / MLS : 0;
  if (!ws || ws_bytes < dla_ml_reduce_ws_bytes(batch)) return DLA_ERR_WORKSPACE;
  double* part = static_cast<double*>(ws);  // per-CTA partials of the fixed-order reduction
  if (nparts > 0) {
    k_ml_partial<<<(unsigned)nparts, MLT, 0, s>>>(batch, n, quad, logdet, abar, part);
    DLAB_LAUNCH_CHECK();
  }
  k_ml_final<<<1, MLT, 0, s>>>(nparts, batch, n, part, lam, out);
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}

}  // extern "C"
