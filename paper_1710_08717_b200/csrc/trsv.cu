// Narrow triangular solve: op(T)^{-1} applied to <= 8 vectors (the GP
// driver's L z = y and L^T s = zbar, dl/models.hpp:99 and its trsm pullback,
// dl/adjoints.hpp:136-137).  A recursive solve would be 2 n/64 dependent
// launches of almost no work each; here ONE launch covers the whole solve:
// CTA i owns block row i (64 rows), streams the blocks S(i, j), j < i, of the
// triangle (block j+1 in flight while block j is awaited) and accumulates
// them against x_j as soon as x_j is published, then applies the inverse of
// its diagonal block (computed before any wait).  x_j is published value by
// value into a scratch vector pre-filled with a sentinel NaN bit pattern, so
// the consumer's poll IS the data load: no fence, no flag round trip on the
// dependent chain.  The triangle is read once (n^2/2 elements), in parallel
// across all CTAs; the chain is one L2 round trip + a 64 x 64 GEMV per block.
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
__device__ __forceinline__ const T* s_ptr(const TrsvGeo& g, MatB<const T> t, int64_t b, int64_t r, int64_t c) {
  const int64_t pr = phys(g, r), pc = phys(g, c);
  return g.s_tt ? t.at(b, pc, pr) : t.at(b, pr, pc);
}

template <typename T>
__device__ __forceinline__ T* x_at(const TrsvGeo& g, MatB<T> x, int64_t b, int64_t r, int v) {
  return g.right ? x.at(b, v, phys(g, r)) : x.at(b, phys(g, r), v);
}

template <typename T>
struct Sentinel;
template <>
struct Sentinel<double> {
  using U = unsigned long long;
  static constexpr U bits = 0xFFFFFFFFFFFFFFFFull;  // a NaN no FP64 operation produces (canonical NaN is 0x7FFF...)
  __device__ static U as_bits(double v) { return (U)__double_as_longlong(v); }
  __device__ static double canon(double v) { return as_bits(v) == bits ? __longlong_as_double(0x7FF8000000000000ll) : v; }
  __device__ static double poll(const double* p) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
  }
};
template <>
struct Sentinel<float> {
  using U = unsigned;
  static constexpr U bits = 0xFFFFFFFFu;
  __device__ static U as_bits(float v) { return (U)__float_as_uint(v); }
  __device__ static float canon(float v) { return as_bits(v) == bits ? __uint_as_float(0x7FC00000u) : v; }
  __device__ static float poll(const float* p) {
    float v;
    asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
  }
};

// One CTA per block row i.  Results are published value-by-value into `pub`
// (pre-filled with the sentinel bit pattern): a consumer knows block j is
// final once none of its values is the sentinel, so publication needs no
// fence or flag round trip.  The blocks S(i, j) stream into a 3-stage
// shared-memory ring by cp.async (they do not depend on any result), warp 0
// polls up to three published blocks per round trip into a ring of x
// buffers, and every thread accumulates its (row, 16-column chunk) products.
constexpr int NS = 3;   // S-block ring stages
constexpr int NY = 4;   // x-block ring slots (3 may be filled ahead)
constexpr int TLD = BR + 1;

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  if (bytes == 8) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
  else asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit8() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait8() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// tile element (r, c) of a staged block: rows of S contiguous (!s_tt) or
// columns contiguous (s_tt), always conflict-free for the r = tid % 64 reads
__device__ __forceinline__ int tidx(bool s_tt, int r, int c) { return s_tt ? c * TLD + r : r * TLD + c; }

// Thread tid copies the elements hi = tid / 64 + 4 k, lo = tid % 64 (k < 16)
// of every staged block; (r, c) = s_tt ? (lo, hi) : (hi, lo), consecutive
// threads on memory-consecutive elements.  phys() is affine, so the source
// address is base + j * dj + k * dk and the shared offset (hi * TLD + lo) is
// the same in both layouts: precomputed once per thread.
struct StageMap {
  int64_t src0, dj, dk;  // element offsets from t.p
  int dst0;
  int krows;             // copy k only while k < krows (partial last block row)
};

template <typename T>
__device__ __forceinline__ StageMap stage_map(const TrsvGeo& g, MatB<const T> t, int64_t b, int64_t r0, int rows) {
  const int lo = threadIdx.x % BR, h0 = threadIdx.x / BR;
  auto off = [&](int hi, int64_t j) {
    const int r = g.s_tt ? lo : hi, c = g.s_tt ? hi : lo;
    return (int64_t)(s_ptr(g, t, b, r0 + r, j * BR + c) - t.p);
  };
  StageMap m;
  m.src0 = off(h0, 0);
  m.dj = off(h0, 1) - m.src0;
  m.dk = off(h0 + 4, 0) - m.src0;
  m.dst0 = h0 * TLD + lo;
  if (g.s_tt) m.krows = lo < rows ? 16 : 0;
  else m.krows = rows > h0 ? (rows - h0 + 3) / 4 : 0;
  return m;
}

template <typename T>
__device__ __forceinline__ void stage_block(const StageMap& m, const T* tp, int64_t j, T* tile) {
  const T* src = tp + m.src0 + j * m.dj;
#pragma unroll
  for (int k = 0; k < 16; ++k)
    if (k < m.krows) cp_async8(tile + m.dst0 + k * 4 * TLD, src + k * m.dk, (int)sizeof(T));
}

template <typename T>
__global__ void __launch_bounds__(TT, 1) k_trsv(TrsvGeo g, MatB<const T> t, MatB<T> x, T alpha, T* pub,
                                             const int32_t* skip, unsigned long long* ticket) {
  using SN = Sentinel<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* S = reinterpret_cast<T*>(smem_raw);  // diagonal block, then partial sums P[4][NR][BR]
  T* Xi = S + BR * SLD;                   // inverse of the diagonal block, vector-major: Xi[v*SLD + r] = Sinv(r, v)
  T* rd = Xi + BR * SLD;
  T(*Y)[NR][BR] = reinterpret_cast<T(*)[NR][BR]>(rd + BR);            // [NY][NR][BR]
  T(*R)[BR] = reinterpret_cast<T(*)[BR]>(rd + BR + NY * NR * BR);     // [NR][BR] right-hand side
  T* ring = rd + BR + (NY + 1) * NR * BR;                             // [NS][BR * TLD]
  // Logical block = an atomic ticket, not blockIdx: block (b, i) waits only on
  // blocks (b, j < i), whose tickets were drawn by CTAs that are already
  // resident, so forward progress never depends on the order in which the
  // hardware dispatches CTAs (concurrent streams, MPS).
  __shared__ unsigned long long tk;
  if (threadIdx.x == 0) tk = atomicAdd(ticket, 1ull);
  __syncthreads();
  const int64_t b = (int64_t)(tk / (unsigned long long)g.nblk), i = (int64_t)(tk % (unsigned long long)g.nblk);
  if (slice_failed(skip, b)) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t r0 = i * BR;
  const int rows = (int)min((int64_t)BR, g.nt - r0);
  const int nv = (int)g.nvec;
  T* pubb = pub + b * g.nvec * g.nt;  // pub[v * nt + logical row]
  // the first NS-1 off-diagonal blocks start streaming immediately
  const StageMap sm = stage_map<T>(g, t, b, r0, rows);
#pragma unroll
  for (int q = 0; q < NS - 1; ++q) {
    if (q < i) stage_block<T>(sm, t.p, q, ring + q * BR * TLD);
    cp_commit8();
  }
  for (int e = tid; e < NR * BR; e += TT) {
    const int v = e / BR, rr = e % BR;
    R[v][rr] = (v < nv && rr < rows) ? alpha * *x_at(g, x, b, r0 + rr, v) : T(0);
  }
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
  const int r = tid % BR, cq = tid / BR;  // (row, 16-column chunk)
  T part[NR];
#pragma unroll
  for (int v = 0; v < NR; ++v) part[v] = T(0);
  int64_t have = 0;  // warp 0: blocks < have already sit in the Y ring
  for (int64_t j = 0; j < i; ++j) {
    cp_wait8<NS - 2>();  // this thread's copies of block j have landed
    if (warp == 0 && have <= j) {
      // one round trip polls blocks j .. j+2: slots of blocks <= j-2 are free
      const int64_t span = min((int64_t)3, i - j);
      int64_t got = 0;
      for (;;) {
        bool ok[3] = {true, true, true};
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          if (q >= span) continue;
          const T* src = pubb + (j + q) * BR;
          T(*Yq)[BR] = Y[(j + q) % NY];
          for (int v = 0; v < nv; ++v) {
            const T y0 = SN::poll(src + v * g.nt + lane), y1 = SN::poll(src + v * g.nt + lane + 32);
            ok[q] &= SN::as_bits(y0) != SN::bits && SN::as_bits(y1) != SN::bits;
            Yq[v][lane] = y0;
            Yq[v][lane + 32] = y1;
          }
        }
        const bool r0k = __all_sync(0xffffffffu, ok[0]);
        const bool r1k = __all_sync(0xffffffffu, ok[1]);
        const bool r2k = __all_sync(0xffffffffu, ok[2]);
        got = !r0k ? 0 : (span < 2 || !r1k) ? 1 : (span < 3 || !r2k) ? 2 : 3;
        if (got > 0) break;
      }
      have = j + got;
    }
    __syncthreads();  // block j staged by every thread; x_j in Y[j % NY]
    {
      const int64_t pf = j + NS - 1;  // refill the stage block j-1 used
      if (pf < i) stage_block<T>(sm, t.p, pf, ring + (pf % NS) * BR * TLD);
      cp_commit8();
    }
    const T* tile = ring + (j % NS) * BR * TLD;
    T(*Yj)[BR] = Y[j % NY];
#pragma unroll
    for (int cc = 0; cc < 16; ++cc) {
      const int c = cq * 16 + cc;
      const T sv = tile[tidx(g.s_tt, r, c)];
#pragma unroll
      for (int v = 0; v < NR; ++v)
        if (v < nv) part[v] += sv * Yj[v][c];
    }
  }
  cp_wait8<0>();
  // right-hand side minus the four column-chunk partial sums
  T* P = S;  // the diagonal block is no longer needed
#pragma unroll
  for (int v = 0; v < NR; ++v) P[(cq * NR + v) * BR + r] = part[v];
  __syncthreads();
  T(*Q)[BR] = R;  // in place: each (v, rr) read and written by one thread
  for (int e = tid; e < NR * BR; e += TT) {
    const int v = e / BR, rr = e % BR;
    Q[v][rr] = R[v][rr] - (P[(0 * NR + v) * BR + rr] + P[(1 * NR + v) * BR + rr] + P[(2 * NR + v) * BR + rr] +
                           P[(3 * NR + v) * BR + rr]);
  }
  __syncthreads();
  // y_i = S_ii^{-1} rhs: four adjacent lanes per (vector, row), 16 columns each
  for (int e0 = 0; e0 < nv * BR * 4; e0 += TT) {
    const int e = e0 + tid, v = e / (BR * 4), rr = (e / 4) % BR, q = e & 3;
    T acc = T(0);
    if (v < nv) {
#pragma unroll
      for (int cc = 0; cc < 16; ++cc) {
        const int c = q * 16 + cc;
        if (c <= rr) acc += Xi[c * SLD + rr] * Q[v][c];
      }
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    if (q == 0 && v < nv && rr < rows) {
      *x_at(g, x, b, r0 + rr, v) = acc;
      pubb[v * g.nt + r0 + rr] = SN::canon(acc);
    }
  }
}

}  // namespace

template <typename T>
bool trsv_eligible(int64_t nt, int64_t nvec) {
  return nt > 64 && nvec >= 1 && nvec <= NR;
}

template <typename T>
size_t ws_trsv(int64_t batch, int64_t m, int64_t n, bool right) {
  (void)right;
  return carve_bound(sizeof(T) * (size_t)(batch * m * n)) + carve_bound(sizeof(unsigned long long));
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
  const size_t pub_bytes = sizeof(T) * (size_t)(batch * g.nvec * g.nt);
  DLAB_SCRATCH(pub, c, pub_bytes);
  DLAB_SCRATCH(tick, c, sizeof(unsigned long long));
  if (cudaMemsetAsync(pub.p, 0xFF, pub_bytes, c.stream) != cudaSuccess) return DLA_ERR_CUDA;  // sentinel
  if (cudaMemsetAsync(tick.p, 0, sizeof(unsigned long long), c.stream) != cudaSuccess) return DLA_ERR_CUDA;
  const size_t sm = sizeof(T) * (2 * BR * SLD + BR + (NY + 1) * NR * BR + NS * BR * TLD);
  ensure_smem_attr(k_trsv<T>, sm);
  k_trsv<T><<<(unsigned)(batch * g.nblk), TT, sm, c.stream>>>(g, t, x, alpha, pub.as<T>(), c.info,
                                                               tick.as<unsigned long long>());
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}

template bool trsv_eligible<double>(int64_t, int64_t);
template bool trsv_eligible<float>(int64_t, int64_t);
template size_t ws_trsv<double>(int64_t, int64_t, int64_t, bool);
template size_t ws_trsv<float>(int64_t, int64_t, int64_t, bool);
template dla_status trsv<double>(const Ctx&, int64_t, int64_t, int64_t, MatB<const double>, MatB<double>, bool, bool,
                                 bool, double);
template dla_status trsv<float>(const Ctx&, int64_t, int64_t, int64_t, MatB<const float>, MatB<float>, bool, bool,
                                bool, float);

}  // namespace dlab
