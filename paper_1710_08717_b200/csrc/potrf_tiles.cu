// Persistent tile-dataflow Cholesky (f64): ONE launch per factorization.
//
// The blocked right-looking loop of dl/cholesky.hpp:43-70 (nb = 64) is a
// DAG of 64 x 64 tile tasks.  Launching it level by level (panel kernel,
// column update, trailing update, x n/64) leaves the GPU idle between the
// dependent launches of the critical chain: at n = 4096 that chain is 64
// steps of ~60 us.  Here every lower tile (i, j) of every matrix is one task,
// owned by one CTA from start to finish (left-looking per tile):
//
//     C      = A(i,j) - sum_{k<j} L(i,k) L(j,k)^T     (FP64 DMMA, cp.async)
//     L(j,j) = chol(C)                    if i == j   (chol_smem64)
//     L(i,j) = C L(j,j)^{-T}              if i >  j   (blocked_fwd_subst)
//
// Persistent CTAs take tasks from an atomic ticket counter in column-major
// order (diagonal first in each column).  A task only waits for tasks with
// smaller tickets, which are held by running CTAs, so any grid size is
// deadlock-free.  Completion is published per tile (global flag, release
// via __threadfence + atomicExch; consumers spin on a volatile load and read
// the tile through L2 with cp.async.cg / ld.global.cg).  The update for
// k-tile k starts as soon as L(i,k) and L(j,k) exist, so the accumulation of
// a tile overlaps the factorization of earlier columns; the critical path
// is one chol + one tile solve + one tile update per column.
//
// A failed pivot records info (global index) and poisons the tile's flag
// (value 2); every dependent task of that matrix then stops and poisons its
// own flag, and the slice is left partially factored (the reference throws
// before returning, dl/cholesky.hpp:49-53).
#include <cstdlib>

#include "chol64.cuh"
#include "common.cuh"
#include "ops.cuh"

namespace dlab {
namespace {

constexpr int TB = 64;           // tile size
constexpr int TK = 16;           // k chunk per pipeline stage
constexpr int TSTAGES = 3;
constexpr int TLD = TK + 4;      // smem row stride of a staged chunk (rows contiguous in k)
constexpr int TTHREADS = 128;    // 4 warps, 32 x 32 warp tiles
constexpr int TSLD = TB + 1;     // chol / solve tiles

#ifdef DLAB_TILES_TRACE
__device__ long long* dlab_tiles_trace;  // [ticket][6]: t0, t_update, t_end, smid, i, j
__device__ __forceinline__ long long gtime() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif

struct TileArgs {
  int64_t batch, n, nt;
  MatB<double> a;
  int64_t kbase;
  int* flags;    // [batch][nt][nt]
  int* ticket;   // [1]
  int32_t* info;
};

__device__ __forceinline__ void cp16(void* smem, const void* gmem, bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(pred ? 16 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ int flag_wait(const int* f) {
  const volatile int* v = f;
  int x;
  while ((x = *v) == 0) __nanosleep(64);
  __threadfence();
  return x;
}

// Decode ticket t (column-major over j, then batch, then i >= j).
__device__ __forceinline__ bool decode_task(const TileArgs& g, int64_t t, int64_t& b, int64_t& i, int64_t& j) {
  for (int64_t c = 0; c < g.nt; ++c) {
    const int64_t per = (g.nt - c) * g.batch;
    if (t < per) {
      b = t / (g.nt - c);
      i = c + t % (g.nt - c);
      j = c;
      return true;
    }
    t -= per;
  }
  return false;
}

// Stage chunk q (k = q * TK .. +TK) of rows of tile-row `ti` and tile-row
// `tj` (both contiguous along k): sa[r][kk] = a(ti*TB + r, q*TK + kk).
__device__ __forceinline__ void load_chunk(const TileArgs& g, const double* base, int64_t ti, int64_t tj, int64_t q,
                                           double* sa, double* sb) {
  // 64 rows x 16 doubles = 512 16-byte pieces per operand; 128 threads x 4
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int c = threadIdx.x + u * TTHREADS;
    const int r = c >> 3, kk = (c & 7) * 2;
    const int64_t ra = ti * TB + r, rb = tj * TB + r, col = q * TK + kk;
    cp16(sa + r * TLD + kk, base + (ra < g.n ? ra : 0) * g.a.ld + col, ra < g.n);
    cp16(sb + r * TLD + kk, base + (rb < g.n ? rb : 0) * g.a.ld + col, rb < g.n);
  }
}

__global__ void __launch_bounds__(TTHREADS, 3) k_potrf_tiles(TileArgs g) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sm = reinterpret_cast<double*>(smem_raw);
  // phase 1 (update): TSTAGES x (A chunk, B chunk); phase 2 (finalize): S, V, rd
  double* sA = sm;
  double* sB = sm + TSTAGES * TB * TLD;
  double* S = sm;
  double* V = sm + TB * TSLD;
  double* rd = V + TB * TSLD;
  __shared__ int64_t s_ticket;
  __shared__ int s_flag, s_abort;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int fr = lane >> 2, fc = lane & 3;
  const int64_t total = g.batch * g.nt * (g.nt + 1) / 2;

  for (;;) {
    if (tid == 0) s_ticket = atomicAdd(reinterpret_cast<unsigned long long*>(g.ticket), 1ull);
    __syncthreads();
    const int64_t t = s_ticket;
    if (t >= total) return;
    int64_t b, i, j;
    decode_task(g, t, b, i, j);
#ifdef DLAB_TILES_TRACE
    long long tr0 = gtime(), tr1 = 0;
#endif
    int* fl = g.flags + b * g.nt * g.nt;
    const double* base = g.a.p + b * g.a.bs;
    if (tid == 0) s_abort = slice_failed(g.info, b) ? 1 : 0;

    double acc[4][4][2];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;

    // ---- update: C -= sum_{k<j} L(i,k) L(j,k)^T, chunks of TK along k
    const int64_t nq = j * (TB / TK);
    auto wait_ktile = [&](int64_t q) {  // before staging the first chunk of a k-tile
      if ((q % (TB / TK)) != 0) return;
      const int64_t k = q / (TB / TK);
      if (tid == 0 && !s_abort) {
        if (flag_wait(fl + i * g.nt + k) == 2 || flag_wait(fl + j * g.nt + k) == 2) s_abort = 1;
      }
      __syncthreads();
    };
    for (int s = 0; s < TSTAGES - 1; ++s) {
      if (s < nq) {
        wait_ktile(s);
        if (!s_abort) load_chunk(g, base, i, j, s, sA + s * TB * TLD, sB + s * TB * TLD);
      }
      cp_commit();
    }
    for (int64_t q = 0; q < nq; ++q) {
      cp_wait<TSTAGES - 2>();
      __syncthreads();
      const int64_t pf = q + TSTAGES - 1;
      if (pf < nq) {
        wait_ktile(pf);
        if (!s_abort) load_chunk(g, base, i, j, pf, sA + (pf % TSTAGES) * TB * TLD, sB + (pf % TSTAGES) * TB * TLD);
      }
      cp_commit();
      if (s_abort) continue;
      const double* a = sA + (q % TSTAGES) * TB * TLD;
      const double* bb = sB + (q % TSTAGES) * TB * TLD;
#pragma unroll
      for (int kk = 0; kk < TK; kk += 4) {
        double af[4], bf[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) af[x] = a[(wm + x * 8 + fr) * TLD + kk + fc];
#pragma unroll
        for (int y = 0; y < 4; ++y) bf[y] = bb[(wn + y * 8 + fr) * TLD + kk + fc];
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(acc[x][y][0]), "+d"(acc[x][y][1])
                         : "d"(af[x]), "d"(bf[y]));
      }
    }
    cp_wait<0>();
    __syncthreads();  // staging buffers are reused below
#ifdef DLAB_TILES_TRACE
    tr1 = gtime();
#endif

    const int rows = (int)min((int64_t)TB, g.n - i * TB);
    const int cols = (int)min((int64_t)TB, g.n - j * TB);
    double* tile = g.a.p + b * g.a.bs + (i * TB) * g.a.ld + j * TB;
    if (s_abort) {
      if (tid == 0) atomicExch(fl + i * g.nt + j, 2);
      continue;
    }
    // ---- C = A(i,j) - acc, into V (vector-major: V[r][c] = C(r, c)) for
    // both cases; the diagonal case factors it in place.
    double* C = (i == j) ? S : V;
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        const int r = wm + x * 8 + fr, c = wn + y * 8 + 2 * fc;
        C[r * TSLD + c] = acc[x][y][0];
        C[r * TSLD + c + 1] = acc[x][y][1];
      }
    __syncthreads();
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // 16 loads in flight per thread, then the smem updates
      double v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int e = tid + (h * 16 + u) * TTHREADS, r = e >> 6, c = e & 63;
        const bool in = r < rows && c < cols && (i != j || c <= r);
        v[u] = in ? __ldcg(tile + r * g.a.ld + c) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int e = tid + (h * 16 + u) * TTHREADS, r = e >> 6, c = e & 63;
        const bool in = r < rows && c < cols && (i != j || c <= r);
        C[r * TSLD + c] = in ? v[u] - C[r * TSLD + c] : 0.0;
      }
    }
    __syncthreads();
    if (i == j) {
      const int failed = chol_smem64<double>(S, rows, &s_flag);
      if (failed >= 0) {
        if (tid == 0) {
          record_failure(g.info, b, DLA_ERR_NOT_SPD, g.kbase + j * TB + failed);
          atomicExch(fl + i * g.nt + j, 2);
        }
        continue;
      }
      for (int e = tid; e < rows * TB; e += TTHREADS) {
        const int r = e >> 6, c = e & 63;
        if (c <= r) tile[r * g.a.ld + c] = S[r * TSLD + c];
      }
    } else {
      if (tid == 0) s_abort = flag_wait(fl + j * g.nt + j) == 2 ? 1 : 0;
      __syncthreads();
      if (s_abort) {
        if (tid == 0) atomicExch(fl + i * g.nt + j, 2);
        continue;
      }
      const double* djj = g.a.p + b * g.a.bs + (j * TB) * g.a.ld + j * TB;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int e = tid + (h * 16 + u) * TTHREADS, r = e >> 6, c = e & 63;
          v[u] = (r < cols && c <= r) ? __ldcg(djj + r * g.a.ld + c) : (r == c ? 1.0 : 0.0);
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int e = tid + (h * 16 + u) * TTHREADS;
          S[(e >> 6) * TSLD + (e & 63)] = v[u];
        }
      }
      __syncthreads();
      if (tid < TB) rd[tid] = 1.0 / S[tid * TSLD + tid];
      __syncthreads();
      blocked_fwd_subst<double>(S, V, rd, cols, rows);  // row r: L(j,j) x = c_r
      for (int e = tid; e < rows * TB; e += TTHREADS) {
        const int r = e >> 6, c = e & 63;
        if (c < cols) tile[r * g.a.ld + c] = V[r * TSLD + c];
      }
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) atomicExch(fl + i * g.nt + j, 1);
#ifdef DLAB_TILES_TRACE
    if (tid == 0) {
      unsigned smid;
      asm("mov.u32 %0, %%smid;" : "=r"(smid));
      long long* r = dlab_tiles_trace + 6 * t;
      r[0] = tr0;
      r[1] = tr1;
      r[2] = gtime();
      r[3] = smid;
      r[4] = i;
      r[5] = j;
    }
#endif
  }
}

}  // namespace

bool potrf_tiles_eligible(int64_t batch, int64_t n, const MatB<double>& a) {
  const uintptr_t p = reinterpret_cast<uintptr_t>(a.p);
  return n > TB && (p % 16) == 0 && (a.ld % 2) == 0 && (a.bs % 2) == 0 && batch * ((n + TB - 1) / TB) <= 4096;
}

size_t ws_potrf_tiles(int64_t batch, int64_t n) {
  const int64_t nt = (n + TB - 1) / TB;
  return carve_bound(sizeof(int) * (size_t)(batch * nt * nt) + 16);
}

dla_status potrf_tiles(const Ctx& c, int64_t batch, int64_t n, MatB<double> a, int64_t kbase) {
  const int64_t nt = (n + TB - 1) / TB;
  const size_t flag_bytes = sizeof(int) * (size_t)(batch * nt * nt);
  DLAB_SCRATCH(ws, c, flag_bytes + 16);
  if (cudaMemsetAsync(ws.p, 0, flag_bytes + 16, c.stream) != cudaSuccess) return DLA_ERR_CUDA;
  TileArgs g;
  g.batch = batch;
  g.n = n;
  g.nt = nt;
  g.a = a;
  g.kbase = kbase;
  g.flags = reinterpret_cast<int*>(static_cast<char*>(ws.p) + 16);
  g.ticket = static_cast<int*>(ws.p);
  g.info = c.info;
  const size_t sm_update = sizeof(double) * 2 * TSTAGES * TB * TLD;
  const size_t sm_final = sizeof(double) * (2 * TB * TSLD + TB);
  const size_t sm = sm_update > sm_final ? sm_update : sm_final;
  ensure_smem_attr(k_potrf_tiles, sm);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_potrf_tiles, TTHREADS, sm);
  if (per_sm < 1) per_sm = 1;
  static const int cap = [] {
    const char* e = getenv("DLA_TILES_PER_SM");  // tuning switch: resident CTAs per SM
    return e ? atoi(e) : 0;
  }();
  const int64_t tasks = batch * nt * (nt + 1) / 2;
  const int64_t grid = min(tasks, (int64_t)c.sms * (cap > 0 ? min(cap, per_sm) : per_sm));
  k_potrf_tiles<<<(unsigned)grid, TTHREADS, sm, c.stream>>>(g);
  DLAB_LAUNCH_CHECK();
  return DLA_OK;
}

}  // namespace dlab
