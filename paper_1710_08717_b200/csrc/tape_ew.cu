// Elementwise / structural node kernels of the device tape.
//
// The reference tape (dl/tape.hpp) evaluates its non-linear-algebra nodes —
// Add/Sub/Mul, Square/Sqrt/Log/Exp/Abs/Neg, ScaleConst/AddConst,
// MulScalar/DivScalar, Sum/SumRows, TileCols/TileRows, ExtractDiag/MakeDiag,
// Tril/TriuMask, ConcatCols (compute_node :615-790) and their pullbacks
// (pull_node :930-1120) — as scalar loops over host matrices.  The device tape
// (paper_1710_08717_b200/tape.py) runs them here: one grid-stride kernel per
// node, the same per-element expression as the reference loop body, in place
// when the memory plan donated the input buffer (out == x), and with an
// accumulate flag that implements Graph::acc (:920-929, out += m) without a
// temporary.  Reductions (Sum, Dot, SumRows, SumCols) are fixed-order trees:
// deterministic run to run (the reference sums sequentially: tolerance-level
// differences only).
#include "common.cuh"

namespace dlab {
namespace {

template <typename T>
__device__ __forceinline__ void put(T* out, int64_t i, T v, bool acc) {
  out[i] = acc ? out[i] + v : v;
}

template <typename T>
__global__ void k_ew_map(int op, int64_t count, const T* x, const T* y, const T* s, T c, T* out, bool acc) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const T xv = x[i];
    T v;
    switch (op) {
      case DLA_EW_COPY: v = xv; break;
      case DLA_EW_ADD: v = xv + y[i]; break;
      case DLA_EW_SUB: v = xv - y[i]; break;
      case DLA_EW_MUL: v = xv * y[i]; break;
      case DLA_EW_SQUARE: v = xv * xv; break;
      case DLA_EW_SQRT: v = sqrt(xv); break;
      case DLA_EW_LOG: v = log(xv); break;
      case DLA_EW_EXP: v = exp(xv); break;
      case DLA_EW_ABS: v = fabs(xv); break;
      case DLA_EW_NEG: v = -xv; break;
      case DLA_EW_SCALE: v = xv * c; break;
      case DLA_EW_ADDC: v = xv + c; break;
      case DLA_EW_MULS: v = xv * s[0]; break;
      case DLA_EW_DIVS: v = xv / s[0]; break;
      case DLA_EW_FILL: v = s[0]; break;
      case DLA_EW_SQUARE_BWD: v = xv * (T(2) * y[i]); break;  // g * (2 x), dl/tape.hpp Square pullback
      case DLA_EW_SQRT_BWD: v = xv / (T(2) * y[i]); break;    // g / (2 y)
      case DLA_EW_LOG_BWD: v = xv / y[i]; break;              // g / x
      case DLA_EW_ABS_BWD: {
        const T w = y[i];
        v = xv * (w > T(0) ? T(1) : (w < T(0) ? T(-1) : T(0)));
        break;
      }
      default: v = T(0); break;
    }
    put(out, i, v, acc);
  }
}

// rows x cols structural maps (output element per thread)
template <typename T>
__global__ void k_ew_struct(int op, int64_t rows, int64_t cols, int64_t aux, const T* x, const T* y, T c, T* out,
                            bool acc) {
  int64_t total;
  switch (op) {
    case DLA_EW_TRIL:
    case DLA_EW_TRIU: total = rows * cols; break;
    case DLA_EW_TILECOLS: total = rows * aux; break;
    case DLA_EW_TILEROWS: total = aux * rows; break;
    case DLA_EW_EXTRACTDIAG: total = rows; break;
    case DLA_EW_MAKEDIAG: total = rows * rows; break;
    case DLA_EW_CONCATCOLS: total = rows * (cols + aux); break;
    case DLA_EW_SLICECOLS: total = rows * cols; break;
    default: total = 0; break;
  }
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    T v = T(0);
    switch (op) {
      case DLA_EW_TRIL: {
        const int64_t i = t / cols, j = t - i * cols;
        v = j <= i ? x[t] : T(0);
        break;
      }
      case DLA_EW_TRIU: {
        const int64_t i = t / cols, j = t - i * cols;
        v = j >= i ? x[t] : T(0);
        break;
      }
      case DLA_EW_TILECOLS: v = x[t / aux]; break;        // x rows x 1 -> rows x aux
      case DLA_EW_TILEROWS: v = x[t % rows]; break;       // x rows x 1 -> aux x rows
      case DLA_EW_EXTRACTDIAG: v = x[t * cols + t]; break;
      case DLA_EW_MAKEDIAG: {
        const int64_t i = t / rows, j = t - i * rows;
        v = i == j ? x[i] : T(0);
        break;
      }
      case DLA_EW_CONCATCOLS: {  // [x | y], x rows x cols, y rows x aux
        const int64_t w = cols + aux, i = t / w, j = t - i * w;
        v = j < cols ? x[i * cols + j] : y[i * aux + (j - cols)];
        break;
      }
      case DLA_EW_SLICECOLS: {  // x rows x aux; columns [c, c + cols)
        const int64_t i = t / cols, j = t - i * cols;
        v = x[i * aux + (int64_t)c + j];
        break;
      }
    }
    put(out, t, v, acc);
  }
}

// Row sums (SumRows) / column sums (SumCols): one warp per output element,
// fixed lane-strided partials + shuffle tree.
template <typename T>
__global__ void k_ew_lines(bool by_rows, int64_t rows, int64_t cols, const T* x, T* out, bool acc) {
  const int64_t nout = by_rows ? rows : cols, len = by_rows ? cols : rows;
  const int lane = threadIdx.x & 31;
  for (int64_t o = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; o < nout;
       o += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    T a = T(0);
    for (int64_t k = lane; k < len; k += 32) a += by_rows ? x[o * cols + k] : x[k * cols + o];
    for (int off = 16; off; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
    if (lane == 0) put(out, o, a, acc);
  }
}

// Sum / Dot over count elements: a fixed grid of partials, then one CTA.
constexpr int RB = 256, RG = 128;
template <typename T>
__global__ void k_ew_reduce_part(int64_t count, const T* x, const T* y, T* part) {
  __shared__ T red[RB];
  T a = T(0);
  for (int64_t i = blockIdx.x * (int64_t)RB + threadIdx.x; i < count; i += (int64_t)gridDim.x * RB)
    a += y ? x[i] * y[i] : x[i];
  red[threadIdx.x] = a;
  __syncthreads();
  for (int st = RB / 2; st; st >>= 1) {
    if (threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}
template <typename T>
__global__ void k_ew_reduce_final(int nparts, const T* part, const T* s, T scale, bool neg_div, T* out, bool acc) {
  __shared__ T red[RG];
  red[threadIdx.x] = threadIdx.x < nparts ? part[threadIdx.x] : T(0);
  __syncthreads();
  for (int st = RG / 2; st; st >>= 1) {
    if (threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    T v = red[0] * scale;
    if (neg_div) v = -v / s[0];  // DivScalar's sbar = -sum(g * y) / s
    put(out, 0, v, acc);
  }
}

}  // namespace

template <typename T>
dla_status tape_ew(int op, int64_t rows, int64_t cols, int64_t aux, const T* x, const T* y, const T* s, T c, T* out,
                   int accumulate, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (rows < 0 || cols < 0 || aux < 0) return DLA_ERR_SHAPE;
  const bool acc = accumulate != 0;
  const int64_t count = rows * cols;
  switch (op) {
    case DLA_EW_COPY:
    case DLA_EW_SQUARE:
    case DLA_EW_SQRT:
    case DLA_EW_LOG:
    case DLA_EW_EXP:
    case DLA_EW_ABS:
    case DLA_EW_NEG:
    case DLA_EW_SCALE:
    case DLA_EW_ADDC:
      if (!x || !out) return DLA_ERR_INVALID;
      break;
    case DLA_EW_ADD:
    case DLA_EW_SUB:
    case DLA_EW_MUL:
    case DLA_EW_SQUARE_BWD:
    case DLA_EW_SQRT_BWD:
    case DLA_EW_LOG_BWD:
    case DLA_EW_ABS_BWD:
      if (!x || !y || !out) return DLA_ERR_INVALID;
      break;
    case DLA_EW_MULS:
    case DLA_EW_DIVS:
      if (!x || !s || !out) return DLA_ERR_INVALID;
      break;
    case DLA_EW_FILL:
      if (!s || !out) return DLA_ERR_INVALID;
      break;
    default:
      break;
  }
  if (op <= DLA_EW_ABS_BWD) {
    if (count == 0) return DLA_OK;
    const T* xx = op == DLA_EW_FILL ? s : x;  // FILL reads no x
    k_ew_map<T><<<blocks_for(count, 256, 148 * 16), 256, 0, st>>>(op, count, op == DLA_EW_FILL ? out : xx, y, s, c,
                                                                  out, acc);
    DLAB_LAUNCH_CHECK();
    return DLA_OK;
  }
  switch (op) {
    case DLA_EW_TRIL:
    case DLA_EW_TRIU:
    case DLA_EW_EXTRACTDIAG:
    case DLA_EW_MAKEDIAG:
      if (op != DLA_EW_MAKEDIAG && rows != cols) return DLA_ERR_SHAPE;
      if (op == DLA_EW_MAKEDIAG && cols != 1) return DLA_ERR_SHAPE;
      [[fallthrough]];
    case DLA_EW_TILECOLS:
    case DLA_EW_TILEROWS:
    case DLA_EW_CONCATCOLS:
    case DLA_EW_SLICECOLS: {
      if (!x || !out || (op == DLA_EW_CONCATCOLS && !y)) return DLA_ERR_INVALID;
      const int64_t work = rows * (cols + aux + rows);
      k_ew_struct<T><<<blocks_for(work, 256, 148 * 16), 256, 0, st>>>(op, rows, cols, aux, x, y, c, out, acc);
      DLAB_LAUNCH_CHECK();
      return DLA_OK;
    }
    case DLA_EW_SUMROWS:
    case DLA_EW_SUMCOLS: {
      if (!x || !out) return DLA_ERR_INVALID;
      const int64_t nout = op == DLA_EW_SUMROWS ? rows : cols;
      k_ew_lines<T><<<blocks_for(nout * 32, 256, 148 * 16), 256, 0, st>>>(op == DLA_EW_SUMROWS, rows, cols, x, out,
                                                                           acc);
      DLAB_LAUNCH_CHECK();
      return DLA_OK;
    }
    case DLA_EW_SUM:
    case DLA_EW_DOT:
    case DLA_EW_DOT_NEG_DIV: {
      if (!x || !out || (op != DLA_EW_SUM && !y) || (op == DLA_EW_DOT_NEG_DIV && !s)) return DLA_ERR_INVALID;
      if (!ws || ws_bytes < sizeof(T) * RG) return DLA_ERR_WORKSPACE;
      T* part = static_cast<T*>(ws);
      const int nb = (int)std::min<int64_t>(RG, std::max<int64_t>(1, (count + RB - 1) / RB));
      k_ew_reduce_part<T><<<nb, RB, 0, st>>>(count, x, op == DLA_EW_SUM ? nullptr : y, part);
      k_ew_reduce_final<T><<<1, RG, 0, st>>>(nb, part, s, T(1), op == DLA_EW_DOT_NEG_DIV, out, acc);
      note_launch(1);
      DLAB_LAUNCH_CHECK();
      return DLA_OK;
    }
    default:
      return DLA_ERR_INVALID;
  }
}

}  // namespace dlab

using namespace dlab;

extern "C" {

size_t dla_tape_ew_ws_bytes(void) { return sizeof(double) * RG; }

dla_status dla_tape_ew_f64(int op, int64_t rows, int64_t cols, int64_t aux, const double* x, const double* y,
                           const double* s, double c, double* out, int accumulate, void* ws, size_t ws_bytes,
                           void* stream) {
  return tape_ew<double>(op, rows, cols, aux, x, y, s, c, out, accumulate, ws, ws_bytes,
                         reinterpret_cast<cudaStream_t>(stream));
}
dla_status dla_tape_ew_f32(int op, int64_t rows, int64_t cols, int64_t aux, const float* x, const float* y,
                           const float* s, float c, float* out, int accumulate, void* ws, size_t ws_bytes,
                           void* stream) {
  return tape_ew<float>(op, rows, cols, aux, x, y, s, c, out, accumulate, ws, ws_bytes,
                        reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
