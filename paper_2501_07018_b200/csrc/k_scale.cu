// Diagonal preconditioning on device (reference rescaling.hpp:44-143):
// 10 Ruiz passes (sqrt of line inf-norms) + 1 Pock-Chambolle pass (sqrt of
// line 1-norms), dividing both layouts, bounds and objective.
//
// Load balance: entries are processed element-parallel through a per-entry
// line map (line_of[k], built once with a max-scan over line heads), so a
// 2,000-entry row costs the same as 2,000 one-entry rows.
//   * inf-norms: atomicMax on the bit patterns of |a| (non-negative doubles
//     order like their bits) — order-free, so exact;
//   * 1-norms:   one thread per line, sequential in storage order — the
//     reference's summation order, run once per solve;
//   * apply:     a /= f_line * f_index elementwise — exact.
// Translation unit compiled with -fmad=false (see common.cuh).

#include <cub/cub.cuh>

#include "common.cuh"
#include "kernels.h"

namespace pdlp {
namespace {

constexpr int kT = 256;

inline int ew_blocks(int64_t n, int64_t cap = 148 * 16) {
  int64_t b = (n + kT - 1) / kT;
  if (b > cap) b = cap;
  return b < 1 ? 1 : static_cast<int>(b);
}

#define GRID_STRIDE(i, n)                                                                   \
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < (n); \
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)

template <class P>
__global__ void mark_heads(const P* __restrict__ start, int64_t dim, int32_t* __restrict__ line_of) {
  GRID_STRIDE(r, dim) {
    const int64_t a = start[r], b = start[r + 1];
    if (a < b) line_of[a] = static_cast<int32_t>(r);
  }
}

// Line inf-norms, warp-coalesced: lane l of a warp takes entry base + l
// (coalesced loads of the values and the line map), a segmented max over the
// warp's 32 entries (a line is a run of equal line_of, which is
// non-decreasing in k) leaves each run's max on its last lane, and that lane
// does one atomicMax on the line's bits.  A 2,000-entry line costs ~63
// atomics; order-free, so exact.
__device__ __forceinline__ void seg_max_flush(int32_t line, unsigned long long a, bool valid,
                                              unsigned long long* __restrict__ bits) {
  const int lane = threadIdx.x & 31;
  if (!valid) line = -1 - lane;  // never joins a run
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xffffffffu, a, o);
    const int32_t tl = __shfl_up_sync(0xffffffffu, line, o);
    if (lane >= o && tl == line) a = t > a ? t : a;
  }
  const int32_t next = __shfl_down_sync(0xffffffffu, line, 1);
  if (valid && (lane == 31 || next != line)) atomicMax(bits + line, a);
}

__device__ __forceinline__ unsigned long long abs_bits(double v) {
  return static_cast<unsigned long long>(__double_as_longlong(fabs(v)));
}

#define WARP_STRIDE(base, n)                                                                    \
  for (int64_t base = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) & ~int64_t(31); \
       base < (n); base += static_cast<int64_t>(gridDim.x) * blockDim.x)

__global__ void absmax_kernel(const double* __restrict__ val, const int32_t* __restrict__ line_of,
                              int64_t nnz, unsigned long long* __restrict__ bits) {
  const int lane = threadIdx.x & 31;
  WARP_STRIDE(base, nnz) {
    const int64_t k = base + lane;
    const bool valid = k < nnz;
    seg_max_flush(valid ? line_of[k] : 0, valid ? abs_bits(val[k]) : 0ull, valid, bits);
  }
}

// One Ruiz pass's division (apply_elem) fused with the next pass's line
// inf-norms of the result (bits_next != nullptr).
__global__ void apply_max_kernel(double* __restrict__ val, const int32_t* __restrict__ idx,
                                 const int32_t* __restrict__ line_of, int64_t nnz,
                                 const double* __restrict__ fp, const double* __restrict__ fs,
                                 unsigned long long* __restrict__ bits_next) {
  const int lane = threadIdx.x & 31;
  WARP_STRIDE(base, nnz) {
    const int64_t k = base + lane;
    const bool valid = k < nnz;
    int32_t line = 0;
    double v = 0.0;
    if (valid) {
      line = line_of[k];
      v = val[k] / (fp[line] * fs[idx[k]]);
      val[k] = v;
    }
    if (bits_next != nullptr) seg_max_flush(line, valid ? abs_bits(v) : 0ull, valid, bits_next);
  }
}

__global__ void factor_from_bits(const unsigned long long* __restrict__ bits, int64_t dim,
                                 double* __restrict__ f) {
  GRID_STRIDE(r, dim) {
    const double mx = __longlong_as_double(static_cast<long long>(bits[r]));
    f[r] = mx > 0.0 ? sqrt(mx) : 1.0;
  }
}

template <class P>
__global__ void onenorm_factor(const P* __restrict__ start, const double* __restrict__ val,
                               int64_t dim, double* __restrict__ f) {
  GRID_STRIDE(r, dim) {
    double a = 0.0;
    for (int64_t k = start[r]; k < start[r + 1]; ++k) a += fabs(val[k]);  // rescaling.hpp:111-116
    f[r] = a > 0.0 ? sqrt(a) : 1.0;
  }
}

__global__ void apply_elem(double* __restrict__ val, const int32_t* __restrict__ idx,
                           const int32_t* __restrict__ line_of, int64_t nnz,
                           const double* __restrict__ fp, const double* __restrict__ fs) {
  GRID_STRIDE(k, nnz) val[k] = val[k] / (fp[line_of[k]] * fs[idx[k]]);
}

__global__ void bits_to_norm(const unsigned long long* __restrict__ bits, int64_t dim,
                             double* __restrict__ norm) {
  GRID_STRIDE(r, dim) norm[r] = __longlong_as_double(static_cast<long long>(bits[r]));
}

template <class P>
__global__ void onenorm_kernel(const P* __restrict__ start, const double* __restrict__ val,
                               int64_t dim, double* __restrict__ norm) {
  GRID_STRIDE(r, dim) {
    double a = 0.0;
    for (int64_t k = start[r]; k < start[r + 1]; ++k) a += fabs(val[k]);
    norm[r] = a;
  }
}

// acc[r] continues the sequential 1-norm of line r over this layout's
// entries (row-sharded: each rank holds one consecutive run of every column).
template <class P>
__global__ void onenorm_continue_kernel(const P* __restrict__ start, const double* __restrict__ val,
                                        int64_t dim, double* __restrict__ acc) {
  GRID_STRIDE(r, dim) {
    double a = acc[r];
    for (int64_t k = start[r]; k < start[r + 1]; ++k) a += fabs(val[k]);
    acc[r] = a;
  }
}

__global__ void norm_factor(double* __restrict__ f, int64_t n) {
  GRID_STRIDE(r, n) {
    const double a = f[r];
    f[r] = a > 0.0 ? sqrt(a) : 1.0;
  }
}

struct MaxOp {
  __device__ __forceinline__ int32_t operator()(int32_t a, int32_t b) const { return a > b ? a : b; }
};

}  // namespace
}  // namespace pdlp

using namespace pdlp;

extern "C" size_t pdlpk_line_of_work_bytes(int64_t nnz) {
  size_t bytes = 0;
  cub::DeviceScan::InclusiveScan(nullptr, bytes, static_cast<int32_t*>(nullptr),
                                 static_cast<int32_t*>(nullptr), MaxOp{}, static_cast<int>(nnz));
  return bytes + 256;
}

extern "C" int pdlpk_line_of(const pdlpk_csr* A, int32_t* line_of, void* work, size_t work_bytes,
                             cudaStream_t s) {
  if (A->nnz == 0) return 0;
  cudaMemsetAsync(line_of, 0, A->nnz * sizeof(int32_t), s);
  if (A->wide) {
    mark_heads<int64_t><<<ew_blocks(A->dim), kT, 0, s>>>(static_cast<const int64_t*>(A->start), A->dim, line_of);
  } else {
    mark_heads<int32_t><<<ew_blocks(A->dim), kT, 0, s>>>(static_cast<const int32_t*>(A->start), A->dim, line_of);
  }
  size_t bytes = work_bytes;
  const cudaError_t e = cub::DeviceScan::InclusiveScan(work, bytes, line_of, line_of, MaxOp{},
                                                       static_cast<int>(A->nnz), s);
  if (e != cudaSuccess) return static_cast<int>(e);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int pdlpk_line_factors(const pdlpk_csr* A, const int32_t* line_of, int32_t one_norm,
                                  double* f, unsigned long long* bits, cudaStream_t s) {
  if (A->dim == 0) return 0;
  if (one_norm) {
    if (A->wide) {
      onenorm_factor<int64_t><<<ew_blocks(A->dim), kT, 0, s>>>(static_cast<const int64_t*>(A->start), A->value, A->dim, f);
    } else {
      onenorm_factor<int32_t><<<ew_blocks(A->dim), kT, 0, s>>>(static_cast<const int32_t*>(A->start), A->value, A->dim, f);
    }
    return static_cast<int>(cudaGetLastError());
  }
  cudaMemsetAsync(bits, 0, A->dim * sizeof(unsigned long long), s);
  if (A->nnz > 0) {
    absmax_kernel<<<ew_blocks(A->nnz), kT, 0, s>>>(A->value, line_of, A->nnz, bits);
  }
  factor_from_bits<<<ew_blocks(A->dim), kT, 0, s>>>(bits, A->dim, f);
  return static_cast<int>(cudaGetLastError());
}

// Ruiz on one GPU (Engine::precondition): the line inf-norms of both layouts
// once, then per pass factors from the bits and the fused division + next
// norms.  Same maxima, same divisions as line_factors + apply_factors.
extern "C" int pdlpk_line_absmax(const pdlpk_csr* A, const int32_t* line_of,
                                 unsigned long long* bits, cudaStream_t s) {
  if (A->dim == 0) return 0;
  cudaMemsetAsync(bits, 0, A->dim * sizeof(unsigned long long), s);
  if (A->nnz > 0) absmax_kernel<<<ew_blocks(A->nnz), kT, 0, s>>>(A->value, line_of, A->nnz, bits);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int pdlpk_factors_from_bits(const unsigned long long* bits, int64_t dim, double* f,
                                       cudaStream_t s) {
  if (dim > 0) factor_from_bits<<<ew_blocks(dim), kT, 0, s>>>(bits, dim, f);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int pdlpk_apply_factors_max(const pdlpk_csr* A, const int32_t* line_of, double* value,
                                       const double* f_primary, const double* f_secondary,
                                       unsigned long long* bits_next, cudaStream_t s) {
  if (bits_next != nullptr && A->dim > 0) {
    cudaMemsetAsync(bits_next, 0, A->dim * sizeof(unsigned long long), s);
  }
  if (A->nnz == 0) return static_cast<int>(cudaGetLastError());
  apply_max_kernel<<<ew_blocks(A->nnz), kT, 0, s>>>(value, A->index, line_of, A->nnz, f_primary,
                                                   f_secondary, bits_next);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int pdlpk_apply_factors(const pdlpk_csr* A, const int32_t* line_of, double* value,
                                   const double* f_primary, const double* f_secondary,
                                   cudaStream_t s) {
  if (A->nnz == 0) return 0;
  apply_elem<<<ew_blocks(A->nnz), kT, 0, s>>>(value, A->index, line_of, A->nnz, f_primary, f_secondary);
  return static_cast<int>(cudaGetLastError());
}

// Row-sharded preconditioning: a rank's K^T block holds partial column norms
// (its rows only); the engine combines them across ranks (max / sum) before
// norm_to_factor.
extern "C" int pdlpk_line_norms(const pdlpk_csr* A, const int32_t* line_of, int32_t one_norm,
                                double* norm, unsigned long long* bits, cudaStream_t s) {
  if (A->dim == 0) return 0;
  if (one_norm) {
    if (A->wide) {
      onenorm_kernel<int64_t><<<ew_blocks(A->dim), kT, 0, s>>>(static_cast<const int64_t*>(A->start), A->value, A->dim, norm);
    } else {
      onenorm_kernel<int32_t><<<ew_blocks(A->dim), kT, 0, s>>>(static_cast<const int32_t*>(A->start), A->value, A->dim, norm);
    }
    return static_cast<int>(cudaGetLastError());
  }
  cudaMemsetAsync(bits, 0, A->dim * sizeof(unsigned long long), s);
  if (A->nnz > 0) {
    absmax_kernel<<<ew_blocks(A->nnz), kT, 0, s>>>(A->value, line_of, A->nnz, bits);
  }
  bits_to_norm<<<ew_blocks(A->dim), kT, 0, s>>>(bits, A->dim, norm);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int pdlpk_norm_to_factor(double* f, int64_t n, cudaStream_t s) {
  if (n > 0) norm_factor<<<ew_blocks(n), kT, 0, s>>>(f, n);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int pdlpk_line_onenorm_continue(const pdlpk_csr* A, double* acc, cudaStream_t s) {
  if (A->dim == 0) return 0;
  if (A->wide) {
    onenorm_continue_kernel<int64_t><<<ew_blocks(A->dim), kT, 0, s>>>(static_cast<const int64_t*>(A->start), A->value, A->dim, acc);
  } else {
    onenorm_continue_kernel<int32_t><<<ew_blocks(A->dim), kT, 0, s>>>(static_cast<const int32_t*>(A->start), A->value, A->dim, acc);
  }
  return static_cast<int>(cudaGetLastError());
}
