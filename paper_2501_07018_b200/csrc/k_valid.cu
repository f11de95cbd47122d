// Problem validation on device (reference problem.hpp:119-154 and
// sparse.hpp:118-133), so a solve never walks the matrix on the host.
//
// First-failure scans reproduce the reference's loop order: each scan
// atomicMin's a key (index << 3 | condition) so the host recovers the first
// failing index and which of its conditions failed first.
//
// layouts_consistent (rebuild the row form from the column form and compare)
// is checked as the equivalent set of conditions:
//   * both row-pointer arrays start at 0, never decrease, end at nnz;
//   * every secondary index is in range; equal nnz;
//   * row lines are strictly increasing (sorted, duplicate free);
//   * every column entry (r, c, v) is found in row r at column c with an
//     equal value (binary search), and each row receives exactly as many
//     column entries as it holds.
// Together these make the column entries a bijection onto the row entries,
// which is what the rebuild comparison asserts.  Large layouts take the
// rebuild itself instead: a stable radix sort of the column entries by row
// (the column layout lists columns in ascending order, so each row's entries
// come out in ascending column order -- the row form) compared entry by
// entry with the row layout: the same rows, columns and values, position for
// position.  (Sort passes instead of a dependent binary search per entry:
// C2, 165.7M entries, 21 -> ~5 ms.)

#include <cub/cub.cuh>

#include "common.cuh"
#include "kernels.h"

namespace pdlp {
namespace {

constexpr int kT = 256;

inline int ew_blocks(int64_t n) {
  int64_t b = (n + kT - 1) / kT;
  if (b > 148 * 16) b = 148 * 16;
  return b < 1 ? 1 : static_cast<int>(b);
}

#define GRID_STRIDE(i, n)                                                                   \
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < (n); \
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)

__device__ __forceinline__ void first_fail(unsigned long long* slot, int64_t i, int code) {
  atomicMin(slot, (static_cast<unsigned long long>(i) << 3) | static_cast<unsigned long long>(code));
}

// keys[0] objective, keys[1] variable bounds, keys[2] constraint bounds,
// keys[3] matrix values (by_row).  Codes follow problem.hpp:127-152.
__global__ void vec_check_kernel(const double* c, const double* lv, const double* uv, int64_t n,
                                 const double* lc, const double* uc, int64_t m,
                                 unsigned long long* keys) {
  GRID_STRIDE(t, n + m) {
    if (t < n) {
      if (!finite_d(c[t])) first_fail(keys + 0, t, 1);
      const double lo = lv[t], hi = uv[t];
      int code = 0;
      if (isnan(lo) || isnan(hi)) code = 1;
      else if (lo == CUDART_INF) code = 2;
      else if (hi == -CUDART_INF) code = 3;
      else if (lo > hi) code = 4;
      if (code) first_fail(keys + 1, t, code);
    } else {
      const int64_t j = t - n;
      const double lo = lc[j], hi = uc[j];
      int code = 0;
      if (isnan(lo) || isnan(hi)) code = 1;
      else if (lo == CUDART_INF) code = 2;
      else if (hi == -CUDART_INF) code = 3;
      else if (lo > hi) code = 4;
      if (code) first_fail(keys + 2, j, code);
    }
  }
}

__global__ void value_check_kernel(const double* v, int64_t nnz, unsigned long long* keys) {
  GRID_STRIDE(k, nnz) {
    if (!finite_d(v[k])) first_fail(keys + 3, k, 1);
  }
}

// Raw int64 row pointers and indices (before the int32 conversion).
template <class T>
__global__ void ptr_check_kernel(const T* start, int64_t dim, int64_t nnz, unsigned* bad) {
  GRID_STRIDE(r, dim + 1) {
    const int64_t a = start[r];
    if (r == 0 && a != 0) atomicOr(bad, 1u);
    if (r == dim && a != nnz) atomicOr(bad, 1u);
    if (r < dim && start[r + 1] < a) atomicOr(bad, 1u);
  }
}

template <class T>
__global__ void index_range_kernel(const T* idx, int64_t count, int64_t bound, unsigned* bad) {
  GRID_STRIDE(k, count) {
    const int64_t v = idx[k];
    if (v < 0 || v >= bound) atomicOr(bad, 2u);
  }
}

// Row lines strictly increasing: consecutive entries of the same line.
__global__ void sorted_check_kernel(const int32_t* idx, const int32_t* line_of, int64_t nnz,
                                    unsigned* bad) {
  GRID_STRIDE(k, nnz - 1) {
    if (line_of[k] == line_of[k + 1] && !(idx[k] < idx[k + 1])) atomicOr(bad, 4u);
  }
}

template <class P>
__global__ void match_kernel(const P* __restrict__ rstart, const int32_t* __restrict__ ridx,
                             const double* __restrict__ rval, const int32_t* __restrict__ cidx,
                             const double* __restrict__ cval, const int32_t* __restrict__ col_of,
                             int64_t nnz, int* __restrict__ row_count, unsigned* bad) {
  GRID_STRIDE(k, nnz) {
    const int32_t r = cidx[k];
    const int32_t c = col_of[k];
    int64_t lo = rstart[r], hi = rstart[r + 1];
    while (lo < hi) {  // lower_bound of c in row r
      const int64_t mid = (lo + hi) >> 1;
      if (ridx[mid] < c) lo = mid + 1; else hi = mid;
    }
    if (lo >= rstart[r + 1] || ridx[lo] != c || !(rval[lo] == cval[k])) atomicOr(bad, 8u);
    atomicAdd(row_count + r, 1);
  }
}

__global__ void narrow_kernel(const int64_t* __restrict__ src, int32_t* __restrict__ dst, int64_t n) {
  GRID_STRIDE(k, n) {
    const int64_t x = src[k];
    dst[k] = x < 0 ? -1 : (x > INT32_MAX ? INT32_MAX : static_cast<int32_t>(x));
  }
}

__global__ void iota_kernel(int32_t* v, int64_t n) {
  GRID_STRIDE(k, n) v[k] = static_cast<int32_t>(k);
}

// Position q of the rebuilt row form: row skeys[q], column col_of[k], value
// cval[k] (k = the column-layout position) against the row layout's entry q.
__global__ void rebuilt_match_kernel(const int32_t* __restrict__ skeys,
                                     const int32_t* __restrict__ svals,
                                     const int32_t* __restrict__ row_of,
                                     const int32_t* __restrict__ ridx,
                                     const double* __restrict__ rval,
                                     const int32_t* __restrict__ col_of,
                                     const double* __restrict__ cval, int64_t nnz, unsigned* bad) {
  GRID_STRIDE(q, nnz) {
    const int32_t k = svals[q];
    if (skeys[q] != row_of[q] || ridx[q] != col_of[k] || !(rval[q] == cval[k])) atomicOr(bad, 8u);
  }
}

template <class P>
__global__ void count_check_kernel(const P* __restrict__ rstart, int64_t dim,
                                   const int* __restrict__ row_count, unsigned* bad) {
  GRID_STRIDE(r, dim) {
    if (static_cast<int64_t>(row_count[r]) != rstart[r + 1] - rstart[r]) atomicOr(bad, 16u);
  }
}

}  // namespace
}  // namespace pdlp

using namespace pdlp;

extern "C" int pdlpk_validate_vectors(const double* c, const double* lv, const double* uv,
                                      int64_t n, const double* lc, const double* uc, int64_t m,
                                      const double* row_values, int64_t nnz,
                                      unsigned long long* keys, cudaStream_t s) {
  cudaMemsetAsync(keys, 0xff, 4 * sizeof(unsigned long long), s);
  if (n + m > 0) vec_check_kernel<<<ew_blocks(n + m), kT, 0, s>>>(c, lv, uv, n, lc, uc, m, keys);
  if (nnz > 0) value_check_kernel<<<ew_blocks(nnz), kT, 0, s>>>(row_values, nnz, keys);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int pdlpk_validate_raw_layout(const int64_t* start, int64_t dim, const int64_t* idx,
                                         int64_t count, int64_t nnz, int64_t bound, unsigned* bad,
                                         cudaStream_t s) {
  if (start != nullptr) ptr_check_kernel<<<ew_blocks(dim + 1), kT, 0, s>>>(start, dim, nnz, bad);
  if (idx != nullptr && count > 0) index_range_kernel<<<ew_blocks(count), kT, 0, s>>>(idx, count, bound, bad);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int pdlpk_validate_raw_layout32(const int32_t* start, int64_t dim, const int32_t* idx,
                                           int64_t count, int64_t nnz, int64_t bound,
                                           unsigned* bad, cudaStream_t s) {
  if (start != nullptr) ptr_check_kernel<<<ew_blocks(dim + 1), kT, 0, s>>>(start, dim, nnz, bad);
  if (idx != nullptr && count > 0) index_range_kernel<<<ew_blocks(count), kT, 0, s>>>(idx, count, bound, bad);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int pdlpk_narrow_i64(const int64_t* src, int32_t* dst, int64_t n, cudaStream_t s) {
  if (n > 0) narrow_kernel<<<ew_blocks(n), kT, 0, s>>>(src, dst, n);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int pdlpk_validate_consistency(const pdlpk_csr* R, const int32_t* row_of,
                                          const pdlpk_csr* Cl, const int32_t* col_of,
                                          int* row_count, unsigned* bad, cudaStream_t s) {
  const int64_t nnz = R->nnz;
  if (nnz > 1) sorted_check_kernel<<<ew_blocks(nnz - 1), kT, 0, s>>>(R->index, row_of, nnz, bad);
  if (nnz >= (int64_t(1) << 20) && nnz < (int64_t(1) << 31)) {
    int end_bit = 1;
    while (end_bit < 31 && (int64_t(1) << end_bit) < R->dim) ++end_bit;
    size_t tmp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, static_cast<const int32_t*>(nullptr),
                                    static_cast<int32_t*>(nullptr), static_cast<const int32_t*>(nullptr),
                                    static_cast<int32_t*>(nullptr), static_cast<int>(nnz), 0, end_bit, s);
    char* buf = nullptr;
    const size_t arr = (static_cast<size_t>(nnz) * 4 + 255) & ~size_t(255);
    if (cudaMallocAsync(reinterpret_cast<void**>(&buf), 3 * arr + tmp_bytes, s) == cudaSuccess) {
      int32_t* skeys = reinterpret_cast<int32_t*>(buf);
      int32_t* vin = reinterpret_cast<int32_t*>(buf + arr);
      int32_t* svals = reinterpret_cast<int32_t*>(buf + 2 * arr);
      iota_kernel<<<ew_blocks(nnz), kT, 0, s>>>(vin, nnz);
      const cudaError_t e = cub::DeviceRadixSort::SortPairs(buf + 3 * arr, tmp_bytes, Cl->index, skeys,
                                                           vin, svals, static_cast<int>(nnz), 0,
                                                           end_bit, s);
      if (e == cudaSuccess) {
        rebuilt_match_kernel<<<ew_blocks(nnz), kT, 0, s>>>(skeys, svals, row_of, R->index,
                                                           R->value_orig, col_of, Cl->value_orig,
                                                           nnz, bad);
      }
      cudaFreeAsync(buf, s);
      if (e != cudaSuccess) return static_cast<int>(e);
      return static_cast<int>(cudaGetLastError());
    }
    cudaGetLastError();  // out of memory: the binary-search form below
  }
  cudaMemsetAsync(row_count, 0, (R->dim > 0 ? R->dim : 1) * sizeof(int), s);
  if (nnz > 0) {
    if (R->wide) {
      match_kernel<int64_t><<<ew_blocks(nnz), kT, 0, s>>>(static_cast<const int64_t*>(R->start),
                                                          R->index, R->value_orig, Cl->index,
                                                          Cl->value_orig, col_of, nnz, row_count, bad);
    } else {
      match_kernel<int32_t><<<ew_blocks(nnz), kT, 0, s>>>(static_cast<const int32_t*>(R->start),
                                                          R->index, R->value_orig, Cl->index,
                                                          Cl->value_orig, col_of, nnz, row_count, bad);
    }
  }
  if (R->dim > 0) {
    if (R->wide) {
      count_check_kernel<int64_t><<<ew_blocks(R->dim), kT, 0, s>>>(static_cast<const int64_t*>(R->start), R->dim, row_count, bad);
    } else {
      count_check_kernel<int32_t><<<ew_blocks(R->dim), kT, 0, s>>>(static_cast<const int32_t*>(R->start), R->dim, row_count, bad);
    }
  }
  return static_cast<int>(cudaGetLastError());
}
