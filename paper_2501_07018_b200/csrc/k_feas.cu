// Elementwise kernels of the Appendix-B fixed-restart feasibility harness
// (reference proj/tests/feasibility_method.hpp:40-85): restarted primal-dual
// steps for  find x >= 0 with A x = b  at a fixed step size.  The products
// are the SpMV kernels (sequential per line in parity mode, matching
// gen_detail::row_product / col_product, generator.hpp:108-136); these
// kernels carry the per-entry arithmetic in the reference's order (built
// with -fmad=false, so no contraction).
#include <cstdint>

#include "kernels.h"

namespace pdlp {
namespace {

constexpr int kT = 256;

inline int blocks(int64_t n) {
  const int64_t b = (n + kT - 1) / kT;
  return static_cast<int>(b < 148 * 16 ? (b < 1 ? 1 : b) : 148 * 16);
}

// feasibility_step, primal half (feasibility_method.hpp:46-52) plus the
// round's running sum (:71):  next = max(0, x - eta aty);  scratch =
// 2 next - x;  x = next;  x_sum += x.  std::max(0.0, v) keeps 0.0 unless
// 0.0 < v (NaN and -0.0 give +0.0).
__global__ void __launch_bounds__(kT) feas_primal_kernel(double* __restrict__ x,
                                                         const double* __restrict__ aty,
                                                         double* __restrict__ scratch,
                                                         double* __restrict__ x_sum, double eta,
                                                         int64_t n) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double xi = x[i];
    const double v = xi - eta * aty[i];
    const double next = 0.0 < v ? v : 0.0;
    scratch[i] = 2.0 * next - xi;
    x[i] = next;
    x_sum[i] = x_sum[i] + next;
  }
}

// Dual half (:54-56):  y -= eta (b - A scratch).
__global__ void __launch_bounds__(kT) feas_dual_kernel(double* __restrict__ y,
                                                       const double* __restrict__ b,
                                                       const double* __restrict__ ax_mid,
                                                       double eta, int64_t m) {
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < m;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    y[j] = y[j] - eta * (b[j] - ax_mid[j]);
  }
}

// End of a round (:73-81) and start of the next (:66-69): x_start = x_sum /
// restart_length; flag[0] = 0 if any entry is not finite; x = x_start,
// x_sum = 0.  (y is reset by the caller.)
__global__ void __launch_bounds__(kT) feas_average_kernel(double* __restrict__ x_start,
                                                          double* __restrict__ x,
                                                          double* __restrict__ x_sum,
                                                          double len, int64_t n,
                                                          int32_t* __restrict__ finite) {
  bool bad = false;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double v = x_sum[i] / len;
    x_start[i] = v;
    x[i] = v;
    x_sum[i] = 0.0;
    bad |= !(v - v == 0.0);  // NaN or +-inf
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) *finite = 0;
}

}  // namespace
}  // namespace pdlp

using namespace pdlp;

extern "C" {

int pdlpk_feas_primal(double* x, const double* aty, double* scratch, double* x_sum, double eta,
                      int64_t n, cudaStream_t s) {
  if (n > 0) feas_primal_kernel<<<blocks(n), kT, 0, s>>>(x, aty, scratch, x_sum, eta, n);
  return static_cast<int>(cudaGetLastError());
}

int pdlpk_feas_dual(double* y, const double* b, const double* ax_mid, double eta, int64_t m,
                    cudaStream_t s) {
  if (m > 0) feas_dual_kernel<<<blocks(m), kT, 0, s>>>(y, b, ax_mid, eta, m);
  return static_cast<int>(cudaGetLastError());
}

int pdlpk_feas_average(double* x_start, double* x, double* x_sum, double len, int64_t n,
                       int32_t* finite, cudaStream_t s) {
  if (n > 0) feas_average_kernel<<<blocks(n), kT, 0, s>>>(x_start, x, x_sum, len, n, finite);
  return static_cast<int>(cudaGetLastError());
}

}  // extern "C"
