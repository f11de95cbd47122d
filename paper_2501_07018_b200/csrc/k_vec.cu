// Cadence-time device operations: plain products, residual screens, ray
// tests, averages, preconditioning and setup conversions.  Each operation
// cites the reference function whose arithmetic it reproduces; in parity
// mode every sum runs in the reference's order (SEQ / SHARD, reduce.cuh).
//
// Translation unit compiled with -fmad=false (see common.cuh).

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "reduce.cuh"
#include "spmv.cuh"

namespace pdlp {
namespace {

constexpr int kT = 256;

inline int ew_blocks(int64_t n) {
  int64_t b = (n + kT - 1) / kT;
  if (b > 148 * 8) b = 148 * 8;
  return b < 1 ? 1 : static_cast<int>(b);
}

// Bitwise OR / AND of the patterns of v (exact, order-free).
__global__ void __launch_bounds__(kT) uniform_bits_kernel(const double* __restrict__ v, int64_t n,
                                                          unsigned long long* or_and) {
  pdl_wait_cadence();
  unsigned long long o = 0ull, a = ~0ull;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v[i]));
    o |= b;
    a &= b;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    o |= __shfl_xor_sync(0xffffffffu, o, d);
    a &= __shfl_xor_sync(0xffffffffu, a, d);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicOr(or_and, o);
    atomicAnd(or_and + 1, a);
  }
}

#define GRID_STRIDE(i, n)                                                                   \
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < (n); \
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)

inline int ok() { return static_cast<int>(cudaGetLastError()); }

// -------------------------------------------------------------- products ---
// cond: optional device flag; the product is skipped when *cond == 0.
template <class P>
__global__ void __launch_bounds__(kT) seq_spmv_kernel(const P* __restrict__ start,
                                                      const int32_t* __restrict__ idx,
                                                      const double* __restrict__ val,
                                                      const double* __restrict__ v,
                                                      double* __restrict__ out, int64_t dim,
                                                      const double* cond) {
  pdl_wait_cadence();
  if (cond != nullptr && *cond == 0.0) return;
  GRID_STRIDE(r, dim) {
    double acc = 0.0;
    for (int64_t k = start[r]; k < start[r + 1]; ++k) acc = acc + val[k] * v[idx[k]];
    out[r] = acc;
  }
}

struct StoreEpi {
  double* out;
  struct Pre {};
  __device__ __forceinline__ Pre load(int64_t) const { return {}; }
  static constexpr int kStaged = 0;
  __device__ __forceinline__ const double* staged_src(int) const { return nullptr; }
  __device__ __forceinline__ bool staged_reused(int) const { return false; }
  __device__ __forceinline__ Pre from_stage(const double* const*, int) const { return {}; }
  __device__ __forceinline__ void reset_acc() {}
  __device__ __forceinline__ void export_acc(double*) const {}
  __device__ __forceinline__ double init(const Pre&) const { return 0.0; }
  __device__ __forceinline__ void prefetch(int64_t) const {}
  __device__ __forceinline__ void line(int64_t r, double acc, const Pre&) { out[r] = acc; }
};

template <class P, int Seg>
__global__ void __launch_bounds__(kSpmvThreads, spmv_min_blocks(Seg)) sched_spmv_kernel(pdlpk_csr A,
                                                                  const double* vals,
                                                                  const double* v, double* out,
                                                                  const double* cond) {
  pdl_wait_cadence();
  if (cond != nullptr && *cond == 0.0) return;
  StoreEpi e{out};
  sched_spmv<P, Seg>(A, vals, v, e);
}

struct LaunchSpmv {
  const pdlpk_csr* A;
  const double* vals;
  const double* v;
  double* out;
  const double* cond;
  cudaStream_t s;
  template <class P, int Seg>
  int go() {
    const int64_t g = sched_blocks(*A);
    if (g > 0) {
      const size_t smem = spmv_smem(*A, Seg);
      allow_smem(sched_spmv_kernel<P, Seg>, smem);
      launch_pdl(PDLPK_PDL_CADENCE, sched_spmv_kernel<P, Seg>, static_cast<unsigned>(g), kSpmvThreads, smem, s,
                 *A, vals, v, out, cond);
    }
    return ok();
  }
};

// ------------------------------------------------------------ elementwise ---
__global__ void fill_kernel(double* x, double v, int64_t n) {
  pdl_wait_cadence();
  GRID_STRIDE(i, n) x[i] = v;
}

__global__ void combine_slots_kernel(const double* all, int world, int stride, uint64_t marked,
                                     uint64_t maxbits, double* slots) {
  pdl_wait_cadence();
  const int i = threadIdx.x;
  if (i >= 64 || !((marked >> i) & 1ull)) return;
  const bool mx = (maxbits >> i) & 1ull;
  double t = all[i];
  for (int r = 1; r < world; ++r) {
    const double v = all[static_cast<int64_t>(r) * stride + i];
    t = mx ? max_keep(t, v) : t + v;
  }
  slots[i] = t;
}

__global__ void accumulate_kernel(double* out, const double* in, int64_t n, int use_max) {
  pdl_wait_cadence();
  GRID_STRIDE(i, n) out[i] = use_max ? max_keep(out[i], in[i]) : out[i] + in[i];
}

__global__ void sub_kernel(const double* a, const double* b, double* out, int64_t n) {
  pdl_wait_cadence();
  GRID_STRIDE(i, n) out[i] = a[i] - b[i];
}

__global__ void scale_div_kernel(const double* scale, const double* v, double* out, int64_t n) {
  pdl_wait_cadence();
  GRID_STRIDE(i, n) out[i] = v[i] / scale[i];
}

__global__ void scale_mul_kernel(const double* scale, const double* v, double* out, int64_t n) {
  pdl_wait_cadence();
  GRID_STRIDE(i, n) out[i] = scale[i] * v[i];
}

__global__ void average_into_kernel(const pdlpk_step_state* st, const double* sx,
                                    const double* sy, double* x, double* y, int64_t n,
                                    int64_t m) {
  pdl_wait_cadence();
  const double inv = 1.0 / st->avg_weight;
  GRID_STRIDE(i, n + m) {
    if (i < n) {
      x[i] = inv * sx[i];
    } else {
      y[i - n] = inv * sy[i - n];
    }
  }
}

__global__ void initial_point_kernel(const double* lv, const double* uv, double* x, int64_t n) {
  pdl_wait_cadence();
  GRID_STRIDE(i, n) x[i] = clampd(0.0, lv[i], uv[i]);
}

__global__ void dual_feas_bounds_kernel(const double* c, const double* lv, const double* uv,
                                        int64_t n, const double* lc, const double* uc,
                                        int64_t m, double* slc, double* suc, double* slv,
                                        double* suv) {
  pdl_wait_cadence();
  GRID_STRIDE(t, n + m) {
    if (t < n) {
      const int64_t i = t;
      const double ci = c[i];
      switch (cone_of_bounds(lv[i], uv[i])) {
        case kZero: slc[i] = ci; suc[i] = ci; break;
        case kNonNeg: slc[i] = -CUDART_INF; suc[i] = ci; break;
        case kNonPos: slc[i] = ci; suc[i] = CUDART_INF; break;
        default: slc[i] = -CUDART_INF; suc[i] = CUDART_INF; break;
      }
    } else {
      const int64_t j = t - n;
      switch (cone_of_bounds(lc[j], uc[j])) {
        case kZero: slv[j] = 0.0; suv[j] = 0.0; break;
        case kNonNeg: slv[j] = 0.0; suv[j] = CUDART_INF; break;
        case kNonPos: slv[j] = -CUDART_INF; suv[j] = 0.0; break;
        default: slv[j] = -CUDART_INF; suv[j] = CUDART_INF; break;
      }
    }
  }
}

__global__ void i64_to_i32_kernel(const int64_t* src, int32_t* dst, int64_t n) {
  pdl_wait_cadence();
  GRID_STRIDE(i, n) dst[i] = static_cast<int32_t>(src[i]);
}

__global__ void radius_kernel(const double* dx2, const double* dy2, double omega, double* out) {
  pdl_wait_cadence();
  *out = sqrt(omega * (*dx2) + (*dy2) / omega);
}

// ------------------------------------------------------ preconditioning ---
// (line norms and matrix scaling live in k_scale.cu)
__global__ void apply_vec_factor_kernel(double* lc, double* uc, double* rs, const double* fr,
                                        int64_t m, double* c, double* lv, double* uv,
                                        double* cs, const double* fc, int64_t n) {
  pdl_wait_cadence();
  GRID_STRIDE(t, m + n) {
    if (t < m) {
      const double f = fr[t];
      lc[t] = lc[t] / f;
      uc[t] = uc[t] / f;
      rs[t] = rs[t] / f;
    } else {
      const int64_t i = t - m;
      const double f = fc[i];
      c[i] = c[i] / f;
      lv[i] = lv[i] * f;
      uv[i] = uv[i] * f;
      cs[i] = cs[i] / f;
    }
  }
}

__global__ void find_nonfinite_kernel(const double* v, int64_t n, int32_t code, int32_t* first) {
  pdl_wait_cadence();
  GRID_STRIDE(i, n) {
    if (!finite_d(v[i])) atomicMin(reinterpret_cast<int*>(first + 1), static_cast<int>(i));
  }
  (void)code;
}

// Reduced cost of coordinate i (recover_reduced_costs_from, residuals.hpp:29-47).
__device__ __forceinline__ double reduced_cost(double c, double aty, double x, double lv,
                                               double uv, int rc_mode) {
  const double v = c - aty;
  if (rc_mode == 0) return cone_project(v, cone_of_bounds(lv, uv));
  if (v > 0.0 && x - lv <= fabs(x)) return v;
  if (v < 0.0 && uv - x <= fabs(x)) return v;
  return 0.0;
}

// Penalty term of dual_objective_value (residuals.hpp:77-96) for multiplier
// value w against bounds (lo, hi): v = -w; hi*v if v > 0, lo*v if v < 0.
__device__ __forceinline__ bool penalty_term(double w, double lo, double hi, double& out) {
  const double v = -w;
  if (v > 0.0) {
    out = mul_zero_inf(hi, v);
    return true;
  }
  if (v < 0.0) {
    out = mul_zero_inf(lo, v);
    return true;
  }
  return false;
}

}  // namespace
}  // namespace pdlp

using namespace pdlp;

// Column panels of the row layout (kernels.h pdlpk_step_args::n_row_panels):
// entry k of row r (rows sorted by column) goes to panel q = its column's
// range, at pp.start[q][r] + its rank among row r's panel-q entries.  Warp per
// row, lanes over the row's entries.
template <class P>
__global__ void __launch_bounds__(kT) panel_scatter_kernel(const P* __restrict__ start,
                                                          const int32_t* __restrict__ idx,
                                                          const double* __restrict__ val, int64_t m,
                                                          pdlpk_panel_ptrs pp) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = w0; r < m; r += nw) {
    const int64_t s = start[r], e = start[r + 1];
    int64_t cum[PDLPK_MAX_ROW_PANELS + 1];
    int64_t pos[PDLPK_MAX_ROW_PANELS];
    cum[0] = 0;
    for (int q = 0; q < pp.np; ++q) {
      pos[q] = pp.start[q][r];
      cum[q + 1] = cum[q] + (pp.start[q][r + 1] - pos[q]);
    }
    for (int64_t k = s + lane; k < e; k += 32) {
      const int64_t o = k - s;
      int q = 0;
      while (q + 1 < pp.np && o >= cum[q + 1]) ++q;
      const int64_t d = pos[q] + (o - cum[q]);
      pp.idx[q][d] = idx[k];
      pp.val[q][d] = val[k];
    }
  }
}

extern "C" {

int64_t pdlpk_red_scratch_doubles(void) { return 8 * kRedMaxBlocks; }

int pdlpk_uniform_bits(const double* v, int64_t n, unsigned long long* or_and, cudaStream_t s) {
  if (n > 0) launch_pdl(PDLPK_PDL_CADENCE, uniform_bits_kernel, static_cast<unsigned>(ew_blocks(n)), kT, 0, s, v, n, or_and);
  return ok();
}

int pdlpk_index_to_i32(const int64_t* src, int32_t* dst, int64_t n, cudaStream_t s) {
  if (n > 0) launch_pdl(PDLPK_PDL_CADENCE, i64_to_i32_kernel, static_cast<unsigned>(ew_blocks(n)), kT, 0, s, src, dst, n);
  return ok();
}

int pdlpk_start_to_i32(const int64_t* src, int32_t* dst, int64_t n, cudaStream_t s) {
  return pdlpk_index_to_i32(src, dst, n, s);
}

int pdlpk_spmv_cond(const pdlpk_csr* A, int32_t orig, const double* v, double* out,
                    int32_t parity, const double* cond, cudaStream_t s) {
  if (A->dim == 0) return 0;
  const double* vals = orig ? A->value_orig : A->value;
  if (parity) {
    const int g = ew_blocks(A->dim);
    if (A->wide) {
      launch_pdl(PDLPK_PDL_CADENCE, seq_spmv_kernel<int64_t>, static_cast<unsigned>(g), kT, 0, s,
                 static_cast<const int64_t*>(A->start), static_cast<const int32_t*>(A->index), vals,
                 v, out, A->dim, cond);
    } else {
      launch_pdl(PDLPK_PDL_CADENCE, seq_spmv_kernel<int32_t>, static_cast<unsigned>(g), kT, 0, s,
                 static_cast<const int32_t*>(A->start), static_cast<const int32_t*>(A->index), vals,
                 v, out, A->dim, cond);
    }
    return ok();
  }
  return dispatch_p(*A, LaunchSpmv{A, vals, v, out, cond, s});
}

int pdlpk_spmv(const pdlpk_csr* A, int32_t orig, const double* v, double* out, int32_t parity,
               cudaStream_t s) {
  return pdlpk_spmv_cond(A, orig, v, out, parity, nullptr, s);
}

int pdlpk_diff_norm_sq(const double* a, const double* b, int64_t n, const pdlpk_red* red,
                       double* slot, cudaStream_t s) {
  auto f = [a, b] __device__(int64_t i, double* v) -> unsigned {
    const double d = a[i] - b[i];
    v[0] = d * d;
    return 1u;
  };
  return multi_reduce<1>(f, n, red->parity ? PDLPK_RED_SHARD : PDLPK_RED_TREE, red->shards, 0u,
                         red->scratch, slot, s);
}

void pdlpk_set_red_log(pdlpk_red_log* log) { g_red_log = log; }

int pdlpk_panel_scatter(const pdlpk_csr* K, const pdlpk_panel_ptrs* pp, cudaStream_t s) {
  if (K->dim <= 0) return 0;
  const unsigned g = static_cast<unsigned>(std::min<int64_t>((K->dim + 7) / 8, 148 * 16));
  if (K->wide) {
    panel_scatter_kernel<<<g, kT, 0, s>>>(static_cast<const int64_t*>(K->start), K->index, K->value,
                                          K->dim, *pp);
  } else {
    panel_scatter_kernel<<<g, kT, 0, s>>>(static_cast<const int32_t*>(K->start), K->index, K->value,
                                          K->dim, *pp);
  }
  return ok();
}

void pdlpk_tile_shape(double avg_len, int32_t budget, int32_t* lines, int32_t* nnz,
                      int32_t* stage_bytes, int32_t staged) {
  const int ns = staged < 0 ? kDefaultStaged : staged;
  const double a = avg_len < 1.0 ? 1.0 : avg_len;
  int L = kTileRows;
  while (L > 32 && static_cast<double>(stage_nnz_for(L, budget, ns)) < a * L) L -= 8;
  const int E = stage_nnz_for(L, budget, ns);
  *lines = L;
  *nnz = E;
  *stage_bytes = static_cast<int32_t>(stage_layout(L, E, ns).bytes);
}

int32_t pdlpk_stage_budget(int32_t nnz) {
  return static_cast<int32_t>(stage_layout(kTileRows, nnz).bytes);
}

int pdlpk_combine_slots(const double* all, int32_t world, int32_t stride, uint64_t marked,
                        uint64_t maxbits, double* slots, cudaStream_t s) {
  if (marked != 0) launch_pdl(PDLPK_PDL_CADENCE, combine_slots_kernel, static_cast<unsigned>(1), 64, 0, s, all, world, stride, marked, maxbits, slots);
  return ok();
}

int pdlpk_accumulate(double* out, const double* in, int64_t n, int32_t use_max, cudaStream_t s) {
  if (n > 0) launch_pdl(PDLPK_PDL_CADENCE, accumulate_kernel, static_cast<unsigned>(ew_blocks(n)), kT, 0, s, out, in, n, use_max);
  return ok();
}

int pdlpk_fill(double* x, double v, int64_t n, cudaStream_t s) {
  if (n > 0) launch_pdl(PDLPK_PDL_CADENCE, fill_kernel, static_cast<unsigned>(ew_blocks(n)), kT, 0, s, x, v, n);
  return ok();
}

int pdlpk_sub(const double* a, const double* b, double* out, int64_t n, cudaStream_t s) {
  if (n > 0) launch_pdl(PDLPK_PDL_CADENCE, sub_kernel, static_cast<unsigned>(ew_blocks(n)), kT, 0, s, a, b, out, n);
  return ok();
}

int pdlpk_average_into(const pdlpk_step_state* st, const double* sum_x, const double* sum_y,
                       double* x, double* y, int64_t n, int64_t m, cudaStream_t s) {
  if (n + m > 0) launch_pdl(PDLPK_PDL_CADENCE, average_into_kernel, static_cast<unsigned>(ew_blocks(n + m)), kT, 0, s, st, sum_x, sum_y, x, y, n, m);
  return ok();
}

int pdlpk_scale_div(const double* scale, const double* v, double* out, int64_t n, cudaStream_t s) {
  if (n > 0) scale_div_kernel<<<ew_blocks(n), kT, 0, s>>>(scale, v, out, n);
  return ok();
}

int pdlpk_scale_mul(const double* scale, const double* v, double* out, int64_t n,
                    cudaStream_t s) {
  if (n > 0) launch_pdl(PDLPK_PDL_CADENCE, scale_mul_kernel, static_cast<unsigned>(ew_blocks(n)), kT, 0, s, scale, v, out, n);
  return ok();
}

int pdlpk_screen(const pdlpk_problem* P, int32_t orig, const double* x, const double* y,
                 const double* ax, const double* aty, int32_t rc_mode, const pdlpk_red* red,
                 double* r_out, double* slots, cudaStream_t s) {
  const int64_t m = P->m, n = P->n;
  const double* c = orig ? P->c_o : P->c;
  const double* lc = orig ? P->lc_o : P->lc;
  const double* uc = orig ? P->uc_o : P->uc;
  const double* lv = orig ? P->lv_o : P->lv;
  const double* uv = orig ? P->uv_o : P->uv;
  const double* rs = orig ? nullptr : P->row_scale;
  const double* cs = orig ? nullptr : P->col_scale;
  // scaled space: bitwise-uniform c / l_v / u_v come from their scalar
  const uint32_t uni = orig ? 0u : P->uniform;
  const double cu = P->c_u, lu = P->lv_u, uu = P->uv_u;
  // values: 0 primal_inf (max), 1 dual_inf (max), 2 pobj (sum), 3 penalty (sum)
  auto f = [=] __device__(int64_t t, double* v) -> unsigned {
    if (t < m) {
      const int64_t j = t;
      const double d = interval_distance(ax[j], lc[j], uc[j]);
      v[0] = rs ? d / rs[j] : d;
      unsigned use = 1u;
      if (penalty_term(y[j], lc[j], uc[j], v[3])) use |= 8u;
      return use;
    }
    const int64_t i = t - m;
    const double xi = x[i];
    const double ci = (uni & 1u) ? cu : c[i], li = (uni & 2u) ? lu : lv[i],
                 ui = (uni & 4u) ? uu : uv[i];
    const double d = interval_distance(xi, li, ui);
    v[0] = cs ? d * cs[i] : d;
    // rc_mode 2: r is given (read from r_out), as in kkt_residuals(p, x, y, r)
    const double ri = rc_mode == 2 ? r_out[i] : reduced_cost(ci, aty[i], xi, li, ui, rc_mode);
    if (r_out && rc_mode != 2) r_out[i] = ri;
    const double dd = fabs(ci - aty[i] - ri);
    v[1] = cs ? dd / cs[i] : dd;
    v[2] = ci * xi;
    unsigned use = 7u;
    if (penalty_term(ri, li, ui, v[3])) use |= 8u;
    return use;
  };
  return multi_reduce<4>(f, m + n, red->parity ? PDLPK_RED_SEQ : PDLPK_RED_TREE, red->shards,
                         0x3u, red->scratch, slots, s);
}

int pdlpk_ray_primal_prep(const pdlpk_problem* P, int32_t orig, const double* yc, double* ray,
                          const pdlpk_red* red, double* slots, cudaStream_t s) {
  const double* lc = orig ? P->lc_o : P->lc;
  const double* uc = orig ? P->uc_o : P->uc;
  // values: 0 |ray|_inf (max), 1 coordinates changed by the projection (count)
  auto f = [=] __device__(int64_t j, double* v) -> unsigned {
    const double y = yc[j];
    const double r = cone_project(y, cone_of_bounds(lc[j], uc[j]));
    ray[j] = r;
    v[0] = fabs(r);
    v[1] = (r != y) ? 1.0 : 0.0;
    return 3u;
  };
  return multi_reduce<2>(f, P->m, PDLPK_RED_TREE, red->shards, 0x1u, red->scratch, slots, s);
}

int pdlpk_ray_primal_finish(const pdlpk_problem* P, int32_t orig, const double* ray,
                            const double* aty, const double* aty_alt, const double* changed,
                            double* rhat, const pdlpk_red* red, double* slots, cudaStream_t s) {
  const int64_t m = P->m, n = P->n;
  const double* lc = orig ? P->lc_o : P->lc;
  const double* uc = orig ? P->uc_o : P->uc;
  const double* lv = orig ? P->lv_o : P->lv;
  const double* uv = orig ? P->uv_o : P->uv;
  // values: 0 residual (max), 1 penalty (sum; dual_objective_value(ray, rhat))
  auto f = [=] __device__(int64_t t, double* v) -> unsigned {
    if (t < m) return penalty_term(ray[t], lc[t], uc[t], v[1]) ? 2u : 0u;
    const int64_t i = t - m;
    const double a = (aty_alt != nullptr && *changed == 0.0) ? aty_alt[i] : aty[i];
    const double rh = cone_project(-a, cone_of_bounds(lv[i], uv[i]));
    rhat[i] = rh;
    v[0] = fabs(a + rh);
    unsigned use = 1u;
    if (penalty_term(rh, lv[i], uv[i], v[1])) use |= 2u;
    return use;
  };
  return multi_reduce<2>(f, m + n, red->parity ? PDLPK_RED_SEQ : PDLPK_RED_TREE, red->shards,
                         0x1u, red->scratch, slots, s);
}

int pdlpk_ray_dual_prep(const pdlpk_problem* P, int32_t orig, const double* xc,
                        const pdlpk_red* red, double* slots, cudaStream_t s) {
  const double* c = orig ? P->c_o : P->c;
  const double* lv = orig ? P->lv_o : P->lv;
  const double* uv = orig ? P->uv_o : P->uv;
  // values: 0 |xc|_inf (max), 1 box residual (max), 2 c'xc (sum)
  auto f = [=] __device__(int64_t i, double* v) -> unsigned {
    const double xi = xc[i];
    v[0] = fabs(xi);
    v[1] = fabs(xi - cone_project(xi, recession_cone(lv[i], uv[i])));
    v[2] = c[i] * xi;
    return 7u;
  };
  return multi_reduce<3>(f, P->n, red->parity ? PDLPK_RED_SEQ : PDLPK_RED_TREE, red->shards,
                         0x3u, red->scratch, slots, s);
}

int pdlpk_ray_dual_finish(const pdlpk_problem* P, int32_t orig, const double* ax,
                          const pdlpk_red* red, double* slots, cudaStream_t s) {
  const double* lc = orig ? P->lc_o : P->lc;
  const double* uc = orig ? P->uc_o : P->uc;
  auto f = [=] __device__(int64_t j, double* v) -> unsigned {
    const double a = ax[j];
    v[0] = fabs(a - cone_project(a, recession_cone(lc[j], uc[j])));
    return 1u;
  };
  return multi_reduce<1>(f, P->m, PDLPK_RED_TREE, red->shards, 0x1u, red->scratch, slots, s);
}

int pdlpk_radius(const double* dx2, const double* dy2, double omega, double* out,
                 cudaStream_t s) {
  launch_pdl(PDLPK_PDL_CADENCE, radius_kernel, static_cast<unsigned>(1), 1, 0, s, dx2, dy2, omega, out);
  return ok();
}

int pdlpk_apply_vec_factors(double* lc, double* uc, double* row_scale, const double* fr,
                            int64_t m, double* c, double* lv, double* uv, double* col_scale,
                            const double* fc, int64_t n, cudaStream_t s) {
  if (m + n > 0) {
    launch_pdl(PDLPK_PDL_CADENCE, apply_vec_factor_kernel, static_cast<unsigned>(ew_blocks(m + n)), kT, 0, s, lc, uc, row_scale, fr, m, c, lv, uv,
                                                           col_scale, fc, n);
  }
  return ok();
}

int pdlpk_abs_max(const double* v, int64_t n, const pdlpk_red* red, double* slot,
                  cudaStream_t s) {
  auto f = [v] __device__(int64_t i, double* o) -> unsigned {
    o[0] = fabs(v[i]);
    return 1u;
  };
  return multi_reduce<1>(f, n, PDLPK_RED_TREE, 1, 0x1u, red->scratch, slot, s);
}

int pdlpk_primal_weight_sums(const double* c, int64_t n, const double* lc, const double* uc,
                             int64_t m, const pdlpk_red* red, double* slots, cudaStream_t s) {
  auto f = [=] __device__(int64_t t, double* v) -> unsigned {
    if (t < n) {
      v[0] = c[t] * c[t];
      return 1u;
    }
    const int64_t j = t - n;
    const double lo = lc[j], hi = uc[j];
    double mag = 0.0;
    if (finite_d(lo)) mag = max_keep(mag, fabs(lo));
    if (finite_d(hi)) mag = max_keep(mag, fabs(hi));
    v[1] = mag * mag;
    return 2u;
  };
  return multi_reduce<2>(f, n + m, red->parity ? PDLPK_RED_SEQ : PDLPK_RED_TREE, red->shards, 0u,
                         red->scratch, slots, s);
}

int pdlpk_initial_point(const double* lv, const double* uv, double* x, int64_t n,
                        cudaStream_t s) {
  if (n > 0) launch_pdl(PDLPK_PDL_CADENCE, initial_point_kernel, static_cast<unsigned>(ew_blocks(n)), kT, 0, s, lv, uv, x, n);
  return ok();
}

int pdlpk_dual_feas_bounds(const double* c, const double* lv, const double* uv, int64_t n,
                           const double* lc, const double* uc, int64_t m, double* sub_lc,
                           double* sub_uc, double* sub_lv, double* sub_uv, cudaStream_t s) {
  if (n + m > 0) {
    launch_pdl(PDLPK_PDL_CADENCE, dual_feas_bounds_kernel, static_cast<unsigned>(ew_blocks(n + m)), kT, 0, s, c, lv, uv, n, lc, uc, m, sub_lc,
                                                           sub_uc, sub_lv, sub_uv);
  }
  return ok();
}

int pdlpk_check_finite(const double* v, int64_t n, int32_t code, int32_t* first,
                       cudaStream_t s) {
  if (n > 0) launch_pdl(PDLPK_PDL_CADENCE, find_nonfinite_kernel, static_cast<unsigned>(ew_blocks(n)), kT, 0, s, v, n, code, first);
  return ok();
}

}  // extern "C"
