// SpMV design lab (measurement probe, not product code): C2-shaped matrices
// generated on the device, candidate row-pass / column-pass kernels timed
// with CUDA events against their algorithmic bytes.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false \
//        -o tools/spmv_lab/lab tools/spmv_lab/lab.cu
//   tools/spmv_lab/lab [m] [n] [sorted]
//
// C2 recipe: column counts ~ discrete power law alpha=2 on [2, 1e4], entries
// of a column at uniform random rows; |a| log-uniform [1e-3, 1e3].
// sorted=1 numbers the columns by decreasing count (degree ordering).
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      std::exit(1);                                                                   \
    }                                                                                 \
  } while (0)

__host__ __device__ inline uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__device__ inline double u01(uint64_t h) { return ((h >> 11) + 1) * (1.0 / 9007199254740992.0); }

__global__ void counts_kernel(int32_t* cnt, int64_t n, uint64_t seed) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    int k = 0;
    for (uint64_t t = 0;; ++t) {
      const double u = u01(mix64(seed ^ (uint64_t(j) * 0x100000001b3ull + t)));
      const double kk = floor(2.0 / u);
      if (kk <= 10000.0) { k = (int)kk; break; }
    }
    cnt[j] = k;
  }
}

// entries of column j: rows at random; key = (row << 24) | col for the row layout
__global__ void entries_kernel(const int64_t* cstart, int64_t n, int64_t m, uint64_t seed,
                               uint64_t* key_row, uint64_t* key_col) {
  const int lane = threadIdx.x & 31;
  for (int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; j < n;
       j += (int64_t)gridDim.x * blockDim.x / 32) {
    for (int64_t e = cstart[j] + lane; e < cstart[j + 1]; e += 32) {
      const uint64_t r = mix64(seed * 31 + e) % uint64_t(m);
      key_row[e] = (r << 24) | uint64_t(j);
      key_col[e] = (uint64_t(j) << 23) | r;
    }
  }
}

__device__ inline double entry_value(uint64_t r, uint64_t c) {
  const uint64_t h = mix64(r * 0x9e3779b97f4a7c15ull ^ c);
  const double mag = exp(log(1e-3) + u01(h) * (log(1e3) - log(1e-3)));
  return (h & 1) ? -mag : mag;
}

__global__ void split_row(const uint64_t* key, int64_t nnz, int32_t* idx, double* val, int32_t* rowcnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t r = key[e] >> 24, c = key[e] & 0xffffff;
    idx[e] = (int32_t)c;
    val[e] = entry_value(r, c);
    atomicAdd(rowcnt + r, 1);
  }
}
__global__ void split_col(const uint64_t* key, int64_t nnz, int32_t* idx, double* val) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t c = key[e] >> 23, r = key[e] & 0x7fffff;
    idx[e] = (int32_t)r;
    val[e] = entry_value(r, c);
  }
}
__global__ void fill_kernel(double* v, int64_t n, uint64_t seed, double lo, double hi) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = lo + (hi - lo) * u01(mix64(seed ^ i));
}
__global__ void i64_to_i32(const int64_t* a, int32_t* b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = (int32_t)a[i];
}

struct Csr {
  int64_t dim = 0, nnz = 0, other = 0;
  int32_t* start = nullptr;  // dim+1
  int32_t* idx = nullptr;
  double* val = nullptr;
  std::vector<int32_t> hstart;
};

// --------------------------------------------------------------- kernels ---
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double clampd(double v, double lo, double hi) { return fmin(fmax(v, lo), hi); }

template <class T>
__device__ __forceinline__ T ldcs(const T* p) { return __ldcs(p); }

// Row-pass epilogue (dual update): R y, l_c, u_c; W y', dy; |dy|^2 partial.
struct RowEpi {
  const double *y, *lc, *uc;
  double *yn, *dy;
  double sigma;
  double acc2 = 0.0;
  struct Pre { double y, lc, uc; };
  __device__ __forceinline__ Pre load(int64_t r) const { return {ldcs(y + r), ldcs(lc + r), ldcs(uc + r)}; }
  __device__ __forceinline__ void line(int64_t r, double s, const Pre& p) {
    const double yhat = p.y - sigma * s;
    const double proj = clampd(yhat / sigma, -p.uc, -p.lc);
    const double yp = yhat - sigma * proj;
    yn[r] = yp;
    const double d = yp - p.y;
    dy[r] = d;
    acc2 += d * d;
  }
  __device__ __forceinline__ void prefetch(int64_t r) const {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(y + r));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(lc + r));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(uc + r));
  }
  static constexpr int kRW = 5;  // 8-byte words per line
};
// Column-pass epilogue: R aty, x, x'; W aty'; |dx|^2, curvature partials.
struct ColEpi {
  const double *aty, *x, *xn;
  double* atyn;
  double acc2 = 0.0, curv = 0.0;
  struct Pre { double a, x, xn; };
  __device__ __forceinline__ Pre load(int64_t i) const { return {ldcs(aty + i), ldcs(x + i), xn[i]}; }
  __device__ __forceinline__ void line(int64_t i, double d, const Pre& p) {
    atyn[i] = p.a + d;
    const double dx = p.xn - p.x;
    acc2 += dx * dx;
    curv += d * dx;
  }
  __device__ __forceinline__ void prefetch(int64_t i) const {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(aty + i));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(x + i));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(xn + i));
  }
  static constexpr int kRW = 4;
};

// Column epilogue without operand loads (measurement: the products and the
// one store only).
struct ColEpiNull {
  double* atyn;
  double acc2 = 0.0;
  struct Pre { double a; };
  __device__ __forceinline__ Pre load(int64_t) const { return {0.0}; }
  __device__ __forceinline__ void prefetch(int64_t) const {}
  __device__ __forceinline__ void line(int64_t i, double d, const Pre&) { atyn[i] = d; acc2 += d; }
};

// Uniform warp items.  Block item {r0, cnt > 0}: lines r0..r0+cnt-1 (<= 63
// lines, <= ITEM entries, each line <= SEQMAX), products in a per-warp shared
// buffer, each lane sums its line in storage order.  Chunk item {r, -1-c,
// slot, nch}: entries [start[r] + c*ITEM, ...) of a long line, lane chains
// + warp tree; multi-chunk lines combine in chunk order in the last arriver.
template <int ITEM, class Epi, int MINB>
__global__ void __launch_bounds__(256, MINB) wb_kernel(const int4* __restrict__ items, int64_t n_items,
                                                       const int32_t* __restrict__ start,
                                                       const int32_t* __restrict__ idx,
                                                       const double* __restrict__ val,
                                                       const double* __restrict__ v, Epi epi,
                                                       double* part, unsigned* cnt, double* out_part) {
  constexpr int J = ITEM / 32;
  __shared__ double sp_all[8][ITEM];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* sp = sp_all[wid];
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t it = gw; it < n_items; it += nw) {
    const int4 d = items[it];
    if (d.y > 0) {
      const int r0 = d.x, cnt_l = d.y;
      const int p0 = lane <= cnt_l ? start[r0 + lane] : 0;
      const int p1 = lane + 32 <= cnt_l ? start[r0 + 32 + lane] : 0;
      const int s0 = __shfl_sync(0xffffffffu, p0, 0);
      const int s1 = cnt_l <= 31 ? __shfl_sync(0xffffffffu, p0, cnt_l & 31)
                                 : __shfl_sync(0xffffffffu, p1, (cnt_l - 32) & 31);
      typename Epi::Pre pre0{}, pre1{};
      if (lane < cnt_l) pre0 = epi.load(r0 + lane);
      if (lane + 32 < cnt_l) pre1 = epi.load(r0 + 32 + lane);
      int ci[J];
      double a[J];
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int k = s0 + j * 32 + lane;
        if (k < s1) {
          ci[j] = ldcs(idx + k);
          a[j] = ldcs(val + k);
        }
      }
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int k = s0 + j * 32 + lane;
        if (k < s1) sp[j * 32 + lane] = a[j] * __ldg(v + ci[j]);
      }
      __syncwarp();
      // line ends: lane l's line is [p(l), p(l+1))
      const int q0 = __shfl_down_sync(0xffffffffu, p0, 1);
      const int p1first = __shfl_sync(0xffffffffu, p1, 0);
      const int e0 = lane == 31 ? p1first : q0;
      if (lane < cnt_l) {
        double acc = 0.0;
        for (int k = p0 - s0; k < e0 - s0; ++k) acc += sp[k];
        epi.line(r0 + lane, acc, pre0);
      }
      const int q1 = __shfl_down_sync(0xffffffffu, p1, 1);
      if (lane + 32 < cnt_l) {
        double acc = 0.0;
        for (int k = p1 - s0; k < q1 - s0; ++k) acc += sp[k];
        epi.line(r0 + 32 + lane, acc, pre1);
      }
      __syncwarp();
    } else {
      const int r = d.x, c = -1 - d.y, nch = d.w;
      const int lo = start[r] + c * ITEM;
      const int e = start[r + 1];
      const int hi = lo + ITEM < e ? lo + ITEM : e;
      typename Epi::Pre pre{};
      if (nch == 1 && lane == 0) pre = epi.load(r);
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      int ci[J];
      double a[J];
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int k = lo + j * 32 + lane;
        if (k < hi) {
          ci[j] = ldcs(idx + k);
          a[j] = ldcs(val + k);
        }
      }
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int k = lo + j * 32 + lane;
        if (k < hi) acc[j & 3] += a[j] * __ldg(v + ci[j]);
      }
      const double t = warp_sum((acc[0] + acc[1]) + (acc[2] + acc[3]));
      if (lane == 0) {
        if (nch == 1) {
          epi.line(r, t, pre);
        } else {
          part[d.z + c] = t;
          __threadfence();
          const unsigned old = atomicAdd(cnt + d.z, 1u);
          if (old == (unsigned)(nch - 1)) {
            __threadfence();
            double tot = 0.0;
            for (int q = 0; q < nch; ++q) tot += __ldcg(part + d.z + q);
            cnt[d.z] = 0;
            epi.line(r, tot, epi.load(r));
          }
        }
      }
    }
  }
  // per-CTA partial (lab: only to keep the epilogue's reduction work)
  double s = warp_sum(epi.acc2);
  if (lane == 0) out_part[blockIdx.x * 8 + wid] = s;
}

// CSR-vector reference: G lanes per line, tree sum (lines <= any length).
template <int G, class Epi, int MINB>
__global__ void __launch_bounds__(256, MINB) vec_kernel(int64_t dim, const int32_t* __restrict__ start,
                                                        const int32_t* __restrict__ idx,
                                                        const double* __restrict__ val,
                                                        const double* __restrict__ v, Epi epi,
                                                        double* out_part) {
  const int lane = threadIdx.x & 31;
  const int sub = lane % G;
  const int64_t g0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
  const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / G;
  for (int64_t base = g0 - (g0 % (32 / G)); base < dim; base += ng) {
    const int64_t r = base + (lane / G);
    double acc = 0.0;
    typename Epi::Pre pre{};
    if (r < dim) {
      if (sub == 0) pre = epi.load(r);
      const int s = start[r], e = start[r + 1];
      for (int k = s + sub; k < e; k += G) acc += ldcs(val + k) * __ldg(v + ldcs(idx + k));
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (r < dim && sub == 0) epi.line(r, acc, pre);
  }
  double s = warp_sum(epi.acc2);
  if (lane == 0) out_part[blockIdx.x * 8 + (threadIdx.x >> 5)] = s;
}

// Column panels: the row layout re-laid out panel-major (entries of column
// panel p of every row, then panel p+1), one pass per panel carrying each
// row's partial sum; only the last pass runs the epilogue.
template <int G, class Epi, int MODE, int MINB>
__global__ void __launch_bounds__(256, MINB) panel_kernel(int64_t dim, const int32_t* __restrict__ start,
                                                          const int32_t* __restrict__ idx,
                                                          const double* __restrict__ val,
                                                          const double* __restrict__ v, Epi epi,
                                                          double* __restrict__ carry, double* out_part) {
  const int lane = threadIdx.x & 31;
  const int sub = lane % G;
  const int64_t g0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
  const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / G;
  for (int64_t base = g0 - (g0 % (32 / G)); base < dim; base += ng) {
    const int64_t r = base + (lane / G);
    double acc = 0.0;
    typename Epi::Pre pre{};
    double cin = 0.0;
    if (r < dim) {
      if (MODE == 2 && sub == 0) pre = epi.load(r);
      if (MODE != 0 && sub == 0) cin = __ldcs(carry + r);
      const int s = start[r], e = start[r + 1];
      for (int k = s + sub; k < e; k += G) acc += ldcs(val + k) * __ldg(v + ldcs(idx + k));
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (r < dim && sub == 0) {
      acc += cin;
      if (MODE == 2) epi.line(r, acc, pre);
      else __stcs(carry + r, acc);
    }
  }
  if (MODE == 2) {
    double s = warp_sum(epi.acc2);
    if (lane == 0) out_part[blockIdx.x * 8 + (threadIdx.x >> 5)] = s;
  }
}

__global__ void panel_count(const int32_t* st, const int32_t* idx, int64_t m, int P, int64_t W, int32_t* cnt) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x)
    for (int k = st[r]; k < st[r + 1]; ++k) cnt[(int64_t)(idx[k] / W) * m + r] += 1;
}
__global__ void panel_scatter(const int32_t* st, const int32_t* idx, const double* val, int64_t m, int P,
                              int64_t W, const int64_t* pst, int32_t* nidx, double* nval) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
    int64_t pos[8];
    for (int p = 0; p < P; ++p) pos[p] = pst[p * m + r];
    for (int k = st[r]; k < st[r + 1]; ++k) {
      const int p = (int)(idx[k] / W);
      nidx[pos[p]] = idx[k];
      nval[pos[p]] = val[k];
      ++pos[p];
    }
  }
}


// ------------------------------------------ sliced ELL (SELL-32-sigma) ---
// Rows in slices of 32 (one lane per row), entries stored slice-column-major
// (entry k of the slice's lane l at off[g] + 32 k + l), so a warp's index and
// value loads are coalesced with no shared-memory staging and each lane sums
// its own row sequentially in storage order (the same sums as the tile
// kernel's storage-order lines).  Rows are sorted by length inside windows of
// SIGMA rows to keep the padding small; perm[] maps a slot to its row.
__global__ void sell_len(const int32_t* st, int64_t m, int64_t sigma, int32_t* len, uint64_t* key, int32_t* rid) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t l = st[r + 1] - st[r];
    len[r] = l;
    key[r] = ((uint64_t)(r / sigma) << 32) | (uint32_t)(0x7fffffff - l);  // window, then longest first
    rid[r] = (int32_t)r;
  }
}
__global__ void sell_width(const int32_t* len, const int32_t* perm, int64_t m, int64_t ng, int64_t* w32) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ng; g += (int64_t)gridDim.x * blockDim.x) {
    int32_t w = 0;
    for (int l = 0; l < 32; ++l) {
      const int64_t s = g * 32 + l;
      if (s < m) w = max(w, len[perm[s]]);
    }
    w32[g] = 32ll * w;
  }
}
__global__ void sell_fill(const int32_t* st, const int32_t* idx, const double* val, const int32_t* perm, int64_t m,
                          const int64_t* off, int32_t* sidx, double* sval) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m; s += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = perm[s];
    const int64_t base = off[s >> 5] + (s & 31);
    const int32_t b = st[r], e = st[r + 1];
    for (int32_t k = b; k < e; ++k) {
      sidx[base + 32ll * (k - b)] = idx[k];
      sval[base + 32ll * (k - b)] = val[k];
    }
  }
}
// MODE 0: first panel (writes carry), 1: middle, 2: last (carry + epilogue), 3: single pass
// SLOT: the row vectors (y, bounds, carry) are stored in slot order (rows renumbered at setup)
template <int U, class Epi, int MODE, int MINB, bool SLOT = false>
__global__ void __launch_bounds__(256, MINB) sell_kernel(int64_t m, int64_t ng, const int64_t* __restrict__ off,
                                                         const int32_t* __restrict__ perm,
                                                         const int32_t* __restrict__ len,
                                                         const int32_t* __restrict__ sidx,
                                                         const double* __restrict__ sval,
                                                         const double* __restrict__ v, Epi epi,
                                                         double* __restrict__ carry, double* out_part) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t g = w0; g < ng; g += nw) {
    const int64_t s = g * 32 + lane;
    const bool live = s < m;
    const int32_t r0 = live ? perm[s] : 0;
    const int32_t n = live ? len[r0] : 0;
    const int64_t r = SLOT ? s : r0;
    const int64_t o = off[g];
    const int32_t w = (int32_t)((off[g + 1] - o) >> 5);
    typename Epi::Pre pre{};
    double acc = 0.0;
    if (live) {
      if (MODE >= 2) pre = epi.load(r);
      if (MODE == 1 || MODE == 2) acc = __ldcs(carry + r);
    }
    const int32_t* pi = sidx + o + lane;
    const double* pv = sval + o + lane;
    for (int32_t k = 0; k < w; k += U) {
      int32_t c[U];
      double a[U], x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool on = k + u < n;
        c[u] = on ? ldcs(pi + 32 * (k + u)) : 0;
        a[u] = on ? ldcs(pv + 32 * (k + u)) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) x[u] = (k + u < n) ? __ldg(v + c[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (k + u < n) acc += a[u] * x[u];
    }
    if (live) {
      if (MODE >= 2) epi.line(r, acc, pre);
      else __stcs(carry + r, acc);
    }
  }
  if (MODE >= 2) {
    double t = warp_sum(epi.acc2);
    if (lane == 0) out_part[blockIdx.x * 8 + (threadIdx.x >> 5)] = t;
  }
}

// Random-gather throughput probe: `count` gathers of v[hash % len], UNROLL
// independent per thread per round (no index stream).
template <int UNROLL>
__global__ void __launch_bounds__(256) gather_probe(const double* __restrict__ v, int64_t len, int64_t count,
                                                    double* out) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  double acc = 0.0;
  for (int64_t b = tid * UNROLL; b < count; b += nt * UNROLL) {
    double g[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      uint32_t h = static_cast<uint32_t>(b + u) * 0x9E3779B1u;
      h ^= h >> 15;
      h *= 0x85EBCA77u;
      h ^= h >> 13;
      g[u] = __ldg(v + __umulhi(h, static_cast<uint32_t>(len)));
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) acc += g[u];
  }
  if (acc == 12345.678) out[0] = acc;
}

// ---------------------------------------------- warp-private TMA rings ---
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}"
               ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ uint64_t evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}
struct WinL { const char* src; uint32_t bytes, shift; };
__device__ __forceinline__ WinL winl(const void* base, int64_t first, int64_t count, int esz) {
  const uintptr_t lo = reinterpret_cast<uintptr_t>(base) + first * esz;
  const uintptr_t hi = lo + count * esz;
  const uintptr_t alo = lo & ~uintptr_t(15), ahi = (hi + 15) & ~uintptr_t(15);
  return WinL{reinterpret_cast<const char*>(alo), count > 0 ? (uint32_t)(ahi - alo) : 0u, (uint32_t)(lo - alo)};
}
struct RingHdr { int r0, cnt, s0, len; uint32_t sh; int pad[3]; };
struct RowStage {  // staged operands of the row epilogue
  static constexpr int kStaged = 3;
};

// Tiles {r0, cnt, s0, len} of consecutive short lines.  Warp 0 lane 0 is the
// producer; consumer warp w owns stages [w][0..S).  Each tile goes to one
// consumer warp whole: gather phase (G gathers in flight per lane, products
// in place), then one lane per line sums in storage order and runs the
// epilogue from the staged operands.
template <int CW, int S, int G, class Epi>
__global__ void __launch_bounds__(32 * (CW + 1), 1) wr_kernel(const int4* __restrict__ tiles, int64_t n_tiles,
                                                              const int32_t* __restrict__ start,
                                                              const int32_t* __restrict__ idx,
                                                              const double* __restrict__ val,
                                                              const double* __restrict__ v, Epi epi,
                                                              const double* st0, const double* st1,
                                                              const double* st2, int E, int L,
                                                              double* out_part) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + CW * S;
  RingHdr* hdr = reinterpret_cast<RingHdr*>(sm + 16 * CW * S);
  const uint32_t o_val = (uint32_t)((4 * E + 32 + 15) & ~15);
  const uint32_t o_ptr = o_val + (uint32_t)((8 * E + 32 + 15) & ~15);
  const uint32_t o_epi = o_ptr + (uint32_t)((4 * (L + 1) + 32 + 15) & ~15);
  const uint32_t epi_stride = (uint32_t)((8 * L + 32 + 15) & ~15);
  const uint32_t stage_bytes = o_epi + 3 * epi_stride;
  unsigned char* stage0 = sm + ((16 * CW * S + sizeof(RingHdr) * CW * S + 127) & ~127);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int q = 0; q < CW * S; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t G0 = gridDim.x;
  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = evict_first();
      int64_t i = 0;
      for (int64_t t = blockIdx.x; t < n_tiles; t += G0, ++i) {
        const int w = (int)(i % CW);
        const int64_t j = i / CW;
        const int s = (int)(j % S);
        const int q = w * S + s;
        if (j >= S) mbar_wait(&empty[q], (uint32_t)(((j / S) - 1) & 1));
        const int4 d = tiles[t];
        unsigned char* buf = stage0 + (size_t)q * stage_bytes;
        const WinL wi = winl(idx, d.z, d.w, 4), wv = winl(val, d.z, d.w, 8), wp = winl(start, d.x, d.y + 1, 4);
        const WinL w0 = winl(st0, d.x, d.y, 8), w1 = winl(st1, d.x, d.y, 8), w2 = winl(st2, d.x, d.y, 8);
        RingHdr h;
        h.r0 = d.x; h.cnt = d.y; h.s0 = d.z; h.len = d.w;
        h.sh = wi.shift | (wv.shift << 4) | (wp.shift << 8) | (w0.shift << 12) | (w1.shift << 16) | (w2.shift << 20);
        hdr[q] = h;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive_expect_tx(&full[q], wi.bytes + wv.bytes + wp.bytes + w0.bytes + w1.bytes + w2.bytes);
        if (wi.bytes) bulk(buf, wi.src, wi.bytes, &full[q], pol);
        if (wv.bytes) bulk(buf + o_val, wv.src, wv.bytes, &full[q], pol);
        if (wp.bytes) bulk(buf + o_ptr, wp.src, wp.bytes, &full[q], pol);
        if (w0.bytes) bulk(buf + o_epi, w0.src, w0.bytes, &full[q], pol);
        if (w1.bytes) bulk(buf + o_epi + epi_stride, w1.src, w1.bytes, &full[q], pol);
        if (w2.bytes) bulk(buf + o_epi + 2 * epi_stride, w2.src, w2.bytes, &full[q], pol);
      }
    }
  } else {
    const int w = warp - 1;
    int64_t j = 0;
    for (int64_t t = blockIdx.x + (int64_t)w * G0; t < n_tiles; t += (int64_t)CW * G0, ++j) {
      const int s = (int)(j % S);
      const int q = w * S + s;
      mbar_wait(&full[q], (uint32_t)((j / S) & 1));
      const RingHdr h = hdr[q];
      unsigned char* buf = stage0 + (size_t)q * stage_bytes;
      const int32_t* s_idx = reinterpret_cast<const int32_t*>(buf + (h.sh & 15u));
      double* s_val = reinterpret_cast<double*>(buf + o_val + ((h.sh >> 4) & 15u));
      const int32_t* s_ptr = reinterpret_cast<const int32_t*>(buf + o_ptr + ((h.sh >> 8) & 15u));
      const double* e0 = reinterpret_cast<const double*>(buf + o_epi + ((h.sh >> 12) & 15u));
      const double* e1 = reinterpret_cast<const double*>(buf + o_epi + epi_stride + ((h.sh >> 16) & 15u));
      const double* e2 = reinterpret_cast<const double*>(buf + o_epi + 2 * epi_stride + ((h.sh >> 20) & 15u));
      for (int e = lane; e < h.len; e += 32 * G) {
        int ci[G];
        double g[G];
#pragma unroll
        for (int u = 0; u < G; ++u)
          if (e + 32 * u < h.len) ci[u] = s_idx[e + 32 * u];
#pragma unroll
        for (int u = 0; u < G; ++u)
          if (e + 32 * u < h.len) g[u] = __ldg(v + ci[u]);
#pragma unroll
        for (int u = 0; u < G; ++u)
          if (e + 32 * u < h.len) s_val[e + 32 * u] *= g[u];
      }
      __syncwarp();
      for (int l = lane; l < h.cnt; l += 32) {
        const int a = s_ptr[l] - h.s0, b = s_ptr[l + 1] - h.s0;
        double acc = 0.0;
        for (int k = a; k < b; ++k) acc += s_val[k];
        epi.line(h.r0 + l, acc, typename Epi::Pre{e0[l], e1[l], e2[l]});
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[q]);
    }
  }
  double s2 = warp_sum(epi.acc2);
  if (lane == 0) out_part[blockIdx.x * 32 + warp] = s2;
}

std::vector<int4> build_tiles(const std::vector<int32_t>& st, int E, int L, int seqmax) {
  std::vector<int4> t;
  const int64_t dim = (int64_t)st.size() - 1;
  int r0 = -1, cnt = 0, nz = 0;
  auto close = [&] {
    if (cnt > 0) t.push_back(make_int4(r0, cnt, st[r0], nz));
    cnt = 0;
    nz = 0;
  };
  for (int64_t r = 0; r < dim; ++r) {
    const int len = st[r + 1] - st[r];
    if (len > seqmax) { close(); continue; }
    if (cnt == L || nz + len > E) close();
    if (cnt == 0) r0 = (int)r;
    ++cnt;
    nz += len;
  }
  close();
  return t;
}

// Stream + gather probe: acc += val[k] * v[idx[k]] over all entries with
// coalesced LDG streams (no line structure): the ceiling of an LDG-fed SpMV.
template <int U>
__global__ void __launch_bounds__(256) stream_gather_probe(const int32_t* __restrict__ idx,
                                                           const double* __restrict__ val,
                                                           const double* __restrict__ v, int64_t nnz,
                                                           double* out) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  const int64_t w = tid >> 5, nw = nt >> 5;
  double acc = 0.0;
  for (int64_t b = w * 32 * U; b < nnz; b += nw * 32 * U) {
    int ci[U];
    double a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = b + u * 32 + lane;
      ci[u] = k < nnz ? __ldcs(idx + k) : 0;
      a[u] = k < nnz ? __ldcs(val + k) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += a[u] * __ldg(v + ci[u]);
  }
  if (acc == 12345.678) out[0] = acc;
}

// Segmented-scan warp spans.  Span {r0, nl > 0, e0, len}: whole lines
// r0..r0+nl-1 (entries [e0, e0+len), no empty line).  Span {r, -1-c, e0, len}
// with (slot, nch) in spanB: chunk c of a long line.  A warp walks its span in
// steps of 256 entries: coalesced index/value loads, 8 gathers per lane,
// then a segmented inclusive scan across lanes (head flags from the line
// starts) with a carry between rows and steps; the lane holding a line's
// last entry runs the epilogue.
__device__ __forceinline__ double seg_scan(double v, bool head, int lane) {
  // inclusive segmented scan over the warp; a head starts a new segment
  unsigned hb = __ballot_sync(0xffffffffu, head);
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double t = __shfl_up_sync(0xffffffffu, v, o);
    // lanes (lane-o, lane] contain no head after lane-o ... include t iff no
    // head in (lane-o, lane]
    const unsigned span = lane >= o ? ((lane == 31 ? 0xffffffffu : ((1u << (lane + 1)) - 1u)) &
                                       ~((1u << (lane - o + 1)) - 1u)) : 0u;
    if (lane >= o && (hb & span) == 0u) v += t;
  }
  return v;
}

template <class Epi, int MINB>
__global__ void __launch_bounds__(256, MINB) seg_kernel(const int4* __restrict__ spans, const int2* __restrict__ spanB,
                                                        int64_t n_spans, const int32_t* __restrict__ start,
                                                        const int32_t* __restrict__ idx,
                                                        const double* __restrict__ val,
                                                        const double* __restrict__ v, Epi epi,
                                                        double* part, unsigned* cnt, double* out_part) {
  __shared__ unsigned masks[8][16];  // per warp: 8 head words, 8 end words
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned* hm = masks[wid];
  unsigned* em = masks[wid] + 8;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t it = gw; it < n_spans; it += nw) {
    const int4 d = spans[it];
    const int e0 = d.z, e1 = d.z + d.w;
    if (d.y < 0) {
      // chunk of a long line: tree sum, ordered combine of the chunks
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int base = e0; base < e1; base += 256) {
        int ci[8];
        double a[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int k = base + 32 * u + lane;
          ci[u] = k < e1 ? ldcs(idx + k) : 0;
          a[u] = k < e1 ? ldcs(val + k) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u & 3] += a[u] * __ldg(v + ci[u]);
      }
      const double t = warp_sum((acc[0] + acc[1]) + (acc[2] + acc[3]));
      if (lane == 0) {
        const int2 b = spanB[it];
        const int c = -1 - d.y, nch = b.y;
        if (nch == 1) {
          epi.line(d.x, t, epi.load(d.x));
        } else {
          part[b.x + c] = t;
          __threadfence();
          const unsigned old = atomicAdd(cnt + b.x, 1u);
          if (old == (unsigned)(nch - 1)) {
            __threadfence();
            double tot = 0.0;
            for (int q = 0; q < nch; ++q) tot += __ldcg(part + b.x + q);
            cnt[b.x] = 0;
            epi.line(d.x, tot, epi.load(d.x));
          }
        }
      }
      continue;
    }
    const int rend = d.x + d.y;  // one past the last line
    int rc = d.x;                // line containing the step's first entry
    double carry = 0.0;          // running sum of the segment open at the step start
    for (int base = e0; base < e1; base += 256) {
      // products
      double p[8];
      {
        int ci[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int k = base + 32 * u + lane;
          ci[u] = k < e1 ? ldcs(idx + k) : 0;
          p[u] = k < e1 ? ldcs(val + k) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) p[u] = p[u] * __ldg(v + ci[u]);
      }
      // head / end masks of this step from the line starts
      if (lane < 16) hm[lane] = 0u;
      __syncwarp();
      for (int j0 = rc; ; j0 += 32) {
        const int r = j0 + lane;
        const int sr = r <= rend ? start[r] : 0x7fffffff;
        if (r <= rend) {
          const int o = sr - base;
          if (o >= 0 && o < 256 && r < rend) atomicOr(&hm[o >> 5], 1u << (o & 31));
          if (o > 0 && o <= 256) atomicOr(&em[(o - 1) >> 5], 1u << ((o - 1) & 31));
        }
        const int last = __shfl_sync(0xffffffffu, sr, 31);
        if (last > base + 256 || j0 + 32 > rend) break;
      }
      __syncwarp();
      // segmented scan row by row, carrying the open segment
      int lines_done = 0;  // lines completed before this row (in this step)
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const unsigned h = hm[u], e = em[u];
        const bool head = (h >> lane) & 1u;
        double s = seg_scan(p[u], head, lane);
        const unsigned upto = lane == 31 ? 0xffffffffu : ((1u << (lane + 1)) - 1u);
        if ((h & upto) == 0u) s += carry;  // still in the segment open at the row start
        // lines completed up to this lane: ends in earlier rows + ends in (.., lane)
        const int rank = lines_done + __popc(e & (upto >> 1));
        if ((e >> lane) & 1u) {
          const int line = rc + rank;
          epi.line(line, s, epi.load(line));
        }
        carry = __shfl_sync(0xffffffffu, s, 31);
        if ((e >> 31) & 1u) carry = 0.0;
        lines_done += __popc(e);
      }
      rc += lines_done;
      __syncwarp();
    }
  }
  double s = warp_sum(epi.acc2);
  if (lane == 0) out_part[blockIdx.x * 8 + wid] = s;
}

// v2: head/end masks precomputed per step (2U words per step: U head words,
// U end words), U rows of 32 entries per step, L2 prefetch of the step's
// epilogue operands.
template <int U, class Epi, int MINB>
__global__ void __launch_bounds__(256, MINB) seg2_kernel(const int4* __restrict__ spans, const int2* __restrict__ spanB,
                                                         const int32_t* __restrict__ step0, const uint32_t* __restrict__ masks,
                                                         int64_t n_spans,
                                                         const int32_t* __restrict__ idx,
                                                         const double* __restrict__ val,
                                                         const double* __restrict__ v, Epi epi,
                                                         double* part, unsigned* cnt, double* out_part) {
  constexpr int STEP = 32 * U;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t it = gw; it < n_spans; it += nw) {
    const int4 d = spans[it];
    const int e0 = d.z, e1 = d.z + d.w;
    if (d.y < 0) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int base = e0; base < e1; base += 256) {
        int ci[8];
        double a[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int k = base + 32 * u + lane;
          ci[u] = k < e1 ? ldcs(idx + k) : 0;
          a[u] = k < e1 ? ldcs(val + k) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u & 3] += a[u] * __ldg(v + ci[u]);
      }
      const double t = warp_sum((acc[0] + acc[1]) + (acc[2] + acc[3]));
      if (lane == 0) {
        const int2 b = spanB[it];
        const int c = -1 - d.y, nch = b.y;
        if (nch == 1) {
          epi.line(d.x, t, epi.load(d.x));
        } else {
          part[b.x + c] = t;
          __threadfence();
          const unsigned old = atomicAdd(cnt + b.x, 1u);
          if (old == (unsigned)(nch - 1)) {
            __threadfence();
            double tot = 0.0;
            for (int q = 0; q < nch; ++q) tot += __ldcg(part + b.x + q);
            cnt[b.x] = 0;
            epi.line(d.x, tot, epi.load(d.x));
          }
        }
      }
      continue;
    }
    int rc = d.x;
    double carry = 0.0;
    int sid = step0[it];
    for (int base = e0; base < e1; base += STEP, ++sid) {
      const uint32_t mw = lane < 2 * U ? __ldg(masks + (int64_t)sid * 2 * U + lane) : 0u;
      double p[U];
      {
        int ci[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int k = base + 32 * u + lane;
          ci[u] = k < e1 ? ldcs(idx + k) : 0;
          p[u] = k < e1 ? ldcs(val + k) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) p[u] = p[u] * __ldg(v + ci[u]);
      }
      // the lines ending in this step: rc .. rc + nend - 1; warm their operands in L2
      int nend = 0;
#pragma unroll
      for (int u = 0; u < U; ++u) nend += __popc(__shfl_sync(0xffffffffu, mw, U + u));
      for (int j = lane; j < nend; j += 32) epi.prefetch(rc + j);
      int lines_done = 0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const unsigned h = __shfl_sync(0xffffffffu, mw, u), e = __shfl_sync(0xffffffffu, mw, U + u);
        const bool head = (h >> lane) & 1u;
        double s = seg_scan(p[u], head, lane);
        const unsigned upto = lane == 31 ? 0xffffffffu : ((1u << (lane + 1)) - 1u);
        if ((h & upto) == 0u) s += carry;
        if ((e >> lane) & 1u) {
          const int line = rc + lines_done + __popc(e & (upto >> 1));
          epi.line(line, s, epi.load(line));
        }
        carry = __shfl_sync(0xffffffffu, s, 31);
        if ((e >> 31) & 1u) carry = 0.0;
        lines_done += __popc(e);
      }
      rc += lines_done;
    }
  }
  double s = warp_sum(epi.acc2);
  if (lane == 0) out_part[blockIdx.x * 8 + wid] = s;
}

// v3: lane-contiguous entries.  Steps of 256 entries start on 8-entry
// boundaries; lane l holds entries [base + 8l, base + 8l + 8) (vector loads),
// sums its line segments sequentially (storage order inside a lane), and one
// segmented scan across lanes joins segments that span lanes; a carry joins
// steps.  Head/end bits: per-step 256-bit masks (8 + 8 words).
__device__ __forceinline__ int warp_excl_scan_int(int v, int lane) {
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += t;
  }
  return x - v;
}

template <class Epi, int MINB>
__global__ void __launch_bounds__(256, MINB) seg3_kernel(const int4* __restrict__ spans, const int2* __restrict__ spanB,
                                                         const int32_t* __restrict__ step0, const uint32_t* __restrict__ masks,
                                                         int64_t n_spans,
                                                         const int32_t* __restrict__ idx,
                                                         const double* __restrict__ val,
                                                         const double* __restrict__ v, Epi epi,
                                                         double* part, unsigned* cnt, double* out_part) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t it = gw; it < n_spans; it += nw) {
    const int4 d = spans[it];
    const int e0 = d.z, e1 = d.z + d.w;
    if (d.y < 0) {
      // chunk of a long line: lane-contiguous products, tree, ordered combine
      double acc = 0.0;
      for (int base = e0 & ~7; base < e1; base += 256) {
        const int k0 = base + 8 * lane;
        if (k0 + 8 > e0 && k0 < e1) {
          const int4 i0 = __ldcs(reinterpret_cast<const int4*>(idx + k0));
          const int4 i1 = __ldcs(reinterpret_cast<const int4*>(idx + k0 + 4));
          const int ci[8] = {i0.x, i0.y, i0.z, i0.w, i1.x, i1.y, i1.z, i1.w};
          double a[8];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const double2 t = __ldcs(reinterpret_cast<const double2*>(val + k0) + q);
            a[2 * q] = t.x;
            a[2 * q + 1] = t.y;
          }
          double g[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) g[u] = (k0 + u >= e0 && k0 + u < e1) ? __ldg(v + ci[u]) : 0.0;
#pragma unroll
          for (int u = 0; u < 8; ++u) acc += (k0 + u >= e0 && k0 + u < e1) ? a[u] * g[u] : 0.0;
        }
      }
      const double t = warp_sum(acc);
      if (lane == 0) {
        const int2 b = spanB[it];
        const int c = -1 - d.y, nch = b.y;
        if (nch == 1) {
          epi.line(d.x, t, epi.load(d.x));
        } else {
          part[b.x + c] = t;
          __threadfence();
          const unsigned old = atomicAdd(cnt + b.x, 1u);
          if (old == (unsigned)(nch - 1)) {
            __threadfence();
            double tot = 0.0;
            for (int q = 0; q < nch; ++q) tot += __ldcg(part + b.x + q);
            cnt[b.x] = 0;
            epi.line(d.x, tot, epi.load(d.x));
          }
        }
      }
      continue;
    }
    int rc = d.x;
    double carry = 0.0;
    int sid = step0[it];
    for (int base = e0 & ~7; base < e1; base += 256, ++sid) {
      const uint32_t mw = lane < 16 ? __ldg(masks + (int64_t)sid * 16 + lane) : 0u;
      const int k0 = base + 8 * lane;
      const bool any = k0 + 8 > e0 && k0 < e1;
      double p[8];
      if (any) {
        const int4 i0 = __ldcs(reinterpret_cast<const int4*>(idx + k0));
        const int4 i1 = __ldcs(reinterpret_cast<const int4*>(idx + k0 + 4));
        const int ci[8] = {i0.x, i0.y, i0.z, i0.w, i1.x, i1.y, i1.z, i1.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double2 t = __ldcs(reinterpret_cast<const double2*>(val + k0) + q);
          p[2 * q] = t.x;
          p[2 * q + 1] = t.y;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) p[u] = (k0 + u >= e0 && k0 + u < e1) ? p[u] * __ldg(v + ci[u]) : 0.0;
      } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) p[u] = 0.0;
      }
      const uint32_t hw = __shfl_sync(0xffffffffu, mw, lane >> 2), ew = __shfl_sync(0xffffffffu, mw, 8 + (lane >> 2));
      const uint32_t hb = (hw >> (8 * (lane & 3))) & 0xffu, eb = (ew >> (8 * (lane & 3))) & 0xffu;
      // lines ending in this step: warm their operands in L2
      const int nend_lane = __popc(eb);
      const int ends_before = warp_excl_scan_int(nend_lane, lane);
      const int nend = __shfl_sync(0xffffffffu, ends_before + nend_lane, 31);
      for (int j = lane; j < nend; j += 32) epi.prefetch(rc + j);
      // pass 1: the open segment at the lane's end
      double tail = 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) tail = ((hb >> u) & 1u) ? p[u] : tail + p[u];
      // segmented exclusive scan of the tails: the sum carried into the lane
      const bool hh = hb != 0u;
      double inc = tail;
      {
        const unsigned hmask = __ballot_sync(0xffffffffu, hh);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double t = __shfl_up_sync(0xffffffffu, inc, o);
          // add lanes (lane-o, lane-1]'s tails only if no head in lanes (lane-o, lane-1] ... i.e. window
          const unsigned win = lane >= o ? (((1u << lane) - 1u) & ~((1u << (lane - o + 1)) - 1u)) : 0u;
          if (lane >= o && (hmask & (win | (1u << lane))) == 0u) inc += t;
        }
        // inc = inclusive sum of tails back to (and including) the nearest
        // lane with a head, excluding that lane's pre-head part (its tail
        // starts at its head).  The carry enters lanes with no head before.
        const unsigned before = hmask & ((1u << lane) - 1u);
        double into = __shfl_up_sync(0xffffffffu, inc, 1);
        if (lane == 0) into = 0.0;
        if (before == 0u) into += carry;
        // pass 2: emit the lines ending in this lane
        double run = into;
        int rank = ends_before;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          run = ((hb >> u) & 1u) ? p[u] : run + p[u];
          if ((eb >> u) & 1u) {
            const int line = rc + rank;
            epi.line(line, run, epi.load(line));
            ++rank;
          }
        }
        // carry out of the step: lane 31's open segment
        double c31 = __shfl_sync(0xffffffffu, run, 31);
        carry = c31;
        const uint32_t eb31 = __shfl_sync(0xffffffffu, eb, 31);
        if ((eb31 >> 7) & 1u) carry = 0.0;
      }
      rc += nend;
    }
  }
  double s = warp_sum(epi.acc2);
  if (lane == 0) out_part[blockIdx.x * 8 + wid] = s;
}

// masks for v3: steps from e0 & ~7 in 256-entry strides, 8 head + 8 end words
std::vector<uint32_t> build_masks3(const std::vector<int32_t>& st, const std::vector<int4>& spans,
                                   std::vector<int32_t>& step0) {
  step0.assign(spans.size(), 0);
  int64_t nsteps = 0;
  for (size_t i = 0; i < spans.size(); ++i) {
    step0[i] = (int32_t)nsteps;
    if (spans[i].y > 0) {
      const int b0 = spans[i].z & ~7;
      nsteps += (spans[i].z + spans[i].w - b0 + 255) / 256;
    }
  }
  std::vector<uint32_t> M((size_t)nsteps * 16 + 16, 0u);
  for (size_t i = 0; i < spans.size(); ++i) {
    const int4 d = spans[i];
    if (d.y <= 0) continue;
    const int b0 = d.z & ~7;
    for (int r = d.x; r < d.x + d.y; ++r) {
      const int oh = st[r] - b0, oe = st[r + 1] - 1 - b0;
      M[(size_t)(step0[i] + oh / 256) * 16 + (oh % 256) / 32] |= 1u << (oh % 32);
      M[(size_t)(step0[i] + oe / 256) * 16 + 8 + (oe % 256) / 32] |= 1u << (oe % 32);
    }
  }
  return M;
}

// per-step masks of a span schedule (host)
std::vector<uint32_t> build_masks(const std::vector<int32_t>& st, const std::vector<int4>& spans, int U,
                                  std::vector<int32_t>& step0) {
  const int STEP = 32 * U;
  step0.assign(spans.size(), 0);
  int64_t nsteps = 0;
  for (size_t i = 0; i < spans.size(); ++i) {
    step0[i] = (int32_t)nsteps;
    if (spans[i].y > 0) nsteps += (spans[i].w + STEP - 1) / STEP;
  }
  std::vector<uint32_t> M((size_t)nsteps * 2 * U + 16, 0u);
  for (size_t i = 0; i < spans.size(); ++i) {
    const int4 d = spans[i];
    if (d.y <= 0) continue;
    for (int r = d.x; r < d.x + d.y; ++r) {
      const int oh = st[r] - d.z, oe = st[r + 1] - 1 - d.z;
      const int64_t sh = step0[i] + oh / STEP, se = step0[i] + oe / STEP;
      M[(size_t)sh * 2 * U + (oh % STEP) / 32] |= 1u << (oh % 32);
      M[(size_t)se * 2 * U + U + (oe % STEP) / 32] |= 1u << (oe % 32);
    }
  }
  return M;
}

std::vector<int4> build_spans(const std::vector<int32_t>& st, int span, std::vector<int2>& B, int64_t& slots) {
  std::vector<int4> out;
  B.clear();
  slots = 0;
  const int64_t dim = (int64_t)st.size() - 1;
  int r0 = -1, nl = 0, nz = 0;
  auto close = [&] {
    if (nl > 0) { out.push_back(make_int4(r0, nl, st[r0], nz)); B.push_back(make_int2(0, 0)); }
    nl = 0; nz = 0;
  };
  for (int64_t r = 0; r < dim; ++r) {
    const int len = st[r + 1] - st[r];
    if (len == 0) { close(); continue; }  // (lab: empty lines skipped)
    if (len > span) {
      close();
      const int nch = (len + span - 1) / span;
      for (int c = 0; c < nch; ++c) {
        const int b = st[r] + c * span;
        out.push_back(make_int4((int)r, -1 - c, b, std::min(span, st[r + 1] - b)));
        B.push_back(make_int2((int)slots, nch));
      }
      slots += nch;
      continue;
    }
    if (nz + len > span) close();
    if (nl == 0) r0 = (int)r;
    ++nl;
    nz += len;
  }
  close();
  return out;
}

__global__ void compare_kernel(const double* a, const double* b, int64_t n, double* out) {
  double mx = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double d = fabs(a[i] - b[i]) / fmax(1e-300, fmax(fabs(a[i]), fabs(b[i])));
    mx = fmax(mx, (fabs(a[i] - b[i]) < 1e-300) ? 0.0 : d);
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<unsigned long long*>(out), __double_as_longlong(mx));
}

__global__ void absdiff_kernel(const double* a, const double* b, int64_t n, double* out) {
  double mx = 0.0, mv = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    mx = fmax(mx, fabs(a[i] - b[i]));
    mv = fmax(mv, fabs(b[i]));
  }
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    mv = fmax(mv, __shfl_xor_sync(0xffffffffu, mv, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(reinterpret_cast<unsigned long long*>(out), __double_as_longlong(mx));
    atomicMax(reinterpret_cast<unsigned long long*>(out) + 1, __double_as_longlong(mv));
  }
}

// ------------------------------------------------------------- schedule ---
std::vector<int4> build_items(const std::vector<int32_t>& st, int item, int seqmax, int64_t& n_slots,
                              bool long_only = false) {
  std::vector<int4> chunks, blocks;
  const int64_t dim = (int64_t)st.size() - 1;
  int64_t slots = 0;
  int r0 = -1, cnt = 0, nz = 0;
  auto close = [&] {
    if (cnt > 0) blocks.push_back(make_int4(r0, cnt, 0, 0));
    cnt = 0;
    nz = 0;
  };
  for (int64_t r = 0; r < dim; ++r) {
    const int len = st[r + 1] - st[r];
    if (len > seqmax) {
      const int nch = (len + item - 1) / item;
      for (int c = 0; c < nch; ++c) chunks.push_back(make_int4((int)r, -1 - c, (int)slots, nch));
      slots += nch;
      continue;  // (a long line does not close the open block: blocks are line runs)
    }
    if (cnt == 63 || nz + len > item || (cnt > 0 && r != r0 + cnt)) close();
    if (cnt == 0) r0 = (int)r;
    ++cnt;
    nz += len;
  }
  close();
  if (long_only) blocks.clear();
  n_slots = slots;
  // long chunks first (they are the same cost per item as blocks)
  std::vector<int4> all = chunks;
  all.insert(all.end(), blocks.begin(), blocks.end());
  return all;
}

// ---------------------------------------------------------------- driver ---
struct Vecs {
  double *xb, *y, *lc, *uc, *yn, *dy;      // row pass: gather xb (n)
  double *aty, *x, *xn, *atyn, *dyg;       // column pass: gather dy (m)
};

template <class F>
float time_it(F&& f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  CK(cudaGetLastError());
  return ms * 1000.0f / reps;
}

int main(int argc, char** argv) {
  const int64_t m = argc > 1 ? atoll(argv[1]) : 5000000;
  const int64_t n = argc > 2 ? atoll(argv[2]) : 10000000;
  const int sorted = argc > 3 ? atoi(argv[3]) : 0;
  const char* only = argc > 4 ? argv[4] : nullptr;  // run the variants whose label contains this
  double peak = 6549.1;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);

  int32_t* cnt;
  CK(cudaMalloc(&cnt, n * 4));
  counts_kernel<<<4096, 256>>>(cnt, n, 12345);
  if (sorted) {  // degree ordering: column 0 has the largest count
    int32_t* tmp;
    CK(cudaMalloc(&tmp, n * 4));
    size_t tb = 0;
    cub::DeviceRadixSort::SortKeysDescending(nullptr, tb, cnt, tmp, (int)n);
    void* t;
    CK(cudaMalloc(&t, tb));
    cub::DeviceRadixSort::SortKeysDescending(t, tb, cnt, tmp, (int)n);
    CK(cudaMemcpy(cnt, tmp, n * 4, cudaMemcpyDeviceToDevice));
    cudaFree(t);
    cudaFree(tmp);
  }
  int64_t* cst;
  CK(cudaMalloc(&cst, (n + 1) * 8));
  CK(cudaMemset(cst, 0, 8));
  {
    size_t tb = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tb, cnt, cst + 1, (int)n);
    void* t;
    CK(cudaMalloc(&t, tb));
    cub::DeviceScan::InclusiveSum(t, tb, cnt, cst + 1, (int)n);
    CK(cudaDeviceSynchronize());
    cudaFree(t);
  }
  int64_t nnz = 0;
  CK(cudaMemcpy(&nnz, cst + n, 8, cudaMemcpyDeviceToHost));
  std::printf("m=%lld n=%lld nnz=%lld sorted=%d\n", (long long)m, (long long)n, (long long)nnz, sorted);
  uint64_t *kr, *kc, *k2;
  CK(cudaMalloc(&kr, nnz * 8));
  CK(cudaMalloc(&kc, nnz * 8));
  CK(cudaMalloc(&k2, nnz * 8));
  entries_kernel<<<4096, 256>>>(cst, n, m, 777, kr, kc);
  Csr K, KT;
  K.dim = m; K.nnz = nnz; K.other = n;
  KT.dim = n; KT.nnz = nnz; KT.other = m;
  CK(cudaMalloc(&K.idx, nnz * 4 + 256));
  CK(cudaMalloc(&K.val, nnz * 8 + 256));
  CK(cudaMalloc(&KT.idx, nnz * 4 + 256));
  CK(cudaMalloc(&KT.val, nnz * 8 + 256));
  {
    size_t tb = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb, kr, k2, nnz, 0, 47);
    void* t;
    CK(cudaMalloc(&t, tb));
    cub::DeviceRadixSort::SortKeys(t, tb, kr, k2, nnz, 0, 47);
    int32_t* rc;
    CK(cudaMalloc(&rc, m * 4));
    CK(cudaMemset(rc, 0, m * 4));
    split_row<<<4096, 256>>>(k2, nnz, K.idx, K.val, rc);
    int64_t* rs64;
    CK(cudaMalloc(&rs64, (m + 1) * 8));
    CK(cudaMemset(rs64, 0, 8));
    size_t tb2 = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tb2, rc, rs64 + 1, (int)m);
    void* t2;
    CK(cudaMalloc(&t2, tb2));
    cub::DeviceScan::InclusiveSum(t2, tb2, rc, rs64 + 1, (int)m);
    CK(cudaMalloc(&K.start, (m + 1) * 4));
    i64_to_i32<<<1024, 256>>>(rs64, K.start, m + 1);
    cub::DeviceRadixSort::SortKeys(t, tb, kc, k2, nnz, 0, 47);
    split_col<<<4096, 256>>>(k2, nnz, KT.idx, KT.val);
    CK(cudaMalloc(&KT.start, (n + 1) * 4));
    i64_to_i32<<<1024, 256>>>(cst, KT.start, n + 1);
    CK(cudaDeviceSynchronize());
    cudaFree(t); cudaFree(t2); cudaFree(rc); cudaFree(rs64);
  }
  cudaFree(kr); cudaFree(kc); cudaFree(k2); cudaFree(cnt); cudaFree(cst);
  K.hstart.resize(m + 1);
  KT.hstart.resize(n + 1);
  CK(cudaMemcpy(K.hstart.data(), K.start, (m + 1) * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(KT.hstart.data(), KT.start, (n + 1) * 4, cudaMemcpyDeviceToHost));

  Vecs V;
  auto vec = [&](int64_t len, double lo, double hi, uint64_t seed) {
    double* p;
    CK(cudaMalloc(&p, len * 8 + 16));
    fill_kernel<<<2048, 256>>>(p, len, seed, lo, hi);
    return p;
  };
  V.xb = vec(n, -1, 1, 1); V.y = vec(m, -1, 1, 2); V.lc = vec(m, -2, -1, 3); V.uc = vec(m, 1, 2, 4);
  V.yn = vec(m, 0, 0, 5); V.dy = vec(m, 0, 0, 6);
  V.aty = vec(n, -1, 1, 7); V.x = vec(n, 0, 1, 8); V.xn = vec(n, 0, 1, 9); V.atyn = vec(n, 0, 0, 10);
  V.dyg = vec(m, -1, 1, 11);
  double* outp;
  CK(cudaMalloc(&outp, 148 * 64 * 8 * 8));
  CK(cudaDeviceSynchronize());

  const double row_bytes = 12.0 * nnz + 4.0 * (m + 1) + 8.0 * n + 8.0 * RowEpi::kRW * m;
  const double col_bytes = 12.0 * nnz + 4.0 * (n + 1) + 8.0 * m + 8.0 * ColEpi::kRW * n;
  RowEpi re{V.y, V.lc, V.uc, V.yn, V.dy, 0.37};
  ColEpi ce{V.aty, V.x, V.xn, V.atyn};
  auto want = [&](const char* label) { return only == nullptr || std::strstr(label, only) != nullptr; };
  auto group = [&](const char* g) { return only == nullptr || std::strstr(only, g) != nullptr; };
  auto report = [&](const char* name, float us, double bytes) {
    std::printf("%-44s %9.1f us  %7.0f GB/s  %.3f of peak\n", name, us, bytes / us / 1e3, bytes / us / 1e3 / peak);
  };
  const int reps = 10;

  auto run_wb = [&](auto tag_item, auto tag_minb, const Csr& A, int seqmax, auto epi, const double* v,
                    double bytes, const char* nm, bool long_only = false) {
    constexpr int ITEM = decltype(tag_item)::value;
    constexpr int MINB = decltype(tag_minb)::value;
    {
      char lb[160];
      std::snprintf(lb, sizeof lb, "%s item=%d seq=%d minb=%d", nm, ITEM, seqmax, MINB);
      if (!want(lb)) return;
    }
    int64_t slots = 0;
    std::vector<int4> items = build_items(A.hstart, ITEM, seqmax, slots, long_only);
    int4* d_items;
    CK(cudaMalloc(&d_items, items.size() * sizeof(int4) + 16));
    CK(cudaMemcpy(d_items, items.data(), items.size() * sizeof(int4), cudaMemcpyHostToDevice));
    double* part;
    unsigned* cntp;
    CK(cudaMalloc(&part, (slots + 1) * 8));
    CK(cudaMalloc(&cntp, (slots + 1) * 4));
    CK(cudaMemset(cntp, 0, (slots + 1) * 4));
    auto k = wb_kernel<ITEM, decltype(epi), MINB>;
    int per = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, 256, 0));
    const int grid = sms * per;
    float us = time_it([&] { k<<<grid, 256>>>(d_items, (int64_t)items.size(), A.start, A.idx, A.val, v, epi, part, cntp, outp); }, reps);
    char buf[160];
    std::snprintf(buf, sizeof buf, "%s item=%d seq=%d minb=%d (%d/SM, %zu items)", nm, ITEM, seqmax, MINB, per, items.size());
    report(buf, us, bytes);
    cudaFree(d_items); cudaFree(part); cudaFree(cntp);
  };
  auto run_vec = [&](auto tag_g, const Csr& A, auto epi, const double* v, double bytes, const char* nm) {
    constexpr int G = decltype(tag_g)::value;
    {
      char lb[160];
      std::snprintf(lb, sizeof lb, "%s vec G=%d", nm, G);
      if (!want(lb)) return;
    }
    auto k = vec_kernel<G, decltype(epi), 4>;
    int per = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, 256, 0));
    const int grid = sms * per;
    float us = time_it([&] { k<<<grid, 256>>>(A.dim, A.start, A.idx, A.val, v, epi, outp); }, reps);
    char buf[160];
    std::snprintf(buf, sizeof buf, "%s vec G=%d (%d/SM)", nm, G, per);
    report(buf, us, bytes);
  };
  using I128 = std::integral_constant<int, 128>;
  using I256 = std::integral_constant<int, 256>;
  using I512 = std::integral_constant<int, 512>;
  using B1 = std::integral_constant<int, 1>;
  using B2 = std::integral_constant<int, 2>;
  using B3 = std::integral_constant<int, 3>;
  using B4 = std::integral_constant<int, 4>;
  using G4 = std::integral_constant<int, 4>;
  using G8 = std::integral_constant<int, 8>;
  using G16 = std::integral_constant<int, 16>;
  using G32 = std::integral_constant<int, 32>;
  // row pass (K x-bar + dual epilogue)
  run_vec(G8{}, K, re, V.xb, row_bytes, "row");
  run_vec(G16{}, K, re, V.xb, row_bytes, "row");
  run_vec(G32{}, K, re, V.xb, row_bytes, "row");
  run_wb(I256{}, B2{}, K, 64, re, V.xb, row_bytes, "row");
  run_wb(I256{}, B3{}, K, 64, re, V.xb, row_bytes, "row");
  run_wb(I256{}, B4{}, K, 64, re, V.xb, row_bytes, "row");
  run_wb(I128{}, B4{}, K, 64, re, V.xb, row_bytes, "row");
  run_wb(I512{}, B2{}, K, 64, re, V.xb, row_bytes, "row");
  // column pass (K^T dy + aty epilogue)
  run_vec(G4{}, KT, ce, V.dyg, col_bytes, "col");
  run_vec(G32{}, KT, ce, V.dyg, col_bytes, "col");
  run_wb(I256{}, B2{}, KT, 64, ce, V.dyg, col_bytes, "col");
  run_wb(I256{}, B3{}, KT, 64, ce, V.dyg, col_bytes, "col");
  run_wb(I256{}, B4{}, KT, 64, ce, V.dyg, col_bytes, "col");
  run_wb(I256{}, B4{}, KT, 32, ce, V.dyg, col_bytes, "col");
  run_wb(I256{}, B4{}, KT, 128, ce, V.dyg, col_bytes, "col");
  run_wb(I128{}, B4{}, KT, 64, ce, V.dyg, col_bytes, "col");
  run_wb(I512{}, B2{}, KT, 64, ce, V.dyg, col_bytes, "col");
  if (group("gather")) {
    double* big;
    const int64_t maxlen = 20000000;
    CK(cudaMalloc(&big, maxlen * 8));
    fill_kernel<<<2048, 256>>>(big, maxlen, 99, -1, 1);
    for (int64_t len : {(int64_t)500000, (int64_t)2500000, (int64_t)5000000, (int64_t)10000000, (int64_t)20000000}) {
      for (int per : {4, 8}) {
        const int grid = sms * per;
        float us = time_it([&] { gather_probe<8><<<grid, 256>>>(big, len, nnz, outp); }, reps);
        std::printf("  (unroll 8) ");
        std::printf("gather probe len=%lld (%.0f MB) grid=%d/SM: %.1f us = %.1f Ggather/s\n", (long long)len,
                    len * 8 / 1e6, per, us, nnz / us / 1e3);
      }
    }
    cudaFree(big);
  }
  // warp-private rings
  auto run_wr = [&](auto tag_cw, auto tag_s, auto tag_g, const Csr& A, int E, int L, int seqmax, auto epi,
                    const double* v, const double* a0, const double* a1, const double* a2, double bytes,
                    const char* nm) {
    constexpr int CW = decltype(tag_cw)::value, S = decltype(tag_s)::value, G = decltype(tag_g)::value;
    char lb[160];
    std::snprintf(lb, sizeof lb, "%s ring cw=%d s=%d g=%d E=%d L=%d", nm, CW, S, G, E, L);
    if (!want(lb)) return;
    std::vector<int4> tiles = build_tiles(A.hstart, E, L, seqmax);
    int4* d_t;
    CK(cudaMalloc(&d_t, tiles.size() * sizeof(int4) + 16));
    CK(cudaMemcpy(d_t, tiles.data(), tiles.size() * sizeof(int4), cudaMemcpyHostToDevice));
    const size_t stage = ((4 * E + 32 + 15) & ~15) + ((8 * E + 32 + 15) & ~15) + ((4 * (L + 1) + 32 + 15) & ~15) +
                         3 * ((8 * L + 32 + 15) & ~15);
    const size_t smem = ((16 * CW * S + sizeof(RingHdr) * CW * S + 127) & ~127) + (size_t)CW * S * stage;
    auto k = wr_kernel<CW, S, G, decltype(epi)>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    int per = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, 32 * (CW + 1), smem));
    if (per < 1) { std::printf("%s: does not fit (%zu B)\n", lb, smem); cudaFree(d_t); return; }
    const int grid = sms * per;
    float us = time_it([&] { k<<<grid, 32 * (CW + 1), smem>>>(d_t, (int64_t)tiles.size(), A.start, A.idx, A.val, v, epi, a0, a1, a2, E, L, outp); }, reps);
    char buf[200];
    std::snprintf(buf, sizeof buf, "%s (%d/SM, %zu KB, %zu tiles)", lb, per, smem / 1024, tiles.size());
    report(buf, us, bytes);
    cudaFree(d_t);
  };
  using C3 = std::integral_constant<int, 3>;
  using C7 = std::integral_constant<int, 7>;
  using C15 = std::integral_constant<int, 15>;
  using S2 = std::integral_constant<int, 2>;
  using S3 = std::integral_constant<int, 3>;
  using Q4 = std::integral_constant<int, 4>;
  using Q8 = std::integral_constant<int, 8>;
  using Q16 = std::integral_constant<int, 16>;
  run_wr(C7{}, S2{}, Q8{}, K, 1024, 64, 64, re, V.xb, V.y, V.lc, V.uc, row_bytes, "row");
  run_wr(C7{}, S2{}, Q16{}, K, 1024, 64, 64, re, V.xb, V.y, V.lc, V.uc, row_bytes, "row");
  run_wr(C7{}, S2{}, Q8{}, K, 2048, 96, 64, re, V.xb, V.y, V.lc, V.uc, row_bytes, "row");
  run_wr(C15{}, S2{}, Q8{}, K, 512, 32, 64, re, V.xb, V.y, V.lc, V.uc, row_bytes, "row");
  run_wr(C15{}, S2{}, Q8{}, K, 768, 32, 64, re, V.xb, V.y, V.lc, V.uc, row_bytes, "row");
  run_wr(C15{}, S3{}, Q8{}, K, 512, 32, 64, re, V.xb, V.y, V.lc, V.uc, row_bytes, "row");
  run_wr(C3{}, S2{}, Q8{}, K, 1024, 64, 64, re, V.xb, V.y, V.lc, V.uc, row_bytes, "row");
  run_wr(C7{}, S3{}, Q4{}, K, 1024, 64, 64, re, V.xb, V.y, V.lc, V.uc, row_bytes, "row");
  // column pass, short lines only (long lines: chunk items, reported separately)
  run_wr(C7{}, S2{}, Q8{}, KT, 1024, 256, 64, ce, V.dyg, V.aty, V.x, V.xn, col_bytes, "colshort");
  run_wr(C15{}, S2{}, Q8{}, KT, 512, 128, 64, ce, V.dyg, V.aty, V.x, V.xn, col_bytes, "colshort");
  run_wb(I256{}, B4{}, KT, 64, ce, V.dyg, col_bytes, "collong", true);
  run_wb(I256{}, B3{}, KT, 64, ce, V.dyg, col_bytes, "collong", true);
  run_wb(I512{}, B2{}, KT, 64, ce, V.dyg, col_bytes, "collong", true);
  if (group("sgp")) {
    for (int per : {4, 8}) {
      const int grid = sms * per;
      float us;
      us = time_it([&] { stream_gather_probe<4><<<grid, 256>>>(KT.idx, KT.val, V.dyg, nnz, outp); }, reps);
      std::printf("sgp col (dy 40MB) U=4 %d/SM: %.1f us = %.1f Gentry/s\n", per, us, nnz / us / 1e3);
      us = time_it([&] { stream_gather_probe<8><<<grid, 256>>>(KT.idx, KT.val, V.dyg, nnz, outp); }, reps);
      std::printf("sgp col (dy 40MB) U=8 %d/SM: %.1f us = %.1f Gentry/s\n", per, us, nnz / us / 1e3);
      us = time_it([&] { stream_gather_probe<16><<<grid, 256>>>(KT.idx, KT.val, V.dyg, nnz, outp); }, reps);
      std::printf("sgp col (dy 40MB) U=16 %d/SM: %.1f us = %.1f Gentry/s\n", per, us, nnz / us / 1e3);
      us = time_it([&] { stream_gather_probe<8><<<grid, 256>>>(K.idx, K.val, V.xb, nnz, outp); }, reps);
      std::printf("sgp row (xb 80MB) U=8 %d/SM: %.1f us = %.1f Gentry/s\n", per, us, nnz / us / 1e3);
    }
  }
  auto run_seg = [&](auto tag_minb, const Csr& A, int span, auto epi, const double* v, double bytes,
                     const char* nm, double* outv, double* refv) {
    constexpr int MINB = decltype(tag_minb)::value;
    char lb[160];
    std::snprintf(lb, sizeof lb, "%s seg span=%d minb=%d", nm, span, MINB);
    if (!want(lb)) return;
    std::vector<int2> B;
    int64_t slots = 0;
    std::vector<int4> sp = build_spans(A.hstart, span, B, slots);
    int4* d_s;
    int2* d_b;
    CK(cudaMalloc(&d_s, sp.size() * sizeof(int4) + 16));
    CK(cudaMalloc(&d_b, B.size() * sizeof(int2) + 16));
    CK(cudaMemcpy(d_s, sp.data(), sp.size() * sizeof(int4), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_b, B.data(), B.size() * sizeof(int2), cudaMemcpyHostToDevice));
    double* part;
    unsigned* cntp;
    CK(cudaMalloc(&part, (slots + 1) * 8));
    CK(cudaMalloc(&cntp, (slots + 1) * 4));
    CK(cudaMemset(cntp, 0, (slots + 1) * 4));
    auto k = seg_kernel<decltype(epi), MINB>;
    int per = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, 256, 0));
    const int grid = sms * per;
    float us = time_it([&] { k<<<grid, 256>>>(d_s, d_b, (int64_t)sp.size(), A.start, A.idx, A.val, v, epi, part, cntp, outp); }, reps);
    char buf[200];
    std::snprintf(buf, sizeof buf, "%s (%d/SM, %zu spans)", lb, per, sp.size());
    report(buf, us, bytes);
    if (refv != nullptr) {
      double* mx;
      CK(cudaMalloc(&mx, 8));
      CK(cudaMemset(mx, 0, 8));
      compare_kernel<<<1024, 256>>>(outv, refv, A.dim, mx);
      double h = 0;
      CK(cudaMemcpy(&h, mx, 8, cudaMemcpyDeviceToHost));
      std::printf("   max rel diff vs vec kernel: %.3e\n", h);
      cudaFree(mx);
    }
    cudaFree(d_s); cudaFree(d_b); cudaFree(part); cudaFree(cntp);
  };
  auto run_seg2 = [&](auto tag_u, auto tag_minb, const Csr& A, int span, auto epi, const double* v, double bytes,
                      const char* nm, double* outv, double* refv) {
    constexpr int U = decltype(tag_u)::value;
    constexpr int MINB = decltype(tag_minb)::value;
    char lb[160];
    std::snprintf(lb, sizeof lb, "%s seg2 U=%d span=%d minb=%d", nm, U, span, MINB);
    if (!want(lb)) return;
    std::vector<int2> B;
    int64_t slots = 0;
    std::vector<int4> sp = build_spans(A.hstart, span, B, slots);
    std::vector<int32_t> s0;
    std::vector<uint32_t> M = build_masks(A.hstart, sp, U, s0);
    int4* d_s;
    int2* d_b;
    int32_t* d_s0;
    uint32_t* d_m;
    CK(cudaMalloc(&d_s, sp.size() * sizeof(int4) + 16));
    CK(cudaMalloc(&d_b, B.size() * sizeof(int2) + 16));
    CK(cudaMalloc(&d_s0, s0.size() * 4 + 16));
    CK(cudaMalloc(&d_m, M.size() * 4 + 16));
    CK(cudaMemcpy(d_s, sp.data(), sp.size() * sizeof(int4), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_b, B.data(), B.size() * sizeof(int2), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_s0, s0.data(), s0.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_m, M.data(), M.size() * 4, cudaMemcpyHostToDevice));
    double* part;
    unsigned* cntp;
    CK(cudaMalloc(&part, (slots + 1) * 8));
    CK(cudaMalloc(&cntp, (slots + 1) * 4));
    CK(cudaMemset(cntp, 0, (slots + 1) * 4));
    auto k = seg2_kernel<U, decltype(epi), MINB>;
    int per = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, 256, 0));
    const int grid = sms * per;
    float us = time_it([&] { k<<<grid, 256>>>(d_s, d_b, d_s0, d_m, (int64_t)sp.size(), A.idx, A.val, v, epi, part, cntp, outp); }, reps);
    char buf[200];
    std::snprintf(buf, sizeof buf, "%s (%d/SM, %zu spans, masks %.0f MB)", lb, per, sp.size(), M.size() * 4 / 1e6);
    report(buf, us, bytes);
    if (refv != nullptr) {
      double* mx;
      CK(cudaMalloc(&mx, 8));
      CK(cudaMemset(mx, 0, 8));
      compare_kernel<<<1024, 256>>>(outv, refv, A.dim, mx);
      double h = 0;
      CK(cudaMemcpy(&h, mx, 8, cudaMemcpyDeviceToHost));
      std::printf("   max rel diff vs vec kernel: %.3e\n", h);
      cudaFree(mx);
    }
    cudaFree(d_s); cudaFree(d_b); cudaFree(d_s0); cudaFree(d_m); cudaFree(part); cudaFree(cntp);
  };
  using U4 = std::integral_constant<int, 4>;
  using U8 = std::integral_constant<int, 8>;
  using B5 = std::integral_constant<int, 5>;
  using B6 = std::integral_constant<int, 6>;
  auto run_seg3 = [&](auto tag_minb, const Csr& A, int span, auto epi, const double* v, double bytes,
                      const char* nm, double* outv, double* refv) {
    constexpr int MINB = decltype(tag_minb)::value;
    char lb[160];
    std::snprintf(lb, sizeof lb, "%s seg3 span=%d minb=%d", nm, span, MINB);
    if (!want(lb)) return;
    std::vector<int2> B;
    int64_t slots = 0;
    std::vector<int4> sp = build_spans(A.hstart, span, B, slots);
    std::vector<int32_t> s0;
    std::vector<uint32_t> M = build_masks3(A.hstart, sp, s0);
    int4* d_s;
    int2* d_b;
    int32_t* d_s0;
    uint32_t* d_m;
    CK(cudaMalloc(&d_s, sp.size() * sizeof(int4) + 16));
    CK(cudaMalloc(&d_b, B.size() * sizeof(int2) + 16));
    CK(cudaMalloc(&d_s0, s0.size() * 4 + 16));
    CK(cudaMalloc(&d_m, M.size() * 4 + 16));
    CK(cudaMemcpy(d_s, sp.data(), sp.size() * sizeof(int4), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_b, B.data(), B.size() * sizeof(int2), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_s0, s0.data(), s0.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_m, M.data(), M.size() * 4, cudaMemcpyHostToDevice));
    double* part;
    unsigned* cntp;
    CK(cudaMalloc(&part, (slots + 1) * 8));
    CK(cudaMalloc(&cntp, (slots + 1) * 4));
    CK(cudaMemset(cntp, 0, (slots + 1) * 4));
    auto k = seg3_kernel<decltype(epi), MINB>;
    int per = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, 256, 0));
    const int grid = sms * per;
    float us = time_it([&] { k<<<grid, 256>>>(d_s, d_b, d_s0, d_m, (int64_t)sp.size(), A.idx, A.val, v, epi, part, cntp, outp); }, reps);
    char buf[200];
    std::snprintf(buf, sizeof buf, "%s (%d/SM, %zu spans, masks %.0f MB)", lb, per, sp.size(), M.size() * 4 / 1e6);
    report(buf, us, bytes);
    if (refv != nullptr) {
      double* mx;
      CK(cudaMalloc(&mx, 8));
      CK(cudaMemset(mx, 0, 8));
      compare_kernel<<<1024, 256>>>(outv, refv, A.dim, mx);
      double h = 0;
      CK(cudaMemcpy(&h, mx, 8, cudaMemcpyDeviceToHost));
      std::printf("   max rel diff vs vec kernel: %.3e\n", h);
      cudaFree(mx);
    }
    cudaFree(d_s); cudaFree(d_b); cudaFree(d_s0); cudaFree(d_m); cudaFree(part); cudaFree(cntp);
  };
  if (group("seg3")) {
    double* ref_col;
    CK(cudaMalloc(&ref_col, n * 8));
    ColEpi ce2 = ce;
    ce2.atyn = ref_col;
    vec_kernel<32, ColEpi, 4><<<sms * 4, 256>>>(KT.dim, KT.start, KT.idx, KT.val, V.dyg, ce2, outp);
    double* ref_row;
    CK(cudaMalloc(&ref_row, m * 8));
    RowEpi re2 = re;
    re2.yn = ref_row;
    vec_kernel<8, RowEpi, 4><<<sms * 4, 256>>>(K.dim, K.start, K.idx, K.val, V.xb, re2, outp);
    CK(cudaDeviceSynchronize());
    ColEpiNull cn{V.atyn};
    run_seg3(B4{}, KT, 2048, cn, V.dyg, col_bytes, "colnull", nullptr, nullptr);
    run_seg3(B5{}, KT, 2048, cn, V.dyg, col_bytes, "colnull", nullptr, nullptr);
    for (int span : {1024, 2048, 4096}) {
      run_seg3(B2{}, KT, span, ce, V.dyg, col_bytes, "col", V.atyn, ref_col);
      run_seg3(B3{}, KT, span, ce, V.dyg, col_bytes, "col", V.atyn, ref_col);
      run_seg3(B4{}, KT, span, ce, V.dyg, col_bytes, "col", V.atyn, ref_col);
      run_seg3(B5{}, KT, span, ce, V.dyg, col_bytes, "col", V.atyn, ref_col);
      run_seg3(B4{}, K, span, re, V.xb, row_bytes, "row", V.yn, ref_row);
    }
    cudaFree(ref_col); cudaFree(ref_row);
  }
  if (group("seg2")) {
    double* ref_col;
    CK(cudaMalloc(&ref_col, n * 8));
    ColEpi ce2 = ce;
    ce2.atyn = ref_col;
    vec_kernel<32, ColEpi, 4><<<sms * 4, 256>>>(KT.dim, KT.start, KT.idx, KT.val, V.dyg, ce2, outp);
    CK(cudaDeviceSynchronize());
    for (int span : {1024, 2048}) {
      run_seg2(U8{}, B3{}, KT, span, ce, V.dyg, col_bytes, "col", V.atyn, ref_col);
      run_seg2(U8{}, B4{}, KT, span, ce, V.dyg, col_bytes, "col", V.atyn, ref_col);
      run_seg2(U4{}, B4{}, KT, span, ce, V.dyg, col_bytes, "col", V.atyn, ref_col);
      run_seg2(U4{}, B5{}, KT, span, ce, V.dyg, col_bytes, "col", V.atyn, ref_col);
      run_seg2(U4{}, B6{}, KT, span, ce, V.dyg, col_bytes, "col", V.atyn, ref_col);
    }
    cudaFree(ref_col);
  }
  if (group("seg")) {
    // reference outputs from the vec kernel (tree sums)
    double* ref_col;
    CK(cudaMalloc(&ref_col, n * 8));
    ColEpi ce2 = ce;
    ce2.atyn = ref_col;
    vec_kernel<32, ColEpi, 4><<<sms * 4, 256>>>(KT.dim, KT.start, KT.idx, KT.val, V.dyg, ce2, outp);
    double* ref_row;
    CK(cudaMalloc(&ref_row, m * 8));
    RowEpi re2 = re;
    re2.yn = ref_row;
    vec_kernel<8, RowEpi, 4><<<sms * 4, 256>>>(K.dim, K.start, K.idx, K.val, V.xb, re2, outp);
    CK(cudaDeviceSynchronize());
    for (int span : {1024, 2048, 4096}) {
      run_seg(B2{}, KT, span, ce, V.dyg, col_bytes, "col", V.atyn, ref_col);
      run_seg(B3{}, KT, span, ce, V.dyg, col_bytes, "col", V.atyn, ref_col);
      run_seg(B4{}, KT, span, ce, V.dyg, col_bytes, "col", V.atyn, ref_col);
      run_seg(B3{}, K, span, re, V.xb, row_bytes, "row", V.yn, ref_row);
    }
    cudaFree(ref_col); cudaFree(ref_row);
  }
  // row pass over P column panels
  for (int P : {2, 3, 4, 6}) {
    {
      char lb[64];
      std::snprintf(lb, sizeof lb, "row panels P=%d", P);
      if (!want(lb)) continue;
    }
    const int64_t W = (n + P - 1) / P;
    int32_t* pc;
    int64_t* pst;
    CK(cudaMalloc(&pc, (int64_t)P * m * 4));
    CK(cudaMalloc(&pst, ((int64_t)P * m + 1) * 8));
    CK(cudaMemset(pc, 0, (int64_t)P * m * 4));
    panel_count<<<2048, 256>>>(K.start, K.idx, m, P, W, pc);
    CK(cudaMemset(pst, 0, 8));
    size_t tb = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tb, pc, pst + 1, (int)(P * m));
    void* t;
    CK(cudaMalloc(&t, tb));
    cub::DeviceScan::InclusiveSum(t, tb, pc, pst + 1, (int)(P * m));
    int32_t* nidx;
    double* nval;
    CK(cudaMalloc(&nidx, nnz * 4 + 16));
    CK(cudaMalloc(&nval, nnz * 8 + 16));
    panel_scatter<<<2048, 256>>>(K.start, K.idx, K.val, m, P, W, pst, nidx, nval);
    int32_t* pst32;
    CK(cudaMalloc(&pst32, ((int64_t)P * m + 1) * 4));
    i64_to_i32<<<1024, 256>>>(pst, pst32, (int64_t)P * m + 1);
    double* carry;
    CK(cudaMalloc(&carry, m * 8));
    CK(cudaDeviceSynchronize());
    auto run_panels = [&](auto tag_g) {
      constexpr int G = decltype(tag_g)::value;
      int per = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, panel_kernel<G, RowEpi, 1, 4>, 256, 0));
      const int grid = sms * per;
      float us = time_it([&] {
        for (int p = 0; p < P; ++p) {
          // panel p's row pointers are pst32[p*m .. p*m+m] (global positions)
          const int32_t* st = pst32 + (int64_t)p * m;
          if (p == 0) panel_kernel<G, RowEpi, 0, 4><<<grid, 256>>>(m, st, nidx, nval, V.xb, re, carry, outp);
          else if (p == P - 1) panel_kernel<G, RowEpi, 2, 4><<<grid, 256>>>(m, st, nidx, nval, V.xb, re, carry, outp);
          else panel_kernel<G, RowEpi, 1, 4><<<grid, 256>>>(m, st, nidx, nval, V.xb, re, carry, outp);
        }
      }, reps);
      char buf[160];
      std::snprintf(buf, sizeof buf, "row panels P=%d G=%d (%d/SM)", P, G, per);
      report(buf, us, row_bytes);
    };
    run_panels(G4{});
    run_panels(G8{});
    cudaFree(t); cudaFree(pc); cudaFree(pst); cudaFree(nidx); cudaFree(nval); cudaFree(pst32); cudaFree(carry);
  }

  // row pass on SELL-32-sigma slices, over P column panels (P = 1: one pass)
  for (int P : {1, 2}) {
    {
      char lb[64];
      std::snprintf(lb, sizeof lb, "row sell P=%d", P);
      if (!want(lb)) continue;
    }
    const int64_t W = (n + P - 1) / P;
    int32_t* pc;
    int64_t* pst;
    CK(cudaMalloc(&pc, (int64_t)P * m * 4));
    CK(cudaMalloc(&pst, ((int64_t)P * m + 1) * 8));
    CK(cudaMemset(pc, 0, (int64_t)P * m * 4));
    panel_count<<<2048, 256>>>(K.start, K.idx, m, P, W, pc);
    CK(cudaMemset(pst, 0, 8));
    size_t tb = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tb, pc, pst + 1, (int)(P * m));
    void* t;
    CK(cudaMalloc(&t, tb));
    cub::DeviceScan::InclusiveSum(t, tb, pc, pst + 1, (int)(P * m));
    int32_t* nidx;
    double* nval;
    CK(cudaMalloc(&nidx, nnz * 4 + 16));
    CK(cudaMalloc(&nval, nnz * 8 + 16));
    panel_scatter<<<2048, 256>>>(K.start, K.idx, K.val, m, P, W, pst, nidx, nval);
    int32_t* pst32;
    CK(cudaMalloc(&pst32, ((int64_t)P * m + 1) * 4));
    i64_to_i32<<<1024, 256>>>(pst, pst32, (int64_t)P * m + 1);
    double *carry, *ref;
    CK(cudaMalloc(&carry, m * 8));
    CK(cudaMalloc(&ref, m * 8));
    CK(cudaDeviceSynchronize());
    // reference result: the CSR panel kernels (same storage-order sums only for G = 1; compare to rounding)
    for (int p = 0; p < P; ++p) {
      const int32_t* st = pst32 + (int64_t)p * m;
      if (P == 1) vec_kernel<8, RowEpi, 4><<<sms * 4, 256>>>(m, st, nidx, nval, V.xb, re, outp);
      else if (p == 0) panel_kernel<8, RowEpi, 0, 4><<<sms * 4, 256>>>(m, st, nidx, nval, V.xb, re, carry, outp);
      else if (p == P - 1) panel_kernel<8, RowEpi, 2, 4><<<sms * 4, 256>>>(m, st, nidx, nval, V.xb, re, carry, outp);
      else panel_kernel<8, RowEpi, 1, 4><<<sms * 4, 256>>>(m, st, nidx, nval, V.xb, re, carry, outp);
    }
    CK(cudaMemcpy(ref, V.yn, m * 8, cudaMemcpyDeviceToDevice));
    for (int64_t sigma : {(int64_t)32, (int64_t)1024, (int64_t)8192, (int64_t)1 << 30}) {
      const int64_t ng = (m + 31) / 32;
      struct Sell { int64_t* off; int32_t *perm, *len, *sidx; double* sval; int64_t slots; } L[4];
      uint64_t *key, *key2;
      int32_t* rid;
      CK(cudaMalloc(&key, m * 8));
      CK(cudaMalloc(&key2, m * 8));
      CK(cudaMalloc(&rid, m * 4));
      double pad_total = 0;
      for (int p = 0; p < P; ++p) {
        const int32_t* st = pst32 + (int64_t)p * m;
        CK(cudaMalloc(&L[p].len, m * 4));
        CK(cudaMalloc(&L[p].perm, m * 4));
        CK(cudaMalloc(&L[p].off, (ng + 1) * 8));
        sell_len<<<2048, 256>>>(st, m, sigma, L[p].len, key, rid);
        size_t sb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, sb, key, key2, rid, L[p].perm, (int)m);
        void* stmp;
        CK(cudaMalloc(&stmp, sb));
        cub::DeviceRadixSort::SortPairs(stmp, sb, key, key2, rid, L[p].perm, (int)m);
        int64_t* w32;
        CK(cudaMalloc(&w32, ng * 8));
        sell_width<<<2048, 256>>>(L[p].len, L[p].perm, m, ng, w32);
        CK(cudaMemset(L[p].off, 0, 8));
        size_t cb = 0;
        cub::DeviceScan::InclusiveSum(nullptr, cb, w32, L[p].off + 1, (int)ng);
        void* ctmp;
        CK(cudaMalloc(&ctmp, cb));
        cub::DeviceScan::InclusiveSum(ctmp, cb, w32, L[p].off + 1, (int)ng);
        CK(cudaMemcpy(&L[p].slots, L[p].off + ng, 8, cudaMemcpyDeviceToHost));
        CK(cudaMalloc(&L[p].sidx, L[p].slots * 4 + 256));
        CK(cudaMalloc(&L[p].sval, L[p].slots * 8 + 256));
        CK(cudaMemset(L[p].sidx, 0, L[p].slots * 4));
        CK(cudaMemset(L[p].sval, 0, L[p].slots * 8));
        sell_fill<<<2048, 256>>>(st, nidx, nval, L[p].perm, m, L[p].off, L[p].sidx, L[p].sval);
        CK(cudaDeviceSynchronize());
        pad_total += (double)L[p].slots;
        cudaFree(stmp); cudaFree(ctmp); cudaFree(w32);
      }
      auto run_sell = [&](auto tag_u, auto tag_minb, auto tag_slot) {
        constexpr int U = decltype(tag_u)::value;
        constexpr int MINB = decltype(tag_minb)::value;
        constexpr bool SLOT = decltype(tag_slot)::value != 0;
        int per = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, sell_kernel<U, RowEpi, 2, MINB, SLOT>, 256, 0));
        const int grid = sms * per;
        CK(cudaMemset(V.yn, 0, m * 8));
        float us = time_it([&] {
          for (int p = 0; p < P; ++p) {
            const Sell& A = L[p];
            if (P == 1) sell_kernel<U, RowEpi, 3, MINB, SLOT><<<grid, 256>>>(m, ng, A.off, A.perm, A.len, A.sidx, A.sval, V.xb, re, carry, outp);
            else if (p == 0) sell_kernel<U, RowEpi, 0, MINB, SLOT><<<grid, 256>>>(m, ng, A.off, A.perm, A.len, A.sidx, A.sval, V.xb, re, carry, outp);
            else if (p == P - 1) sell_kernel<U, RowEpi, 2, MINB, SLOT><<<grid, 256>>>(m, ng, A.off, A.perm, A.len, A.sidx, A.sval, V.xb, re, carry, outp);
            else sell_kernel<U, RowEpi, 1, MINB, SLOT><<<grid, 256>>>(m, ng, A.off, A.perm, A.len, A.sidx, A.sval, V.xb, re, carry, outp);
          }
        }, reps);
        char buf[200];
        std::snprintf(buf, sizeof buf, "row sell P=%d sigma=%lld U=%d (%d/SM) pad=%.3f%s", P, (long long)sigma, U, per,
                      pad_total / nnz, SLOT ? " slot-order vectors" : "");
        report(buf, us, row_bytes);
        if (!SLOT) {  // the epilogue's output is rounding noise where the projection is inactive: absolute check
          double* mx;
          CK(cudaMalloc(&mx, 16));
          CK(cudaMemset(mx, 0, 16));
          absdiff_kernel<<<1024, 256>>>(V.yn, ref, m, mx);
          double h[2] = {0, 0};
          CK(cudaMemcpy(h, mx, 16, cudaMemcpyDeviceToHost));
          std::printf("   max |diff| vs CSR kernel: %.3e (max |value| %.3e)\n", h[0], h[1]);
          cudaFree(mx);
        }
      };
      using S0 = std::integral_constant<int, 0>;
      using S1 = std::integral_constant<int, 1>;
      run_sell(U8{}, B4{}, S0{});
      run_sell(U8{}, B3{}, S0{});
      run_sell(U4{}, B6{}, S0{});
      run_sell(U8{}, B4{}, S1{});
      run_sell(U8{}, B3{}, S1{});
      run_sell(U4{}, B6{}, S1{});
      for (int p = 0; p < P; ++p) {
        cudaFree(L[p].off); cudaFree(L[p].perm); cudaFree(L[p].len); cudaFree(L[p].sidx); cudaFree(L[p].sval);
      }
      cudaFree(key); cudaFree(key2); cudaFree(rid);
    }
    cudaFree(t); cudaFree(pc); cudaFree(pst); cudaFree(nidx); cudaFree(nval); cudaFree(pst32); cudaFree(carry); cudaFree(ref);
  }
  // a copy of the same bytes, for calibration
  {
    double *a, *b;
    const int64_t words = (int64_t)(row_bytes / 16);
    CK(cudaMalloc(&a, words * 8));
    CK(cudaMalloc(&b, words * 8));
    float us = time_it([&] { cudaMemcpyAsync(b, a, words * 8, cudaMemcpyDeviceToDevice); }, reps);
    report("memcpy (same bytes as row pass)", us, 16.0 * words);
    cudaFree(a); cudaFree(b);
  }
  return 0;
}
