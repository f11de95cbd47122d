// Multi-vector products for the cadence (perf mode): out_q = A v_q for up
// to four operand vectors in one pass over a layout with a segmented-span
// schedule (spmv.cuh seg_spans).  The operands are packed interleaved
// (pack[i * VEC + q] = v_q[i]), so each entry costs one 8*VEC-byte gather --
// one L2 sector for VEC <= 4 -- and the index / value streams are read once
// for all VEC products.  The gathers, not the bytes, bound these products
// (DESIGN.md §4), so VEC products cost little more than one.
//
// Per vector the arithmetic is exactly seg_spans': lane-contiguous 8-entry
// segments summed in storage order, the same segmented scan across lanes,
// chunked long lines combined in chunk order by the last-arriving chunk --
// each out_q is bit-identical to a single-vector product on the same
// schedule.  Translation unit compiled with -fmad=false.

#include "common.cuh"
#include "kernels.h"
#include "spmv.cuh"

#include <algorithm>

namespace pdlp {
namespace {

constexpr int kT = 256;

template <int VEC>
__global__ void __launch_bounds__(kT) pack_kernel(pdlpk_multi_vecs in, int64_t n, double* pack) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
#pragma unroll
    for (int q = 0; q < VEC; ++q) pack[i * VEC + q] = in.v[q][i];
  }
}

template <int VEC>
__device__ __forceinline__ void gather_vec(const double* __restrict__ pack, int c, double (&g)[VEC]) {
  const double2* p = reinterpret_cast<const double2*>(pack + static_cast<int64_t>(c) * VEC);
#pragma unroll
  for (int q = 0; q < VEC / 2; ++q) {
    const double2 t = __ldg(p + q);
    g[2 * q] = t.x;
    g[2 * q + 1] = t.y;
  }
}

template <int VEC>
__global__ void __launch_bounds__(kT, 2) seg_multi_kernel(pdlpk_csr A, const double* __restrict__ vals,
                                                         const double* __restrict__ pack,
                                                         pdlpk_multi_vecs out, double* part) {
  const int32_t* __restrict__ idx = A.index;
  const int lane = threadIdx.x & 31;
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint64_t pol = l2_first_policy();
  for (int64_t it = gw; it < A.n_seg_spans; it += nw) {
    const int4 d = A.seg_spans[it];
    const int64_t e0 = static_cast<int64_t>(static_cast<uint32_t>(d.z)) |
                       (static_cast<int64_t>(A.seg_aux[it].w) << 32);
    const int64_t e1 = e0 + d.w;
    if (d.y < 0) {
      double acc[VEC];
#pragma unroll
      for (int q = 0; q < VEC; ++q) acc[q] = 0.0;
      for (int64_t base = e0 & ~int64_t(7); base < e1; base += 256) {
        const int64_t k0 = base + 8 * lane;
        if (k0 + 8 > e0 && k0 < e1) {
          const int4 i0 = ld_stream_ef(reinterpret_cast<const int4*>(idx + k0), pol);
          const int4 i1 = ld_stream_ef(reinterpret_cast<const int4*>(idx + k0 + 4), pol);
          const int ci[8] = {i0.x, i0.y, i0.z, i0.w, i1.x, i1.y, i1.z, i1.w};
          double a[8];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const double2 t = ld_stream_ef(reinterpret_cast<const double2*>(vals + k0) + q, pol);
            a[2 * q] = t.x;
            a[2 * q + 1] = t.y;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (k0 + u >= e0 && k0 + u < e1) {
              double g[VEC];
              gather_vec<VEC>(pack, ci[u], g);
#pragma unroll
              for (int q = 0; q < VEC; ++q) acc[q] = mac(acc[q], a[u], g[q]);
            }
          }
        }
      }
      double t[VEC];
#pragma unroll
      for (int q = 0; q < VEC; ++q) t[q] = warp_sum(acc[q]);
      if (lane == 0) {
        const int4 x = A.seg_aux[it];
        const int c = -1 - d.y, nch = x.y;
        if (nch == 1) {
#pragma unroll
          for (int q = 0; q < VEC; ++q) out.v[q][d.x] = 0.0 + t[q];
        } else {
#pragma unroll
          for (int q = 0; q < VEC; ++q) part[(static_cast<int64_t>(x.x) + c) * VEC + q] = t[q];
          __threadfence();
          const unsigned arrived = atomicAdd(A.chunk_cnt + x.x, 1u);
          if (arrived == static_cast<unsigned>(nch - 1)) {
            __threadfence();
#pragma unroll
            for (int q = 0; q < VEC; ++q) {
              double tot = 0.0;
              for (int r = 0; r < nch; ++r) tot += __ldcg(part + (static_cast<int64_t>(x.x) + r) * VEC + q);
              out.v[q][d.x] = 0.0 + tot;
            }
            A.chunk_cnt[x.x] = 0;
          }
        }
      }
      continue;
    }
    int64_t rc = d.x;
    double carry[VEC];
#pragma unroll
    for (int q = 0; q < VEC; ++q) carry[q] = 0.0;
    int64_t sid = A.seg_step0[it];
    for (int64_t base = e0 & ~int64_t(7); base < e1; base += 256, ++sid) {
      const uint32_t mw = lane < 16 ? __ldg(A.seg_masks + sid * 16 + lane) : 0u;
      const int64_t k0 = base + 8 * lane;
      double p[8][VEC];
      if (k0 + 8 > e0 && k0 < e1) {
        const int4 i0 = ld_stream_ef(reinterpret_cast<const int4*>(idx + k0), pol);
        const int4 i1 = ld_stream_ef(reinterpret_cast<const int4*>(idx + k0 + 4), pol);
        const int ci[8] = {i0.x, i0.y, i0.z, i0.w, i1.x, i1.y, i1.z, i1.w};
        double a[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double2 t = ld_stream_ef(reinterpret_cast<const double2*>(vals + k0) + q, pol);
          a[2 * q] = t.x;
          a[2 * q + 1] = t.y;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (k0 + u >= e0 && k0 + u < e1) {
            double g[VEC];
            gather_vec<VEC>(pack, ci[u], g);
#pragma unroll
            for (int q = 0; q < VEC; ++q) p[u][q] = a[u] * g[q];
          } else {
#pragma unroll
            for (int q = 0; q < VEC; ++q) p[u][q] = 0.0;
          }
        }
      } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
#pragma unroll
          for (int q = 0; q < VEC; ++q) p[u][q] = 0.0;
        }
      }
      const uint32_t hw = __shfl_sync(0xffffffffu, mw, lane >> 2);
      const uint32_t ew = __shfl_sync(0xffffffffu, mw, 8 + (lane >> 2));
      const uint32_t hb = (hw >> (8 * (lane & 3))) & 0xffu, eb = (ew >> (8 * (lane & 3))) & 0xffu;
      const int nend_lane = __popc(eb);
      const int ends_before = warp_excl_scan_i(nend_lane, lane);
      const int nend = __shfl_sync(0xffffffffu, ends_before + nend_lane, 31);
      const unsigned hmask = __ballot_sync(0xffffffffu, hb != 0u);
#pragma unroll
      for (int q = 0; q < VEC; ++q) {
        double tail = 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) tail = ((hb >> u) & 1u) ? p[u][q] : tail + p[u][q];
        double inc = tail;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double t = __shfl_up_sync(0xffffffffu, inc, o);
          const unsigned win = lane >= o ? (((2u << lane) - 1u) & ~((1u << (lane - o + 1)) - 1u)) : 0u;
          if (lane >= o && (hmask & win) == 0u) inc += t;
        }
        double into = __shfl_up_sync(0xffffffffu, inc, 1);
        if (lane == 0) into = 0.0;
        if ((hmask & ((1u << lane) - 1u)) == 0u) into += carry[q];
        double run = into;
        int64_t line = rc + ends_before;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          run = ((hb >> u) & 1u) ? p[u][q] : run + p[u][q];
          if ((eb >> u) & 1u) {
            out.v[q][line] = 0.0 + run;
            ++line;
          }
        }
        carry[q] = __shfl_sync(0xffffffffu, run, 31);
        if ((__shfl_sync(0xffffffffu, eb, 31) >> 7) & 1u) carry[q] = 0.0;
      }
      rc += nend;
    }
  }
}

}  // namespace
}  // namespace pdlp

using namespace pdlp;

extern "C" int pdlpk_spmv_multi(const pdlpk_csr* A, int32_t orig, int32_t vec,
                                const pdlpk_multi_vecs* in, int64_t operand_len, double* pack,
                                const pdlpk_multi_vecs* out, double* part, cudaStream_t s) {
  if (!A->seg_mode || (vec != 2 && vec != 4)) return static_cast<int>(cudaErrorInvalidValue);
  const double* vals = orig ? A->value_orig : A->value;
  const unsigned pg = static_cast<unsigned>(std::min<int64_t>((operand_len + kT - 1) / kT, 148 * 8));
  if (operand_len > 0) {
    if (vec == 2) pack_kernel<2><<<pg > 0 ? pg : 1, kT, 0, s>>>(*in, operand_len, pack);
    else pack_kernel<4><<<pg > 0 ? pg : 1, kT, 0, s>>>(*in, operand_len, pack);
  }
  static int per_sm[2] = {0, 0};
  int& occ = per_sm[vec == 2 ? 0 : 1];
  if (occ == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &occ, vec == 2 ? seg_multi_kernel<2> : seg_multi_kernel<4>, kT, 0) != cudaSuccess ||
        occ < 1) {
      cudaGetLastError();
      occ = 1;
    }
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned g = static_cast<unsigned>(sms * occ);
  if (vec == 2) seg_multi_kernel<2><<<g, kT, 0, s>>>(*A, vals, pack, *out, part);
  else seg_multi_kernel<4><<<g, kT, 0, s>>>(*A, vals, pack, *out, part);
  return static_cast<int>(cudaGetLastError());
}
