// Host -> device upload through a pinned staging ring.
//
// A pageable cudaMemcpyAsync moves ~5-7 GB/s: the driver copies the source
// into its own small pinned buffers with one thread, then DMAs.  The solve's
// inputs are ~390 MB on the bench workload (two CSR layouts with 64-bit
// indices plus the bound vectors), so the stager does the same job with a
// process-wide ring of pinned chunks that a pool of host threads fills in
// parallel while the copy engine drains the previous chunks on the caller's
// stream.  Semantics match a pageable cudaMemcpyAsync: the source has been
// read when the call returns; the device copy completes in stream order.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace pdlp_host {

// Copies `bytes` from pageable host memory to device memory in stream order.
// Small copies go straight to cudaMemcpyAsync.  Thread-safe (one upload at a
// time through the ring).
void stage_h2d(void* dst, const void* src, size_t bytes, cudaStream_t s);

// Uploads `count` int64 values narrowed to int32 (saturating: a value outside
// int32 becomes -1 or INT32_MAX, so range checks still reject it): half the
// bytes over PCIe for indices and line starts.
void stage_h2d_narrow(int32_t* dst, const int64_t* src, size_t count, cudaStream_t s);

// Device -> pageable host download through the same ring: the copy engine
// fills pinned chunks while the pool copies finished chunks out.  Runs after
// the work already in `s`; returns with `dst` filled (synchronous, like a
// pageable cudaMemcpy).
void stage_d2h(void* dst, const void* src, size_t bytes, cudaStream_t s);

// Whether p is page-locked host memory (uploads from / downloads into it
// bypass the ring: one DMA, indices narrowed on the device).
bool is_pinned(const void* p);

// Staged upload time since the last call: waiting for ring slots (DMA-bound)
// vs host copies into them (copy-bound), and the bytes staged.
void stage_report(double* wait_s, double* copy_s, double* mbytes);

}  // namespace pdlp_host
