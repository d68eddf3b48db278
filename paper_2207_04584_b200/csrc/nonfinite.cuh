// nonfinite.cuh -- non-finite sample values (NaN / +-Inf) in Eq. 1.
//
// Eq. 1 sums V[s_n] w over the samples within R of a cell; in IEEE
// arithmetic a NaN or Inf value therefore makes exactly those cells' values NaN / +-Inf
// (the oracle's fp64 sum does the same; reading R15: no masking).  The engines multiply a
// sample's value by the weights of a whole block of cells, most of them zero, and
// 0 * NaN = NaN would poison cells outside the sample's support.  So the value loaders
// replace a non-finite value by 0 (the finite part of every sum stays exact) and record
// (plan position, channel); after the launch, k_nonfinite_fix combines each recorded value
// into the cells within its support, with IEEE semantics (NaN wins, +Inf with -Inf gives
// NaN), order-independent.  Records that do not fit set the overflow flag, and the fix-up
// then scans every value instead.  With hegrid_opts.nonfinite = MASK the fix-up instead
// recomputes the affected (cell, channel) values over the finite values only.
#pragma once

#include <float.h>

#include "common.cuh"

namespace hg {

// Device record buffer: hdr[0] = count, hdr[1] = overflow; rec[k] = plan position |
// channel << 32.  Allocated per launch (stream-ordered), capacity kNfCap.
constexpr uint32_t kNfCap = 1u << 16;
struct NfBuf {
    uint32_t* hdr;
    unsigned long long* rec;
};

__device__ __forceinline__ bool nf_bad(float s) { return !(fabsf(s) <= FLT_MAX); }

static __device__ __noinline__ void nf_record(NfBuf nf, uint32_t p, uint32_t ch) {
    const uint32_t k = atomicAdd(&nf.hdr[0], 1u);
    if (k < kNfCap)
        nf.rec[k] = (unsigned long long)p | ((unsigned long long)ch << 32);
    else
        atomicExch(&nf.hdr[1], 1u);
}

hegrid_status nonfinite_alloc(const hegrid_plan_s* p, NfBuf* nf, cudaStream_t st);
hegrid_status nonfinite_fix(const hegrid_plan_s* p, const float* d_v, int64_t ldv, int C, NfBuf nf,
                            float* d_out, cudaStream_t st);

}  // namespace hg
