// permute.cu -- reorder sample values into plan order (paper step 3, PAPER.md:191:
// "the location of coordinates and sampling value in memory ... was adjusted according to
// their pixel_idx"), fused with the [C][N] -> [N][C] transpose the hot loop wants.
//
// Iterates in ORIGINAL sample order so both sides stay coalesced: a 32-sample x 32-channel
// tile is read as 32 rows of 128 B from the user's [C][ld] array, transposed in shared
// memory, and each sample's 32 channels are written as one 128 B run of plan row
// iperm[n].  Samples that cannot reach any cell (plan position >= n_used) are skipped.
#include "common.cuh"

namespace hg {

__global__ void __launch_bounds__(256) k_permute(const float* __restrict__ src, int64_t ld_src,
                                                 int C, int64_t n, const int32_t* __restrict__ iperm,
                                                 int64_t n_used, float* __restrict__ dst,
                                                 int64_t ld_dst) {
    __shared__ float t[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
    const int64_t n0 = (int64_t)blockIdx.x * 32;
    const int c0 = blockIdx.y * 32;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int c = c0 + ty + 8 * r;
        const int64_t s = n0 + tx;
        t[ty + 8 * r][tx] = (c < C && s < n) ? src[(int64_t)c * ld_src + s] : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int sl = ty + 8 * r;
        const int64_t s = n0 + sl;
        if (s < n) {
            const int64_t pos = iperm[s];
            const int c = c0 + tx;
            if (pos < n_used && c < C) dst[pos * ld_dst + c] = t[tx][sl];
        }
    }
}

hegrid_status launch_permute(const hegrid_plan_s* p, const float* d_user, int64_t n_channels,
                             int64_t ld_user, float* d_plan, int64_t ld_plan, cudaStream_t st) {
    if (n_channels <= 0 || p->n == 0) return HEGRID_OK;
    int64_t gx = (p->n + 31) / 32;
    int64_t gy = (n_channels + 31) / 32;
    if (gy > 65535) return HEGRID_EINVAL;
    k_permute<<<dim3((unsigned)gx, (unsigned)gy), 256, 0, st>>>(
        d_user, ld_user, (int)n_channels, p->n, p->d_iperm, p->n_used, d_plan, ld_plan);
    count_launch();
    return cuda_status(cudaGetLastError());
}

}  // namespace hg
