// walk_pairs.cu -- the walk kernel (walk_kernel.cuh) instantiated for the (RSS, BIC)
// record layout (bnreg_run_pairs, the bench's layout), the launch dispatch and the
// walk's resource queries.
#include "walk_kernel.cuh"

namespace bnr {

cudaError_t launch_walk_tables(const TravParams& P, int grid, cudaStream_t st);   // walk_tables.cu

size_t walk_cta_smem(int m, int k, int SA, int g, int lw) { return walk_cta_smem_h(m, k, SA, g, lw); }
int walk_tmem_cols(int k, int jbmax) { return walk_tmem_cols_h(k, jbmax); }

cudaError_t launch_walk(const TravParams& P, int grid, cudaStream_t st)
{
    if (P.lw != 3 || P.k > 8 || P.jbmax > 7) return cudaErrorInvalidValue;   // 8 workers per warp, k <= 8
    if (!P.out_pairs) return launch_walk_tables(P, grid, st);
    return P.jbmax <= 4 ? launch_w<false, false, true, 4>(P, grid, st) : launch_w<false, false, true, 7>(P, grid, st);
}

int walk_max_ctas_per_sm(int m, int k, int S_alloc, int g, int jbmax)
{
    // computed from the limits directly: cudaOccupancyMaxActiveBlocksPerMultiprocessor
    // reports 1 CTA per SM for this kernel (measured on B200, CUDA 12.9), although the
    // SM runs 4 (ncu launch__occupancy_limit_*)
    TravParams P{};
    P.m = m; P.k = k; P.S_alloc = S_alloc; P.g = g; P.lw = 3; P.jbmax = jbmax;
    P.tm_cols = walk_tmem_cols(k, jbmax);
    const size_t smem = walk_launch_smem(P);
    auto f = jbmax <= 4 ? walk_kernel<false, false, true, 4> : walk_kernel<false, false, true, 7>;
    if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, f) != cudaSuccess) return 0;
    int dev = 0, smem_sm = 0, regs_sm = 0, thr_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&thr_sm, cudaDevAttrMaxThreadsPerMultiProcessor, dev);
    const int threads = 32 << g;
    const int regs_warp = ((fa.numRegs * 32 + 255) / 256) * 256;
    const int by_regs = regs_sm / (regs_warp * (threads / 32));
    const int by_smem = (int)((size_t)smem_sm / (smem + fa.sharedSizeBytes + 1024));
    const int by_thr = thr_sm / threads;
    return std::max(0, std::min(std::min(by_regs, by_smem), std::min(by_thr, 512 / P.tm_cols)));
}

}  // namespace bnr
