// walks_pairs.cu -- the slot-split walk kernel (walks_kernel.cuh, design S)
// instantiated for the (RSS, BIC) record layout (bnreg_run_pairs, the bench's layout).
#include "walks_kernel.cuh"

namespace bnr {

cudaError_t launch_walks_tables(const TravParams& P, int grid, cudaStream_t st);   // walks_tables.cu

size_t walks_cta_smem(int k, int S_alloc) { return walks_cta_smem_h(k, S_alloc); }

cudaError_t launch_walks(const TravParams& P, int grid, cudaStream_t st)
{
    // 32 workers per CTA (3 warp + 2 gang variables), k <= 8, at most 4 back entries per lane
    if (P.lw != 3 || P.p != 3 || P.g != 2 || P.k > 8 || P.jbmax > 4) return cudaErrorInvalidValue;
    if (!P.out_pairs) return launch_walks_tables(P, grid, st);
    return launch_ws<false, false, true>(P, grid, st);
}

}  // namespace bnr
