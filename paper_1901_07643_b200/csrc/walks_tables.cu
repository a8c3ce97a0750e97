// walks_tables.cu -- the slot-split walk kernel (walks_kernel.cuh, design S) instantiated
// for the separate RSS / BIC table layouts (bnreg_run, bnreg_all_rss, bnreg_bic).
#include "walks_kernel.cuh"

namespace bnr {

cudaError_t launch_walks_tables(const TravParams& P, int grid, cudaStream_t st)
{
    const int key = (P.out_rss ? 2 : 0) | (P.out_bic ? 1 : 0);
    switch (key) {
        case 3: return launch_ws<true, true, false>(P, grid, st);
        case 2: return launch_ws<true, false, false>(P, grid, st);
        case 1: return launch_ws<false, true, false>(P, grid, st);
        default: return launch_ws<false, false, false>(P, grid, st);
    }
}

}  // namespace bnr
