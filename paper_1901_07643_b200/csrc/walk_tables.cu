// walk_tables.cu -- the walk kernel (walk_kernel.cuh) instantiated for the separate
// RSS / BIC table layouts (bnreg_run, bnreg_all_rss, bnreg_bic).
#include "walk_kernel.cuh"

namespace bnr {

template <int JBMAX>
static cudaError_t launch_tab(const TravParams& P, int grid, cudaStream_t st)
{
    const int key = (P.out_rss ? 2 : 0) | (P.out_bic ? 1 : 0);
    switch (key) {
        case 3: return launch_w<true, true, false, JBMAX>(P, grid, st);
        case 2: return launch_w<true, false, false, JBMAX>(P, grid, st);
        case 1: return launch_w<false, true, false, JBMAX>(P, grid, st);
        default: return launch_w<false, false, false, JBMAX>(P, grid, st);
    }
}

cudaError_t launch_walk_tables(const TravParams& P, int grid, cudaStream_t st)
{
    return P.jbmax <= 4 ? launch_tab<4>(P, grid, st) : launch_tab<7>(P, grid, st);
}

}  // namespace bnr
