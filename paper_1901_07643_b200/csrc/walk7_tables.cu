// walk7_tables.cu -- walk7_kernel.cu instantiated for the separate RSS / BIC tables
// (bnreg_run, bnreg_all_rss, bnreg_bic), in its own translation unit (parallel build).
#define BNREG_WALK7_TABLES 1
#include "walk7_kernel.cu"
