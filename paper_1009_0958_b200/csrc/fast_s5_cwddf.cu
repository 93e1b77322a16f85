// Instantiation unit: window 5x5, CWDDF (centre-weighted DDF applied to every window, filters.py:296-328), Minkowski order p = 2, and the family launcher.
#include "dfg_fast.cuh"
DFG_DEFINE_LAUNCH_PAIRED_PC(5, dfg::FAM_CWDDF, cwddf, p2, dfg::PC_2)
DFG_DEFINE_LAUNCH_PAIRED_DISPATCH(5, cwddf)
