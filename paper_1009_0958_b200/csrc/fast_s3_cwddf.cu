// Instantiation unit: window 3x3, CWDDF (centre-weighted DDF applied to every window, filters.py:296-328), Minkowski order p = 2, and the family launcher.
#include "dfg_w3.cuh"
DFG_DEFINE_LAUNCH_PAIRED_PC(3, dfg::FAM_CWDDF, cwddf, p2, dfg::PC_2)
DFG_DEFINE_LAUNCH_PAIRED_DISPATCH(3, cwddf)
