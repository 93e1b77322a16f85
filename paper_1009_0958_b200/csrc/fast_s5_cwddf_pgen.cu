// Instantiation unit: window 5x5, CWDDF (centre-weighted DDF applied to every window, filters.py:296-328), general Minkowski order p.
#include "dfg_fast.cuh"
DFG_DEFINE_LAUNCH_PAIRED_PC(5, dfg::FAM_CWDDF, cwddf, pgen, dfg::PC_GEN)
