// Instantiation unit: window 3x3, CWDDF (centre-weighted DDF applied to every window, filters.py:296-328), general Minkowski order p.
#include "dfg_w3.cuh"
DFG_DEFINE_LAUNCH_PAIRED_PC(3, dfg::FAM_CWDDF, cwddf, pgen, dfg::PC_GEN)
