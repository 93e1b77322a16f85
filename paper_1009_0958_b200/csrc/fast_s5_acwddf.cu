// Instantiation unit: window 5x5, ACWDDF (_engine.py:451-487).
#include "dfg_fast.cuh"
DFG_DEFINE_LAUNCH_PAIRED(5, dfg::FAM_ACWDDF, acwddf)
