// Instantiation unit: window 7x7, ACWDDF (_engine.py:451-487).
#include "dfg_fast.cuh"
DFG_DEFINE_LAUNCH_PAIRED(7, dfg::FAM_ACWDDF, acwddf)
