// Instantiation unit: window 3x3, ACWDDF (_engine.py:451-487).
#include "dfg_w3.cuh"
DFG_DEFINE_LAUNCH_PAIRED(3, dfg::FAM_ACWDDF, acwddf)
