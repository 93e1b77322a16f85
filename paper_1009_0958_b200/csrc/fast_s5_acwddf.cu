// Instantiation unit: window 5x5, ACWDDF (_engine.py:451-487), Minkowski order p = 2, and the family launcher.
#include "dfg_fast.cuh"
DFG_DEFINE_LAUNCH_PAIRED_PC(5, dfg::FAM_ACWDDF, acwddf, p2, dfg::PC_2)
DFG_DEFINE_LAUNCH_PAIRED_DISPATCH(5, acwddf)
