// Instantiation unit: window 7x7, ACWDDF (_engine.py:451-487), Minkowski order p = 2, and the family launcher.
#include "dfg_fast.cuh"
DFG_DEFINE_LAUNCH_PAIRED_PC(7, dfg::FAM_ACWDDF, acwddf, p2, dfg::PC_2)
DFG_DEFINE_LAUNCH_PAIRED_DISPATCH(7, acwddf)
