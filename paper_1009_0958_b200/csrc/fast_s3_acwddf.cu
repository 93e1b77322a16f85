// Instantiation unit: window 3x3, ACWDDF (_engine.py:451-487), Minkowski order p = 2, and the family launcher.
#include "dfg_w3.cuh"
DFG_DEFINE_LAUNCH_PAIRED_PC(3, dfg::FAM_ACWDDF, acwddf, p2, dfg::PC_2)
DFG_DEFINE_LAUNCH_PAIRED_DISPATCH(3, acwddf)
