// Instantiation unit: window 5x5, ACWDDF (_engine.py:451-487), Minkowski order p = 1.
#include "dfg_fast.cuh"
DFG_DEFINE_LAUNCH_PAIRED_PC(5, dfg::FAM_ACWDDF, acwddf, p1, dfg::PC_1)
