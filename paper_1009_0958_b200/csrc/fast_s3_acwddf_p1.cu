// Instantiation unit: window 3x3, ACWDDF (_engine.py:451-487), Minkowski order p = 1.
#include "dfg_w3.cuh"
DFG_DEFINE_LAUNCH_PAIRED_PC(3, dfg::FAM_ACWDDF, acwddf, p1, dfg::PC_1)
