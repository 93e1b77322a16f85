// Instantiation unit: window 7x7, ACWDDF (_engine.py:451-487), general Minkowski order p.
#include "dfg_fast.cuh"
DFG_DEFINE_LAUNCH_PAIRED_PC(7, dfg::FAM_ACWDDF, acwddf, pgen, dfg::PC_GEN)
