// Instantiation unit: window 7x7, DDF (_engine.py:435-448), Minkowski order p = 1.
#include "dfg_fast.cuh"
DFG_DEFINE_LAUNCH_PAIRED_PC(7, dfg::FAM_DDF, ddf, p1, dfg::PC_1)
