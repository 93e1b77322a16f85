// Instantiation unit: window 5x5, DDF (_engine.py:435-448), Minkowski order p = 1.
#include "dfg_fast.cuh"
DFG_DEFINE_LAUNCH_PAIRED_PC(5, dfg::FAM_DDF, ddf, p1, dfg::PC_1)
