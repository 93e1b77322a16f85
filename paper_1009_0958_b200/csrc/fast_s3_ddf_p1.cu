// Instantiation unit: window 3x3, DDF (_engine.py:435-448), Minkowski order p = 1.
#include "dfg_w3.cuh"
DFG_DEFINE_LAUNCH_PAIRED_PC(3, dfg::FAM_DDF, ddf, p1, dfg::PC_1)
