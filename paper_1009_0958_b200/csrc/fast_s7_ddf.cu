// Instantiation unit: window 7x7, DDF (_engine.py:435-448), Minkowski order p = 2, and the family launcher.
#include "dfg_fast.cuh"
DFG_DEFINE_LAUNCH_PAIRED_PC(7, dfg::FAM_DDF, ddf, p2, dfg::PC_2)
DFG_DEFINE_LAUNCH_PAIRED_DISPATCH(7, ddf)
