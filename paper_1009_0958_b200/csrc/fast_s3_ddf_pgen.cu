// Instantiation unit: window 3x3, DDF (_engine.py:435-448), general Minkowski order p.
#include "dfg_w3.cuh"
DFG_DEFINE_LAUNCH_PAIRED_PC(3, dfg::FAM_DDF, ddf, pgen, dfg::PC_GEN)
