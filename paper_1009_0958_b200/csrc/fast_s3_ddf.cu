// Instantiation unit: window 3x3, DDF (_engine.py:435-448).
#include "dfg_w3.cuh"
DFG_DEFINE_LAUNCH_PAIRED(3, dfg::FAM_DDF, ddf)
