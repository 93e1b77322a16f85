// Instantiation unit: window 5x5, DDF (_engine.py:435-448).
#include "dfg_fast.cuh"
DFG_DEFINE_LAUNCH_PAIRED(5, dfg::FAM_DDF, ddf)
