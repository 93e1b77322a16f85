// Instantiation unit: window 7x7, DDF (_engine.py:435-448).
#include "dfg_fast.cuh"
DFG_DEFINE_LAUNCH_PAIRED(7, dfg::FAM_DDF, ddf)
