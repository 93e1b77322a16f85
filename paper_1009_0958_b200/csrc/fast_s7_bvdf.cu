// Instantiation unit: window 7x7, BVDF (_engine.py:421-432).
#include "dfg_fast.cuh"
DFG_DEFINE_LAUNCH_BVDF(7)
