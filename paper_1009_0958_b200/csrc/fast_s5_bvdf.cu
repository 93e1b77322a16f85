// Instantiation unit: window 5x5, BVDF (_engine.py:421-432).
#include "dfg_fast.cuh"
DFG_DEFINE_LAUNCH_BVDF(5)
