// Instantiation unit: window 3x3, BVDF (_engine.py:421-432).
#include "dfg_w3.cuh"
DFG_DEFINE_LAUNCH_BVDF(3)
