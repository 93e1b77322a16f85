// Instantiation unit: window 3x3, VMF (vector median, _engine.py:409-418).
#include "dfg_w3.cuh"
DFG_DEFINE_LAUNCH_VMF(3)
