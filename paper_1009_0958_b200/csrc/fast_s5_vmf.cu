// Instantiation unit: window 5x5, VMF (vector median, _engine.py:409-418).
#include "dfg_fast.cuh"
DFG_DEFINE_LAUNCH_VMF(5)
