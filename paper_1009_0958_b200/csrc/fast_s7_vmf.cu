// Instantiation unit: window 7x7, VMF (vector median, _engine.py:409-418).
#include "dfg_fast.cuh"
DFG_DEFINE_LAUNCH_VMF(7)
