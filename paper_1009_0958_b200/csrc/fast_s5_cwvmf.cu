// Instantiation unit: window 5x5, CWVMF (centre-weighted VMF applied to every window, filters.py:331-337).
#include "dfg_fast.cuh"
DFG_DEFINE_LAUNCH_CWVMF(5)
