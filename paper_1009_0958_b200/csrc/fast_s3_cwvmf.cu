// Instantiation unit: window 3x3, CWVMF (centre-weighted VMF applied to every window, filters.py:331-337).
#include "dfg_w3.cuh"
DFG_DEFINE_LAUNCH_CWVMF(3)
