// Instantiation unit: window 7x7, CWVMF (centre-weighted VMF applied to every window, filters.py:331-337).
#include "dfg_fast.cuh"
DFG_DEFINE_LAUNCH_CWVMF(7)
