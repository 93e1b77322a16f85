// dfg_fixup.cu -- host-callable probe of the double-double arccos used by the
// float64 re-decision stage (dfg_f64.cuh), for CPU verification against a
// high-precision reference and against glibc (tests/test_abi.py).
#include <math.h>

#include "dfg_f64.cuh"

extern "C" DFG_API double dfg_cr_acos_host(double z, int32_t perturb_ulps)
{
    double y0 = acos(z);
    for (int k = 0; k < (perturb_ulps > 0 ? perturb_ulps : -perturb_ulps); k++)
        y0 = nextafter(y0, perturb_ulps > 0 ? 10.0 : -10.0);
    return dfg::cr_acos_from(z, y0);
}
