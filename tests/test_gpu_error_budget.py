"""GPU: the FP32 aggregates of the decision kernel stay inside the error
budget the kernel uses to decide which pixels need the float64 re-decision
(dfg_api.cu error_budget).  If this fails, a flagged-pixel criterion could
miss a decision flip, so it guards the exactness argument of DESIGN.md."""

import ctypes

import numpy as np
import pytest

import oracle
from paper_1009_0958_b200 import _lib, parse_filter_spec, synth

pytestmark = pytest.mark.gpu


def budget(spec):
    n = spec.window ** 2
    kind = spec.strategy.kind if spec.family != "vmf" else "exact"
    p = spec.acwddf.p if spec.family == "acwddf" else spec.p
    er_pair, ea_pair = 8e-7, 1e-10
    if kind == "minimax":
        er_pair, ea_pair = 1.2e-6, 8e-8
    if kind == "chromaticity":
        er_pair, ea_pair = 8e-7, 1e-9
    if p not in (1.0, 2.0):
        er_pair += 4e-6 * p
    return 1.25 * (er_pair + (n - 1) * 6e-8), 1.25 * n * ea_pair


@pytest.mark.parametrize("spec", ["bvdf:exact", "bvdf:minimax", "bvdf:minimax:q=3", "bvdf:rgb", "ddf:exact:window=5",
                                  "ddf:minimax:window=7", "ddf:rgb:window=5", "vmf:p=3", "ddf:exact:p=1:window=7",
                                  "bvdf:rgb:p=3"])
def test_fp32_aggregates_within_budget(cuda, spec):
    torch = cuda
    s = parse_filter_spec(spec)
    n = s.window ** 2
    rng = np.random.default_rng(5)
    imgs = [synth.noisy_image(40, 64, 31, ("uncorrelated", 0.1)), rng.integers(0, 256, (40, 64, 3)).astype(np.uint8),
            np.clip(synth.clean_image(40, 64, 8).astype(int) + rng.integers(-2, 3, (40, 64, 3)), 0, 255).astype(np.uint8)]
    er, ea = budget(s)
    worst_a = worst_l = 0.0
    for img in imgs:
        want = oracle.aggregates(img, s)
        x = torch.from_numpy(img).cuda()
        vals = torch.empty((40, 64, 2, n), dtype=torch.float32, device="cuda")
        prm = _lib.params_from_spec(s, "replicate")
        _lib.check(_lib.lib().dfg_debug_values(ctypes.c_void_p(x.data_ptr()), 40, 64, 192,
                                               ctypes.c_void_p(vals.data_ptr()), ctypes.byref(prm), None))
        got = vals.cpu().numpy().astype(np.float64)
        if s.family != "vmf":
            A, A64 = got[:, :, 0], want[:, :, 0]
            worst_a = max(worst_a, float((np.abs(A - A64) / (er * np.abs(A64) + ea)).max()))
        if s.family in ("vmf", "ddf", "acwddf"):
            L, L64 = got[:, :, 1], want[:, :, 1]
            worst_l = max(worst_l, float((np.abs(L - L64) / (er * np.abs(L64) + 1e-30)).max()))
    print(f"{spec}: worst angular error / budget = {worst_a:.3f}, Minkowski = {worst_l:.3f}")
    assert worst_a < 0.5 and worst_l < 0.5
