"""CPU: bench.py's multi-GPU work split -- C5a row strips with their halo
rows (strong scaling) and the C5b frame split -- partitions the work exactly
once per pixel at 1/2/4/8 ranks, and strips filtered independently (oracle,
global border policy) reproduce the whole-frame result bit for bit.  Config
shapes are shrunk so the check runs in seconds; the split logic is the one
the GPU bench uses."""

import numpy as np
import pytest

import bench
import oracle
from paper_1009_0958_b200 import parse_filter_spec, synth


@pytest.fixture
def small_configs(monkeypatch):
    cfgs = {k: dict(v) for k, v in synth.CONFIGS.items()}
    cfgs["c5a"]["shape"] = (83, 29)
    cfgs["c5b"]["shape"] = (12, 17)
    cfgs["c5b"]["frames"] = 8
    monkeypatch.setattr(synth, "CONFIGS", cfgs)
    img = synth.noisy_image(83, 29, cfgs["c5a"]["seed"], cfgs["c5a"]["noise"])
    monkeypatch.setattr(synth, "config_input", lambda name, frames=None: img)
    return cfgs, img


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_c5a_strips_partition_and_match(small_configs, world):
    cfgs, img = small_configs
    spec = parse_filter_spec(cfgs["c5a"]["spec"])
    H = img.shape[0]
    want = oracle.filter_image(img, spec, threads=1)
    covered = np.zeros(H, int)
    total = 0
    for rank in range(world):
        wl = bench.workload("c5a", rank, world)
        if world == 1:
            assert wl["kind"] == "image" and wl["x"] is img
            covered += 1
            total += wl["px"]
            continue
        r0, n, i0 = wl["out_row0"], wl["out_rows"], wl["in_row0"]
        assert wl["kind"] == "rows" and wl["scaling"] == "strong" and wl["total_px"] == img.shape[0] * img.shape[1]
        assert (wl["x"] == img[i0:i0 + wl["x"].shape[0]]).all()
        assert i0 == max(0, r0 - 3) and i0 + wl["x"].shape[0] == min(H, r0 + n + 3)  # 7x7: 3-row halo
        covered[r0:r0 + n] += 1
        total += wl["px"]
        full = np.zeros_like(img)
        full[i0:i0 + wl["x"].shape[0]] = wl["x"]  # global row index, only the strip + halo present
        got = oracle.filter_image(full, spec, threads=1, rows=(r0, r0 + n))[r0:r0 + n]
        assert (got == want[r0:r0 + n]).all(), (world, rank)
    assert (covered == 1).all() and total == img.shape[0] * img.shape[1]


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_c5b_frame_split(small_configs, world):
    cfgs, _ = small_configs
    c = cfgs["c5b"]
    seen = []
    for rank in range(world):
        wl = bench.workload("c5b", rank, world)
        assert wl["kind"] == "batch" and wl["total_px"] == c["frames"] * 12 * 17
        per = -(-c["frames"] // world)
        for j, fr in enumerate(wl["x"]):
            f = rank * per + j
            assert (fr == synth.noisy_image(12, 17, c["seed"] + f, c["noise"])).all()
            seen.append(f)
    assert sorted(seen) == list(range(c["frames"]))
