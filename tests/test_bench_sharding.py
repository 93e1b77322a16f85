"""CPU: bench.py's work split and its command-line contract.

* C5a at N > 1 is row-strip sharded through parallel.StripJob (the halo
  exchange + chunked gather that tests/test_parallel.py runs multi-rank
  with gloo); here: the workload kinds, scaling and pixel totals at 1/2/4/8
  ranks, and that the strips StripJob cuts partition the frame.
* C5b frames are split across ranks exactly once, each with its seed.
* Both arms print the same ``config`` dict.
* ``--gpus N`` outside torchrun re-launches the script under
  torch.distributed.run with N ranks (exercised with the CPU reference arm:
  rank 0 prints exactly one JSON line with n_gpus = N)."""

import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import bench
from paper_1009_0958_b200 import synth
from paper_1009_0958_b200.parallel import strip_rows

ROOT = Path(__file__).resolve().parent.parent


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
def test_c5a_strips(small_configs, world):
    cfgs, img = small_configs
    H, W = img.shape[:2]
    covered = np.zeros(H, int)
    for rank in range(world):
        wl = bench.workload("c5a", rank, world)
        assert wl["total_px"] == H * W
        if world == 1:
            assert wl["kind"] == "image" and wl["x"] is img and wl["scaling"] == "weak"
            covered += 1
            continue
        assert wl["kind"] == "strips" and wl["scaling"] == "strong" and wl["x"] is img
        r0, r1, i0, i1 = strip_rows(H, world, rank, 7)
        assert i0 == max(0, r0 - 3) and i1 == min(H, r1 + 3)  # 7x7: 3-row halo
        covered[r0:r1] += 1
    assert (covered == 1).all()


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


def test_default_workload_is_c5a():
    assert bench.DEFAULT_CONFIG == "c5a"
    d = bench.config_dict("c5a", 1)
    assert d["workload"] == "c5a" and d["shape"] == [8192, 8192] and d["spec"] == "ddf:exact:window=7"


def test_gpus_flag_relaunches_under_torchrun():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--impl", "reference",
                        "--config", "c1", "--steps", "1", "--warmup", "3"],
                       capture_output=True, text=True, timeout=600, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["config"] == bench.config_dict("c1", 2)
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] in ("reference", "port")
