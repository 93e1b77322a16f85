"""CPU (gloo, world size 2): the multi-GPU strip sharding host logic --
strip bounds, neighbour halo exchange, all-gather -- reproduces the
single-process result bit for bit (the reference's row-partition
equivalence, T/test_filters.py:434-439).  The per-strip filter is the float64
oracle here (test infrastructure); on GPUs it is filter_rows_device."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1009_0958_b200 import parse_filter_spec, synth
from paper_1009_0958_b200.parallel import filter_strips, frame_split, strip_rows


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_rows(strip, H, i0, r0, rows, spec, policy):
    """Oracle on a strip: rebuild the global index frame so the border
    policy applies at the true image edges (what dfg_filter_rows does)."""
    full = np.zeros((H,) + tuple(strip.shape[1:]), dtype=np.uint8)
    full[i0:i0 + strip.shape[0]] = strip.numpy()
    out = oracle.filter_image(full, spec, policy, threads=1, rows=(r0, r0 + rows))
    return torch.from_numpy(out[r0:r0 + rows].astype(np.uint8))


def _worker(rank, world, port, spec_text, border, H, W, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        spec = parse_filter_spec(spec_text)
        img = synth.noisy_image(H, W, 9, ("correlated", 0.2))
        r0, r1, _, _ = strip_rows(H, world, rank, spec.window, border)
        own = torch.from_numpy(img[r0:r1].copy())
        full = filter_strips(own, r0, r1, H, spec, border, filter_fn=_oracle_rows, gather=True)
        if rank == 0:
            q.put(full.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("spec_text,border", [("ddf:exact:window=7", "replicate"), ("acwddf:rgb:window=5", "reflect"),
                                              ("bvdf:minimax", "replicate")])
def test_two_rank_strips_equal_single_process(spec_text, border):
    H, W = 37, 29
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, spec_text, border, H, W, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    img = synth.noisy_image(H, W, 9, ("correlated", 0.2))
    want = oracle.filter_image(img, parse_filter_spec(spec_text), border, threads=2)
    assert (got == want).all()


def test_strip_bounds_cover_every_row():
    for H in (1, 7, 100, 8192):
        for world in (1, 2, 3, 4, 8):
            for s in (3, 5, 7):
                rows = []
                for r in range(world):
                    r0, r1, i0, i1 = strip_rows(H, world, r, s)
                    assert i0 <= r0 <= r1 <= i1 or r0 == r1
                    if r1 > r0:
                        assert r0 - i0 <= s // 2 and i1 - r1 <= s // 2
                    rows.extend(range(r0, r1))
                assert rows == list(range(H))


def test_frame_split_partitions_batch():
    for B in (1, 5, 64):
        for world in (1, 2, 4, 8):
            got = []
            for r in range(world):
                f0, f1 = frame_split(B, world, r)
                got.extend(range(f0, f1))
            assert got == list(range(B))
