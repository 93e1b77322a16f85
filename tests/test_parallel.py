"""CPU (gloo, world sizes 2-8): the multi-GPU strip sharding host logic --
strip bounds, neighbour halo exchange, chunked gather to the root (the
exact code bench.py times on GPUs, parallel.StripJob) -- reproduces the
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
from paper_1009_0958_b200.parallel import StripJob, frame_split, strip_rows


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_filter(spec, border):
    """filter_fn for StripJob: the oracle on a strip, rebuilt into the global
    row index so the border policy applies at the true image edges (what
    dfg_filter_rows does)."""
    def fn(strip, H, i0, r0, rows, out):
        full = np.zeros((H,) + tuple(strip.shape[1:]), dtype=np.uint8)
        full[i0:i0 + strip.shape[0]] = strip.numpy()
        res = oracle.filter_image(full, spec, border, threads=1, rows=(r0, r0 + rows))
        out.copy_(torch.from_numpy(res[r0:r0 + rows].astype(np.uint8)))
    return fn


def _worker(rank, world, port, spec_text, border, H, W, gather, chunks, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        spec = parse_filter_spec(spec_text)
        img = synth.noisy_image(H, W, 9, ("correlated", 0.2))
        try:
            job = StripJob(H, W, spec.window, border=border, gather=gather, chunks=chunks)
        except ValueError as e:  # every rank raises alike (no rank left waiting)
            q.put((rank, "ValueError", str(e)))
            return
        job.own.copy_(torch.from_numpy(img[job.r0:job.r1]))
        out = job.run(_oracle_filter(spec, border))
        q.put((rank, (job.r0, job.r1), out.numpy().copy()))
    finally:
        dist.destroy_process_group()


def _run(world, spec_text, border, H, W, gather=True, chunks=3):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, spec_text, border, H, W, gather, chunks, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, a, b = q.get(timeout=180)
        res[rank] = (a, b)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world,spec_text,border,H,W", [
    (2, "ddf:exact:window=7", "replicate", 37, 29), (2, "acwddf:rgb:window=5", "reflect", 37, 29),
    (3, "bvdf:minimax", "replicate", 40, 23), (4, "ddf:exact", "replicate", 2, 11),  # ranks 2, 3 own no rows
    (4, "ddf:exact:window=7", "replicate", 13, 9)])
def test_strips_gather_to_root_equal_single_process(world, spec_text, border, H, W):
    """Halo exchange into the strip buffers, chunked filtering and the
    chunk-by-chunk gather to rank 0 reproduce the single-process frame --
    including ranks that own no rows (they neither send nor receive)."""
    res = _run(world, spec_text, border, H, W, gather=True, chunks=3)
    img = synth.noisy_image(H, W, 9, ("correlated", 0.2))
    want = oracle.filter_image(img, parse_filter_spec(spec_text), border, threads=2)
    assert (res[0][1] == want).all()


def test_strips_resident_output():
    """Without the gather every rank keeps exactly its own filtered rows."""
    H, W, spec_text = 41, 17, "acwddf:exact"
    res = _run(3, spec_text, "replicate", H, W, gather=False)
    img = synth.noisy_image(H, W, 9, ("correlated", 0.2))
    want = oracle.filter_image(img, parse_filter_spec(spec_text), "replicate", threads=2)
    for rank, ((r0, r1), out) in res.items():
        assert (out == want[r0:r1]).all(), rank


def test_too_many_ranks_raise_everywhere():
    """Strips thinner than the halo cannot be served by neighbours alone:
    every rank raises ValueError instead of waiting on a peer."""
    res = _run(8, "ddf:exact:window=7", "replicate", 9, 5)
    assert all(a == "ValueError" for a, _ in res.values())


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
