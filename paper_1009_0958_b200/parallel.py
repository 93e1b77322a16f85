"""Multi-GPU partitioning of the directional-filter path (one process per GPU).

Reference analogue: ``apply_filter(..., workers=k)`` splits the output rows
into contiguous bands (filters.py:416-430), every band reading the shared
padded image; results are bit-identical to the sequential run
(T/test_filters.py:434-439).  Here each rank owns one band ("strip") of a
frame that is resident on the GPUs as strips:

* ``strip_rows``  -- output rows [r0, r1) of a rank and the input rows
  [i0, i1) its windows need (halo of s//2 rows, clipped at the image edges,
  where the global border policy applies instead: dfg_filter_rows resolves
  border rows against the global height).
* ``StripJob`` -- the per-rank buffers of one sharded frame and its step:
  halo exchange with the neighbours (point-to-point send/recv straight into
  the strip buffer's halo rows: NCCL over NVLink on GPUs, gloo in the CPU
  tests), the strip filter in row chunks, and -- optionally -- the gather of
  the filtered rows to a root rank, each chunk sent as soon as its kernel is
  enqueued so the transfer overlaps the next chunk's filtering.  The halo
  exchange and the gather are the only data-path collectives.
* ``frame_split`` -- batch workloads (C5b) split whole frames, no halo.

The per-chunk filter call is injected (``filter_fn``) so the multi-rank host
logic runs on CPU with gloo in the tests; on GPUs it is the CUDA
``filter_rows_device``.
"""

from __future__ import annotations

import math


def strip_rows(H: int, world: int, rank: int, window: int, border: str = "replicate"):
    """Rows of rank ``rank``: output [r0, r1), input [i0, i1) incl. halo.
    Ranks past the last row own nothing: (H, H, H, H)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    h = window // 2
    per = math.ceil(H / world)
    r0, r1 = min(H, rank * per), min(H, (rank + 1) * per)
    if r1 <= r0:
        return r0, r0, r0, r0
    if border == "replicate" or (H > 2 * h and r1 - r0 >= h):
        # replicate clamps; reflect mirrors rows -h..-1 onto 0..h-1, which an
        # edge strip of >= h rows already holds
        i0, i1 = max(0, r0 - h), min(H, r1 + h)
    else:
        i0, i1 = 0, H  # tiny images: mirrored indices can land anywhere
    return r0, r1, i0, i1


def frame_split(B: int, world: int, rank: int):
    """Frames [f0, f1) of rank ``rank`` for a batch of B frames."""
    per = math.ceil(B / world)
    return min(B, rank * per), min(B, (rank + 1) * per)


def check_exchangeable(H: int, world: int, window: int, border: str = "replicate") -> None:
    """The neighbour exchange moves halo rows between adjacent ranks only,
    so every strip followed by another non-empty strip must hold at least
    s//2 rows, and reflect strips must be the replicate-like kind (no
    whole-image fallback).  Raises ValueError (on every rank alike)."""
    h = window // 2
    for r in range(world):
        r0, r1, i0, i1 = strip_rows(H, world, r, window, border)
        if r1 <= r0:
            continue
        if r1 < H and r1 - r0 < h:
            raise ValueError(f"strip of rank {r} holds {r1 - r0} rows < window//2 = {h}: too many ranks for H={H}")
        if (i0, i1) != (max(0, r0 - h), min(H, r1 + h)):
            raise ValueError("reflect border on a frame too small to shard with a neighbour halo")


def _halo_ops(dist, strip, r0, r1, i0, i1, H, world, rank, window, group):
    """Point-to-point ops of the halo exchange, receiving straight into the
    strip buffer (rows [i0, i1); own rows already at [r0 - i0, r1 - i0))."""
    if r1 <= r0:  # an empty rank neither sends nor receives
        return []
    h = window // 2
    ops = []
    own = strip[r0 - i0:r1 - i0]
    n = r1 - r0
    below_owns = rank + 1 < world and strip_rows(H, world, rank + 1, window)[1] > strip_rows(H, world, rank + 1,
                                                                                              window)[0]
    if rank > 0:  # my first h rows are the halo below rank - 1; its last rows are my top halo
        ops.append(dist.P2POp(dist.isend, own[:min(h, n)], rank - 1, group))
        if r0 - i0 > 0:
            ops.append(dist.P2POp(dist.irecv, strip[:r0 - i0], rank - 1, group))
    if below_owns:
        ops.append(dist.P2POp(dist.isend, own[n - min(h, n):], rank + 1, group))
        if i1 - r1 > 0:
            ops.append(dist.P2POp(dist.irecv, strip[r1 - i0:], rank + 1, group))
    return ops


def halo_exchange_into(strip, r0: int, r1: int, i0: int, i1: int, H: int, window: int, group=None):
    """Fill the halo rows of this rank's strip buffer from its neighbours.
    Collective over the group (every rank calls it, empty ranks included)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    ops = _halo_ops(dist, strip, r0, r1, i0, i1, H, world, rank, window, group)
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return strip


def halo_exchange(own, r0: int, r1: int, H: int, window: int, group=None):
    """Given this rank's own rows ``own`` ((r1-r0, W, 3)), return
    (strip, i0): a new buffer holding rows [i0, i1) incl. the neighbours'
    halo rows.  Collective over the group."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    check_exchangeable(H, world, window)
    _, _, i0, i1 = strip_rows(H, world, rank, window)
    strip = torch.empty((max(0, i1 - i0),) + tuple(own.shape[1:]), dtype=own.dtype, device=own.device)
    if r1 > r0:
        strip[r0 - i0:r1 - i0] = own
    halo_exchange_into(strip, r0, r1, i0, i1, H, window, group)
    return strip, i0


class StripJob:
    """One rank's share of a row-strip sharded (H, W, 3) frame.

    ``strip`` holds input rows [i0, i1); the caller writes its own rows
    [r0, r1) into ``own`` (the frame arrives sharded).  ``run(filter_fn)`` is
    the multi-GPU step: halo exchange, then the strip's output rows in
    ``chunks`` row chunks -- ``filter_fn(strip, H, i0, out_row0, rows, out)``
    writes output rows [out_row0, out_row0 + rows) into ``out`` -- and, with
    ``gather``, every chunk is sent to ``root`` right after its filter is
    enqueued, the root receiving all ranks' chunk c in one group call into
    its full-frame ``out`` (overlapping the transfer with the next chunk).
    Without ``gather`` the filtered rows stay resident on their rank
    (``out`` then holds rows [r0, r1))."""

    def __init__(self, H: int, W: int, window: int, group=None, border: str = "replicate", root: int = 0,
                 gather: bool = True, chunks: int = 4, device=None):
        import torch
        import torch.distributed as dist

        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        check_exchangeable(H, self.world, window, border)
        self.H, self.W, self.window, self.group = H, W, window, group
        self.root, self.gather = root, gather
        self.r0, self.r1, self.i0, self.i1 = strip_rows(H, self.world, self.rank, window, border)
        self.strip = torch.zeros((max(0, self.i1 - self.i0), W, 3), dtype=torch.uint8, device=device)
        self.own = self.strip[self.r0 - self.i0:self.r1 - self.i0]
        if gather and self.rank == root:
            self.out = torch.empty((H, W, 3), dtype=torch.uint8, device=device)
            self.my_out = self.out[self.r0:self.r1]
        else:
            self.out = torch.empty((self.r1 - self.r0, W, 3), dtype=torch.uint8, device=device)
            self.my_out = self.out
        # chunk boundaries (relative to each rank's r0); identical formula on
        # every rank so the root knows every sender's chunks
        self.chunks = max(1, chunks)

    def _chunk_bounds(self, rank: int):
        r0, r1, _, _ = strip_rows(self.H, self.world, rank, self.window)
        n = r1 - r0
        k = self.chunks if self.gather else 1
        cuts = [r0 + (n * c) // k for c in range(k + 1)]
        return [(a, b) for a, b in zip(cuts[:-1], cuts[1:])]

    def run(self, filter_fn):
        import torch.distributed as dist

        halo_exchange_into(self.strip, self.r0, self.r1, self.i0, self.i1, self.H, self.window, self.group)
        reqs = []
        send = self.gather and self.rank != self.root
        if self.gather and self.rank == self.root:
            # all chunk receives up front (they wait on the communication
            # stream, not on the root's own filtering)
            per_rank = {k: self._chunk_bounds(k) for k in range(self.world) if k != self.root}
            for c in range(self.chunks):
                ops = [dist.P2POp(dist.irecv, self.out[b[c][0]:b[c][1]], k, self.group)
                       for k, b in per_rank.items() if b[c][1] > b[c][0]]
                if ops:
                    reqs.extend(dist.batch_isend_irecv(ops))
        for a, b in self._chunk_bounds(self.rank):
            if b <= a:
                continue
            dst = self.my_out[a - self.r0:b - self.r0]
            filter_fn(self.strip, self.H, self.i0, a, b - a, dst)
            if send:
                reqs.extend(dist.batch_isend_irecv([dist.P2POp(dist.isend, dst, self.root, self.group)]))
        for r in reqs:
            r.wait()
        return self.out


def filter_strips(own, r0: int, r1: int, H: int, spec, policy, group=None, filter_fn=None, gather: bool = False,
                  chunks: int = 4):
    """Filter a frame sharded by rows across the group: halo exchange, local
    strip filter, optional gather of the whole frame to rank 0 (returned
    there; other ranks return their own filtered rows).  ``filter_fn(strip,
    H, i0, out_row0, rows, out)``; default the CUDA ``filter_rows_device``."""
    import torch.distributed as dist

    if filter_fn is None:
        from .filters import filter_rows_device

        def filter_fn(strip, H_, i0, a, n, out):
            filter_rows_device(strip, H_, i0, a, n, spec, policy, out=out)
    border = getattr(policy, "mode", policy)
    job = StripJob(H, int(own.shape[1]) if own.dim() == 3 else 0, int(spec.window), group, border,
                   gather=gather, chunks=chunks, device=own.device)
    if (job.r0, job.r1) != (r0, r1):
        raise ValueError(f"rank {dist.get_rank(group)} owns rows [{job.r0}, {job.r1}), got [{r0}, {r1})")
    job.own.copy_(own)
    return job.run(filter_fn)
