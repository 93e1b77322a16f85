"""Multi-GPU partitioning of the directional-filter path (one process per GPU).

Reference analogue: ``apply_filter(..., workers=k)`` splits the output rows
into contiguous bands (filters.py:416-430), every band reading the shared
padded image; results are bit-identical to the sequential run
(T/test_filters.py:434-439).  Here each rank owns one band ("strip"):

* ``strip_rows``  -- output rows [r0, r1) of a rank and the input rows
  [i0, i1) its window needs (halo of s//2 rows, clipped at the image edges
  where the global border policy applies instead -- dfg_filter_rows resolves
  border rows against the global height).
* ``halo_exchange`` -- when every rank holds only its own rows (e.g. the
  frame was produced sharded by an upstream stage), fetch the h rows above
  and below from the neighbours with point-to-point send/recv (NCCL over
  NVLink on GPUs, gloo in the CPU tests).  This is the only data-path
  collective, and only for pre-sharded frames; a frame staged from the host
  is cut with its halos and needs no exchange.
* ``gather_rows`` -- optional all-gather of the filtered strips (the
  "gather" of SURVEY 8(e)) for callers that need the whole frame on every
  rank; rank-local results need no collective.
* ``frame_split`` -- batch workloads (C5b) split whole frames, no halo.

The per-strip filter call is injected (``filter_fn``) so the multi-rank
host logic can be exercised on CPU with gloo; the default is the CUDA path.
"""

from __future__ import annotations

import math


def strip_rows(H: int, world: int, rank: int, window: int, border: str = "replicate"):
    """Rows of rank ``rank``: output [r0, r1), input [i0, i1) incl. halo."""
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


def halo_exchange(own, r0: int, r1: int, H: int, window: int, group=None):
    """Given this rank's own rows ``own`` (tensor (r1-r0, W, 3)) of a frame of
    H rows split by ``strip_rows``, return (strip, i0): the rows [i0, i1)
    including the neighbours' halo rows, using send/recv with the ranks
    above and below.  Collective over the group (every rank calls it)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    h = window // 2
    if math.ceil(H / world) < h:
        raise ValueError("strips must hold at least window//2 rows for a neighbour halo exchange")
    i0, i1 = max(0, r0 - h), min(H, r1 + h)
    top_n, bot_n = r0 - i0, i1 - r1
    ops, bufs = [], {}
    W = own.shape[1]
    # my first h rows go to the rank above, my last h rows to the rank below
    if rank > 0 and r1 > r0:
        n_up = min(h, r1 - r0)
        ops.append(dist.P2POp(dist.isend, own[:n_up].contiguous(), rank - 1, group))
    if rank < world - 1 and r1 > r0:
        n_dn = min(h, r1 - r0)
        ops.append(dist.P2POp(dist.isend, own[r1 - r0 - n_dn:].contiguous(), rank + 1, group))
    if top_n > 0:
        bufs["top"] = torch.empty((top_n, W, 3), dtype=own.dtype, device=own.device)
        ops.append(dist.P2POp(dist.irecv, bufs["top"], rank - 1, group))
    if bot_n > 0:
        bufs["bot"] = torch.empty((bot_n, W, 3), dtype=own.dtype, device=own.device)
        ops.append(dist.P2POp(dist.irecv, bufs["bot"], rank + 1, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    parts = [bufs["top"]] if "top" in bufs else []
    parts.append(own)
    if "bot" in bufs:
        parts.append(bufs["bot"])
    return torch.cat(parts, 0), i0


def gather_rows(strip_out, H: int, window: int, group=None):
    """All-gather the filtered strips into the full (H, W, 3) frame."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    per = math.ceil(H / world)
    W = strip_out.shape[1]
    padded = torch.zeros((per, W, 3), dtype=strip_out.dtype, device=strip_out.device)
    padded[: strip_out.shape[0]] = strip_out
    outs = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(outs, padded, group=group)
    full = torch.cat(outs, 0)
    return full[:H]


def filter_strips(own, r0: int, r1: int, H: int, spec, policy, group=None, filter_fn=None, gather: bool = False):
    """Filter a frame sharded by rows across the group: halo exchange, local
    strip filter (``filter_fn(strip, H, i0, r0, rows, spec, policy)``;
    default the CUDA ``filter_rows_device``), optional all-gather."""
    if filter_fn is None:
        from .filters import filter_rows_device

        filter_fn = filter_rows_device
    strip, i0 = halo_exchange(own, r0, r1, H, int(spec.window), group)
    out = filter_fn(strip, H, i0, r0, r1 - r0, spec, policy) if r1 > r0 else own[:0]
    if gather:
        return gather_rows(out, H, int(spec.window), group)
    return out
