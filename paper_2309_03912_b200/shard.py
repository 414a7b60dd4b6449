"""Multi-GPU sharding.

Configs C2/C5 (many files):

Units never resolve symbols across files (sema.py:152-218 works on one unit),
so a corpus shards across ranks with no data-path collective: each rank takes
a contiguous, byte-balanced range of the path-sorted corpus, analyses it on
its own GPU, and the ordered per-file results are gathered to rank 0 in rank
order -- which is path order, the order ``Diagnostic.sort_key`` imposes
(diagnostics.py:73-74).  One process per GPU, ``torch.distributed`` for the
plumbing (NCCL on the GPU box, gloo in the CPU tests).

Config C4 (one huge unit): ``analyze_unit_sharded`` -- every rank runs the
front end on the unit, walks its share of each level's work items, and the
library exchanges the levels' new instances, the edge slots, launch seeds and
diagnostics through an all-gather this module supplies
(``torch.distributed.all_gather``; include/exspace_b200.h exs_set_collective).
"""
from __future__ import annotations

import bisect
from typing import Callable, Optional, Sequence


def shard_ranges(sizes: Sequence[int], world: int) -> list:
    """Contiguous ranges [lo, hi) of ``sizes`` with near-equal byte totals.

    Rank r gets the files whose byte prefix midpoints fall in
    [r * total / world, (r + 1) * total / world); every file lands on exactly
    one rank and ranks stay in input order.
    """
    if world < 1:
        raise ValueError("world must be >= 1")
    n = len(sizes)
    prefix = [0]
    for s in sizes:
        prefix.append(prefix[-1] + int(s))
    total = prefix[-1]
    if total == 0:
        # equal counts when there is nothing to balance
        return [(n * r // world, n * (r + 1) // world) for r in range(world)]
    mids = [(prefix[i] + prefix[i + 1]) / 2.0 for i in range(n)]
    bounds = [bisect.bisect_left(mids, total * r / world) for r in range(world)] + [n]
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def my_shard(units: Sequence, rank: int, world: int, size_of: Callable = None) -> tuple:
    size_of = size_of or (lambda u: len(u[1].encode("utf-8", "surrogateescape")))
    lo, hi = shard_ranges([size_of(u) for u in units], world)[rank]
    return lo, hi


def merge_results(parts: Sequence) -> tuple:
    """Concatenate per-shard columnar results (recs, text, unit_first) in
    shard order: unit indices and message offsets move past the earlier
    shards' (exs_result layout, include/exspace_b200.h)."""
    import numpy as np
    from ._native import RESULT_DTYPE
    recs, texts, firsts = [], [], [np.zeros(1, dtype=np.uint64)]
    units = 0
    tbase = 0
    rbase = 0
    for r, t, f in parts:
        r = np.array(r, dtype=RESULT_DTYPE, copy=True)
        r["unit"] += units
        r["msg_off"] += tbase
        recs.append(r)
        texts.append(np.asarray(t, dtype=np.uint8))
        firsts.append(np.asarray(f[1:], dtype=np.uint64) + rbase)
        units += len(f) - 1
        tbase += len(t)
        rbase += len(r)
    return (np.concatenate(recs) if recs else np.zeros(0, dtype=RESULT_DTYPE),
            np.concatenate(texts) if texts else np.zeros(0, dtype=np.uint8),
            np.concatenate(firsts))


def gather_results(recs, text, unit_first, rank: int, world: int, device=None, group=None):
    """Gather every rank's columnar results to rank 0 in rank order (None on
    other ranks) with point-to-point collectives: an all-gather of the three
    sizes, then one variable-size send/recv per rank of each byte buffer.
    ``device``: where the byte tensors live (a CUDA device for NCCL, None for
    CPU / gloo)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from ._native import RESULT_DTYPE
    if world == 1:
        return recs, text, unit_first
    dev = torch.device(device) if device is not None else torch.device("cpu")
    bufs = [np.ascontiguousarray(recs).view(np.uint8).reshape(-1),
            np.ascontiguousarray(text, dtype=np.uint8).reshape(-1),
            np.ascontiguousarray(unit_first, dtype=np.uint64).view(np.uint8).reshape(-1)]
    sizes = torch.tensor([b.size for b in bufs], dtype=torch.int64, device=dev)
    allsz = [torch.zeros_like(sizes) for _ in range(world)]
    dist.all_gather(allsz, sizes, group=group)
    allsz = [x.tolist() for x in allsz]
    if rank != 0:
        for b in bufs:
            if b.size:
                dist.send(torch.from_numpy(b).to(dev), dst=0, group=group)
        return None
    parts = [tuple(bufs)]
    for src in range(1, world):
        got = []
        for k in range(3):
            t = torch.empty(allsz[src][k], dtype=torch.uint8, device=dev)
            if allsz[src][k]:
                dist.recv(t, src=src, group=group)
            got.append(t.cpu().numpy())
        parts.append(tuple(got))
    return merge_results([(p[0].view(RESULT_DTYPE), p[1], p[2].view(np.uint64)) for p in parts])


def analyze_sharded(units: Sequence, rank: int, world: int, analyze_batch: Optional[Callable] = None,
                    device: Optional[int] = None, comm_device=None):
    """Analyse this rank's shard and gather the results to rank 0.

    ``units`` are (path, text[, profile, mode, cfg]) sorted by path.
    ``analyze_batch(shard) -> (recs, text, unit_first)`` defaults to the GPU
    engine on ``device``.  Returns, on rank 0, one Analysis per unit of the
    whole corpus in input order (None on other ranks)."""
    from . import exspace as X
    lo, hi = my_shard(units, rank, world)
    shard = list(units[lo:hi])
    if analyze_batch is None:
        dev = rank if device is None else device
        eng = X.get_engine(dev)
        X.analyze_corpus(shard, device=dev, engine=eng)
        local = eng.handle.results(copy=True)
    else:
        local = analyze_batch(shard)
    merged = gather_results(*local, rank, world, device=comm_device)
    if merged is None:
        return None
    res = X.CorpusResults(*merged, [u[0] for u in units])
    out = []
    for f, u in enumerate(units):
        prof = u[2] if len(u) > 2 else X.CompileProfile()
        mode = u[3] if len(u) > 3 else X.Mode.CLASSIC
        out.append(X.Analysis(u[0], prof, mode, res, f))
    return out


class _CudaBytes:
    """A raw device pointer as a uint8 CUDA array (torch.as_tensor reads it)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "|u1", "data": (ptr, False), "version": 2}


def make_allgather(device=None, group=None, stage_host=False):
    """An exs_allgather_fn over torch.distributed: variable-size byte buffers,
    padded to the largest, all-gathered, then packed in rank order.  device
    None: the buffers are host memory (gloo; the EMU build in the CPU tests);
    else CUDA memory on that device (NCCL), or, with stage_host, CUDA memory
    exchanged through host copies over a CPU backend (gloo: the functional GPU
    test that runs two ranks on one device)."""
    import ctypes as C
    import numpy as np
    from ._native import ALLGATHER_FN

    def fn(ctx, send, nbytes, recv, sizes):
        try:
            import torch
            import torch.distributed as dist
            world = dist.get_world_size(group)
            szs = [int(sizes[r]) for r in range(world)]
            mx = max(szs + [1])
            if device is None:
                t = torch.zeros(mx, dtype=torch.uint8)
                if nbytes:
                    t[:nbytes] = torch.from_numpy(np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(send)).copy())
                outs = [torch.empty(mx, dtype=torch.uint8) for _ in range(world)]
                dist.all_gather(outs, t, group=group)
                if sum(szs):
                    dst = np.ctypeslib.as_array((C.c_uint8 * sum(szs)).from_address(recv))
                    off = 0
                    for r in range(world):
                        dst[off:off + szs[r]] = outs[r][:szs[r]].numpy()
                        off += szs[r]
            elif stage_host:
                dev = torch.device(device)
                t = torch.zeros(mx, dtype=torch.uint8)
                if nbytes:
                    t[:nbytes] = torch.as_tensor(_CudaBytes(send, nbytes), device=dev).cpu()
                outs = [torch.empty(mx, dtype=torch.uint8) for _ in range(world)]
                dist.all_gather(outs, t, group=group)
                if sum(szs):
                    cat = torch.cat([outs[r][:szs[r]] for r in range(world)])
                    torch.as_tensor(_CudaBytes(recv, sum(szs)), device=dev).copy_(cat.to(dev))
                torch.cuda.synchronize(dev)
            else:
                dev = torch.device(device)
                t = torch.zeros(mx, dtype=torch.uint8, device=dev)
                if nbytes:
                    t[:nbytes].copy_(torch.as_tensor(_CudaBytes(send, nbytes), device=dev))
                outs = [torch.empty(mx, dtype=torch.uint8, device=dev) for _ in range(world)]
                dist.all_gather(outs, t, group=group)
                if sum(szs):
                    dst = torch.as_tensor(_CudaBytes(recv, sum(szs)), device=dev)
                    off = 0
                    for r in range(world):
                        dst[off:off + szs[r]].copy_(outs[r][:szs[r]])
                        off += szs[r]
                torch.cuda.synchronize(dev)
            return 0
        except Exception:  # the library reports a failed collective
            import traceback
            traceback.print_exc()
            return 1

    return ALLGATHER_FN(fn)


def analyze_unit_sharded(text: str, path: str, rank: int, world: int, profile=None, mode=None, cfg=None,
                         engine=None, device=None, want_walks: bool = False, stage_host: bool = False):
    """One unit analysed by `world` ranks together (the walk split across
    them); every rank returns the same Analysis.  device: CUDA device of the
    collective's buffers (None for host memory: gloo with the EMU build);
    stage_host: exchange CUDA buffers through host copies (make_allgather)."""
    from . import exspace as X
    eng = engine or X.get_engine(rank if device is None else device)
    eng.handle.set_collective(rank, world, make_allgather(device, stage_host=stage_host))
    try:
        unit = (text, path, profile or X.CompileProfile(), mode or X.Mode.CLASSIC, cfg or X.TraitConfig())
        return eng.run_batch([unit], want_walks=want_walks)[0]
    finally:
        eng.handle.set_collective(0, 1, None)

