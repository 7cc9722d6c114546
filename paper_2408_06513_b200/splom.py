"""Scatterplot-matrix (SPLOM) batches: many independent plots regularized at once
(BASELINE.json configs[3]: 256 plots x 500k points, 1024^2, 10 iterations).

Plots are independent (no cross-plot term anywhere in the reference's regularize.py:
40-80), so the batch is partitioned across ranks into contiguous blocks with no
data-path communication.  Inside a rank the block runs as ONE batched run
(inim_run_batched): every stage of every iteration is a single launch over all plots
with the plot index in grid.z, so the 1024^2 kernels of the whole block fill the GPU
together, captured once into a CUDA graph and replayed.  One collective at the end
gathers the final positions of every plot (NCCL all-gather over NVLink on GPUs; gloo
in the CPU tests).

The reference runs the same workload as a process pool over host cores
(tests/test_acceptance.py:107-128), one regularize.run per plot.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional, Sequence

import numpy as np


def shard(nplots: int, world: int, rank: int) -> range:
    """Contiguous block of plot indices owned by `rank` (sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(nplots, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def _chunk_bounds(nb: int, chunk: int, lead: int) -> list:
    """[b0, b1) plot ranges for run_host.  The copy in of the first chunk and the copy out
    of the last are the parts nothing overlaps, so the chunks ramp: `lead` plots, then
    doubling up to `chunk`, the middle in near-equal chunks of at most `chunk`, and the
    mirror image at the end (a batched run computes a plot in about twice the time its
    copy takes, so each chunk's copy hides behind the previous chunk's run)."""
    if lead <= 0 or lead >= chunk or nb < 3 * lead:
        sizes = [chunk] * (nb // chunk) + ([nb % chunk] if nb % chunk else [])
    else:
        ramp = []
        c = lead
        while c < chunk and 2 * (sum(ramp) + c) + c <= nb:  # leaves a middle at least c
            ramp.append(c)
            c *= 2
        mid = nb - 2 * sum(ramp)
        k = -(-mid // chunk)
        sizes = ramp + [mid // k + (1 if q < mid % k else 0) for q in range(k)] + ramp[::-1]
    out, b0 = [], 0
    for n in sizes:
        out.append((b0, b0 + n))
        b0 += n
    return out


def splom_plot(idx: int, n: int, seed: int = 2408) -> np.ndarray:
    """Synthetic plot `idx` of the batch: a Gaussian mixture of 1-8 clusters (PCG64
    stream seeded by (seed, idx), the reference suite's seeding pattern,
    datasets.py:140-149), float32-representable, resampled into [0, 1]^2."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence((seed, idx))))
    m = int(rng.integers(1, 9))
    w = rng.uniform(0.5, 2.0, size=m)
    counts = np.floor(w / w.sum() * n).astype(np.int64)
    counts[: n - int(counts.sum())] += 1
    centres = rng.uniform(0.12, 0.88, size=(m, 2))
    sig = rng.uniform(0.005, 0.02, size=m)
    parts = []
    for c in range(m):
        p = rng.normal(centres[c], sig[c], size=(int(counts[c]), 2))
        for _ in range(64):
            bad = np.any((p < 0) | (p > 1), axis=1)
            if not bad.any():
                break
            p[bad] = rng.normal(centres[c], sig[c], size=(int(bad.sum()), 2))
        parts.append(np.clip(p, 0, 1))
    return np.concatenate(parts).astype(np.float32).astype(np.float64)


@dataclass
class SplomConfig:
    nplots: int = 256
    points: int = 500_000
    k: int = 10
    kernel_size: int = 8
    iterations: int = 10
    max_batch: int = 256        # plots per batched launch (bounds the workspace: ~43 MB per plot at C4)
    collect_metrics: bool = False  # per-frame binned_stddev / overplotting of every plot ("basic")
    stop: str = "fixed"         # or "displacement": each plot stops at its own iteration (regularize.py:76-79)
    epsilon: float = 1e-4


class DeviceSplom:
    """Runs this rank's block of plots as batched runs of up to `max_batch` plots."""

    def __init__(self, cfg: SplomConfig, plot_ids: Sequence[int], device=None):
        import torch

        from . import _device as D
        from . import _lib

        self.torch, self.D, self._lib = torch, D, _lib
        self.lib = D.require_cuda()
        D.check_grid(cfg.k)
        self.cfg = cfg
        self.ids = list(plot_ids)
        self.dev = device or D.device()
        n = cfg.points
        nb = len(self.ids)
        self.inputs = torch.empty((nb, n, 2), dtype=torch.float32, device=self.dev)
        self.work = torch.empty_like(self.inputs)
        # plots of an odd size cannot share 16-byte aligned batch strides: one per launch
        self.batch = max(1, min(cfg.max_batch, nb)) if n % 2 == 0 else 1
        self.chunks = [(b0, min(b0 + self.batch, nb)) for b0 in range(0, nb, self.batch)]
        wsb = int(self.lib.inim_workspace_bytes(cfg.k, n, self.batch))
        self.ws = torch.empty(wsb, dtype=torch.uint8, device=self.dev)
        self.stats = (torch.zeros((nb, cfg.iterations, 3), dtype=torch.int64, device=self.dev)
                      if cfg.collect_metrics else None)
        if cfg.stop not in ("fixed", "displacement"):
            raise ValueError("a batched run stops on a fixed count or on displacement")
        self.eps = 0.0
        if cfg.stop == "displacement":
            if not cfg.epsilon > 0:
                raise ValueError("epsilon must be > 0")
            self.eps = max(float(np.float32(cfg.epsilon)), float(np.finfo(np.float32).smallest_subnormal))
        self.states = torch.zeros((nb, 4), dtype=torch.int32, device=self.dev) if self.eps > 0 else None

    def load(self, make_plot: Callable[[int], np.ndarray]):
        for q, idx in enumerate(self.ids):
            self.inputs[q].copy_(self.torch.from_numpy(make_plot(idx).astype(np.float32)))

    def run(self, on_chunk: Optional[Callable[[int, int], None]] = None):
        """All plots, `iterations` each, on the current stream; inputs stay untouched
        (results in .work).  on_chunk(b0, b1) is called after each batched run of plots
        [b0, b1) is enqueued (a pipelined gather starts that chunk's collective there)."""
        D, lib, cfg = self.D, self.lib, self.cfg
        self.work.copy_(self.inputs)
        stream = D.stream()
        for b0, b1 in self.chunks:
            stats = D.ptr(self.stats[b0:b1]) if self.stats is not None else None
            self._lib.check(lib.inim_run_batched(D.ptr(self.work[b0:b1]), cfg.points, b1 - b0, cfg.k,
                                                 cfg.kernel_size, 0.0, cfg.iterations, self.eps,
                                                 D.ptr(self.states[b0:b1]) if self.states is not None else None,
                                                 stats, D.ptr(self.ws),
                                                 stream), "splom run")
            if on_chunk is not None:
                on_chunk(b0, b1)
        return self.work

    def run_host(self, host_in, host_out, chunk: int = 96, lead: int = 8):
        """The whole block from page-locked host buffers: (B, n, 2) float32 in, final
        positions out.  The plots go in chunks of about `chunk`: chunk c + 1 is copied in
        on one copy stream and chunk c - 1 copied out on another while chunk c runs (the
        copy engines work beside the SMs), so the step costs about max(compute,
        transfers) instead of their sum.  The chunks ramp from `lead` plots up and back
        down (_chunk_bounds): the first copy in and the last copy out are the parts
        nothing overlaps.  Returns host_out."""
        torch, D, lib, cfg = self.torch, self.D, self.lib, self.cfg
        nb = len(self.ids)
        chunk = max(1, min(chunk, self.batch))
        cur = torch.cuda.current_stream(self.dev)
        h2d, d2h = torch.cuda.Stream(device=self.dev), torch.cuda.Stream(device=self.dev)
        start = torch.cuda.Event()
        start.record(cur)
        h2d.wait_event(start)
        d2h.wait_event(start)
        copied, ran = [], []
        bounds = _chunk_bounds(nb, chunk, min(lead, chunk))
        for b0, b1 in bounds:  # all copies in, in order, on their own stream
            with torch.cuda.stream(h2d):
                self.work[b0:b1].copy_(host_in[b0:b1], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(h2d)
                copied.append(ev)
        for (b0, b1), ev in zip(bounds, copied):
            cur.wait_event(ev)
            stats = D.ptr(self.stats[b0:b1]) if self.stats is not None else None
            self._lib.check(lib.inim_run_batched(D.ptr(self.work[b0:b1]), cfg.points, b1 - b0, cfg.k,
                                                 cfg.kernel_size, 0.0, cfg.iterations, self.eps,
                                                 D.ptr(self.states[b0:b1]) if self.states is not None else None,
                                                 stats, D.ptr(self.ws),
                                                 D.stream()), "splom run")
            done = torch.cuda.Event()
            done.record(cur)
            ran.append(done)
            with torch.cuda.stream(d2h):
                d2h.wait_event(done)
                host_out[b0:b1].copy_(self.work[b0:b1], non_blocking=True)
        fin = torch.cuda.Event()
        fin.record(d2h)
        cur.wait_event(fin)
        return host_out

    def iterations_done(self) -> list:
        """Iterations each plot ran (all of them for stop="fixed")."""
        if self.states is None:
            return [self.cfg.iterations] * len(self.ids)
        return [int(v) for v in self.states[:, 1].cpu().tolist()]

    def metrics(self):
        """Per plot and frame 1..iterations: (binned_stddev, overplotting) as the
        reference's record_for_frame (metrics.py:46-71, 147-168), from the device
        occupancy statistics."""
        from .metrics import overplotting_from_stats, stddev_from_stats

        if self.stats is None:
            raise ValueError("SplomConfig(collect_metrics=True) is needed")
        st = self.stats.cpu().numpy()
        n, k = self.cfg.points, self.cfg.k
        done = self.iterations_done()
        return [[(stddev_from_stats(int(st[q, t, 1]), int(st[q, t, 2]), k), overplotting_from_stats(int(st[q, t, 0]), n))
                 for t in range(done[q])] for q in range(len(self.ids))]


def gather_results(local, nplots: int, world: int, group=None):
    """All-gather every rank's block of final positions into (nplots, n, 2) on every
    rank.  Blocks are padded to the largest shard so one all_gather_into_tensor moves
    everything; padding rows are dropped afterwards."""
    import torch
    import torch.distributed as dist

    if world == 1:
        return local
    per = max(len(shard(nplots, world, r)) for r in range(world))
    shape = (per,) + tuple(local.shape[1:])
    buf = torch.zeros(shape, dtype=local.dtype, device=local.device)
    buf[: local.shape[0]].copy_(local)
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world,) + shape, dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(out, buf, group=group)  # one NCCL all-gather over NVLink
        blocks = [out[r] for r in range(world)]
    else:  # gloo (CPU tests): list form
        blocks = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(blocks, buf, group=group)
    parts = [blocks[r][: len(shard(nplots, world, r))] for r in range(world)]
    return torch.cat(parts, dim=0)


def pipeline_parts(nplots: int, world: int, parts: int) -> list:
    """Offsets [b0, b1) within every rank's block of the pipelined gather's sub-batches
    (the same on every rank: blocks are padded to the largest shard)."""
    per = max(len(shard(nplots, world, r)) for r in range(world))
    step = max(1, -(-per // max(1, parts)))
    return [(b0, min(b0 + step, per)) for b0 in range(0, per, step)]


class GatherPipeline:
    """The gather of the final positions split into sub-batches, each started as soon as
    its batched run is enqueued (asynchronous collective: NCCL runs it on its own stream
    after the compute stream reaches that point), so the transfer of sub-batch q
    overlaps the compute of sub-batch q + 1.  finish() waits and reassembles the plots in
    global order (rank blocks, padding dropped)."""

    def __init__(self, nplots: int, world: int, rank: int, parts: int, like, group=None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist, self.group = torch, dist, group
        self.nplots, self.world, self.rank = nplots, world, rank
        self.bounds = pipeline_parts(nplots, world, parts)
        self.nccl = world > 1 and dist.get_backend(group) == "nccl"
        self.shape = tuple(like.shape[1:])
        self.dtype, self.device = like.dtype, like.device
        self.counts = [len(shard(nplots, world, r)) for r in range(world)]
        self.works, self.outs = [], []

    def ready(self, local, b1: int):
        """This rank's plots [0, b1) of its block (`local`) are computed (enqueued): start
        every sub-batch collective they complete, in order (the same order on every
        rank; a short block completes its later sub-batches at once)."""
        n = local.shape[0]
        while len(self.outs) < len(self.bounds):
            c0, c1 = self.bounds[len(self.outs)]
            if min(c1, n) > b1:
                break
            self._submit(local, len(self.outs))

    def _submit(self, local, q: int):
        torch, dist = self.torch, self.dist
        c0, c1 = self.bounds[q]
        width = c1 - c0
        have = max(0, min(local.shape[0], c1) - c0)
        if have == width:
            src = local[c0:c1]
        else:  # a short (or empty) last block: pad to the common width
            src = torch.zeros((width,) + self.shape, dtype=self.dtype, device=self.device)
            if have:
                src[:have].copy_(local[c0:c0 + have])
        if self.world == 1:
            self.outs.append([src])
            return
        if self.nccl:
            out = torch.empty((self.world, width) + self.shape, dtype=self.dtype, device=self.device)
            self.works.append(dist.all_gather_into_tensor(out, src.contiguous(), group=self.group, async_op=True))
            self.outs.append([out[r] for r in range(self.world)])
        else:  # gloo (CPU tests): list form
            blocks = [torch.empty_like(src) for _ in range(self.world)]
            self.works.append(dist.all_gather(blocks, src.contiguous(), group=self.group, async_op=True))
            self.outs.append(blocks)

    def finish(self, local):
        self.ready(local, local.shape[0])
        for w in self.works:
            w.wait()
        parts = []
        for r in range(self.world):
            for q, (c0, c1) in enumerate(self.bounds):
                n = max(0, min(self.counts[r], c1) - c0)
                if n:
                    parts.append(self.outs[q][r][:n])
        self.works, self.outs = [], []
        return self.torch.cat(parts, dim=0)


def run_distributed(cfg: SplomConfig, rank: int, world: int, make_plot: Optional[Callable] = None, group=None,
                    gather_parts: int = 1):
    """One rank's share of the batch + the gather; returns all final positions.  With
    gather_parts > 1 the rank's block runs as that many sub-batches, each gathered while
    the next one computes."""
    ids = shard(cfg.nplots, world, rank)
    if gather_parts > 1:
        cfg = SplomConfig(**{**cfg.__dict__, "max_batch": pipeline_parts(cfg.nplots, world, gather_parts)[0][1]})
    job = DeviceSplom(cfg, ids)
    job.load(make_plot or (lambda i: splom_plot(i, cfg.points)))
    pipe = GatherPipeline(cfg.nplots, world, rank, gather_parts, job.work, group)
    job.run(on_chunk=lambda b0, b1: pipe.ready(job.work, b1))
    return pipe.finish(job.work)
