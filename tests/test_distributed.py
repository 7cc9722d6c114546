"""Multi-process (gloo, world_size 2) tests of the SPLOM sharding and result gather on
CPU.  The per-plot compute is the GPU path and cannot run here; the distributed
plumbing (shard ownership, padded all-gather, reassembly order) is what these cover."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_partition():
    from paper_2408_06513_b200.splom import shard

    for nplots in (1, 7, 256, 255):
        for world in (1, 2, 3, 4, 8):
            got = [list(shard(nplots, world, r)) for r in range(world)]
            flat = [i for g in got for i in g]
            assert flat == list(range(nplots))
            sizes = [len(g) for g in got]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard(4, 2, 2)


def test_splom_plot_generator_deterministic():
    from paper_2408_06513_b200.splom import splom_plot

    a, b = splom_plot(3, 1000), splom_plot(3, 1000)
    assert np.array_equal(a, b) and a.shape == (1000, 2)
    assert a.min() >= 0 and a.max() <= 1
    assert np.array_equal(a, a.astype(np.float32).astype(np.float64))
    assert not np.array_equal(a, splom_plot(4, 1000))


def _worker(rank, world, port, nplots, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2408_06513_b200.splom import gather_results, shard

        ids = shard(nplots, world, rank)
        # stand-in per-plot result: plot index in every coordinate (checks the reassembly order)
        local = torch.stack([torch.full((5, 2), float(i)) for i in ids]) if len(ids) else torch.zeros((0, 5, 2))
        allres = gather_results(local, nplots, world)
        out_q.put((rank, allres[:, 0, 0].tolist()))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # surface worker failures instead of a queue timeout
        out_q.put((rank, repr(e)))


@pytest.mark.parametrize("nplots", [7, 8])
def test_gather_world2(nplots):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, nplots, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        assert res[r] == [float(i) for i in range(nplots)]


def _bench_worker(rank, world, port, out_q):
    """bench.py's distributed skeleton (barrier, max-over-ranks timing) on gloo."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t = torch.tensor([1.0 + rank], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    out_q.put((rank, float(t.item())))
    dist.destroy_process_group()


def test_max_over_ranks_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: 2.0, 1: 2.0}


def test_bench_gpus2_self_launch_shard_gather_on_gloo():
    """`bench.py --gpus 2` outside torchrun re-launches itself with two ranks
    (torch.distributed.run), each rank takes its contiguous block of the SPLOM batch,
    runs it (compute stubbed on the CPU: --cpu-stub) and the step all-gathers every
    plot's positions; rank 0 prints one line with n_gpus = 2 and the reassembled order
    checked, the max-over-ranks timing in ms_per_step."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    env = dict(os.environ)
    for v in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(v, None)
    out = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--cpu-stub", "--plots", "7",
                          "--splom-points", "16", "--steps", "2", "--warmup", "3"],
                         capture_output=True, text=True, timeout=600, env=env, cwd=str(root))
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["scaling"] == "strong"
    assert rec["collective"]["world"] == 2 and rec["collective"]["backend"] == "gloo"
    assert rec["collective"]["gather_ok"] is True
    assert rec["plots_per_rank"] == 4  # rank 0's block of 7 plots over 2 ranks
    assert rec["value"] > 0 and rec["ms_per_step"] > 0


def test_bench_rejects_mismatched_world():
    """--gpus N under a torchrun world of a different size fails loudly."""
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--cpu-stub"],
                         capture_output=True, text=True, timeout=300, env=env, cwd=str(root))
    assert out.returncode != 0 and "WORLD_SIZE=1" in out.stderr


def _pipe_worker(rank, world, port, nplots, parts, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2408_06513_b200.splom import GatherPipeline, pipeline_parts, shard

        ids = list(shard(nplots, world, rank))
        local = torch.stack([torch.full((3, 2), float(i)) for i in ids]) if ids else torch.zeros((0, 3, 2))
        pipe = GatherPipeline(nplots, world, rank, parts, torch.zeros((1, 3, 2)))
        step = pipeline_parts(nplots, world, parts)[0][1]
        for b0 in range(0, len(ids), step):  # the chunked run's callbacks
            pipe.ready(local, min(b0 + step, len(ids)))
        allres = pipe.finish(local)
        out_q.put((rank, allres[:, 0, 0].tolist()))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:
        out_q.put((rank, repr(e)))


@pytest.mark.parametrize("nplots,parts", [(7, 2), (8, 3), (3, 2), (9, 4), (8, 1)])
def test_pipelined_gather_world2(nplots, parts):
    """Sub-batched gather: every rank submits the same collectives in the same order
    (short blocks pad, empty sub-batches included) and the plots come back in global
    order."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pipe_worker, args=(r, 2, port, nplots, parts, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        assert res[r] == [float(i) for i in range(nplots)], res[r]
