"""CPU, world_size 2 over gloo: the host-side logic of the batch-sharded step -- the reference's contiguous chunking
with ranks as workers (src/trainer.cpp:93,107-108) and the algebra the SUM all-reduce relies on: the gradient
accumulator marks untouched rows with -0.0f, and IEEE addition keeps that marker exactly when every rank left the row
untouched."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2311_15439_b200.trainer import chunk_bounds  # noqa: E402  (needs the built library to import the package)


def test_chunk_bounds_match_reference_worker_chunks():
    for batch, workers in [(2048, 8), (10, 3), (7, 8), (1, 1), (262144, 8), (5, 2), (64, 3)]:
        chunk = (batch + workers - 1) // workers  # src/trainer.cpp:93
        covered = []
        for t in range(workers):
            begin = t * chunk
            end = min(batch, begin + chunk)  # :107-108 (workers with begin >= end do not start)
            b, e = chunk_bounds(batch, workers, t)
            if begin >= end:
                assert b == e
            else:
                assert (b, e) == (begin, end)
            covered += list(range(b, e))
        assert covered == list(range(batch))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    neg0 = np.float32(-0.0)
    # rows: [untouched everywhere, touched with +0 on rank 1 only, value on rank 0 only, values on both, cancel exactly]
    mine = {0: [neg0, neg0, 1.5, 0.25, 3.0], 1: [neg0, 0.0, neg0, -1.0, -3.0]}[rank]
    t = torch.tensor(np.array(mine, dtype=np.float32))
    dist.all_reduce(t)  # SUM, what Trainer.distributed_step issues on the table-gradient view
    loss = torch.tensor([0.5 + rank], dtype=torch.float64)
    dist.all_reduce(loss)
    # every rank holds the full deterministic batch and takes its contiguous chunk
    batch = torch.arange(10)
    b, e = chunk_bounds(10, world, rank)
    part = torch.zeros(10, dtype=torch.int64)
    part[b:e] = batch[b:e] + 1
    dist.all_reduce(part)
    if rank == 0:
        out.put((t.numpy().view(np.uint32).tolist(), float(loss.item()), part.tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_gradient_allreduce_keeps_the_untouched_marker():
    ctx = mp.get_context("spawn")
    out = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    bits, loss, part = out.get()
    f = np.array(bits, dtype=np.uint32).view(np.float32)
    assert bits[0] == 0x80000000            # -0 + -0 = -0 : still untouched
    assert bits[1] == 0x00000000            # -0 + +0 = +0 : touched with a zero gradient
    assert f[2] == 1.5 and f[3] == -0.75    # -0 + v = v ; plain sums
    assert bits[4] == 0x00000000            # exact cancellation is +0 : touched
    assert loss == 2.0
    assert part == list(range(1, 11))       # the chunks tile the batch exactly once


def test_level_ranges_cover_every_level_once():
    from paper_2311_15439_b200.trainer import level_ranges
    for levels in (1, 3, 8, 16, 17):
        for chunks in (1, 2, 4, 5, 16, 64):
            r = level_ranges(levels, chunks)
            assert len(r) <= max(1, min(chunks, levels))
            covered = [l for f, c in r for l in range(f, f + c)]
            assert covered == list(range(levels)), (levels, chunks, r)
            assert all(c >= 1 for _, c in r)


def _chunk_worker(rank, world, port, out):
    """The exchange of Trainer.distributed_step on CPU tensors: the level-major accumulator is all-reduced one level range
    at a time, asynchronously, while 'the next range computes'; the result must equal one all-reduce of the whole buffer."""
    from paper_2311_15439_b200.trainer import level_ranges
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    levels, per_level = 16, 64
    g = torch.Generator().manual_seed(100 + rank)
    whole = torch.randn(levels * per_level, generator=g)
    whole[torch.rand(levels * per_level, generator=g) < 0.3] = -0.0  # untouched rows of this rank
    chunked = whole.clone()
    dist.all_reduce(whole)
    pending = []
    for first, count in level_ranges(levels, 4):
        sl = chunked[first * per_level:(first + count) * per_level]  # contiguous slice of the level-major buffer
        pending.append(dist.all_reduce(sl, async_op=True))
    for w in pending:
        w.wait()
    if rank == 0:
        out.put(bool(torch.equal(whole.view(torch.int32), chunked.view(torch.int32))))
    dist.barrier()
    dist.destroy_process_group()


def test_level_chunked_exchange_equals_the_whole_buffer_allreduce():
    ctx = mp.get_context("spawn")
    out = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_chunk_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert out.get() is True
