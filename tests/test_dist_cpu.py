"""Host logic of the multi-GPU path on the CPU: stream sharding and the final
metrics gather over a gloo process group with world size 2."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2011_03910_b200.dist import gather_metrics, shard_streams, summarize


def test_shard_streams_partition():
    for total in (0, 1, 7, 64, 512, 513):
        for world in (1, 2, 3, 4, 8):
            shards = [shard_streams(total, world, r) for r in range(world)]
            assert sum(s.n_streams for s in shards) == total
            pos = 0
            for s in shards:
                assert s.stream_begin == pos
                pos += s.n_streams
            sizes = [s.n_streams for s in shards]
            assert max(sizes) - min(sizes) <= 1
    assert shard_streams(512, 8, 3).n_streams == 64
    with pytest.raises(ValueError):
        shard_streams(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shard = shard_streams(512, world, rank)
    m = {"frames": shard.n_streams * 8 * 10, "ids_issued": 100 + rank, "elapsed_ms": 10.0 + rank,
         "live_tracks": 50, "candidates": 1, "detections": 1, "records": 1}
    out = gather_metrics(m)
    q.put((rank, out, summarize(out)))
    dist.barrier()
    dist.destroy_process_group()


def test_gather_metrics_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, per_rank, summ in res:
        assert [m["ids_issued"] for m in per_rank] == [100.0, 101.0]
        assert summ["frames"] == 512 * 8 * 10
        assert summ["max_elapsed_ms"] == 11.0                  # max over ranks
        assert summ["frames_per_s"] == pytest.approx(512 * 8 * 10 / 0.011)


def test_gather_without_process_group():
    out = gather_metrics({"frames": 5, "elapsed_ms": 2.0})
    assert out[0]["frames"] == 5.0 and summarize(out)["frames_per_s"] == pytest.approx(2500.0)
