"""N>1 path on CPU with the gloo backend, world_size 2 (⑤): the scene batch
is replicas-only — each rank owns an independent scene; the only collective
gathers per-scene stats and takes the max-over-ranks time. Also checks that
per-rank host-side work (partition / hierarchy, the native host code every
rank runs) is identical across ranks for identical scenes."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        import paper_2411_06224_b200 as P
        from paper_2411_06224_b200 import scenes

        # per-rank scene work (host side of the hot path): identical scenes
        # must give identical hierarchies on every rank
        sc = scenes.CONFIGS["cfg1_soft_cube"]()
        l0 = P.partition_block_graph(sc.n_blocks, sc.rest_edges, 16)
        h = P.build_hierarchy(l0, sc.rest_edges, 4)
        sig = [int(L["n_nodes"]) for L in h.levels] + [int(np.sum(L["agg"])) for L in h.levels]
        stats = dict(total_ms=10.0 + rank, pcg_ms=5.0 + 2 * rank, iters=100 + rank, conv=True, sig=sig)
        gathered, agg = bench.gather_scene_stats(stats, world, dist)
        q.put((rank, gathered, agg))
    finally:
        dist.destroy_process_group()


def test_scene_batch_stats_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, gathered, agg in results:
        assert len(gathered) == world
        assert agg["max_total_ms"] == 11.0       # max over ranks
        assert agg["max_pcg_ms"] == 7.0
        assert agg["iters"] == 201               # work summed over the batch
        assert gathered[0]["sig"] == gathered[1]["sig"]


def test_single_rank_stats_without_dist():
    import bench

    g, agg = bench.gather_scene_stats(dict(total_ms=3.0, pcg_ms=2.0, iters=7, conv=True), 1, None)
    assert agg == {"max_total_ms": 3.0, "max_pcg_ms": 2.0, "iters": 7, "converged": True}


if __name__ == "__main__":
    pytest.main([__file__, "-q"])
