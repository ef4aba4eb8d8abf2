"""N>1 path on CPU: world_size-2 gloo processes.

The multi-GPU path shards independent camera streams over ranks with no
data-path collective; the only collectives are the timing barrier and the
max-over-ranks reduction. These tests run that host logic (paper_1704_04313_b200.shard)
under torch.distributed/gloo with two processes and check that (1) the shards
are disjoint and cover the global stream set, (2) max_over_ranks is the max,
(3) per-stream results (oracle forward_frame on each owned stream's clip) are
independent of the world size -- what sharding by stream relies on.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from netutil import tiny_spec

S_PER_RANK = 2
FRAMES = 3


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _clip_cfg(seed):
    return dict(channels=2, height=16, width=16, sprites=[(4, 2, 0.9)], noise=0.0, seed=seed)


def _run_stream(orc, weights, g):
    net = orc.load_network(tiny_spec(0.01), weights)
    cfg = _clip_cfg(__import__("paper_1704_04313_b200.shard", fromlist=["x"]).stream_seed(g))
    out = []
    for f in range(FRAMES):
        r = net.forward_frame(orc.synth_frame(cfg, f))
        out.append(np.asarray(r["labels"]))
    return np.stack(out)


def _worker(rank, world, port, outdir):
    import torch.distributed as dist

    from oracle import Oracle
    from paper_1704_04313_b200 import shard

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        mine = shard.streams_for_rank(S_PER_RANK, rank, world)
        orc = Oracle()
        w = orc.generate_weights(tiny_spec(0.01), 1)
        for g in mine:
            np.save(os.path.join(outdir, f"s{g}.npy"), _run_stream(orc, w, g))
        shard.barrier()
        m = shard.max_over_ranks(1.5 + rank)
        with open(os.path.join(outdir, f"max{rank}.txt"), "w") as f:
            f.write(f"{m}\n{','.join(map(str, mine))}\n")
    finally:
        dist.destroy_process_group()


def test_shard_partition():
    from paper_1704_04313_b200 import shard
    for world in (1, 2, 4, 8):
        got = sorted(g for r in range(world) for g in shard.streams_for_rank(3, r, world))
        assert got == list(range(3 * world))
    with pytest.raises(ValueError):
        shard.streams_for_rank(1, 2, 2)
    assert shard.aggregate_rate(2, 8, 1000.0) == 16.0
    assert shard.max_over_ranks(3.25) == 3.25  # no process group: identity


def test_gloo_world2_streams_sharded(tmp_path, orc):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    owned = []
    for r in range(world):
        m, streams = open(tmp_path / f"max{r}.txt").read().split()
        assert float(m) == 1.5 + (world - 1)
        owned.append([int(x) for x in streams.split(",")])
    assert sorted(owned[0] + owned[1]) == list(range(world * S_PER_RANK))
    assert not set(owned[0]) & set(owned[1])
    # a single process running every stream sees identical per-stream results
    w = orc.generate_weights(tiny_spec(0.01), 1)
    for g in range(world * S_PER_RANK):
        np.testing.assert_array_equal(np.load(tmp_path / f"s{g}.npy"), _run_stream(orc, w, g))
