"""CPU (gloo, world_size 2) tests of the multi-GPU plumbing: query sharding
and the single end-of-run gather of per-query records.  The per-query solve
here is the CPU oracle standing in for each rank's GPU; on the GPU box the
same shard/gather code runs under NCCL in bench.py."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1705_02403_b200.shard import gather_records, records, shard_range, weak_range


def test_shard_range_partitions():
    for total in (0, 1, 7, 64, 4096, 4097):
        for world in (1, 2, 3, 4, 8):
            parts = [shard_range(total, world, r) for r in range(world)]
            flat = [q for p in parts for q in p]
            assert flat == list(range(total))
            sizes = [len(p) for p in parts]
            assert max(sizes) - min(sizes) <= 1
    assert list(weak_range(512, 3)) == list(range(1536, 2048))
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    import oracle
    from paper_1705_02403_b200 import problem as P
    from tests.helpers import oracle_instance

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    port_lib = oracle.port()

    class S:  # PlanSummary-shaped
        pass

    sums = []
    for q in shard_range(total, world, rank):
        spec = P.random_forest_query(99, q, n=300)
        o = oracle_instance(port_lib, spec)
        r = port_lib.gmt_plan(spec, o["coords"], len(o["goal_idx"]), o["graph"], o["init"], 1.0,
                              o["radius"])
        s = S()
        s.status, s.cost, s.iterations = r.status, r.cost, r.iterations
        s.total_collision_checks, s.path_len = r.total_collision_checks, len(r.path_indices)
        s.num_stats = len(r.group_sizes)
        sums.append(s)
    got = gather_records(records(sums))
    if rank == 0:
        np.save(os.path.join(out_dir, "gathered.npy"), got)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shard_and_gather(tmp_path):
    total = 7  # uneven split: 4 + 3
    mp.spawn(_worker, args=(2, _free_port(), total, str(tmp_path)), nprocs=2, join=True)
    got = np.load(os.path.join(tmp_path, "gathered.npy"))
    assert got.shape == (total, 6)

    import oracle
    from paper_1705_02403_b200 import problem as P
    from tests.helpers import oracle_instance
    port_lib = oracle.port()
    for q in range(total):
        spec = P.random_forest_query(99, q, n=300)
        o = oracle_instance(port_lib, spec)
        r = port_lib.gmt_plan(spec, o["coords"], len(o["goal_idx"]), o["graph"], o["init"], 1.0,
                              o["radius"])
        assert got[q, 0] == r.status and got[q, 2] == r.iterations
        assert got[q, 3] == r.total_collision_checks
        assert got[q, 1] == r.cost or (np.isinf(got[q, 1]) and np.isinf(r.cost))
