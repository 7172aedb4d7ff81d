"""Multi-rank protocol of the sharded encode on CPU (gloo, world size 2).

Each rank encodes its shard (top-level blocks t % W == rank, with their subtrees) -- here with
the oracle standing in for the GPU encode, since this container has no GPU -- and the product's
gather (paper_1501_04140_b200.dist.gather_records, the same call the NCCL path uses) must
reassemble exactly the single-process code after canonical ordering (B desc, ry, rx).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from fic_inputs import config, image_for
        from paper_1501_04140_b200.dist import gather_records

        cfg = config("C2", seed=1)
        cfg["N"] = 128
        cfg["tau"] = [-1.0, 4.5, -1.0, 2.6]
        from fic_inputs import make_image
        img = make_image(128, 5)
        local = oracle.encode_cfg(cfg, img, shard=rank, n_shards=world)
        t = torch.from_numpy(local.view(np.uint8).reshape(-1, 40).copy())
        allrec, counts, stride = gather_records(t)
        if rank == 0:
            a = allrec.numpy()
            parts = [a[r * stride: r * stride + counts[r]] for r in range(world)]
            merged = np.concatenate(parts).reshape(-1).view(oracle.RECORD_DTYPE)
            order = np.lexsort((merged["rx"], merged["ry"], -merged["B"]))
            full = oracle.encode_cfg(cfg, img)
            fields = ("rx", "ry", "B", "dom", "dx", "dy", "iso", "s_idx", "o_code", "accepted", "err")
            ok = len(merged) == len(full) and all(np.array_equal(merged[order][f], full[f]) for f in fields)
            result[0] = 1 if ok else 0
            result[1] = len(full)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gather_two_ranks_gloo():
    port = _free_port()
    result = torch.zeros(2, dtype=torch.int64).share_memory_()
    mp.spawn(_worker, args=(2, port, result), nprocs=2, join=True)
    assert result[1] > 0
    assert result[0] == 1
