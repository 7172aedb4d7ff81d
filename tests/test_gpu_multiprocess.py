"""The multi-rank protocol of the sharded encode with real GPU processes.

Two and three worker processes, each with its own CUDA context on the box's one GPU, form a
gloo process group.  Every rank runs the library's shard encode (fic_encode with shard = rank,
n_shards = W: the top-level blocks t % W == rank and their subtrees, every pool built by the rank
itself), the codes are all-gathered (paper_1501_04140_b200.dist.gather_records; CPU tensors over
gloo, because NCCL cannot place two ranks on one device) and merged on each rank's GPU with
fic_merge_shards.  Every rank must end with the one-GPU code byte for byte, and a rank-0 oracle
check closes the loop.  (fic_encode_nccl itself runs the same shard / gather / merge steps with
ncclAllGather; on this one-GPU box it is exercised on a one-rank communicator in
test_gpu_parity.py.)
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg_name, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1501_04140_b200 as p
        from paper_1501_04140_b200.dist import gather_records
        from fic_inputs import config, image_for

        cfg = config(cfg_name)
        img_np = image_for(cfg)
        img = torch.from_numpy(img_np).cuda()
        ctx = p.Context(0)
        local = ctx.encode_cfg(cfg, img, shard=rank, n_shards=world).cpu()
        allrec, counts, stride = gather_records(local)
        merged = ctx.merge_shards(allrec.cuda(), counts, stride).cpu().numpy().tobytes()
        full = ctx.encode_cfg(cfg, img).cpu().numpy().tobytes()
        ok = merged == full
        if rank == 0:
            import oracle
            ref = oracle.encode_cfg(cfg, img_np)
            got = np.frombuffer(merged, dtype=oracle.RECORD_DTYPE)
            ok = ok and len(got) == len(ref) and all(np.array_equal(got[f], ref[f]) for f in ref.dtype.names)
        result[rank] = 1 if ok else 0
        ctx.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_encode_processes(world):
    assert torch.cuda.is_available()
    from paper_1501_04140_b200 import build as b
    b.build()
    port = _free_port()
    result = torch.zeros(world, dtype=torch.int64).share_memory_()
    mp.spawn(_worker, args=(world, port, "C2", result), nprocs=world, join=True)
    assert result.tolist() == [1] * world
