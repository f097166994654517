"""N > 1 host logic with world_size 2 over gloo on CPU: the communicator-id broadcast,
row sharding, max-over-ranks timing and result gathering used by bench.py's torchrun
path (the device exchange itself is covered on one GPU by the virtual-rank parity tests)."""
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


def _worker(rank, world, port, n, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2311_14908_b200 import shard_rows
    from paper_2311_14908_b200.dist import broadcast_uid, gather_rows, max_over_ranks
    dev = torch.device("cpu")
    uid = bytes(range(128)) if rank == 0 else None
    got = broadcast_uid(uid, dev)
    blocks = shard_rows(n, world)
    lo, hi = blocks[rank]
    local = torch.arange(lo, hi, dtype=torch.float64) * 0.5
    full = gather_rows(local, blocks, dev)
    t = max_over_ranks(1.0 + rank, dev)
    # OvO: each rank trains its share of the pairs; gather_models assembles all of them
    from paper_2311_14908_b200.multiclass import OvOModel, enumerate_pairs, gather_models
    mdl = OvOModel(4, 1, 0.5)
    for k, pair in enumerate(enumerate_pairs(4)):
        if k % world == rank:
            mdl.models[pair] = dict(b=float(k), coef=np.arange(k, dtype=np.float64))
    gather_models(mdl)
    np.save(os.path.join(out_dir, f"m{rank}.npy"), np.array([mdl.models[p]["b"] for p in enumerate_pairs(4)]))
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), uid=np.frombuffer(got, np.uint8), full=full.numpy(),
             t=t, lo=lo, hi=hi)
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [7, 1000, 32561])
def test_two_rank_host_path(tmp_path, n):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), n, str(tmp_path)), nprocs=world,
                       start_method="spawn")
    r = [np.load(os.path.join(tmp_path, f"r{k}.npz")) for k in range(world)]
    for k in range(world):
        assert bytes(r[k]["uid"]) == bytes(range(128))
        np.testing.assert_array_equal(r[k]["full"], np.arange(n) * 0.5)
        assert float(r[k]["t"]) == 2.0
    assert int(r[0]["lo"]) == 0 and int(r[1]["hi"]) == n and int(r[0]["hi"]) == int(r[1]["lo"])
    for k in range(world):
        assert np.load(os.path.join(tmp_path, f"m{k}.npy")).tolist() == [float(i) for i in range(6)]
