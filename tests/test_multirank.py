"""The N > 1 path on CPU (gloo, world size 2): keys shard by GLOBAL index with no data exchange
(SURVEY.md section 8(e)).  Each rank computes its key range through the
oracle (test infrastructure) exactly as bench.py shards the GPU work (first_key_index = rank * n);
the gathered bytes must equal one process computing the whole range, and the step time reported
is the max over ranks (bench.py's all_reduce MAX)."""
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
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    first = rank * n                                   # bench.py: first_key_index = rank * n
    res = O.keygen_many(761, 2, np.arange(first, first + n, dtype=np.uint64))
    pk = torch.from_numpy(np.ascontiguousarray(res["pk"]))
    sk = torch.from_numpy(np.ascontiguousarray(res["sk"]))
    pks = [torch.empty_like(pk) for _ in range(world)]
    sks = [torch.empty_like(sk) for _ in range(world)]
    dist.all_gather(pks, pk)
    dist.all_gather(sks, sk)
    # max-over-ranks step time, as bench.py reduces its CUDA-event times
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        np.save(os.path.join(out_dir, "pk.npy"), torch.cat(pks).numpy())
        np.save(os.path.join(out_dir, "sk.npy"), torch.cat(sks).numpy())
        np.save(os.path.join(out_dir, "t.npy"), t.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_equals_single_process(tmp_path, O):
    world, n = 2, 6
    mp.spawn(_worker, args=(world, _free_port(), n, str(tmp_path)), nprocs=world, join=True)
    pk = np.load(tmp_path / "pk.npy")
    sk = np.load(tmp_path / "sk.npy")
    ref = O.keygen_many(761, 2, np.arange(world * n, dtype=np.uint64))
    assert np.array_equal(pk, ref["pk"]) and np.array_equal(sk, ref["sk"])
    assert float(np.load(tmp_path / "t.npy")[0]) == float(world)
