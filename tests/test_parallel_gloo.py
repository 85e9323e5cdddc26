"""N > 1 host logic on CPU (gloo, world_size 2): head sharding partitions the heads,
needs no exchange (each rank's oracle result on its slice equals the matching slice
of the unsharded result), and the timing reduction takes the max over ranks."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_16710_b200.parallel import (LORA_PARAMS_LLAMA3_8B_R8, LayerBucketReducer, allreduce_grad_bucket,
                                            head_shard, max_over_ranks)


def test_head_shard_partition():
    for hq, hkv, world in ((32, 8, 1), (32, 8, 2), (32, 8, 4), (32, 8, 8), (6, 2, 2)):
        seen_q, seen_kv = [], []
        for r in range(world):
            s = head_shard(hq, hkv, world, r)
            seen_q += list(range(*s.q_heads))
            seen_kv += list(range(*s.kv_heads))
            G = hq // hkv
            assert all(h // G in range(*s.kv_heads) for h in range(*s.q_heads))
        assert seen_q == list(range(hq)) and seen_kv == list(range(hkv))
    with pytest.raises(ValueError):
        head_shard(32, 8, 3, 0)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import chunkwise as OC
        from synth import make_inputs
        hq, hkv, S, d, c = 4, 2, 48, 8, 16
        x = make_inputs(hq, hkv, S, d, seed=3, bf16=False)
        s = head_shard(hq, hkv, world, rank)
        sl_q, sl_kv = slice(*s.q_heads), slice(*s.kv_heads)
        r = OC.seco_step(x.q[sl_q], x.k[sl_kv], x.v[sl_kv], x.do[sl_q], [c] * (S // c))
        # gather every rank's shard of dK to rank 0 (test only; the product path has no collective)
        dk = torch.from_numpy(r["dk"])
        parts = [torch.zeros_like(dk) for _ in range(world)]
        dist.all_gather(parts, dk)
        t = max_over_ranks(10.0 + rank)
        bucket = torch.full((1000,), float(rank + 1))
        allreduce_grad_bucket(bucket)
        if rank == 0:
            full = OC.seco_step(x.q, x.k, x.v, x.do, [c] * (S // c))
            out["dk_err"] = float(np.abs(torch.cat(parts).numpy() - full["dk"]).max())
            out["tmax"] = t
            out["bucket"] = float(bucket[0])
    finally:
        dist.destroy_process_group()


def test_sharded_oracle_equals_unsharded_gloo():
    world = 2
    port = 29500 + (os.getpid() % 1000)
    ctx = mp.get_context("spawn")
    with ctx.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True, start_method="spawn")
        assert out["dk_err"] == 0.0          # bit-identical: shards share nothing
        assert out["tmax"] == 11.0           # max over ranks
        assert out["bucket"] == 3.0          # batch-mode gradient bucket summed over ranks


def test_max_over_ranks_single_process():
    assert max_over_ranks(3.5) == 3.5


def test_lora_bucket_size():
    """LLaMA3-8B, r=8 on q,k,v,o x 32 layers = 6.82 M params = 27.3 MB fp32."""
    assert LORA_PARAMS_LLAMA3_8B_R8 == 6_815_744
    assert abs(LORA_PARAMS_LLAMA3_8B_R8 * 4 / 1e6 - 27.3) < 0.05


def _bucket_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        buckets = [torch.full((100 + l,), float((rank + 1) * (l + 1))) for l in range(3)]
        red = LayerBucketReducer()
        for l in (2, 1, 0):                  # top-down, as the last chunk's backward finishes layers
            red.layer_final(l, buckets[l])
        red.wait()
        if rank == 0:
            out["sent"] = list(red.sent)
            out["vals"] = [float(b[0]) for b in buckets] + [float(b[-1]) for b in buckets]
    finally:
        dist.destroy_process_group()


def test_layer_bucket_reducer_gloo():
    """per-layer buckets are all-reduced (async) in the order layers become final."""
    world = 2
    port = 29700 + (os.getpid() % 1000)
    ctx = mp.get_context("spawn")
    with ctx.Manager() as m:
        out = m.dict()
        mp.spawn(_bucket_worker, args=(world, port, out), nprocs=world, join=True, start_method="spawn")
        assert out["sent"] == [2, 1, 0]
        assert out["vals"] == [3.0, 6.0, 9.0] * 2


def test_layer_bucket_reducer_single_process_noop():
    red = LayerBucketReducer()
    b = torch.ones(4)
    red.layer_final(0, b)
    red.wait()
    assert red.sent == [0] and float(b.sum()) == 4.0
