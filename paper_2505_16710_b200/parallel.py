"""Multi-GPU plumbing for the chunked-attention hot path (one process per GPU).

KV-head groups are independent units of the method: every forward and gradient
term of the q-heads of group g touches only K / V / dKV of kv-head g (GQA map
h -> h // G, reading Z3).  Head sharding therefore needs no collective
on the data path; ranks only meet at the timing barrier and the max-over-ranks
reduction of the measured time.  Batch mode gives every rank its own sequence.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class HeadShard:
    q_heads: tuple      # [h0, h1) global q-head range of this rank
    kv_heads: tuple     # [g0, g1) global kv-head range of this rank

    @property
    def hq(self):
        return self.q_heads[1] - self.q_heads[0]

    @property
    def hkv(self):
        return self.kv_heads[1] - self.kv_heads[0]


def head_shard(hq: int, hkv: int, world: int, rank: int) -> HeadShard:
    """Contiguous kv-head groups per rank: rank r owns kv-heads [r*Hkv/N, (r+1)*Hkv/N)
    and the G q-heads of each.  Requires Hkv % N == 0 (no group is split, so no
    exchange is ever needed)."""
    if hq % hkv:
        raise ValueError("hq must be a multiple of hkv")
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    if hkv % world:
        raise ValueError(f"head sharding needs Hkv % N == 0 (Hkv={hkv}, N={world})")
    G = hq // hkv
    per = hkv // world
    g0, g1 = rank * per, (rank + 1) * per
    return HeadShard((g0 * G, g1 * G), (g0, g1))


def max_over_ranks(value: float, device=None) -> float:
    """MAX of a per-rank scalar (the timed region) over all ranks; identity when
    torch.distributed is not initialised."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# LLaMA3-8B, LoRA r = 8 on the q, k, v, o projections of 32 layers: per layer
# q: 8*(4096+4096), k: 8*(4096+1024), v: 8*(4096+1024), o: 8*(4096+4096) parameters.
LORA_PARAMS_LLAMA3_8B_R8 = 32 * 8 * ((4096 + 4096) + 2 * (4096 + 1024) + (4096 + 4096))


def allreduce_grad_bucket(bucket):
    """Batch-of-sequences mode (BASELINE configs[4]): every rank ran the chunked step on
    its own sequence; the per-rank fp32 LoRA-gradient bucket is summed over ranks with
    one all_reduce (NCCL over NVLink on the GPU box, gloo in the CPU tests).  The only
    device-to-device exchange of the method; a no-op on one rank."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(bucket, op=dist.ReduceOp.SUM)
    return bucket


class LayerBucketReducer:
    """Per-layer gradient buckets all-reduced as soon as each is final.

    In a SeCO / SpaCO step the last processed chunk (the smallest selected index) finishes the
    layers top-down, so the all_reduce of layer l's LoRA-gradient bucket (NCCL, async, on its
    own stream) overlaps the backward of layers l-1 .. 0.  `wait()` joins them at step end.
    A no-op on one rank or without torch.distributed."""

    def __init__(self):
        self.handles = []
        self.sent = []            # layer indices in the order their buckets were sent

    def layer_final(self, layer: int, bucket):
        import torch.distributed as dist
        self.sent.append(layer)
        if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
            self.handles.append(dist.all_reduce(bucket, op=dist.ReduceOp.SUM, async_op=True))

    def wait(self):
        for h in self.handles:
            h.wait()
        self.handles.clear()
