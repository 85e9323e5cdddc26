"""SeCO / SpaCO step driver for one attention layer (Alg. 1, Alg. 2
P:319-338).  Owns the persistent device buffers of a step (outputs O / LSE, the
fp32 checkpoint-gradient buffer dKV, dQ, workspace) and issues the chunk calls
in the algorithm's order on one CUDA stream.  Torch is used for memory and
streams only; all arithmetic is in libseco.so."""
from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import ops
from .flops import seco_step_flops, spaco_step_flops


_CALL_NAMES = {"f": "seco_chunk_forward", "b": "seco_chunk_backward", "z": "spaco_chunk_skip"}


@dataclass
class StepResult:
    selected: list = field(default_factory=list)   # chunk indices processed in stage 2 (descending)
    relay_scale: float = 1.0
    seed_scale: float = 1.0
    flops: float = 0.0                               # algorithmic FLOPs of the step (flops.py)
    launches: int = 0                                # kernels enqueued by libseco.so


class ChunkedAttention:
    """Buffers + call sequence for one causal GQA attention layer over a sequence
    of k chunks.  dkv[0] / dkv[1] hold, after a step, the gradient of every
    chunk's own K / V (slot j = total own-chunk gradient after chunk j's relay)."""

    def __init__(self, hq, hkv, d, seq, chunk, dtype=torch.bfloat16, device="cuda", softmax_scale=0.0,
                 own_copies=False, deterministic=False, layout="hsd"):
        """layout "hsd": Q, dO, O, dQ are [hq][S][d] and the KV cache [hkv][S][d] (contiguous);
        "shd": sequence-major storage [S][h][d] (the projection output layout, where a chunk
        is one contiguous block), passed and exposed as [h][S][d] views (x.transpose(0, 1))."""
        if seq % chunk:
            raise ValueError("seq must be a multiple of chunk")
        self.hq, self.hkv, self.d, self.seq, self.chunk = hq, hkv, d, seq, chunk
        self.k = seq // chunk
        dev = torch.device(device)
        if dev.type == "cuda" and dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.dtype, self.device = dtype, dev
        dev = self.device
        if layout not in ("hsd", "shd"):
            raise ValueError("layout must be 'hsd' or 'shd'")
        self.layout = layout

        def buf(h):
            if layout == "hsd":
                return torch.empty(h, seq, d, dtype=dtype, device=dev)
            return torch.empty(seq, h, d, dtype=dtype, device=dev).transpose(0, 1)

        self.o = buf(hq)
        self.lse = torch.empty(self.k, hq, chunk, dtype=torch.float32, device=dev)   # LSE_j dense [hq][c]
        self.dq = buf(hq)
        self.dkv = torch.empty(2, hkv, seq, d, dtype=torch.float32, device=dev)
        self.own = torch.empty(2, hkv, chunk, d, dtype=dtype, device=dev) if own_copies else None
        probe_q = self.o
        probe_k = buf(hkv)
        self.shape = ops.make_shape(probe_q, probe_k, chunk, softmax_scale, deterministic)
        # stage-1 forwards of chunks j >= 1 follow the previous chunk's forward, which neither
        # writes their inputs nor reads their outputs: SECO_FLAG_PREV_INDEPENDENT lets each one
        # start in its predecessor's last wave (programmatic dependent launch)
        self.shape_chain = ops.make_shape(probe_q, probe_k, chunk, softmax_scale, deterministic,
                                          prev_independent=True)
        self.ws = torch.empty(max(ops.seco_workspace_size(self.shape) // 4, 1), dtype=torch.float32, device=dev)

    # ---- per-chunk calls -------------------------------------------------------------
    def _lse(self, j):
        return self.lse[j]

    def lse_full(self):
        """LSE as [hq][S] (a copy)."""
        return self.lse.permute(1, 0, 2).reshape(self.hq, self.seq)

    def forward_chunk(self, q, k_cache, v_cache, j, stream=None, chained=False):
        """chained: the previous kernel on the stream is the previous chunk's stage-1 forward."""
        shape = self.shape_chain if chained else self.shape
        ops.seco_chunk_forward(shape, j, ops.chunk_view(q, self.shape, j), k_cache, v_cache,
                               ops.chunk_view(self.o, self.shape, j), self._lse(j), self.ws, stream)
        return ops.last_launch_count()

    def backward_chunk(self, q, k_cache, v_cache, do, j, relay_scale=1.0, grad_scale=1.0, stream=None):
        dk_own = self.own[0] if self.own is not None else None
        dv_own = self.own[1] if self.own is not None else None
        ops.seco_chunk_backward(self.shape, j, ops.chunk_view(q, self.shape, j), k_cache, v_cache,
                                ops.chunk_view(self.o, self.shape, j), ops.chunk_view(do, self.shape, j),
                                self._lse(j), relay_scale, grad_scale, self.dkv,
                                ops.chunk_view(self.dq, self.shape, j), dk_own, dv_own, self.ws, stream)
        return ops.last_launch_count()

    def skip_chunk(self, j, stream=None):
        """SpaCO chunk outside the sample (reading Z11), at its place in the descending walk."""
        dk_own = self.own[0] if self.own is not None else None
        dv_own = self.own[1] if self.own is not None else None
        ops.spaco_chunk_skip(self.shape, j, self.dkv, ops.chunk_view(self.dq, self.shape, j), dk_own, dv_own,
                             stream)
        return ops.last_launch_count()

    def plan(self, selected=None):
        """The step's chunk calls in the algorithm's order: [("f", j, chained) | ("b", j) |
        ("z", j)].  Stage 1: forward of every chunk, ascending (Alg. 1/2 lines 1-3).  Stage 2:
        j = k-1 .. 0; a selected j (default: all) is rebuilt (forward) and backpropagated with
        the relay (Alg. 1 lines 4-7; Alg. 2 lines 5-8), any other j is skipped (its gradients
        zero, its checkpoint gradient dropped: reading Z11)."""
        sel = set(range(self.k)) if selected is None else set(int(i) for i in selected)
        order = [("f", j, j > 0) for j in range(self.k)]
        for j in reversed(range(self.k)):
            order += [("f", j, False), ("b", j)] if j in sel else [("z", j)]
        return order

    def run(self, order, q, k_cache, v_cache, do, relay_scale=1.0, grad_scale=1.0, stream=None, events=None,
            nvtx=False):
        """Issue a plan on one stream (the checkpoint gradients start at zero: dkv is zeroed
        first).  events: optional per-call (start, end) CUDA event pairs; nvtx: one NVTX range
        per chunk call (for a profiler timeline).  Returns the number of kernel launches."""
        # checkpoint grads m'.grad start at zero each step (caller-owned buffer), zeroed on the
        # stream the chunk calls go to
        if stream is None:
            self.dkv.zero_()
        else:
            with torch.cuda.stream(stream):
                self.dkv.zero_()
        launches = 0
        for n, op in enumerate(order):
            if nvtx:
                torch.cuda.nvtx.range_push(f"{_CALL_NAMES[op[0]]} j={op[1]}")
            if events is not None:
                events[n][0].record(stream or torch.cuda.current_stream())
            if op[0] == "f":
                launches += self.forward_chunk(q, k_cache, v_cache, op[1], stream, chained=op[2])
            elif op[0] == "b":
                launches += self.backward_chunk(q, k_cache, v_cache, do, op[1], relay_scale, grad_scale, stream)
            else:
                launches += self.skip_chunk(op[1], stream)
            if events is not None:
                events[n][1].record(stream or torch.cuda.current_stream())
            if nvtx:
                torch.cuda.nvtx.range_pop()
        return launches

    # ---- whole steps ---------------------------------------------------------------
    def _check(self, q, k_cache, v_cache, do):
        for t, h in ((q, self.hq), (do, self.hq), (k_cache, self.hkv), (v_cache, self.hkv)):
            if t.shape != (h, self.seq, self.d) or t.dtype != self.dtype or t.device != self.device:
                raise ValueError("input tensor shape / dtype / device mismatch")
            want = (self.seq * self.d, self.d, 1) if self.layout == "hsd" else (self.d, h * self.d, 1)
            if t.stride() != want:
                raise ValueError(f"inputs must be {self.layout}-laid-out [heads][seq][d] (strides {want})")

    def step(self, q, k_cache, v_cache, do, selected=None, relay_scale=1.0, grad_scale=1.0, stream=None):
        """One SeCO (selected=None) or SpaCO step (selected = the sampled set I): plan() issued
        on one CUDA stream."""
        self._check(q, k_cache, v_cache, do)
        sel = sorted(set(range(self.k)) if selected is None else set(int(i) for i in selected), reverse=True)
        self.last_selected = sel
        launches = self.run(self.plan(selected), q, k_cache, v_cache, do, relay_scale, grad_scale, stream)
        if selected is None:
            fl = seco_step_flops(self.hq, self.d, self.seq, self.chunk)
        else:
            fl = spaco_step_flops(self.hq, self.d, self.seq, self.chunk, sel)
        return StepResult(sel, relay_scale, grad_scale, fl, launches)

    def seco_step(self, q, k_cache, v_cache, do, stream=None):
        return self.step(q, k_cache, v_cache, do, None, 1.0, 1.0, stream)

    def spaco_step(self, q, k_cache, v_cache, do, t, seed, cap=2.0, mode=ops._lib.SPACO_PAPER, stream=None):
        idx, gamma, s = ops.spaco_sample_and_scale(self.k, t, seed, cap, mode)
        r = self.step(q, k_cache, v_cache, do, idx, gamma, s, stream)
        r.selected, r.relay_scale, r.seed_scale = idx, gamma, s
        return r

    def memory_ledger(self):
        """Device bytes by role (the memory claim P:175-177, 'reduces the
        memory requirements for storing forward activations by a factor of k').  What scales
        with the sequence: the KV checkpoints (caller's), their fp32 gradient buffer dKV and
        the per-token inputs / outputs.  What a chunk call needs on top: the workspace and
        the chunk-j views of Q, O, dO, dQ, LSE -- O(c), independent of k (the library never
        allocates; tests/test_gpu_fullsize.py checks that a step allocates nothing)."""
        el = torch.finfo(self.dtype).bits // 8
        hq, hkv, S, c, d = self.hq, self.hkv, self.seq, self.chunk, self.d
        return {
            "kv_cache_bytes": 2 * hkv * S * d * el,                     # caller-owned checkpoints
            "dkv_fp32_bytes": self.dkv.numel() * 4,                       # persistent m'.grad
            "q_do_bytes": 2 * hq * S * d * el,                            # caller-owned inputs
            "o_dq_lse_bytes": (self.o.numel() + self.dq.numel()) * el + self.lse.numel() * 4,
            "per_call_chunk_bytes": 4 * hq * c * d * el + hq * c * 4,     # Q_j, O_j, dO_j, dQ_j, LSE_j (views)
            "per_call_workspace_bytes": self.ws.numel() * 4,
        }

    @property
    def dk(self):
        """Gradient of every chunk's own K after the last step (a view of dkv[0]): slot j is
        the total own-chunk gradient after chunk j's relay, and zero for a chunk a SpaCO step
        skipped (spaco_chunk_skip, reading Z11)."""
        return self.dkv[0]

    @property
    def dv(self):
        return self.dkv[1]

    def own_grads(self):
        """(dK, dV) of each chunk's own K/V after the last step (copies of dkv[0], dkv[1]:
        the library has already zeroed the slots of non-sampled chunks)."""
        return self.dkv[0].clone(), self.dkv[1].clone()
