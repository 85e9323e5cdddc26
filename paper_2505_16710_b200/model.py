"""Multi-layer integration: an L-layer attention stack with RoPE and
LoRA-adapted projections trained chunk-wise with SeCO / SpaCO, the chunk attention of every
layer running in libseco.so.

The model is the one oracle/multilayer.py defines (reading Z18): per layer
    Q = rope(x W'_q), K = rope(x W'_k), V = x W'_v,  x <- x + attn(Q, K, V) W'_o,
    W'_p = W_p + A_p B_p (LoRA; W frozen, A and B trained), loss J = sum <x_L, G>.
The gradient reaches earlier chunks only through the KV caches (Eq. 2-3): chunk
j's backward in layer l deposits dK/dV into that layer's fp32 checkpoint-gradient buffer for
slots < j, and when chunk i is processed later (descending order) the relayed slot-i gradient
(`grad_hook`) is handed to autograd as the gradient of K_i, V_i of layer l, which
carries it through W'_k, W'_v into x_i of layer l and on into layer l-1 -- the multi-hop
chains of Eq. 3.

Torch does the base projections (library GEMMs, cuBLAS) and the autograd bookkeeping; every
attention forward / backward and every LoRA-gradient accumulation (SURVEY f2:
`seco_lora_grad`, fp32 per-layer buckets summed over the chunks of a step) is a libseco.so
call through the C ABI (ops.py).  A layer's bucket is final once the step's last chunk has
passed through it, and is handed to a `LayerBucketReducer` right then, so with several
data-parallel ranks its all_reduce overlaps the backward of the layers below.  The KV cache
is kept sequence-major ([S][Hkv][d], the projection output layout) and Q/O/dO/dQ of a chunk
are [c][Hq][d] -- the ABI's strided layouts, no transposes.
"""
from __future__ import annotations

import torch

from . import _lib, ops
from .parallel import LayerBucketReducer

_DT = {torch.bfloat16: _lib.SECO_BF16, torch.float32: _lib.SECO_FP32_DEBUG}
PROJ = ("q", "k", "v", "o")


class _LayerState:
    """Per-layer buffers: KV cache (the checkpoints m_j), LSE per chunk, the fp32
    checkpoint-gradient buffer dKV (m'.grad), workspace."""

    def __init__(self, hq, hkv, d, seq, chunk, dtype, device, deterministic):
        k = seq // chunk
        self.chunk = chunk
        self.k_cache = torch.zeros(seq, hkv, d, dtype=dtype, device=device)
        self.v_cache = torch.zeros(seq, hkv, d, dtype=dtype, device=device)
        self.lse = torch.empty(k, hq, chunk, dtype=torch.float32, device=device)
        self.dkv = torch.zeros(2, hkv, seq, d, dtype=torch.float32, device=device)
        self.own = torch.empty(2, hkv, chunk, d, dtype=dtype, device=device)    # dk_own / dv_own
        self.shape = _lib.SecoShape(hq, hkv, d, chunk, k, 0.0, _DT[dtype], d, hq * d, d, hkv * d,
                                    _lib.SECO_FLAG_DETERMINISTIC if deterministic else 0)
        self.ws = torch.empty(max(ops.seco_workspace_size(self.shape) // 4, 1), dtype=torch.float32,
                              device=device)


class _ChunkAttention(torch.autograd.Function):
    """O_j = attn(Q_j; K/V slots 0..j) with libseco.so; backward = the chunk-local backward
    with relay (Alg. 1 lines 6-7 / Alg. 2 line 6): returns dQ_j and, as the gradient of
    K_j, V_j, the layer's checkpoint-gradient slot j after the call (gamma x deposits of
    later chunks + this chunk's own share)."""

    @staticmethod
    def forward(ctx, q, k, v, st, j, relay):
        o = torch.empty_like(q)
        ops.seco_chunk_forward(st.shape, j, q, st.k_cache, st.v_cache, o, st.lse[j], st.ws)
        ctx.save_for_backward(q, o)
        ctx.st, ctx.j, ctx.relay = st, j, relay
        return o

    @staticmethod
    def backward(ctx, do):
        q, o = ctx.saved_tensors
        st, j = ctx.st, ctx.j
        do = do.contiguous()
        dq = torch.empty_like(q)
        ops.seco_chunk_backward(st.shape, j, q, st.k_cache, st.v_cache, o, do, st.lse[j], ctx.relay, 1.0,
                                st.dkv, dq, st.own[0], st.own[1], st.ws)
        # dk_own / dv_own: slot j of dKV after the relay, converted by the library ([hkv][c][d]);
        # autograd takes them as the gradients of K_j, V_j ([c][hkv][d] views)
        return dq, st.own[0].transpose(0, 1), st.own[1].transpose(0, 1), None, None, None


class _LoRAProj(torch.autograd.Function):
    """Y = X W + (X A) B.  Backward: dA, dB accumulate in fp32 into the layer's bucket via
    seco_lora_grad (which also returns u = dY B^T); dX = dY W^T + u A^T (cuBLAS)."""

    @staticmethod
    def forward(ctx, x, W, A, B, model, li, name):
        ctx.save_for_backward(x, W, A, B)
        ctx.model, ctx.li, ctx.name = model, li, name
        return x @ W + (x @ A) @ B

    @staticmethod
    def backward(ctx, dy):
        x, W, A, B = ctx.saved_tensors
        m, li, name = ctx.model, ctx.li, ctx.name
        dy = dy.contiguous()
        u = torch.empty(x.shape[0], A.shape[1], dtype=torch.float32, device=x.device)
        shape = ops.lora_shape(x, dy, A.shape[1], deterministic=m.deterministic)
        ws = m._lora_ws(ops.seco_lora_workspace_size(shape))
        dA, dB = m.lora_views[li]["A" + name], m.lora_views[li]["B" + name]
        ops.seco_lora_grad(shape, x, dy, A, B, dA, dB, u, ws)
        dx = dy @ W.t() + u.to(x.dtype) @ A.t()
        m._lora_done(li)
        return dx, None, None, None, None, None, None


class ChunkedLoRAStack:
    """L attention blocks; `params[l]` holds W_p (frozen) and A_p, B_p (trainable leaves)."""

    def __init__(self, layers, hq, hkv, d, seq, chunk, dtype=torch.bfloat16, device="cuda",
                 deterministic=False, rope_base=10000.0):
        if seq % chunk:
            raise ValueError("seq must be a multiple of chunk")
        self.hq, self.hkv, self.d, self.seq, self.chunk, self.k = hq, hkv, d, seq, chunk, seq // chunk
        self.dtype = dtype
        self.device = torch.device(device)
        self.params = []
        for p in layers:
            t = {}
            for name, val in p.items():
                t[name] = torch.as_tensor(val).contiguous().to(device=self.device, dtype=dtype)
            self.params.append(t)
        # fp32 LoRA-gradient bucket per layer (views dA_p [n_in][r], dB_p [r][n_out])
        self.buckets, self.lora_views = [], []
        for t in self.params:
            sizes = [t[ab + n].numel() for n in PROJ for ab in "AB"]
            bucket = torch.zeros(sum(sizes), dtype=torch.float32, device=self.device)
            views, off = {}, 0
            for n in PROJ:
                for ab in "AB":
                    num = t[ab + n].numel()
                    views[ab + n] = bucket[off:off + num].view(t[ab + n].shape)
                    off += num
            self.buckets.append(bucket)
            self.lora_views.append(views)
        self._ws = torch.empty(0, dtype=torch.float32, device=self.device)
        self.reducer = LayerBucketReducer()
        self._final_chunk = False
        self._pending = [0] * len(self.params)
        self.deterministic = deterministic
        self.state = [_LayerState(hq, hkv, d, seq, chunk, dtype, self.device, deterministic) for _ in layers]
        half = d // 2
        inv = rope_base ** (-torch.arange(half, dtype=torch.float64) * 2.0 / d)
        ang = torch.arange(seq, dtype=torch.float64)[:, None] * inv[None, :]
        self.cos = torch.cos(ang).to(self.device, torch.float32)[:, None, :]    # [S][1][d/2]
        self.sin = torch.sin(ang).to(self.device, torch.float32)[:, None, :]

    # ------------------------------------------------------------------ pieces
    def _rope(self, t, j):
        c, half = self.chunk, self.d // 2
        cos, sin = self.cos[j * c:(j + 1) * c], self.sin[j * c:(j + 1) * c]
        tf = t.float()
        t1, t2 = tf[..., :half], tf[..., half:]
        return torch.cat([t1 * cos - t2 * sin, t2 * cos + t1 * sin], dim=-1).to(self.dtype)

    def _proj(self, x, p, n, li=None):
        if li is None:                                     # no graph (stage 1)
            return x @ p["W" + n] + (x @ p["A" + n]) @ p["B" + n]
        return _LoRAProj.apply(x, p["W" + n], p["A" + n], p["B" + n], self, li, n)

    def _lora_ws(self, nbytes):
        if self._ws.numel() * 4 < nbytes:
            self._ws = torch.empty((nbytes + 3) // 4, dtype=torch.float32, device=self.device)
        return self._ws

    def _lora_done(self, li):
        """Called after each LoRA accumulation; on the step's last chunk, the fourth one of a
        layer makes its bucket final."""
        if self._final_chunk:
            self._pending[li] -= 1
            if self._pending[li] == 0:
                self.reducer.layer_final(li, self.buckets[li])

    def _block(self, li, x, j, relay, grad):
        p, st, c = self.params[li], self.state[li], self.chunk
        gl = li if grad else None
        q = self._rope(self._proj(x, p, "q", gl).view(c, self.hq, self.d), j).contiguous()
        k = self._rope(self._proj(x, p, "k", gl).view(c, self.hkv, self.d), j).contiguous()
        v = self._proj(x, p, "v", gl).view(c, self.hkv, self.d).contiguous()
        st.k_cache[j * c:(j + 1) * c].copy_(k.detach())         # checkpoint m_j of this layer
        st.v_cache[j * c:(j + 1) * c].copy_(v.detach())
        if grad:
            o = _ChunkAttention.apply(q, k, v, st, j, relay)
        else:
            o = torch.empty_like(q)
            ops.seco_chunk_forward(st.shape, j, q, st.k_cache, st.v_cache, o, st.lse[j], st.ws)
        return x + self._proj(o.view(c, self.hq * self.d), p, "o", gl)

    # ------------------------------------------------------------------ steps
    def step(self, x0, G, selected=None, relay_scale=1.0, seed_scale=1.0):
        """One SeCO (selected=None) or SpaCO step (selected = sampled chunk indices, Alg. 2):
        stage 1 forwards every chunk through all layers (no graph); stage 2 rebuilds each
        selected chunk, descending, and backpropagates J_j * seed_scale, relaying through the
        per-layer checkpoint gradients with relay_scale.  Returns dJ/dx0 (zero rows for chunks
        not processed); the LoRA gradients (fp32) are in lora_views / buckets, and their
        all_reduce over data-parallel ranks (if any) has completed when this returns."""
        c = self.chunk
        x0 = x0.to(self.device, self.dtype)
        G = G.to(self.device, torch.float32)
        for st in self.state:
            st.dkv.zero_()
        for b in self.buckets:
            b.zero_()
        sel = list(range(self.k)) if selected is None else sorted(set(int(i) for i in selected))
        with torch.no_grad():
            for j in range(self.k):                                    # stage 1 (Alg. 1 lines 1-3)
                x = x0[j * c:(j + 1) * c]
                for li in range(len(self.params)):
                    x = self._block(li, x, j, 1.0, grad=False)
        dx0 = torch.zeros_like(x0)
        self._pending = [len(PROJ)] * len(self.params)
        for j in reversed(sel):                                        # stage 2, descending
            self._final_chunk = j == sel[0]
            xin = x0[j * c:(j + 1) * c].detach().clone().requires_grad_(True)
            x = xin
            for li in range(len(self.params)):
                x = self._block(li, x, j, relay_scale, grad=True)
            loss = (x.float() * G[j * c:(j + 1) * c]).sum() * seed_scale
            loss.backward()
            dx0[j * c:(j + 1) * c] = xin.grad
        self._final_chunk = False
        if not sel:
            # an empty sample (possible with SPACO_BERNOULLI): no chunk finished any layer, but
            # every rank must still send every layer's (zero) bucket, top-down like a
            # non-empty step, or the ranks that did sample chunks would wait forever
            for li in reversed(range(len(self.params))):
                self.reducer.layer_final(li, self.buckets[li])
        self.reducer.wait()
        return dx0

    def lora_grads(self):
        """{(layer, 'A'+p / 'B'+p): grad} as float64 CPU arrays (result extraction)."""
        return {(li, key): v.double().cpu().numpy() for li, views in enumerate(self.lora_views)
                for key, v in views.items()}
