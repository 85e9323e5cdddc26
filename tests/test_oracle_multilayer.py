"""Pins for O9 (oracle/multilayer.py): the L-layer RoPE + LoRA attention stack and its exact
gradients, checked against things other than the oracle itself:
  * RoPE against complex multiplication (x1 + i x2) e^{i p theta_i) and its adjoint identity;
  * all gradients against torch autograd (float64, CPU) of the same model, whose attention
    is torch's scaled_dot_product_attention (an independent implementation);
  * directional central finite differences of the loss;
  * L = 1 with zero LoRA factors reduces to a single attention call (O1)."""
import numpy as np
import pytest
import torch

from oracle import attention as OA
from oracle import multilayer as OM
from synth import make_stack_inputs


def test_rope_is_complex_rotation():
    rng = np.random.default_rng(0)
    S, H, d = 9, 3, 16
    x = rng.standard_normal((S, H, d))
    pos = np.arange(S) * 7 + 3
    z = x[..., : d // 2] + 1j * x[..., d // 2:]
    theta = 10000.0 ** (-np.arange(d // 2) * 2.0 / d)
    zr = z * np.exp(1j * pos[:, None, None] * theta[None, None, :])
    want = np.concatenate([zr.real, zr.imag], axis=-1)
    assert np.abs(OM.rope(x, pos) - want).max() < 1e-12
    assert np.abs(OM.rope(x, np.zeros(S)) - x).max() == 0.0
    g = rng.standard_normal((S, H, d))
    assert abs((OM.rope(x, pos) * g).sum() - (x * OM.rope_bwd(g, pos)).sum()) < 1e-10   # adjoint
    assert np.abs(OM.rope(OM.rope_bwd(g, pos), pos) - g).max() < 1e-12                   # orthogonal


def _torch_grads(inp, hq, hkv, d):
    x0 = torch.tensor(inp.x0, dtype=torch.float64, requires_grad=True)
    params = [{k: torch.tensor(v, dtype=torch.float64, requires_grad=True) for k, v in p.items()}
              for p in inp.layers]
    S = x0.shape[0]
    half = d // 2
    inv = 10000.0 ** (-torch.arange(half, dtype=torch.float64) * 2.0 / d)
    ang = torch.arange(S, dtype=torch.float64)[:, None] * inv[None, :]
    cos, sin = torch.cos(ang)[:, None, :], torch.sin(ang)[:, None, :]

    def rope(t):
        t1, t2 = t[..., :half], t[..., half:]
        return torch.cat([t1 * cos - t2 * sin, t2 * cos + t1 * sin], dim=-1)

    x = x0
    for p in params:
        w = {n: p["W" + n] + p["A" + n] @ p["B" + n] for n in OM.PROJ}
        q = rope((x @ w["q"]).view(S, hq, d)).transpose(0, 1)
        k = rope((x @ w["k"]).view(S, hkv, d)).transpose(0, 1)
        v = (x @ w["v"]).view(S, hkv, d).transpose(0, 1)
        o = torch.nn.functional.scaled_dot_product_attention(q[None], k[None], v[None], is_causal=True,
                                                             enable_gqa=True)[0]
        x = x + o.transpose(0, 1).reshape(S, hq * d) @ w["o"]
    J = (x * torch.tensor(inp.G)).sum()
    J.backward()
    return [{k: t.grad.numpy() for k, t in p.items()} for p in params], x0.grad.numpy(), J.item()


@pytest.mark.parametrize("L,hq,hkv", [(1, 2, 1), (2, 4, 2), (3, 3, 3)])
def test_stack_grads_match_torch_autograd(L, hq, hkv):
    d, hd, r, S = 8, 12, 3, 20
    inp = make_stack_inputs(L, hd, hq, hkv, d, r, S, seed=L)
    grads, dx0 = OM.stack_grads(inp.x0, inp.layers, inp.G, hq, hkv, d)
    tg, tdx0, tJ = _torch_grads(inp, hq, hkv, d)
    assert abs(OM.stack_loss(inp.x0, inp.layers, inp.G, hq, hkv, d) - tJ) < 1e-9 * max(1.0, abs(tJ))
    assert np.abs(dx0 - tdx0).max() < 1e-10 * max(1.0, np.abs(tdx0).max())
    for g, t in zip(grads, tg):
        for key in t:
            assert np.abs(g[key] - t[key]).max() < 1e-10 * max(1.0, np.abs(t[key]).max()), key


def test_stack_grads_finite_differences():
    L, hq, hkv, d, hd, r, S = 2, 2, 1, 8, 8, 2, 12
    inp = make_stack_inputs(L, hd, hq, hkv, d, r, S, seed=7)
    grads, dx0 = OM.stack_grads(inp.x0, inp.layers, inp.G, hq, hkv, d)
    rng = np.random.default_rng(1)
    u = [{k: rng.standard_normal(v.shape) for k, v in p.items()} for p in inp.layers]
    ux = rng.standard_normal(inp.x0.shape)
    eps = 1e-6

    def J(sign):
        ls = [{k: p[k] + sign * eps * uu[k] for k in p} for p, uu in zip(inp.layers, u)]
        return OM.stack_loss(inp.x0 + sign * eps * ux, ls, inp.G, hq, hkv, d)

    fd = (J(+1) - J(-1)) / (2 * eps)
    an = sum((g[k] * uu[k]).sum() for g, uu in zip(grads, u) for k in g) + (dx0 * ux).sum()
    assert abs(fd - an) < 1e-6 * max(1.0, abs(an))


def test_single_layer_without_lora_is_one_attention():
    hq, hkv, d, hd, S = 2, 1, 8, 6, 10
    inp = make_stack_inputs(1, hd, hq, hkv, d, 2, S, seed=3)
    p = inp.layers[0]
    for n in OM.PROJ:
        p["A" + n] = np.zeros((p["W" + n].shape[0], 2))
    x = inp.x0
    pos = np.arange(S)
    q = OM.rope((x @ p["Wq"]).reshape(S, hq, d), pos).transpose(1, 0, 2)
    k = OM.rope((x @ p["Wk"]).reshape(S, hkv, d), pos).transpose(1, 0, 2)
    v = (x @ p["Wv"]).reshape(S, hkv, d).transpose(1, 0, 2)
    o, _ = OA.full_attn_fwd(q, k, v)
    want = x + o.transpose(1, 0, 2).reshape(S, hq * d) @ p["Wo"]
    assert np.abs(OM.stack_forward(x, [p], hq, hkv, d) - want).max() < 1e-12


def test_lora_grads_match_torch_autograd():
    rng = np.random.default_rng(4)
    rows, n_in, n_out, r = 37, 24, 20, 4
    x, dy = rng.standard_normal((rows, n_in)), rng.standard_normal((rows, n_out))
    A, B, W = rng.standard_normal((n_in, r)), rng.standard_normal((r, n_out)), rng.standard_normal((n_in, n_out))
    dA, dB, u = OM.lora_grads(x, dy, A, B)
    tx = torch.tensor(x, requires_grad=True)
    tA, tB = torch.tensor(A, requires_grad=True), torch.tensor(B, requires_grad=True)
    y = tx @ torch.tensor(W) + (tx @ tA) @ tB
    (y * torch.tensor(dy)).sum().backward()
    assert np.abs(dA - tA.grad.numpy()).max() < 1e-10
    assert np.abs(dB - tB.grad.numpy()).max() < 1e-10
    # dX = dY W^T + u A^T
    assert np.abs(dy @ W.T + u @ A.T - tx.grad.numpy()).max() < 1e-10
