"""Multi-layer integration on the GPU: an L-layer RoPE + LoRA attention
stack trained chunk-wise (paper_2505_16710_b200/model.py, attention through the C ABI)
against the exact full-sequence gradients of oracle/multilayer.py (O9):
  * SeCO = full-sequence backward (SeCO is exact), fp32 debug kernels and bf16;
  * SpaCO with independent Bernoulli(rho) selection and s = gamma = 1/rho is unbiased at any
    depth (reading Z7): the probability-weighted sum over all 2^k selections equals SeCO --
    the multi-hop chains of Eq. 3 across 2 layers included;
  * SpaCO selecting every chunk with gamma = s = 1 reproduces SeCO bit for bit
    (deterministic mode)."""
import itertools

import numpy as np
import pytest
import torch

from oracle import multilayer as OM
from synth import make_stack_inputs
from tests.gpu_util import BF16_TOL, err

pytestmark = pytest.mark.gpu


def _stack(inp, hq, hkv, d, S, c, dtype, deterministic=False):
    from paper_2505_16710_b200.model import ChunkedLoRAStack
    return ChunkedLoRAStack(inp.layers, hq, hkv, d, S, c, dtype=dtype, deterministic=deterministic)


def _inputs(inp, dtype):
    return torch.tensor(inp.x0, dtype=dtype), torch.tensor(inp.G, dtype=torch.float32)


def _check(model, dx0, inp, hq, hkv, d, tol):
    grads, rdx0 = OM.stack_grads(inp.x0, inp.layers, inp.G, hq, hkv, d)
    got = model.lora_grads()
    worst = 0.0
    for li, g in enumerate(grads):
        for n in OM.PROJ:
            for ab in "AB":
                e = err(got[(li, ab + n)], g[ab + n])
                worst = max(worst, e)
                assert e <= tol, (li, ab + n, e)
    e = err(dx0.double().cpu().numpy(), rdx0)
    assert e <= tol, ("dx0", e)
    return max(worst, e)


@pytest.fixture(autouse=True)
def _no_tf32():
    old = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    yield
    torch.backends.cuda.matmul.allow_tf32 = old


@pytest.mark.parametrize("L,hq,hkv,d,hd,S,c", [(2, 4, 2, 16, 32, 64, 16), (3, 2, 1, 32, 48, 96, 32)])
def test_fp32_seco_stack_matches_full_gradient(L, hq, hkv, d, hd, S, c):
    inp = make_stack_inputs(L, hd, hq, hkv, d, 4, S, seed=L)
    model = _stack(inp, hq, hkv, d, S, c, torch.float32)
    x0, G = _inputs(inp, torch.float32)
    dx0 = model.step(x0, G)
    torch.cuda.synchronize()
    _check(model, dx0, inp, hq, hkv, d, 1e-4)
    assert model.reducer.sent == list(reversed(range(L)))   # buckets final top-down on the last chunk


@pytest.mark.parametrize("d,S,c", [(64, 512, 128), (128, 512, 128), (128, 600, 200)])
def test_bf16_seco_stack_matches_full_gradient(d, S, c):
    L, hq, hkv, hd = 2, 4, 2, 128                    # c = 200: ragged chunks through the stack
    inp = make_stack_inputs(L, hd, hq, hkv, d, 8, S, seed=11, bf16=True)
    model = _stack(inp, hq, hkv, d, S, c, torch.bfloat16)
    x0, G = _inputs(inp, torch.bfloat16)
    dx0 = model.step(x0, G)
    torch.cuda.synchronize()
    _check(model, dx0, inp, hq, hkv, d, BF16_TOL)    # north-star 2e-2; measured worst 1.1e-2 (two bf16 layers)


def test_fp32_spaco_bernoulli_unbiased_across_layers():
    L, hq, hkv, d, hd, S, c = 2, 2, 1, 16, 24, 64, 16
    k, rho = S // c, 0.5
    inp = make_stack_inputs(L, hd, hq, hkv, d, 4, S, seed=5)
    model = _stack(inp, hq, hkv, d, S, c, torch.float32)
    x0, G = _inputs(inp, torch.float32)
    model.step(x0, G)
    seco = model.lora_grads()
    mean = {key: np.zeros_like(v) for key, v in seco.items()}
    for n in range(k + 1):
        for sel in itertools.combinations(range(k), n):
            w = rho ** n * (1 - rho) ** (k - n)
            model.reducer.sent.clear()
            dx0 = model.step(x0, G, selected=sel, relay_scale=1 / rho, seed_scale=1 / rho)
            # every layer's bucket is sent once per step, top-down, even for an empty sample
            assert model.reducer.sent == list(reversed(range(L)))
            if n == 0:                         # no chunk selected: zero gradient
                torch.cuda.synchronize()
                assert float(dx0.abs().max()) == 0.0
                assert all(np.abs(v).max() == 0.0 for v in model.lora_grads().values())
            for key, v in model.lora_grads().items():
                mean[key] += w * v
    torch.cuda.synchronize()
    for key in seco:
        assert err(mean[key], seco[key]) <= 1e-4, key


def test_bf16_spaco_all_chunks_is_seco():
    L, hq, hkv, d, hd, S, c = 2, 4, 2, 64, 128, 512, 128
    inp = make_stack_inputs(L, hd, hq, hkv, d, 8, S, seed=2, bf16=True)
    model = _stack(inp, hq, hkv, d, S, c, torch.bfloat16, deterministic=True)
    x0, G = _inputs(inp, torch.bfloat16)
    a = model.step(x0, G).clone()
    ga = model.lora_grads()
    b = model.step(x0, G, selected=list(range(S // c)), relay_scale=1.0, seed_scale=1.0)
    gb = model.lora_grads()
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    for key in ga:
        assert np.array_equal(ga[key], gb[key]), key


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("rows,n_in,n_out,r", [(512, 256, 384, 8), (129, 72, 40, 4), (2048, 1024, 1024, 16),
                                              (2048, 4096, 1024, 8), (300, 1024, 512, 4), (64, 256, 256, 1),
                                              (17, 512, 2048, 2), (4001, 4096, 4096, 8), (256, 4096, 8192, 8),
                                              (40, 128, 4096, 16)])
@pytest.mark.parametrize("det", [False, True])
def test_lora_grad_kernel_matches_oracle(dtype, rows, n_in, n_out, r, det):
    """seco_lora_grad against oracle.multilayer.lora_grads: dA, dB accumulate (two
    calls give twice the gradient), u = dY B^T; X is a strided view (padded rows).  bf16 with
    n_in, n_out multiples of 128 up to 4096 takes the fused persistent kernel (ragged row counts
    and fewer row blocks than clusters included), bf16 multiples of 256 beyond that the two-pass
    tensor-core kernels (4096 -> 8192), everything else the CUDA-core ones."""
    from paper_2505_16710_b200 import ops
    from synth import round_to_bf16
    rng = np.random.default_rng(rows + r)

    def draw(shape):
        a = rng.standard_normal(shape).astype(np.float32)
        return round_to_bf16(a) if dtype == torch.bfloat16 else a

    x_np, dy_np, a_np, b_np = draw((rows, n_in)), draw((rows, n_out)), draw((n_in, r)), draw((r, n_out))
    xpad = torch.zeros(rows, n_in + 8, dtype=dtype, device="cuda")
    xpad[:, :n_in] = torch.from_numpy(x_np).to(dtype)
    x = xpad[:, :n_in]
    dy = torch.from_numpy(dy_np).to("cuda", dtype)
    a = torch.from_numpy(a_np).to("cuda", dtype)
    b = torch.from_numpy(b_np).to("cuda", dtype)
    da = torch.zeros(n_in, r, device="cuda")
    db = torch.zeros(r, n_out, device="cuda")
    u = torch.empty(rows, r, device="cuda")
    shape = ops.lora_shape(x, dy, r, deterministic=det)
    ws = torch.empty(ops.seco_lora_workspace_size(shape) // 4, device="cuda")
    for _ in range(2):
        ops.seco_lora_grad(shape, x, dy, a, b, da, db, u, ws)
    torch.cuda.synchronize()
    if det:   # fixed summation order: a repeat from zero reproduces the first call bit for bit
        da1, db1 = torch.zeros_like(da), torch.zeros_like(db)
        ops.seco_lora_grad(shape, x, dy, a, b, da1, db1, u, ws)
        da2, db2 = torch.zeros_like(da), torch.zeros_like(db)
        ops.seco_lora_grad(shape, x, dy, a, b, da2, db2, u, ws)
        assert torch.equal(da1, da2) and torch.equal(db1, db2)
    rdA, rdB, ru = (np.asarray(t) for t in __import__("oracle").multilayer.lora_grads(x_np, dy_np, a_np, b_np))
    assert err(da.cpu().numpy(), 2 * rdA) <= 1e-5
    assert err(db.cpu().numpy(), 2 * rdB) <= 1e-5
    assert err(u.cpu().numpy(), ru) <= 1e-5
