"""Helpers for the GPU parity tests: upload synth inputs, run steps through the
C ABI, compare against the oracle with the north-star error metric
(reading Z13: err = max|X_gpu - X_ref| / max|X_ref| per tensor)."""
import numpy as np
import torch

from synth import make_inputs

BF16_TOL = 2e-2     # north star: max relative error <= 2e-2 in bf16
FP32_TOL = 1e-4     # north star: <= 1e-4 in the fp32 debug build


def err(gpu, ref):
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.abs(gpu - ref).max() / max(np.abs(ref).max(), 1e-30))


def to_dev(x, bits, dtype):
    if dtype == torch.bfloat16:
        return torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16).cuda()
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def upload(x, dtype):
    return tuple(to_dev(a, b, dtype) for a, b in ((x.q, x.q_bits), (x.k, x.k_bits), (x.v, x.v_bits),
                                                  (x.do, x.do_bits)))


def host(t):
    return t.float().cpu().numpy()


def inputs(hq, hkv, seq, d, seed=0, peaky=False, dtype=torch.bfloat16):
    return make_inputs(hq, hkv, seq, d, seed=seed, peaky=peaky, bf16=(dtype == torch.bfloat16))
