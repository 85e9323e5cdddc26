"""Quick diagnostic run on a GPU box: prints parity errors per tensor instead of asserting."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from oracle import chunkwise as OC
from tests.gpu_util import err, host, inputs, upload
from paper_2505_16710_b200.step import ChunkedAttention


def run(hq, hkv, seq, d, c, dtype, peaky=False, fwd_only=False):
    x = inputs(hq, hkv, seq, d, seed=3, peaky=peaky, dtype=dtype)
    q, k, v, do = upload(x, dtype)
    L = ChunkedAttention(hq, hkv, d, seq, c, dtype=dtype)
    t0 = time.time()
    if fwd_only:
        L.dkv.zero_()
        for j in range(L.k):
            L.forward_chunk(q, k, v, j)
    else:
        L.seco_step(q, k, v, do)
    torch.cuda.synchronize()
    dt = time.time() - t0
    ref = OC.seco_step(x.q, x.k, x.v, x.do, [c] * (seq // c))
    out = dict(o=err(host(L.o), ref["o"]), lse=err(host(L.lse_full()), ref["lse"]))
    if not fwd_only:
        out.update(dq=err(host(L.dq), ref["dq"]), dk=err(host(L.dk), ref["dk"]), dv=err(host(L.dv), ref["dv"]))
    print(f"{dtype} hq={hq} hkv={hkv} S={seq} d={d} c={c} peaky={peaky} fwd_only={fwd_only} t={dt:.3f}s",
          {k_: f"{v_:.2e}" for k_, v_ in out.items()}, flush=True)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("all", "fp32"):
        run(2, 1, 64, 16, 16, torch.float32)
        run(4, 1, 1024, 64, 256, torch.float32)
    if what in ("all", "fwd"):
        run(8, 2, 512, 128, 128, torch.bfloat16, fwd_only=True)
        run(4, 1, 1024, 128, 256, torch.bfloat16, fwd_only=True)
        run(3, 1, 768, 128, 384, torch.bfloat16, fwd_only=True)
    if what in ("all", "bwd"):
        run(8, 2, 512, 128, 128, torch.bfloat16)
        run(4, 1, 1024, 128, 256, torch.bfloat16)
        run(4, 1, 1024, 128, 256, torch.bfloat16, peaky=True)
