"""Systematic (round-toward-zero) bias of the tcgen05 complex GEMM.

    TNX_GEMM_PROMOTE=3 python tools/gemm_bias.py [M N K]

Prints one JSON line: the bias b = Re<r, g - r> / <r, r> (a uniform relative
shrink of the result shows up as b < 0), the residual normwise error once the
bias is removed, and the plain normwise error, for random CN(0,1) operands
against a complex128 reference.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2002_01935_b200 import _native as nat  # noqa: E402


def main():
    M, N, K = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (2048, 2048, 4096)
    lib = nat.load()
    g = torch.Generator(device="cuda").manual_seed(0)
    a = torch.randn(1, M, K, dtype=torch.complex64, device="cuda", generator=g)
    b = torch.randn(1, N, K, dtype=torch.complex64, device="cuda", generator=g)
    c = torch.empty(1, M, N, dtype=torch.complex64, device="cuda")
    s = torch.cuda.Stream()
    prec = int(os.environ.get("PREC", "1"))  # 1 = 3xtf32, 2 = tf32-bf16x
    nat.check(lib.tnx_gemm_c64(a.data_ptr(), b.data_ptr(), c.data_ptr(), 1, M, N, K, prec, s.cuda_stream))
    torch.cuda.synchronize()
    ref = torch.einsum("bmk,bnk->bmn", a.to(torch.complex128), b.to(torch.complex128))
    d = c.to(torch.complex128) - ref
    rr = (ref.abs() ** 2).sum().item()
    bias = (ref.conj() * d).sum().real.item() / rr
    resid = (d - bias * ref).norm().item() / ref.norm().item()
    out = {"M": M, "N": N, "K": K, "prec": prec, "env": {k: v for k, v in os.environ.items() if k.startswith("TNX_")},
           "bias": bias, "resid": resid, "err": d.norm().item() / ref.norm().item()}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
