"""Standalone tcgen05 complex GEMM micro-benchmark: C[b,m,n] = sum_k A[b,m,k] B[b,n,k].
Usage: python tools/run_gemm.py M N K [batch] [reps]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2002_01935_b200 import _native as nat
M, N, K = (int(x) for x in sys.argv[1:4])
B = int(sys.argv[4]) if len(sys.argv) > 4 else 1
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 5
lib = nat.load()
a = torch.randn(B, M, K, dtype=torch.complex64, device="cuda")
b = torch.randn(B, N, K, dtype=torch.complex64, device="cuda")
c = torch.empty(B, M, N, dtype=torch.complex64, device="cuda")
s = torch.cuda.Stream()
for r in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    nat.check(lib.tnx_gemm_c64(a.data_ptr(), b.data_ptr(), c.data_ptr(), B, M, N, K, 1, s.cuda_stream))
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
print(f"M={M} N={N} K={K} B={B}: {ms:.3f} ms incl. pack+alloc, {8*B*M*N*K/ms/1e9:.1f} TFLOP/s (8MNK)")
ref = torch.einsum("bmk,bnk->bmn", a.to(torch.complex128), b.to(torch.complex128))
err = ((c.to(torch.complex128) - ref).norm() / ref.norm()).item()
print("rel err", err)
