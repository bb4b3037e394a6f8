"""TF/s of the tile kernel's generic contraction per operand majorness (dev tool)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17599_b200 as fce
M = N = K = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
torch.manual_seed(0)
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
At, Bt = A.t().contiguous(), B.t().contiguous()
ref = (A.float() @ B.float().t())
for a_mn, b_mn in [(0, 0), (0, 1), (1, 0), (1, 1)]:
    a = At if a_mn else A
    b = Bt if b_mn else B
    C = fce.gemm_bf16(a, b, a_mn, b_mn)
    err = ((C - ref).abs().max() / ref.abs().max()).item()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    for _ in range(2): fce.gemm_bf16(a, b, a_mn, b_mn, out=C)
    e0.record()
    for _ in range(5): fce.gemm_bf16(a, b, a_mn, b_mn, out=C)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"a_mn={a_mn} b_mn={b_mn} M=N=K={M}: {ms:.3f} ms  {2*M*N*K/ms/1e9:.0f} TF/s  err={err:.2e}", flush=True)
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(5): torch.matmul(A, B.t())
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"cuBLAS bf16 (bf16 out) {ms:.3f} ms {2*M*N*K/ms/1e9:.0f} TF/s")
