import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17599_b200 as fce
def run(M, N, K, a_mn, b_mn, acc, it=5):
    A = torch.randn((K, M) if a_mn else (M, K), device="cuda").to(torch.bfloat16)
    B = torch.randn((K, N) if b_mn else (N, K), device="cuda").to(torch.bfloat16)
    C = torch.zeros(M if acc != 2 else 1, N, device="cuda")
    h = fce.default_handle(0)
    import ctypes
    def f():
        fce._check(h.lib.fce_gemm_bf16(h.raw, A.data_ptr(), A.stride(0), a_mn, B.data_ptr(), B.stride(0), b_mn, M, N, K, C.data_ptr(), C.stride(0), acc))
    f(); f()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(it): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / it
    print(f"M={M} N={N} K={K} a_mn={a_mn} b_mn={b_mn} acc={acc}: {ms:.3f} ms {2*M*N*K/ms/1e9:.0f} TF/s", flush=True)
import sys as _s
h0 = fce.default_handle(0)
h0.set_option("gemm_pair", int(_s.argv[1]) if len(_s.argv) > 1 else 1)
# correctness of the selected path against torch
for a_mn, b_mn in [(0, 0), (0, 1), (1, 0), (1, 1)]:
    M, N, K = 1000, 520, 700
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16); B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    C = fce.gemm_bf16(A.t().contiguous() if a_mn else A, B.t().contiguous() if b_mn else B, a_mn, b_mn)
    ref = A.float() @ B.float().t()
    print("check", a_mn, b_mn, ((C - ref).abs().max() / ref.abs().max()).item(), flush=True)
for acc in (2, 0, 1):
    run(8192, 8192, 8192, 0, 0, acc)
run(16384, 32768, 4096, 0, 0, 2)
run(16384, 32768, 4096, 1, 1, 2)
run(8192, 4096, 2048, 0, 1, 1)   # dH-like unit mix
run(2048, 4096, 8192, 1, 1, 0)   # dW-like
run(8192, 2048, 4096, 0, 0, 2)   # grad-like (no epilogue)
