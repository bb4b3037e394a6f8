import os, sys, torch, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17599_b200 as fce
h = fce.default_handle(0)
def run(M, N, K, a_mn, b_mn, acc, pair=1, it=5):
    h.set_option("gemm_pair", pair)
    A = torch.randn((K, M) if a_mn else (M, K), device="cuda").to(torch.bfloat16)
    B = torch.randn((K, N) if b_mn else (N, K), device="cuda").to(torch.bfloat16)
    C = torch.zeros(M if acc != 2 else 1, N, device="cuda")
    def f():
        fce._check(h.lib.fce_gemm_bf16(h.raw, A.data_ptr(), A.stride(0), a_mn, B.data_ptr(), B.stride(0), b_mn, M, N, K, C.data_ptr(), C.stride(0), acc))
    f(); f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(it): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / it
    print(f"pair={pair} M={M} N={N} K={K} a_mn={a_mn} b_mn={b_mn} acc={acc}: {ms:.3f} ms {2*M*N*K/ms/1e9:.0f} TF/s", flush=True)
run(8192, 8192, 8192, 0, 0, 2)
run(8192, 8192, 8192, 0, 0, 0)
run(16384, 32768, 4096, 0, 0, 2)
run(16384, 65536, 4096, 0, 0, 2)
run(16384, 32768, 4096, 1, 1, 2)
run(16384, 32768, 4096, 0, 1, 2)
