import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17599_b200 as fce
h = fce.default_handle(0)
M, N, K = 16384, 32768, 4096
for a_mn, b_mn in [(0, 0), (1, 0), (0, 1), (1, 1)]:
    A = torch.randn((K, M) if a_mn else (M, K), device="cuda").to(torch.bfloat16)
    B = torch.randn((K, N) if b_mn else (N, K), device="cuda").to(torch.bfloat16)
    C = torch.zeros(1, N, device="cuda")
    def f():
        fce._check(h.lib.fce_gemm_bf16(h.raw, A.data_ptr(), A.stride(0), a_mn, B.data_ptr(), B.stride(0), b_mn, M, N, K, C.data_ptr(), C.stride(0), 2))
    for _ in range(2): f()
    torch.cuda.synchronize()
    if len(sys.argv) > 1: torch.cuda.cudart().cudaProfilerStart()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); f(); e1.record(); torch.cuda.synchronize()
    if len(sys.argv) > 1: torch.cuda.cudart().cudaProfilerStop()
    ms = e0.elapsed_time(e1)
    print(f"a_mn={a_mn} b_mn={b_mn}: {ms:.3f} ms {2*M*N*K/ms/1e9:.0f} TF/s", flush=True)
