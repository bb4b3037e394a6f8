"""Per-clock efficiency of the contraction kernels (dev tool): each variant runs
~1.5 s while nvidia-smi samples the SM clock; reports TF/s and % of the
tensor peak at the observed clock (148 SMs x 8192 flop/clk)."""
import os, subprocess, statistics, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17599_b200 as fce
h = fce.default_handle(0)
M, N, K = 16384, 16384, 4096

def sample(fn, seconds=1.5):
    f = open("/tmp/clk.csv", "w")
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits", "-lms", "50"], stdout=f)
    time.sleep(0.2)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    n = 0
    e0.record()
    t0 = time.time()
    while time.time() - t0 < seconds:
        fn(); n += 1
        if n % 10 == 0: torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    p.terminate(); p.wait(); f.close()
    clks = [float(x) for x in open("/tmp/clk.csv").read().split() if x.strip()]
    clk = statistics.median(clks[len(clks)//4:]) if clks else float("nan")
    return e0.elapsed_time(e1) / n, clk

for pair, a_mn, b_mn in [(1, 0, 0), (1, 0, 1), (1, 1, 1), (0, 0, 0), (0, 0, 1), (1, 0, 0)]:
    h.set_option("gemm_pair", pair)
    A = torch.randn((K, M) if a_mn else (M, K), device="cuda").to(torch.bfloat16)
    B = torch.randn((K, N) if b_mn else (N, K), device="cuda").to(torch.bfloat16)
    C = torch.zeros(1, N, device="cuda")
    def f():
        fce._check(h.lib.fce_gemm_bf16(h.raw, A.data_ptr(), A.stride(0), a_mn, B.data_ptr(), B.stride(0), b_mn, M, N, K, C.data_ptr(), C.stride(0), 2))
    f(); torch.cuda.synchronize()
    ms, clk = sample(f)
    tf = 2 * M * N * K / ms / 1e9
    peak = 148 * 8192 * clk * 1e6 / 1e12
    print(f"pair={pair} a_mn={a_mn} b_mn={b_mn}: {ms:.3f} ms {tf:.0f} TF/s at {clk:.0f} MHz -> {100*tf/peak:.1f}% of clock peak", flush=True)
    del A, B
