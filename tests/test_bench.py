"""bench.py contract: one JSON line per run with the keys the driver reads, the
reference arm under torchrun (rank 0 prints, the other ranks exit 0), and the
native vocab-parallel (NCCL) path of the GPU arm under torchrun."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _json_lines(out: str):
    return [json.loads(l) for l in out.splitlines() if l.strip().startswith("{")]


def _torchrun(nproc: int, port: int, *args, timeout=600):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "bench.py"), *args]
    return subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout)


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "small",
                        "--steps", "1", "--warmup", "0"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = _json_lines(r.stdout)
    assert len(lines) == 1
    d = lines[0]
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["unit"] == "tokens/s"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1


def test_reference_arm_under_torchrun_prints_once():
    r = _torchrun(2, 29561, "--impl", "reference", "--gpus", "2", "--config", "small", "--steps", "1",
                  "--warmup", "0")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1 and lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2


@pytest.mark.gpu
def test_gpu_arm_native_vocab_parallel_under_torchrun(cuda):
    """The path `bench.py --gpus N` takes under torchrun (NCCL communicator,
    fce_vp_forward / fce_vp_backward), on one rank."""
    r = _torchrun(1, 29563, "--gpus", "1", "--force-vp", "--config", "small", "--steps", "2", "--warmup", "3",
                  "--e2e-steps", "2", "--no-cpu-baseline")
    assert r.returncode == 0, r.stderr[-3000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1
    d = lines[0]
    assert BASE_KEYS <= set(d) and {"roofline", "clocks", "gpu_launches"} <= set(d)
    assert d["config"]["parallelism"].startswith("vocab-parallel x1 (NCCL")
    assert d["gpu_launches"] > 0 and d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    # same loss as the single-GPU path on the same seeded instance
    r1 = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "small", "--steps", "2",
                         "--warmup", "3", "--e2e-steps", "2", "--no-cpu-baseline"], cwd=ROOT, capture_output=True,
                        text=True, timeout=600)
    assert r1.returncode == 0, r1.stderr[-3000:]
    d1 = _json_lines(r1.stdout)[0]
    assert abs(d["loss"] - d1["loss"]) <= 1e-6 * abs(d1["loss"])


@pytest.mark.gpu
def test_gpu_arm_self_launches_k_ranks_without_torchrun(cuda):
    """`bench.py --gpus 3` launched plainly on a box with fewer GPUs runs the 3
    ranks of the vocab-parallel path in-process (local transport) and prints
    one JSON line whose loss equals the single-GPU path's."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "3", "--config", "small",
                        "--steps", "2", "--warmup", "3", "--e2e-steps", "2", "--no-cpu-baseline"], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1
    d = lines[0]
    assert BASE_KEYS <= set(d) and d["config"]["ranks"] == 3
    assert "local transport" in d["config"]["parallelism"]
    assert d["e2e_with_grads"]["d2h_bytes_per_step"] > d["e2e"]["d2h_bytes_per_step"]
    r1 = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "small", "--steps", "2",
                         "--warmup", "3", "--e2e-steps", "2", "--no-cpu-baseline"], cwd=ROOT, capture_output=True,
                        text=True, timeout=600)
    assert r1.returncode == 0, r1.stderr[-3000:]
    d1 = _json_lines(r1.stdout)[0]
    assert abs(d["loss"] - d1["loss"]) <= 1e-5 * abs(d1["loss"])


def test_cpu_baseline_fit_is_the_marginal_cost():
    sys.path.insert(0, ROOT)
    import bench
    alpha, beta = bench._fit([(16, 10.0), (208, 14.8), (16, 10.2), (208, 15.0)])
    assert abs(beta - 0.025) < 1e-9 and abs(alpha - (10.1 - 0.025 * 16)) < 1e-9


@pytest.mark.gpu
def test_gpu_arm_ipc_transport_processes(cuda):
    """`bench.py --gpus 2 --transport ipc`: two processes (torch.distributed.run,
    gloo for the launcher's barrier) sharing this GPU, vocab-parallel over
    libfce's own IPC collectives; one JSON line, the single-GPU loss."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--transport", "ipc",
                        "--config", "small", "--steps", "2", "--warmup", "3", "--e2e-steps", "2", "--no-cpu-baseline",
                        "--no-e2e-grads"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1
    d = lines[0]
    assert d["config"]["ranks"] == 2 and "IPC transport" in d["config"]["parallelism"]
    r1 = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "small", "--steps", "2",
                         "--warmup", "3", "--e2e-steps", "2", "--no-cpu-baseline", "--no-e2e-grads", "--no-dropin"],
                        cwd=ROOT, capture_output=True, text=True, timeout=600)
    d1 = _json_lines(r1.stdout)[0]
    assert abs(d["loss"] - d1["loss"]) <= 1e-5 * abs(d1["loss"])


def test_committed_traffic_matches_the_sources():
    """profiles/traffic.json (ncu --set full DRAM bytes per launch) must have been
    captured on the current csrc/*: otherwise bench.py would report no traffic."""
    sys.path.insert(0, ROOT)
    import bench
    for cfg in ("llama3-8b", "qwen2.5-7b", "gemma2-2b"):
        for kernel in ("fce_fwd_sm100", "fce_bwd_persistent_sm100"):
            t = bench._traffic_from_profile(cfg, kernel)
            assert t is not None and t["bytes"] > 0, (cfg, kernel)
