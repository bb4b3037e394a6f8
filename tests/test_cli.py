"""The fusedce-style CLI (reference tests/test_cli.cpp): exit codes, verify
suites, bench CSV schema (bench.cpp:200-211)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(*args):
    return subprocess.run([sys.executable, "-m", "paper_2511_17599_b200.cli", *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=600)


def test_usage_errors_exit_2():
    assert run().returncode == 2
    assert run("bench", "--methods", "bogus").returncode == 2
    assert run("--help").returncode == 0


@pytest.mark.gpu
def test_verify_passes(cuda):
    r = run("verify", "--loss-instances", "12", "--grad-instances", "4")
    assert r.returncode == 0, r.stdout + r.stderr
    for suite in ("loss_equivalence", "gradient_recompute", "window_sweep", "shard_invariance", "stability",
                  "vocab_parallel_ranks"):
        assert suite in r.stdout
    assert "overall: PASS" in r.stdout


@pytest.mark.gpu
def test_bench_csv_schema(cuda, tmp_path):
    out = tmp_path / "b.csv"
    r = run("bench", "--bt", "256", "--vocab", "2048", "--hidden", "128", "--repeats", "2", "--warmup", "1",
            "--methods", "canonical,fused,fused_windowed,fused_partial_grad", "--window", "512",
            "--output", str(out))
    assert r.returncode == 0, r.stderr
    lines = out.read_text().strip().splitlines()
    assert lines[0] == "bt,vocab,hidden,method,precision,latency_s,latency_min_s,latency_max_s,aux_peak_bytes,loss"
    assert len(lines) == 5 and all(len(l.split(",")) == 10 for l in lines)
    losses = [float(l.split(",")[9]) for l in lines[1:]]
    assert max(losses) - min(losses) < 1e-3 * abs(losses[0])  # every method computes the same loss


@pytest.mark.gpu
def test_bench_losses_match_the_oracle(cuda, tmp_path):
    """The CLI's device results against the CPU oracle on the same seeded
    instance (the CLI draws make_random_instance bit for bit on the device)."""
    sys.path.insert(0, ROOT)
    from oracle import bindings as ob
    out = tmp_path / "b.csv"
    r = run("bench", "--bt", "200,333", "--vocab", "1500", "--hidden", "136", "--repeats", "1", "--warmup", "0",
            "--methods", "fused,fused_windowed,fused_partial_grad", "--window", "384", "--reduction", "sum",
            "--seed", "7", "--output", str(out))
    assert r.returncode == 0, r.stderr
    for line in out.read_text().strip().splitlines()[1:]:
        bt, vocab, hidden, method = line.split(",")[:4]
        loss = float(line.split(",")[9])
        H, W, Y = ob.make_instance(int(bt), int(hidden), int(vocab), 7)
        _, _, ref = ob.forward(H, W, Y, "sum")
        assert abs(loss - ref) <= 1e-3 * abs(ref), (method, bt, loss, ref)


@pytest.mark.gpu
def test_bench_extended_columns(cuda, tmp_path):
    out = tmp_path / "e.csv"
    r = run("bench", "--bt", "512", "--vocab", "4096", "--hidden", "256", "--repeats", "2", "--warmup", "1",
            "--methods", "canonical,fused", "--extended", "--output", str(out))
    assert r.returncode == 0, r.stderr
    lines = out.read_text().strip().splitlines()
    assert lines[0].endswith(",tokens_per_s,tflops,pct_peak,peak_hbm_bytes,gpus")
    for l in lines[1:]:
        f = l.split(",")
        assert len(f) == 15 and float(f[10]) > 0 and float(f[11]) > 0 and int(f[13]) > 0 and f[14] == "1"
