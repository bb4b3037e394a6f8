"""Summarise ncu captures into profiles/ (dev tool).

usage: python scripts/ncu_summary.py <round-tag> <config> <launches.csv> <full.ncu-rep> [bench.json]
Writes profiles/<tag>_launches.csv (copy), profiles/<tag>_ncu_summary.md and
profiles/traffic.json: DRAM bytes per launch of each kernel of <config>, with
the hash of the kernel sources captured (bench.py reports the number only
while the sources are unchanged).
"""
import collections, csv, io, json, os, shutil, subprocess, sys

tag, config, launches, rep = sys.argv[1:5]
bench = json.load(open(sys.argv[5])) if len(sys.argv) > 5 else None
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root)
from bench import _source_hash  # noqa: E402
prof = os.path.join(root, "profiles")
os.makedirs(prof, exist_ok=True)
shutil.copy(launches, os.path.join(prof, f"{tag}_launches.csv"))

def short(name):
    if "fce_bwd_persistent" in name: return "fce_bwd_persistent_sm100"
    if "fce_tile_kernel<0>" in name or "fce_tile_kernel<0, " in name: return "fce_fwd_sm100"
    if "fce_tile_kernel<1>" in name: return "fce_bwd_grad_sm100"
    if "fce_tile_kernel<2>" in name: return "fce_bwd_gemm_sm100"
    return name.split("(")[0].replace("void ", "")

rows = list(csv.reader(open(launches)))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr, data = rows[hi], rows[hi + 1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.OrderedDict()
for r in data:
    v = float(r[vi].replace(",", ""))
    v *= {"msecond": 1e3, "ms": 1e3, "usecond": 1.0, "us": 1.0, "nsecond": 1e-3, "ns": 1e-3, "second": 1e6, "s": 1e6}.get(r[ui], 1.0)
    k = short(r[ki])
    c, t = agg.get(k, (0, 0.0))
    agg[k] = (c + 1, t + v)
tot = sum(t for _, t in agg.values())

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h2, units, kd = rr[0], rr[1], rr[2:]
want = {
    "gpu__time_duration.sum": "duration",
    "sm__cycles_elapsed.avg.per_second": "SM clock",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor pipe active",
    "dram__bytes_read.sum": "DRAM read",
    "dram__bytes_write.sum": "DRAM write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "DRAM throughput",
    "lts__t_sector_hit_rate.pct": "L2 hit rate",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "L2 throughput",
    "launch__registers_per_thread": "registers/thread",
    "launch__grid_size": "grid",
    "launch__cluster_dim_x": "cluster x",
}
scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}
traffic = {}
lines = [f"# ncu summary — {tag} ({config})", "",
         "Captured under gpurun on one B200 with `--clock-control none` (cold cache, serialised",
         "launches: compare shares, not absolute times with the bench).", "",
         "## Launch list (one fwd+bwd step, `ncu --metrics gpu__time_duration.sum`)", "",
         "| kernel | launches | total µs | share |", "|---|---|---|---|"]
for k, (c, t) in agg.items():
    lines.append(f"| {k} | {c} | {t:.1f} | {100 * t / tot:.1f}% |")
lines += ["", f"Step total under ncu: {tot / 1e3:.2f} ms", "", "## `--set full` per kernel", ""]
for r in kd:
    name = short(r[h2.index("Kernel Name")])
    lines.append(f"### {name}")
    lines.append("")
    for key, label in want.items():
        if key in h2:
            i = h2.index(key)
            lines.append(f"- {label}: {r[i]} {units[i]}")
    try:
        rd = float(r[h2.index("dram__bytes_read.sum")]) * scale.get(units[h2.index("dram__bytes_read.sum")], 1)
        wr = float(r[h2.index("dram__bytes_write.sum")]) * scale.get(units[h2.index("dram__bytes_write.sum")], 1)
        if rd == rd and wr == wr:  # ncu reports NaN for some very long launches
            traffic[name] = rd + wr
        lines.append(f"- DRAM traffic per launch: {(rd + wr) / 1e9:.2f} GB")
    except (ValueError, KeyError):
        pass
    lines.append("")
if bench:
    lines += ["## Bench line of the same build", "", "```json", json.dumps(bench, indent=1), "```", ""]
open(os.path.join(prof, f"{tag}_ncu_summary.md"), "w").write("\n".join(lines))
tp = os.path.join(prof, "traffic.json")
old = json.load(open(tp)) if os.path.exists(tp) else {}
old = {k: v for k, v in old.items() if isinstance(v, dict)}  # drop the round-1 flat format
sha = _source_hash()
old[config] = {k: {"dram_bytes": v, "source_sha": sha, "capture": f"{tag}_ncu_summary.md"}
               for k, v in traffic.items()}
json.dump(old, open(tp, "w"), indent=1)
print("\n".join(lines[:40]))
