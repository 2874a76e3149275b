"""Summarise ncu outputs into profiles/ (launch list shares + per-kernel full-capture metrics)."""
import collections
import csv
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def launches(csv_path: Path, out: Path) -> None:
    rows = list(csv.reader(open(csv_path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    idx = [i for i, d in enumerate(data) if "timestep_freq" in d["Kernel Name"]]
    step = data[idx[-1]:]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in step:
        k = d["Kernel Name"].split("(")[0][:60] + "  grid=" + d["Grid Size"]
        agg[k][0] += 1
        agg[k][1] += float(d["Metric Value"])
    tot = sum(v[1] for v in agg.values())
    lines = [f"# one STDiT3-XL/2 240p x 51 CFG step, DoP 1: {len(step)} launches, "
             f"sum of ncu per-launch gpu__time_duration = {tot / 1e6:.3f} ms (serialised, cold)",
             f"{'ms':>9} {'n':>5} {'avg_us':>9} {'share':>6}  kernel"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{v[1] / 1e6:9.3f} {v[0]:5d} {v[1] / v[0] / 1e3:9.1f} {100 * v[1] / tot:5.1f}%  {k}")
    out.write_text("\n".join(lines) + "\n")
    print("\n".join(lines[:12]))


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second"]


def full(rep: Path, out: Path) -> list[dict]:
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    rows = list(csv.reader(txt))
    hdr, units = rows[0], rows[1]
    res = []
    lines = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:80], "grid": r[hdr.index("Grid Size")]}
        for w in WANT:
            if w in hdr:
                d[w] = f"{r[hdr.index(w)]} {units[hdr.index(w)]}".strip()
        res.append(d)
        lines.append(json.dumps(d))
    out.write_text("\n".join(lines) + "\n")
    return res


if __name__ == "__main__":
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    go = ROOT / "gpurun_out"
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    if (go / f"launches_{tag}.csv").exists():
        launches(go / f"launches_{tag}.csv", prof / f"{tag}_step_launches_240p.txt")
    for name in ("gemm", "fmha"):
        rep = go / f"{name}_{tag}.ncu-rep"
        if rep.exists():
            res = full(rep, prof / f"{tag}_{name}_ncu_full.jsonl")
            for d in res:
                print(d)
