"""Summarise ncu outputs into committed profiles/.

  python tools/profile_summary.py <tag> <launches.csv> <k1.ncu-rep> [bench.json] [c3launches.csv]

Writes profiles/<tag>_launches.md (per-kernel mean device time and share of
the step from the `--metrics gpu__time_duration.sum` launch list),
profiles/<tag>_k1_ncu.md (key counters of the `--set full` capture of K1) and
profiles/k1_traffic.json (DRAM bytes per K1 launch, read by bench.py for the
roofline `traffic` field), and with a C3 launch list profiles/<tag>_c3_launches.md
(per-kernel totals of the last full C3 step).
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

K1_METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum.per_second",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
    "lts__t_bytes.sum",
    "sm__cycles_elapsed.avg.per_second",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                name = d["Kernel Name"]
                unit = d.get("Metric Unit", "ns")
                v = float(d["Metric Value"].replace(",", ""))
                v = v / 1e3 if unit == "ns" else (v * 1e3 if unit == "ms" else v)
                agg[name].append(v)
    total = sum(sum(v) for v in agg.values())
    out = ["| kernel | launches | mean µs | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        short = k.split("(")[0][:70]
        out.append(f"| `{short}` | {len(v)} | {sum(v) / len(v):.2f} | {sum(v) / total:.3f} |")
    return "\n".join(out), agg


def ncu_raw(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {}
        for i, h in enumerate(hdr):
            if h in K1_METRICS:
                d[h] = (vals[i], units[i])
        res.append(d)
    return res


def to_bytes(v, u):
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def c3_step(path):
    """Per-kernel totals of the last complete C3 forward (embed_kernel starts one)."""
    rows = list(csv.reader(open(path)))
    hdr = None
    seq = []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                v = float(d["Metric Value"].replace(",", ""))
                v = v / 1e3 if d.get("Metric Unit", "ns") == "ns" else v
                seq.append((int(d["ID"]), d["Kernel Name"], v))
    seq.sort()
    starts = [i for i, (_, k, _) in enumerate(seq) if "embed_kernel" in k]
    last = seq[starts[-1]:] if starts else seq
    agg = defaultdict(lambda: [0, 0.0])
    for _, k, v in last:
        agg[k.split("(")[0][:70]][0] += 1
        agg[k.split("(")[0][:70]][1] += v
    total = sum(v[1] for v in agg.values())
    out = [f"Last full step: {len(last)} kernels, {total / 1e3:.2f} ms serialised.\n",
           "| kernel | launches | total µs | share |", "|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {n} | {t:.1f} | {t / total:.3f} |")
    return "\n".join(out)


def main():
    tag, lcsv, rep = sys.argv[1:4]
    bench = json.load(open(sys.argv[4])) if len(sys.argv) > 4 else None
    os.makedirs(PROF, exist_ok=True)
    table, _ = launches(lcsv)
    with open(os.path.join(PROF, f"{tag}_launches.md"), "w") as f:
        f.write(f"# {tag}: launch list (ncu --metrics gpu__time_duration.sum --clock-control none)\n\n")
        f.write("Cold-cache, serialised per-launch times: compare SHARES, not absolutes.\n\n")
        f.write(table + "\n")
    metrics = ncu_raw(rep)
    with open(os.path.join(PROF, f"{tag}_k1_ncu.md"), "w") as f:
        f.write(f"# {tag}: K1 tree attention, ncu --set full --clock-control none\n\n")
        for i, d in enumerate(metrics):
            f.write(f"## launch {i}\n\n| metric | value | unit |\n|---|---|---|\n")
            for k in K1_METRICS:
                if k in d:
                    f.write(f"| {k} | {d[k][0]} | {d[k][1]} |\n")
            f.write("\n")
        if bench:
            r = bench.get("roofline", {})
            f.write(f"bench.py (same build): K1 {r.get('us_per_launch', 0):.1f} µs/launch, "
                    f"{r.get('achieved', 0):.0f} GB/s = {r.get('frac', 0):.3f} of the measured "
                    f"{r.get('peak')} GB/s copy peak; algorithmic bytes/launch "
                    f"{r.get('bytes_per_launch')}\n")
    if metrics and "dram__bytes_read.sum" in metrics[0]:
        d = metrics[0]
        traffic = to_bytes(*d["dram__bytes_read.sum"]) + to_bytes(*d["dram__bytes_write.sum"])
        json.dump({"tag": tag, "dram_bytes_per_launch": traffic,
                   "source": f"profiles/{tag}_k1_ncu.md"},
                  open(os.path.join(PROF, "k1_traffic.json"), "w"), indent=1)
    if len(sys.argv) > 5:
        with open(os.path.join(PROF, f"{tag}_c3_launches.md"), "w") as f:
            f.write(f"# {tag}: C3 full stack (bench.py --config c3), one step, ncu launch list\n\n")
            f.write("`nvjet_*` are cuBLAS GEMMs (QKV batched, WO / W2 with the residual as beta=1, "
                    "W1, LM head); `tree_attn_tc_kernel` is K1 per layer.\n\n")
            f.write(c3_step(sys.argv[5]) + "\n")
    print("wrote", PROF)


if __name__ == "__main__":
    main()
