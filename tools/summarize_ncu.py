"""Summarise an ncu launch list (gpu__time_duration per launch) and --set full
captures into a markdown table for profiles/. Usage:
    python tools/summarize_ncu.py <tag> [launches.csv] [report.ncu-rep ...]
Writes profiles/<tag>_launches.csv (kernel, duration_ns per launch) and prints
markdown."""
import collections
import csv
import io
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def short(name):
    return name.split("(")[0].replace("void ", "").replace("adipc_gpu::", "").replace("<unnamed>::", "").strip()


def launch_list(path, tag):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(d["Metric Unit"], 1)
        out.append((short(d["Kernel Name"]), v))
    with open(os.path.join(ROOT, "profiles", f"{tag}_launches.csv"), "w") as f:
        f.write("kernel,duration_ns\n")
        for k, v in out:
            f.write(f"\"{k}\",{v:.0f}\n")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for k, v in out:
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v[1] for v in agg.values())
    lines = ["| kernel | launches | total ms | share | avg us |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:20]:
        lines.append(f"| `{k}` | {v[0]} | {v[1] / 1e6:.2f} | {100 * v[1] / tot:.1f}% | {v[1] / v[0] / 1e3:.2f} |")
    return "\n".join(lines)


WANT = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "L1 %"),
    ("sm__warps_active.avg.per_cycle_active", "warps/SM"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
]


def full_report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = ["| kernel | " + " | ".join(w[1] for w in WANT) + " | top stalls |",
             "|---" * (len(WANT) + 2) + "|"]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        cells = []
        for k, _ in WANT:
            cells.append(f"{d.get(k, '?')} {u.get(k, '')}".strip())
        ks = [k for k in hdr if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
        tot = sum(float(d[k].replace(",", "") or 0) for k in ks) or 1
        top = sorted(ks, key=lambda k: -float(d[k].replace(",", "") or 0))[:3]
        stalls = ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * float(d[k].replace(',', '')) / tot:.0f}%"
                           for k in top)
        lines.append(f"| `{short(d['Kernel Name'])}` | " + " | ".join(cells) + f" | {stalls} |")
    return "\n".join(lines)


if __name__ == "__main__":
    tag = sys.argv[1]
    if len(sys.argv) > 2:
        print(f"### Launch list ({tag}): one warm bench step, ncu serialised, cold caches\n")
        print(launch_list(sys.argv[2], tag))
    for rep in sys.argv[3:]:
        print(f"\n### `ncu --set full` — {os.path.basename(rep)}\n")
        print(full_report(rep))
