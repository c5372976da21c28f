"""Summarise ncu captures for profiles/ (runs on the CPU box: `ncu -i`).

    python tools/ncu_summary.py full <report.ncu-rep> [label]     # per-launch key metrics + top stalls
    python tools/ncu_summary.py launches <launches.csv>            # per-kernel share of the launch list
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct_of_peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_pct"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1_smem_pct"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor_pipe_pct"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
    ("smsp__inst_executed.sum", "warp_instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "lds_bank_conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "lds_wavefronts"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def stalls(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        st = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(d[k])) for k in hdr
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
              and d[k] not in ("", "n/a")]
        tot = sum(v for _, v in st) or 1.0
        res.append(sorted(((k, round(100 * v / tot, 1)) for k, v in st), key=lambda x: -x[1])[:6])
    return res


def full(rep, label=""):
    runs, units = raw(rep)
    st = stalls(rep)
    print(f"### {label or rep}\n")
    for i, d in enumerate(runs):
        print(f"- launch {i}: `{d.get('Kernel Name', '')[:60]}`")
        for k, name in KEYS:
            if k in d:
                print(f"  - {name}: {d[k]} {units.get(k, '')}")
        print(f"  - top stall reasons (% of samples): {st[i]}")
    print()


def launches(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rd = csv.DictReader(io.StringIO("".join(lines)))
    per = defaultdict(lambda: [0.0, 0])
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        if unit == "usecond":
            v *= 1e3
        elif unit == "msecond":
            v *= 1e6
        name = r["Kernel Name"].split("(")[0]
        per[name][0] += v
        per[name][1] += 1
    tot = sum(v for v, _ in per.values())
    print("| kernel | launches | total ns | share |\n|---|---|---|---|")
    for k, (v, n) in sorted(per.items(), key=lambda x: -x[1][0]):
        print(f"| {k} | {n} | {v:.0f} | {100 * v / tot:.1f}% |")


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
    else:
        launches(sys.argv[2])
