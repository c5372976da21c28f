"""Writes profiles/<kernel>_dram_traffic.json from an ncu launch list (run where the capture ran,
so the stamp is the hash of the sources that were profiled):

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
        -k regex:hydro --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline
    python tools/traffic_json.py gpurun_out/launches.csv hydro_classifier_kernel > gpurun_out/k4_dram_traffic.json

bytes_per_launch = mean of dram__bytes_read.sum + dram__bytes_write.sum over the kernel's launches
that evaluated a hop (early-exit slot launches, < 1 MB moved, are the ones the device timers skip).
bench.py uses it only when csrc_sha16 matches the current sources.
"""
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(path, kernel):
    from bench import csrc_sha16

    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    hdr = rows[hdr_i]
    launches = {}
    for r in rows[hdr_i + 1:]:
        d = dict(zip(hdr, r))
        if kernel not in d.get("Kernel Name", ""):
            continue
        key = d["ID"]
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                 "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}.get(unit, 1)
        launches.setdefault(key, {})[d["Metric Name"]] = v * scale
    work = [l for l in launches.values()
            if l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0) > 1e6]
    tot = [l["dram__bytes_read.sum"] + l["dram__bytes_write.sum"] for l in work]
    out = {"source": f"ncu launch list {os.path.basename(path)} (cold-cache, serialised launches)",
           "kernel": kernel, "csrc_sha16": csrc_sha16(), "working_launches": len(work),
           "bytes_per_launch": sum(tot) / max(len(tot), 1),
           "seconds_per_launch": sum(l.get("gpu__time_duration.sum", 0) for l in work) / max(len(work), 1),
           "per_launch_bytes": tot}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "hydro_classifier_kernel")
