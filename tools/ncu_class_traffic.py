"""Per-launch DRAM traffic of a kernel class from an ncu --set full capture of
several launches (e.g. every cfg5 layer of the dominant class, captured with
tools/prof_stack_layers.py): mean dram__bytes_read.sum + dram__bytes_write.sum
per launch, written to profiles/ncu_traffic.json under `key` (bench.py's
roofline.traffic), plus a summary of the launches.

    python tools/ncu_class_traffic.py REPORT.ncu-rep KEY NAME LAYER1,LAYER2,...
"""
import csv
import io
import json
import os
import subprocess
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(rep, key, name, layers):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__throughput.avg.pct_of_peak_sustained_active", "gpc__cycles_elapsed.max", "sm__cycles_active.avg"]
    launches = []
    for i, r in enumerate(rows[2:]):
        d = {"layer": layers[i] if i < len(layers) else None, "kernel": r[hdr.index("Kernel Name")][:100]}
        for k in keys:
            if k in hdr:
                j = hdr.index(k)
                v = float(r[j].replace(",", "")) if r[j] else 0.0
                d[k] = v * UNITS.get(units[j], 1) if "bytes" in k else v
        launches.append(d)
    dram = [d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in launches]
    mean = sum(dram) / len(dram)
    os.makedirs("profiles", exist_ok=True)
    with open(f"profiles/{name}.json", "w") as f:
        json.dump({"report": os.path.basename(rep), "key": key, "launches": launches,
                   "mean_dram_bytes_per_launch": mean}, f, indent=1)
    tpath = "profiles/ncu_traffic.json"
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    traffic[key] = {"bytes": mean, "source": name, "launches": len(dram)}
    json.dump(traffic, open(tpath, "w"), indent=1)
    print(key, len(dram), "launches, mean dram bytes per launch", mean)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4].split(","))
