"""Summarise an ncu report into profiles/: key metrics of the captured
kernel(s) and dram traffic per launch (consumed by bench.py's roofline)."""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "smsp__cycles_active.avg", "sm__warps_active.avg.pct_of_peak_sustained_active"]


def main(rep, name, workload):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:120]}
        for k in KEYS:
            if k in hdr:
                d[k] = f"{r[hdr.index(k)]} {units[hdr.index(k)]}".strip()
        res.append(d)
    os.makedirs("profiles", exist_ok=True)
    with open(f"profiles/{name}.json", "w") as f:
        json.dump({"report": os.path.basename(rep), "workload": workload, "kernels": res}, f, indent=1)
    # dram traffic per launch for bench.py
    tpath = "profiles/ncu_traffic.json"
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    k0 = res[0]

    def val(key):
        v, u = k0[key].split()[:2] if " " in k0[key] else (k0[key], "byte")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        return float(v.replace(",", "")) * scale

    traffic[workload] = {"bytes": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"), "source": name}
    json.dump(traffic, open(tpath, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3])
