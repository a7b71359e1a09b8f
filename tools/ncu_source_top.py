"""Summarise an ncu --page source --csv --print-source sass dump: top stall
instructions with their dominant stall reasons (for reading captures here)."""
import csv
import sys


def main(path, n=30, ctx=0):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    data = rows[2:]
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(float(r[i_s] or 0) for r in data) or 1
    order = sorted(range(len(data)), key=lambda k: -float(data[k][i_s] or 0))[:n]
    for k in order:
        r = data[k]
        rs = sorted(((float(r[hdr.index(x)] or 0), x) for x in reasons), reverse=True)[:2]
        why = ", ".join(f"{x[6:]}={v:.0f}" for v, x in rs if v > 0)
        print(f"{float(r[i_s]) / tot * 100:5.1f}% [{k:4d}] {r[1][:90]:90s} {why}")
        for j in range(max(0, k - ctx), k):
            print(f"              [{j:4d}] {data[j][1][:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30, int(sys.argv[3]) if len(sys.argv) > 3 else 0)
