"""Per-region summary of an ncu source-page CSV (--page source --csv
--print-source sass): executed warp instructions per unit (e.g. per tile)
and stall samples, in blocks of `block` SASS lines."""
import collections
import csv
import sys


def main(path, units=1.0, block=48):
    rows = list(csv.reader(open(path)))
    hdr, data = rows[1], rows[2:]
    ie = hdr.index("Instructions Executed")
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    cnt = [float(r[ie] or 0) / units for r in data]
    st = [float(r[i_s] or 0) for r in data]
    tot = sum(st) or 1
    print(f"total instr/unit {sum(cnt):.0f}")
    for b in range(0, len(data), block):
        c, s = sum(cnt[b:b + block]), sum(st[b:b + block])
        if c > 100 or s / tot > 0.02:
            t = collections.Counter()
            for r in data[b:b + block]:
                for x in reasons:
                    t[x[6:]] += float(r[hdr.index(x)] or 0)
            top = ", ".join(f"{x}={int(v)}" for x, v in t.most_common(3))
            print(f"{b:5d} instr/unit {c:7.0f} stall {s / tot * 100:5.1f}%  {data[b][1][:48]:48s} {top}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1.0, int(sys.argv[3]) if len(sys.argv) > 3 else 48)
