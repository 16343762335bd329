"""Summarise an ncu --csv launch list (gpu__time_duration.sum, dram__bytes_read.sum).

    python tools/launch_table.py gpurun_out/launches.csv [--min-us 0]

Prints per-kernel launch count, mean time, share, DRAM bytes per launch and
GB/s. ncu serialises launches (no PDL overlap) and runs them cold: compare
SHARES, not absolute times, with the live bench.
"""
import argparse
import collections
import csv


def load(path):
    hdr, per = None, collections.OrderedDict()
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            key = (int(d["ID"]), d["Kernel Name"], d["Grid Size"])
            per.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return per


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--min-us", type=float, default=0.0, help="drop launches shorter than this")
    a = ap.parse_args()
    per = load(a.csv)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for (i, k, g), m in per.items():
        t = m.get("gpu__time_duration.sum", 0.0)
        if t / 1e3 < a.min_us:
            continue
        x = agg[k.split("(")[0][:60]]
        x[0] += 1
        x[1] += t
        x[2] += m.get("dram__bytes_read.sum", 0.0)
    tot = sum(v[1] for v in agg.values()) or 1.0
    print(f"{'launches':>8} {'mean us':>9} {'share':>7} {'MB/launch':>10} {'GB/s':>7}  kernel")
    for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{n:8d} {t / n / 1e3:9.1f} {t / tot * 100:6.1f}% {b / n / 1e6:10.1f} {b / t if t else 0:7.0f}  {k}")
    print(f"total {tot / 1e6:.3f} ms over {sum(v[0] for v in agg.values())} launches")


if __name__ == "__main__":
    main()
