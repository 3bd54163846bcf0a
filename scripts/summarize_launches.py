"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel."""
import collections
import csv
import sys


def main(path, out=None):
    rows = list(csv.reader(open(path)))
    hdr = None
    data = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        name = d["Kernel Name"].split("(")[0].replace("<unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"]) * scale.get(d["Metric Unit"], 1.0)
    tot = sum(v[1] for v in agg.values())
    lines = [f"launches: {len(data)}  total device time: {tot / 1e3:.2f} ms (ncu, serialised, cold L2)", "",
             "| kernel | launches | total ms | avg us | share |", "|---|---:|---:|---:|---:|"]
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {v[0]} | {v[1] / 1e3:.2f} | {v[1] / v[0]:.1f} | {v[1] / tot:.3f} |")
    txt = "\n".join(lines)
    if out:
        open(out, "w").write(txt + "\n")
    print(txt)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
