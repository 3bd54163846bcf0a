"""Summarise ncu --set full reports (raw page) into a markdown table."""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram rd"),
    ("dram__bytes_write.sum", "dram wr"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM thru %"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem thru %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 thru %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 thru %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


_SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3}


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, units = r[0], r[1]
    for row in r[2:]:
        d, raw = {}, {}
        for m, short in METRICS:
            if m in h:
                i = h.index(m)
                d[short] = f"{row[i]} {units[i]}".strip()
                try:
                    raw[m] = float(row[i].replace(",", "")) * _SCALE.get(units[i], 1.0)
                except ValueError:
                    pass
        d["kernel"] = row[h.index("Kernel Name")].split("(")[0].replace("<unnamed>::", "")[:48]
        d["_raw"] = raw
        yield d


def main(paths, out=None, json_out=None):
    import json

    cols = ["kernel"] + [s for _, s in METRICS]
    lines = ["| " + " | ".join(cols) + " |", "|" + "---|" * len(cols)]
    js = []
    for p in paths:
        for d in rows(p):
            lines.append("| " + " | ".join(d.get(c, "") for c in cols) + " |")
            raw = d["_raw"]
            js.append({"kernel": d["kernel"], "report": p, "time_us": raw.get("gpu__time_duration.sum"),
                       "dram_read_bytes": raw.get("dram__bytes_read.sum"),
                       "dram_write_bytes": raw.get("dram__bytes_write.sum"),
                       "tensor_pipe_pct": raw.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
                       "fp64_pipe_pct": raw.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                       "fma_pipe_pct": raw.get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                       "sm_throughput_pct": raw.get("sm__throughput.avg.pct_of_peak_sustained_elapsed")})
    txt = "\n".join(lines)
    if out:
        open(out, "w").write(txt + "\n")
    if json_out:
        open(json_out, "w").write(json.dumps(js, indent=1) + "\n")
    print(txt)


if __name__ == "__main__":
    args = sys.argv[1:]
    out = json_out = None
    if "-o" in args:
        i = args.index("-o")
        out = args[i + 1]
        args = args[:i] + args[i + 2:]
    if "--json" in args:
        i = args.index("--json")
        json_out = args[i + 1]
        args = args[:i] + args[i + 2:]
    main(args, out, json_out)
