"""Per-launch table from tools/ncu_tensor.sh: time, SM clock, tensor-pipe %, DRAM bytes vs
algorithmic flops, plus fused vs unfused DRAM totals."""
import csv
import json
import re
import sys
from pathlib import Path


def rows(path):
    lines = Path(path).read_text().splitlines()
    st = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    per = {}
    for r in csv.DictReader(lines[st:]):
        try:
            v = float(r["Metric Value"].replace(",", ""))
        except ValueError:
            continue
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6,
                 "msecond": 1e-3, "ms": 1e-3, "Ghz": 1e9, "GHz": 1e9, "Mhz": 1e6, "MHz": 1e6, "hz": 1, "%": 1}.get(r.get("Metric Unit", ""), 1)
        d = per.setdefault(int(r["ID"]), {"name": r["Kernel Name"]})
        d[r["Metric Name"]] = v * scale
    return [per[i] for i in sorted(per)]


def main():
    launches = rows(sys.argv[1])
    tags = json.loads(Path(sys.argv[2]).read_text())
    assert len(tags) == len(launches), (len(tags), len(launches))
    print("| launch | ms | SM GHz | tensor pipe % | DRAM GB | TFLOP/s |")
    print("|---|---|---|---|---|---|")
    tot_t = tot_b = tot_f = 0.0
    for tag, d in zip(tags, launches):
        t = d["gpu__time_duration.sum"]
        b = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
        m = re.search(r"(\d+)x(\d+)x(\d+)", tag)
        fl = 2.0 * int(m.group(1)) * int(m.group(2)) * int(m.group(3)) if m else 0.0
        tp = d.get("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed", 0.0)
        clk = d.get("sm__cycles_elapsed.avg.per_second", 0.0) / 1e9
        tot_t += t
        tot_b += b
        tot_f += fl
        print(f"| {tag} | {t * 1e3:.3f} | {clk:.2f} | {tp:.1f} | {b / 1e9:.2f} | "
              f"{(fl / t / 1e12) if fl else 0:.0f} |")
    print(f"| **step** | {tot_t * 1e3:.3f} | | | {tot_b / 1e9:.2f} | {tot_f / tot_t / 1e12:.0f} |")
    for name in ("fused", "unfused"):
        p = Path(sys.argv[1]).parent / f"ncu_bytes_{name}_c4.csv"
        if p.exists():
            rr = rows(p)
            b = sum(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in rr)
            t = sum(d["gpu__time_duration.sum"] for d in rr)
            print(f"\n{name}: {len(rr)} launches, DRAM {b / 1e9:.2f} GB, serialised kernel time {t * 1e3:.2f} ms")


if __name__ == "__main__":
    main()
