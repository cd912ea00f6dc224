"""Per-launch table (time, SM clock, tensor pipe %, DRAM GB, TFLOP/s) of one measured step
from an ncu CSV of bench.py --ncu and its launch tags.

    python tools/ncu_launch_table.py gpurun_out/<dir>/ncu_launches_c4.csv gpurun_out/<dir>/launch_tags_c4.json
"""
import csv
import json
import re
import sys
from pathlib import Path

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3,
         "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6, "Ghz": 1.0, "Mhz": 1e-3, "hz": 1e-9, "%": 1.0}


def main():
    lines = Path(sys.argv[1]).read_text().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    tags = json.loads(Path(sys.argv[2]).read_text())
    per = {}
    for r in rows:
        i = int(r["ID"])
        v = float(r["Metric Value"].replace(",", "")) * SCALE.get(r.get("Metric Unit", ""), 1.0)
        per.setdefault(i, {})[r["Metric Name"]] = v
    print("| launch | ms | SM GHz | tensor pipe % | DRAM GB | TFLOP/s |\n|---|---|---|---|---|---|")
    tot_ms = tot_b = tot_f = 0.0
    for i in sorted(per):
        m = per[i]
        tag = tags[i] if i < len(tags) else {}
        name = tag.get("tag", tag.get("name", "?")) if isinstance(tag, dict) else str(tag)
        flops = tag.get("flops", 0.0) if isinstance(tag, dict) else 0.0
        if not flops:
            mm = re.search(r"(\d+)x(\d+)x(\d+)", name)
            flops = 2.0 * int(mm[1]) * int(mm[2]) * int(mm[3]) if mm else 0.0
        ms = m.get("gpu__time_duration.sum", 0.0)
        ghz = m.get("sm__cycles_elapsed.avg.per_second", 0.0)
        tp = next((v for k, v in m.items() if "pipe_tensor" in k), 0.0)
        gb = (m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)) / 1e9
        tf = flops / (ms * 1e-3) / 1e12 if ms else 0.0
        tot_ms, tot_b, tot_f = tot_ms + ms, tot_b + gb, tot_f + flops
        print(f"| {name} | {ms:.3f} | {ghz:.2f} | {tp:.1f} | {gb:.2f} | {tf:.0f} |")
    print(f"| **step** | {tot_ms:.3f} | | | {tot_b:.2f} | {tot_f / (tot_ms * 1e-3) / 1e12:.0f} |")


if __name__ == "__main__":
    main()
