"""Fold an ncu per-launch DRAM-bytes CSV of one measured step into profiles/traffic.json.

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx \\
        --nvtx-include "measure/" --csv --log-file gpurun_out/ncu_dram_c4.csv \\
        python bench.py --ncu --steps 1 --warmup 1          # also writes gpurun_out/launch_tags_c4.json
    python tools/traffic_json.py gpurun_out/ncu_dram_c4.csv gpurun_out/launch_tags_c4.json c4

Keys are "<config>:<launch tag>", values DRAM bytes (read + write) per launch (mean over
repeated tags within the step).
"""
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def main():
    csv_path, tags_path, config = sys.argv[1], sys.argv[2], sys.argv[3]
    lines = Path(csv_path).read_text().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    per = {}
    for r in rows:
        if not r["Metric Name"].startswith("dram__bytes"):
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "byte")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        per.setdefault(int(r["ID"]), [r["Kernel Name"], 0.0])[1] += v * scale
    launches = [per[k] for k in sorted(per)]
    tags = json.loads(Path(tags_path).read_text())
    if len(tags) != len(launches):
        sys.exit(f"{len(tags)} tags vs {len(launches)} ncu launches: not one measured step")
    out_path = ROOT / "profiles" / "traffic.json"
    out = json.loads(out_path.read_text()) if out_path.exists() else {}
    out = {k: v for k, v in out.items() if not k.startswith(config + ":")}   # drop stale launches
    import subprocess
    import time

    sha = subprocess.run(["git", "rev-parse", "--short=12", "HEAD"], capture_output=True, text=True,
                         cwd=str(ROOT)).stdout.strip()
    meta = out.setdefault("_meta", {})
    meta[config] = {"source": str(Path(csv_path).name), "git": sha, "date": time.strftime("%Y-%m-%d"),
                    "how": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none, "
                           "one measured step of bench.py --ncu"}
    acc = {}
    for tag, (_, b) in zip(tags, launches):
        acc.setdefault(tag, []).append(b)
    for tag, bs in acc.items():
        out[f"{config}:{tag}"] = int(sum(bs) / len(bs))
    out_path.write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps({k: v for k, v in out.items() if k.startswith(config + ":")}, indent=1))


if __name__ == "__main__":
    main()
