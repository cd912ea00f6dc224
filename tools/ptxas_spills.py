"""Summarise ptxas -v output: registers and spills per kernel (flags decoded for coda_gemm_fast)."""
import re
import subprocess
import sys
from pathlib import Path

log = Path(sys.argv[1] if len(sys.argv) > 1 else Path(__file__).resolve().parents[1] /
           "paper_2605_19269_b200/_lib/ptxas.log").read_text().splitlines()
fn = None
for line in log:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        fn = m.group(1)
        try:
            fn = subprocess.run(["c++filt", fn], capture_output=True, text=True).stdout.strip()
        except Exception:
            pass
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and fn:
        st = (int(m.group(2)), int(m.group(3)))
        if st != (0, 0) or "-a" in sys.argv:
            print(f"spill st/ld {st[0]:4d}/{st[1]:4d}  {fn[:150]}")
    m = re.search(r"Used (\d+) registers", line)
    if m and fn and "-r" in sys.argv:
        print(f"regs {m.group(1):>4}  {fn[:150]}")
