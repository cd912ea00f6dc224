"""Efficiency of each GEMM launch vs the tcgen05 MMA floor at the launch's own SM clock."""
import collections
import csv
import sys

# C4 step launch order (fast GEMMs, aux kernels interleaved) -> (M, N, K)
C4 = [("K4a", 16384, 4096, 4096), ("K6", 16384, 28672, 4096), ("K4b", 16384, 4096, 14336),
      ("K7", 16384, 12288, 4096), ("K9b", 16384, 4096, 12288), ("wgrad_qkv", 4096, 12288, 16384),
      ("K10", 16384, 14336, 4096), ("wgrad_down", 14336, 4096, 16384), ("K9a", 16384, 4096, 28672),
      ("wgrad_gu", 4096, 28672, 16384), ("dgrad_x", 16384, 4096, 4096), ("wgrad_out", 4096, 4096, 16384)]


def floor_cycles(m, n, k, units=74):
    tiles = -(-m // 256) * -(-n // 256)
    return -(-tiles // units) * -(-k // 64) * 512


rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr, data = rows[hi], rows[hi + 1:]
ik, im, iv, iu, iid = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
per = collections.defaultdict(dict)
names = {}
for r in data:
    if not r[iv]:
        continue
    v = float(r[iv].replace(",", ""))
    scale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9,
             "Ghz": 1e9, "GHz": 1e9, "Mhz": 1e6, "MHz": 1e6, "hz": 1, "cycle": 1}.get(r[iu], 1)
    per[int(r[iid])][r[im]] = v * scale
    names[int(r[iid])] = r[ik]
gemms = [i for i in sorted(per) if "coda_gemm" in names[i]]
tot_t = 0.0
for (label, m, n, k), i in zip(C4, gemms):
    t = per[i]["gpu__time_duration.sum"]
    clk = per[i]["sm__cycles_elapsed.avg.per_second"]
    cyc = t * clk
    fl = floor_cycles(m, n, k)
    tot_t += t
    print(f"{label:11s} {t*1e3:7.3f} ms  clk {clk/1e9:5.3f} GHz  floor {fl/1e6:6.3f} Mcyc  used {cyc/1e6:6.3f} Mcyc"
          f"  eff {fl/cyc*100:5.1f}%  {2*m*n*k/t/1e12:6.0f} TFLOP/s")
others = [i for i in sorted(per) if "coda_gemm" not in names[i]]
for i in others:
    print(f"{names[i][:40]:40s} {per[i]['gpu__time_duration.sum']*1e3:7.3f} ms")
print(f"GEMM total {tot_t*1e3:.3f} ms")
