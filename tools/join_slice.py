"""Join the executor's launch order ([rcsg-order] lines) with an ncu launch
list (time, DRAM read/write bytes) of the same slice: the i-th tcgen05 GEMM
mark is the i-th gemm_tc_persistent launch.  Prints the launches by time with
algorithmic bytes, DRAM bytes and their ratio, achieved GB/s and TF/s."""
import csv, sys
from collections import defaultdict

marks = []
for line in open(sys.argv[1]):
    if line.startswith("[rcsg-order]"):
        f = line.split()
        marks.append(dict(i=int(f[1]), cat=f[2], step=int(f[3]), m=int(f[4]), n=int(f[5]), k=int(f[6]),
                          batch=int(f[7]), work=float(f[8]), bytes=float(f[9])))
rows = [r for r in csv.DictReader(l for l in open(sys.argv[2]) if l.startswith('"'))]
launch = defaultdict(dict)
names = {}
for r in rows:
    i = int(r["ID"])
    launch[i][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    names[i] = r["Kernel Name"]
ids = sorted(launch)
tc = [i for i in ids if "gemm_tc_persistent" in names[i]]
tcm = [m for m in marks if m["cat"] == "gemm_tc"]
total_ns = sum(launch[i].get("gpu__time_duration.sum", 0) for i in ids)
print(f"launches {len(ids)}, device time {total_ns / 1e6:.3f} ms; tcgen05 launches {len(tc)}, marks {len(tcm)}")
out = []
for i, m in zip(tc, tcm):
    L = launch[i]
    ns = L.get("gpu__time_duration.sum", 0)
    dram = L.get("dram__bytes_read.sum", 0) + L.get("dram__bytes_write.sum", 0)
    out.append((ns, m, L, dram, names[i]))
other = total_ns - sum(o[0] for o in out)
out.sort(key=lambda o: -o[0])
print(f"{'ms':>8} {'share':>6} {'step':>5} {'m':>9} {'n':>7} {'k':>7} {'bat':>4} {'TF/s':>7} {'algoGB':>7} "
      f"{'dramGB':>7} {'rd/wr GB':>13} {'x':>5} {'GB/s':>7}  kernel")
for ns, m, L, dram, name in out:
    s = ns * 1e-9
    print(f"{ns / 1e6:8.3f} {ns / total_ns:6.3f} {m['step']:5d} {m['m']:9d} {m['n']:7d} {m['k']:7d} {m['batch']:4d} "
          f"{m['work'] / s / 1e12:7.1f} {m['bytes'] / 1e9:7.3f} {dram / 1e9:7.3f} "
          f"{L.get('dram__bytes_read.sum', 0) / 1e9:6.2f}/{L.get('dram__bytes_write.sum', 0) / 1e9:6.2f} "
          f"{dram / m['bytes'] if m['bytes'] else 0:5.2f} {dram / s / 1e9:7.0f}  {name[:60]}")
print(f"non-tcgen05 launches: {other / 1e6:.3f} ms")
