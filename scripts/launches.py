"""Summarise an ncu launch-list CSV: one line per kernel launch of a steady frame."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hi]
ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
per = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) > vi:
        per.setdefault(r[ii], {"name": r[ki]})[r[mi]] = r[vi]
# the bench's own kernels only (clip synthesis and torch's elementwise/decode helpers excluded)
seq = [d for d in per.values()
       if not any(k in d["name"] for k in ("synth_kernel", "elementwise", "decode_u8", "vectorized", "unrolled"))]
start = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n = int(sys.argv[3]) if len(sys.argv) > 3 else len(seq)
tot = 0.0
for i, d in enumerate(seq[start:start + n]):
    t = float(d.get("gpu__time_duration.sum", 0)) / 1000.0
    tot += t
    rd = float(d.get("dram__bytes_read.sum", 0)) / 1e6
    wr = float(d.get("dram__bytes_write.sum", 0)) / 1e6
    print(f"{start + i:4d} {d['name'].split('(')[0][-34:]:34s} {t:9.2f} us  rd {rd:8.2f} MB  wr {wr:7.2f} MB  "
          f"regs {d.get('launch__registers_per_thread', '')}  warps {d.get('sm__warps_active.avg.pct_of_peak_sustained_active', '')}")
print(f"total {tot:.2f} us")
