"""Top SASS instructions of one kernel in an ncu report by warp-stall samples
(and executed instructions / shared-memory conflicts).

  python scripts/ncu_hot.py REPORT.ncu-rep KERNEL_REGEX [N] [launch_index]
"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name",
                      "regex:" + kre, "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = rows[0]
ci = {c: i for i, c in enumerate(h)}
data = rows[1:]
def f(r, c):
    try:
        return float(r[ci[c]])
    except (ValueError, KeyError, IndexError):
        return 0.0
tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
tot_i = sum(f(r, "Instructions Executed") for r in data)
print(lines[0][:120], f"samples={tot:.0f} inst={tot_i:.0f}")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:n]:
    top = sorted(((f(r, c), c[6:]) for c in reasons), reverse=True)[:2]
    if len(r) <= ci['Source']:
        continue
    print(f"{f(r, 'Warp Stall Sampling (All Samples)'):6.0f} {f(r, 'Instructions Executed'):9.0f} "
          f"{f(r, 'L1 Conflicts Shared N-Way'):4.0f}  {r[ci['Source']].strip()[:60]:60s} " +
          " ".join(f"{c}={v:.0f}" for v, c in top if v))
