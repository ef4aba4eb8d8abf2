"""Summarise an `ncu --set full` capture of one steady frame (scripts/gpu_full.sh)
into a markdown table and profiles/traffic.json (DRAM bytes per launch of
each kernel, used by bench.py's roofline.traffic).

  python scripts/ncu_summary.py gpurun_out/TAG_frame.ncu-rep profiles/rN_ncu_frame_table.md profiles/traffic.json
"""
import csv
import io
import json
import subprocess
import sys

# launch order of a steady frame of paper_like (f16, 8-bit frames): bench.py's kernel names
# (FRAME_F32: the fp32-frame path of round 1)
FRAME = ["detect[0]", "dilate_compact[0]", "conv_tc[0]", "pool[1]", "dilate_compact[2]",
         "conv_tc[2]", "pool[3]:scan", "pool[3]:work", "dilate_compact[4]", "conv_tc_tail[4]"]
FRAME_F32 = ["detect[0]", "dilate_compact[0]", "conv_exact[0]", "pool[1]:scan", "pool[1]:work", "dilate_compact[2]",
             "conv_tc[2]", "pool[3]:scan", "pool[3]:work", "dilate_compact[4]", "conv_tc_tail[4]"]
METRICS = [
    ("gpu__time_duration.sum", "us", 1e-3),
    ("dram__bytes_read.sum", "MB rd", 1e-6),
    ("dram__bytes_write.sum", "MB wr", 1e-6),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %", 1),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor %", 1),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %", 1),
    ("lts__t_sector_hit_rate.pct", "L2 hit %", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %", 1),
    ("sm__inst_executed.avg.per_cycle_active", "IPC", 1),
]


def main(rep, out_md, out_json):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}

    def val(r, m):
        try:
            v = float(r[col[m]].replace(",", ""))
        except (KeyError, ValueError):
            return None
        u = units[col[m]]
        scale = {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "byte": 1, "Kbyte": 1e3,
                 "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        return v * scale

    lines = ["| # | kernel | bench name | " + " | ".join(m[1] for m in METRICS) + " |",
             "|---|---|---|" + "---|" * len(METRICS)]
    traffic = {}
    for i, r in enumerate(data):
        name = r[col["Kernel Name"]].split("(")[0].replace("void ", "")[-40:]
        bench = FRAME[i] if i < len(FRAME) else "?"
        cells = []
        for m, label, sc in METRICS:
            v = val(r, m)
            cells.append("" if v is None else f"{v * sc:.2f}")
        lines.append(f"| {i} | `{name}` | {bench} | " + " | ".join(cells) + " |")
        key = bench.split(":")[0]
        rd, wr, t = val(r, "dram__bytes_read.sum") or 0, val(r, "dram__bytes_write.sum") or 0, val(r, "gpu__time_duration.sum") or 0
        e = traffic.setdefault(key, {"dram_bytes": 0, "ncu_us": 0.0})
        e["dram_bytes"] += int(rd + wr)
        e["ncu_us"] = round(e["ncu_us"] + t * 1e-3, 3)
    open(out_md, "w").write("\n".join(lines) + "\n")
    json.dump({"source": f"{out_md} (ncu --set full --clock-control none, steady frame 1 of one lane = 8 of 16 x 1080p streams; "
                         "default cache control: caches flushed before each kernel)", "kernels": traffic},
              open(out_json, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:4])
