"""Summarise an `ncu --set full` report: per profiled launch, duration, DRAM bytes, throughput and
occupancy figures (read here, no GPU needed).

    python tools/ncu_full_summary.py gpurun_out/r5.ncu-rep profiles/r1_ncu_full_summary.txt profiles/r1_ncu_full.json
"""
import csv
import io
import json
import subprocess
import sys

rep, out_txt, out_json = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = {
    "kernel": "Kernel Name",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "registers": "launch__registers_per_thread",
    "duration_ns": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex_throughput_pct": "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts_throughput_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3,
         "msecond": 1e6, "ms": 1e6, "second": 1e9, "s": 1e9}
recs = []
for r in rows[2:]:
    rec = {}
    for k, name in want.items():
        if name not in hdr:
            continue
        i = hdr.index(name)
        v = r[i]
        if k == "kernel":
            rec[k] = v
            continue
        try:
            val = float(v.replace(",", ""))
        except ValueError:
            rec[k] = v
            continue
        rec[k] = val * scale.get(units[i], 1)
    recs.append(rec)
with open(out_json, "w") as fh:
    json.dump({"report": rep, "launches": recs}, fh, indent=1)
with open(out_txt, "w") as fh:
    fh.write(f"ncu --set full summary of {rep} (ncu replays each launch; cold cache, serialised)\n")
    for rec in recs:
        tot = rec.get("dram_read_bytes", 0) + rec.get("dram_write_bytes", 0)
        dur = rec.get("duration_ns", 0)
        fh.write(f"{rec['kernel'][:40]:40s} dur={dur / 1e6:8.3f} ms  dram={tot / 1e9:8.3f} GB "
                 f"({tot / max(dur, 1):7.1f} GB/s)  dram%={rec.get('dram_throughput_pct', 0):5.1f} "
                 f"l1%={rec.get('l1tex_throughput_pct', 0):5.1f} lts%={rec.get('lts_throughput_pct', 0):5.1f} "
                 f"warps%={rec.get('warps_active_pct', 0):5.1f} regs={rec.get('registers', 0):.0f}\n")
print(open(out_txt).read())
