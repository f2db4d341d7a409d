"""DRAM traffic and pipe utilisation of one kernel launch from an `ncu --set full` report, as the JSON that
bench.py's roofline reads (`traffic`, `compute`).
   python tools/ncu_traffic.py report.ncu-rep "workload" > profiles/<round>_ncu_fwd_bwd_traffic.json"""
import csv
import io
import json
import subprocess
import sys

rep, workload = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]


def val(name):
    if name not in hdr:
        return None
    i = hdr.index(name)
    v = float(vals[i].replace(",", ""))
    u = units[i]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
             "nsecond": 1e-9, "msecond": 1e-3}.get(u, 1)
    return v * scale


rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
out = {
    "kernel": vals[hdr.index("Kernel Name")],
    "workload": workload,
    "dram_bytes_read": rd,
    "dram_bytes_write": wr,
    "duration_s": val("gpu__time_duration.sum"),
    "capture": "ncu --set full --clock-control none (cache control all: cold caches per replay)",
    "traffic_bytes": (rd or 0) + (wr or 0),
    "sm_throughput_pct_of_peak": val("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    "issue_active_pct_of_peak": val("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "fp64_pipe_active_pct_of_peak": val("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    "fma_pipe_active_pct_of_peak": val("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    "alu_pipe_active_pct_of_peak": val("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
    "note": "sm__throughput / smsp__issue_active / sm__pipe_{fp64,fma,alu}_cycles_active from the same capture: "
            "the kernel is issue/latency bound (exact double-double reduction, no-FMA parity arithmetic), not DRAM bound",
}
print(json.dumps(out, indent=1))
