"""Summarise one `ncu --set full` capture of K4 into profiles/ncu_k4_summary.json.

    python tools/ncu_summary.py gpurun_out/k4.ncu-rep hv720 "<how it was captured>"

Reads `ncu -i <rep> --page raw --csv`; bench.py takes `traffic` (DRAM bytes per
launch) from the resulting file.
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

rep, config = sys.argv[1], sys.argv[2]
source = sys.argv[3] if len(sys.argv) > 3 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]


def get(name, scale=1.0):
    i = hdr.index(name)
    u = units[i]
    v = float(vals[i].replace(",", ""))
    mult = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12, "ms": 1.0, "us": 1e-3,
            "ns": 1e-6, "Ghz": 1.0, "Mhz": 1e-3}.get(u, 1.0)
    return v * mult * scale


out = {
    "kernel": vals[hdr.index("Kernel Name")],
    "source": source,
    "gpu_time_ms": get("gpu__time_duration.sum"),
    "dram_bytes_read": get("dram__bytes_read.sum"),
    "dram_bytes_write": get("dram__bytes_write.sum"),
    "l2_to_sm_bytes": get("l1tex__m_xbar2l1tex_read_bytes.sum"),
    "l2_hit_rate_pct": get("lts__t_sector_hit_rate.pct"),
    "tensor_pipe_active_pct": get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
    "issue_active_pct": get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "xu_pipe_pct": get("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
    "registers_per_thread": int(get("launch__registers_per_thread")),
    "sm_clock_ghz": get("sm__cycles_elapsed.avg.per_second"),
}
out["dram_bytes_per_launch"] = out["dram_bytes_read"] + out["dram_bytes_write"]
p = Path(__file__).resolve().parents[1] / "profiles" / "ncu_k4_summary.json"
data = json.loads(p.read_text()) if p.exists() else {}
data[config] = out
p.write_text(json.dumps(data, indent=2) + "\n")
print(json.dumps(out, indent=2))
