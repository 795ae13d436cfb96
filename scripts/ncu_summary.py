"""Summarises one kernel of an ncu --set full report as JSON (dev tool):
python scripts/ncu_summary.py REPORT.ncu-rep [LABEL] [FLOPS]."""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu_time_us": "gpu__time_duration.sum",
    "sm_cycles_active_avg": "sm__cycles_active.avg",
    "tensor_pipe_active_pct_of_active": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "tensor_pipe_active_pct_of_elapsed":
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "xu_pipe_pct_of_active": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "elapsed_cycles": "gpc__cycles_elapsed.max",
    "sm_clock_ghz": "smsp__cycles_elapsed.avg.per_second",
}


def main():
    rep = sys.argv[1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, vals = rows[0], rows[1], rows[2]
    col = {h: i for i, h in enumerate(head)}
    out = {"report": rep.split("/")[-1], "kernel": vals[col["Kernel Name"]] if "Kernel Name" in col else None}
    if len(sys.argv) > 2:
        out["label"] = sys.argv[2]
    for k, m in KEYS.items():
        if m in col:
            try:
                out[k] = float(vals[col[m]])
            except ValueError:
                out[k] = vals[col[m]]
            out[k + "_unit"] = units[col[m]]
    if len(sys.argv) > 3 and "gpu_time_us" in out:
        fl = float(sys.argv[3])
        out["algorithmic_flops"] = fl
        out["achieved_tflops_at_capture_clock"] = fl / (out["gpu_time_us"] * 1e-6) / 1e12
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
