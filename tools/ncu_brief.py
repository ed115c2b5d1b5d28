"""Key metrics of every kernel in an ncu report (ncu -i ... --page raw --csv)."""
import csv
import io
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__inst_executed.sum": "inst",
    "smsp__inst_executed.avg.per_cycle_active": "ipc_smsp",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__sass_thread_inst_executed_op_dfma_pred_on.sum": "dfma_thread_inst",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum": "dfma_thread_inst",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
}
STALLS = "smsp__pcsamp_warps_issue_stalled_"


def brief(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], dict(zip(rows[0], rows[1]))
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", "?").split("(")[0]
        vals = {v: (d[k] + (units.get(k) or "")) for k, v in KEYS.items() if k in d}
        stalls = sorted(((k[len(STALLS):], float(d[k].replace(",", "") or 0)) for k in hdr
                         if k.startswith(STALLS) and not k.endswith("not_issued") and d[k]),
                        key=lambda x: -x[1])[:6]
        out.append(f"{name}: " + ", ".join(f"{k}={v}" for k, v in vals.items()))
        out.append("   top stalls: " + ", ".join(f"{k}={int(v)}" for k, v in stalls))
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(p)
        print(brief(p))
