"""Summarise ncu --set full reports into the JSON kept under profiles/.

    python tools/ncu_summary.py OUT.json NAME=report.ncu-rep [NAME=report.ncu-rep ...]

Per kernel launch in each report: duration, DRAM bytes and throughput,
issue activity, pipe utilisation (FP64, FMA, ALU, tensor), occupancy and the
warp-stall shares from the PC sampler."""
import csv
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "sm__cycles_elapsed.avg.per_second",
]


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    head, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        d = dict(zip(head, row))
        u = dict(zip(head, units))
        k = {"Kernel Name": d.get("Kernel Name", "")[:120]}
        for key in KEYS:
            if key in d:
                k[key] = d[key] + (f" {u[key]}" if u.get(key) else "")
        st = {}
        for key, v in d.items():
            if key.startswith("smsp__pcsamp_warps_issue_stalled_") and not key.endswith("not_issued"):
                try:
                    st[key.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v)
                except ValueError:
                    pass
        tot = sum(st.values()) or 1.0
        k["stall_share"] = {a: round(b / tot, 3) for a, b in
                            sorted(st.items(), key=lambda x: -x[1])[:10]}
        res.append(k)
    return res


def main():
    out = sys.argv[1]
    doc = {"source": "ncu --set full --clock-control none (one B200); tools/ncu_summary.py",
           "reports": {}}
    for arg in sys.argv[2:]:
        name, rep = arg.split("=", 1)
        doc["reports"][name] = summarise(rep)
    with open(out, "w") as f:
        json.dump(doc, f, indent=1)


if __name__ == "__main__":
    main()
