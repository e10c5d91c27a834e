"""Summarise an ncu report: time, DRAM bytes, throughput, issue, stalls.
    python tools/ncu_summary.py rep.ncu-rep [...]"""
import csv, io, subprocess, sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy%"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__inst_executed.sum", "inst"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("smsp__average_warp_latency_per_inst_issued.ratio", "cyc/inst"),
]
STALLS = ["long_scoreboard", "short_scoreboard", "wait", "barrier", "math_pipe_throttle",
          "mio_throttle", "lg_throttle", "not_selected", "selected", "no_instruction",
          "dispatch_stall", "drain", "membar", "sleeping", "branch_resolving", "tex_throttle",
          "imc_miss", "misc"]

for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        print(f"== {rep}: {r[idx['Kernel Name']][:80]}")
        for k, short in KEYS:
            if k in idx:
                print(f"   {short:12s} {r[idx[k]]} {units[idx[k]]}")
        st = []
        for s in STALLS:
            k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if k in idx:
                try:
                    st.append((float(r[idx[k]]), s))
                except ValueError:
                    pass
        st.sort(reverse=True)
        print("   stalls/issue:", ", ".join(f"{s}={v:.2f}" for v, s in st[:8]))
