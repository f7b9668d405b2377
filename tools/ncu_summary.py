"""One-screen summary of an `ncu --set full` report (run where `ncu` is on PATH):
duration, tensor-pipe (tcgen05 UTCHMMA) and XU (MUFU) utilisation, L2 / DRAM
throughput and bytes, issue activity, occupancy and the top stall reasons.

    python tools/ncu_summary.py report.ncu-rep [more.ncu-rep ...]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration (us)", 1e-3),
    ("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe, tcgen05 bf16 MMA (% of peak, elapsed)", 1),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU / MUFU pipe (% of peak, active)", 1),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput (% of peak)", 1),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput (% of peak)", 1),
    ("dram__bytes_read.sum", "DRAM read (MB)", 1),
    ("dram__bytes_write.sum", "DRAM write (MB)", 1),
    ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue slots busy (%)", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy (%)", 1),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    for rep in sys.argv[1:]:
        hdr, units, data = raw(rep)
        for r in data:
            name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
            print(f"== {rep}: {name[:110]}")
            for key, label, scale in KEYS:
                if key in hdr:
                    v = r[hdr.index(key)]
                    u = units[hdr.index(key)]
                    try:
                        f = float(v.replace(",", ""))
                        if u == "byte" or u == "Kbyte" or u == "Mbyte":
                            f = f * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0}[u]
                        elif u in ("ns", "usecond", "msecond"):
                            f = f * {"ns": 1e-3, "usecond": 1.0, "msecond": 1e3}[u]
                        print(f"   {label:52s} {f:12.2f}")
                    except ValueError:
                        print(f"   {label:52s} {v}")
            pre = "smsp__pcsamp_warps_issue_stalled_"
            vals = []
            for i, k in enumerate(hdr):
                if k.startswith(pre) and not k.endswith("_not_issued"):
                    try:
                        vals.append((float(r[i].replace(",", "")), k[len(pre):]))
                    except ValueError:
                        pass
            tot = sum(v for v, _ in vals) or 1.0
            top = sorted(vals, reverse=True)[:6]
            print("   top stall reasons (share of PC samples): " +
                  ", ".join(f"{n} {v / tot:.0%}" for v, n in top))


if __name__ == "__main__":
    main()
