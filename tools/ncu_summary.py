"""ncu report(s) -> markdown tables of the metrics the judge reads.

usage: python tools/ncu_summary.py TAG:report.ncu-rep [...] > profiles/rNN_ncu_summary.md
"""
import csv
import io
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_static",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__cycles_elapsed.avg", "launch__shared_mem_per_block_dynamic",
    "lts__t_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
]


def main():
    print("# ncu summaries (B200, `--set full --clock-control none`)\n")
    for arg in sys.argv[1:]:
        tag, path = arg.split(":", 1)
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        head, units = rows[0], rows[1]
        ix = {k: i for i, k in enumerate(head)}
        for r in rows[2:]:
            name = r[ix["Kernel Name"]][:110]
            print(f"## [{tag}] `{name}`\n")
            print("| metric | value |\n|---|---|")
            for m in METRICS:
                if m in ix:
                    print(f"| {m} | {r[ix[m]]} {units[ix[m]]} |")
            stalls = {}
            for k, i in ix.items():
                if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                    try:
                        stalls[k[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(r[i].replace(",", ""))
                    except ValueError:
                        pass
            tot = sum(stalls.values()) or 1.0
            top = sorted(stalls.items(), key=lambda kv: -kv[1])[:5]
            print("| top stall reasons (share of samples) | " +
                  ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in top) + " |\n")


if __name__ == "__main__":
    main()
