"""Key metrics of an ncu --set full report (per captured launch) as text.
usage: python tools/ncu_summary.py REPORT.ncu-rep [title]"""
import csv
import io
import subprocess
import sys

KEYS = ["Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__icc_request_hit_rate.pct", "sm__cycles_elapsed.avg.per_second"]
STALLS = "smsp__pcsamp_warps_issue_stalled_"


def main():
    rep = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else rep
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    print(f"ncu --set full --clock-control none: {title}")
    for r in rows[2:]:
        print("-" * 100)
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"{k:70s} {r[i]} {units[i]}")
        st = [(float(r[i].replace(",", "") or 0), h[len(STALLS):]) for i, h in enumerate(hdr)
              if h.startswith(STALLS) and not h.endswith("_not_issued") and r[i] not in ("", "n/a")]
        tot = sum(v for v, _ in st) or 1.0
        print("warp stall reasons (share of PC samples):")
        for v, nm in sorted(st, reverse=True)[:10]:
            print(f"  {nm:40s} {100 * v / tot:5.1f}%")


if __name__ == "__main__":
    main()
