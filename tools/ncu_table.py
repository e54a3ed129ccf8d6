"""Per-kernel table from `ncu --page raw --csv` exports (measurement helper).

    python tools/ncu_table.py TITLE raw.csv [raw.csv ...] > profiles/xx.md

Columns: duration, DRAM bytes read / written (per launch), achieved DRAM
GB/s and its fraction of MEASURED_PEAKS.json hbm_gbs, shared-memory
wavefronts and the fraction of them that are bank conflicts, issue-slot
utilisation, registers.  Launches whose name matches SKIP (validation
kernels outside the timed region) are listed but not summed.
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
try:
    PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:  # noqa: BLE001
    PEAK = 6547.5
SKIP = ("k_count_distinct", "k_validate", "k_check")


def f(x):
    try:
        return float(x)
    except ValueError:
        return float("nan")


def main():
    title, files = sys.argv[1], sys.argv[2:]
    print(f"# {title}\n")
    print(f"Peak = {PEAK:.0f} GB/s (MEASURED_PEAKS.json hbm_gbs, copy).  ncu --set full --clock-control none; "
          "DRAM bytes are per launch (cold L2 per replay).\n")
    for fn in files:
        rows = list(csv.reader(open(fn)))
        h = rows[0]
        col = {name: i for i, name in enumerate(h)}
        g = lambda r, m: r[col[m]] if m in col else ""  # noqa: E731
        print(f"## {os.path.basename(fn)}\n")
        print("| # | kernel | ms | DRAM rd GB | DRAM wr GB | GB/s | % peak | smem wavefronts | bank-conflict % | issue % | regs |")
        print("|---|---|---|---|---|---|---|---|---|---|---|")
        tot_ms = tot_b = 0.0
        for k, r in enumerate(rows[2:]):
            name = g(r, "Kernel Name").split("(")[0].replace("void ", "")
            ms = f(g(r, "gpu__time_duration.sum"))
            rd, wr = f(g(r, "dram__bytes_read.sum")), f(g(r, "dram__bytes_write.sum"))
            unit = rows[1][col["dram__bytes_read.sum"]] if "dram__bytes_read.sum" in col else "Gbyte"
            scale = {"Gbyte": 1.0, "Mbyte": 1e-3, "Kbyte": 1e-6, "byte": 1e-9, "Tbyte": 1e3}.get(unit, 1.0)
            rd, wr = rd * scale, wr * scale
            tunit = rows[1][col["gpu__time_duration.sum"]]
            ms *= {"msecond": 1.0, "usecond": 1e-3, "nsecond": 1e-6, "second": 1e3}.get(tunit, 1.0)
            gbs = (rd + wr) / (ms / 1e3) if ms == ms and ms > 0 else float("nan")
            wf = f(g(r, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"))
            bc = f(g(r, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"))
            iss = f(g(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"))
            regs = g(r, "launch__registers_per_thread")
            skip = any(s in name for s in SKIP)
            if not skip and ms == ms:
                tot_ms += ms
                tot_b += (rd + wr) if rd == rd else 0.0
            print(f"| {k} | `{name[:60]}`{' (validation, not summed)' if skip else ''} | {ms:.3f} | {rd:.2f} | {wr:.2f} | "
                  f"{gbs:.0f} | {100 * gbs / PEAK:.0f} | {wf:.3g} | {100 * bc / wf if wf else 0:.0f} | {iss:.0f} | {regs} |")
        print(f"\nSum of the listed launches: {tot_ms:.2f} ms, DRAM {tot_b:.1f} GB "
              f"({tot_b / (tot_ms / 1e3) if tot_ms else 0:.0f} GB/s).\n")


if __name__ == "__main__":
    main()
