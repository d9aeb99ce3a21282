"""Summarise ncu output into the markdown committed under profiles/.

  python tools/ncu_summary.py --rep gpurun_out/prof.ncu-rep [--launches gpurun_out/launches.csv] > profiles/rN_ncu.md

--rep: a `ncu --set full` report; prints one row per profiled launch with
duration, DRAM bytes (read + write = the roofline `traffic`), achieved DRAM
GB/s, SM / ALU / FMA / LSU pipe utilisation, registers and occupancy.
--launches: a `ncu --metrics gpu__time_duration.sum --csv` launch list;
prints each kernel's share of the summed device time (cold-cache, serialised:
compare shares, not absolutes).
"""
import argparse
import collections
import csv
import io
import subprocess
import sys

METRICS = {
    "dur_us": "gpu__time_duration.sum",
    "dram_rd": "dram__bytes_read.sum",
    "dram_wr": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "alu_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "fma_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "lsu_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "occ": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "bank_conf": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "issue_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "fmaheavy_pct": "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "warp_inst_M": "smsp__inst_executed.sum",
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3,
              "ns": 1e-3, "us": 1, "ms": 1e3}


def rep_rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        rec = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")[:48],
               "grid": r[hdr.index("Grid Size")]}
        for k, m in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    rec[k] = float(r[i].replace(",", "")) * UNIT_SCALE.get(units[i], 1)
                except ValueError:
                    rec[k] = None
        yield rec


def fmt(v, p=1):
    return "-" if v is None else f"{v:.{p}f}"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    a = ap.parse_args()
    if a.rep:
        print("| kernel | grid | us | DRAM MB (rd+wr) | DRAM GB/s | DRAM % | SM % | ALU % | FMA % | LSU % | regs | warps % | smem bank conflicts | issue % | fmaheavy % | warp-inst M |")
        print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
        for rep in a.rep.split(","):
          for r in rep_rows(rep):
            tb = (r.get("dram_rd") or 0) + (r.get("dram_wr") or 0)
            gbs = tb / (r["dur_us"] * 1e-6) / 1e9 if r.get("dur_us") else None
            wi = r.get("warp_inst_M")
            print(f"| {r['kernel']} | {r['grid']} | {fmt(r.get('dur_us'))} | {tb / 1e6:.1f} | {fmt(gbs, 0)} | "
                  f"{fmt(r.get('dram_pct'))} | {fmt(r.get('sm_pct'))} | {fmt(r.get('alu_pct'))} | "
                  f"{fmt(r.get('fma_pct'))} | {fmt(r.get('lsu_pct'))} | {fmt(r.get('regs'), 0)} | "
                  f"{fmt(r.get('occ'))} | {fmt(r.get('bank_conf'), 0)} | {fmt(r.get('issue_pct'))} | "
                  f"{fmt(r.get('fmaheavy_pct'))} | {fmt(wi / 1e6 if wi else None)} |")
    if a.launches:
        text = open(a.launches).read()
        lines = [l for l in text.splitlines() if l.startswith('"')]
        rows = list(csv.reader(io.StringIO("\n".join(lines))))
        hdr = rows[0]
        ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
        ui = hdr.index("Metric Unit")
        tot = collections.Counter()
        cnt = collections.Counter()
        for r in rows[1:]:
            if r[mi] != "gpu__time_duration.sum":
                continue
            k = r[ki].split("(")[0].replace("void ", "")[:60]
            tot[k] += float(r[vi].replace(",", "")) * UNIT_SCALE.get(r[ui], 1)
            cnt[k] += 1
        s = sum(tot.values())
        print(f"\nlaunch list: {sum(cnt.values())} launches, {s / 1e3:.2f} ms summed device time\n")
        print("| kernel | launches | total us | share |")
        print("|---|---|---|---|")
        for k, v in tot.most_common():
            print(f"| {k} | {cnt[k]} | {v:.0f} | {100 * v / s:.1f}% |")


if __name__ == "__main__":
    sys.exit(main())
