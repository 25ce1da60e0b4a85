"""Summarise an ncu report (.ncu-rep) into the numbers quoted in profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--sass]  > profiles/<name>.md

Per kernel: duration, DRAM bytes, FMA-pipe and issue utilisation, shared-memory wavefronts
and bank conflicts, registers, top stall reasons; with --sass, the share of warp-stall samples
per barrier-delimited SASS region of the first kernel.
"""

import csv
import io
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__cluster_dim_x", "sm__cycles_active.avg",
]


def ncu(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    rows = ncu(rep, "--page", "raw", "--csv")
    hdr, units = rows[0], rows[1]
    print(f"# ncu summary of `{rep}`\n")
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        print(f"## {name[:120]}\n")
        print("| metric | value |\n|---|---|")
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                print(f"| {m} | {r[i]} {units[i]} |")
        stall = [(float(r[i]) if r[i] else 0.0, h) for i, h in enumerate(hdr)
                 if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio")]
        stall.sort(reverse=True)
        print("\nTop stall reasons (warps per issued instruction):\n")
        for v, h in stall[:8]:
            print(f"- {h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}: {v:.3f}")
        print()
    if "--sass" in sys.argv:
        rows = ncu(rep, "--page", "source", "--csv", "--print-source=sass")
        hdr = rows[1]
        ia, isrc = hdr.index("Address"), hdr.index("Source")
        isamp = hdr.index("Warp Stall Sampling (All Samples)")
        seen, data = set(), []
        for r in rows[2:]:
            if len(r) != len(hdr) or r[0] == "Address":
                continue
            if r[ia] in seen:
                break
            seen.add(r[ia])
            data.append(r)

        def f(x):
            try:
                return float(x)
            except ValueError:
                return 0.0
        tot = sum(f(r[isamp]) for r in data) or 1.0
        base = int(data[0][ia], 16)
        segs, cur = [], []
        for r in data:
            cur.append(r)
            op = r[isrc]
            if "BAR." in op or "UCGABAR_WAIT" in op or "EXIT" in op or "SYNCS" in op:
                segs.append(cur)
                cur = []
        segs.append(cur)
        print("## Warp-stall samples by barrier-delimited SASS region (first kernel)\n")
        print("| region | share | instructions | FFMA | ends with |\n|---|---|---|---|---|")
        for sgm in segs:
            samp = sum(f(r[isamp]) for r in sgm)
            if samp / tot < 0.005:
                continue
            a0, a1 = int(sgm[0][ia], 16) - base, int(sgm[-1][ia], 16) - base
            nffma = sum(1 for r in sgm if "FFMA" in r[isrc])
            print(f"| {a0:#07x}-{a1:#07x} | {samp / tot * 100:.1f}% | {len(sgm)} | {nffma} | `{sgm[-1][isrc].strip()[:40]}` |")


if __name__ == "__main__":
    main()
