"""Summarise an .ncu-rep: headline metrics, stall reasons, SASS opcode mix."""
import collections, csv, io, subprocess, sys

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[2:]

def main(rep, top=20):
    hdr, rows = raw(rep)
    keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__warps_active.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "l1tex__throughput.avg.pct_of_peak_sustained_active",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
    for r in rows:
        for k in keys:
            if k in hdr:
                print(f"{k} = {r[hdr.index(k)]}")
        pipes = [(h, r[i]) for i, h in enumerate(hdr)
                 if ("pipe" in h or "mio" in h or "lsu" in h) and h.endswith("pct_of_peak_sustained_active")]
        pipes = sorted(((h, float(v)) for h, v in pipes if v not in ("", "n/a")), key=lambda x: -x[1])
        print("pipes:", ", ".join(f"{h.replace('.avg.pct_of_peak_sustained_active','')}={v:.1f}" for h, v in pipes[:14]))
        st = [(h, r[i]) for i, h in enumerate(hdr) if "smsp__average_warps_issue_stalled" in h and "not_issued" not in h]
        st = sorted(st, key=lambda x: -float(x[1] or 0))
        print("stalls:", ", ".join(f"{h.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio','')}={float(v):.2f}" for h, v in st[:8]))
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(out)))
    if len(srows) > 2:
        h = srows[1]; ie = h.index("Instructions Executed"); src = h.index("Source")
        ops = collections.Counter()
        for r in srows[2:]:
            t = r[src].split()
            if t:
                ops[t[1] if t[0].startswith("@") else t[0]] += int(r[ie] or 0)
        tot = sum(ops.values())
        print("opcode mix:", ", ".join(f"{op} {100*c/tot:.1f}%" for op, c in ops.most_common(top)))

if __name__ == "__main__":
    main(sys.argv[1])
