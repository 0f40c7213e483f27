"""Summarise ncu --set full reports and launch-list CSVs into markdown (profiles/)."""
import csv, io, subprocess, sys, collections

METRICS = [("gpu__time_duration.sum", "duration"), ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
           ("sm__inst_executed_pipe_uc.avg.pct_of_peak_sustained_active", "uc pipe %"),
           ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
           ("dram__bytes_read.sum", "dram read"), ("dram__bytes_write.sum", "dram write"),
           ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
           ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"),
           ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
           ("l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed", "smem wavefronts %")]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    lines = ["| kernel | " + " | ".join(m[1] for m in METRICS) + " |", "|" + "---|" * (len(METRICS) + 1)]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")[-40:]
        vals = []
        for m, _ in METRICS:
            if m in hdr:
                i = hdr.index(m)
                vals.append(f"{r[i]} {units[i]}".strip())
            else:
                vals.append("n/a")
        lines.append(f"| {name} | " + " | ".join(vals) + " |")
    return "\n".join(lines)


def launches(path, top=14):
    rows = [l for l in open(path) if l.startswith('"')]
    r = [x for x in csv.DictReader(io.StringIO("".join(rows))) if x["Metric Name"] == "gpu__time_duration.sum"]
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for x in r:
        k = x["Kernel Name"].split("(")[0].replace("void ", "").replace("unnamed>::", "")
        tot[k] += float(x["Metric Value"]) / 1e3
        cnt[k] += 1
    T = sum(tot.values())
    lines = [f"{len(r)} launches, {T/1e3:.2f} ms total (serialised, cold-cache: compare shares)", "",
             "| kernel | launches | total ms | avg us | share |", "|---|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda z: -z[1])[:top]:
        lines.append(f"| {k} | {cnt[k]} | {v/1e3:.2f} | {v/cnt[k]:.1f} | {100*v/T:.1f}% |")
    return "\n".join(lines)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"### {p}\n")
        print(report(p) if p.endswith(".ncu-rep") else launches(p))
        print()
