"""Summarise ncu launch-list CSVs (gpu__time_duration + dram bytes) into markdown tables.

usage: launch_summary.py bench.csv refresh.csv > profiles/rNN_launches.md
bench.csv: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size
           --csv --log-file ... python bench.py --steps 2 --warmup 3 --skip-cpu --skip-e2e --skip-adam`
           -> the LAST plain step (from its k_prepare) is split into phases;
refresh.csv: the same metrics over scripts/refresh_t50.py (--profile-from-start off: the t=50 step)."""
import collections, csv, json, re, sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hi]
    ki, mi, vi, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) > vi:
            per.setdefault(r[ii], {"name": r[ki]})[r[mi]] = r[vi]
    out = []
    for l in per.values():
        n = re.sub(r"shampoo::(<unnamed>::)?", "", l["name"].replace("void ", "").split("(")[0])
        f = lambda k: float(l.get(k, "0").replace(",", ""))
        out.append((n, f("gpu__time_duration.sum") / 1e3, (f("dram__bytes_read.sum") + f("dram__bytes_write.sum")) / 1e6,
                    l.get("launch__grid_size", "")))
    return out


def table(launches, title):
    agg = collections.OrderedDict()
    for n, t, b, g in launches:
        a = agg.setdefault(n, [0, 0.0, 0.0])
        a[0] += 1
        a[1] += t
        a[2] += b
    tot = sum(a[1] for a in agg.values())
    lines = [f"### {title}: {len(launches)} launches, {tot / 1e3:.3f} ms (ncu: serialised, cold caches)", "",
             "| kernel | launches | µs | share | DRAM MB | GB/s |", "|---|---|---|---|---|---|"]
    for n, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{n}` | {c} | {t:.1f} | {100 * t / tot:.1f}% | {b:.1f} | {b / t * 1e3 if t else 0:.0f} |")
    return "\n".join(lines), tot


def main():
    bench = load(sys.argv[1])
    start = max(i for i, l in enumerate(bench) if l[0].startswith("k_prepare"))
    plain = bench[start:]
    names = [l[0] for l in plain]
    gv = next(i for i, n in enumerate(names) if n.startswith("grouped_gemv") or i > 0 and n.startswith("k_oz_rowexp") and
              names[:i].count("k_oz_gemm<double, 8>") >= 1)
    sq = next(i for i, n in enumerate(names) if n.startswith("k_sumsq"))
    phases = {"stats (k_prepare .. thin)": plain[:gv], "precondition": plain[gv:sq], "graft/momentum/apply": plain[sq:]}
    out = ["## Plain step (bench workload, last step of the launch list)", ""]
    traffic = {}
    for title, ls in phases.items():
        t, tot = table(ls, title)
        out += [t, ""]
        traffic[title] = sum(l[2] for l in ls) * 1e6
    if len(sys.argv) > 2:
        rf = load(sys.argv[2])
        t, tot = table(rf, "Refresh step t=50 (root inverse + the step's other phases)")
        out += ["## Refresh step", "", t, ""]
        traffic["refresh_step"] = sum(l[2] for l in rf) * 1e6
    print("\n".join(out))
    print("<!-- traffic bytes per phase: " + json.dumps({k: round(v) for k, v in traffic.items()}) + " -->")


main()
