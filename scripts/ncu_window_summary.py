"""Summarise an ncu launch list of bench.py's profiled window (SHAMPOO_BENCH_PROFILE=1) into markdown.

    ncu --profile-from-start off --clock-control none --csv --log-file W.csv \
        --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        env SHAMPOO_BENCH_PROFILE=1 python bench.py --steps 3 --skip-cpu --skip-e2e --skip-adam
    python scripts/ncu_window_summary.py W.csv > profiles/rNN_window.md

Steps are split at each `k_finite` launch (the first kernel of every step); the window starts at a
refresh step, so step 0 is the refresh step and the others are plain steps.  ncu serialises the
launches with cold caches: compare SHARES with bench.py's phase split, not absolutes.
"""
import collections
import csv
import re
import sys


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
        base = l["name"].replace("void ", "").split("(")[0]
        lt = base.find("<") if "<" in base else len(base)
        n = base[base.rfind("::", 0, lt) + 2:] if "::" in base[:lt] else base
        f = lambda k: float(l.get(k, "0").replace(",", ""))
        out.append((n, f("gpu__time_duration.sum") / 1e3,
                    (f("dram__bytes_read.sum") + f("dram__bytes_write.sum")) / 1e6))
    return out


def table(launches, title):
    agg = collections.OrderedDict()
    for n, us, mb in launches:
        a = agg.setdefault(n, [0, 0.0, 0.0])
        a[0] += 1
        a[1] += us
        a[2] += mb
    tot = sum(a[1] for a in agg.values())
    print(f"### {title}: {len(launches)} launches, {tot / 1e3:.3f} ms (ncu: serialised, cold caches)\n")
    print("| kernel | launches | µs | share | DRAM MB | GB/s |")
    print("|---|---|---|---|---|---|")
    for n, (c, us, mb) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        if us < 0.002 * tot:
            continue
        print(f"| `{n}` | {c} | {us:.1f} | {100 * us / tot:.1f}% | {mb:.1f} | {mb / us * 1e3 if us else 0:.0f} |")
    print()


def main():
    launches = load(sys.argv[1])
    steps, cur = [], []
    for l in launches:
        if l[0].startswith("k_finite") and cur:
            steps.append(cur)
            cur = []
        cur.append(l)
    if cur:
        steps.append(cur)
    table(steps[0], "Refresh step (steady state)")
    for k, st in enumerate(steps[1:], 1):
        table(st, f"Plain step {k}")


if __name__ == "__main__":
    main()
