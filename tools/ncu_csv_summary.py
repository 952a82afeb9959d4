#!/usr/bin/env python
"""Summaries of ncu --csv metric logs (tools/profile_r02.sh): per kernel, the launch count and
the mean of every metric; with --launches, the per-kernel time shares of a launch list."""
import argparse
import collections
import csv
import re


def load(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hi]
    ik, im, iv, iu = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    iid = hdr.index("ID")
    out = collections.OrderedDict()
    for r in rows[hi + 1:]:
        name = re.sub(r"\(anonymous namespace\)::|lm::|void ", "", r[ik].split("(")[0])
        try:
            v = float(r[iv].replace(",", ""))
        except ValueError:
            continue
        out.setdefault(name, collections.defaultdict(dict))[f"{r[im]} [{r[iu]}]"][r[iid]] = v
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--launches", action="store_true")
    a = ap.parse_args()
    k = load(a.csv)
    if a.launches:
        tot = {n: sum(m["gpu__time_duration.sum [ns]"].values()) for n, m in k.items()}
        cnt = {n: len(m["gpu__time_duration.sum [ns]"]) for n, m in k.items()}
        allt = sum(tot.values())
        print(f"# {a.csv}: {sum(cnt.values())} launches, {allt / 1e3:.1f} us total (cold, serialised)")
        print(f"{'kernel':70s} {'n':>5s} {'total us':>10s} {'avg us':>9s} {'share':>6s}")
        for n in sorted(tot, key=lambda x: -tot[x]):
            print(f"{n[:70]:70s} {cnt[n]:5d} {tot[n] / 1e3:10.1f} {tot[n] / cnt[n] / 1e3:9.1f} {tot[n] / allt:6.1%}")
        return
    for n, m in k.items():
        print(n, f"({len(next(iter(m.values())))} launches, means)")
        for mm, vs in m.items():
            print(f"    {mm:75s} {sum(vs.values()) / len(vs):.4g}")


if __name__ == "__main__":
    main()
