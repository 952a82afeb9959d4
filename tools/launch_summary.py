"""Per-kernel share / mean duration from an ncu `--metrics gpu__time_duration.sum --csv` launch list."""
import collections
import csv
import sys


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[2:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        name = r[ki].split("(")[0].replace("lm::<unnamed>::", "").replace("void ", "")
        tot[name] += v
        cnt[name] += 1
    total = sum(tot.values())
    print("  share     avg_us      n  kernel")
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
        print(f"{100 * v / total:6.2f}% {v / cnt[k] / 1e3:9.1f} {cnt[k]:6d}  {k}")


if __name__ == "__main__":
    main()
