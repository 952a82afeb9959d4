"""Per-CUDA-source-line instruction and stall shares of one kernel in an ncu report
(`--page source --print-source cuda,sass`; the kernel must be compiled with -lineinfo).

  python tools/ncu_lines.py REPORT KERNEL_REGEX [--top N]
"""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("kernel")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--regions", default="", help="name:first-last,... line ranges of the kernel's file to total")
    a = ap.parse_args()
    txt = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "-k", "regex:" + a.kernel], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    out, hdr, fname = [], None, "?"
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if len(r) > 4 and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr) or not r[0]:
            continue
        try:
            e = float(r[hdr.index("Instructions Executed")] or 0)
            s = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except ValueError:
            continue
        out.append((e, s, f"{fname}:{r[0]}", r[1].strip()[:96]))
    te = sum(x[0] for x in out) or 1.0
    ts = sum(x[1] for x in out) or 1.0
    print(f"# {a.kernel}: {te:.3e} warp instructions, {ts:.0f} stall samples")
    for e, s, loc, src in sorted(out, key=lambda x: -x[1])[: a.top]:
        print(f"{100 * e / te:5.1f}% inst {100 * s / ts:5.1f}% stall  {loc:>16s}  {src}")
    if a.regions:
        print("# regions")
        for spec in a.regions.split(","):
            name, rng = spec.split(":")
            lo, hi = (int(x) for x in rng.split("-"))
            e = sum(x[0] for x in out if lo <= int(x[2].split(":")[-1]) <= hi)
            st = sum(x[1] for x in out if lo <= int(x[2].split(":")[-1]) <= hi)
            print(f"{100 * e / te:5.1f}% inst {100 * st / ts:5.1f}% stall  {name} ({lo}-{hi})")


if __name__ == "__main__":
    main()
