#!/usr/bin/env python
"""Per-source-line warp-stall attribution from an ncu report (the cuda,sass source page):
   python tools/ncu_source_lines.py REPORT.ncu-rep [--kernel REGEX] [--top N]
Prints, for the top-N lines by stall samples, the share of samples, the share of executed
warp instructions and the three largest stall reasons."""
import argparse
import csv
import io
import re
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--kernel", default=None)
    ap.add_argument("--top", type=int, default=40)
    args = ap.parse_args()
    cmd = ["ncu", "-i", args.report, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if args.kernel:
        cmd += ["--kernel-name", f"regex:{args.kernel}"]
    txt = subprocess.run(cmd, capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, fname, out, func = None, None, {}, None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            func = r[1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr and r[0].isdigit() and len(r) > 8:
            try:
                s, ex = int(r[4]), int(r[7])
            except ValueError:
                continue
            stalls = {hdr[i]: float(r[i] or 0) for i in range(len(hdr))
                      if hdr[i].startswith("stall_") and "Not Issued" not in hdr[i] and r[i] not in ("", "-")}
            out[(fname, int(r[0]))] = (s, ex, r[1].strip()[:80], stalls)
    tot = sum(v[0] for v in out.values()) or 1
    totex = sum(v[1] for v in out.values()) or 1
    print(f"# {func}: {tot} stall samples, {totex} warp instructions executed")
    for (f, ln), (s, ex, src, st) in sorted(out.items(), key=lambda kv: -kv[1][0])[:args.top]:
        top3 = ", ".join(f"{k[6:]} {v / max(s, 1) * 100:.0f}%" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3] if v)
        print(f"{100 * s / tot:5.1f}% ex {100 * ex / totex:5.1f}%  {f}:{ln:<5d} [{top3}] {src}")


if __name__ == "__main__":
    main()
