"""Summarise an ncu --set full report: headline metrics, pipe utilisation, stall reasons and
(with --source) the hottest source lines by warp stall samples. Used to write profiles/*.txt."""
import argparse
import csv
import io
import subprocess
import sys

KEYS = (
    "gpu__time_duration.sum", "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
)


def ncu(args):
    return subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--source", type=int, default=0, help="print the N hottest source lines")
    a = ap.parse_args()
    rows = list(csv.reader(io.StringIO(ncu(["-i", a.rep, "--page", "raw", "--csv"]))))
    h, units = rows[0], rows[1]
    for row in rows[2:]:
        d = dict(zip(h, row))
        u = dict(zip(h, units))
        print(f"kernel: {d.get('Kernel Name', '?')[:100]}")
        for k in KEYS:
            if k in d:
                print(f"  {k} = {d[k]} {u.get(k, '')}")
        for k in sorted(h):
            if k.startswith("sm__inst_executed_pipe_") and k.endswith("avg.pct_of_peak_sustained_active"):
                try:
                    if float(d[k]) >= 1.0:
                        print(f"  {k} = {d[k]}")
                except ValueError:
                    pass
        st = []
        for k in h:
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(d[k]), k))
                except ValueError:
                    pass
        for v, k in sorted(st, reverse=True)[:8]:
            print(f"  stall {k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]} = {v:.3f}")
    if a.source:
        txt = ncu(["-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"])
        r = list(csv.reader(io.StringIO(txt)))
        if len(r) < 2:
            return
        r = r[1:]
        hh = r[0]
        try:
            ci = hh.index("Warp Stall Sampling (All Samples)")
        except ValueError:
            print("no stall sampling column", hh[:8])
            return
        li, si = hh.index("Address"), hh.index("Source")
        body = []
        for x in r[1:]:
            try:
                body.append((float(x[ci] or 0), x[li], x[si].strip()[:110]))
            except (ValueError, IndexError):
                pass
        tot = sum(b[0] for b in body) or 1.0
        print(f"  hottest SASS instructions (share of warp stall samples):")
        for v, ln, src in sorted(body, reverse=True)[: a.source]:
            print(f"    {100 * v / tot:5.1f}%  {ln[-5:]}: {src}")
        ops = {}
        for v, _, src in body:
            op = src.split()[0] if src.split() else "?"
            if op.startswith("@"):
                op = src.split()[1] if len(src.split()) > 1 else op
            op = op.split(".")[0]
            ops[op] = ops.get(op, 0.0) + v
        print("  stall samples by opcode: " + ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in
                                                        sorted(ops.items(), key=lambda t: -t[1])[:14]))


if __name__ == "__main__":
    sys.exit(main())
