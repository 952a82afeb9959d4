"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) and executed warp
instructions (smsp__inst_executed.sum) of the step's kernels from
ncu --set full reports -> profiles/ncu_traffic.json, read by bench.py for the roofline `traffic` key.

  python tools/ncu_traffic.py OUT.json REPORT.ncu-rep [REPORT.ncu-rep ...]
"""
import csv
import io
import json
import subprocess
import sys

PHASE = {"raster_bwd": "raster_bwd", "raster_fwd": "raster_fwd", "dec1_": "decoder", "dec2_": "decoder",
         "dec_reduce": "decoder", "tile_sort": "bin", "scatter_kernel": "bin", "project_kernel": "bin",
         "project_bwd": "project_bwd", "adam_update": "adam"}


def main():
    out, reps = sys.argv[1], sys.argv[2:]
    per_kernel = {}
    for rep in reps:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(txt)))
        h, units = rows[0], rows[1]
        for r in rows[2:]:
            d = dict(zip(h, r))
            name = d["Kernel Name"].split("(")[0].split("::")[-1]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            b = 0.0
            for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                b += float(d[k]) * scale[dict(zip(h, units))[k]]
            tu = dict(zip(h, units))["gpu__time_duration.sum"]
            us = float(d["gpu__time_duration.sum"]) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[tu]
            wi = float(d.get("smsp__inst_executed.sum", "0") or 0)
            per_kernel.setdefault(name, []).append((b, us, wi))
    res = {"source": reps, "kernels": {}}
    for name, v in per_kernel.items():
        res["kernels"][name] = {"bytes_per_launch": sum(x[0] for x in v) / len(v),
                                "ncu_us_per_launch": sum(x[1] for x in v) / len(v), "launches": len(v),
                                "warp_instructions_per_launch": sum(x[2] for x in v) / len(v),
                                "phase": next((p for k, p in PHASE.items() if k in name), None)}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res["kernels"], indent=1))


if __name__ == "__main__":
    main()
