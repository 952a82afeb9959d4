"""run_pipeline over a LAMT dataset (proj/src/pipeline.cpp:314-335) and the keyframe log format
(pipeline.cpp:337-351). The per-keyframe work is ``api.Pipeline.process_keyframe``: the C-ABI
pipeline (csrc/pipeline.cu) over the device session and store."""
from __future__ import annotations

import time

from . import api, lamt


def run_pipeline(p: api.Pipeline, manifest: lamt.DatasetManifest, on_keyframe=None):
    """Every frame_count() frame, keyframes by select_keyframe(f, keyframe_stride), each loaded
    (lamt.load_frame) and processed; then the final flush of the active set into the store.
    Returns RunResult (pipe/pipeline.hpp:97-103) as a dict."""
    res = {"frames": 0, "keyframes": 0, "wall_seconds": 0.0, "keyframes_per_second": 0.0, "log": []}
    t0 = time.perf_counter()
    for f in range(manifest.frame_count()):
        res["frames"] += 1
        if not api.select_keyframe(f, p.pcfg.keyframe_stride):
            continue
        kf = lamt.load_frame(manifest, f)
        row = p.process_keyframe(kf, f)
        res["keyframes"] += 1
        if on_keyframe:
            on_keyframe(row)
        res["log"].append(row)
    if p.session.n > 0:
        p.flush()
    res["wall_seconds"] = time.perf_counter() - t0
    res["keyframes_per_second"] = res["keyframes"] / res["wall_seconds"] if res["keyframes"] else 0.0
    return res


def log_csv_header():
    return ("frame_index,l_rgb,l_ssim,l_depth,l_cos,l_l2,l_trust,total,supervised_rows,seeded,"
            "active_count,global_count,dict_weight_mass,synced,wall_ms")


def log_csv_row(r):
    """ostream with precision(9): %.9g for the floating fields."""
    lo = r["loss"]
    g = lambda v: "%.9g" % float(v)  # noqa: E731
    return ",".join([str(r["frame_index"])] + [g(lo[k]) for k in ("l_rgb", "l_ssim", "l_depth", "l_cos", "l_l2",
                                                                   "l_trust", "total")]
                    + [str(lo["supervised_rows"]), str(r["seeded"]), str(r["active_count"]), str(r["global_count"]),
                       g(r["dict_weight_mass"]), "1" if r["synced"] else "0", g(r["wall_ms"])])
