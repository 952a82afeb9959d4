"""Pipeline host logic without a GPU: the reference's Config defaults for the pipeline fields
(core/config.hpp:10-58), select_keyframe (pipeline.cpp:14-17) and the CSV log format
(pipeline.cpp:337-351)."""
import numpy as np
import pytest

from paper_2602_12314_b200 import _capi, api, pipeline as pl


def test_default_pipeline_config_matches_reference():
    pc = api.default_pipeline_config()
    assert (pc.query_dim, pc.embed_dim, pc.dict_size) == (32, 64, 2000)
    assert (pc.stage1_iters, pc.stage2_iters, pc.history_sample, pc.history_capacity) == (1, 5, 5, 200)
    assert pc.voxel_size == pytest.approx(0.01) and pc.local_radius == 5.0 and pc.sync_distance == 1.0
    assert pc.hash_capacity == 1 << 20 and pc.local_mapping == 1 and pc.keyframe_stride == 4 and pc.seed == 0
    assert pc.dict_init == 0 and pc.dict_decay == 1.0 and pc.trust_anchor_persistent == 0
    assert api.default_pipeline_config(dict_init="random").dict_init == 1


def test_select_keyframe():
    assert [api.select_keyframe(f, 4) for f in range(6)] == [True, False, False, False, True, False]
    assert api.select_keyframe(3, 1)
    with pytest.raises(_capi.InvalidArgument):
        api.select_keyframe(0, 0)


def test_log_csv_format():
    f = lambda v: float(np.float32(v))  # noqa: E731  (LossBreakdown<float> fields)
    row = {"frame_index": 8, "loss": {"l_rgb": f(0.1), "l_ssim": f(0.25), "l_depth": 0.0, "l_cos": f(1 / 3),
                                      "l_l2": 2.0, "l_trust": 0.0, "total": 12.5, "supervised_rows": 307200},
           "seeded": 17, "active_count": 1000, "global_count": 5000, "dict_weight_mass": 48.0, "synced": True,
           "wall_ms": 12.25}
    assert pl.log_csv_header().count(",") == 14
    assert pl.log_csv_row(row) == ("8,0.100000001,0.25,0,0.333333343,2,0,12.5,307200,17,1000,5000,48,1,12.25")
