"""latmap::Config text format (src/config.cpp): parse / validate / serialise, and the split into
the C-ABI configs. CPU only."""
import numpy as np
import pytest

from paper_2602_12314_b200 import api, config_io
from paper_2602_12314_b200._capi import InvalidArgument


def test_default_serialisation_round_trips():
    d = config_io.default_config()
    text = config_io.serialize_config(d)
    lines = text.splitlines()
    assert lines[0] == "query_dim = 32" and lines[-1] == "feature_supervision = pixel"
    assert "lr_position = 9.99999975e-05" in lines and "local_mapping = true" in lines
    assert "hash_capacity = 1048576" in lines and len(lines) == len(config_io.FIELDS)
    assert config_io.parse_config(text) == d


def test_parse_rules():
    c = config_io.parse_config("# comment\n\n  lambda_feat = 2.5   # trailing\nseed=18446744073709551615\r\n"
                               "dict_init = random\nlocal_mapping = 0\n")
    assert c["lambda_feat"] == 2.5 and c["seed"] == (1 << 64) - 1 and c["dict_init"] == "random"
    assert c["local_mapping"] is False and c["query_dim"] == 32
    for bad, msg in (("query_dim 3", "line 1: missing '='"), ("\nnope = 1", "line 2: unknown key 'nope'"),
                     ("lambda_cos = 1.0x", "bad float value '1.0x'"), ("dict_learn = yes", "bad bool value"),
                     ("stage1_iters = 1e3", "bad int value"), ("dict_init = other", "dict_init must be kmeans|random"),
                     ("query_dim = 100", "query_dim must be <= embed_dim"), ("dict_decay = 0", "dict_decay")):
        with pytest.raises(InvalidArgument, match=msg):
            config_io.parse_config(bad)
    with pytest.raises(OverflowError):
        config_io.parse_config("query_dim = 4294967296")


def test_float_values_round_trip_exactly():
    g = np.random.default_rng(0)
    c = config_io.default_config()
    for k in ("lambda_cos", "lr_dict", "voxel_size", "softmax_temp"):
        c[k] = float(np.float32(g.uniform(0.001, 3)))
    c2 = config_io.parse_config(config_io.serialize_config(c))
    assert all(c2[k] == c[k] for k in c)


def test_save_load(tmp_path):
    c = config_io.default_config()
    c["stage2_iters"] = 3
    config_io.save_config(c, str(tmp_path / "c.txt"))
    assert config_io.load_config(str(tmp_path / "c.txt")) == c
    with pytest.raises(RuntimeError, match="cannot open config file"):
        config_io.load_config(str(tmp_path / "missing.txt"))


def test_to_latmap_matches_library_defaults():
    cfg, pc = config_io.to_latmap(config_io.default_config())
    ref = api.default_config()
    for f, _ in cfg._fields_:
        assert getattr(cfg, f) == getattr(ref, f), f
    pref = api.default_pipeline_config()
    for f, _ in pc._fields_:
        assert getattr(pc, f) == getattr(pref, f), f
    c = config_io.parse_config("feature_supervision = segment\ndict_learn = false\ndict_init = random\n")
    cfg, pc = config_io.to_latmap(c)
    assert cfg.segment_mode == 1 and cfg.dict_learn == 0 and pc.dict_init == 1
