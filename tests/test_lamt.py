"""LAMT named-tensor files, the dataset layout and the map / dictionary dumps (SURVEY.md §8(f)
row 4), pinned by the reference's own container cases (proj/tests/test_io.cpp:37-125) and the
byte layout of io/tensor_file.hpp:46-50. CPU only."""
import json
import os

import numpy as np
import pytest

from paper_2602_12314_b200 import lamt
from paper_2602_12314_b200._capi import InvalidArgument


def test_empty_container_round_trips():
    b = lamt.write_tensor(lamt.TensorContainer())
    assert b == b"LAMT" + bytes([1, 0, 0, 0, 0, 0, 0, 0])
    back = lamt.read_tensor(b)
    assert back.entries == [] and lamt.write_tensor(back) == b


def test_golden_bytes_single_entry():
    """The byte layout by hand: magic | version | count | name_len | name | dtype | ndim | dims | payload."""
    c = lamt.TensorContainer()
    c.add_f32("x", np.array([1.0, -2.0], np.float32), (2,))
    want = (b"LAMT" + (1).to_bytes(4, "little") + (1).to_bytes(4, "little") + (1).to_bytes(4, "little") + b"x"
            + bytes([1, 1]) + (2).to_bytes(8, "little") + bytes.fromhex("0000803f000000c0"))
    assert lamt.write_tensor(c) == want


def test_typed_entries_round_trip_exactly():
    c = lamt.TensorContainer()
    w = np.array([1.5, -2.25, 0.0, 1e-20, 3e20, -0.625, 7, 8, 9, 10, 11, 12], np.float32)
    c.add_f32("W", w, (3, 4))
    d = np.array([0, 1, 65535, 1234, 40000, 7], np.uint16)
    c.add_u16("depth", d, (2, 3))
    a = np.array([-1, 0, 2147483647, -2147483648], np.int32)
    c.add_i32("assign", a, (4,))
    b = lamt.write_tensor(c)
    # name_len + name + dtype + ndim + dims + payload per entry. test_io.cpp:55-56 writes the "W"
    # term as 4 + 1 + 1 + 2 + 16 + 48 (one byte more than its writer emits, tensor_file.cpp:170-177,
    # so that CHECK cannot pass against the reference's own writer); the writer is followed here.
    assert len(b) == 12 + (4 + 1 + 1 + 1 + 16 + 48) + (4 + 5 + 1 + 1 + 16 + 12) + (4 + 6 + 1 + 1 + 8 + 16)
    back = lamt.read_tensor(b)
    assert np.array_equal(back.get_f32("W"), w)
    assert np.array_equal(back.get_u16("depth"), d)
    assert np.array_equal(back.get_i32("assign"), a)
    assert lamt.write_tensor(back) == b
    with pytest.raises(RuntimeError, match="is not u16"):
        back.get_u16("W")
    with pytest.raises(RuntimeError, match="missing entry 'nope'"):
        back.get_f32("nope")


def test_matrix_helpers_round_trip():
    m = np.random.default_rng(5).standard_normal((7, 3)).astype(np.float32)
    c = lamt.TensorContainer()
    c.add_matrix("m", m)
    assert np.array_equal(lamt.read_tensor(lamt.write_tensor(c)).get_matrix("m"), m)
    with pytest.raises(RuntimeError, match="not 2-D"):
        c2 = lamt.TensorContainer()
        c2.add_vector("v", m[0])
        c2.get_matrix("v")


def test_truncation_fuzzing_always_format_error():
    c = lamt.TensorContainer()
    c.add_f32("weights", np.arange(1, 7, dtype=np.float32), (2, 3))
    c.add_i32("labels", np.array([9, 8, 7, 6], np.int32), (2, 2))
    b = lamt.write_tensor(c)
    for n in range(len(b)):
        with pytest.raises(lamt.FormatError) as e:
            lamt.read_tensor(b[:n])
        assert e.value.offset <= n
    lamt.read_tensor(b)


def test_bad_magic_version_dtype_duplicates_trailing():
    c = lamt.TensorContainer()
    c.add_f32("x", np.ones(1, np.float32), (1,))
    good = bytearray(lamt.write_tensor(c))
    for pos, val, msg in ((0, ord("X"), "bad magic"), (4, 99, "unsupported version 99"),
                          (12 + 4 + 1, 7, "bad dtype code 7")):
        bad = bytearray(good)
        bad[pos] = val
        with pytest.raises(lamt.FormatError, match=msg):
            lamt.read_tensor(bytes(bad))
    with pytest.raises(lamt.FormatError, match="trailing bytes"):
        lamt.read_tensor(bytes(good) + b"\0")
    dup = lamt.TensorContainer()
    dup.add_f32("x", np.ones(1, np.float32), (1,))
    dup.add_f32("x", np.ones(1, np.float32), (1,))
    with pytest.raises(InvalidArgument, match="duplicate"):
        lamt.write_tensor(dup)
    assert isinstance(InvalidArgument("x"), ValueError)  # std::invalid_argument


def test_reader_rejects_overflowing_dims():
    c = lamt.TensorContainer()
    c.add_f32("x", np.ones(1, np.float32), (1,))
    b = bytearray(lamt.write_tensor(c))
    # ndim = 2 with dims (2^63, 4): the product overflows u64
    e = b[:12 + 4 + 1 + 1] + bytes([2]) + (1 << 63).to_bytes(8, "little") + (4).to_bytes(8, "little")
    with pytest.raises(lamt.FormatError, match="dimension overflow"):
        lamt.read_tensor(bytes(e))
    e = b[:12 + 4 + 1 + 1] + bytes([1]) + (1 << 63).to_bytes(8, "little")
    with pytest.raises(lamt.FormatError, match="payload size overflow"):
        lamt.read_tensor(bytes(e))


def c_round_quantize(d):
    """dataset.cpp:139-141 for one value, scalar: float division, std::round, clamp."""
    q = np.float32(np.float32(d) / lamt.DEPTH_QUANTUM)
    if np.isnan(q):
        return 0
    if np.isinf(q):
        return 65535 if q > 0 else 0
    import math
    r = math.floor(float(q) + 0.5) if q >= 0 else -math.floor(-float(q) + 0.5)
    return int(min(65535.0, max(0.0, r)))


def test_depth_quantization_matches_reference_rounding():
    vals = np.array([0, 0.000125, 0.000375, 0.00025, 1.0, 2.5, 16.38375, 16.38376, 100.0, -0.1, np.nan,
                     np.inf, -np.inf, 0.0001249], np.float32)
    g = np.random.default_rng(0)
    vals = np.concatenate([vals, g.uniform(0, 17, 2000).astype(np.float32)])
    q = lamt.quantize_depth(vals)
    assert [int(v) for v in q] == [c_round_quantize(v) for v in vals]
    back = q.astype(np.float32) * lamt.DEPTH_QUANTUM
    ok = np.isfinite(vals) & (vals >= 0) & (vals < 16.38)
    assert np.abs(back[ok] - vals[ok]).max() <= 0.000125 + 1e-6


def make_frames(h=6, w=8, n=3, seed=0):
    g = np.random.default_rng(seed)
    out = []
    for i in range(n):
        q = g.standard_normal(4)
        q /= np.linalg.norm(q)
        out.append(lamt.Keyframe(tuple(q), tuple(g.standard_normal(3)), g.uniform(0, 1, (h, w, 3)).astype(np.float32),
                                 (lamt.quantize_depth(g.uniform(0, 5, (h, w))).astype(np.float32) * lamt.DEPTH_QUANTUM),
                                 g.integers(-1, 4, (h, w)).astype(np.int32),
                                 g.standard_normal((4, 16)).astype(np.float32), timestamp=0.5 * i, frame_index=i,
                                 labels=g.integers(0, 3, (h, w)).astype(np.int32) if i == 1 else None))
    return out


def test_dataset_round_trip(tmp_path):
    intr = lamt.Intrinsics(50.0, 51.5, 4.0, 3.0, 8, 6)
    frames = make_frames()
    lamt.save_dataset(str(tmp_path), intr, frames)
    m = lamt.load_manifest(str(tmp_path))
    assert m.intrinsics == intr and m.frame_count() == 3
    assert m.frame_path(2).endswith(os.path.join("frames", "frame_000002.lamt"))
    for i, f in enumerate(frames):
        k = lamt.load_frame(m, i)
        assert np.array_equal(k.rgb, f.rgb) and np.array_equal(k.depth, f.depth)
        assert np.array_equal(k.assignment, f.assignment) and np.array_equal(k.features, f.features)
        assert k.timestamp == f.timestamp and k.frame_index == i
        assert np.allclose(k.pose_rot, f.pose_rot, atol=1e-7) and np.allclose(k.pose_trans, f.pose_trans, atol=1e-7)
        assert (k.labels is None) == (f.labels is None)
        if f.labels is not None:
            assert np.array_equal(k.labels.reshape(f.labels.shape), f.labels)
        p = lamt.load_frame(m, i, want_embeddings=False)
        assert (p.assignment == -1).all() and p.features.shape == (0, 0)
    with pytest.raises(IndexError):
        lamt.load_frame(m, 3)
    assert lamt.load_prototypes(str(tmp_path)).shape == (0, 0)
    c = lamt.TensorContainer()
    protos = np.eye(3, 16, dtype=np.float32)
    c.add_matrix("prototypes", protos)
    lamt.save_tensor(c, str(tmp_path / "prototypes.lamt"))
    assert np.array_equal(lamt.load_prototypes(str(tmp_path)), protos)


def test_dataset_errors(tmp_path):
    d = tmp_path
    (d / "intrinsics.txt").write_text("50 50 4 3 8 6\n")
    (d / "poses.txt").write_text("# idx tx ty tz qx qy qz qw\n0 0 0 0 0 0 0 2\n\n1 1 2 3 0 0 0 1\n")
    m = lamt.load_manifest(str(d))
    assert m.poses[0] == ((1.0, 0.0, 0.0, 0.0), (0.0, 0.0, 0.0))  # normalised (w, x, y, z)
    with pytest.raises(RuntimeError, match="frame 0"):
        lamt.load_frame(m, 0)  # file missing
    (d / "poses.txt").write_text("0 0 0 0 0 0 0 1\n2 0 0 0 0 0 0 1\n")
    with pytest.raises(RuntimeError, match="non-contiguous frame index 2"):
        lamt.load_manifest(str(d))
    (d / "poses.txt").write_text("0 0 0 0 0 0 0 0\n")
    with pytest.raises(RuntimeError, match="zero quaternion"):
        lamt.load_manifest(str(d))
    (d / "poses.txt").write_text("0 0 0 x\n")
    with pytest.raises(RuntimeError, match="malformed pose line"):
        lamt.load_manifest(str(d))
    (d / "intrinsics.txt").write_text("50 50 9 3 8 6\n")  # cx >= width
    with pytest.raises(RuntimeError, match="invalid intrinsics"):
        lamt.load_manifest(str(d))
    (d / "intrinsics.txt").write_text("50 50\n")
    with pytest.raises(RuntimeError, match="malformed intrinsics"):
        lamt.load_manifest(str(d))


def test_frame_assignment_out_of_range(tmp_path):
    intr = lamt.Intrinsics(50.0, 50.0, 4.0, 3.0, 8, 6)
    f = make_frames(n=1)[0]
    f.assignment[0, 0] = 4  # 4 feature rows
    lamt.save_dataset(str(tmp_path), intr, [f])
    with pytest.raises(RuntimeError, match="assignment index out of range"):
        lamt.load_frame(lamt.load_manifest(str(tmp_path)), 0)


def test_intrinsics_and_poses_text_format(tmp_path):
    lamt.save_intrinsics(lamt.Intrinsics(525.0, 525.0, 319.5, 239.5, 640, 480), str(tmp_path / "i.txt"))
    assert (tmp_path / "i.txt").read_text() == "525 525 319.5 239.5 640 480\n"
    lamt.save_poses([((1, 0, 0, 0), (0.1, 0, -2))], str(tmp_path / "p.txt"))
    assert (tmp_path / "p.txt").read_text() == "0 0.100000001 0 -2 0 0 0 1\n"


class FakeStore:
    def __init__(self, recs, keys):
        self._r, self._k, self.ds, self.capacity = recs, keys, recs.shape[1] - 14, 1 << 10

    def records(self):
        return self._r, self._k

    def size(self):
        return self._r.shape[0]

    def stats(self):
        return dict(inserted=5, updated=1, rejected_duplicate=2, rejected_overflow=0, probe_steps=9)


def test_map_dump_round_trip(tmp_path):
    g = np.random.default_rng(3)
    recs = g.standard_normal((5, 14 + 8)).astype(np.float32)
    keys = g.integers(-100, 100, (5, 3)).astype(np.int32)
    st = FakeStore(recs, keys)
    lamt.save_map_store(st, str(tmp_path / "map.lamt"))
    c = lamt.load_tensor(str(tmp_path / "map.lamt"))
    assert [e.name for e in c.entries] == ["positions", "rotations", "colors", "log_scales", "opacity_logits",
                                          "features", "voxel_keys"]
    assert c.require("opacity_logits").dims == (5,) and c.require("features").dims == (5, 8)
    lm = lamt.load_map_store(str(tmp_path / "map.lamt"))
    assert np.array_equal(lm.records(), recs) and np.array_equal(lm.keys, keys)
    lamt.save_store_counters(st, str(tmp_path / "counters.json"))
    j = json.loads((tmp_path / "counters.json").read_text())
    assert list(j) == ["records", "capacity", "inserted", "updated", "rejected_duplicate", "rejected_overflow",
                       "probe_steps"]
    assert j["records"] == 5 and j["capacity"] == 1024
    # a dump whose fields disagree in size
    c.entries[0] = lamt.TensorEntry("positions", lamt.F32, (4, 3), recs[:4, :3].tobytes())
    lamt.save_tensor(c, str(tmp_path / "bad.lamt"))
    with pytest.raises(RuntimeError, match="size mismatch in positions"):
        lamt.load_map_store(str(tmp_path / "bad.lamt"))


def test_dictionary_dump_round_trip(tmp_path):
    g = np.random.default_rng(4)
    d = lamt.DictionaryState(g.standard_normal((6, 10)).astype(np.float32), g.standard_normal((6, 10)).astype(np.float32),
                             g.standard_normal((4, 10)).astype(np.float32), g.uniform(0, 3, 6).astype(np.float32), 2.0)
    lamt.save_dictionary(d, str(tmp_path / "dict.lamt"))
    e = lamt.load_dictionary(str(tmp_path / "dict.lamt"))
    for f in ("atoms", "anchor", "proj", "weights"):
        assert np.array_equal(getattr(e, f), getattr(d, f))
    assert e.temperature == 2.0
    names = [x.name for x in lamt.load_tensor(str(tmp_path / "dict.lamt")).entries]
    assert names == ["atoms", "anchor", "projection", "weights", "temperature"]
