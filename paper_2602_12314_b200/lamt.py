"""LAMT named-tensor files and the artifacts either side of the hot path.

Host-side byte formats only, no device work. Restates:

- the container of ``io/tensor_file.hpp:46-85`` and ``src/tensor_file.cpp:1-230``: magic "LAMT",
  version u32, entry count u32, then per entry name_len u32 | name | dtype u8 | ndim u8 |
  dims u64[ndim] | payload, little-endian, row-major. The reader raises ``FormatError`` with
  the reference's messages and byte offsets;
- the dataset layout of ``io/dataset.hpp:9-35`` / ``src/dataset.cpp``: ``intrinsics.txt``,
  ``poses.txt``, ``frames/frame_%06d.lamt`` (u16 depth in 0.25 mm steps) and ``prototypes.lamt``;
- the dumps of ``src/artifacts.cpp``: the global map as SoA tensors plus voxel keys, the store
  counters sidecar, and the dictionary.

Files written here load in the reference and the reverse. Two places may differ from the
reference's float bits. First, text floats are parsed to double and then rounded to float. That
is exact for the ``%.9g`` text both sides write. Second, the pose quaternion norm is a sequential
float sum. Real Eigen's reduction order is unpinned.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass, field

import numpy as np

from ._capi import InvalidArgument

MAGIC = b"LAMT"
VERSION = 1
F32, U16, I32 = 1, 2, 3
_NP = {F32: np.dtype("<f4"), U16: np.dtype("<u2"), I32: np.dtype("<i4")}
_NAMES = {F32: "f32", U16: "u16", I32: "i32"}
_U64 = (1 << 64) - 1
DEPTH_QUANTUM = np.float32(0.00025)  # dataset.hpp:26 kDepthQuantum, metres per u16 step


class FormatError(RuntimeError):
    """tensor_file.hpp:13-22: parse failure; ``offset`` is the reader's byte position."""

    def __init__(self, what, offset):
        super().__init__(f"{what} (at byte {offset})")
        self.offset = offset


def dtype_size(dt):
    if dt not in _NP:
        raise InvalidArgument("unknown dtype")
    return _NP[dt].itemsize


@dataclass
class TensorEntry:
    name: str
    dtype: int = F32
    dims: tuple = ()
    payload: bytes = b""

    def element_count(self):
        n = 1
        for d in self.dims:
            n *= int(d)
        return n

    def array(self):
        """The payload as a numpy array of shape ``dims`` (a copy, native byte order)."""
        return np.frombuffer(self.payload, _NP[self.dtype]).astype(_NP[self.dtype].newbyteorder("="))\
            .reshape(tuple(int(d) for d in self.dims))


class TensorContainer:
    """tensor_file.hpp:46-78: ordered named entries; names must be unique when written."""

    def __init__(self, entries=None):
        self.entries = list(entries or [])

    def find(self, name):
        for e in self.entries:
            if e.name == name:
                return e
        return None

    def require(self, name):
        e = self.find(name)
        if e is None:
            raise RuntimeError(f"tensor container: missing entry '{name}'")
        return e

    def _add(self, name, dt, data, dims):
        a = np.asarray(data)
        dims = tuple(int(d) for d in (a.shape if dims is None else dims))
        e = TensorEntry(name, dt, dims)
        flat = np.ascontiguousarray(a, _NP[dt]).reshape(-1)
        if flat.size != e.element_count():
            raise InvalidArgument(f"tensor container: {flat.size} values for dims {dims} in '{name}'")
        e.payload = flat.tobytes()
        self.entries.append(e)
        return e

    def add_f32(self, name, data, dims=None):
        return self._add(name, F32, data, dims)

    def add_u16(self, name, data, dims=None):
        return self._add(name, U16, data, dims)

    def add_i32(self, name, data, dims=None):
        return self._add(name, I32, data, dims)

    def add_matrix(self, name, m):
        m = np.asarray(m)
        if m.ndim != 2:
            raise InvalidArgument(f"add_matrix: '{name}' is not 2-D")
        return self.add_f32(name, m, m.shape)

    def add_vector(self, name, v):
        v = np.asarray(v).reshape(-1)
        return self.add_f32(name, v, (v.size,))

    def _get(self, name, dt):
        e = self.require(name)
        if e.dtype != dt:
            raise RuntimeError(f"entry '{name}' is not {_NAMES[dt]}")
        return np.frombuffer(e.payload, _NP[dt]).astype(_NP[dt].newbyteorder("="))

    def get_f32(self, name):
        return self._get(name, F32)

    def get_u16(self, name):
        return self._get(name, U16)

    def get_i32(self, name):
        return self._get(name, I32)

    def get_matrix(self, name):
        e = self.require(name)
        if len(e.dims) != 2:
            raise RuntimeError(f"entry '{name}' is not 2-D")
        return self.get_f32(name).reshape(int(e.dims[0]), int(e.dims[1]))

    def get_vector(self, name):
        return self.get_f32(name)


def write_tensor(c: TensorContainer) -> bytes:
    """tensor_file.cpp:159-180."""
    names = set()
    for e in c.entries:
        if e.name in names:
            raise InvalidArgument(f"tensor container: duplicate entry name '{e.name}'")
        names.add(e.name)
    out = [MAGIC, np.array([VERSION, len(c.entries)], "<u4").tobytes()]
    for e in c.entries:
        if len(e.payload) != e.element_count() * dtype_size(e.dtype):
            raise InvalidArgument(f"tensor container: payload size mismatch for '{e.name}'")
        nm = e.name.encode("utf-8", "surrogateescape")
        out += [np.array([len(nm)], "<u4").tobytes(), nm, bytes([e.dtype, len(e.dims)]),
                np.array(e.dims, "<u8").tobytes(), bytes(e.payload)]
    return b"".join(out)


class _Reader:
    def __init__(self, data):
        self.data, self.size, self.pos = data, len(data), 0

    def need(self, n, what):
        if self.pos + n > self.size:
            raise FormatError(f"truncated: {what}", self.pos)

    def u8(self, what):
        self.need(1, what)
        self.pos += 1
        return self.data[self.pos - 1]

    def u32(self, what):
        self.need(4, what)
        self.pos += 4
        return int.from_bytes(self.data[self.pos - 4:self.pos], "little")

    def u64(self, what):
        self.need(8, what)
        self.pos += 8
        return int.from_bytes(self.data[self.pos - 8:self.pos], "little")


def read_tensor(data) -> TensorContainer:
    """tensor_file.cpp:182-214: every malformed or truncated input raises FormatError."""
    data = bytes(data)
    r = _Reader(data)
    r.need(4, "magic")
    if data[:4] != MAGIC:
        raise FormatError("bad magic", 0)
    r.pos = 4
    version = r.u32("version")
    if version != VERSION:
        raise FormatError(f"unsupported version {version}", 4)
    count = r.u32("entry count")
    c = TensorContainer()
    names = set()
    for _ in range(count):
        name_len = r.u32("name length")
        r.need(name_len, "name")
        name = data[r.pos:r.pos + name_len].decode("utf-8", "surrogateescape")
        r.pos += name_len
        if name in names:
            raise FormatError(f"duplicate entry name '{name}'", r.pos)
        names.add(name)
        dt = r.u8("dtype")
        if dt < 1 or dt > 3:
            raise FormatError(f"bad dtype code {dt}", r.pos - 1)
        ndim = r.u8("ndim")
        elems, dims = 1, []
        for _ in range(ndim):
            dim = r.u64("dim")
            if dim != 0 and elems > _U64 // dim:
                raise FormatError("dimension overflow", r.pos - 8)
            elems *= dim
            dims.append(dim)
        if elems > _U64 // dtype_size(dt):
            raise FormatError("payload size overflow", r.pos)
        nbytes = elems * dtype_size(dt)
        if nbytes > r.size - r.pos:
            raise FormatError("truncated: payload", r.pos)
        c.entries.append(TensorEntry(name, dt, tuple(dims), data[r.pos:r.pos + nbytes]))
        r.pos += nbytes
    if r.pos != r.size:
        raise FormatError("trailing bytes after last entry", r.pos)
    return c


def save_tensor(c: TensorContainer, path):
    b = write_tensor(c)
    try:
        with open(path, "wb") as f:
            f.write(b)
    except OSError as e:
        raise RuntimeError(f"cannot write {path}") from e


def load_tensor(path) -> TensorContainer:
    try:
        with open(path, "rb") as f:
            b = f.read()
    except OSError as e:
        raise RuntimeError(f"cannot open {path}") from e
    return read_tensor(b)


# ---- dataset layout (io/dataset.hpp, src/dataset.cpp) ----

@dataclass
class Intrinsics:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    def valid(self):
        """types.hpp:46-49."""
        return (self.fx > 0 and self.fy > 0 and self.width > 0 and self.height > 0 and 0 <= self.cx < self.width
                and 0 <= self.cy < self.height)


@dataclass
class Keyframe:
    """KeyframeT<float> (types.hpp:225-234) on the host: pose camera-to-world, rotation (w, x, y, z);
    rgb H x W x 3, depth H x W (metres, 0 = invalid), features n_set x d_f, assignment H x W
    (-1 = unsupervised), labels H x W or None. Field names match what Session.set_frames reads."""
    pose_rot: tuple
    pose_trans: tuple
    rgb: np.ndarray
    depth: np.ndarray
    assignment: np.ndarray
    features: np.ndarray
    timestamp: float = 0.0
    frame_index: int = 0
    labels: np.ndarray | None = None


@dataclass
class DatasetManifest:
    dir: str
    intrinsics: Intrinsics
    poses: list = field(default_factory=list)  # [(rotation (w,x,y,z), translation)] float32

    def frame_count(self):
        return len(self.poses)

    def frame_path(self, index):
        return os.path.join(self.dir, "frames", "frame_%06d.lamt" % index)


def load_manifest(d) -> DatasetManifest:
    """dataset.cpp:20-55."""
    p = os.path.join(d, "intrinsics.txt")
    try:
        toks = open(p).read().split()
    except OSError as e:
        raise RuntimeError(f"dataset: cannot open {p}") from e
    try:
        intr = Intrinsics(*[float(np.float32(t)) for t in toks[:4]], int(toks[4]), int(toks[5]))
    except (ValueError, IndexError) as e:
        raise RuntimeError("dataset: malformed intrinsics.txt") from e
    if not intr.valid():
        raise RuntimeError("dataset: invalid intrinsics")
    m = DatasetManifest(d, intr)
    p = os.path.join(d, "poses.txt")
    try:
        lines = open(p).read().splitlines()
    except OSError as e:
        raise RuntimeError(f"dataset: cannot open {p}") from e
    for line in lines:
        if not line or line[0] == "#":
            continue
        t = line.split()
        try:
            idx = int(t[0])
            tx, ty, tz, qx, qy, qz, qw = (np.float32(v) for v in t[1:8])
        except (ValueError, IndexError) as e:
            raise RuntimeError(f"dataset: malformed pose line: {line}") from e
        if idx != len(m.poses):
            raise RuntimeError(f"dataset: non-contiguous frame index {idx}")
        q = np.array([qw, qx, qy, qz], np.float32)
        s = np.float32(0)
        for v in q:
            s = np.float32(s + v * v)
        n = np.float32(np.sqrt(s))
        if not n > 0:
            raise RuntimeError("dataset: zero quaternion in poses.txt")
        m.poses.append((tuple(float(v) for v in q / n), (float(tx), float(ty), float(tz))))
    return m


def save_intrinsics(intr, path):
    with open(path, "w") as f:
        f.write("%.9g %.9g %.9g %.9g %d %d\n" % (intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height))


def save_poses(poses, path):
    """poses: [(rotation (w,x,y,z), translation)]; written as index tx ty tz qx qy qz qw."""
    with open(path, "w") as f:
        for i, (q, t) in enumerate(poses):
            q = [float(np.float32(v)) for v in q]
            t = [float(np.float32(v)) for v in t]
            f.write("%d %.9g %.9g %.9g %.9g %.9g %.9g %.9g\n" % (i, t[0], t[1], t[2], q[1], q[2], q[3], q[0]))


def quantize_depth(depth):
    """dataset.cpp:139-141: u16(min(65535, max(0, round(d / 0.25 mm)))), round half away from
    zero, NaN -> 0."""
    q = np.asarray(depth, np.float32) / DEPTH_QUANTUM
    qd = q.astype(np.float64)  # float32 + 0.5 is exact in double: std::round without double rounding
    r = np.where(qd >= 0, np.floor(qd + 0.5), -np.floor(-qd + 0.5))
    r = np.where(np.isnan(r), 0.0, np.clip(r, 0.0, 65535.0))
    return r.astype(np.uint16)


def load_frame(manifest: DatasetManifest, index, want_embeddings=True) -> Keyframe:
    """dataset.cpp:73-125."""
    if index < 0 or index >= manifest.frame_count():
        raise IndexError("dataset: frame index out of range")
    try:
        c = load_tensor(manifest.frame_path(index))
    except Exception as e:
        raise RuntimeError(f"dataset: frame {index}: {e}") from e
    h, w = manifest.intrinsics.height, manifest.intrinsics.width
    ts = c.get_f32("timestamp")
    rgb = c.get_f32("rgb")
    if rgb.size != h * w * 3:
        raise RuntimeError(f"dataset: rgb size mismatch in frame {index}")
    dq = c.get_u16("depth")
    if dq.size != h * w:
        raise RuntimeError(f"dataset: depth size mismatch in frame {index}")
    depth = (dq.astype(np.float32) * DEPTH_QUANTUM).reshape(h, w)
    rot, trans = manifest.poses[index]
    kf = Keyframe(rot, trans, rgb.reshape(h, w, 3), depth, np.full((h, w), -1, np.int32),
                  np.zeros((0, 0), np.float32), 0.0 if ts.size == 0 else float(ts[0]), index)
    if want_embeddings:
        if len(c.require("features").dims) != 2:
            raise RuntimeError("dataset: features entry must be 2-D")
        kf.features = c.get_matrix("features")
        a = c.get_i32("assignment")
        if a.size != h * w:
            raise RuntimeError("dataset: assignment size mismatch")
        if a.size and a.max() >= kf.features.shape[0]:
            raise RuntimeError("dataset: assignment index out of range")
        kf.assignment = a.reshape(h, w)
        if c.find("labels") is not None:
            kf.labels = c.get_i32("labels")
    return kf


def save_frame(kf: Keyframe, path):
    """dataset.cpp:127-150."""
    rgb = np.asarray(kf.rgb, np.float32)
    h, w = rgb.shape[0], rgb.shape[1]
    c = TensorContainer()
    c.add_f32("timestamp", np.float32(kf.timestamp), (1,))
    c.add_f32("rgb", rgb, (h, w, 3))
    dep = np.asarray(kf.depth, np.float32)
    c.add_u16("depth", quantize_depth(dep), (dep.shape[0], dep.shape[1]))
    feats = np.asarray(kf.features, np.float32)
    c.add_matrix("features", feats.reshape(feats.shape[0], -1) if feats.ndim == 2 else feats.reshape(0, 0))
    a = np.asarray(kf.assignment, np.int32)
    eh, ew = (a.shape if a.ndim == 2 else (h, w))
    c.add_i32("assignment", a, (eh, ew))
    if kf.labels is not None and np.asarray(kf.labels).size:
        c.add_i32("labels", kf.labels, (eh, ew))
    save_tensor(c, path)


def save_dataset(d, intr, frames):
    """The layout load_manifest reads: intrinsics.txt, poses.txt, frames/frame_%06d.lamt."""
    os.makedirs(os.path.join(d, "frames"), exist_ok=True)
    save_intrinsics(intr, os.path.join(d, "intrinsics.txt"))
    save_poses([(f.pose_rot, f.pose_trans) for f in frames], os.path.join(d, "poses.txt"))
    for i, f in enumerate(frames):
        save_frame(f, os.path.join(d, "frames", "frame_%06d.lamt" % i))


def load_prototypes(d):
    """dataset.cpp:152-156: the C x d_f class prototypes, or an empty matrix when absent."""
    p = os.path.join(d, "prototypes.lamt")
    if not os.path.exists(p):
        return np.zeros((0, 0), np.float32)
    return load_tensor(p).get_matrix("prototypes")


# ---- artifacts (src/artifacts.cpp) ----

MAP_FIELDS = (("positions", 3), ("rotations", 4), ("colors", 3), ("log_scales", 3), ("opacity_logits", 1))


@dataclass
class LoadedMap:
    """artifacts.hpp LoadedMap: the record pool as SoA arrays plus voxel keys (n x 3 int32)."""
    positions: np.ndarray
    rotations: np.ndarray
    colors: np.ndarray
    log_scales: np.ndarray
    opacity_logits: np.ndarray
    features: np.ndarray
    keys: np.ndarray

    def records(self):
        """The store's AoS record rows [position 3 | rotation 4 | color 3 | log_scale 3 |
        opacity 1 | features d_s]."""
        n = self.positions.shape[0]
        return np.concatenate([self.positions, self.rotations, self.colors, self.log_scales,
                               self.opacity_logits.reshape(n, 1), self.features], axis=1)


def _map_container(recs, keys, ds):
    c = TensorContainer()
    n = recs.shape[0]
    col = 0
    for name, w in MAP_FIELDS:
        blk = recs[:, col:col + w]
        c.add_f32(name, blk, (n, w) if w > 1 else (n,))
        col += w
    c.add_f32("features", recs[:, col:col + ds], (n, ds))
    c.add_i32("voxel_keys", keys, (n, 3))
    return c


def save_map_store(store, path):
    """artifacts.cpp:40-52: the store's record pool (insertion order) as named SoA tensors plus
    the voxel key of each record."""
    recs, keys = store.records()
    save_tensor(_map_container(recs, keys, store.ds), path)


def load_map_store(path) -> LoadedMap:
    """artifacts.cpp:19-37, 54-63."""
    c = load_tensor(path)
    feat = c.require("features")
    n, ds = int(feat.dims[0]), int(feat.dims[1])
    out = {}
    for name, w in MAP_FIELDS + (("features", ds),):
        v = c.get_f32(name)
        if v.size != n * w:
            raise RuntimeError(f"map artifact: size mismatch in {name}")
        out[name] = v.reshape(n, w) if name != "opacity_logits" else v
    keys = c.get_i32("voxel_keys")
    return LoadedMap(**out, keys=keys[:keys.size // 3 * 3].reshape(-1, 3))


def restore_store(ctx, loaded: LoadedMap, capacity):
    """A Store holding a loaded dump: each record inserted under its stored key in dump order
    (so record indices equal the dump's)."""
    from .api import Store
    st = Store(ctx, capacity, loaded.features.shape[1])
    st.insert_keyed(loaded.keys, loaded.records())
    return st


def save_store_counters(store, path):
    """artifacts.cpp:65-74: one JSON line of the store's size, capacity and counters."""
    s = store.stats()
    with open(path, "w") as f:
        f.write(json.dumps({"records": store.size(), "capacity": store.capacity, **s}, separators=(",", ":")) + "\n")


@dataclass
class DictionaryState:
    """DictionaryStateT<float> (dict/dictionary.hpp:14-27)."""
    atoms: np.ndarray
    anchor: np.ndarray
    proj: np.ndarray
    weights: np.ndarray
    temperature: float


def save_dictionary(d, path):
    """artifacts.cpp:76-85. ``d``: a DictionaryState or an api.Session (its device dictionary,
    anchor, atom weights and the configured softmax temperature)."""
    if not isinstance(d, DictionaryState):
        atoms, proj = d.get_dictionary()
        d = DictionaryState(atoms, d.get_anchor(), proj, d.dict_weights(), d.cfg.softmax_temp)
    c = TensorContainer()
    c.add_matrix("atoms", d.atoms)
    c.add_matrix("anchor", d.anchor)
    c.add_matrix("projection", d.proj)
    c.add_vector("weights", d.weights)
    c.add_f32("temperature", np.float32(d.temperature), (1,))
    save_tensor(c, path)


def load_dictionary(path) -> DictionaryState:
    """artifacts.cpp:87-96."""
    c = load_tensor(path)
    t = c.get_f32("temperature")
    if t.size < 1:
        raise IndexError("dictionary artifact: empty temperature")
    return DictionaryState(c.get_matrix("atoms"), c.get_matrix("anchor"), c.get_matrix("projection"),
                           c.get_vector("weights"), float(t[0]))


def apply_dictionary(session, d: DictionaryState):
    """Load a DictionaryState into a device session (atoms, anchor, proj, atom weights). The
    temperature is part of the session's Config and is checked, not changed."""
    if abs(float(np.float32(session.cfg.softmax_temp)) - float(np.float32(d.temperature))) > 0:
        raise InvalidArgument("dictionary temperature differs from the session's softmax_temp")
    session.set_dictionary(d.atoms, d.anchor, d.proj)
    session.set_dict_weights(d.weights)
