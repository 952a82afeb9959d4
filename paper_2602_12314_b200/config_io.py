"""latmap::Config as the reference reads and writes it (core/config.hpp:10-71, src/config.cpp):
flat ``key = value`` lines, '#' comments, blank lines ignored, unknown keys a hard error,
Config::validate after parsing, and serialisation in the reference's field order with ``%.9g``
floats. ``to_latmap`` splits a parsed config into the C-ABI's objective config and pipeline config.

Host-side text format only. One difference from the reference: float values are parsed to double
and then rounded to float32, where ``std::stof`` rounds the text directly. The two agree for every
``%.9g`` text, which is what ``serialize_config`` writes.
"""
from __future__ import annotations

import math
import re
from fractions import Fraction

import numpy as np

from ._capi import InvalidArgument

# (name, kind, default) in the order of config.cpp:84-99 (serialisation order)
FIELDS = (
    ("query_dim", "int", 32), ("embed_dim", "int", 64), ("dict_size", "int", 2000),
    ("trust_delta", "float", 0.1), ("lambda_cos", "float", 0.5), ("lambda_l2", "float", 0.5),
    ("lambda_trust", "float", 0.2), ("lambda_i1", "float", 0.2), ("lambda_i2", "float", 0.8),
    ("lambda_rgb", "float", 1.0), ("lambda_depth", "float", 0.1), ("lambda_feat", "float", 5.0),
    ("lr_proj", "float", 0.01), ("lr_dict", "float", 0.01), ("lr_position", "float", 1e-4),
    ("lr_rotation", "float", 1e-3), ("lr_color", "float", 2.5e-3), ("lr_log_scale", "float", 5e-3),
    ("lr_opacity", "float", 5e-2), ("lr_feature", "float", 2.5e-3), ("scene_extent", "float", 1.0),
    ("stage1_iters", "int", 1), ("stage2_iters", "int", 5), ("history_sample", "int", 5),
    ("history_capacity", "int", 200), ("voxel_size", "float", 0.01), ("local_radius", "float", 5.0),
    ("sync_distance", "float", 1.0), ("hash_capacity", "i64", 1 << 20), ("local_mapping", "bool", True),
    ("keyframe_stride", "int", 4), ("seed", "u64", 0), ("num_threads", "int", 0),
    ("dict_init", "str", "kmeans"), ("dict_learn", "bool", True), ("dict_decay", "float", 1.0),
    ("softmax_temp", "float", 1.0), ("trust_anchor_persistent", "bool", False),
    ("feature_supervision", "str", "pixel"),
)
_KIND = {n: k for n, k, _ in FIELDS}
_RANGE = {"int": (-(1 << 31), (1 << 31) - 1), "i64": (-(1 << 63), (1 << 63) - 1), "u64": (0, (1 << 64) - 1)}


def default_config() -> dict:
    """Config{} (config.hpp:10-58): float fields as float32 values."""
    return {n: (float(np.float32(d)) if k == "float" else d) for n, k, d in FIELDS}


_DEC = re.compile(r"[+-]?(\d+\.?\d*|\.\d+)([eE][+-]?\d+)?")
_HEX = re.compile(r"[+-]?0[xX]([0-9a-fA-F]+\.?[0-9a-fA-F]*|\.[0-9a-fA-F]+)([pP][+-]?\d+)?")
_SPECIAL = re.compile(r"[+-]?(inf|infinity|nan(\([0-9A-Za-z_]*\))?)", re.IGNORECASE)
_FLT_MIN = 2.0 ** -126


def _exact_value(v):
    """The exact rational value of a decimal or hexadecimal strtof literal."""
    if _HEX.fullmatch(v):
        sign = -1 if v[0] == "-" else 1
        body = v.lstrip("+-")[2:]
        mant, _, exp = body.partition("p") if "p" in body else body.partition("P")
        ip, _, fp = mant.partition(".")
        digits = (ip or "0") + fp
        return sign * Fraction(int(digits, 16), 16 ** len(fp)) * Fraction(2) ** int(exp or "0")
    return Fraction(v)


def _round_f32(f):
    """Round an exact rational to the nearest float32, ties to even (strtof's result); +-inf past
    the rounding boundary of FLT_MAX."""
    big = Fraction(2) ** 128  # the next "float" past FLT_MAX, for the rounding decision
    mag = abs(f)
    fmax = Fraction(float(np.finfo(np.float32).max))
    if mag > fmax:
        mid = (fmax + big) / 2
        r = math.inf if mag >= mid else float(fmax)  # a tie rounds to the even side: 2^128
        return -r if f < 0 else r
    d = float(mag)  # correctly rounded to double
    with np.errstate(over="ignore"):
        r = float(np.float32(d))
    if r != d:  # double rounding is only possible on a float32 midpoint: decide on the exact value
        nb = float(np.nextafter(np.float32(r), np.float32(0) if r > d else np.float32(np.finfo(np.float32).max)))
        a, b = (nb, r) if nb < r else (r, nb)
        mid = (Fraction(a) + Fraction(b)) / 2
        if mag < mid:
            r = a
        elif mag > mid:
            r = b
        else:
            r = a if int(np.float32(a).view(np.uint32)) % 2 == 0 else b
    return -r if f < 0 else r


def parse_float(v):
    """std::stof with the whole string consumed (config.cpp:28-33), as glibc strtof parses it:
    leading whitespace, decimal and hexadecimal literals, inf / infinity / nan(...). Raises
    std::out_of_range (OverflowError) when the value overflows float, or when it rounds inexactly
    to a subnormal or zero (strtof's ERANGE; checked against this image's std::stof)."""
    t = v.lstrip(" \t\n\v\f\r")
    if _SPECIAL.fullmatch(t):
        return float(np.float32(float(t.lower().split("(")[0])))
    if not (_DEC.fullmatch(t) or _HEX.fullmatch(t)):
        raise InvalidArgument(f"bad float value '{v}'")
    f = _exact_value(t)
    if f == 0:
        return -0.0 if t.startswith("-") else 0.0
    r = _round_f32(f)
    if not math.isfinite(r):
        raise OverflowError(f"float value out of range '{v}'")  # std::out_of_range
    if abs(r) < _FLT_MIN:
        # underflow (ERANGE) when the subnormal result is inexact. glibc's hexadecimal path first
        # forms a 24-bit mantissa (round bit = the 25th bit, sticky = anything beyond) and then
        # tests only the mantissa bits shifted out below 2^-149 and the sticky bit -- not that
        # round bit (measured: 0x1.000001p-149 parses, 0x1.00000000001p-149 is out of range)
        if _HEX.fullmatch(t):
            mag = abs(f)
            e = mag.numerator.bit_length() - mag.denominator.bit_length()
            if Fraction(2) ** e > mag:
                e -= 1
            elif Fraction(2) ** (e + 1) <= mag:
                e += 1
            unit = Fraction(2) ** (e - 23)
            m24 = int(mag / unit)
            rem = mag - m24 * unit
            sticky = rem != 0 and rem != unit / 2
            drop = -126 - e
            dropped = m24 if drop >= 24 else m24 % (1 << drop) if drop > 0 else 0
            inexact = dropped != 0 or sticky
        else:
            inexact = Fraction(r) != f
        if inexact:
            raise OverflowError(f"float value out of range '{v}'")  # std::out_of_range
    return r


def _parse(kind, v):
    if kind == "float":
        return parse_float(v)
    if kind in _RANGE:
        try:
            if "_" in v:
                raise ValueError
            i = int(v, 10)
        except ValueError:
            raise InvalidArgument(f"bad int value '{v}'") from None
        lo, hi = _RANGE[kind]
        if not lo <= i <= hi:
            raise OverflowError(f"int value out of range '{v}'")  # std::out_of_range
        return i
    if kind == "bool":
        if v in ("true", "1"):
            return True
        if v in ("false", "0"):
            return False
        raise InvalidArgument(f"bad bool value '{v}'")
    return v


def validate(c: dict):
    """Config::validate (config.cpp:110-133)."""
    def req(ok, msg):
        if not ok:
            raise InvalidArgument("config: " + msg)
    req(c["query_dim"] >= 1 and c["embed_dim"] >= 1, "dimensions must be >= 1")
    req(c["query_dim"] <= c["embed_dim"], "query_dim must be <= embed_dim")
    req(c["dict_size"] >= 1, "dict_size must be >= 1")
    req(all(c[k] >= 0 for k in ("lambda_cos", "lambda_l2", "lambda_trust", "lambda_i1", "lambda_i2", "lambda_rgb",
                                "lambda_depth", "lambda_feat")), "loss weights must be >= 0")
    req(c["trust_delta"] >= 0, "trust_delta must be >= 0")
    req(c["stage1_iters"] >= 0 and c["stage2_iters"] >= 0, "iteration counts must be >= 0")
    req(c["keyframe_stride"] >= 1, "keyframe_stride must be >= 1")
    req(c["history_sample"] >= 0 and c["history_capacity"] >= 1, "history sizes invalid")
    req(c["voxel_size"] > 0, "voxel_size must be > 0")
    req(c["local_radius"] > 0 and c["sync_distance"] >= 0, "sync geometry invalid")
    req(c["hash_capacity"] >= 1, "hash_capacity must be >= 1")
    req(c["softmax_temp"] > 0, "softmax_temp must be > 0")
    req(0 < c["dict_decay"] <= 1, "dict_decay must be in (0,1]")
    req(c["dict_init"] in ("kmeans", "random"), "dict_init must be kmeans|random")
    req(c["feature_supervision"] in ("pixel", "segment"), "feature_supervision must be pixel|segment")
    req(c["num_threads"] >= 0, "num_threads must be >= 0")


def parse_config(text: str) -> dict:
    """parse_config (config.cpp:135-165)."""
    c = default_config()
    for lineno, line in enumerate(text.split("\n"), 1):
        line = line.split("#", 1)[0].strip(" \t\r\n")
        if not line:
            continue
        if "=" not in line:
            raise InvalidArgument(f"config line {lineno}: missing '='")
        key, value = line.split("=", 1)
        key, value = key.strip(" \t\r\n"), value.strip(" \t\r\n")
        if key not in _KIND:
            raise InvalidArgument(f"config line {lineno}: unknown key '{key}'")
        c[key] = _parse(_KIND[key], value)
    validate(c)
    return c


def load_config(path) -> dict:
    try:
        with open(path, "rb") as f:
            text = f.read().decode()
    except OSError as e:
        raise RuntimeError(f"cannot open config file: {path}") from e
    return parse_config(text)


def serialize_config(c: dict) -> str:
    """serialize_config (config.cpp:175-179): every field, reference order, %.9g floats."""
    out = []
    for n, k, _ in FIELDS:
        v = c[n]
        if k == "float":
            s = "%.9g" % float(np.float32(v))
        elif k == "bool":
            s = "true" if v else "false"
        else:
            s = str(v)
        out.append(f"{n} = {s}\n")
    return "".join(out)


def save_config(c: dict, path):
    try:
        with open(path, "wb") as f:
            f.write(serialize_config(c).encode())
    except OSError as e:
        raise RuntimeError(f"cannot write config file: {path}") from e


def to_latmap(c: dict):
    """(latmap_config, latmap_pipeline_config) for the C-ABI from a parsed Config.
    num_threads has no meaning on the device and is dropped."""
    from . import api
    obj_fields = ("lambda_cos", "lambda_l2", "lambda_trust", "trust_delta", "lambda_i1", "lambda_i2", "lambda_rgb",
                  "lambda_depth", "lambda_feat", "lr_proj", "lr_dict", "lr_position", "lr_rotation", "lr_color",
                  "lr_log_scale", "lr_opacity", "lr_feature", "scene_extent", "softmax_temp")
    cfg = api.default_config(**{k: c[k] for k in obj_fields})
    cfg.dict_learn = int(bool(c["dict_learn"]))
    cfg.segment_mode = int(c["feature_supervision"] == "segment")
    pc = api.default_pipeline_config(
        query_dim=c["query_dim"], embed_dim=c["embed_dim"], dict_size=c["dict_size"], stage1_iters=c["stage1_iters"],
        stage2_iters=c["stage2_iters"], history_sample=c["history_sample"], history_capacity=c["history_capacity"],
        voxel_size=c["voxel_size"], local_radius=c["local_radius"], sync_distance=c["sync_distance"],
        hash_capacity=c["hash_capacity"], local_mapping=int(bool(c["local_mapping"])),
        keyframe_stride=c["keyframe_stride"], seed=c["seed"], dict_init=c["dict_init"], dict_decay=c["dict_decay"],
        trust_anchor_persistent=int(bool(c["trust_anchor_persistent"])))
    return cfg, pc
