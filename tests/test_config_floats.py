"""config_io.parse_float against this image's own std::stof (the reference's parse_float,
proj/src/config.cpp:28-33): value bits or the exception kind on ~3000 literals -- random decimals
over the whole float range (overflow, FLT_MAX rounding, subnormals), hex floats, specials and
malformed text. The C++ side is compiled here from a 15-line program."""
import shutil
import subprocess

import numpy as np
import pytest

from paper_2602_12314_b200 import config_io
from paper_2602_12314_b200._capi import InvalidArgument

PROG = r"""
#include <cstdio>
#include <iostream>
#include <stdexcept>
#include <string>
int main() {
  std::string v;
  while (std::getline(std::cin, v)) {
    try { size_t pos = 0; float f = std::stof(v, &pos);
      if (pos != v.size()) std::puts("invalid"); else std::printf("%a\n", (double)f); }
    catch (std::out_of_range&) { std::puts("range"); }
    catch (std::invalid_argument&) { std::puts("invalid"); }
  }
}
"""


@pytest.fixture(scope="module")
def stof(tmp_path_factory):
    if not shutil.which("g++"):
        pytest.skip("no g++")
    d = tmp_path_factory.mktemp("stof")
    (d / "stof.cpp").write_text(PROG)
    subprocess.run(["g++", "-O1", "-o", str(d / "stof"), str(d / "stof.cpp")], check=True)
    return str(d / "stof")


def literals():
    rng = np.random.default_rng(7)
    out = ["0", "-0.0", "1.5", ".5", "5.", "inf", "-INF", "Infinity", "nan", "nan(x1)", "1e", ".", "", "+", "1.5x",
           "0x", "0x.p1", "0x1p", "1e+", "--1", "3.4028235e38", "3.40282357e38", "3.4028236e38", "1.17549435e-38",
           "1.1754942e-38", "1.4e-45", "7e-46", "0x1p-149", "0x1p-150", "0x1.000001p-149", " 1", "1 "]
    for _ in range(1500):  # decimals across the range
        m = rng.integers(1, 10 ** rng.integers(1, 12))
        e = rng.integers(-50, 45)
        s = f"{'-' if rng.random() < 0.3 else ''}{m}e{e}"
        if rng.random() < 0.5:
            t = str(m)
            k = rng.integers(0, len(t) + 1)
            s = f"{'-' if rng.random() < 0.3 else ''}{t[:k]}.{t[k:]}e{e}"
        out.append(s)
    for _ in range(800):  # hex floats
        mant = "".join(rng.choice(list("0123456789abcdef"), rng.integers(1, 9)))
        k = rng.integers(0, len(mant) + 1)
        out.append(f"0x{mant[:k]}.{mant[k:]}p{rng.integers(-160, 130)}")
    for _ in range(600):  # float32 values printed with 9 significant digits (round trips)
        x = np.float32(rng.standard_normal() * 10.0 ** rng.integers(-40, 39))
        out.append(f"{float(x):.9g}")
    return out


def test_parse_float_matches_std_stof(stof):
    lits = literals()
    res = subprocess.run([stof], input="\n".join(lits) + "\n", capture_output=True, text=True, check=True)
    ref = res.stdout.splitlines()
    assert len(ref) == len(lits)
    for lit, r in zip(lits, ref):
        try:
            got = config_io.parse_float(lit)
            kind = "value"
        except OverflowError:
            kind = "range"
        except InvalidArgument:
            kind = "invalid"
        if r in ("range", "invalid"):
            assert kind == r, (lit, kind, r)
        else:
            assert kind == "value", (lit, kind, r)
            want = float.fromhex(r) if "nan" not in r else float("nan")
            if want != want:
                assert got != got, lit
            else:
                assert np.float32(got).view(np.uint32) == np.float32(want).view(np.uint32), (lit, got, want)
