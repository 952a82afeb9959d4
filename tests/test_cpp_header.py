"""The C++ host header (include/latmap_b200.hpp) compiles against the C-ABI header and links
against liblatmap_b200.so (no GPU needed: the program only checks that a context cannot be
created without a device and that the status -> exception mapping matches the reference)."""
import os
import subprocess
import shutil

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SRC = r'''
#include <cstdio>
#include <stdexcept>
#include "latmap_b200.hpp"
int main() {
  latmap_config cfg;
  latmap_default_config(&cfg);
  if (cfg.lambda_feat != 5.0f) return 2;
  try { latmap_b200::check(LATMAP_ERR_INVALID_ARGUMENT, nullptr); return 3; } catch (const std::invalid_argument&) {}
  try { latmap_b200::check(LATMAP_ERR_STALE_CACHE, nullptr); return 4; } catch (const std::runtime_error&) {}
  try { latmap_b200::Context ctx(0); std::puts("has-gpu"); } catch (const latmap_b200::device_error&) { std::puts("no-gpu"); }
  return 0;
}
'''


@pytest.mark.skipif(shutil.which("g++") is None, reason="g++ missing")
def test_cpp_header_compiles_and_links(tmp_path):
    src = tmp_path / "t.cpp"
    src.write_text(SRC)
    exe = tmp_path / "t"
    libdir = os.path.join(ROOT, "paper_2602_12314_b200")
    subprocess.run(["g++", "-std=c++17", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"), str(src), "-o",
                    str(exe), "-L", libdir, "-llatmap_b200", f"-Wl,-rpath,{libdir}",
                    "-L/usr/local/cuda/lib64", "-lcudart"], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert out.stdout.strip() in ("no-gpu", "has-gpu")
