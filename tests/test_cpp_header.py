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
  // template instantiations of the k-means entry points (std::mt19937_64 through the callback)
  std::mt19937_64 rng(12);
  if (latmap_b200::uniform01_trampoline<std::mt19937_64>(&rng) != 0.18722118704556479) return 5;
  {
    std::mt19937_64 a(7), b(7);
    auto got = latmap_b200::sample_history(10, 4, a);
    std::vector<size_t> idx(10);
    for (size_t i = 0; i < 10; ++i) idx[i] = i;
    for (int k = 0; k < 4; ++k) {  // the reference's loop (pipeline.cpp:29-34)
      std::uniform_int_distribution<size_t> pick(size_t(k), 9);
      std::swap(idx[size_t(k)], idx[pick(b)]);
      if (got[size_t(k)] != idx[size_t(k)]) return 6;
    }
    if (latmap_b200::sample_history(3, 5, a).size() != 3 || !latmap_b200::sample_history(0, 5, a).empty()) return 7;
  }
  if (!latmap_b200::select_keyframe(8, 4) || latmap_b200::select_keyframe(9, 4)) return 8;
  try { latmap_b200::select_keyframe(1, 0); return 9; } catch (const std::invalid_argument&) {}
  latmap_pipeline_config pc;
  latmap_default_pipeline_config(&pc);
  if (pc.stage2_iters != 5 || pc.history_capacity != 200) return 10;
  if (cfg.lambda_feat < 0) {
    latmap_b200::Context ctx(0);
    latmap_intrinsics in{1, 1, 0, 0, 1, 1};
    latmap_b200::Pipeline p(ctx, cfg, pc, in);
    p.flush();
  }
  if (cfg.lambda_feat < 0) {
    latmap_b200::Context ctx(0);
    std::vector<float> pts(8, 0.f), w(4, 1.f);
    auto r = latmap_b200::weighted_kmeans(ctx, pts, w, 2, 2, rng);
    (void)r;
  }
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
