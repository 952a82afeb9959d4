// dropin_check.cpp — drives the reference's own Eigen-typed API (proj/include/latmap/**) for
// T = float, which this binary links to the drop-in layer (latmap_dropin.o -> the B200 kernels),
// on seeded inputs, and writes inputs and outputs as .npy files into argv[1]. The GPU test
// (tests/test_gpu_dropin.py) replays the same inputs through the CPU oracle and compares; it also
// checks the exception contract recorded in errors.npy.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "latmap/dict/dictionary.hpp"
#include "latmap/obj/losses.hpp"
#include "latmap/obj/objective.hpp"
#include "latmap/splat/render.hpp"

using namespace latmap;

namespace {

std::string g_dir;

void save(const std::string& name, const void* data, const std::vector<size_t>& shape, const char* descr,
          size_t elem) {
  std::string dict = std::string("{'descr': '") + descr + "', 'fortran_order': False, 'shape': (";
  size_t count = 1;
  for (size_t i = 0; i < shape.size(); ++i) {
    dict += std::to_string(shape[i]) + (shape.size() == 1 ? "," : (i + 1 < shape.size() ? ", " : ""));
    count *= shape[i];
  }
  dict += "), }";
  while ((10 + dict.size() + 1) % 64) dict += ' ';
  dict += '\n';
  std::ofstream f(g_dir + "/" + name + ".npy", std::ios::binary);
  const char magic[] = "\x93NUMPY\x01\x00";
  f.write(magic, 8);
  const uint16_t hl = uint16_t(dict.size());
  f.write(reinterpret_cast<const char*>(&hl), 2);
  f.write(dict.data(), std::streamsize(dict.size()));
  f.write(static_cast<const char*>(data), std::streamsize(count * elem));
}
void savef(const std::string& n, const float* d, std::vector<size_t> s) { save(n, d, s, "<f4", 4); }
void savei(const std::string& n, const int32_t* d, std::vector<size_t> s) { save(n, d, s, "<i4", 4); }
template <class M>
void savem(const std::string& n, const M& m) {
  savef(n, m.data(), {size_t(m.rows()), size_t(m.cols())});
}
void savev(const std::string& n, const VecX<float>& v) { savef(n, v.data(), {size_t(v.size())}); }
void saveimg(const std::string& n, const Image& im) {
  savef(n, im.data.data(), {size_t(im.height), size_t(im.width), size_t(im.channels)});
}

GaussianMap random_map(int n, int ds, std::mt19937_64& rng) {
  std::uniform_real_distribution<float> u(0.f, 1.f);
  std::normal_distribution<float> g(0.f, 1.f);
  GaussianMap m;
  m.resize(n, ds);
  for (int i = 0; i < n; ++i) {
    m.positions.row(i) << (u(rng) * 2 - 1) * 1.6f, (u(rng) * 2 - 1) * 1.2f, 1.5f + u(rng) * 3.5f;
    Vec4f q(g(rng), g(rng), g(rng), g(rng));
    q.normalize();
    m.rotations.row(i) = q.transpose();
    m.colors.row(i) << u(rng), u(rng), u(rng);
    m.log_scales.row(i) << -3.3f + 0.4f * g(rng), -3.3f + 0.4f * g(rng), -3.3f + 0.4f * g(rng);
    m.opacity_logits(i) = g(rng);
    for (int c = 0; c < ds; ++c) m.features(i, c) = g(rng);
  }
  return m;
}

MatX<float> randn(int r, int c, std::mt19937_64& rng, float s = 1.f) {
  std::normal_distribution<float> g(0.f, s);
  MatX<float> m(r, c);
  for (Eigen::Index i = 0; i < m.size(); ++i) m.data()[i] = g(rng);
  return m;
}

template <class F>
int32_t throws(F f, int kind) {  // 1 = std::invalid_argument, 2 = other std::runtime_error, 0 = none
  try {
    f();
  } catch (const std::invalid_argument&) {
    return kind == 1 ? 1 : -1;
  } catch (const std::runtime_error&) {
    return kind == 2 ? 2 : -2;
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: dropin_check OUTDIR\n");
    return 2;
  }
  g_dir = argv[1];
  std::mt19937_64 rng(0x4c41544d44ull);
  const int N = 6000, ds = 8, K = 32, df = 64, W = 128, H = 96;
  Intrinsics intr;
  intr.fx = intr.fy = 110.f, intr.cx = 64.f, intr.cy = 48.f, intr.width = W, intr.height = H;
  GaussianMap map = random_map(N, ds, rng);
  Pose pose;
  pose.rotation = Vec4f(0.9995f, 0.01f, -0.03f, 0.005f);
  pose.rotation.normalize();
  pose.translation = Vec3f(0.05f, -0.02f, 0.1f);
  savem("positions", map.positions), savem("rotations", map.rotations), savem("colors", map.colors);
  savem("log_scales", map.log_scales), savev("opacity_logits", map.opacity_logits), savem("features", map.features);
  const float pv[7] = {pose.rotation(0), pose.rotation(1), pose.rotation(2), pose.rotation(3),
                       pose.translation(0), pose.translation(1), pose.translation(2)};
  savef("pose", pv, {7});

  // ---- render + backward
  const RenderOutput out = render<float>(map, pose, intr, 4);
  saveimg("color", out.color), saveimg("depth", out.depth), saveimg("query", out.query), saveimg("alpha", out.alpha);
  std::vector<int32_t> sp;
  for (const auto& s : out.splats) sp.insert(sp.end(), {s.source, s.x0, s.x1, s.y0, s.y1});
  savei("splats", sp.data(), {out.splats.size(), 5});
  Image dcol(H, W, 3), ddep(H, W, 1), dq(H, W, ds);
  {
    std::normal_distribution<float> g(0.f, 1.f);
    for (auto& v : dcol.data) v = g(rng);
    for (auto& v : ddep.data) v = g(rng);
    for (auto& v : dq.data) v = g(rng);
  }
  saveimg("up_color", dcol), saveimg("up_depth", ddep), saveimg("up_query", dq);
  RenderUpstream<float> up;
  up.d_color = &dcol, up.d_depth = &ddep, up.d_query = &dq;
  const MapGradients mg = render_backward<float>(map, pose, intr, out, up, 4);
  savem("g_positions", mg.positions), savem("g_rotations", mg.rotations), savem("g_colors", mg.colors);
  savem("g_log_scales", mg.log_scales), savev("g_opacity_logits", mg.opacity_logits);
  savem("g_features", mg.features);

  // ---- decoder
  DictionaryState dict;
  dict.init(K, ds, df);
  dict.atoms = randn(K, df, rng);
  for (int k = 0; k < K; ++k) dict.atoms.row(k) /= dict.atoms.row(k).norm();
  dict.anchor = dict.atoms + randn(K, df, rng, 0.08f);
  dict.proj = randn(ds, df, rng, 0.5f);
  dict.temperature = 2.0f;
  savem("atoms", dict.atoms), savem("anchor", dict.anchor), savem("proj", dict.proj);
  const MatX<float> Q = randn(500, ds, rng);
  AttentionCache<float> cache;
  const MatX<float> rec = reconstruct<float>(Q, dict, &cache);
  const MatX<float> dF = randn(500, df, rng);
  const DictionaryGrads<float> dg = reconstruct_backward<float>(dict, cache, dF);
  savem("Q", Q), savem("rec", rec), savem("attention", cache.attention), savem("dF", dF);
  savem("dg_queries", dg.d_queries), savem("dg_proj", dg.d_proj), savem("dg_atoms", dg.d_atoms);
  MatX<float> tgrad;
  const float pen = trust_region_penalty<float>(dict.atoms, dict.anchor, 0.1f, &tgrad);
  savef("trust", &pen, {1}), savem("trust_grad", tgrad);

  // ---- losses on the rendered images
  Image obs(H, W, 3), odep(H, W, 1);
  {
    std::uniform_real_distribution<float> u(0.f, 1.f);
    for (auto& v : obs.data) v = u(rng);
    for (size_t i = 0; i < odep.data.size(); ++i) odep.data[i] = u(rng) < 0.2f ? 0.f : 1.f + 4.f * u(rng);
  }
  saveimg("obs_rgb", obs), saveimg("obs_depth", odep);
  const RgbLoss<float> rl = rgb_loss<float>(out.color, obs, 0.2f, 0.8f, true);
  const float rv[3] = {rl.value, rl.l1, rl.ssim_loss};
  savef("rgb_loss", rv, {3}), saveimg("rgb_grad", rl.grad);
  const ScalarLoss<float> dl = depth_loss<float>(out.depth, odep, out.alpha, true);
  const float dv[2] = {dl.value, dl.flagged ? 1.f : 0.f};
  savef("depth_loss", dv, {2}), saveimg("depth_grad", dl.grad);
  Image sg;
  const float sv = ssim<float>(out.color, obs, &sg);
  savef("ssim", &sv, {1}), saveimg("ssim_grad", sg);
  const MatX<float> tgt = randn(500, df, rng);
  const FeatureLoss<float> fl = feature_loss<float>(rec, tgt, dict.atoms, dict.anchor, 0.1f, 0.5f, 0.5f, 0.2f, true);
  const float fv[5] = {fl.value, fl.cos_term, fl.l2_term, fl.trust_term, fl.zero_norm_flagged ? 1.f : 0.f};
  savem("feat_target", tgt), savef("feature_loss", fv, {5}), savem("feat_grad", fl.d_reconstructed);
  savem("feat_trust_grad", fl.d_atoms_trust);

  // ---- total_objective over two keyframes (second one posed), with gradients
  std::vector<Keyframe> kfs(2);
  for (int b = 0; b < 2; ++b) {
    Keyframe& kf = kfs[size_t(b)];
    kf.pose = b == 0 ? Pose() : pose;
    kf.rgb = obs;
    kf.depth = odep;
    kf.embeddings.height = H, kf.embeddings.width = W;
    const int nset = 12;
    kf.embeddings.features = randn(nset, df, rng);
    for (int r = 0; r < nset; ++r) kf.embeddings.features.row(r) /= kf.embeddings.features.row(r).norm();
    std::uniform_int_distribution<int> pick(-1, nset - 1);
    kf.embeddings.assignment.resize(size_t(H) * W);
    for (auto& a : kf.embeddings.assignment) a = pick(rng);
    savem("kf" + std::to_string(b) + "_features", kf.embeddings.features);
    savei("kf" + std::to_string(b) + "_assignment", kf.embeddings.assignment.data(), {size_t(H), size_t(W)});
  }
  Config cfg;
  cfg.lambda_i2 = 0.8f;
  ObjectiveGrads<float> og;
  const LossBreakdown<float> lb = total_objective<float>(map, dict, {&kfs[0], &kfs[1]}, intr, cfg, &og, {});
  const float lv[7] = {lb.l_rgb, lb.l_ssim, lb.l_depth, lb.l_cos, lb.l_l2, lb.l_trust, lb.total};
  savef("obj_loss", lv, {7});
  savem("og_positions", og.map.positions), savem("og_rotations", og.map.rotations), savem("og_colors", og.map.colors);
  savem("og_log_scales", og.map.log_scales), savev("og_opacity_logits", og.map.opacity_logits);
  savem("og_features", og.map.features), savem("og_proj", og.d_proj), savem("og_atoms", og.d_atoms);

  // ---- the exception contract (render.cpp:136,256-260; dictionary.cpp:28-33,59-64,87-88;
  // losses.cpp:203-204,229-230,261-262; objective.cpp:72)
  Intrinsics bad = intr;
  bad.fx = 0;
  DictionaryState other = dict;
  other.atoms(0, 0) += 1.f;
  Pose moved = pose;
  moved.translation(0) += 0.5f;
  const Image small(4, 4, 3);
  std::vector<int32_t> errs = {
      throws([&] { render<float>(map, pose, bad, 1); }, 1),
      throws([&] { render_backward<float>(map, moved, intr, out, up, 1); }, 2),
      throws([&] { reconstruct<float>(randn(3, ds + 1, rng), dict, nullptr); }, 1),
      throws([&] { reconstruct_backward<float>(other, cache, dF); }, 2),
      throws([&] { trust_region_penalty<float>(dict.atoms, dict.proj, 0.1f, nullptr); }, 1),
      throws([&] { rgb_loss<float>(out.color, small, 0.2f, 0.8f, true); }, 1),
      throws([&] { depth_loss<float>(out.depth, small, out.alpha, true); }, 1),
      throws([&] { feature_loss<float>(rec, dF.topRows(10), dict.atoms, dict.anchor, 0.1f, 0.5f, 0.5f, 0.2f, true); }, 1),
      throws([&] { total_objective<float>(map, dict, {}, intr, cfg, nullptr, {}); }, 1),
  };
  savei("errors", errs.data(), {errs.size()});
  std::printf("dropin_check: wrote %s\n", g_dir.c_str());
  return 0;
}
