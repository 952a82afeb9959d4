// Test helper: libstdc++'s std::mt19937_64 and the distributions the reference pipeline draws
// with (proj/src/pipeline.cpp:19-73, 106-121, 136-153; stream_kmeans.cpp:58-71), exposed to the
// Python tests so a test-side composition of the pipeline can consume the generator in the
// reference's order. Test infrastructure only; compiled at test time.
#include <cstdint>
#include <random>
#include <utility>
#include <vector>

extern "C" {
void* rng_new(uint64_t seed) { return new std::mt19937_64(seed); }
void rng_free(void* h) { delete static_cast<std::mt19937_64*>(h); }
double rng_uniform01(void* h) {
  std::uniform_real_distribution<double> u(0.0, 1.0);
  return u(*static_cast<std::mt19937_64*>(h));
}
// one fresh std::normal_distribution<float>(0, stddev), n draws (seed_gaussians, PipelineState ctor)
void rng_normal(void* h, float stddev, int64_t n, float* out) {
  std::normal_distribution<float> g(0.0f, stddev);
  for (int64_t i = 0; i < n; ++i) out[i] = g(*static_cast<std::mt19937_64*>(h));
}
// sample_history (pipeline.cpp:19-37) over indices 0..n-1
int64_t rng_sample_history(void* h, int64_t n, int32_t count, int64_t* out) {
  auto& rng = *static_cast<std::mt19937_64*>(h);
  if (n == 0 || count <= 0) return 0;
  if (n <= count) {
    for (int64_t i = 0; i < n; ++i) out[i] = i;
    return n;
  }
  std::vector<size_t> idx((size_t)n);
  for (size_t i = 0; i < (size_t)n; ++i) idx[i] = i;
  for (int k = 0; k < count; ++k) {
    std::uniform_int_distribution<size_t> pick(size_t(k), size_t(n) - 1);
    std::swap(idx[size_t(k)], idx[pick(rng)]);
    out[k] = (int64_t)idx[size_t(k)];
  }
  return count;
}
}
