// Compile-and-run check of the C++ facade (include/hpsim_b200.hpp): the
// reference's hpsim::Cluster usage pattern, and ConfigError on the reference's
// invalid configurations (host-side validation; no GPU needed).
#include <cstdio>
#include <cstring>
#include <string>

#include "hpsim_b200.hpp"

using namespace hpsim_b200;

static ModelSpec tiny() {
  ModelSpec s;
  s.conv_layers = {{3, 32, 5, 1, 2, true}, {32, 32, 4, 2, 1, true}, {32, 64, 4, 2, 1, true}};
  s.fc_layers = {{4096, 256, true}, {256, 10, false}};
  s.input_shape = {3, 32, 32};
  s.num_classes = 10;
  return s;
}

int main(int argc, char** argv) {
  int fails = 0;
  auto expect_config_error = [&](const ModelSpec& s, const ClusterConfig& c, const char* needle) {
    try {
      Cluster cl(s, c);
      std::printf("FAIL: no error for %s\n", needle);
      ++fails;
    } catch (const ConfigError& e) {
      if (std::string(e.what()).find(needle) == std::string::npos) {
        std::printf("FAIL: message '%s' lacks '%s'\n", e.what(), needle);
        ++fails;
      }
    }
  };
  ClusterConfig c;
  c.workers = 3;
  c.scheme = Scheme::C;
  expect_config_error(tiny(), c, "is not divisible by 3");
  c = ClusterConfig{};
  c.workers = 2;
  c.scheme = Scheme::A;
  c.variable_batch = true;
  expect_config_error(tiny(), c, "scheme A has a single fc pass");
  ModelSpec bad = tiny();
  bad.fc_layers[0].in_dim = 100;
  expect_config_error(bad, ClusterConfig{}, "model.fc_layers[0].in_dim: expected 4096");
  if (argc > 1 && std::strcmp(argv[1], "gpu") == 0) {  // full step on a B200
    ClusterConfig g;
    g.workers = 2;
    g.per_worker_batch = 8;
    g.scheme = Scheme::C;
    Cluster cl(tiny(), g);
    std::vector<float> x(8 * 3 * 32 * 32, 0.5f), t(8 * 10, 0.f);
    for (int i = 0; i < 8; ++i) t[i * 10 + i % 10] = 1.f;
    auto r = cl.run_step(std::vector<const float*>{x.data(), x.data()}, std::vector<const float*>{t.data(), t.data()},
                         HyperParams{}, 0.01);
    if (r.trace.pass_count() != 2 + 2 * 2) ++fails;
    std::printf("loss %.6f passes %d\n", r.metrics.loss, r.trace.pass_count());
    // the reference's Tensor-based signature (span under C++20, vector otherwise)
    std::vector<Tensor> xb{Tensor({8, 3, 32, 32}, x), Tensor({8, 3, 32, 32}, x)};
    std::vector<Tensor> tb{Tensor({8, 10}, t), Tensor({8, 10}, t)};
#if __cplusplus >= 202002L
    r = cl.run_step(std::span<const Tensor>(xb), std::span<const Tensor>(tb), HyperParams{}, 0.01);
#else
    r = cl.run_step(xb, tb, HyperParams{}, 0.01);
#endif
    if (r.trace.pass_count() != 6) ++fails;
    try {
      std::vector<Tensor> wrong{Tensor({8, 3, 32, 31}), Tensor({8, 3, 32, 31})};
      cl.run_step(wrong, tb, HyperParams{}, 0.01);
      std::printf("FAIL: no DimensionError for a wrong batch shape\n");
      ++fails;
    } catch (const DimensionError&) {
    }
    // worker(i) snapshot and gathered_model(): conv = worker 0's replica, fc =
    // the shards pasted back by column (cluster.cpp:417-437)
    const WorkerState w0 = cl.worker(0), w1 = cl.worker(1);
    const Model m = cl.gathered_model();
    for (std::size_t l = 0; l < m.conv.size(); ++l)
      for (std::int64_t i = 0; i < m.conv[l].kernels.size(); ++i)
        if (m.conv[l].kernels.data()[i] != w0.conv_params[l].kernels.data()[i] ||
            w1.conv_params[l].kernels.data()[i] != w0.conv_params[l].kernels.data()[i]) {
          std::printf("FAIL: conv layer %zu differs from worker 0\n", l);
          ++fails;
          break;
        }
    for (std::size_t l = 0; l < m.fc.size(); ++l) {
      const std::int64_t in = m.fc[l].weight.dim(0), out = m.fc[l].weight.dim(1);
      std::int64_t col = 0;
      for (const WorkerState* w : {&w0, &w1}) {
        const Tensor& sh = w->fc_shard[l].weight;
        for (std::int64_t r = 0; r < in; ++r)
          for (std::int64_t j = 0; j < sh.dim(1); ++j)
            if (sh.data()[r * sh.dim(1) + j] != m.fc[l].weight.data()[r * out + col + j]) {
              std::printf("FAIL: fc layer %zu shard column mismatch\n", l);
              ++fails;
              r = in;
              break;
            }
        col += sh.dim(1);
      }
      if (col != out) ++fails;
    }
    if (w0.bytes.sent[0] + w0.bytes.sent[1] + w0.bytes.sent[2] + w0.bytes.sent[3] <= 0) ++fails;
  }
  std::printf(fails ? "FAILED\n" : "facade ok\n");
  return fails ? 1 : 0;
}
