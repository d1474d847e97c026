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
    auto r = cl.run_step({x.data(), x.data()}, {t.data(), t.data()}, HyperParams{}, 0.01);
    if (r.trace.pass_count() != 2 + 2 * 2) ++fails;
    std::printf("loss %.6f passes %d\n", r.metrics.loss, r.trace.pass_count());
  }
  std::printf(fails ? "FAILED\n" : "facade ok\n");
  return fails ? 1 : 0;
}
