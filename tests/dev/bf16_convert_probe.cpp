// Dev: host f32 -> bf16 (RN-even) conversion throughput of one AlexNet batch (19.3M floats), T threads.
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
#include <cstdlib>
static void conv(const float* __restrict__ s, uint16_t* __restrict__ d, long n) {
  for (long i = 0; i < n; ++i) {
    uint32_t u;
    std::memcpy(&u, s + i, 4);
    u += 0x7fffu + ((u >> 16) & 1u);
    d[i] = static_cast<uint16_t>(u >> 16);
  }
}
int main(int argc, char** argv) {
  const long n = 128L * 3 * 224 * 224;
  int T = argc > 1 ? atoi(argv[1]) : 8;
  std::vector<float> s(n);
  for (long i = 0; i < n; ++i) s[i] = (i % 1000) * 0.001f;
  std::vector<uint16_t> d(n);
  for (int rep = 0; rep < 5; ++rep) {
    auto a = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t) {
      long b = n * t / T, e = n * (t + 1) / T;
      th.emplace_back([&, b, e] { conv(s.data() + b, d.data() + b, e - b); });
    }
    for (auto& x : th) x.join();
    auto z = std::chrono::steady_clock::now();
    printf("T=%d %.3f ms\n", T, std::chrono::duration<double, std::milli>(z - a).count());
  }
}
