// Host narrowing throughput in isolation (csrc/narrow.cpp): one parallel pass
// over 8M x 256 int32 rows (like torch's copy) vs the host pipeline's 64-MB
// chunks, with N threads.  g++ -O3 -std=c++17 -pthread tools/narrow_bench.cpp \
//   paper_1905_13746_b200/csrc/narrow.cpp -o tools/narrow_bench
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

namespace gnb {
bool narrow_rows_block(int bits, const int32_t* s, int32_t F, int64_t ldx, uint8_t* d,
                       int64_t dpitch, int64_t r0, int64_t r1);
}

int main(int argc, char** argv) {
  const int64_t n = 8000000;
  const int F = 256;
  const int T = argc > 1 ? atoi(argv[1]) : (int)std::thread::hardware_concurrency();
  std::vector<int32_t> x(size_t(n) * F);
  for (size_t i = 0; i < x.size(); ++i) x[i] = int32_t(i * 2654435761u >> 28);
  std::vector<uint8_t> d(size_t(n) * F / 2);
  auto pass = [&](int64_t chunk_rows, int block) {
    auto t0 = std::chrono::steady_clock::now();
    for (int64_t c0 = 0; c0 < n; c0 += chunk_rows) {
      const int64_t cn = std::min(chunk_rows, n - c0);
      std::vector<std::thread> th;
      for (int w = 0; w < T; ++w)
        th.emplace_back([&, w] {
          const int64_t lo = c0 + cn * w / T, hi = c0 + cn * (w + 1) / T;
          for (int64_t r = lo; r < hi; r += block)
            gnb::narrow_rows_block(4, x.data(), F, F, d.data(), F / 2, r, std::min<int64_t>(r + block, hi));
        });
      for (auto& t : th) t.join();
    }
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return n * F * 4.0 / s / 1e9;
  };
  pass(n, 64);
  printf("{\"threads\": %d, \"one_pass_gbs\": %.1f, \"chunk64mb_gbs\": %.1f, \"chunk256mb_gbs\": %.1f, "
         "\"one_pass_block1024_gbs\": %.1f}\n",
         T, pass(n, 64), pass(65536, 64), pass(262144, 64), pass(n, 1024));
  return 0;
}
