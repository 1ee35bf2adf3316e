// Golden vectors from the C++ standard library for the two pieces of the
// reference's data kit that are defined by it: std::to_chars(double)
// shortest formatting (datakit.hpp:225-230, used by every CSV / report
// writer) and std::mt19937_64 + rng::uniform_real (rng.hpp:14-21, the
// synthesize noise stream).  Built and run by make_std_vectors.py.
#include <charconv>
#include <cstdint>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <random>
#include <vector>

int main() {
  std::vector<double> vals = {0.0, -0.0, 1.0, -1.0, 0.5, 0.1, 0.2, 0.3, 1.5, 2.0, 10.0, 100.0,
                              123456.0, 1e15, 1e16, 1e17, 1e21, 1e22, 1e23, 1.5e300, 5e-324,
                              2.2250738585072014e-308, 1e-5, 1e-4, 1e-3, 0.001234, 123.456,
                              1.0 / 3.0, 2.0 / 3.0, 123456789012345680.0, 9007199254740993.0,
                              4.35e-7, 3.14159265358979, 5.375, 84.0, 65536.0, 1048576.0,
                              12345678.9, 1e7, 1.25e7, 0.000123, 436.0, 1.3};
  std::mt19937_64 seeds(12345);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  for (int i = 0; i < 200; ++i) {
    double x = std::ldexp(u(seeds), (int)(seeds() % 200) - 100);
    vals.push_back(x);
  }
  std::printf("{\n  \"to_chars\": [\n");
  for (size_t i = 0; i < vals.size(); ++i) {
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof(buf), vals[i]);
    *r.ptr = 0;
    std::printf("    [\"%a\", \"%s\"]%s\n", vals[i], buf, i + 1 < vals.size() ? "," : "");
  }
  std::printf("  ],\n");
  {
    std::mt19937_64 g;  // default seed 5489
    unsigned long long x = 0;
    for (int i = 0; i < 10000; ++i) x = g();
    std::printf("  \"mt19937_64_default_10000th\": \"%llu\",\n", x);
  }
  std::printf("  \"uniform_real\": {\n");
  const unsigned long long sd[] = {0ull, 42ull, 18446744073709551615ull};
  for (int k = 0; k < 3; ++k) {
    std::mt19937_64 g(sd[k]);
    std::printf("    \"%llu\": [", sd[k]);
    for (int i = 0; i < 64; ++i) {
      const double c = static_cast<double>(g() >> 11) * 0x1.0p-53;
      volatile double span = 0.03 - (-0.03);
      volatile double t = span * c;
      double v = -0.03 + t;
      std::printf("\"%a\"%s", v, i + 1 < 64 ? ", " : "");
    }
    std::printf("]%s\n", k + 1 < 3 ? "," : "");
  }
  std::printf("  }\n}\n");
  return 0;
}
