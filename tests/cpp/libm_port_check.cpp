// Host build of the generated libm restatements (csrc/libm_port.cuh) against
// the libm the reference links: bitwise on random inputs drawn from the
// ranges the Dubins steering feeds them (angles, differences of angles,
// direction components, cosines) plus random bit patterns and specials.
//   libm_port_check FUNC COUNT SEED  -> "FUNC checked N mismatches M" (+ the first few)
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>
#include <atomic>

#include "libm_port.cuh"

using namespace lmport;

static bool same(double a, double b) {
  if (a != a && b != b) return true;
  return lm_b(a) == lm_b(b);
}

static double draw(std::mt19937_64& g) {
  const unsigned k = g() % 8;
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  switch (k) {
    case 0: return u(g) * 3.5;                    // an angle
    case 1: return u(g) * 7.0;                    // a sum / difference of angles
    case 2: return u(g) * 64.0;                   // scaled distances
    case 3: return u(g) * 1e-3;                   // small
    case 4: {                                     // a random exponent
      const int e = static_cast<int>(g() % 80) - 60;
      return std::ldexp(u(g), e);
    }
    case 5: {                                     // near a multiple of pi/4
      const double m = static_cast<double>(static_cast<int>(g() % 64) - 32) * 0.78539816339744830962;
      return m + std::ldexp(u(g), -static_cast<int>(g() % 50));
    }
    case 6: return u(g) * 1e6;
    default: {                                     // raw bits (finite or not)
      const u64 b = g();
      return lm_f(b);
    }
  }
}

int main(int argc, char** argv) {
  const std::string fn = argv[1];
  const long long count = std::atoll(argv[2]);
  const unsigned long long seed = std::strtoull(argv[3], nullptr, 10);
  const unsigned threads = std::max(1u, std::thread::hardware_concurrency());
  std::atomic<long long> bad{0};
  std::vector<std::thread> th;
  std::vector<std::string> first(threads);
  for (unsigned t = 0; t < threads; ++t) {
    th.emplace_back([&, t] {
      std::mt19937_64 g(seed * 1000003ull + t);
      const long long n = count / threads + (t < count % threads ? 1 : 0);
      for (long long i = 0; i < n; ++i) {
        double a = draw(g), b = draw(g), want, got;
        if ((fn == "sin" || fn == "cos") && !(std::fabs(a) < 105414350.0)) continue;  // (__branred's domain)
        if (fn == "sin") {
          want = std::sin(a), got = lm_sin(a);
        } else if (fn == "cos") {
          want = std::cos(a), got = lm_cos(a);
        } else if (fn == "hypot") {
          want = std::hypot(a, b), got = lm_hypot(a, b);
        } else if (fn == "atan2") {
          want = std::atan2(a, b), got = lm_atan2(a, b);
        } else {  // acos: mostly inside [-1, 1]
          if (g() % 4) a = std::fmod(a, 1.0);
          if (g() % 8 == 0) a = (g() % 2 ? 1.0 : -1.0) - std::ldexp(static_cast<double>(g() % 1000), -52) * (a < 0 ? -1 : 1);
          want = std::acos(a), got = lm_acos(a);
        }
        if (!same(want, got)) {
          if (bad.fetch_add(1) < 8) {
            char buf[256];
            std::snprintf(buf, sizeof buf, "  %s(%a, %a) libm %a port %a\n", fn.c_str(), a, b, want, got);
            first[t] += buf;
          }
        }
      }
    });
  }
  for (auto& x : th) x.join();
  std::printf("%s checked %lld mismatches %lld\n", fn.c_str(), count, bad.load());
  for (auto& s : first) std::fputs(s.c_str(), stdout);
  return bad.load() ? 1 : 0;
}
