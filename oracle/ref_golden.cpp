// TEST INFRASTRUCTURE ONLY (oracle pin). Compiled against the reference's own
// Eigen-free headers where they lie under /root/reference (never copied):
//   proj/include/vmfa/rng.hpp      (splitmix64, hash_combine, hash3, Rng, uniform_component)
//   proj/include/vmfa/numerics.hpp (kLog2Pi, log_sum_exp)
// Output: JSON golden vectors, committed as tests/golden/rng_ref.json by
// oracle/make_ref_golden.sh. The rest of the reference needs Eigen3 (absent
// here), so it is treated as unbuildable.
#include <cmath>
#include <cstdio>
#include <vector>
#include "vmfa/rng.hpp"
#include "vmfa/numerics.hpp"

static void list_u64(const char* name, const std::vector<unsigned long long>& v, bool last = false) {
  std::printf("  \"%s\": [", name);
  for (size_t i = 0; i < v.size(); ++i) std::printf("%s\"%llu\"", i ? ", " : "", v[i]);
  std::printf("]%s\n", last ? "" : ",");
}
static void list_f64(const char* name, const std::vector<double>& v, bool last = false) {
  std::printf("  \"%s\": [", name);
  for (size_t i = 0; i < v.size(); ++i) {
    if (std::isfinite(v[i])) std::printf("%s%.17g", i ? ", " : "", v[i]);
    else std::printf("%s\"%s\"", i ? ", " : "", std::isnan(v[i]) ? "nan" : (v[i] > 0 ? "inf" : "-inf"));
  }
  std::printf("]%s\n", last ? "" : ",");
}

int main() {
  std::printf("{\n");
  // uniform_component over the BASELINE configs' C and N-1, iterations 0,1,7 and a few seeds
  const int Cs[] = {100, 1000, 4000, 10000, 50000};
  const unsigned long long Ns[] = {19999ULL, 199999ULL, 999999ULL, 9999999ULL, 49999999ULL};
  std::printf("  \"uniform_component\": [\n");
  bool first = true;
  for (int ci = 0; ci < 5; ++ci)
    for (unsigned long long seed : {0ULL, 1ULL, 12345ULL})
      for (unsigned long long it : {0ULL, 1ULL, 7ULL, 1000ULL}) {
        unsigned long long ns[] = {0ULL, 1ULL, 2ULL, 12345ULL, Ns[ci]};
        for (unsigned long long n : ns) {
          int r = vmfa::uniform_component(seed, it, n, Cs[ci]);
          std::printf("%s    [\"%llu\", \"%llu\", \"%llu\", %d, %d]", first ? "" : ",\n", seed, it, n, Cs[ci], r);
          first = false;
        }
      }
  std::printf("\n  ],\n");
  std::vector<unsigned long long> h;
  for (unsigned long long a : {0ULL, 1ULL, 2ULL, 0xdeadbeefULL})
    for (unsigned long long b : {0ULL, 3ULL, 0x1217f01dULL})
      h.push_back(vmfa::hash_combine(a, b));
  list_u64("hash_combine_a0_1_2_deadbeef_x_b0_3_1217f01d", h);
  h.clear();
  h.push_back(vmfa::hash3(0, 0, 0));
  h.push_back(vmfa::hash3(1, 2, 3));
  h.push_back(vmfa::hash3(7, 11, 13));
  list_u64("hash3_000_123_71113", h);
  // Rng streams used by the trainer (trainer.cpp:36, :107 salts)
  for (unsigned long long salt : {0x1217f01dULL, 0x7a57a7e5ULL}) {
    vmfa::Rng r(vmfa::hash_combine(0, salt));
    std::vector<unsigned long long> v;
    for (int i = 0; i < 16; ++i) v.push_back(r.next_u64());
    char name[64];
    std::snprintf(name, sizeof name, "rng_next_u64_seed0_salt_%llx", salt);
    list_u64(name, v);
  }
  {
    vmfa::Rng r(42);
    std::vector<double> v;
    for (int i = 0; i < 9; ++i) v.push_back(r.gaussian());
    v.push_back(r.uniform());
    for (int i = 0; i < 6; ++i) v.push_back(r.gaussian());
    list_f64("rng42_gaussian9_uniform1_gaussian6", v);
  }
  {
    vmfa::Rng r(7);
    std::vector<unsigned long long> v;
    for (long long b : {1000LL, 1LL, 2LL, 3LL, 1000000007LL, 50000000LL, 100LL})
      v.push_back((unsigned long long)r.uniform_int(b));
    list_u64("rng7_uniform_int_1000_1_2_3_1e9p7_5e7_100", v);
  }
  {
    std::vector<double> a = {-1.0, -2.0, -3.0};
    std::vector<double> b = {-1e3, -1e3 - 1e-9, -745.0, -2000.0};
    std::vector<double> c = {vmfa::kNegInf, vmfa::kNegInf};
    std::vector<double> d = {vmfa::kNegInf, 0.5};
    list_f64("log_sum_exp_abcd", {vmfa::log_sum_exp(a), vmfa::log_sum_exp(b), vmfa::log_sum_exp(c), vmfa::log_sum_exp(d)});
  }
  std::printf("  \"kLog2Pi\": %.17g\n", vmfa::kLog2Pi);
  std::printf("}\n");
  return 0;
}
