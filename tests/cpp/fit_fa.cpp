// The fit_fa_per_cluster loop of the reference (kmeans.cpp:195-210) through
// the C++ drop-in (include/vmfa_b200.hpp): one cluster's rows as a single-
// component FA (C = C' = G = 1, every K row = {0}, every responsibility 1):
// accumulate_suffstats with the caller's K and resp, update_params (+
// precompute), truncated_free_energy over the caller's ksets, until
// check_convergence(epsilon) -- exactly the reference's sequence of calls.
// Args: data.mfad params.mfam floor.bin max_iters epsilon out.mfam
// Prints "it F joints" per iteration.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <vector>

#include "vmfa_b200.hpp"

int main(int argc, char** argv) {
  if (argc < 7) return 2;
  using namespace vmfa_b200;
  try {
    const Dataset cell = load_dataset(argv[1]);
    MfaParams fa = load_checkpoint(argv[2]);
    std::vector<double> floor(cell.D);
    FILE* f = std::fopen(argv[3], "rb");
    if (!f || std::fread(floor.data(), sizeof(double), floor.size(), f) != floor.size()) return 2;
    std::fclose(f);
    const int max_iters = std::atoi(argv[4]);
    const double epsilon = std::atof(argv[5]);
    Session s(cell, 1, fa.H, 1, 1);
    s.set_floor(floor);
    s.upload(fa);  // + precompute_all
    const std::vector<int32_t> ksets(cell.N, 0);      // ksets.idx.assign(n, 0)
    const std::vector<double> resp(cell.N, 1.0);      // resp(n, 1.0)
    EvalCounter tally;
    double prev = std::numeric_limits<double>::quiet_NaN();
    for (int it = 0; it < max_iters; ++it) {
      const SuffStats stats = accumulate_suffstats(s, ksets, resp);
      fa = update_params(s, stats);  // + precompute_all on the device
      const double F = truncated_free_energy(s, ksets, tally);
      std::printf("%d %.12e %llu\n", it, F, static_cast<unsigned long long>(tally.joints));
      if (std::isfinite(prev) && check_convergence(prev, F, epsilon)) break;
      prev = F;
    }
    save_checkpoint(fa, argv[6]);
  } catch (const DeviceError& e) {
    std::fprintf(stderr, "device error: %s\n", e.what());
    return 3;
  }
  return 0;
}
