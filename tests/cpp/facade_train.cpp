// Drop-in usage of the C++ mirror (include/vmfa_b200.hpp): config-1 data,
// the reference's initialisation, then train_vmfa's loop with fixed counts.
// Prints one line per iteration: warmup F F_estep joints.
#include <cstdio>
#include <string>
#include <vector>

#include "vmfa_b200.hpp"

int main(int argc, char** argv) {
  const int64_t N = argc > 1 ? std::atoll(argv[1]) : 20000;
  vmfa_synth_spec sp{};
  sp.kind = 0; sp.n_total = N; sp.D = 64; sp.C_true = 100; sp.H_true = 4; sp.dirichlet = 0;
  sp.mu_std = 4.0; sp.lam_std = 0.5; sp.psi_lo = 0.1; sp.psi_hi = 1.0; sp.data_seed = 0;
  vmfa_b200::Dataset data;
  data.N = N;
  data.D = 64;
  data.rows.resize(size_t(N) * 64);
  vmfa_b200::check(vmfa_gen_synthetic(&sp, 0, N, data.rows.data(), nullptr, 0));
  const int C = 100, H = 4, Cp = 3, G = 5;
  vmfa_b200::MfaParams p;
  p.C = C, p.D = 64, p.H = H;
  p.pi.resize(C); p.mu.resize(C * 64); p.Lambda.resize(C * 64 * H); p.dnoise.resize(C * 64);
  vmfa_b200::VarState st;
  st.C = C, st.Cprime = Cp, st.G = G;
  st.K.resize(N * Cp); st.g.resize(C * G); st.g_count.resize(C);
  std::vector<double> floor(64);
  std::vector<int64_t> seeds(C);
  vmfa_b200::check(vmfa_host_initialize(data.rows.data(), N, 64, C, H, Cp, G, 0, 0.1, 1, floor.data(),
                                        p.pi.data(), p.mu.data(), p.Lambda.data(), p.dnoise.data(),
                                        st.K.data(), st.g.data(), st.g_count.data(), seeds.data()));
  try {
    vmfa_b200::Session s(data, C, H, Cp, G);
    s.set_floor(floor);
    s.upload(p);
    s.upload(st);
    if (argc > 2 && std::string(argv[2]) == "converge") {  // train_vmfa's convergence-gated loop
      vmfa_b200::TrainConfig cfg;
      cfg.epsilon = 1e-4;
      cfg.max_iters = 60;
      cfg.eval_nll_every = 5;
      cfg.warmup_epsilon = 1e-3;
      cfg.halt_on_max_iters = false;
      const auto rep = vmfa_b200::train_vmfa(s, cfg);
      for (const auto& r : rep.iterations)
        std::printf("%d %.10f %.10f %llu\n", r.warmup ? 1 : 0, r.F, r.nll_train,
                    static_cast<unsigned long long>(r.joint_evals));
      std::printf("final %d %d %.10f\n", rep.converged ? 1 : 0, rep.main_iterations, rep.nll_train);
    } else {
      for (const auto& r : vmfa_b200::train_fixed(s, 0, 2, 20))
        std::printf("%d %.10f %.10f %llu\n", r.warmup ? 1 : 0, r.F, r.F_estep,
                    static_cast<unsigned long long>(r.joint_evals));
    }
  } catch (const vmfa_b200::DeviceError& e) {
    std::fprintf(stderr, "device error: %s\n", e.what());
    return 3;
  }
  return 0;
}
