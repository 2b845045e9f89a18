// The reference's experiment driver, cmd_run (experiment.cpp:79-199, compiled in place
// into oracle/_ref), writing its CSV artifacts.  Built twice by tests/cpp/Makefile:
//   cmd_run_ref  -- the reference as is;
//   cmd_run_gpu  -- with PKRR_GPU_INTERPOSE: this executable defines pkrr::grid_search,
//                   pkrr::standardize and pkrr::auto_sigma_grid over the GPU adapter
//                   (include/pkrr_gpu.hpp), which ELF symbol interposition substitutes
//                   for the library's own definitions inside cmd_run -- the drop-in at
//                   the seam INTEGRATION.md describes, without editing the reference.
// tests/test_gpu_adapter.py compares the two runs' artifacts.
#include <cstdio>
#include <string>

#include "pkrr/experiment.hpp"
#include "pkrr_gpu.hpp"

#ifdef PKRR_GPU_INTERPOSE
namespace pkrr {
GridResult grid_search(StrategyKind kind, const Dataset& train, const Dataset& test, std::size_t p,
                       std::span<const double> lambdas, std::span<const double> sigmas, std::uint64_t seed,
                       const GridOptions& options) {
  return gpu::grid_search(kind, train, test, p, lambdas, sigmas, seed, options);
}
StandardizeResult standardize(const Dataset& train, const Dataset& test) { return gpu::standardize(train, test); }
std::vector<double> auto_sigma_grid(const Dataset& train, std::uint64_t seed) {
  return gpu::auto_sigma_grid(train, seed);
}
}  // namespace pkrr
#endif

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s <out_dir>\n", argv[0]);
    return 2;
  }
  pkrr::ExperimentConfig cfg;
  cfg.use_synthetic = true;
  cfg.synth.n = 4000;
  cfg.synth.d = 8;
  cfg.synth.c = 4;
  cfg.synth.noise = 0.1;
  cfg.strategies = {pkrr::StrategyKind::kk2, pkrr::StrategyKind::bk2, pkrr::StrategyKind::dc};
  cfg.p = 4;
  cfg.lambda_grid = {1e-4, 1e-2};  // sigma grid: auto_sigma_grid (interposed in the GPU build)
  cfg.seed = 7;
  cfg.workers = 1;
  cfg.out_dir = argv[1];
  pkrr::cmd_run(cfg);
  return 0;
}
