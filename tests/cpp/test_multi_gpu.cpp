// The C++ drop-in's multi-GPU path: with R1_NUM_GPUS=N, rank1::hoscf /
// rank1::ihoscf split the DenseTensor into slabs over N GPUs (one thread per
// GPU, NCCL group exchange per sweep).  Prints lambda, iterations and the
// factors bit-exactly so two runs (default vs R1_NUM_GPUS) can be compared
// (tests/test_cpp_dropin.py).
#include <cstdio>
#include <vector>

#include "rank1/solvers.hpp"
#include "rank1/tensor.hpp"

int main() {
    const std::vector<std::size_t> dims = {30, 20, 25};
    rank1::DenseTensor a(dims);
    for (std::size_t i = 0; i < a.size(); ++i) a[i] = static_cast<double>((i * 7919) % 1009) / 1009.0 - 0.5;
    for (const char* alg : {"hoscf", "ihoscf"}) {
        rank1::SolveOptions o;
        o.tol = 1e-10;
        o.seed = 3;
        const rank1::SolveReport r = rank1::solve(alg, a, o);
        std::printf("%s %d %d %.17g\n", alg, r.iterations, r.converged ? 1 : 0, r.result.lambda);
        for (const auto& u : r.result.factors)
            for (double v : u) std::printf("%a\n", v);
    }
    return 0;
}
